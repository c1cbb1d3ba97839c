# cfg4 critical path: trace on the GPU, analysis on the box's host (the trace is too big to bring back)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-c4}
SN_TRACE_DUMP=/tmp/trace_cfg4_${TAG}.npz timeout 900 python tools/sn_probe.py cfg4 --engines sn --reps 2 --stamps --no-parity > gpurun_out/probe_cfg4_${TAG}.jsonl 2> gpurun_out/probe_cfg4_${TAG}.err; echo "probe rc=$?"
timeout 1200 python tools/sn_critpath.py cfg4 /tmp/trace_cfg4_${TAG}.npz > gpurun_out/crit_cfg4_${TAG}.txt 2>&1; echo "crit rc=$?"
cat gpurun_out/crit_cfg4_${TAG}.txt
timeout 600 python tools/sn_occupancy.py /tmp/trace_cfg4_${TAG}.npz > gpurun_out/occ_cfg4_${TAG}.txt 2>&1; echo "occ rc=$?"
cat gpurun_out/occ_cfg4_${TAG}.txt
