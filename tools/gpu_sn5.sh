cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-sn5}
timeout -s ABRT 600 python -X faulthandler -m pytest tests/test_gpu_sn.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_sn_${TAG}.log 2>&1
echo "pytest sn rc=$?"; tail -3 gpurun_out/pytest_sn_${TAG}.log
SN_TRACE_DUMP=gpurun_out/trace_g400_${TAG}.npz timeout 600 python tools/sn_probe.py g400 --engines sn --reps 3 --stamps --no-parity > gpurun_out/probe_${TAG}.jsonl 2> gpurun_out/probe_${TAG}.err; echo "probe rc=$?"
timeout 600 python tools/sn_probe.py cfg4 --engines sn --reps 3 --stamps >> gpurun_out/probe_${TAG}.jsonl 2>> gpurun_out/probe_${TAG}.err; echo "probe rc=$?"
tail -3 gpurun_out/probe_${TAG}.err
cut -c1-400 gpurun_out/probe_${TAG}.jsonl
