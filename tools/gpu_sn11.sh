cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-sn11}
timeout -s ABRT 600 python -X faulthandler -m pytest tests/test_gpu_sn.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_sn_${TAG}.log 2>&1
echo "pytest sn rc=$?"; tail -3 gpurun_out/pytest_sn_${TAG}.log
for A in 0 1; do
SN_ASSIGN=$A SN_TRACE_DUMP=gpurun_out/trace_g400_${TAG}_a$A.npz timeout 600 python tools/sn_probe.py g400 --engines sn --reps 3 --stamps --no-parity > gpurun_out/probe_${TAG}_a$A.jsonl 2> gpurun_out/probe_${TAG}_a$A.err; echo "probe g400 assign=$A rc=$?"
SN_ASSIGN=$A timeout 600 python tools/sn_probe.py cfg4 --engines sn --reps 3 --no-parity >> gpurun_out/probe_${TAG}_a$A.jsonl 2>> gpurun_out/probe_${TAG}_a$A.err; echo "probe cfg4 assign=$A rc=$?"
cut -c1-200 gpurun_out/probe_${TAG}_a$A.jsonl
done
