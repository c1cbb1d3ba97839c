cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-sn16}
timeout -s ABRT 600 python -X faulthandler -m pytest tests/test_gpu_sn.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_sn_${TAG}.log 2>&1
echo "pytest sn rc=$?"; tail -3 gpurun_out/pytest_sn_${TAG}.log
for A in 0 2 1; do
SN_ASSIGN=$A timeout 900 python tools/sn_probe.py g400 cfg4 --engines sn --reps 3 --stamps --no-parity > gpurun_out/probe_${TAG}_a$A.jsonl 2> gpurun_out/probe_${TAG}_a$A.err; echo "probe assign=$A rc=$?"
cut -c1-150 gpurun_out/probe_${TAG}_a$A.jsonl
done
