# supernodal dataflow engine: GPU parity tests, then g400 / cfg4 timing + per-task trace
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-sn3}
timeout -s ABRT 600 python -X faulthandler -m pytest tests/test_gpu_sn.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_sn_${TAG}.log 2>&1
echo "pytest sn rc=$?"; tail -15 gpurun_out/pytest_sn_${TAG}.log
timeout 900 python tools/sn_probe.py g400 cfg4 --engines sn --reps 3 --stamps > gpurun_out/probe_${TAG}.jsonl 2> gpurun_out/probe_${TAG}.err; echo "probe rc=$?"
tail -5 gpurun_out/probe_${TAG}.err
cut -c1-600 gpurun_out/probe_${TAG}.jsonl
