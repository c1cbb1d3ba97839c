cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout -s ABRT 600 python -X faulthandler -m pytest tests/test_gpu_sn.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_sn.log 2>&1
echo "pytest sn rc=$?"; tail -2 gpurun_out/pytest_sn.log
timeout 900 python tools/sn_probe.py g400 cfg4 --engines sn --reps 2 --stamps --no-parity > gpurun_out/probe6.jsonl 2> gpurun_out/probe6.err; echo "probe rc=$?"
tail -5 gpurun_out/probe6.err
