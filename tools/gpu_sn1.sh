cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout -s ABRT 600 python -X faulthandler -m pytest tests/test_gpu_sn.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_sn.log 2>&1
echo "pytest sn rc=$?"; tail -3 gpurun_out/pytest_sn.log
timeout 600 python tools/sn_probe.py g200 g400 --engines sn --reps 3 --stamps > gpurun_out/probe3.jsonl 2> gpurun_out/probe3.err; echo "probe rc=$?"
cat gpurun_out/probe3.jsonl; tail -5 gpurun_out/probe3.err
timeout 900 python tools/sn_probe.py cfg4 --engines sn --reps 2 --stamps --no-parity > gpurun_out/probe_cfg4b.jsonl 2> gpurun_out/probe_cfg4b.err; echo "probe cfg4 rc=$?"
cat gpurun_out/probe_cfg4b.jsonl; tail -5 gpurun_out/probe_cfg4b.err
