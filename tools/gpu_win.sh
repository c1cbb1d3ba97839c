# window-walk experiment: supernodal GPU tests, then same-process A/B of GLU_SN_WINDOW
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-win}
timeout -s ABRT 900 python -X faulthandler -m pytest tests/test_gpu_sn.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_sn_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_sn_${TAG}.log
timeout 900 python tools/sn_ab.py ${CFGS:-g400 cfg4} --var ${VAR:-GLU_SN_WINDOW} --vals ${VALS:-0,1} --reps ${REPS:-6} > gpurun_out/ab_${TAG}.jsonl 2> gpurun_out/ab_${TAG}.err
echo "ab rc=$?"; cat gpurun_out/ab_${TAG}.jsonl; tail -3 gpurun_out/ab_${TAG}.err
