# pinned-result API path: its GPU test, then the bench (cfg4) e2e legs
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-api}
timeout -s ABRT 900 python -X faulthandler -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${TAG}.log
timeout 900 python bench.py --no-cpu-baseline --no-batch > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_${TAG}.err
python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}.json')); print('ms', d['ms_per_step'], 'parity', d['parity'], 'e2e', d['e2e']['ms_per_matrix'], 'api', d['e2e_api']['ms_per_matrix'])"
