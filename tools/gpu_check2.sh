# after a cleanup: all GPU tests, engine 2 on cfg2 (bench line), the default cfg4 bench (e2e legs)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-chk}
timeout -s ABRT 1200 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest gpu rc=$?"; tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 600 python bench.py --config cfg2 --no-cpu-baseline --no-batch --steps 20 --warmup 5 > gpurun_out/bench_cfg2_${TAG}.json 2> gpurun_out/bench_cfg2_${TAG}.err; echo "cfg2 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg2_${TAG}.json')); print('cfg2 ms', round(d['ms_per_step'],3), d['parity'], 'factor', round(d['roofline']['kernel_ms'],3), 'e2e', round(d['e2e']['ms_per_matrix'],3), 'api', round(d['e2e_api']['ms_per_matrix'],2))"
timeout 900 python bench.py --no-cpu-baseline --no-batch > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}.json')); print('cfg4 ms', round(d['ms_per_step'],3), d['parity'], 'e2e', round(d['e2e']['ms_per_matrix'],2), 'api', round(d['e2e_api']['ms_per_matrix'],2))"
