#!/bin/bash
# One gpurun call: parity tests, smoke, per-level timing, bench.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout -s ABRT ${PYTEST_TIMEOUT:-600} python -X faulthandler -m pytest tests -m gpu -x -q --durations 8 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
for c in ${DIAG_CFGS:-cfg1 cfg2}; do for k in 1 0; do timeout 180 python tools/diag_levels.py $c $k 2>&1 | tail -1; done; done
if [ -n "${BENCH:-1}" ]; then
  timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --cpu-budget 10 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
  tail -3 gpurun_out/bench_cfg2.err; cat gpurun_out/bench_cfg2.json
fi
