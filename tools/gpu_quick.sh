#!/bin/bash
# Quick GPU iteration: parity tests, per-level timing, short bench.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout -s ABRT ${PYTEST_TIMEOUT:-400} python -X faulthandler -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for c in ${DIAG_CFGS:-cfg2}; do for k in 1 0; do timeout 180 python tools/diag_levels.py $c $k 2>&1 | tail -1 | cut -c1-400; done; done
timeout 300 python bench.py --config ${CFG:-cfg2} --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -3 gpurun_out/bench_quick.err; cat gpurun_out/bench_quick.json | cut -c1-600
