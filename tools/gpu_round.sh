#!/bin/bash
# Round evidence in one gpurun call: GPU parity tests, smoke, the default
# bench (with the CPU baseline), the reference arm, ncu launch list and one
# `--set full` capture of each of our kernels.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout -s ABRT 600 python -X faulthandler -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
cat gpurun_out/bench_${TAG}.json | cut -c1-400
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2>&1; echo "ref rc=$?"
cut -c1-300 gpurun_out/bench_ref_${TAG}.json
timeout 600 python bench.py --batch 32 --steps 5 --warmup 3 > gpurun_out/bench_batch32_${TAG}.json 2> gpurun_out/bench_batch32_${TAG}.err; echo "batch rc=$?"
cut -c1-300 gpurun_out/bench_batch32_${TAG}.json
timeout 900 python bench.py --config cfg3 --steps 10 --warmup 3 > gpurun_out/bench_cfg3_${TAG}.json 2> gpurun_out/bench_cfg3_${TAG}.err; echo "cfg3 rc=$?"
cut -c1-300 gpurun_out/bench_cfg3_${TAG}.json
timeout 300 python tools/solve_bench.py cfg2 > gpurun_out/solve_${TAG}.json 2>&1; echo "solve rc=$?"; cut -c1-300 gpurun_out/solve_${TAG}.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 2 -c 1 \
  -f -o gpurun_out/prof_factor_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_factor_${TAG}.log 2>&1; echo "ncu factor rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 2 -c 1 \
  -f -o gpurun_out/prof_tail_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_tail_${TAG}.log 2>&1; echo "ncu tail rc=$?"
