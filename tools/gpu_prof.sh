#!/bin/bash
# One gpurun call: ncu launch list of a short bench run + one `--set full`
# capture of the persistent factor kernel.  Usage: CFG=cfg2 TAG=r1 tools/gpu_prof.sh
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${CFG:-cfg2}; TAG=${TAG:-r1}; CON=${CON:-B}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}_${CFG}.csv \
  python bench.py --config $CFG --contract $CON --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_launch_bench_${TAG}_${CFG}.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 2 -c 1 \
  -f -o gpurun_out/prof_${TAG}_${CFG} \
  python bench.py --config $CFG --contract $CON --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_full_${TAG}_${CFG}.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full_${TAG}_${CFG}.log
