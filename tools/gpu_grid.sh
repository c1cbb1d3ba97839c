#!/bin/bash
# G3-family scaling points (bench.py --config gNNN) with peak host memory.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
free -g | head -2
for cfg in ${CFGS:-g600}; do
  python - "$cfg" > gpurun_out/bench_${cfg}.json 2> gpurun_out/bench_${cfg}.err <<'PY'
import resource, runpy, sys
cfg = sys.argv[1]
sys.argv = ["bench.py", "--config", cfg, "--steps", "5", "--warmup", "3"]
try:
    runpy.run_path("bench.py", run_name="__main__")
finally:
    print(f"peak RSS {resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6:.1f} GB", file=sys.stderr)
PY
  echo "$cfg rc=$?"; cut -c1-600 gpurun_out/bench_${cfg}.json; tail -3 gpurun_out/bench_${cfg}.err
done
