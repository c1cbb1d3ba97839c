#!/bin/bash
# Same-box A/B of a plan/tuning environment variable: VAR=name VALS="a b" CFGS="cfg2" tools/ab_env.sh
set -u
mkdir -p gpurun_out
for cfg in ${CFGS:-cfg2}; do
  for v in ${VALS}; do
    env "$VAR=$v" timeout 600 python bench.py --config $cfg --no-cpu-baseline --steps 20 --warmup 5 \
      > gpurun_out/ab.json 2> gpurun_out/ab_${cfg}_${v}.err
    python -c "
import json,sys
try:
    d=json.loads(open('gpurun_out/ab.json').read()); r=d['roofline']
    print('$cfg', '$VAR=$v', round(d['ms_per_matrix'],3), 'factor', round(r['kernel_ms'],3), 'items', d['config']['plan']['items'])
except Exception as e:
    print('$cfg', '$VAR=$v', 'FAILED'); print(open('gpurun_out/ab_${cfg}_${v}.err').read()[-600:])
"
  done
done
