#!/bin/bash
# batched-launch throughput of the current library: bench --batch 8, twice
for rep in 1 2; do
  timeout 600 python bench.py --batch 8 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batch8', round(d['value'],1), '/s', d.get('parity'))"
done
