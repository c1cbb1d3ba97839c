set -u
for v in 32 200 1000 32 200; do
  GLU_POLL_NS=$v timeout 600 python bench.py --batch 8 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batch8 poll', $v, round(d['value'],1), '/s')"
done
for v in 32 200 32 200; do
  GLU_POLL_NS=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('single poll', $v, round(d['ms_per_matrix'],3), 'ms')"
done
