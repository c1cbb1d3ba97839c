for v in 100000000 6000 100000000 6000; do
  GLU_CRIT_WIDE=$v timeout 600 python bench.py --batch 8 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batch8 crit_wide', $v, round(d['value'],1), '/s')"
done
