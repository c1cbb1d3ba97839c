set -u
cp paper_1908_00204_b200/libglu_b200.so /tmp/new.so
for v in new old new old; do
  if [ $v = old ]; then cp tools/instr_lib/old/libglu_b200.so paper_1908_00204_b200/libglu_b200.so; else cp /tmp/new.so paper_1908_00204_b200/libglu_b200.so; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', round(d['ms_per_matrix'],3), 'factor', round(r['kernel_ms'],3), 'tail', round(d.get('roofline_tail',{}).get('kernel_ms',0),3))"
done
