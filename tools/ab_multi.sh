#!/bin/bash
# Same-box comparison of several prebuilt libraries: LIBS="old A B" (tools/instr_lib/<name>/libglu_b200.so)
set -u
cp paper_1908_00204_b200/libglu_b200.so /tmp/cur.so
for rep in 1 2; do
  for v in ${LIBS}; do
    cp tools/instr_lib/$v/libglu_b200.so paper_1908_00204_b200/libglu_b200.so
    timeout 600 python bench.py --no-cpu-baseline --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', round(d['ms_per_matrix'],3), 'factor', round(r['kernel_ms'],3), 'tail', round(d.get('roofline_tail',{}).get('kernel_ms',0),3))"
  done
done
cp /tmp/cur.so paper_1908_00204_b200/libglu_b200.so
