#!/bin/bash
# batched-launch throughput of several prebuilt libraries (LIBS="old new")
cp paper_1908_00204_b200/libglu_b200.so /tmp/cur_b.so
for v in ${LIBS}; do
  cp tools/instr_lib/$v/libglu_b200.so paper_1908_00204_b200/libglu_b200.so
  timeout 600 python bench.py --batch 32 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v batch32', round(d['value'],1), '/s', d.get('parity'))"
done
cp /tmp/cur_b.so paper_1908_00204_b200/libglu_b200.so
