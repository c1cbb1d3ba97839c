# library-swap A/B on cfg2 (engine 2): tools/instr_lib/old vs the working tree's library
cd "${GRAFT_REPO_ROOT:-/root/repo}"
cp paper_1908_00204_b200/libglu_b200.so /tmp/new.so
for v in old new old new old new; do
  if [ $v = old ]; then cp tools/instr_lib/old/libglu_b200.so paper_1908_00204_b200/libglu_b200.so; else cp /tmp/new.so paper_1908_00204_b200/libglu_b200.so; fi
  timeout 600 python bench.py --config ${CFG:-cfg2} --no-cpu-baseline --no-batch --no-e2e --no-parity --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', round(d['ms_per_matrix'],3), 'factor', round(r['kernel_ms'],3))"
done
cp /tmp/new.so paper_1908_00204_b200/libglu_b200.so
