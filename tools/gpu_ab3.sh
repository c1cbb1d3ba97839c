# TRSM fast-path experiment: sn GPU tests (fast path on), knob A/B in one process, library swap vs tools/instr_lib/old
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-ab3}
timeout -s ABRT 900 python -X faulthandler -m pytest tests/test_gpu_sn.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_sn_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_sn_${TAG}.log
echo "knob"; timeout 900 python tools/sn_ab.py cfg4 g400 --var GLU_SN_TRSM_FAST --vals 0,1 --reps 6 2>> gpurun_out/ab_${TAG}.err
cp paper_1908_00204_b200/libglu_b200.so /tmp/new.so
for v in old new old new; do
  if [ $v = old ]; then cp tools/instr_lib/old/libglu_b200.so paper_1908_00204_b200/libglu_b200.so; else cp /tmp/new.so paper_1908_00204_b200/libglu_b200.so; fi
  echo "lib=$v"; timeout 600 python tools/sn_ab.py cfg4 --vals 1 --reps 5 2>> gpurun_out/ab_${TAG}.err
done
cp /tmp/new.so paper_1908_00204_b200/libglu_b200.so
