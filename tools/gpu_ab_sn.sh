# supernodal-kernel change: sn GPU tests, then library swap (tools/instr_lib/old vs working tree) on cfg4 and g400
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-absn}
timeout -s ABRT 900 python -X faulthandler -m pytest tests/test_gpu_sn.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_sn_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_sn_${TAG}.log
cp paper_1908_00204_b200/libglu_b200.so /tmp/new.so
for v in old new old new; do
  if [ $v = old ]; then cp tools/instr_lib/old/libglu_b200.so paper_1908_00204_b200/libglu_b200.so; else cp /tmp/new.so paper_1908_00204_b200/libglu_b200.so; fi
  echo "lib=$v"; timeout 600 python tools/sn_ab.py ${CFGS:-cfg4 g400} --vals 1 --reps 5 2>> gpurun_out/ab_${TAG}.err
done
cp /tmp/new.so paper_1908_00204_b200/libglu_b200.so
