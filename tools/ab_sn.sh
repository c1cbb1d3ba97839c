# A/B of prebuilt libglu_b200.so variants (tools/ab_so/<name>/, git-ignored)
# on the supernodal engine: GPU sn tests once per variant, then cfg4 / g400
# timings interleaved.  VARIANTS="base u2 ..." TAG=... bash tools/ab_sn.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-ab}
for v in $VARIANTS; do
  cp tools/ab_so/$v/libglu_b200.so paper_1908_00204_b200/libglu_b200.so
  timeout -s ABRT 600 python -m pytest tests/test_gpu_sn.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_${TAG}_$v.log 2>&1
  echo "$v pytest rc=$? $(tail -1 gpurun_out/pytest_${TAG}_$v.log)"
done
for rep in 1 2; do
  for v in $VARIANTS; do
    cp tools/ab_so/$v/libglu_b200.so paper_1908_00204_b200/libglu_b200.so
    for cfg in g400 cfg4; do
      timeout 600 python tools/sn_probe.py $cfg --engines sn --reps 3 --no-parity 2>>gpurun_out/ab_${TAG}.err | python -c "import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['config'], round(d['ms'],2))"
    done
  done
done
