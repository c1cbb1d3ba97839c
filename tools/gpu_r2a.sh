# round-2 check pass: GPU tests, reference suite under the levlu alias, smoke, cfg4 bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r2a} bash tools/gpu_tests.sh
timeout 900 python bench.py > gpurun_out/b_cfg4_${TAG:-r2a}.json 2> gpurun_out/b_cfg4_${TAG:-r2a}.err; echo "bench cfg4 rc=$?"; tail -3 gpurun_out/b_cfg4_${TAG:-r2a}.err
