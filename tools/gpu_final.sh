# round-2 final evidence pass: GPU tests + the reference's suite + smoke, the
# default bench (cfg4 + cfg5), the reference arm, ncu launch list + one
# --set full capture of sn_kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r2f}
TAG=$TAG bash tools/gpu_tests.sh
TAG=$TAG bash tools/gpu_round2.sh
