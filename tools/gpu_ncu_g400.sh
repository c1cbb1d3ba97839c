cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-x}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sn_kernel -s 1 -c 1 -f -o gpurun_out/prof_sn_g400_${TAG} \
   python tools/sn_probe.py g400 --engines sn --reps 1 --no-parity > gpurun_out/ncu_g400_${TAG}.log 2>&1; echo "ncu rc=$?"
