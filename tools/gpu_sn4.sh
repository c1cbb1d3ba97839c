cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-sn4}
timeout -s ABRT 600 python -X faulthandler -m pytest tests/test_gpu_sn.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_sn_${TAG}.log 2>&1
echo "pytest sn rc=$?"; tail -3 gpurun_out/pytest_sn_${TAG}.log
timeout 600 python tools/sn_probe.py g400 --engines sn --reps 3 --no-parity > gpurun_out/probe_${TAG}.jsonl 2> gpurun_out/probe_${TAG}.err; echo "probe rc=$?"
cut -c1-300 gpurun_out/probe_${TAG}.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sn_kernel -s 1 -c 1 -f -o gpurun_out/prof_sn_g400_${TAG} \
   python tools/sn_probe.py g400 --engines sn --reps 1 --no-parity > gpurun_out/ncu_g400_${TAG}.log 2>&1; echo "ncu rc=$?"
