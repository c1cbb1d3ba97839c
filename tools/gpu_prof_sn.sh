# ncu evidence for the supernodal engine on cfg4: launch list of a short
# bench run, then one --set full capture of sn_kernel (1 GPU, never multi-rank)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_cfg4_${TAG}.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parity --no-e2e --no-batch \
  > gpurun_out/ncu_launch_cfg4_${TAG}.log 2>&1; echo "launch rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:sn_kernel -s 1 -c 1 \
  -f -o gpurun_out/prof_sn_cfg4_${TAG} python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  --no-parity --no-e2e --no-batch > gpurun_out/ncu_sn_cfg4_${TAG}.log 2>&1; echo "ncu sn rc=$?"
tail -3 gpurun_out/ncu_sn_cfg4_${TAG}.log
