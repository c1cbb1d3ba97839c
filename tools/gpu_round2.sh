# round-2 evidence pass: default bench (cfg4 + cfg5 batch), the reference arm,
# ncu launch list and one --set full capture of sn_kernel (1 GPU)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r2c}
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_${TAG}.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4_${TAG}.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parity --no-e2e --no-batch > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "launch rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:sn_kernel -s 1 -c 1 -f -o gpurun_out/prof_sn_cfg4_${TAG} \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity --no-e2e --no-batch > gpurun_out/ncu_sn_${TAG}.log 2>&1; echo "ncu rc=$?"
