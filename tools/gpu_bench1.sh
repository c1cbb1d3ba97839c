cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python bench.py --config g200 --steps 3 --warmup 2 --batch-total 64 > gpurun_out/b_g200.json 2> gpurun_out/b_g200.err; echo "bench g200 rc=$?"; tail -3 gpurun_out/b_g200.err; cut -c1-300 gpurun_out/b_g200.json
timeout 900 python bench.py > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err; echo "bench cfg4 rc=$?"; tail -3 gpurun_out/b_cfg4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err; echo "ref rc=$?"; tail -3 gpurun_out/b_ref.err
timeout -s ABRT 900 python -X faulthandler -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
