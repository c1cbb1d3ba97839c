cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python tools/sn_probe.py g400 --engines sn --reps 2 --stamps --no-parity > gpurun_out/probe6.jsonl 2> gpurun_out/probe6.err; echo "probe rc=$?"
tail -5 gpurun_out/probe6.err
