# ASAP-order latency model: hand-off latency (GLU_SN_HOP, host-side plan order only; same kernel binary)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for hop in ${HOPS:-2.5 1.5 4.0 6.0 2.5}; do
  GLU_SN_HOP=$hop timeout 600 python tools/sn_probe.py ${CFG:-cfg4} --engines sn --reps 5 --no-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('hop=$hop', round(d['ms'],3), [round(x,3) for x in d['ms_all']])"
done
