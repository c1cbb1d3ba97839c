cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for X in 0 5 30 200; do
GLU_SN_EXPRESS_SLACK=$X timeout 900 python tools/sn_probe.py g400 cfg4 --engines sn --reps 3 --no-parity > gpurun_out/probe_ex_$X.jsonl 2> gpurun_out/probe_ex_$X.err; echo "slack=$X rc=$?"
python -c "
import json
for l in open('gpurun_out/probe_ex_$X.jsonl'):
    d=json.loads(l); print(d['config'], round(d['ms'],2))
"
done
