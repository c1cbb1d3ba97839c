cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for A in rr load sim; do
GLU_SN_ASSIGN=$A timeout 900 python tools/sn_probe.py g400 cfg4 --engines sn --reps 3 --no-parity > gpurun_out/probe_as_$A.jsonl 2> gpurun_out/probe_as_$A.err; echo "assign=$A rc=$?"
python -c "
import json
for l in open('gpurun_out/probe_as_$A.jsonl'):
    d=json.loads(l); print(d['config'], round(d['ms'],2))
"
done
