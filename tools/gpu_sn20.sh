cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-sn20}
for A in 1 0.7 0.4 0; do
GLU_SN_ORDER_ALPHA=$A timeout 900 python tools/sn_probe.py g400 cfg4 --engines sn --reps 3 --no-parity > gpurun_out/probe_${TAG}_a$A.jsonl 2> gpurun_out/probe_${TAG}_a$A.err; echo "alpha=$A rc=$?"
python -c "
import json
for l in open('gpurun_out/probe_${TAG}_a$A.jsonl'):
    d=json.loads(l); print(d['config'], round(d['ms'],2))
"
done
