# round-2 data points beside the headline: cfg3 (engine 2) bench line, G3-family grids on the supernodal engine with oracle parity
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg3 --no-batch > gpurun_out/bench_cfg3_fam.json 2> gpurun_out/bench_cfg3_fam.err; echo "cfg3 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg3_fam.json')); print('cfg3 ms', round(d['ms_per_step'],3), d['parity'], 'e2e', round(d['e2e']['ms_per_matrix'],3), 'cpu', d['cpu_baseline']['ms_per_matrix'])"
timeout 1500 python tools/sn_probe.py g400 g600 g800 --engines sn --reps 5 > gpurun_out/family_sn.jsonl 2> gpurun_out/family_sn.err; echo "family rc=$?"
python -c "
import json
for l in open('gpurun_out/family_sn.jsonl'):
    d=json.loads(l); print(d['config'], d['n'], d['macs'], 'ms', round(d['ms'],3), d['parity'], 'cpu_s', d['ref_s'])"
