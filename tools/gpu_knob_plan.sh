# host-side plan knob sweep (same kernel binary): VAR=GLU_SN_MINGATHER VALS="3 2 5 8 3" CFG=cfg4
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in ${VALS}; do
  env "$VAR=$v" timeout 600 python tools/sn_probe.py ${CFG:-cfg4} --engines sn --reps 5 ${PARITY:---no-parity} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', '${CFG:-cfg4}', round(d['ms'],3), 'med', round(sorted(d['ms_all'])[2],3), d['parity'], 'tasks', (d.get('sn') or {}).get('tasks'), 'rg', (d.get('sn') or {}).get('rg_tasks'))"
done
