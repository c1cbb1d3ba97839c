#!/bin/bash
# express-queue parameter sweep (diagnostics): R K MAX per line
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for cfgl in "0 3 3000" "8 3 3000" "16 3 3000" "8 1 3000" "8 5 3000" "16 5 5000" "24 4 5000"; do
  set -- $cfgl
  GLU_EXPRESS_R=$1 GLU_EXPRESS_K=$2 GLU_EXPRESS_MAX=$3 timeout 200 python tools/diag_levels.py cfg2 1 2>&1 | tail -1 | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('R=$1 K=$2 MAX=$3', round(d['total_ms'],3), 'ms', 'express', d['plan'].get('express_items'))"
done
