"""Per-panel timeline of the dense-tail cluster kernel (glu_set_option 13).

    python tools/tail_trace.py [cfg2]

Prints the kernel's phases (column load, panel loop, store, divide) and,
per panel p, its owner's hand-off latency (observed p-1 minus the previous
owner's publish), look-ahead apply, panel column sweep, write-back and
publish times.
"""
import json
import os
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1908_00204_b200 as glu  # noqa: E402
from paper_1908_00204_b200 import _lib, synthetic  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
a = synthetic.make(cfg)
fp = glu.symbolic_fillin(a.pattern)
s = glu.levelize(glu.detect_relaxed(fp))
fz = glu.get_factorizer(fp, s.level_of, _lib.CONTRACT_B)
fz.set_input(a.col_ptr, a.row_idx)
fz.set_option(13, 1)
for _ in range(4):
    lu, rc = fz.factor_host(a.values, 1e-14)
    assert rc == -1 or os.environ.get("TRACE_NOCHECK"), rc  # timing-only variants: wrong values
buf = np.zeros(8 + 6 * 4096, dtype=np.int64)
w = int(_lib.lib.glu_tail_trace_read(fz.handle, _lib.ptr(buf), len(buf)))
t = buf[:w].astype(np.float64)
t0 = t[0]
ph = {"load_us": (t[1] - t[0]) / 1e3, "panels_us": (t[2] - t[1]) / 1e3,
      "store_divide_us": (t[4] - t[2]) / 1e3, "total_us": (t[4] - t[0]) / 1e3}
npan = (w - 8) // 6
P = t[8:8 + 6 * npan].reshape(npan, 6)  # observed, applied, block factored, factored, published
rows = []
for p in range(1, npan):
    if P[p, 0] == 0:
        continue
    rows.append({"p": p, "handoff_us": (P[p, 0] - P[p - 1, 4]) / 1e3, "apply_us": (P[p, 1] - P[p, 0]) / 1e3,
                 "factor_us": (P[p, 2] - P[p, 1]) / 1e3, "writeback_us": (P[p, 3] - P[p, 2]) / 1e3,
                 "publish_us": (P[p, 4] - P[p, 3]) / 1e3})
mean = {k: float(np.mean([r[k] for r in rows]))
        for k in ("handoff_us", "apply_us", "factor_us", "writeback_us", "publish_us")}
print(json.dumps({"config": cfg, "panels": npan, "phases": ph, "per_panel_mean": mean,
                  "panel0_factor_us": (P[0, 3] - P[0, 1]) / 1e3,
                  "handoff_all_us": [round(r["handoff_us"], 2) for r in rows],
                  "first_panels": rows[:6], "last_panels": rows[-4:]}, indent=1))
