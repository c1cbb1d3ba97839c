import sys, pathlib, numpy as np
sys.path.insert(0, ".")
import paper_1908_00204_b200 as glu
from paper_1908_00204_b200 import _lib, synthetic
a = synthetic.make("cfg2"); fp = glu.symbolic_fillin(a.pattern); s = glu.levelize(glu.detect_relaxed(fp))
fz = glu.get_factorizer(fp, s.level_of, _lib.CONTRACT_B); fz.set_input(a.col_ptr, a.row_idx); fz.set_option(13, 1)
for _ in range(3): fz.factor_host(a.values, 1e-14)
buf = np.zeros(8 + 6 * 64, dtype=np.int64); w = int(_lib.lib.glu_tail_trace_read(fz.handle, _lib.ptr(buf), len(buf)))
t = buf.astype(float); t0 = t[0]
P = t[8:8 + 6 * 37].reshape(37, 6)
print("CTA0 loaded", (t[1]-t0)/1e3, "CTA3 loaded", (t[5]-t0)/1e3, "CTA3 umax done", (t[6]-t0)/1e3, "CTA3 before await(2)", (t[7]-t0)/1e3)
print("publish times p0..p3:", [(P[p,4]-t0)/1e3 for p in range(4)], "CTA3 observed p2:", (P[3,0]-t0)/1e3)
