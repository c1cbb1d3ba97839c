"""Stage clocks of the owner's look-ahead apply in the tail kernel
(instrumented library only: loads / panel rows / rows below)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1908_00204_b200 as glu
from paper_1908_00204_b200 import _lib, synthetic
a = synthetic.make("cfg2"); fp = glu.symbolic_fillin(a.pattern); s = glu.levelize(glu.detect_relaxed(fp))
fz = glu.get_factorizer(fp, s.level_of, _lib.CONTRACT_B); fz.set_input(a.col_ptr, a.row_idx); fz.set_option(13, 1)
for _ in range(3):
    fz.factor_host(a.values, 1e-14)
buf = np.zeros(8 + 10 * 64, dtype=np.int64); w = int(_lib.lib.glu_tail_trace_read(fz.handle, _lib.ptr(buf), len(buf)))
npan = (w - 8) // 10
C = buf[8 + 6 * npan: 8 + 10 * npan].reshape(npan, 4)[1:]
d = np.diff(C, axis=1)
print("cycles loads / panel rows / rows below (median):", np.median(d, axis=0).astype(int).tolist())
print("per panel (every 6th):", d[::6].tolist())
