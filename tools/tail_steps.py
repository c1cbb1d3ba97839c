"""Per-column-step clocks of the tail panel sweep (instrumented library only:
tools/instr_lib/libglu_b200.so built with per-step clock64 stamps)."""
import pathlib, sys
import numpy as np
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1908_00204_b200 as glu
from paper_1908_00204_b200 import _lib, synthetic
a = synthetic.make("cfg2")
fp = glu.symbolic_fillin(a.pattern)
s = glu.levelize(glu.detect_relaxed(fp))
fz = glu.get_factorizer(fp, s.level_of, _lib.CONTRACT_B)
fz.set_input(a.col_ptr, a.row_idx)
fz.set_option(13, 1)
for _ in range(3):
    fz.factor_host(a.values, 1e-14)
buf = np.zeros(8 + 24 * 64, dtype=np.int64)
w = int(_lib.lib.glu_tail_trace_read(fz.handle, _lib.ptr(buf), len(buf)))
npan = (w - 8) // 24
C = buf[8 + 6 * npan: 8 + 6 * npan + 18 * npan].reshape(npan, 18)
d = np.diff(C[:, :17], axis=1)  # cycles per step (k -> k+1), last = write-back start
print("panels", npan)
print("median cycles per step:", np.median(d[1:], axis=0).astype(int).tolist())
print("panel totals (cycles):", (C[1:6, 16] - C[1:6, 0]).tolist())
tot = C[:, 16] - C[:, 0]
print("per-panel sweep cycles, every 4th panel:", tot[::4].tolist())
