"""Host-only plan statistics for a synthetic config (no GPU needed)."""
import sys, time, ctypes, pathlib
import numpy as np
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1908_00204_b200 as glu
from paper_1908_00204_b200 import synthetic, _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
contract = int(sys.argv[2]) if len(sys.argv) > 2 else 1
T = int(sys.argv[3]) if len(sys.argv) > 3 else 0
D = int(sys.argv[4]) if len(sys.argv) > 4 else 0
a = synthetic.make(cfg)
fp = glu.symbolic_fillin(a.pattern)
s = glu.levelize(glu.detect_relaxed(fp))
t = time.time()
pp = ctypes.c_void_p()
rc = _lib.lib.glu_plan_build(a.n, _lib.ptr(fp.full.col_ptr), _lib.ptr(fp.full.row_idx),
                             _lib.ptr(fp.diag_pos), _lib.ptr(_lib.i64(s.level_of)), contract, T, D,
                             int(sys.argv[5]) if len(sys.argv) > 5 else 0, 0,
                             ctypes.byref(pp))
print("plan build s", round(time.time() - t, 2), rc)
info = np.zeros(16, np.int64)
_lib.lib.glu_plan_info(pp, _lib.ptr(info))
names = ("levels", "items", "chunks", "macs", "max_item_macs", "max_chunks", "deferred", "bytes",
         "deep_items", "deep_macs", "epochs", "push_macs", "targets", "tail_t0", "tail_macs")
print(dict(zip(names, info.tolist())))
nl, ni, nc, nd = info[0], info[1], info[2], info[9]
lip = np.zeros(nl + 1, np.int64); items = np.zeros(ni * 8, np.int64); ch = np.zeros(nc * 5, np.int64)
dp = np.zeros(max(nd, 1) * 3, np.int64)
_lib.lib.glu_plan_export(pp, _lib.ptr(lip), _lib.ptr(items), _lib.ptr(ch), _lib.ptr(dp), None, None)
items = items.reshape(-1, 8); ch = ch.reshape(-1, 5)
ipl = np.diff(lip)
cs = np.concatenate([[0], np.cumsum(items[:, 6])]); mpl = cs[lip[1:]] - cs[lip[:-1]]
push = items[items[:, 7] == 0]; deep = items[items[:, 7] == 1]
print("items/level pct", np.percentile(ipl, [0, 10, 50, 90, 100]))
print("macs/level pct", np.percentile(mpl, [0, 10, 50, 90, 100]))
print("push item macs pct", np.percentile(push[:, 6], [10, 50, 90, 99, 100]))
print("push chunks/item pct", np.percentile(push[:, 4], [10, 50, 90, 99, 100]))
print("push targets/item pct", np.percentile(push[:, 5], [10, 50, 90, 99, 100]))
if len(deep):
    print("deep item macs pct", np.percentile(deep[:, 6], [10, 50, 90, 99, 100]))
ep = np.concatenate([[0], np.cumsum(ch[:, 4])])
epi = ep[push[:, 3] + push[:, 4]] - ep[push[:, 3]]
print("epochs/push item pct", np.percentile(epi, [10, 50, 90, 99, 100]))
