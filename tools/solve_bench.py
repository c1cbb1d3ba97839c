"""Triangular-solve timing (level-scheduled solve_kernel), cfg2: one and
several right-hand sides, device-resident factors."""
import sys, os, json, pathlib, ctypes
import numpy as np
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
import paper_1908_00204_b200 as glu
from paper_1908_00204_b200 import synthetic, _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
a = synthetic.make(cfg)
fp = glu.symbolic_fillin(a.pattern)
s = glu.levelize(glu.detect_relaxed(fp))
fz = glu.get_factorizer(fp, s.level_of, 0)
fz.set_input(a.col_ptr, a.row_idx)
tblock = int(os.environ.get("GLU_SOLVE_TBLOCK", "-1"))
if tblock >= 0:
    fz.set_option(10, tblock)
multi = int(os.environ.get("GLU_SOLVE_MULTI", "1"))
fz.set_option(11, multi)
stail = int(os.environ.get("GLU_SOLVE_TAIL", "1"))
fz.set_option(14, stail)
long_row = int(os.environ.get("GLU_SOLVE_LONG", "-1"))
if long_row >= 0:
    fz.set_option(12, long_row)
lu, rc = fz.factor_host(a.values, 1e-14)
assert rc == -1
dev = torch.device("cuda", 0)
lu_d = torch.from_numpy(lu).to(dev)
st = torch.cuda.current_stream()
out = {"config": cfg, "tblock": tblock, "multi": multi, "tail_cta": stail, "long_row": long_row, "n": a.n, "lsolve_levels": fz.handle_info["lsolve_levels"],
       "usolve_levels": fz.handle_info["usolve_levels"]}
for k in (1, 8, 32):
    x = torch.randn((k, a.n), dtype=torch.float64, device=dev)
    for _ in range(2):
        _lib.lib.glu_solve_multi_device(fz.handle, glu.numeric._dptr(lu_d), glu.numeric._dptr(x), k, a.n, 0,
                                        ctypes.c_void_p(st.cuda_stream))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    reps = 5
    for _ in range(reps):
        _lib.lib.glu_solve_multi_device(fz.handle, glu.numeric._dptr(lu_d), glu.numeric._dptr(x), k, a.n, 0,
                                        ctypes.c_void_p(st.cuda_stream))
    e1.record(st)
    torch.cuda.synchronize()
    out[f"nrhs{k}_ms"] = e0.elapsed_time(e1) / reps
# L only / U only, one right-hand side
for part, name in ((1, "lower1_ms"), (2, "upper1_ms")):
    x = torch.randn((1, a.n), dtype=torch.float64, device=dev)
    for _ in range(2):
        _lib.lib.glu_solve_multi_device(fz.handle, glu.numeric._dptr(lu_d), glu.numeric._dptr(x), 1, a.n, part,
                                        ctypes.c_void_p(st.cuda_stream))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5):
        _lib.lib.glu_solve_multi_device(fz.handle, glu.numeric._dptr(lu_d), glu.numeric._dptr(x), 1, a.n, part,
                                        ctypes.c_void_p(st.cuda_stream))
    e1.record(st)
    torch.cuda.synchronize()
    out[name] = e0.elapsed_time(e1) / 5
# batch solves: nb sets, each its own factors (replicas here) and right-hand side
for nbs in (8, 32):
    L = lu_d.repeat(nbs, 1).reshape(nbs, -1).contiguous()
    X = torch.randn((nbs, a.n), dtype=torch.float64, device=dev)
    status = np.zeros(nbs, dtype=np.int64)
    def run():
        rc = _lib.lib.glu_solve_batch_device(fz.handle, glu.numeric._dptr(L), L.shape[1], glu.numeric._dptr(X),
                                             nbs, a.n, _lib.ptr(status), ctypes.c_void_p(st.cuda_stream))
        assert rc == -1, _lib.last_error()
    for _ in range(2):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5):
        run()
    e1.record(st)
    torch.cuda.synchronize()
    out[f"batch{nbs}_ms"] = e0.elapsed_time(e1) / 5
# residual of one solve through the public API
b = np.random.default_rng(0).standard_normal(a.n)
xs = glu.solve(glu.LuFactors(fp, lu), b)
import scipy.sparse as sp
A = sp.csc_matrix((a.values, a.row_idx, a.col_ptr), shape=(a.n, a.n))
out["residual"] = float(np.linalg.norm(A @ xs - b) / np.linalg.norm(b))
print(json.dumps(out))
