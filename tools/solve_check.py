"""Triangular solves on one config: GPU dataflow solve (1 and 32 right-hand
sides, device-resident factors, CUDA events) against the CPU oracle's
lower/upper solve on the same factors (bitwise check, single thread).

    python tools/solve_check.py cfg4
"""
import ctypes
import json
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import paper_1908_00204_b200 as glu
    from paper_1908_00204_b200 import _lib, numeric, synthetic
    from oracle import oracle as orc

    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    a = synthetic.make(cfg)
    fp = glu.symbolic_fillin(a.pattern)
    lv = numeric._relaxed_levels(fp)
    fz = numeric.get_factorizer(fp, lv, _lib.CONTRACT_A)
    fz.set_input(a.col_ptr, a.row_idx)
    fz.set_option(1, 0)
    lu, rc = fz.factor_host(a.values, 1e-14)
    assert rc == -1
    dev = torch.device("cuda", 0)
    lu_d = torch.from_numpy(lu).to(dev)
    st = torch.cuda.current_stream()
    b = np.random.default_rng(0).standard_normal(a.n)
    out = {"config": cfg, "n": a.n, "nnz": fp.nnz, "engine": fz.engine}
    for k in (1, 32):
        x0 = torch.from_numpy(np.tile(b, (k, 1))).to(dev)
        ts = []
        for _ in range(3):
            x = x0.clone()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _lib.lib.glu_solve_multi_device(fz.handle, numeric._dptr(lu_d), numeric._dptr(x), k, a.n, 0,
                                            ctypes.c_void_p(st.cuda_stream))
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[f"gpu_ms_k{k}"] = min(ts)
        if k == 1:
            xg = x[0].cpu().numpy()
    pat = orc.Pattern.from_fp(fp)
    t0 = time.perf_counter()
    xr, bad = orc.upper_solve(pat, lu, orc.lower_solve(pat, lu, b))
    out["cpu_oracle_ms_k1"] = (time.perf_counter() - t0) * 1e3
    out["bitwise_k1"] = bool(bad == -1 and np.array_equal(xg, xr))
    # solution residual ||A x - b|| / ||b|| (north_star: <= 1e-10)
    import scipy.sparse as sp

    A = sp.csc_matrix((a.values, a.row_idx, a.col_ptr), shape=(a.n, a.n))
    out["residual_k1"] = float(np.linalg.norm(A @ xg - b) / np.linalg.norm(b))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
