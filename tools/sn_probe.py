"""Supernodal vs per-MAC engine on one config: device time per
refactorization (CUDA events), plan size and setup time, bitwise parity vs
the CPU oracle (factor_parallel deterministic on all host cores).

    python tools/sn_probe.py g400 [cfg4 ...] [--engines sn,plan] [--reps 5]
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def task_profile(fz, fp, a_d, v, st):
    """Per-task timestamps of one factorization ({start, source ready, target
    ready, done}, glu_sn_trace): kernel span, the plan model's critical
    path, and per kind / width class the execution time after the last wait
    and the wait times."""
    import torch

    sys.path.insert(0, str(ROOT / "tests"))
    import sn_emul
    from paper_1908_00204_b200 import _lib

    plan = sn_emul.build(fp)
    tasks = plan["tasks"]
    ntasks = len(tasks)
    fz.set_option(15, 1)
    fz.scatter_device(a_d, v, st)
    fz.factor_device_async(v, 1e-14, st)
    torch.cuda.synchronize()
    tr = np.zeros((ntasks, 6), dtype=np.int64)
    _lib.lib.glu_sn_trace(fz.handle, _lib.ptr(tr), ntasks)
    fz.set_option(15, 0)
    warp = tr[:, 4].copy()
    clk = tr[:, 5].copy()
    tr = tr[:, :4]
    t0 = tr[:, 0].min()
    if os.environ.get("SN_TRACE_DUMP"):
        np.savez_compressed(os.environ["SN_TRACE_DUMP"], trace=((tr - t0) // 10).astype(np.int32),
                            warp=warp.astype(np.int32), clk=clk)
    tr = (tr - t0).astype(np.float64) * 1e-3  # us from kernel start
    kind = (tasks[:, 0].view(np.uint32) >> 29).astype(np.int64)
    w = tasks[:, 3] - tasks[:, 2]
    wcls = np.select([w <= 1, w <= 2, w <= 4, w <= 8], [1, 2, 4, 8], 16)
    out = {"span_us": float(tr[:, 3].max()), "model_crit_us": plan["info"]["crit_ns"] * 1e-3, "tasks": ntasks}
    execd = tr[:, 3] - tr[:, 2]
    wait_src = tr[:, 1] - tr[:, 0]
    wait_tgt = tr[:, 2] - tr[:, 1]
    by = {}
    for k, name in ((0, "trsm"), (1, "rect"), (2, "uw"), (3, "rg"), (4, "wb")):
        for wc in (1, 2, 4, 8, 16):
            m = (kind == k) & (wcls == wc)
            if m.any():
                by[f"{name}{wc}"] = [int(m.sum()), round(float(np.median(execd[m])), 2),
                                     round(float(np.percentile(execd[m], 90)), 2),
                                     round(float(np.median(wait_src[m])), 2), round(float(np.median(wait_tgt[m])), 2),
                                     round(float(execd[m].sum() * 1e-3), 1)]
    out["by_kind_width[n,exec_med,exec_p90,wait_src_med,wait_tgt_med,exec_sum_ms]"] = by
    m = (kind == 0) & (w >= 9)
    if m.any():  # TRSM phase cycles (loads, block, rows)
        c = clk[m]
        out["trsm_wide_cycles_med[loads,block,rows]"] = [int(np.median((c >> s) & ((1 << 21) - 1))) for s in (0, 21, 42)]
    m = (kind == 1) & (w >= 9)
    if m.any():  # RECT phase cycles after the target wait (loads, U solve, MACs + stores)
        c = clk[m]
        out["rect_wide_cycles_med[loads,usolve,macs]"] = [int(np.median((c >> s) & ((1 << 21) - 1))) for s in (0, 21, 42)]
    # busy fraction: sum of (done - start) over all warps / (warps x span)
    out["sum_exec_ms"] = float(execd.sum() * 1e-3)
    out["sum_wait_ms"] = float((tr[:, 2] - tr[:, 0]).sum() * 1e-3)
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("configs", nargs="+")
    p.add_argument("--engines", default="sn,plan")
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--no-parity", action="store_true")
    p.add_argument("--stamps", action="store_true", help="per-task trace profile (sn)")
    args = p.parse_args()
    import torch

    import paper_1908_00204_b200 as glu
    from paper_1908_00204_b200 import numeric, synthetic
    from oracle import oracle as orc

    dev = torch.device("cuda", 0)
    for name in args.configs:
        t0 = time.perf_counter()
        a = synthetic.make(name) if name in synthetic.CONFIGS else synthetic.grid5(int(name[1:]), seed=0)
        fp = glu.symbolic_fillin(a.pattern)
        lv = numeric._relaxed_levels(fp)
        t_an = time.perf_counter() - t0
        macs = numeric.pattern_flops(fp)[0]
        ref = None
        if not args.no_parity:
            t0 = time.perf_counter()
            pat = orc.Pattern.from_fp(fp)
            ref, bad = orc.scatter(pat, a.col_ptr, a.row_idx, a.values)
            s = glu.levelize(glu.detect_relaxed(fp))
            lp = np.concatenate([[0], np.cumsum([len(c) for c in s.levels])]).astype(np.int64)
            lc = np.concatenate(s.levels).astype(np.int64)
            ncpu = orc.cpu_count()
            caps = orc.concurrency_caps([int(x) for x in np.diff(lp)], ncpu, n=a.n)
            assert orc.factor_parallel(pat, ref, lp, lc, caps, True) == -1
            t_ref = time.perf_counter() - t0
        for eng in args.engines.split(","):
            if eng == "plan" and macs > 1.5e10:
                continue
            t0 = time.perf_counter()
            fz = numeric.Factorizer(fp, lv, 0, engine=eng)
            t_setup = time.perf_counter() - t0
            fz.set_input(a.col_ptr, a.row_idx)
            fz.set_option(1, 0)
            fz.set_option(2, 1)
            a_d = torch.from_numpy(a.values).to(dev)
            v = torch.empty(fp.nnz, dtype=torch.float64, device=dev)
            st = torch.cuda.current_stream()
            ts = []
            for r in range(args.reps + 1):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                fz.scatter_device(a_d, v, st)
                e0.record(st)
                fz.factor_device_async(v, 1e-14, st)
                e1.record(st)
                torch.cuda.synchronize()
                rc = fz.status(st)
                assert rc == -1, rc
                if r:
                    ts.append(e0.elapsed_time(e1))
            out = v.cpu().numpy()
            prof = None
            if args.stamps and eng == "sn":
                prof = task_profile(fz, fp, a_d, v, st)
            par = None
            if ref is not None:
                par = "bitwise" if np.array_equal(out, ref) else \
                    f"MISMATCH max|d|={np.max(np.abs(out - ref)):.3e} n_diff={int(np.sum(out != ref))}"
            rec = dict(config=name, engine=eng, n=a.n, nnz=fp.nnz, macs=macs, analysis_s=round(t_an, 2),
                       setup_s=round(t_setup, 2), ms=min(ts), ms_all=[round(x, 3) for x in ts],
                       parity=par, plan=fz.plan_info.get("plan_bytes"),
                       sn=getattr(fz, "sn_info", None), device_bytes=fz.handle_info["device_bytes"],
                       ref_s=round(t_ref, 2) if ref is not None else None, profile=prof)
            print(json.dumps(rec), flush=True)
            fz.close()
            del v, a_d
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
