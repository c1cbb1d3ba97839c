"""Supernodal vs per-MAC engine on one config: device time per
refactorization (CUDA events), plan size and setup time, bitwise parity vs
the CPU oracle (factor_parallel deterministic on all host cores).

    python tools/sn_probe.py g400 [cfg4 ...] [--engines sn,plan] [--reps 5]
"""

from __future__ import annotations

import argparse
import json
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def phase_profile(fz, fp, a_d, v, st):
    """Per-phase durations from the kernel's completion stamps, grouped by
    the kind of tasks the phase holds (0 DIAG, 1 TRSM/TRI, 2 RECT)."""
    import torch

    sys.path.insert(0, str(ROOT / "tests"))
    import sn_emul
    from paper_1908_00204_b200 import _lib

    plan = sn_emul.build(fp)
    fz.set_option(15, 2)
    fz.scatter_device(a_d, v, st)
    fz.factor_device_async(v, 1e-14, st)
    torch.cuda.synchronize()
    nph = len(plan["phase_ptr"]) - 1
    buf = np.zeros(nph + 1, dtype=np.int64)
    _lib.lib.glu_sn_stamps(fz.handle, _lib.ptr(buf), nph + 1)
    ntasks = len(plan["tasks"])
    tr = np.zeros((ntasks, 4), dtype=np.int64)
    _lib.lib.glu_sn_trace(fz.handle, _lib.ptr(tr), ntasks)
    fz.set_option(15, 0)
    dur = np.diff(buf).astype(np.float64) * 1e-3  # us
    tasks, pp = plan["tasks"], plan["phase_ptr"]
    kinds = np.array([int(tasks[pp[p], 0]) >> 28 for p in range(nph)])  # 0 trsm/tri/diag-ish, 1 rect
    kinds = np.array([min(int(k), 1) + 1 for k in kinds])  # 1: phase led by TRSM/TRI, 2: RECT/DIAG
    ntask = np.diff(pp)
    out = {"total_us": float(dur.sum()), "phases": nph}
    for k, name in ((0, "diag"), (1, "trsm_tri"), (2, "rect")):
        d = dur[kinds == k]
        if len(d):
            out[name] = {"n": int(len(d)), "sum_us": float(d.sum()), "median_us": float(np.median(d)),
                         "p90_us": float(np.percentile(d, 90)), "max_us": float(d.max()),
                         "tasks_median": float(np.median(ntask[kinds == k]))}
    # phases by task count
    for lo, hi in ((1, 1), (2, 8), (9, 64), (65, 512), (513, 1 << 30)):
        m = (ntask >= lo) & (ntask <= hi)
        if m.any():
            out[f"tasks_{lo}_{hi}"] = {"n": int(m.sum()), "sum_us": float(dur[m].sum()),
                                       "median_us": float(np.median(dur[m]))}
    # per phase: wake (previous phase complete -> first / last task past its
    # wait), execution (longest task), flush (last task done -> phase complete)
    ph_of = np.repeat(np.arange(nph), ntask)
    t1, t2 = tr[:, 1].astype(np.float64), tr[:, 2].astype(np.float64)
    first_wait = np.full(nph, np.inf)
    last_wait = np.zeros(nph)
    last_done = np.zeros(nph)
    exec_max = np.zeros(nph)
    np.minimum.at(first_wait, ph_of, t1)
    np.maximum.at(last_wait, ph_of, t1)
    np.maximum.at(last_done, ph_of, t2)
    np.maximum.at(exec_max, ph_of, t2 - t1)
    prev = buf[:-1].astype(np.float64)
    comp = {"wake_first_us": (first_wait - prev) * 1e-3, "wake_last_us": (last_wait - prev) * 1e-3,
            "exec_max_us": exec_max * 1e-3, "flush_us": (buf[1:] - last_done) * 1e-3}
    for k, x in comp.items():
        out[k] = {"sum": float(x.sum()), "median": float(np.median(x)), "p90": float(np.percentile(x, 90))}
    kinds_t = (tasks[:, 0] >> 28)  # (kind << 27) >> 28 = kind index
    for k, name in ((0, "diag"), (1, "trsm"), (2, "tri"), (3, "rect")):
        m = kinds_t == k
        if m.any():
            d = (t2[m] - t1[m]) * 1e-3
            out[f"task_{name}_us"] = {"n": int(m.sum()), "median": float(np.median(d)),
                                     "p90": float(np.percentile(d, 90)), "max": float(d.max())}
    wd = tasks[:, 3] - tasks[:, 2]
    wcls = np.select([wd <= 1, wd <= 2, wd <= 4, wd <= 8, wd <= 16], [1, 2, 4, 8, 16], 32)
    npair = tasks[:, 7] - tasks[:, 6]
    by = {}
    for k, name in ((0, "diag"), (1, "trsm"), (2, "tri"), (3, "rect")):
        for wc in (1, 2, 4, 8, 16, 32):
            m = (kinds_t == k) & (wcls == wc)
            if m.any():
                d = (t2[m] - t1[m]) * 1e-3
                by[f"{name}{wc}"] = [int(m.sum()), round(float(np.median(d)), 2),
                                     round(float(np.percentile(d, 90)), 2), round(float(d.max()), 2),
                                     round(float(npair[m].mean()), 1)]
    out["by_kind_width[n,med,p90,max,npair]"] = by
    top = np.argsort(dur)[::-1][:8]
    out["top"] = [(int(p), int(kinds[p]), int(ntask[p]), round(float(dur[p]), 1)) for p in top]
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("configs", nargs="+")
    p.add_argument("--engines", default="sn,plan")
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--no-parity", action="store_true")
    p.add_argument("--stamps", action="store_true", help="per-phase completion profile (sn)")
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
                prof = phase_profile(fz, fp, a_d, v, st)
            par = None
            if ref is not None:
                par = "bitwise" if np.array_equal(out, ref) else \
                    f"MISMATCH max|d|={np.max(np.abs(out - ref)):.3e} n_diff={int(np.sum(out != ref))}"
            rec = dict(config=name, engine=eng, n=a.n, nnz=fp.nnz, macs=macs, analysis_s=round(t_an, 2),
                       setup_s=round(t_setup, 2), ms=min(ts), ms_all=[round(x, 3) for x in ts],
                       parity=par, plan=fz.plan_info.get("plan_bytes"),
                       sn=getattr(fz, "sn_info", None), device_bytes=fz.handle_info["device_bytes"],
                       ref_s=round(t_ref, 2) if ref is not None else None, phases=prof)
            print(json.dumps(rec), flush=True)
            fz.close()
            del v, a_d
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
