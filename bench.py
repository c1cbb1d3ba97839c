"""Benchmark: GLU3.0 numeric (re)factorization on the B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4]
                    [--impl ours|reference] [--engine auto|sn|plan]
                    [--batch-config cfg2] [--batch-total 1024] [--no-batch]

Headline (BASELINE.json metric, first half): numeric factorization of the
north-star configuration cfg4 -- the G3_circuit-like 1258 x 1258 grid,
n = 1,582,564, 184 M filled entries, 3.8e10 MACs -- on one B200.  One step =
one refactorization of the analysed pattern with a new value set: device
scatter of A's values into the filled pattern (_kernels.py:15-34) + the
factorization kernel(s) + the pivot check.  Analysis, plan and scatter map
are built once, outside the timed region.  At N > 1 every
rank refactors its own cfg4 value sets (independent matrices, no collective
in the data path: weak scaling).

Second half of the metric ("refactorizations/s at 1/2/4/8 GPUs"): the
`batch` object -- cfg5, 1,024 same-pattern refactorizations of cfg2's
pattern sharded over the N ranks (batched launches, 16 sets per launch), the
only collective the final all-gather of (set, status, LU digest).

value = whole-job refactorizations/s from the max-over-ranks device time;
e2e = the same through the reference-facing C-ABI call with pinned host
buffers (A values in, LU values out, copies inside the timed region);
e2e_api = through factor_parallel, the reference's own Python entry point
(pageable numpy in and out).
--impl reference times the reference algorithm on the host cores (the C
restatement in oracle/; the reference itself is Python+numba that does not
travel to the GPU box), analysis included, on the same config.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import pathlib
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "numeric factorization ms/matrix (1 GPU) & refactorizations/sec at 1/2/4/8 GPUs"
CONFIG_DESC = {
    "cfg1": "synthetic circuit-like n=2,000 (2-D local, deg 4, radius 2), SuperLU MMD order",
    "cfg2": "synthetic rajat-style circuit n=100,000 + 4 dense power/ground hubs (10%), "
            "SuperLU MMD order",
    "cfg3": "synthetic ASIC_680k-like n=680,000 (1-D local +-40, 6 hubs x 1%), SuperLU MMD order",
    "cfg4": "synthetic G3_circuit-like 5-point 2-D grid 1258x1258 (n=1,582,564), geometric "
            "nested dissection",
    "g400": "G3-family 5-point grid 400x400 (n=160,000), geometric nested dissection",
    "g600": "G3-family 5-point grid 600x600 (n=360,000), geometric nested dissection",
    "g800": "G3-family 5-point grid 800x800 (n=640,000), geometric nested dissection",
}
# above this many MACs only the parallel reference paths are timed (a single
# thread takes minutes on cfg4)
BIG_MACS = 2_000_000_000


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="cfg4")
    p.add_argument("--contract", default="A", choices=["A", "B"])
    p.add_argument("--engine", default="auto", choices=["auto", "sn", "plan"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--cpu-budget", type=float, default=30.0, help="seconds of CPU baseline work")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-parity", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--batch-config", default="cfg2")
    p.add_argument("--batch-total", type=int, default=1024, help="cfg5: value sets over all ranks")
    p.add_argument("--batch-steps", type=int, default=2)
    p.add_argument("--no-batch", action="store_true")
    p.add_argument("--ref-budget", type=float, default=150.0,
                   help="reference arm: stop timing after this many seconds")
    return p.parse_args()


def init_dist(world, local):
    """One process per GPU over NCCL.  GLU_DIST_BACKEND=gloo (test only) lets
    several ranks share one GPU to exercise the multi-rank code path."""
    import torch

    ndev = max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("GLU_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    return dev


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_config(name):
    from paper_1908_00204_b200 import synthetic

    return synthetic.make(name)


def value_sets(a, seed0, count):
    """cfg5-style perturbed value sets on the pattern."""
    from paper_1908_00204_b200 import synthetic

    return [synthetic.perturb_values(a, seed0 + i) for i in range(count)]


def config_dict(name, a, nnz, levels, macs):
    """Identical in both arms (same_config)."""
    return {"workload": f"{name}: {CONFIG_DESC.get(name, '')}", "n": int(a.n), "nz": int(len(a.row_idx)),
            "nnz": int(nnz), "levels": int(levels), "macs": int(macs),
            "values": "seeded perturbed value sets (synthetic.perturb_values), one per step"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# CPU reference (oracle port of levlu's factor_parallel / left-looking)
# ---------------------------------------------------------------------------
def oracle_analysis(a):
    """The reference's analysis (symbolic_fillin, relaxed deps, levelize),
    restated in oracle/ -- the reference arm loads no product library."""
    from oracle import oracle as orc

    pat = orc.symbolic_fillin(a.n, a.col_ptr, a.row_idx)
    dp, di = orc.relaxed_deps(pat)
    level_of, lp, lc = orc.levelize(a.n, dp, di)
    return pat, lp, lc


def cpu_paths(a, pat, lp, lc, big):
    """Callables for the reference's CPU paths on this box.
    Each returns the LU values of the value set it is given."""
    from oracle import oracle as orc

    sizes = [int(x) for x in np.diff(lp)]
    ncpu = orc.cpu_count()

    def scatter(vals):
        v, bad = orc.scatter(pat, a.col_ptr, a.row_idx, vals)
        assert bad == -1
        return v

    def left(vals):
        v = scatter(vals)
        assert orc.factor_left_looking(pat, v) == -1
        return v

    def par(det, w):
        caps = orc.concurrency_caps(sizes, w, n=a.n)

        def run(vals):
            v = scatter(vals)
            assert orc.factor_parallel(pat, v, lp, lc, caps, det) == -1
            return v
        return run

    paths = {f"factor_parallel det w={ncpu}": (par(True, ncpu), ncpu)}
    if not big:
        paths.update({"left_looking w=1": (left, 1),
                      "factor_parallel det w=1": (par(True, 1), 1),
                      f"factor_parallel atomic w={ncpu}": (par(False, ncpu), ncpu)})
    return paths, ncpu


def cpu_baseline(paths, ncpu, vals, budget_s, big):
    """Best reference path on this host (value = refactorizations/s);
    returns (baseline dict, LU values of the fastest path's last run)."""
    per, last = {}, {}
    share = budget_s / len(paths)
    for name, (fn, cores) in paths.items():
        ts = []
        t_end = time.perf_counter() + share
        while not ts or (time.perf_counter() < t_end and len(ts) < 5):
            t0 = time.perf_counter()
            last[name] = fn(vals)
            ts.append(time.perf_counter() - t0)
        per[name] = {"ms": min(ts) * 1e3, "reps": len(ts), "cores": cores}
    best = min(per, key=lambda k: per[k]["ms"])
    ms = per[best]["ms"]
    skipped = " (single-thread paths not timed above 2e9 MACs)" if big else ""
    return ({"value": 1e3 / ms, "unit": "refactorizations/s", "cores": per[best]["cores"],
             "kind": "port", "ms_per_matrix": ms,
             "sample": f"full '{best}' factorizations of the bench's value set (C restatement of "
                       f"levlu, oracle/levlu_oracle.c), best of reps; paths: "
                       + ", ".join(f"{k} {v['ms']:.1f} ms x{v['reps']}" for k, v in per.items()) + skipped,
             "host_cpus": ncpu, "cpu_model": cpu_model()}, last[best])


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    t0 = time.perf_counter()
    a = load_config(args.config)
    pat, lp, lc = oracle_analysis(a)
    from oracle import oracle as orc

    macs, _ = orc.pattern_flops(pat)
    setup_s = time.perf_counter() - t0
    big = macs > BIG_MACS
    paths, ncpu = cpu_paths(a, pat, lp, lc, big)
    sets = value_sets(a, 1000, 2)
    # fastest reference path during warm-up, then K timed steps of it (time-boxed)
    best, best_t = None, float("inf")
    for name, (fn, cores) in paths.items():
        t1 = time.perf_counter()
        fn(sets[0])
        dt = time.perf_counter() - t1
        if dt < best_t:
            best, best_t = name, dt
    fn, cores = paths[best]
    for i in range(max(min(args.warmup, 2) - 1, 0)):
        fn(sets[i % 2])
    times = []
    t_all = time.perf_counter()
    for i in range(args.steps):
        t1 = time.perf_counter()
        fn(sets[i % 2])
        times.append(time.perf_counter() - t1)
        if time.perf_counter() - t_all > args.ref_budget:
            break
    ms = 1e3 * sum(times) / len(times)
    val = 1e3 / ms
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "refactorizations/s",
            "n_gpus": world, "steps": len(times), "steps_requested": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "ms_per_matrix": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, perturbed value sets)",
            "config": config_dict(args.config, a, pat.nnz, len(lp) - 1, macs),
            "setup_s": round(setup_s, 1),
            "cpu_baseline": {"value": val, "unit": "refactorizations/s", "cores": cores, "kind": "port",
                             "sample": f"{len(times)} full factorizations (of {args.steps} requested, "
                                       f"time box {args.ref_budget:.0f} s), path '{best}' (fastest of "
                                       f"{list(paths)}), C restatement of levlu; analysis by the "
                                       f"oracle's restatement of symbolic_fillin/detect_relaxed/levelize",
                             "host_cpus": ncpu, "cpu_model": cpu_model()},
            "e2e": {"value": val, "unit": "refactorizations/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, index):
        self.path = ROOT / "gpurun_out" / f"clocks_{os.getpid()}.csv"
        self.proc = None
        self.index = index

    def __enter__(self):
        try:
            self.path.parent.mkdir(exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()

    def summary(self):
        if not self.proc:
            return None
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                rows.append(parts)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def measured_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except (OSError, ValueError):
        return {}


def profiled_traffic(config, kernel):
    """DRAM bytes per launch (dram__bytes_read + write) from one ncu --set full
    capture of the kernel, recorded in profiles/traffic.json."""
    try:
        d = json.loads((ROOT / "profiles" / "traffic.json").read_text())
        return d.get(f"{config}/{kernel}")
    except (OSError, ValueError):
        return None


def l2_roof(traffic, kernel_ms):
    """L2 traffic of the kernel (ncu lts__t_sectors x 32 B, profiles/traffic.json)
    against the measured L2 read bandwidth (tools/ubench/l2bw.cu,
    profiles/l2_peak.json)."""
    try:
        peak = json.loads((ROOT / "profiles" / "l2_peak.json").read_text())["l2_read_gbs"]
    except (OSError, ValueError, KeyError):
        return None
    b = traffic.get("l2_bytes_per_launch")
    if not b or not kernel_ms:
        return {"peak_gbs": peak, "achieved_gbs": None, "frac": None}
    a = b / (kernel_ms * 1e-3) / 1e9
    return {"bytes": b, "achieved_gbs": a, "peak_gbs": peak, "frac": a / peak,
            "source": "ncu lts__t_sectors.sum x 32 B (one --set full capture) / this run's kernel time; "
                      "peak: tools/ubench/l2bw.cu"}


def max_over_ranks(x, dev, world):
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t[0])


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    dev = init_dist(world, local)
    import paper_1908_00204_b200 as glu
    from paper_1908_00204_b200 import _lib, numeric

    a = load_config(args.config)
    t0 = time.perf_counter()
    fp = glu.symbolic_fillin(a.pattern)
    s = glu.levelize(glu.detect_relaxed(fp))
    analysis_s = time.perf_counter() - t0
    macs, divs = glu.pattern_flops(fp)
    contract = _lib.CONTRACT_B if args.contract == "B" else _lib.CONTRACT_A
    engine = numeric.pick_engine(fp, contract) if args.engine == "auto" else args.engine
    t0 = time.perf_counter()
    fz = numeric.get_factorizer(fp, numeric.plan_levels(fp, s.level_of, contract), contract, engine=engine)
    setup_s = time.perf_counter() - t0
    fz.set_input(a.col_ptr, a.row_idx)
    fz.set_option(1, 0)
    fz.set_option(2, 1)
    nsets = 2
    sets = value_sets(a, 1000 + rank * nsets, nsets)
    a_dev = [torch.from_numpy(x).to(dev) for x in sets]
    v = torch.empty(fp.nnz, dtype=torch.float64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()
    thresh = 1e-14

    def step(i, ev=None):
        if ev:
            ev[0].record(stream)
        fz.scatter_device(a_dev[i % nsets], v, stream)
        fz.factor_device_async(v, thresh, stream)
        if ev:
            ev[1].record(stream)

    for i in range(args.warmup):
        flush.zero_()
        step(i)
    torch.cuda.synchronize()
    assert fz.status(stream) == -1
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    fz.set_option(8, args.steps)  # per-kernel CUDA events on the launch stream (ring of K)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with Clocks(dev.index) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 flush outside the timed events
            step(i, evs[i])
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    status = fz.status(stream)
    assert status == -1, f"pivot failure {status}"
    step_ms = [e[0].elapsed_time(e[1]) for e in evs]
    kt = np.zeros(2 * args.steps, dtype=np.float64)
    nk = _lib.lib.glu_kernel_times(fz.handle, _lib.ptr(kt), args.steps)
    main_ms = float(kt[0:2 * nk:2].mean()) if nk else None
    tail_ms = float(kt[1:2 * nk:2].mean()) if nk else None
    fz.set_option(8, 0)
    ms_step = max_over_ranks(sum(step_ms) / args.steps, dev, world)
    lu_last = v.cpu().numpy()
    last_set = (args.steps - 1) % nsets

    # parity of the last step vs the CPU oracle (rank 0) + the CPU baseline on
    # the same value set (the fastest reference path's output is the check)
    parity = cpu = None
    if rank == 0 and not (args.no_parity and args.no_cpu_baseline):
        from oracle import oracle as orc

        pat = orc.Pattern.from_fp(fp)
        lp = np.concatenate([[0], np.cumsum([len(c) for c in s.levels])]).astype(np.int64)
        lc = np.concatenate(s.levels).astype(np.int64)
        big = macs > BIG_MACS
        paths, ncpu = cpu_paths(a, pat, lp, lc, big)
        if args.no_cpu_baseline:
            ref = paths[f"factor_parallel det w={ncpu}"][0](sets[last_set])
        else:
            cpu, ref = cpu_baseline(paths, ncpu, sets[last_set], args.cpu_budget, big)
        if contract == _lib.CONTRACT_B:
            ref, bad = orc.scatter(pat, a.col_ptr, a.row_idx, sets[last_set])
            orc.factor_parallel(pat, ref, lp, lc, np.ones(len(lp) - 1, np.int64), False)
        parity = "bitwise" if np.array_equal(ref, lu_last) else \
            f"MISMATCH ({int(np.sum(ref != lu_last))} entries)"

    # e2e: the reference-facing C-ABI call with pinned host buffers
    e2e = e2e_api = None
    if not args.no_e2e:
        a_host = [torch.from_numpy(x).pin_memory() for x in sets]
        lu_host = torch.empty(fp.nnz, dtype=torch.float64).pin_memory()

        def e2e_step(i):
            rc = _lib.lib.glu_factor_host(fz.handle, ctypes.c_void_p(a_host[i % nsets].data_ptr()),
                                          ctypes.c_void_p(lu_host.data_ptr()), thresh)
            assert rc == -1, rc

        for i in range(min(args.warmup, 2)):
            e2e_step(i)
        if world > 1:
            torch.distributed.barrier()
        t1 = time.perf_counter()
        for i in range(args.steps):
            e2e_step(i)
        e2e_ms = max_over_ranks((time.perf_counter() - t1) * 1e3 / args.steps, dev, world)
        e2e = {"value": world * 1e3 / e2e_ms, "unit": "refactorizations/s", "ms_per_matrix": e2e_ms,
               "h2d_bytes_per_step": 8 * len(a.row_idx), "d2h_bytes_per_step": 8 * fp.nnz,
               "api": "glu_factor_host (C ABI, pinned host buffers): H2D A values, scatter, factor, "
                      "pivot check, D2H LU values, status read"}
        del a_host, lu_host
        # the reference's own entry point: factor_parallel with numpy (pageable) arrays
        plans = glu.plan_schedule(s, glu.level_stats(fp, s), a.n, glu.B200_RESOURCE)
        opts = glu.FactorOptions(deterministic=contract == _lib.CONTRACT_A)
        mats = [glu.CscMatrix(a.n, a.col_ptr, a.row_idx, x) for x in sets]
        os.environ["GLU_LEVEL_TIMES"] = "0"
        for i in range(2):  # warm-up in the timed loop's shape: the previous result stays alive
            lu, _ = glu.factor_parallel(mats[i % nsets], fp, s, plans, opts)
        reps = max(2, min(args.steps, 5))
        t1 = time.perf_counter()
        for i in range(reps):
            lu, _ = glu.factor_parallel(mats[i % nsets], fp, s, plans, opts)
        api_ms = max_over_ranks((time.perf_counter() - t1) * 1e3 / reps, dev, world)
        e2e_api = {"value": world * 1e3 / api_ms, "unit": "refactorizations/s", "ms_per_matrix": api_ms,
                   "steps": reps, "api": "factor_parallel(a, fp, schedule, plans, opts) -> LuFactors "
                                         "(levlu/numeric.py:241; numpy in, numpy out: LU values in "
                                         "recycled page-locked buffers, numeric._PinnedPool)"}
        del lu, mats

    batch = None
    if not args.no_batch:
        del a_dev, v, flush
        torch.cuda.empty_cache()
        batch = run_batch(args, rank, world, dev)

    if rank == 0:
        peaks = measured_peaks()
        hbm = peaks.get("hbm_gbs")
        info = fz.handle_info
        kname = "sn_kernel" if engine == "sn" else "factor_kernel"
        tail_macs = int(fz.plan_info.get("tail_macs", 0)) if engine == "plan" else 0
        t0c = int(fz.plan_info.get("tail_t0", a.n)) if engine == "plan" else a.n
        nnz_tail = int(fp.full.col_ptr[a.n] - fp.full.col_ptr[t0c])
        # SURVEY 8(d)'s per-unit figure: 16 B per MAC (target read + write) + 16 B
        # per value of the columns the kernel owns -- a no-reuse count
        bytes_survey = 16 * (macs - tail_macs) + 16 * (fp.nnz - nnz_tail)
        if engine == "sn":
            # the supernodal kernel keeps a panel's targets in registers / shared
            # memory across its sources, so the 16 B/MAC count exceeds any bandwidth
            # (frac > 1): its algorithmic bytes are the compulsory ones -- every
            # value read and written once (16 B per filled entry) and the plan read
            # once -- and its binding limit is the dependency chain (latency_floor)
            bytes_main = 16 * fp.nnz + int(fz.sn_info["plan_bytes"])
            formula = ("compulsory bytes: 16 * nnz(A_s) (every value read and written once) + the plan "
                       "(read once); SURVEY 8(d)'s 16 B/MAC no-reuse count is `survey_formula`")
        else:
            bytes_main = bytes_survey
            formula = "SURVEY 8(d): 16*MACs + 16*nnz(A_s) of the kernel's columns per launch"
        achieved = bytes_main / (main_ms * 1e-3) / 1e9 if main_ms else None
        traffic = profiled_traffic(args.config, kname) or {}
        # FP64 issue roof: every MAC is a DMUL + a DADD (no FMA: bitwise parity,
        # _kernels.py:4-6); 64 FP64 lanes per SM
        sm_mhz = peaks.get("sm_max_mhz", 1965.0)
        fp64_macs_peak = info["sms"] * 64 * sm_mhz * 1e6 / 2
        line = {
            "metric": METRIC,
            "value": world * 1e3 / ms_step,
            "unit": "refactorizations/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step,
            "ms_per_matrix": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded generator, perturbed value sets)",
            "config": config_dict(args.config, a, fp.nnz, s.level_count, macs),
            "run": {"engine": engine, "contract": args.contract, "plan": fz.plan_info,
                    "sn": getattr(fz, "sn_info", None), "device_bytes": info["device_bytes"],
                    "grid_ctas": info["grid"], "analysis_s": round(analysis_s, 2),
                    "setup_s": round(setup_s, 2), "l2": "flushed (512 MiB write) between timed steps",
                    "parallelism": f"{world} independent refactorizations (one per GPU)"},
            "parity": parity,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": (achieved / hbm) if (hbm and achieved) else None,
                         "traffic": traffic.get("bytes_per_launch"),
                         "kernel": kname, "kernel_ms": main_ms, "bytes_alg": bytes_main,
                         "formula": formula,
                         "binding": ("dependency latency: the critical path of the task graph "
                                     "(latency_floor), not bytes or FP64 issue" if engine == "sn" else
                                     "dependency latency: levels x cross-SM hand-off"),
                         "survey_formula": {"bytes": bytes_survey,
                                            "effective_gbs": bytes_survey / (main_ms * 1e-3) / 1e9
                                            if main_ms else None},
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)",
                         "traffic_source": traffic.get("source"),
                         "l2": l2_roof(traffic, main_ms)},
            "roofline_fp64": {"achieved_macs_per_s": macs / (main_ms * 1e-3) if main_ms else None,
                              "peak_macs_per_s": fp64_macs_peak,
                              "frac": macs / (main_ms * 1e-3) / fp64_macs_peak if main_ms else None,
                              "peak_source": f"derived: {info['sms']} SMs x 64 FP64 lanes x {sm_mhz:.0f} MHz "
                                             f"/ 2 instructions per MAC (DMUL + DADD, no FMA)"},
            "latency_floor": ({"model_critical_path_ms": fz.sn_info["crit_ns"] * 1e-6,
                               "frac": fz.sn_info["crit_ns"] * 1e-6 / main_ms if main_ms else None,
                               "note": "longest dependency chain of the dataflow plan under its latency "
                                       "model (2.5 us per hand-off + per-task cost, calibrated on B200 "
                                       "traces; glu_snode.cpp step 6); tools/sn_critpath.py splits the "
                                       "measured path into execution, hand-offs and warp-busy time"}
                              if engine == "sn" else None),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_api": e2e_api,
            "batch": batch,
            "clocks": clk.summary(),
            "gpu_launches": (4 + (1 if fz.sn_info["dblk"] > 0 else 0)) * args.steps if engine == "sn" else
            (3 + (1 if t0c < a.n else 0)) * args.steps,
        }
        if engine == "plan" and tail_ms:
            line["roofline_tail"] = {"kernel": "tail_kernel", "kernel_ms": tail_ms,
                                     "bytes_alg": 16 * tail_macs + 16 * nnz_tail}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_batch(args, rank, world, dev):
    """cfg5: --batch-total value sets of --batch-config's pattern sharded over
    the ranks, each rank refactoring its shard in batched launches; the
    final all-gather of (set, status, LU digest) is the only collective.
    Returns the line's `batch` object on rank 0."""
    import torch

    import paper_1908_00204_b200 as glu
    from paper_1908_00204_b200 import batch as glu_batch
    from paper_1908_00204_b200 import numeric, synthetic

    a = load_config(args.batch_config)
    fp = glu.symbolic_fillin(a.pattern)
    s = glu.levelize(glu.detect_relaxed(fp))
    macs, _ = glu.pattern_flops(fp)
    mine = list(glu_batch.shard(args.batch_total, rank, world))
    B = len(mine)
    fz = numeric.get_factorizer(fp, numeric.plan_levels(fp, None, 0), 0, tail=False)
    fz.set_input(a.col_ptr, a.row_idx)
    fz.set_option(1, 0)
    fz.set_option(2, 1)
    sets = np.stack([synthetic.perturb_values(a, 1000 + b) for b in mine]) if B else \
        np.zeros((0, len(a.row_idx)))
    a_dev = torch.from_numpy(sets).to(dev)
    v = torch.empty((max(B, 1), fp.nnz), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        for b in range(B):
            fz.scatter_device(a_dev[b], v[b], stream)
        return fz.factor_batch_device(v[:B], 1e-14, stream) if B else np.zeros(0, np.int64)

    assert np.all(step() == -1)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.batch_steps):
        fails = step()  # status read per step (synchronizes: part of the API)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.batch_steps, dev, world)
    digests = [glu_batch.set_digest(v[b].cpu().numpy()) for b in range(B)]
    if world > 1:
        idx, status, dg = glu_batch.gather_results(mine, fails.tolist(), digests)
    else:
        idx, status, dg = np.array(mine), np.asarray(fails), np.array(digests)
    out = None
    if rank == 0:
        from oracle import oracle as orc

        pat = orc.Pattern.from_fp(fp)
        checked = []
        for b in sorted({0, args.batch_total - 1}):
            ref, _ = orc.scatter(pat, a.col_ptr, a.row_idx, synthetic.perturb_values(a, 1000 + b))
            orc.factor_left_looking(pat, ref)
            checked.append(glu_batch.set_digest(ref) == int(dg[list(idx).index(b)]))
        # CPU throughput ceiling: nproc independent single-thread factorizations
        ref, _ = orc.scatter(pat, a.col_ptr, a.row_idx, sets[0] if B else a.values)
        t1 = time.perf_counter()
        orc.factor_left_looking(pat, ref)
        t_one = time.perf_counter() - t1
        ncpu = orc.cpu_count()
        out = {"workload": f"cfg5: {args.batch_total} same-pattern refactorizations of "
                           f"{args.batch_config} ({CONFIG_DESC.get(args.batch_config, '')}), perturbed "
                           f"value sets, sharded over {world} GPU(s)",
               "value": args.batch_total * 1e3 / ms, "unit": "refactorizations/s",
               "ms_per_step": ms, "ms_per_matrix_per_gpu": ms / max(len(mine), 1),
               "steps": args.batch_steps, "sets_per_gpu": B, "n_gpus": world,
               "scaling": "strong (fixed 1,024 sets)", "statuses_ok": bool(np.all(np.asarray(status) == -1)),
               "gathered_sets": int(len(idx)),
               "parity": "bitwise (digest of sets 0 and last vs oracle)" if all(checked) else "MISMATCH",
               "n": a.n, "nnz": fp.nnz, "macs": macs,
               "launches_per_step": B + (B + 15) // 16 * 2 if B else 0,
               "cpu_ceiling": {"value": ncpu / t_one, "unit": "refactorizations/s",
                               "sample": f"{ncpu} x one single-thread left-looking factorization "
                                         f"({t_one * 1e3:.1f} ms), perfect scaling assumed"}}
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
