"""Benchmark: GLU3.0 numeric (re)factorization on the B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2]
                    [--contract B|A] [--impl ours|reference]

One step = one numeric refactorization of the configuration's pattern on
every GPU: device scatter of A's new values into the filled pattern
(_kernels.py:15-34) + the persistent level kernel (factor + pivot check +
divide).  Pattern analysis, plan and scatter map are built once, outside
the timed region.  N > 1 (torchrun): every rank refactors
its own value sets -- independent matrices, no collective in the data path
(weak scaling); the only collective is the final all-gather of per-rank
checksums after the timed region.

value = whole-job refactorizations/s (max-over-ranks device time); e2e = the
same through the reference-facing C-ABI call with host buffers (pinned A
values in, LU values out, copies inside the timed region).
--impl reference times the reference algorithm on the host cores (the C
restatement in oracle/, the reference itself being Python+numba that does
not travel to the GPU box).
"""

from __future__ import annotations

import argparse
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
    "g400": "G3-family 5-point grid 400x400 (n=160,000), geometric nested dissection",
    "g600": "G3-family 5-point grid 600x600 (n=360,000), geometric nested dissection",
    "g800": "G3-family 5-point grid 800x800 (n=640,000), geometric nested dissection",
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="cfg2")
    p.add_argument("--contract", default="B", choices=["A", "B"])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU baseline work")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--batch", type=int, default=0,
                   help="cfg5-style: value sets per GPU per step, factored by batched launches")
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


def analyze(a):
    import paper_1908_00204_b200 as glu

    fp = glu.symbolic_fillin(a.pattern)
    s = glu.levelize(glu.detect_relaxed(fp))
    return fp, s


def value_sets(a, rank, count):
    """cfg5-style perturbed value sets on the pattern, distinct per rank."""
    from paper_1908_00204_b200 import synthetic

    return [synthetic.perturb_values(a, 1000 + rank * count + i) for i in range(count)]


def level_arrays(s):
    lp = np.concatenate([[0], np.cumsum([len(c) for c in s.levels])]).astype(np.int64)
    return lp, np.concatenate(s.levels).astype(np.int64)


# ---------------------------------------------------------------------------
# CPU reference (oracle port of levlu's factor_parallel / left-looking)
# ---------------------------------------------------------------------------
def cpu_paths(a, fp, s):
    """Callables for the reference's CPU paths on this box."""
    from oracle import oracle as orc

    pat = orc.Pattern.from_fp(fp)
    lp, lc = level_arrays(s)
    sizes = [int(x) for x in np.diff(lp)]
    ncpu = orc.cpu_count()

    def scatter():
        v, bad = orc.scatter(pat, a.col_ptr, a.row_idx, a.values)
        assert bad == -1
        return v

    def left():
        v = scatter()
        assert orc.factor_left_looking(pat, v) == -1
        return v

    def par(det, w):
        caps = orc.concurrency_caps(sizes, w, n=a.n)

        def run():
            v = scatter()
            assert orc.factor_parallel(pat, v, lp, lc, caps, det) == -1
            return v
        return run

    paths = {"left_looking w=1": (left, 1),
             "factor_parallel det w=1": (par(True, 1), 1),
             f"factor_parallel det w={ncpu}": (par(True, ncpu), ncpu),
             f"factor_parallel atomic w={ncpu}": (par(False, ncpu), ncpu)}
    return paths, ncpu


def time_cpu(fn, budget_s, min_reps=1):
    ts = []
    t_end = time.perf_counter() + budget_s
    while len(ts) < min_reps or (time.perf_counter() < t_end and len(ts) < 5):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts), len(ts)


def cpu_baseline(a, fp, s, budget_s):
    paths, ncpu = cpu_paths(a, fp, s)
    per = {}
    share = budget_s / len(paths)
    for name, (fn, cores) in paths.items():
        fn()  # warm
        best, reps = time_cpu(fn, share)
        per[name] = {"ms": best * 1e3, "reps": reps, "cores": cores}
    best_name = min(per, key=lambda k: per[k]["ms"])
    ms = per[best_name]["ms"]
    return {"value": 1e3 / ms, "unit": "refactorizations/s", "cores": per[best_name]["cores"],
            "kind": "port", "ms_per_matrix": ms,
            "sample": f"full {best_name} factorizations of the same matrix (C restatement of "
                      f"levlu, oracle/levlu_oracle.c), best of reps; all paths: "
                      + ", ".join(f"{k} {v['ms']:.1f} ms" for k, v in per.items()),
            "host_cpus": ncpu, "cpu_model": cpu_model()}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    a = load_config(args.config)
    fp, s = analyze(a)
    paths, ncpu = cpu_paths(a, fp, s)
    # pick the fastest reference path during warm-up, then time K steps of it
    best, best_t = None, float("inf")
    for name, (fn, cores) in paths.items():
        t0 = time.perf_counter()
        fn()
        dt = time.perf_counter() - t0
        if dt < best_t:
            best, best_t = name, dt
    fn, cores = paths[best]
    for _ in range(max(args.warmup - 1, 0)):
        fn()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fn()
    el = time.perf_counter() - t0
    ms = el * 1e3 / args.steps
    val = 1e3 / ms
    import paper_1908_00204_b200 as glu

    macs, divs = glu.pattern_flops(fp)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "refactorizations/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "ms_per_matrix": ms,
            "config": {"workload": f"{args.config}: {CONFIG_DESC.get(args.config, '')}",
                       "n": a.n, "nnz": fp.nnz, "levels": s.level_count, "macs": macs},
            "cpu_baseline": {"value": val, "unit": "refactorizations/s", "cores": cores,
                             "kind": "port", "sample": f"{args.steps} full factorizations, path "
                             f"'{best}' (fastest of {list(paths)}), C restatement of levlu",
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


def profiled_traffic(config, contract):
    """DRAM bytes per launch (dram__bytes_read + write) from one ncu --set full
    capture per kernel, recorded in profiles/traffic.json."""
    try:
        d = json.loads((ROOT / "profiles" / "traffic.json").read_text())
        return d.get(f"{config}/{contract}")
    except (OSError, ValueError):
        return None


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    dev = init_dist(world, local)
    import paper_1908_00204_b200 as glu

    a = load_config(args.config)
    fp, s = analyze(a)
    macs, divs = glu.pattern_flops(fp)
    contract = 1 if args.contract == "B" else 0
    t0 = time.perf_counter()
    fz = glu.Factorizer(fp, s.level_of, contract)
    setup_s = time.perf_counter() - t0
    fz.set_input(a.col_ptr, a.row_idx)
    fz.set_option(1, 0)
    nsets = 4
    sets = value_sets(a, rank, nsets)
    a_dev = [torch.from_numpy(x).to(dev) for x in sets]
    v = torch.empty(fp.nnz, dtype=torch.float64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()
    thresh = 1e-14

    def step(i, ev=None):
        if ev:
            ev[0].record(stream)
        fz.scatter_device(a_dev[i % nsets], v, stream)
        if ev:
            ev[1].record(stream)
        fz.factor_device_async(v, thresh, stream)
        if ev:
            ev[2].record(stream)

    for i in range(args.warmup):
        flush.zero_()
        step(i)
    torch.cuda.synchronize()
    assert fz.status(stream) == -1
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
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
    step_ms = [e[0].elapsed_time(e[2]) for e in evs]
    fac_ms = [e[1].elapsed_time(e[2]) for e in evs]
    from paper_1908_00204_b200 import _lib
    kt = np.zeros(2 * args.steps, dtype=np.float64)
    nk = _lib.lib.glu_kernel_times(fz.handle, _lib.ptr(kt), args.steps)
    main_ms = float(kt[0:2 * nk:2].mean()) if nk else None
    tail_ms = float(kt[1:2 * nk:2].mean()) if nk else None
    fz.set_option(8, 0)
    tot = torch.tensor([sum(step_ms), sum(fac_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(tot, op=torch.distributed.ReduceOp.MAX)
    ms_step = float(tot[0]) / args.steps
    ms_fac = float(tot[1]) / args.steps

    # parity spot check of the last step vs the CPU oracle (rank 0), and the
    # final gather of per-rank checksums (the only collective)
    lu_last = v.cpu().numpy()
    from paper_1908_00204_b200 import batch as glu_batch

    last_set = rank * nsets + (args.steps - 1) % nsets  # global value-set id
    if world > 1:  # (set id, status, LU checksum) of every rank: the only collective
        glu_batch.gather_results([last_set], [fz.status(stream)], [glu_batch.set_digest(lu_last)])
    parity = None
    cpu = None
    if rank == 0:
        from oracle import oracle as orc

        pat = orc.Pattern.from_fp(fp)
        ref, bad = orc.scatter(pat, a.col_ptr, a.row_idx, sets[(args.steps - 1) % nsets])
        lp, lc = level_arrays(s)
        orc.factor_parallel(pat, ref, lp, lc, np.ones(len(lp) - 1, np.int64), contract == 0)
        parity = "bitwise" if np.array_equal(ref, lu_last) else "MISMATCH"
        if not args.no_cpu_baseline:
            cpu = cpu_baseline(a, fp, s, args.cpu_budget)

    # e2e through the host-buffer C-ABI call (pinned buffers)
    a_host = [torch.from_numpy(x).pin_memory() for x in sets]
    lu_host = torch.empty(fp.nnz, dtype=torch.float64).pin_memory()
    from paper_1908_00204_b200 import _lib
    import ctypes

    def e2e_step(i):
        rc = _lib.lib.glu_factor_host(fz.handle, ctypes.c_void_p(a_host[i % nsets].data_ptr()),
                                      ctypes.c_void_p(lu_host.data_ptr()), thresh)
        assert rc == -1, rc

    for i in range(args.warmup):
        e2e_step(i)
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        e2e_step(i)
    e2e_s = time.perf_counter() - t0
    e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(e2e_t, op=torch.distributed.ReduceOp.MAX)
    e2e_ms = float(e2e_t[0]) * 1e3 / args.steps

    if rank == 0:
        peaks = measured_peaks()
        hbm = peaks.get("hbm_gbs")
        # algorithmic bytes per launch: 16 B per MAC (target read +
        # write, L and multiplier in registers) + 16 B per value of the columns
        # the kernel owns; the dense tail's MACs belong to tail_kernel
        tail_macs = int(fz.plan_info.get("tail_macs", 0))
        t0c = int(fz.plan_info.get("tail_t0", a.n))
        nnz_tail = int(fp.full.col_ptr[a.n] - fp.full.col_ptr[t0c])
        bytes_main = 16 * (macs - tail_macs) + 16 * (fp.nnz - nnz_tail)
        bytes_tail = 16 * tail_macs + 16 * nnz_tail
        achieved = bytes_main / (main_ms * 1e-3) / 1e9
        traffic = profiled_traffic(args.config, args.contract) or {}
        info = fz.handle_info
        line = {
            "metric": METRIC,
            "value": world * 1e3 / ms_step,
            "unit": "refactorizations/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step,
            "ms_per_matrix": ms_step,
            "factor_kernel_ms": ms_fac,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded generator, perturbed value sets)",
            "config": {"workload": f"{args.config}: {CONFIG_DESC.get(args.config, '')}",
                       "n": a.n, "nz": a.nnz, "nnz": fp.nnz, "levels": s.level_count,
                       "macs": macs, "contract": args.contract,
                       "plan": fz.plan_info, "grid_ctas": info["grid"],
                       "threads_per_cta": info["threads"], "setup_s": round(setup_s, 3),
                       "l2": "flushed (512 MiB write) between timed steps",
                       "parallelism": f"{world} independent refactorizations (one per GPU)"},
            "parity": parity,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": (achieved / hbm) if hbm else None,
                         "traffic": traffic.get("factor_kernel"),
                         "kernel": "factor_kernel", "kernel_ms": main_ms,
                         "bytes_alg": bytes_main,
                         "formula": "16*(MACs - tail MACs) + 16*nnz(A_s outside the tail) per launch",
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)",
                         "traffic_source": traffic.get("source")},
            "roofline_tail": ({"kernel": "tail_kernel", "kernel_ms": tail_ms, "bytes_alg": bytes_tail,
                               "achieved": bytes_tail / (tail_ms * 1e-3) / 1e9, "unit": "GB/s",
                               "frac": bytes_tail / (tail_ms * 1e-3) / 1e9 / hbm if hbm else None,
                               "traffic": traffic.get("tail_kernel"), "tail_columns": a.n - t0c,
                               "tail_macs": tail_macs} if tail_ms else None),
            "cpu_baseline": cpu,
            "e2e": {"value": world * 1e3 / e2e_ms, "unit": "refactorizations/s",
                    "ms_per_matrix": e2e_ms,
                    "h2d_bytes_per_step": 8 * a.nnz, "d2h_bytes_per_step": 8 * fp.nnz,
                    "api": "glu_factor_host (C ABI, pinned host buffers)"},
            "clocks": clk.summary(),
            "gpu_launches": (3 + (1 if fz.plan_info.get("tail_t0", a.n) < a.n else 0)) * args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_batch(args):
    """cfg5-style throughput: each step, every rank refactors its shard of
    `--batch` value sets of the configuration's pattern through batched
    launches (up to 8 sets per launch share each item's plan loads,
    dependency wait and release).  value = whole-job refactorizations/s."""
    import torch

    rank, world, local = dist_env()
    dev = init_dist(world, local)
    import paper_1908_00204_b200 as glu
    from paper_1908_00204_b200 import batch as glu_batch

    a = load_config(args.config)
    fp, s = analyze(a)
    macs, _ = glu.pattern_flops(fp)
    contract = 1 if args.contract == "B" else 0
    fz = glu.Factorizer(fp, s.level_of, contract, max_item_macs=64)  # dense tail: one cluster per set
    fz.set_input(a.col_ptr, a.row_idx)
    B = args.batch
    sets = np.stack(value_sets(a, rank, B))
    a_dev = torch.from_numpy(sets).to(dev)
    v = torch.empty((B, fp.nnz), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        for b in range(B):
            fz.scatter_device(a_dev[b], v[b], stream)
        return fz.factor_batch_device(v, 1e-14, stream)

    for _ in range(args.warmup):
        assert np.all(step() == -1)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(dev.index) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            fails = step()  # status read per step (synchronizes: part of the API)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(ms, op=torch.distributed.ReduceOp.MAX)
    ms = float(ms[0])
    digests = [glu_batch.set_digest(v[b].cpu().numpy()) for b in range(B)]
    idx = list(range(rank * B, rank * B + B))
    if world > 1:
        glu_batch.gather_results(idx, fails.tolist(), digests)
    parity = None
    if rank == 0:
        from oracle import oracle as orc

        pat = orc.Pattern.from_fp(fp)
        lp, lc = level_arrays(s)
        ref, _ = orc.scatter(pat, a.col_ptr, a.row_idx, sets[B - 1])
        orc.factor_parallel(pat, ref, lp, lc, np.ones(len(lp) - 1, np.int64), contract == 0)
        parity = "bitwise" if np.array_equal(ref, v[B - 1].cpu().numpy()) else "MISMATCH"
        line = {"metric": METRIC, "value": world * B * 1e3 / ms, "unit": "refactorizations/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "ms_per_matrix": ms / B, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded generator, perturbed value sets)",
                "config": {"workload": f"cfg5-style batch of {B} value sets per GPU on "
                                       f"{args.config}'s pattern",
                           "n": a.n, "nnz": fp.nnz, "levels": s.level_count, "macs": macs,
                           "contract": args.contract, "batch_per_gpu": B,
                           "launches_per_step": (B + 7) // 8,
                           "parallelism": f"{world} ranks x {B} independent value sets"},
                "parity": parity, "clocks": clk.summary(),
                "gpu_launches": args.steps * (2 * B + (B + 7) // 8)}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.batch > 0:
        run_batch(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
