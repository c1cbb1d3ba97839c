"""Command-line harness for the B200 path.

    python -m paper_1908_00204_b200 factor MATRIX.mtx [--sequential left|right | --parallel]
        [--atomic] [--threads T] [--deps relaxed|upward [--allow-unsafe]] [--detect-races]
        [--perm P | --row-perm R --col-perm C] [--check-residual] [--stats-out R.json|R.csv]
    python -m paper_1908_00204_b200 solve MATRIX.mtx RHS.txt [--out x.txt]
    python -m paper_1908_00204_b200 deps-compare MATRIX.mtx [--csv PATH|-]
    python -m paper_1908_00204_b200 level-stats MATRIX.mtx [--deps D] [--warps W]

Mirrors `levlu` (levlu/cli.py:69-359): same subcommands and flags, same
report lines, the same `checksum` line (first 16 hex digits of sha256 over
the LU values, levlu/cli.py:201) -- identical to the reference's because
the factors are bit-identical -- the same RunReport JSON/CSV, the same
deps-compare / level-stats CSV, and the same exit codes (0 ok, 1 usage or
I/O error, 2 pivot breakdown, 3 schedule hazard; levlu/cli.py:23-26).  The
numeric work runs on the B200 through the package API; there is no CPU
path.  Differences: the deps line adds `device=cuda`; `--precision single`
factors fp32 values in fp64 arithmetic and rounds the factors to fp32
(numeric._value_dtype).
"""

from __future__ import annotations

import argparse
import csv
import hashlib
import json
import sys
import time
from collections import Counter
from dataclasses import asdict, dataclass, field

import numpy as np

from . import depgraph, numeric, resource, sparse, symbolic

EXIT_OK, EXIT_USAGE, EXIT_PIVOT, EXIT_HAZARD = 0, 1, 2, 3

_DETECTORS = {"upward": depgraph.detect_upward, "exact": depgraph.detect_double_u_exact,
              "relaxed": depgraph.detect_relaxed}


class CliError(Exception):
    def __init__(self, msg, code=EXIT_USAGE):
        super().__init__(msg)
        self.code = code


@dataclass
class RunReport:
    """Per-run record written by --stats-out (levlu/cli.py:29-60)."""

    matrix: str
    n: int
    nz: int
    nnz: int
    deps_method: str
    level_count: int
    times: dict = field(default_factory=dict)
    residual: float | None = None
    mode_histogram: dict = field(default_factory=dict)
    workers: int = 1
    device: str = "cuda"

    def write(self, path: str) -> None:
        if path.endswith(".json"):
            with open(path, "w") as fh:
                json.dump(asdict(self), fh, indent=2)
                fh.write("\n")
        elif path.endswith(".csv"):
            row = {k: getattr(self, k) for k in
                   ("matrix", "n", "nz", "nnz", "deps_method", "level_count")}
            row.update({f"time_{k}_s": v for k, v in self.times.items()})
            row.update({"residual": "" if self.residual is None else self.residual,
                        "workers": self.workers, "device": self.device})
            with open(path, "w", newline="") as fh:
                w = csv.DictWriter(fh, fieldnames=list(row))
                w.writeheader()
                w.writerow(row)
        else:
            raise CliError("--stats-out must end in .csv or .json")


def _read_perm(path: str, n: int) -> sparse.Permutation:
    try:
        with open(path) as fh:
            return sparse.load_permutation(fh, n)
    except OSError as e:
        raise CliError(f"cannot read permutation: {e}")
    except ValueError as e:
        raise CliError(f"{path}: {e}")


def _load_matrix(args) -> sparse.CscMatrix:
    dtype = np.float32 if getattr(args, "precision", "double") == "single" else np.float64
    try:
        with open(args.matrix) as fh:
            a = sparse.to_csc(sparse.load_matrix_market(fh), dtype=dtype)
    except OSError as e:
        raise CliError(f"cannot read {args.matrix}: {e}")
    except (sparse.MatrixFormatError, ValueError) as e:
        raise CliError(f"{args.matrix}: {e}")
    perm, rperm, cperm = (getattr(args, k, None) for k in ("perm", "row_perm", "col_perm"))
    if perm and (rperm or cperm):
        raise CliError("--perm conflicts with --row-perm/--col-perm")
    if perm:
        p = _read_perm(perm, a.n)
        a = sparse.permute(a, p, p)
    elif rperm or cperm:
        if not (rperm and cperm):
            raise CliError("--row-perm and --col-perm must be given together")
        a = sparse.permute(a, _read_perm(rperm, a.n), _read_perm(cperm, a.n))
    return a


def _resource_model(args) -> resource.ResourceModel:
    return resource.ResourceModel(total_warps=args.warps, stream_threshold=args.stream_threshold,
                                  memory_budget_bytes=args.mem_budget,
                                  scalar_size_bytes=4 if getattr(args, "precision", "double") == "single" else 8)


def _analyze(a, method: str):
    t0 = time.perf_counter()
    fp = symbolic.symbolic_fillin(a.pattern)
    t1 = time.perf_counter()
    graph = _DETECTORS[method](fp)
    t2 = time.perf_counter()
    schedule = depgraph.levelize(graph)
    t3 = time.perf_counter()
    return fp, schedule, {"symbolic": t1 - t0, "detection": t2 - t1, "levelization": t3 - t2}


def cmd_factor(args) -> int:
    if args.sequential and args.parallel:
        raise CliError("--sequential and --parallel are mutually exclusive")
    if not args.sequential:
        args.parallel = True
    if args.parallel and args.deps == "upward" and not args.allow_unsafe:
        raise CliError("--deps upward with --parallel requires --allow-unsafe")
    a = _load_matrix(args)
    fp, schedule, times = _analyze(a, args.deps)
    rm = _resource_model(args)
    plans = resource.plan_schedule(schedule, depgraph.level_stats(fp, schedule), a.n, rm)
    opts = numeric.FactorOptions(deterministic=args.deterministic, worker_count=args.threads,
                                 resource=rm, detect_races=args.detect_races)
    modes: Counter = Counter()
    t0 = time.perf_counter()
    try:
        if args.sequential == "left":
            lu = numeric.factor_left_looking(a, fp, opts)
        elif args.sequential == "right":
            lu = numeric.factor_right_looking_seq(a, fp, opts)
        else:
            lu, stats = numeric.factor_parallel(a, fp, schedule, plans, opts)
            modes = Counter(stats.level_modes)
    except numeric.PivotError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_PIVOT
    except numeric.ScheduleHazardError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_HAZARD
    times["numeric"] = time.perf_counter() - t0
    res = numeric.residual(a, lu) if args.check_residual else None
    report = RunReport(matrix=args.matrix, n=a.n, nz=fp.nz_before, nnz=fp.nnz,
                       deps_method=args.deps, level_count=schedule.level_count, times=times,
                       residual=res, mode_histogram=dict(sorted(modes.items())),
                       workers=args.threads if args.parallel else 1)
    checksum = hashlib.sha256(np.ascontiguousarray(lu.values).tobytes()).hexdigest()[:16]
    cpu_time = times["symbolic"] + times["detection"] + times["levelization"]
    print(f"matrix {args.matrix}: n={a.n} nz={fp.nz_before} nnz={fp.nnz}")
    print(f"deps={args.deps} levels={schedule.level_count} workers={report.workers} device=cuda")
    print(f"cpu-phase time {cpu_time * 1e3:.3f} ms, numeric time {times['numeric'] * 1e3:.3f} ms")
    if modes:
        print("modes: " + ", ".join(f"{m}={c}" for m, c in sorted(modes.items())))
    if res is not None:
        print(f"residual {res:.3e}")
    print(f"checksum {checksum}")
    if args.stats_out:
        report.write(args.stats_out)
    return EXIT_OK


def cmd_solve(args) -> int:
    a = _load_matrix(args)
    try:
        b = np.loadtxt(args.rhs, dtype=a.values.dtype, ndmin=1)
    except OSError as e:
        raise CliError(f"cannot read {args.rhs}: {e}")
    except ValueError as e:
        raise CliError(f"{args.rhs}: {e}")
    if len(b) != a.n:
        raise CliError(f"rhs has {len(b)} entries, expected {a.n}")
    fp, schedule, _ = _analyze(a, args.deps)
    rm = _resource_model(args)
    plans = resource.plan_schedule(schedule, depgraph.level_stats(fp, schedule), a.n, rm)
    try:
        lu, _ = numeric.factor_parallel(a, fp, schedule, plans,
                                        numeric.FactorOptions(worker_count=args.threads,
                                                              resource=rm))
        x = numeric.solve(lu, b)
    except numeric.PivotError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_PIVOT
    np.savetxt(args.out, x)
    cols = np.repeat(np.arange(a.n), np.diff(a.col_ptr))
    r = np.bincount(a.row_idx, weights=a.values * x[cols], minlength=a.n) - b
    scale = np.abs(b).max() if len(b) else 0.0
    res = float(np.abs(r).max() / scale) if scale else float(np.abs(r).max(initial=0.0))
    print(f"wrote {args.out}")
    print(f"residual {res:.3e}")
    return EXIT_OK


def cmd_deps_compare(args) -> int:
    """The three detectors side by side (levlu/cli.py:237-264): edges,
    levels, time; the upward <= exact <= relaxed edge-set ordering is
    checked (exit 3 if violated)."""
    a = _load_matrix(args)
    fp = symbolic.symbolic_fillin(a.pattern)
    results = []
    for name in ("upward", "exact", "relaxed"):
        t0 = time.perf_counter()
        graph = _DETECTORS[name](fp)
        dt = time.perf_counter() - t0
        results.append((name, graph, depgraph.levelize(graph).level_count, dt))
    edges = {name: g.edge_set() for name, g, _, _ in results}
    if not (edges["upward"] <= edges["exact"] <= edges["relaxed"]):
        print("error: detector superset ordering violated", file=sys.stderr)
        return EXIT_HAZARD
    for name, g, levels, dt in results:
        print(f"{name:8s} edges={g.edge_count:8d} levels={levels:6d} time={dt * 1e3:.3f} ms")
    if args.csv:
        out = sys.stdout if args.csv == "-" else open(args.csv, "w")
        try:
            out.write("method,edges,levels\n")
            for name, g, levels, _ in results:
                out.write(f"{name},{g.edge_count},{levels}\n")
        finally:
            if out is not sys.stdout:
                out.close()
    return EXIT_OK


def cmd_level_stats(args) -> int:
    """Per-level size, max subcolumns and kernel mode as CSV (levlu/cli.py:
    267-279), modes from plan_schedule under the given resource model."""
    a = _load_matrix(args)
    fp, schedule, _ = _analyze(a, args.deps)
    st = depgraph.level_stats(fp, schedule)
    resource.plan_schedule(schedule, st, a.n, _resource_model(args))
    out = sys.stdout
    out.write("level,size,max_subcolumns,mode\n")
    for lvl in range(st.level_count):
        out.write(f"{lvl},{st.sizes[lvl]},{st.max_subcolumns[lvl]},{st.modes[lvl]}\n")
    return EXIT_OK


def _add_common(p: argparse.ArgumentParser) -> None:
    p.add_argument("matrix", help="Matrix Market coordinate file")
    p.add_argument("--deps", choices=sorted(_DETECTORS), default="relaxed")
    p.add_argument("--threads", type=int, default=1)
    p.add_argument("--warps", type=int, default=96)
    p.add_argument("--stream-threshold", type=int, default=16)
    p.add_argument("--mem-budget", type=int, default=1 << 30)
    p.add_argument("--precision", choices=["single", "double"], default="double")
    p.add_argument("--device", choices=["cuda"], default="cuda")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1908_00204_b200", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("factor", help="factorize a matrix on the B200 and report")
    _add_common(p)
    p.add_argument("--perm", help="symmetric permutation file (one 0-based index per line)")
    p.add_argument("--row-perm", help="row permutation file")
    p.add_argument("--col-perm", help="column permutation file")
    p.add_argument("--sequential", choices=["left", "right"])
    p.add_argument("--parallel", action="store_true")
    p.add_argument("--deterministic", action="store_true", default=True)
    p.add_argument("--atomic", dest="deterministic", action="store_false",
                   help="level-major (atomic-mode) accumulation order")
    p.add_argument("--check-residual", action="store_true")
    p.add_argument("--detect-races", action="store_true")
    p.add_argument("--allow-unsafe", action="store_true")
    p.add_argument("--stats-out", help="write the run report to PATH.csv or PATH.json")
    p.set_defaults(func=cmd_factor)
    p = sub.add_parser("solve", help="factor and solve A x = b on the B200")
    _add_common(p)
    p.add_argument("rhs", help="right-hand side, one scalar per line")
    p.add_argument("--out", default="x.txt", help="solution output file")
    p.set_defaults(func=cmd_solve)
    p = sub.add_parser("deps-compare", help="compare the three dependency detectors")
    p.add_argument("matrix", help="Matrix Market coordinate file")
    p.add_argument("--perm", help="symmetric permutation file (one 0-based index per line)")
    p.add_argument("--row-perm", help="row permutation file")
    p.add_argument("--col-perm", help="column permutation file")
    p.add_argument("--precision", choices=["single", "double"], default="double")
    p.add_argument("--csv", help="write method,edges,levels CSV to PATH ('-' for stdout)")
    p.set_defaults(func=cmd_deps_compare)
    p = sub.add_parser("level-stats", help="emit per-level statistics as CSV")
    _add_common(p)
    p.add_argument("--perm", help="symmetric permutation file (one 0-based index per line)")
    p.add_argument("--row-perm", help="row permutation file")
    p.add_argument("--col-perm", help="column permutation file")
    p.set_defaults(func=cmd_level_stats)
    return ap


def main(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as e:  # argparse exits 2, which here would read as a pivot failure
        return EXIT_OK if e.code == 0 else EXIT_USAGE
    try:
        return args.func(args)
    except CliError as e:
        print(f"error: {e}", file=sys.stderr)
        return e.code
    except (symbolic.SymbolicError, numeric.PatternMismatchError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
