"""cProfile of the reference-facing path (factor_parallel with numpy in and
out) on one config: where the host time goes around the kernel.

    python tools/api_profile.py cfg4 [--reps 3]
"""
import cProfile
import pathlib
import pstats
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    import paper_1908_00204_b200 as glu
    from paper_1908_00204_b200 import synthetic

    a = synthetic.make(name)
    fp = glu.symbolic_fillin(a.pattern)
    s = glu.levelize(glu.detect_relaxed(fp))
    plans = glu.plan_schedule(s, glu.level_stats(fp, s), a.n, glu.B200_RESOURCE)
    opts = glu.FactorOptions(deterministic=True)
    mats = [glu.CscMatrix(a.n, a.col_ptr, a.row_idx, synthetic.perturb_values(a, seed=k)) for k in range(2)]
    glu.factor_parallel(mats[0], fp, s, plans, opts)  # setup + warm pool
    glu.factor_parallel(mats[1], fp, s, plans, opts)
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    for i in range(reps):
        lu, st = glu.factor_parallel(mats[i % 2], fp, s, plans, opts)
        del lu
    pr.disable()
    print(f"{name}: factor_parallel {(time.perf_counter() - t0) * 1e3 / reps:.1f} ms per call (under cProfile)")
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)


if __name__ == "__main__":
    main()
