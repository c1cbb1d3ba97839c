"""Supernodal engine vs the CPU oracle on one config: where do the values
differ (column, row, panel, width)?  Diagnostics only.

    python tools/sn_debug.py cfg1
"""
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import torch  # noqa: F401

    import paper_1908_00204_b200 as glu
    from paper_1908_00204_b200 import numeric, synthetic
    import sn_emul
    from oracle import oracle as orc

    name = sys.argv[1]
    a = synthetic.make(name) if name in synthetic.CONFIGS else synthetic.grid5(int(name[1:]), seed=0)
    fp = glu.symbolic_fillin(a.pattern)
    pat = orc.Pattern.from_fp(fp)
    ref, bad = orc.scatter(pat, a.col_ptr, a.row_idx, a.values)
    assert orc.factor_left_looking(pat, ref, 1e-14) == -1
    lv = numeric._relaxed_levels(fp)
    fz = numeric.Factorizer(fp, lv, 0, engine="sn")
    fz.set_input(a.col_ptr, a.row_idx)
    fz.set_option(1, 0)
    fz.set_option(2, 1)
    plan = sn_emul.build(fp)
    pan = plan["pan"]
    pan_of = np.zeros(fp.n, dtype=np.int64)
    for p in range(len(pan)):
        pan_of[pan[p, 0]:pan[p, 1]] = p
    cols = np.repeat(np.arange(fp.n), np.diff(fp.full.col_ptr))
    rows = fp.full.row_idx
    for rep in range(3):
        vals, rc = fz.factor_host(a.values, 1e-14)
        d = np.flatnonzero(vals != ref)
        print(f"rep {rep}: rc {rc}, {len(d)} differing slots of {fp.nnz}")
        for q in d[:12]:
            c, r = int(cols[q]), int(rows[q])
            p = int(pan_of[c])
            print(f"  slot {q} col {c} row {r} {'U' if r < c else ('D' if r == c else 'L')} panel {p} "
                  f"[{pan[p, 0]},{pan[p, 1]}) row-panel {int(pan_of[r])} got {vals[q]!r} ref {ref[q]!r}")
        if len(d):
            first = int(cols[d].min())
            print("  first differing column", first, "panel", int(pan_of[first]),
                  "width", int(pan[pan_of[first], 1] - pan[pan_of[first], 0]))


if __name__ == "__main__":
    main()
