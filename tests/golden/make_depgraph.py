"""Goldens for the reference's debugging detectors, by running the REFERENCE:
detect_double_u_exact (levlu/depgraph.py:129-156) and simulate_hazards
(:173-205) under the upward and relaxed schedules.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_depgraph.py

Writes tests/golden/depgraph/<case>.npz (inputs are the existing
tests/golden/<case>.npz matrices).
"""

from __future__ import annotations

import os
import pathlib
import sys

import numpy as np

REF = pathlib.Path("/root/reference/pkg/src")
HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import levlu as lv  # noqa: E402  (the reference)

CASES = ["conflict8", "random_dd_s1_n40", "random_dd_s2_n80", "random_dd_s3_n120", "random_dd_s5_n100",
         "block_arrow_4x24", "banded_n200", "cfg1"]


def csr_of(g):
    lens = np.array([len(d) for d in g.deps], dtype=np.int64)
    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = np.concatenate(g.deps).astype(np.int64) if ptr[-1] else np.empty(0, np.int64)
    return ptr, idx


def hazards(fp, s):
    rep = lv.simulate_hazards(fp, s)
    return np.array([[h.level, h.writer, h.reader, h.element[0], h.element[1]] for h in rep.hazards],
                    dtype=np.int64).reshape(-1, 5)


def main():
    out_dir = HERE / "depgraph"
    out_dir.mkdir(exist_ok=True)
    for name in CASES:
        with np.load(HERE / f"{name}.npz") as d:
            a = lv.CscMatrix(int(d["n"]), d["a_col_ptr"], d["a_row_idx"], d["a_values"])
        fp = lv.symbolic_fillin(a.pattern)
        ex_ptr, ex_idx = csr_of(lv.detect_double_u_exact(fp))
        up = lv.levelize(lv.detect_upward(fp))
        rel = lv.levelize(lv.detect_relaxed(fp))
        np.savez_compressed(out_dir / f"{name}.npz", exact_ptr=ex_ptr, exact_idx=ex_idx,
                            hz_upward=hazards(fp, up), hz_relaxed=hazards(fp, rel),
                            upward_level_of=up.level_of)
        print(name, len(ex_idx), len(hazards(fp, up)), flush=True)


if __name__ == "__main__":
    main()
