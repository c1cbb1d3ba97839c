"""Pin the analysis at the BASELINE configs' scale by running the REFERENCE.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_digests.py cfg2 cfg3 cfg4

For each config the reference's own symbolic_fillin (levlu/symbolic.py:92-145),
make_csr_view (sparse.py:267-278), detect_relaxed + levelize
(depgraph.py:113-170) run on the seeded synthetic matrix, and sha256 digests
of col_ptr, row_idx, diag_pos, csc_pos and level_of (int64, little endian)
go to tests/golden/analysis_digests.json (cfg4's analysis takes minutes in the
reference; the arrays themselves are GBs, so only digests are committed).
tests/test_analysis.py compares the product's C++ analysis against them.
"""

from __future__ import annotations

import hashlib
import json
import os
import pathlib
import sys
import time

import numpy as np

REF = pathlib.Path("/root/reference/pkg/src")
HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(1, str(HERE.parent.parent))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import levlu as lv  # noqa: E402  (the reference)

from paper_1908_00204_b200 import synthetic  # noqa: E402  (matrix generators only)


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()


def main(names):
    out_path = HERE / "analysis_digests.json"
    out = json.loads(out_path.read_text()) if out_path.exists() else {}
    for name in names:
        m = synthetic.make(name)
        a = lv.CscMatrix(m.n, m.col_ptr, m.row_idx, m.values)
        t0 = time.time()
        fp = lv.symbolic_fillin(a.pattern)
        t1 = time.time()
        s = lv.levelize(lv.detect_relaxed(fp))
        t2 = time.time()
        out[name] = {"n": int(fp.n), "nnz": int(fp.full.row_idx.shape[0]), "levels": int(s.level_count),
                     "col_ptr": digest(fp.full.col_ptr), "row_idx": digest(fp.full.row_idx),
                     "diag_pos": digest(fp.diag_pos), "csc_pos": digest(fp.csr.csc_pos),
                     "level_of": digest(s.level_of),
                     "reference_seconds": {"symbolic_fillin": round(t1 - t0, 1),
                                           "detect_relaxed+levelize": round(t2 - t1, 1)}}
        print(name, out[name], flush=True)
        out_path.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg2", "cfg3", "cfg4"])
