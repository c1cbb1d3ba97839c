"""Same-process A/B of a supernodal-kernel knob read at every launch
(GLU_SN_WINDOW): one factorizer per config, the values interleaved rep by
rep, device time per factorization from CUDA events (L2 flushed before
each launch), and every result compared bit for bit with the first value's
(the path the GPU tests validate against the oracle).

    python tools/sn_ab.py cfg4 g400 --var GLU_SN_WINDOW --vals 0,1 --reps 6
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("configs", nargs="+")
    p.add_argument("--var", default="GLU_SN_WINDOW")
    p.add_argument("--vals", default="0,1")
    p.add_argument("--reps", type=int, default=6)
    args = p.parse_args()
    import torch

    import paper_1908_00204_b200 as glu
    from paper_1908_00204_b200 import numeric, synthetic

    dev = torch.device("cuda", 0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    vals = args.vals.split(",")
    for name in args.configs:
        a = synthetic.make(name) if name in synthetic.CONFIGS else synthetic.grid5(int(name[1:]), seed=0)
        fp = glu.symbolic_fillin(a.pattern)
        fz = numeric.Factorizer(fp, numeric._relaxed_levels(fp), 0, engine="sn")
        fz.set_input(a.col_ptr, a.row_idx)
        fz.set_option(1, 0)
        fz.set_option(2, 1)
        a_d = torch.from_numpy(a.values).to(dev)
        v = torch.empty(fp.nnz, dtype=torch.float64, device=dev)
        st = torch.cuda.current_stream()
        ts = {x: [] for x in vals}
        first = None
        same = {x: True for x in vals}
        for r in range(args.reps + 1):
            for x in vals:
                os.environ[args.var] = x
                fz.scatter_device(a_d, v, st)
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                fz.factor_device_async(v, 1e-14, st)
                e1.record(st)
                torch.cuda.synchronize()
                assert fz.status(st) == -1
                out = v.cpu().numpy()
                if first is None:
                    first = out
                elif not np.array_equal(out, first):
                    same[x] = False
                if r:
                    ts[x].append(e0.elapsed_time(e1))
        rec = {"config": name, "var": args.var,
               "ms_min": {x: round(min(ts[x]), 3) for x in vals},
               "ms_med": {x: round(float(np.median(ts[x])), 3) for x in vals},
               "bitwise_same_as_first": same}
        print(json.dumps(rec), flush=True)
        fz.close()
        del v, a_d
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
