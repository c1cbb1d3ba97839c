"""Per-item timestamp trace of chosen phases (diagnostics, glu_set_option
3/4 + glu_trace_read) together with per-phase completion times."""
import sys, json, pathlib
import numpy as np
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
import paper_1908_00204_b200 as glu
from paper_1908_00204_b200 import synthetic, _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
contract = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ranges = [(0, 2), (10, 2), (300, 4), (690, 2)]
a = synthetic.make(cfg)
fp = glu.symbolic_fillin(a.pattern)
s = glu.levelize(glu.detect_relaxed(fp))
fz = glu.Factorizer(fp, s.level_of, contract)
fz.set_input(a.col_ptr, a.row_idx)
import os
if 'GLU_POLL' in os.environ:
    fz.set_option(6, int(os.environ['GLU_POLL']))
dev = torch.device("cuda", 0)
ad = torch.from_numpy(a.values).to(dev)
v = torch.empty(fp.nnz, dtype=torch.float64, device=dev)
st = torch.cuda.current_stream()
for _ in range(2):
    fz.scatter_device(ad, v, st); fz.factor_device(v, 1e-14, st)
out = {}
for l0, nl in ranges:
    if l0 + nl > s.level_count:
        continue
    fz.set_option(1, 1)
    fz.set_option(3, l0)
    fz.set_option(4, nl)
    fz.scatter_device(ad, v, st)
    rc = fz.factor_device(v, 1e-14, st)
    lt = np.array(fz.level_times_s()) * 1e9
    ends = np.cumsum(lt)  # ns since kernel start, per phase completion
    rec = np.zeros((200000, 8), dtype=np.int64)
    m = _lib.lib.glu_trace_read(fz.handle, _lib.ptr(rec), len(rec))
    rec = rec[:m]
    out[f"r{l0}"] = rec
    out[f"ends{l0}"] = ends
    fz.set_option(4, 0)
    if not len(rec):
        continue
    t0 = rec[:, 2].min()
    lv = rec[:, 0] >> 32
    for l in range(l0, l0 + nl):
        r = rec[lv == l]
        if not len(r):
            continue
        prev_done = r[:, 4].min()  # earliest wait release
        print(json.dumps({"phase": l, "items": len(r), "warps": len(set(r[:, 1].tolist())),
              "start_us": round((r[:, 2].min() - t0) / 1e3, 2),
              "wait_done_us(min/max)": [round((r[:, 4].min() - t0) / 1e3, 2), round((r[:, 4].max() - t0) / 1e3, 2)],
              "load_us(med/max)": [float(np.median(r[:, 5] - r[:, 4])) / 1e3, float((r[:, 5] - r[:, 4]).max()) / 1e3],
              "apply_store_us(med/max)": [float(np.median(r[:, 6] - r[:, 5])) / 1e3, float((r[:, 6] - r[:, 5]).max()) / 1e3],
              "last_store_us": round((r[:, 6].max() - t0) / 1e3, 2),
              "phase_len_us": round(lt[l] / 1e3, 2)}))
np.savez(ROOT / "gpurun_out" / f"trace_{cfg}_{contract}{os.environ.get('TAG', '')}.npz", **out)
# deep items of the traced phases
for key in list(out):
    if not key.startswith("r"):
        continue
    rec = out[key]
    dp = rec[(rec[:, 7] > 0)]
    if len(dp):
        g = dp[:, 7]
        tot = (dp[:, 6] - dp[:, 4]) / 1e3
        print(json.dumps({"range": key, "deep_items": int(len(dp)), "groups_max": int(g.max()),
                          "loop_us_max": float(tot.max()), "us_per_group_med": float(np.median(tot / g)),
                          "first_group_us_med": float(np.median(dp[:, 5] - dp[:, 4]) / 1e3),
                          "setup_us_med": float(np.median(dp[:, 4] - dp[:, 3]) / 1e3)}))
