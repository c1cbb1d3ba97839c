"""Plan-parameter sweep (diagnostics): item MAC cap T and deep threshold D."""
import sys, json, pathlib, time
import numpy as np
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
import paper_1908_00204_b200 as glu
from paper_1908_00204_b200 import synthetic

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
a = synthetic.make(cfg)
fp = glu.symbolic_fillin(a.pattern)
s = glu.levelize(glu.detect_relaxed(fp))
dev = torch.device("cuda", 0)
ad = torch.from_numpy(a.values).to(dev)
v = torch.empty(fp.nnz, dtype=torch.float64, device=dev)
st = torch.cuda.current_stream()
for T, D in [(0, 0), (64, 0), (32, 0), (128, 0), (0, 16), (0, 32), (0, 4)]:
    fz = glu.Factorizer(fp, s.level_of, 1, max_item_macs=T, deep_min=D)
    fz.set_input(a.col_ptr, a.row_idx)
    for _ in range(3):
        fz.scatter_device(ad, v, st); assert fz.factor_device(v, 1e-14, st) == -1
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        fz.scatter_device(ad, v, st)
        e0.record(st); fz.factor_device_async(v, 1e-14, st); e1.record(st); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"T": T, "D": D, "ms": round(min(ts), 3), "items": fz.plan_info["items"],
                      "deep_items": fz.plan_info["deep_items"]}), flush=True)
    fz.close()
