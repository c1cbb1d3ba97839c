"""Per-level GPU timing of one factorization (globaltimer stamps written by
the persistent kernel) next to the plan's per-level items / MACs."""
import os, sys, time, json, pathlib
import numpy as np
ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
import paper_1908_00204_b200 as glu
from paper_1908_00204_b200 import synthetic, _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
contract = int(sys.argv[2]) if len(sys.argv) > 2 else 1
a = synthetic.make(cfg)
fp = glu.symbolic_fillin(a.pattern)
s = glu.levelize(glu.detect_relaxed(fp))
fz = glu.Factorizer(fp, s.level_of, contract)
fz.set_input(a.col_ptr, a.row_idx)
dev = torch.device("cuda", 0)
ad = torch.from_numpy(a.values).to(dev)
v = torch.empty(fp.nnz, dtype=torch.float64, device=dev)
st = torch.cuda.current_stream()
fz.set_option(1, 0)
if "GLU_POLL" in os.environ:
    fz.set_option(6, int(os.environ["GLU_POLL"]))
for _ in range(3):
    fz.scatter_device(ad, v, st); fz.factor_device(v, 1e-14, st)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
fz.scatter_device(ad, v, st)
e0.record(st); fz.factor_device_async(v, 1e-14, st); e1.record(st); torch.cuda.synchronize()
tot = e0.elapsed_time(e1)
fz.set_option(1, 1)
fz.scatter_device(ad, v, st); rc = fz.factor_device(v, 1e-14, st)
lt = np.array(fz.level_times_s()) * 1e3
out = ROOT / "gpurun_out" / f"levels_{cfg}_{contract}{os.environ.get('TAG', '')}.npz"
out.parent.mkdir(exist_ok=True)
np.savez(out, level_ms=lt, total_ms=tot)
print(json.dumps({"cfg": cfg, "contract": contract, "rc": rc, "total_ms": tot,
                  "sum_level_ms": float(lt.sum()), "levels": len(lt),
                  "pct_level_us": np.percentile(lt * 1e3, [0, 10, 50, 90, 99, 100]).tolist(),
                  "plan": fz.plan_info, "handle": fz.handle_info}))
