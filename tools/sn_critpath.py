"""Critical path of one supernodal factorization from its per-task trace
(tools/sn_probe.py with SN_TRACE_DUMP=... --stamps): walks back from the
last task to finish through whatever it waited on last -- a counter it
needed (the task whose completion reached the count) or, when it started
late, the previous task of its warp -- and splits the path into execution,
hand-off latency and warp-busy delay.  Diagnostics only.

    python tools/sn_critpath.py g400 gpurun_out/trace_g400.npz [--grid 296]
"""

from __future__ import annotations

import argparse
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("config")
    p.add_argument("trace")
    p.add_argument("--grid", type=int, default=296, help="CTAs of the launch (8 warps each)")
    args = p.parse_args()
    import paper_1908_00204_b200 as glu
    from paper_1908_00204_b200 import synthetic
    import sn_emul

    name = args.config
    a = synthetic.make(name) if name in synthetic.CONFIGS else synthetic.grid5(int(name[1:]), seed=0)
    fp = glu.symbolic_fillin(a.pattern)
    plan = sn_emul.build(fp)
    tasks, panm = plan["tasks"], plan["panm"]
    tr = np.load(args.trace)["trace"].astype(np.float64) * 1e-2  # us
    n = len(tasks)
    assert tr.shape[0] == n
    d = sn_emul._decode(tasks)
    kind, P, K, need = d["kind"], d["P"], d["K"], d["need"]
    w = d["p1"] - d["p0"]
    # completion times per counter: in[K] by RECT tasks, f[P] by TRSM tasks
    done = tr[:, 3]
    comp = {}
    # an RG task adds all its pushes at once: expand it into that many completions
    rgi = np.flatnonzero(kind == 3)
    for cnt, sel, key in ((0, kind == 1, K), (1, kind == 0, P)):
        idx = np.flatnonzero(sel)
        if cnt == 0 and len(rgi):
            idx = np.concatenate([idx, np.repeat(rgi, d["p1"][rgi])])  # ta.w = RECT chunks
        order = np.lexsort((done[idx], key[idx]))
        idx = idx[order]
        keys = key[idx]
        starts = np.searchsorted(keys, np.arange(len(panm) + 1))
        comp[cnt] = (idx, starts)

    def nth(cnt, panel, k):
        """Task whose completion made counter (cnt, panel) reach k."""
        idx, starts = comp[cnt]
        return int(idx[starts[panel] + k - 1])

    z = np.load(args.trace)
    if "warp" in z:
        warp_of = z["warp"]
    else:  # static deal
        warp_of = (np.arange(n) % args.grid) * 8 + (np.arange(n) // args.grid) % 8
    prev_on_warp = np.full(n, -1)
    last = {}
    for i in np.argsort(tr[:, 0], kind="stable"):  # each warp's tasks in the order it ran them
        wv = int(warp_of[i])
        prev_on_warp[i] = last.get(wv, -1)
        last[wv] = i

    def deps(i):
        k = int(kind[i])
        if k == 0:
            return [(0, int(P[i]), int(panm[P[i], 0]))]
        if k == 4:  # WB
            return [(1, int(P[i]), int(panm[P[i], 1]))]
        if k == 1:
            return [(1, int(P[i]), int(panm[P[i], 1])), (0, int(K[i]), int(need[i]))]
        if k == 3:  # RG: the target, then each push's source panel
            x0, c = int(d["r0"][i]), int(d["r1"][i])
            return [(0, int(K[i]), int(need[i]))] + [(1, int(plan["push"][x, 0]), int(panm[plan["push"][x, 0], 1]))
                                                     for x in range(x0, x0 + c)]
        return [(0, int(K[i]), int(need[i]) + int(panm[P[i], 1]))]

    i = int(np.argmax(done))
    path = []
    ex = hop = busy = 0.0
    kinds = np.zeros(5)
    links = {}
    while i >= 0:
        best, bt, bc = -1, -1.0, -1
        for c, p_, k in deps(i):
            if k <= 0:
                continue
            j = nth(c, p_, k)
            if done[j] > bt:
                best, bt, bc = j, done[j], c
        pw = int(prev_on_warp[i])
        pw_done = done[pw] if pw >= 0 else 0.0
        ready = tr[i, 2]
        ex += done[i] - ready
        kinds[int(kind[i])] += done[i] - ready
        if best >= 0 and bt >= pw_done:
            lk = ("tgt" if bc == 0 else "src", int(kind[i]), int(kind[best]))
            links[lk] = links.get(lk, 0) + 1
            hop += ready - bt
            path.append((i, "dep", ready - bt))
            i = best
        elif pw >= 0:
            busy += ready - pw_done
            path.append((i, "warp", ready - pw_done))
            i = pw
        else:
            path.append((i, "start", ready))
            break
    span = float(done.max() - tr[:, 0].min())
    print(f"{name}: span {span:.0f} us, critical path {len(path)} tasks: execution {ex:.0f} us "
          f"(TRSM {kinds[0]:.0f}, RECT {kinds[1]:.0f}, UW {kinds[2]:.0f}, RG {kinds[3]:.0f}), hand-offs {hop:.0f} us, "
          f"warp-busy {busy:.0f} us")
    hops = np.array([x[2] for x in path if x[1] == "dep"])
    if len(hops):
        print(f"  hand-off latency per dependency: median {np.median(hops):.2f} us, p90 "
              f"{np.percentile(hops, 90):.2f}, n {len(hops)}")
    exs = np.array([done[x[0]] - tr[x[0], 2] for x in path])
    print(f"  execution per task on the path: median {np.median(exs):.2f} us, p90 {np.percentile(exs, 90):.2f}")
    nb = sum(1 for x in path if x[1] == "warp")
    print(f"  warp-busy links: {nb}")
    names = {0: "TRSM", 1: "RECT", 2: "UW", 3: "RG", 4: "WB"}
    print("  dependency links (waited on, task <- predecessor):",
          ", ".join(f"{a} {names[b]}<-{names[c]}: {v}" for (a, b, c), v in sorted(links.items(), key=lambda z: -z[1])))
    for kk, nm in ((0, "TRSM"), (1, "RECT"), (2, "UW"), (3, "RG"), (4, "WB")):
        m = [x for x in path if kind[x[0]] == kk]
        if m:
            ww = np.array([max(int(w[x[0]]), 1) for x in m])
            print(f"  {nm}: {len(m)} on the path, widths {np.bincount(np.minimum(ww, 16))[1:].tolist()}")


if __name__ == "__main__":
    main()
