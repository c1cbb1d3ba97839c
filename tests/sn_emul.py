"""CPU emulation of the supernodal plan (glu_snode.cpp) -- test helper.

Runs the plan's warp tasks phase by phase with the kernel's arithmetic
(glu_snode.cu: every MAC `t - l * u` as two IEEE roundings, every divide
correctly rounded -- Python floats do exactly that) and with phase-snapshot
semantics: every task reads the values as they were when its phase began
and no two tasks of a phase may write the same slot, nor may one read a
slot another writes.  So the emulation checks both the plan's per-target
MAC order (against the oracle, bit for bit) and its race freedom.
"""

from __future__ import annotations

import ctypes

import numpy as np

from paper_1908_00204_b200 import _lib

W = 32


def build(fp, level_of=None):
    """Supernodal plan of fp as numpy arrays (glu_plan_build_sn + export)."""
    n = fp.n
    cp, ri, dp = _lib.i64(fp.full.col_ptr), _lib.i64(fp.full.row_idx), _lib.i64(fp.diag_pos)
    rp, ci, cs = _lib.i64(fp.csr.row_ptr), _lib.i64(fp.csr.col_idx), _lib.i64(fp.csr.csc_pos)
    lv = _lib.i64(np.zeros(n) if level_of is None else level_of)
    plan = ctypes.c_void_p()
    rc = _lib.lib.glu_plan_build_sn(n, _lib.ptr(cp), _lib.ptr(ri), _lib.ptr(dp), _lib.ptr(rp),
                                    _lib.ptr(ci), _lib.ptr(cs), _lib.ptr(lv), 2, ctypes.byref(plan))
    if rc != _lib.GLU_OK:
        raise RuntimeError(f"glu_plan_build_sn: {rc} {_lib.last_error()}")
    try:
        info = np.zeros(12, dtype=np.int64)
        _lib.lib.glu_sn_plan_info(plan, _lib.ptr(info))
        ns, npan, npair, nmap, npush, ntask, nph = (int(x) for x in info[:7])
        arr = dict(sn=np.zeros((ns, 4), np.int32), pan=np.zeros((npan, 4), np.int32),
                   pairs=np.zeros((npair, 4), np.int32), relmap=np.zeros(nmap, np.int32),
                   push=np.zeros((npush, 4), np.int32), tasks=np.zeros((ntask, 8), np.int32),
                   phase_ptr=np.zeros(nph + 1, np.int32), col_a=np.zeros(n, np.int32))
        _lib.lib.glu_sn_plan_export(plan, *(_lib.ptr(arr[k]) for k in
                                            ("sn", "pan", "pairs", "relmap", "push", "tasks",
                                             "phase_ptr", "col_a")))
        arr["info"] = dict(zip(("supernodes", "panels", "pairs", "map", "pushes", "tasks", "phases",
                                "stages", "macs", "bytes"), info[:10].tolist()))
    finally:
        _lib.lib.glu_plan_free(plan)
    return arr


class _Phase:
    def __init__(self, v):
        self.v0 = v
        self.writes = {}
        self.reads = set()

    def rd(self, q):
        q = int(q)
        self.reads.add((self.task, q))
        return self.v0[q]

    def wr(self, q, x):
        q = int(q)
        prev = self.writes.get(q)
        assert prev is None or prev[0] == self.task, f"slot {q} written by two tasks of a phase"
        self.writes[q] = (self.task, x)


def emulate(plan, fp, v, thresh=1e-14, fail_level=None):
    """Factor A_s values v (after the scatter) through the plan; returns
    (values, failing column key or -1) like the device path."""
    cp, dp = fp.full.col_ptr, fp.diag_pos
    n = fp.n
    v = np.array(v, dtype=np.float64)
    cmax = np.zeros(n)
    pairs, relmap = plan["pairs"], plan["relmap"]
    col_a = plan["col_a"]
    tasks, pptr = plan["tasks"], plan["phase_ptr"]

    def factor_block(E, p0, p1, clo, record):
        """The w x w diagonal block factored from the phase-start values
        (DIAG, or TRSM / TRI with the local flag)."""
        w = p1 - p0
        B = {}
        for c in range(w):
            dc = int(dp[p0 + c])
            if record:
                for q in range(int(cp[p0 + c]), dc - (c - clo[c])):
                    mx(p0 + c, E.rd(q))
            for r in range(clo[c], w):
                B[c, r] = E.rd(dc + r - c)
        for j in range(w):
            if record:
                for r in range(clo[j], w):
                    mx(p0 + j, B[j, r])
            piv = B[j, j]
            for r in range(j + 1, w):
                B[j, r] = B[j, r] / piv
            for r in range(j + 1, w):
                for c in range(j + 1, w):
                    if j >= clo[c]:
                        B[c, r] = B[c, r] - B[j, r] * B[c, j]
        return B

    def mx(c, x):
        a = abs(x)
        if a == a and a > cmax[c]:
            cmax[c] = a

    for ph in range(len(pptr) - 1):
        E = _Phase(v.copy())
        for ti in range(pptr[ph], pptr[ph + 1]):
            kc, tph, p0, p1, s1, h, r0, r1 = (int(x) for x in tasks[ti])
            code, chunk = kc >> 27, kc & ((1 << 27) - 1)
            kind, local = code >> 1, code & 1
            assert tph == ph
            E.task = ti
            if kind == 0:  # DIAG
                w = p1 - p0
                clo = [max(int(col_a[p0 + c]) - p0, 0) for c in range(w)]
                B = factor_block(E, p0, p1, clo, True)
                for c in range(w):
                    for r in range(clo[c], w):
                        E.wr(int(dp[p0 + c]) + r - c, B[c, r])
            elif kind == 1:  # TRSM
                w = p1 - p0
                clo = [max(int(col_a[p0 + c]) - p0, 0) for c in range(w)]
                if local:
                    U = factor_block(E, p0, p1, clo, False)
                else:
                    U = {}
                    for c in range(w):
                        for r in range(clo[c], c + 1):
                            U[c, r] = E.rd(int(dp[p0 + c]) + r - c)
                for t in range(chunk * 32, min(h, chunk * 32 + 32)):
                    x = [E.rd(int(dp[p0 + c]) + (p1 - p0 - c) + t) for c in range(w)]
                    for j in range(w):
                        mx(p0 + j, x[j])
                        d = x[j] / U[j, j]
                        x[j] = d
                        for c in range(j + 1, w):
                            if j >= clo[c]:
                                x[c] = x[c] - d * U[c, j]
                    for c in range(w):
                        E.wr(int(dp[p0 + c]) + (p1 - p0 - c) + t, x[c])
            elif kind == 2:  # TRI
                w = p1 - p0
                if local:
                    clo = [max(int(col_a[p0 + c]) - p0, 0) for c in range(w)]
                    B = factor_block(E, p0, p1, clo, False)
                    Lb = {(j, r): B[j, r] for j in range(w) for r in range(j + 1, w)}
                else:
                    Lb = {(j, r): E.rd(int(dp[p0 + j]) + r - j) for j in range(w) for r in range(j + 1, w)}
                for q in range(r0, r1):
                    k, a, base, mp = (int(x) for x in pairs[q])
                    if a >= p1:
                        continue
                    lo = max(a - p0, 0)
                    u = {r: E.rd(base - (s1 - (p0 + r))) for r in range(lo, w)}
                    for j in range(lo, w):
                        for r in range(j + 1, w):
                            u[r] = u[r] - Lb[j, r] * u[j]
                    for r in range(lo + 1, w):
                        E.wr(base - (s1 - (p0 + r)), u[r])
            else:  # RECT
                w = p1 - p0
                in_sn = s1 - p1
                rows = range(chunk * 32, min(h, chunk * 32 + 32))
                L = {t: [E.rd(int(dp[p0 + j]) + (p1 - p0 - j) + t) for j in range(w)] for t in rows}
                for q in range(r0, r1):
                    k, a, base, mp = (int(x) for x in pairs[q])
                    if a >= p1:
                        continue
                    lo = max(a - p0, 0)
                    uu = {j: E.rd(base - (s1 - (p0 + j))) for j in range(lo, w)}
                    for t in rows:
                        if t < in_sn:
                            pos = base - (in_sn - t)
                        else:
                            pos = int(relmap[mp + t - in_sn]) if mp >= 0 else base + t - in_sn
                        x = E.rd(pos)
                        for j in range(lo, w):
                            x = x - L[t][j] * uu[j]
                        E.wr(pos, x)
        written = {}
        for q, (t, x) in E.writes.items():
            v[q] = x
            written[q] = t
        for t, q in E.reads:
            wt = written.get(q)
            assert wt is None or wt == t, f"phase {ph}: task {t} reads slot {q} written by task {wt}"
    fail = -1
    best = None
    for c in range(n):
        piv = v[dp[c]]
        if abs(piv) <= thresh * cmax[c]:
            key = (c,) if fail_level is None else (int(fail_level[c]), c)
            if best is None or key < best:
                best = key
                fail = c
    return v, fail
