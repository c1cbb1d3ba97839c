"""CPU emulation of the supernodal dataflow plan (glu_snode.cpp) -- test helper.

Runs the plan's warp tasks with the kernel's arithmetic (glu_snode.cu: every
MAC `t - l * u` as two IEEE roundings, every divide correctly rounded --
Python floats do exactly that) and the kernel's synchronisation: a task may
run once the counters it waits on (TRSM: in[P]; RECT: f[P] and in[K]; UW:
in[K]) reach their targets, and counts itself when done.

Execution is in rounds: every round runs a set of ready tasks concurrently
against a snapshot of the values; no two tasks of a round may write the same
slot, nor may one read a slot another writes (a race the counters fail to
order).  `schedule` picks the round's tasks: "all" (maximal concurrency),
"random" (a random half, seeded) or "serial" (the ready task with the
smallest index, one per round).  The static list order is also checked to be
topological (the kernel's deadlock-freedom argument).  So the emulation
checks the plan's per-target MAC order (against the oracle, bit for bit) and
its race freedom.
"""

from __future__ import annotations

import ctypes

import numpy as np

from paper_1908_00204_b200 import _lib

TRSM, RECT, UW, RG, WB = 0, 1, 2, 3, 4
TRI_F, WRITE_U = 1, 2


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
        info = np.zeros(16, dtype=np.int64)
        _lib.lib.glu_sn_plan_info(plan, _lib.ptr(info))
        ns, npan, npair, nmap, npush, ntask = (int(x) for x in info[:6])
        nrg, nslot, nidx, nuidx = (int(x) for x in info[10:14])
        arr = dict(sn=np.zeros((ns, 4), np.int32), pan=np.zeros((npan, 4), np.int32),
                   panm=np.zeros((npan, 4), np.int32), pairs=np.zeros((npair, 4), np.int32),
                   relmap=np.zeros(nmap, np.int32), push=np.zeros((npush, 4), np.int32),
                   push_need=np.zeros(npush, np.int32), tasks=np.zeros((ntask, 12), np.int32),
                   col_a=np.zeros(n, np.int32), rg=np.zeros((nrg, 4), np.int32),
                   rg_slot=np.zeros(nslot, np.int32), rg_idx=np.zeros(nidx, np.uint16),
                   rg_uidx=np.zeros(nuidx, np.uint16))
        _lib.lib.glu_sn_plan_export(plan, *(_lib.ptr(arr[k]) for k in
                                            ("sn", "pan", "panm", "pairs", "relmap", "push", "push_need",
                                             "tasks", "col_a", "rg", "rg_slot", "rg_idx", "rg_uidx")))
        arr["info"] = dict(zip(("supernodes", "panels", "pairs", "map", "pushes", "tasks", "dblk",
                                "crit_ns", "macs", "bytes", "rg_tasks", "rg_slots", "rg_macs", "rg_pairs"),
                               info[:14].tolist()))
    finally:
        _lib.lib.glu_plan_free(plan)
    return arr


class _Round:
    """Values as they were when the round began; writes collected per task."""

    def __init__(self, v, dblk):
        self.v0, self.d0 = v, dblk
        self.writes = {}
        self.reads = set()
        self.local = {}
        self._task = -1

    @property
    def task(self):
        return self._task

    @task.setter
    def task(self, t):
        self._task = t
        self.local = {}  # a task sees its own writes, never another task's of the round

    def rd(self, q):
        q = int(q)
        own = self.local.get(q)
        if own is not None:
            return own
        self.reads.add((self.task, q))
        return self.v0[q]

    def wr(self, q, x):
        self._w(int(q), x)

    def rdd(self, p, e):
        key = ("d", int(p), int(e))
        self.reads.add((self.task, key))
        return self.d0[key[1:]]

    def wrd(self, p, e, x):
        self._w(("d", int(p), int(e)), x)

    def _w(self, key, x):
        prev = self.writes.get(key)
        assert prev is None or prev[0] == self.task, f"slot {key} written by tasks {prev[0]} and {self.task}"
        self.writes[key] = (self.task, x)
        if not isinstance(key, tuple):
            self.local[key] = x


def _decode(tasks):
    code = (tasks[:, 0].view(np.uint32) >> 27).astype(np.int64)
    return dict(kind=code >> 2, flags=code & 3, chunk=tasks[:, 0] & ((1 << 27) - 1), P=tasks[:, 1],
                p0=tasks[:, 2], p1=tasks[:, 3], s1=tasks[:, 4], h=tasks[:, 5], r0=tasks[:, 6],
                r1=tasks[:, 7], K=tasks[:, 8], need=tasks[:, 9])


def _waits(d, plan, i):
    """[(counter, panel, target)] task i waits on; counter 0 = in, 1 = f.
    An RG task waits for its target once, then for each push's source panel
    as it reaches that push (here: all of them up front)."""
    panm = plan["panm"]
    k, P = int(d["kind"][i]), int(d["P"][i])
    if k == TRSM:
        return [(0, P, int(panm[P, 0]))]
    if k == WB:
        return [(1, P, int(panm[P, 1]))]
    K, need = int(d["K"][i]), int(d["need"][i])
    if k == RECT:
        return [(1, P, int(panm[P, 1])), (0, K, need)]
    if k == RG:
        x0, cnt = int(d["r0"][i]), int(d["r1"][i])  # RG: tb = {first slot, slots, first push, pushes}
        return [(0, K, need)] + [(1, int(plan["push"][x, 0]), int(panm[plan["push"][x, 0], 1]))
                                 for x in range(x0, x0 + cnt)]
    return [(0, K, need + int(panm[P, 1]))]


def _signal(d, i):
    """(counter, panel, increment) task i adds when done, or None."""
    k = int(d["kind"][i])
    if k == TRSM:
        return (1, int(d["P"][i]), 1)
    if k == RECT:
        return (0, int(d["K"][i]), 1)
    if k == RG:
        return (0, int(d["K"][i]), int(d["p1"][i]))  # ta.w: the RECT chunks of its pushes
    return None


def check_topological(plan):
    """Every task's waits are met by the tasks before it in the list."""
    d = _decode(plan["tasks"])
    cnt = np.zeros((2, len(plan["pan"])), dtype=np.int64)
    for i in range(len(plan["tasks"])):
        for c, p, need in _waits(d, plan, i):
            assert cnt[c, p] >= need, f"task {i} waits on a later task (counter {c}, panel {p})"
        s = _signal(d, i)
        if s is not None:
            cnt[s[0], s[1]] += s[2]


def emulate(plan, fp, v, thresh=1e-14, fail_level=None, schedule="all", seed=0):
    """Factor A_s values v (after the scatter) through the plan; returns
    (values, failing column key or -1) like the device path."""
    cp, dp = fp.full.col_ptr, fp.diag_pos
    n = fp.n
    v = np.array(v, dtype=np.float64)
    dblk = {}
    cmax = np.zeros(n)
    pairs, relmap, col_a, panm = plan["pairs"], plan["relmap"], plan["col_a"], plan["panm"]
    tasks = plan["tasks"]
    d = _decode(tasks)
    check_topological(plan)
    rng = np.random.default_rng(seed)

    def mx(c, x):
        a = abs(x)
        if a == a and a > cmax[c]:
            cmax[c] = a

    def clo_of(p0, w):
        return [max(int(col_a[p0 + c]) - p0, 0) for c in range(w)]

    def factor_block(E, p0, p1, clo, record):
        """The w x w diagonal block factored from the current (unfactored)
        values; B[c, r] = element (row p0 + r, column p0 + c)."""
        w = p1 - p0
        B = {}
        for c in range(w):
            dc = int(dp[p0 + c])
            for r in range(w):
                B[c, r] = E.rd(dc + r - c) if r >= clo[c] else 0.0
        for j in range(w):
            if record:
                for r in range(j + 1, w):
                    mx(p0 + j, B[j, r])
            piv = B[j, j]
            for r in range(j + 1, w):
                B[j, r] = B[j, r] / piv
            for r in range(j + 1, w):
                for c in range(j + 1, w):
                    if j >= clo[c]:
                        B[c, r] = B[c, r] - B[j, r] * B[c, j]
        return B

    def solve_u(E, i, P, p0, w, s1, lo, base):
        uu = {j: E.rd(base - (s1 - (p0 + j))) for j in range(lo, w)}
        for j in range(lo, w - 1):
            for r in range(j + 1, w):
                uu[r] = uu[r] - E.rdd(P, j * w + r) * uu[j]
        return uu

    def run_rg(E, i):
        """One-chunk pushes from one-column panels, in order, on the RG's
        staged slots (the kernel's shared-memory list): every MAC and every
        multiplier U(p0, k) through its u16 index."""
        slot0, nslot = int(d["s1"][i]), int(d["h"][i])
        idx0, uidx0 = int(d["P"][i]), int(d["p0"][i])  # ta = {code | pushes, first MAC index, first U index, 0}
        slots = plan["rg_slot"][slot0:slot0 + nslot]
        val = [E.rd(q) for q in slots]
        for x in range(int(d["r0"][i]), int(d["r0"][i]) + int(d["r1"][i])):
            P, r0, r1, _K = (int(y) for y in plan["push"][x])
            p0, p1, _S, h = (int(y) for y in plan["pan"][P])
            s1 = p1  # a one-column panel is a one-column supernode
            assert h <= 128
            L = [E.rd(int(dp[p0]) + 1 + t) for t in range(h)]
            for q in range(r0, r1):
                k, a, base, mp = (int(y) for y in pairs[q])
                ui = int(plan["rg_uidx"][uidx0])
                uidx0 += 1
                ix = plan["rg_idx"][idx0:idx0 + h]
                idx0 += h
                if a >= p1:
                    continue
                assert int(slots[ui]) == base - (s1 - p0), "RG multiplier index"
                u = val[ui]
                for t in range(h):
                    pos = int(relmap[mp + t]) if mp >= 0 else base + t
                    assert int(slots[ix[t]]) == pos, "RG slot index"
                    val[ix[t]] = val[ix[t]] - L[t] * u
        for q, x in zip(slots, val):
            E.wr(q, x)

    def run(E, i):
        kind, flags, chunk = int(d["kind"][i]), int(d["flags"][i]), int(d["chunk"][i])
        if kind == RG:
            run_rg(E, i)
            return
        if kind == WB:  # the factored block back in place
            P_, p0_, p1_ = int(d["P"][i]), int(d["p0"][i]), int(d["p1"][i])
            w_ = p1_ - p0_
            clo = clo_of(p0_, w_)
            for c in range(w_):
                for r in range(clo[c], w_):
                    E.wr(int(dp[p0_ + c]) + r - c, E.rdd(P_, c * w_ + r))
            return
        P, p0, p1, s1, h = (int(d[k][i]) for k in ("P", "p0", "p1", "s1", "h"))
        w = p1 - p0
        rows = range(chunk * 32, min(h, chunk * 32 + 32))
        if kind == TRSM:
            clo = clo_of(p0, w)
            B = factor_block(E, p0, p1, clo, chunk == 0)
            if chunk == 0 and w >= 2:
                for c in range(w):
                    for r in range(w):
                        E.wrd(P, c * w + r, B[c, r])
            for t in rows:
                x = [E.rd(int(dp[p0 + c]) + (p1 - p0 - c) + t) for c in range(w)]
                for j in range(w):
                    mx(p0 + j, x[j])
                    dd = x[j] / B[j, j]
                    x[j] = dd
                    for c in range(j + 1, w):
                        if j >= clo[c]:
                            x[c] = x[c] - dd * B[c, j]
                for c in range(w):
                    E.wr(int(dp[p0 + c]) + (p1 - p0 - c) + t, x[c])
            return
        in_sn = s1 - p1
        tri = bool(flags & TRI_F) and kind == RECT or kind == UW
        L = {t: [E.rd(int(dp[p0 + j]) + (p1 - p0 - j) + t) for j in range(w)] for t in rows} if kind == RECT else {}
        for q in range(int(d["r0"][i]), int(d["r1"][i])):
            k, a, base, mp = (int(x) for x in pairs[q])
            if a >= p1:
                continue
            lo = max(a - p0, 0)
            uu = solve_u(E, i, P, p0, w, s1, lo, base) if tri else \
                {j: E.rd(base - (s1 - (p0 + j))) for j in range(lo, w)}
            if kind == UW or flags & WRITE_U:
                for r in range(lo + 1, w):
                    E.wr(base - (s1 - (p0 + r)), uu[r])
            if kind == UW:
                continue
            for t in rows:
                if t < in_sn:
                    pos = base - (in_sn - t)
                else:
                    pos = int(relmap[mp + t - in_sn]) if mp >= 0 else base + t - in_sn
                x = E.rd(pos)
                for j in range(lo, w):
                    x = x - L[t][j] * uu[j]
                E.wr(pos, x)

    ntask = len(tasks)
    cnt = np.zeros((2, len(plan["pan"])), dtype=np.int64)
    waits = [_waits(d, plan, i) for i in range(ntask)]
    done = np.zeros(ntask, dtype=bool)
    left = ntask
    while left:
        ready = [i for i in np.flatnonzero(~done) if all(cnt[c, p] >= need for c, p, need in waits[i])]
        assert ready, "no ready task: the plan deadlocks"
        if schedule == "serial":
            ready = ready[:1]
        elif schedule == "random":
            keep = rng.uniform(size=len(ready)) < 0.5
            ready = [t for t, k in zip(ready, keep) if k] or [ready[int(rng.integers(len(ready)))]]
        E = _Round(v, dblk)
        for i in ready:
            E.task = i
            run(E, i)
        owner = {}
        for key, (t, x) in E.writes.items():
            owner[key] = t
            if isinstance(key, tuple):
                dblk[key[1:]] = x
            else:
                v[key] = x
        for t, key in E.reads:
            wt = owner.get(key)
            assert wt is None or wt == t, f"task {t} reads {key} written by concurrent task {wt}"
        for i in ready:
            done[i] = True
            s = _signal(d, i)
            if s is not None:
                cnt[s[0], s[1]] += s[2]
        left -= len(ready)
    # the pivot check
    fail = -1
    best = None
    for c in range(n):
        m = cmax[c]
        for q in range(int(cp[c]), int(dp[c]) + 1):
            a = abs(v[q])
            if a == a and a > m:
                m = a
        if abs(v[dp[c]]) <= thresh * m:
            key = (c,) if fail_level is None else (int(fail_level[c]), c)
            if best is None or key < best:
                best = key
                fail = c
    return v, fail
