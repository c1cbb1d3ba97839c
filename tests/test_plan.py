"""The update plan (glu_plan_build) reproduces the reference's MAC order.

A numpy emulation of exactly what the device kernel does with the plan
(items in any order inside a phase, chunks in order inside an item, targets
by searching the item's segment, on-the-fly division, final pivot/divide
pass) must give the reference's values bit for bit: contract A = the
left-looking / deterministic values, contract B = the atomic-mode values.
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

import paper_1908_00204_b200 as glu
from paper_1908_00204_b200 import _lib
from conftest import csc_from_golden, load_golden


def export_plan(fp, level_of, contract, max_item_macs=0, deep_min=0, tail_max=0):
    cp, ri, dp = _lib.i64(fp.full.col_ptr), _lib.i64(fp.full.row_idx), _lib.i64(fp.diag_pos)
    lv = _lib.i64(level_of)
    h = ctypes.c_void_p()
    rc = _lib.lib.glu_plan_build(fp.n, _lib.ptr(cp), _lib.ptr(ri), _lib.ptr(dp), _lib.ptr(lv),
                                 contract, max_item_macs, deep_min, tail_max, 2, ctypes.byref(h))
    assert rc == _lib.GLU_OK, _lib.last_error()
    info = np.zeros(16, dtype=np.int64)
    _lib.lib.glu_plan_info(h, _lib.ptr(info))
    nl, ni, nc, nd = int(info[0]), int(info[1]), int(info[2]), int(info[9])
    nm, nt = int(info[11]), int(info[12])
    lip = np.zeros(nl + 1, dtype=np.int64)
    items = np.zeros((max(ni, 1), 8), dtype=np.int64)
    chunks = np.zeros((max(nc, 1), 5), dtype=np.int64)
    deep = np.zeros((max(nd, 1), 3), dtype=np.int64)
    map8 = np.zeros(max(nm, 1), dtype=np.uint8)
    tgt = np.zeros(max(nt, 1), dtype=np.int64)
    _lib.lib.glu_plan_export(h, _lib.ptr(lip), _lib.ptr(items), _lib.ptr(chunks), _lib.ptr(deep),
                             _lib.ptr(map8), _lib.ptr(tgt))
    _lib.lib.glu_plan_free(h)
    return dict(info=info, lip=lip, items=items[:ni], chunks=chunks[:nc], deep=deep[:nd],
                map8=map8[:nm], tgt=tgt[:nt])


def emulate(fp, level_of, plan, v, thresh, rng=None):
    """What factor_kernel does with the plan: items of a phase in any order;
    a push item stages its targets, applies its chunks in order (entries of
    one epoch must hit distinct targets) and writes every target back once."""
    ri = fp.full.row_idx
    lip, items, chunks, map8, tgt = plan["lip"], plan["items"], plan["chunks"], plan["map8"], plan["tgt"]
    for l in range(len(lip) - 1):
        order = np.arange(lip[l], lip[l + 1])
        if rng is not None:
            rng.shuffle(order)  # items of a phase are independent
        for it in order:
            moff, toff, base, c0, nch, ntgt, macs, kind = items[it]
            if kind == 1:  # deep: one target, ordered contributions
                for l_, d, m in plan["deep"][moff:moff + macs]:
                    v[base] = v[base] - (v[l_] / v[d]) * v[m]
                continue
            assert nch <= 32 and macs <= 128 and ntgt <= macs
            slots = base + tgt[toff:toff + ntgt]
            assert np.all(np.diff(slots) > 0)
            stage = v[slots].copy()
            e = moff
            touched = set()
            for m, j, p0, cnt, ep in chunks[c0:c0 + nch]:
                d = fp.diag_pos[j]
                p = np.arange(p0, p0 + cnt)
                u = map8[e:e + cnt].astype(np.int64)
                e += cnt
                # the staged slot is the row the MAC targets
                assert np.array_equal(ri[slots[u]], ri[p])
                if ep:
                    touched = set()
                assert touched.isdisjoint(u.tolist())
                touched.update(u.tolist())
                stage[u] = stage[u] - (v[p] / v[d]) * v[m]
            assert e == moff + macs
            v[slots] = stage
    # dense tail: columns >= t0, one source column at a time in index order
    t0 = int(plan["info"][13])
    cp_, dp_ = fp.full.col_ptr, fp.diag_pos
    for j in range(t0, fp.n):
        lrows = ri[dp_[j] + 1:cp_[j + 1]]
        for t in range(fp.csr.row_ptr[j], fp.csr.row_ptr[j + 1]):
            k = fp.csr.col_idx[t]
            if k <= j:
                continue
            m = fp.csr.csc_pos[t]
            rows_k = ri[cp_[k]:cp_[k + 1]]
            q = cp_[k] + np.searchsorted(rows_k, lrows)
            p = np.arange(dp_[j] + 1, cp_[j + 1])
            v[q] = v[q] - (v[p] / v[dp_[j]]) * v[m]
    fail = None
    cp, dp = fp.full.col_ptr, fp.diag_pos
    for j in range(fp.n):
        col = v[cp[j]:cp[j + 1]]
        cmax = 0.0
        for x in np.abs(col):
            if x > cmax:
                cmax = x
        piv = v[dp[j]]
        if abs(piv) <= thresh * cmax:
            key = (int(level_of[j]), j)
            fail = key if fail is None or key < fail else fail
            continue
        v[dp[j] + 1:cp[j + 1]] = v[dp[j] + 1:cp[j + 1]] / piv
    return fail


CASES = ["conflict8", "random_dd_s2_n80", "random_dd_s3_n120", "random_dd_s5_n100",
         "random_dd_s11_n300", "random_dd_s12_n500", "block_arrow_4x24", "banded_n200", "cfg1",
         "singular_2x2", "threshold_fail"]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("contract", [_lib.CONTRACT_A, _lib.CONTRACT_B])
@pytest.mark.parametrize("max_item_macs,deep_min,tail_max", [(0, 0, 0), (7, 0, 0), (0, 2, 0),
                                                              (5, 1000, 0), (0, 0, 1000)])
def test_plan_emulation_bitwise(case, contract, max_item_macs, deep_min, tail_max):
    g = load_golden(case)
    a = csc_from_golden(g)
    fp = glu.symbolic_fillin(a.pattern)
    level_of = g["level_of"]
    plan = export_plan(fp, level_of, contract, max_item_macs, deep_min, tail_max)
    assert int(plan["info"][3]) == glu.pattern_flops(fp)[0]  # every MAC planned once
    assert int(plan["info"][11]) + int(plan["info"][9]) + int(plan["info"][14]) == int(plan["info"][3])
    push = plan["items"][plan["items"][:, 7] == 0]
    assert int(push[:, 6].sum()) == int(plan["info"][11])
    assert int(push[:, 5].sum()) == int(plan["info"][12])
    if max_item_macs:
        assert np.all(push[:, 6] <= max_item_macs)
    v = np.zeros(fp.nnz)
    from oracle import oracle as orc
    v, bad = orc.scatter(orc.Pattern.from_fp(fp), a.col_ptr, a.row_idx, a.values)
    fail = emulate(fp, level_of, plan, v, float(g["thresh"]), np.random.default_rng(0))
    tag = "a" if contract == _lib.CONTRACT_A else "b"
    if int(g[f"fail_{tag}"]) >= 0:
        assert fail is not None and fail[1] == int(g[f"fail_{tag}"])
    else:
        assert fail is None
        assert np.array_equal(v, g[f"lu_{tag}"])


def test_contract_a_defers_only_when_needed():
    g = load_golden("cfg1")
    fp = glu.symbolic_fillin(csc_from_golden(g).pattern)
    pa = export_plan(fp, g["level_of"], _lib.CONTRACT_A)
    pb = export_plan(fp, g["level_of"], _lib.CONTRACT_B)
    assert pb["info"][6] == 0
    assert 0 < pa["info"][6] < pa["info"][3]


def _levels_arrays(level_of):
    order = np.argsort(level_of, kind="stable")
    counts = np.bincount(level_of)
    return np.concatenate([[0], np.cumsum(counts)]).astype(np.int64), order.astype(np.int64)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("workers", [1, 2])
def test_upward_schedule_matches_reference(case, workers):
    """factor_parallel accepts any LevelSchedule (levlu/numeric.py:241-351).
    Under levelize(detect_upward(fp)) the reference's deterministic mode
    still gives left-looking values, and its atomic mode reads multipliers
    that same-level sources update first: the plan (contract A on the
    relaxed schedule, contract B on the refined sub-levels) must give the
    oracle's factor_parallel values bit for bit."""
    from oracle import oracle as orc

    g = load_golden(case)
    a = csc_from_golden(g)
    fp = glu.symbolic_fillin(a.pattern)
    s = glu.levelize(glu.detect_upward(fp))
    lp, lc = _levels_arrays(s.level_of)
    pat = orc.Pattern.from_fp(fp)
    thresh = float(g["thresh"])
    for det, contract in ((True, _lib.CONTRACT_A), (False, _lib.CONTRACT_B)):
        ref, bad = orc.scatter(pat, a.col_ptr, a.row_idx, a.values)
        caps = np.full(len(lp) - 1, workers, dtype=np.int64)
        err = orc.factor_parallel(pat, ref, lp, lc, caps, det, thresh)
        phases = glu.numeric.plan_levels(fp, s.level_of, contract)
        if contract == _lib.CONTRACT_B:
            # sub-levels keep the caller's level order
            assert np.all(np.diff(s.level_of[np.argsort(phases, kind="stable")]) >= 0)
        plan = export_plan(fp, phases, contract)
        v, _ = orc.scatter(pat, a.col_ptr, a.row_idx, a.values)
        fail = emulate(fp, s.level_of if contract == _lib.CONTRACT_A else phases, plan, v, thresh,
                       np.random.default_rng(1))
        if err >= 0:
            assert fail is not None and fail[1] == err
        else:
            assert fail is None and np.array_equal(v, ref), (case, det)


def test_schedule_with_late_source_raises():
    """A source column placed after its target: the reference would read an
    unfinished column; the B200 path refuses instead of returning other bits."""
    g = load_golden("conflict8")
    fp = glu.symbolic_fillin(csc_from_golden(g).pattern)
    lv = np.zeros(fp.n, dtype=np.int64)
    lv[0] = 1  # column 0 is a source of column 1 (conflict8 deps)
    with pytest.raises(glu.ScheduleHazardError):
        glu.numeric.plan_levels(fp, lv, _lib.CONTRACT_A)
