"""Seeded synthetic circuit-like matrices for the BASELINE configs.

The reference ships no matrices beyond two tiny fixtures; BASELINE.json names
synthetic analogues, generated here:

  cfg1  2-D-local random graph, n=2000, deg 4, radius 2
  cfg2  as cfg1 with n=100,000 and 4 hub nodes (power/ground nets) each
        coupled to 10% of the nodes
  cfg3  1-D-local random graph, n=680,000, deg 2.4, window +-40, 6 hubs x 1%
  cfg4  5-point 2-D grid 1258 x 1258 (G3_circuit-like), entries x U(0.9,1.1)
  cfg5  1,024 value sets on cfg2's pattern, off-diagonals x (1+0.05 U(-1,1))

All are structurally symmetric, numerically unsymmetric and strictly
diagonally dominant (no pivot breakdown).  cfg1-3 use SuperLU's MMD
ordering on A^T+A, as the survey did; cfg4 (where MMD took 1,225 s) uses
geometric nested dissection on the grid coordinates, O(n log n).  Fill and
level counts are reported next to every number.
"""

from __future__ import annotations

import numpy as np

from .sparse import CscMatrix, Permutation, Triplets, permute, to_csc


def _sym_edges(u: np.ndarray, v: np.ndarray, n: int) -> tuple[np.ndarray, np.ndarray]:
    """Unique undirected edges (u < v)."""
    a, b = np.minimum(u, v), np.maximum(u, v)
    keep = a != b
    key = np.unique(a[keep].astype(np.int64) * n + b[keep])
    return key // n, key % n


def _assemble(n, eu, ev, rng, diag_margin=1.0, scale=None) -> CscMatrix:
    """Both directions with independent U(-1,1) values (or stencil values),
    diagonal = off-diagonal absolute row sum + margin."""
    rows = np.concatenate([eu, ev])
    cols = np.concatenate([ev, eu])
    if scale is None:
        vals = rng.uniform(-1.0, 1.0, size=len(rows))
    else:
        vals = scale * rng.uniform(0.9, 1.1, size=len(rows))
    rowsum = np.bincount(rows, weights=np.abs(vals), minlength=n)
    d = np.arange(n, dtype=np.int64)
    return to_csc(Triplets(n, n, np.concatenate([rows, d]), np.concatenate([cols, d]),
                           np.concatenate([vals, rowsum + diag_margin])))


def nested_dissection(coords: np.ndarray, indptr: np.ndarray, indices: np.ndarray,
                      leaf: int = 64) -> np.ndarray:
    """Geometric nested dissection.  coords (m, d) float; adjacency in CSR.
    Returns order[new] = old.  Each node set is cut at the median of its
    widest coordinate; the separator is the set of right-side endpoints of
    the cut edges; order = ND(left) + ND(right - sep) + sep."""
    m = len(coords)
    side = np.zeros(m, dtype=np.int8)
    out = []
    stack = [(np.arange(m, dtype=np.int64), 0)]
    # explicit post-order: entries are (nodes, state); state 1 = emit separator
    while stack:
        item, state = stack.pop()
        if state == 1:
            out.append(item)
            continue
        S = item
        if len(S) <= leaf:
            c = coords[S]
            out.append(S[np.lexsort(c.T[::-1])])
            continue
        c = coords[S]
        ext = c.max(axis=0) - c.min(axis=0)
        ax = int(np.argmax(ext))
        x = c[:, ax]
        cut = np.median(x)
        left_mask = x < cut
        if left_mask.all() or not left_mask.any():
            left_mask = x <= cut
            if left_mask.all() or not left_mask.any():
                out.append(S[np.argsort(x, kind="stable")])
                continue
        L, R = S[left_mask], S[~left_mask]
        side[L] = 1
        side[R] = 2
        # right nodes with a neighbour on the left form the separator
        deg = indptr[R + 1] - indptr[R]
        owner = np.repeat(np.arange(len(R)), deg)
        starts = np.repeat(indptr[R], deg)
        offs = np.arange(len(owner)) - np.repeat(np.cumsum(deg) - deg, deg)
        nb = indices[starts + offs]
        hit = np.zeros(len(R), dtype=bool)
        hit[owner[side[nb] == 1]] = True
        side[S] = 0
        sep, R2 = R[hit], R[~hit]
        sep = sep[np.lexsort(coords[sep].T[::-1])]
        stack.append((sep, 1))
        stack.append((R2, 0))
        stack.append((L, 0))
    order = np.concatenate(out) if out else np.empty(0, dtype=np.int64)
    assert len(order) == m
    return order


def _csr_adj(n: int, eu: np.ndarray, ev: np.ndarray):
    r = np.concatenate([eu, ev])
    c = np.concatenate([ev, eu])
    o = np.argsort(r, kind="stable")
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(indptr, r + 1, 1)
    np.cumsum(indptr, out=indptr)
    return indptr, c[o].astype(np.int64)


def mmd_order(a: CscMatrix) -> np.ndarray:
    """SuperLU's multiple-minimum-degree ordering on A^T + A (the survey's
    ordering for cfg1-3), as forward[old] = new.  scipy factors the matrix
    on the way; only the column permutation is kept."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as sla

    A = sp.csc_matrix((a.values, a.row_idx, a.col_ptr), shape=(a.n, a.n))
    lu = sla.splu(A, permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0,
                  options=dict(SymmetricMode=True))
    return np.asarray(lu.perm_c, dtype=np.int64)


def _order_and_permute(a: CscMatrix, coords, eu, ev, n_geo: int, method: str = "nd") -> CscMatrix:
    """Symmetric fill-reducing permutation: SuperLU MMD, or geometric nested
    dissection over the nodes [0, n_geo) with the hubs (>= n_geo) last."""
    if method == "mmd":
        p = Permutation(mmd_order(a))
        return permute(a, p, p)
    geo = (eu < n_geo) & (ev < n_geo)
    indptr, indices = _csr_adj(n_geo, eu[geo], ev[geo])
    order = nested_dissection(coords, indptr, indices)
    order = np.concatenate([order, np.arange(n_geo, a.n, dtype=np.int64)])
    fwd = np.empty(a.n, dtype=np.int64)
    fwd[order] = np.arange(a.n, dtype=np.int64)
    p = Permutation(fwd)
    return permute(a, p, p)


def _hub_edges(rng, n_geo, hubs, frac):
    eu, ev = [], []
    for h in range(hubs):
        k = max(1, int(frac * n_geo))
        nodes = rng.choice(n_geo, size=k, replace=False)
        eu.append(np.full(k, n_geo + h, dtype=np.int64))
        ev.append(nodes.astype(np.int64))
    if not eu:
        return np.empty(0, np.int64), np.empty(0, np.int64)
    return np.concatenate(eu), np.concatenate(ev)


def circuit_like(n: int = 2000, deg: float = 4.0, radius: int = 2, hubs: int = 0,
                 hub_frac: float = 0.10, seed: int = 0, ordering: str = "mmd") -> CscMatrix:
    """cfg1 / cfg2: nodes on a ceil(sqrt)-wide grid, random links within
    Chebyshev radius ``radius``, plus ``hubs`` dense power/ground nodes."""
    rng = np.random.default_rng(seed)
    n_geo = n - hubs
    w = int(np.ceil(np.sqrt(n_geo)))
    m = int(round(n_geo * deg / 2))
    u = rng.integers(0, n_geo, size=m)
    dx = rng.integers(-radius, radius + 1, size=m)
    dy = rng.integers(-radius, radius + 1, size=m)
    x, y = u % w + dx, u // w + dy
    v = y * w + x
    ok = (x >= 0) & (x < w) & (y >= 0) & (v < n_geo) & (v >= 0)
    eu, ev = _sym_edges(u[ok], v[ok], n)
    hu, hv = _hub_edges(rng, n_geo, hubs, hub_frac)
    if len(hu):
        hu2, hv2 = _sym_edges(hu, hv, n)
        eu, ev = np.concatenate([eu, hu2]), np.concatenate([ev, hv2])
    a = _assemble(n, eu, ev, rng)
    coords = np.stack([np.arange(n_geo) % w, np.arange(n_geo) // w], axis=1).astype(np.float64)
    return _order_and_permute(a, coords, eu, ev, n_geo, ordering)


def asic_like(n: int = 680_000, deg: float = 2.4, window: int = 40, hubs: int = 6,
              hub_frac: float = 0.01, seed: int = 0, ordering: str = "mmd") -> CscMatrix:
    """cfg3: 1-D-local random links within +-window, plus hubs."""
    rng = np.random.default_rng(seed)
    n_geo = n - hubs
    m = int(round(n_geo * deg / 2))
    u = rng.integers(0, n_geo, size=m)
    off = rng.integers(1, window + 1, size=m) * rng.choice([-1, 1], size=m)
    v = u + off
    ok = (v >= 0) & (v < n_geo)
    eu, ev = _sym_edges(u[ok], v[ok], n)
    hu, hv = _hub_edges(rng, n_geo, hubs, hub_frac)
    if len(hu):
        hu2, hv2 = _sym_edges(hu, hv, n)
        eu, ev = np.concatenate([eu, hu2]), np.concatenate([ev, hv2])
    a = _assemble(n, eu, ev, rng)
    coords = np.arange(n_geo, dtype=np.float64)[:, None]
    return _order_and_permute(a, coords, eu, ev, n_geo, ordering)


def grid5(k: int = 1258, drop: float = 0.0, seed: int = 0) -> CscMatrix:
    """cfg4: 5-point k x k grid; stencil -1 off-diagonal x U(0.9,1.1),
    diagonal = |off-diagonal| row sum + 0.1.  ``drop`` removes that fraction
    of grid edges (fill closer to the real G3_circuit)."""
    rng = np.random.default_rng(seed)
    n = k * k
    idx = np.arange(n, dtype=np.int64).reshape(k, k)
    eu = np.concatenate([idx[:, :-1].ravel(), idx[:-1, :].ravel()])
    ev = np.concatenate([idx[:, 1:].ravel(), idx[1:, :].ravel()])
    if drop > 0:
        keep = rng.uniform(size=len(eu)) >= drop
        eu, ev = eu[keep], ev[keep]
    a = _assemble(n, eu, ev, rng, diag_margin=0.1, scale=-1.0)
    coords = np.stack([np.arange(n) % k, np.arange(n) // k], axis=1).astype(np.float64)
    return _order_and_permute(a, coords, eu, ev, n)


def perturb_values(a: CscMatrix, seed: int, eps: float = 0.05) -> np.ndarray:
    """cfg5 value set: off-diagonals x (1 + eps U(-1,1)), diagonal recomputed
    as off-diagonal |row sum| + 1.  Same pattern as ``a``."""
    rng = np.random.default_rng(seed)
    cols = np.repeat(np.arange(a.n, dtype=np.int64), np.diff(a.col_ptr))
    diag = a.row_idx == cols
    v = a.values * (1.0 + eps * rng.uniform(-1.0, 1.0, size=len(a.values)))
    off = np.where(diag, 0.0, np.abs(v))
    rowsum = np.bincount(a.row_idx, weights=off, minlength=a.n)
    v[diag] = rowsum[a.row_idx[diag]] + 1.0
    return v


CONFIGS = {
    "cfg1": lambda: circuit_like(2000, seed=0),
    "cfg2": lambda: circuit_like(100_000, hubs=4, hub_frac=0.10, seed=0),
    "cfg3": lambda: asic_like(680_000, seed=0),
    "cfg4": lambda: grid5(1258, seed=0),
    # G3-family grids between cfg1 and cfg4 (parity at intermediate sizes)
    "g200": lambda: grid5(200, seed=0),
    "g400": lambda: grid5(400, seed=0),
    "g600": lambda: grid5(600, seed=0),
    "g800": lambda: grid5(800, seed=0),
}


def make(name: str) -> CscMatrix:
    return CONFIGS[name]()
