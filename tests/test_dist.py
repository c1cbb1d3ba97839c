"""Multi-process batch path on the host (gloo, world size 2): sharding and
the final gather are exactly what bench.py / batch.py run over NCCL on
GPUs; the per-set factorization here is the CPU oracle standing in for the
device (no GPU needed)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1908_00204_b200 import batch


def test_shard_covers_batch_exactly():
    for total in (0, 1, 7, 1024, 1025):
        for world in (1, 2, 3, 8):
            got = [list(batch.shard(total, r, world)) for r in range(world)]
            flat = [i for g in got for i in g]
            assert flat == list(range(total))
            assert max(len(g) for g in got) - min(len(g) for g in got) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    from paper_1908_00204_b200 import synthetic

    import paper_1908_00204_b200 as glu

    a = synthetic.make("cfg1")
    fp = glu.symbolic_fillin(a.pattern)
    s = glu.levelize(glu.detect_relaxed(fp))
    pat = orc.Pattern.from_fp(fp)
    lp = np.concatenate([[0], np.cumsum([len(c) for c in s.levels])])
    lc = np.concatenate(s.levels)
    idx, st, dg = [], [], []
    for b in batch.shard(total, rank, world):
        vals = synthetic.perturb_values(a, 1000 + b)
        if b == 3:
            vals = np.zeros_like(vals)  # a singular set: fails at its first pivot
        v, bad = orc.scatter(pat, a.col_ptr, a.row_idx, vals)
        rc = orc.factor_parallel(pat, v, lp, lc, np.ones(len(lp) - 1, np.int64), False)
        idx.append(b)
        st.append(rc)
        dg.append(batch.set_digest(v))
    i, status, digest = batch.gather_results(idx, st, dg)
    if rank == 0:
        out.put((i.tolist(), status.tolist(), digest.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_shard_and_gather_match_single_process():
    total = 6
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, out)) for r in range(2)]
    for p in procs:
        p.start()
    res = out.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    i, status, digest = res
    assert i == list(range(total))
    assert status[3] >= 0 and all(s == -1 for k, s in enumerate(status) if k != 3)
    # the same sets factored in one process give the same bits
    from oracle import oracle as orc
    from paper_1908_00204_b200 import synthetic

    import paper_1908_00204_b200 as glu

    a = synthetic.make("cfg1")
    fp = glu.symbolic_fillin(a.pattern)
    s = glu.levelize(glu.detect_relaxed(fp))
    pat = orc.Pattern.from_fp(fp)
    lp = np.concatenate([[0], np.cumsum([len(c) for c in s.levels])])
    lc = np.concatenate(s.levels)
    for b in (0, 5):
        v, _ = orc.scatter(pat, a.col_ptr, a.row_idx, synthetic.perturb_values(a, 1000 + b))
        assert orc.factor_parallel(pat, v, lp, lc, np.ones(len(lp) - 1, np.int64), False) == -1
        assert batch.set_digest(v) == digest[b]
