"""Multi-rank batch refactorization on the DEVICE: two ranks (gloo, both on
cuda:0 -- the test box has one GPU) each refactor their shard of a cfg5-style
batch through refactorize_batch (batched sm_100a launches), then all-gather
(set, status, LU digest) -- the same code path bench.py runs over NCCL on
N GPUs.  Every set's digest must equal the CPU oracle's, bit for bit."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

TOTAL = 10
SINGULAR = 4


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sets(a):
    from paper_1908_00204_b200 import synthetic

    out = []
    for b in range(TOTAL):
        vals = synthetic.perturb_values(a, 1000 + b)
        if b == SINGULAR:
            vals = np.zeros_like(vals)  # fails at its first pivot
        out.append(vals)
    return np.stack(out)


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1908_00204_b200 as glu
    from paper_1908_00204_b200 import batch, synthetic

    a = synthetic.make("cfg1")
    fp = glu.symbolic_fillin(a.pattern)
    lu0 = glu.factor_left_looking(a, fp)  # pattern resident on this rank's device
    mine = list(batch.shard(TOTAL, rank, world))
    vals, status = glu.refactorize_batch(lu0, a, _sets(a)[mine])
    digests = [batch.set_digest(v) for v in vals]
    i, st, dg = batch.gather_results(mine, status.tolist(), digests)
    if rank == 0:
        out.put((i.tolist(), st.tolist(), dg.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_device_batch_matches_oracle():
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    i, status, digest = out.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert i == list(range(TOTAL))
    from oracle import oracle as orc
    from paper_1908_00204_b200 import batch, synthetic

    import paper_1908_00204_b200 as glu

    a = synthetic.make("cfg1")
    fp = glu.symbolic_fillin(a.pattern)
    pat = orc.Pattern.from_fp(fp)
    sets = _sets(a)
    for b in range(TOTAL):
        v, _ = orc.scatter(pat, a.col_ptr, a.row_idx, sets[b])
        err = orc.factor_left_looking(pat, v)
        if b == SINGULAR:
            assert err >= 0 and status[b] == err
        else:
            assert err == -1 and status[b] == -1
            assert batch.set_digest(v) == digest[b], b
