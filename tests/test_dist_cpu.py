"""Multi-rank host logic on CPU (gloo, world size 2): the experience step's
single collective — all-gather of the whitening/metric partials summed in rank
order — reproduces single-process whitening over the union of the shards."""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp


def _worker(rank, world, port, shards, out_q):
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2405_01481_b200.dist import allgather_sum_fn
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle(threads=1)
    adv = shards[rank]
    kl = np.full(len(adv), 0.5 * (rank + 1))
    part = np.array([len(adv), adv.sum(), (adv * adv).sum(), kl.sum(), 3.0 * (rank + 1), 1.0], np.float64)
    allgather_sum_fn()(part.ctypes.data, 6, None)
    w = o.whiten_apply(adv, part[:3])
    out_q.put((rank, part.copy(), w))
    dist.barrier()
    dist.destroy_process_group()


def test_whitening_collective_world2():
    from oracle.oracle import Oracle
    rng = np.random.default_rng(4)
    shards = [rng.normal(1.0, 3.0, size=97), rng.normal(-2.0, 0.5, size=203)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shards, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (part, w)) for r, part, w in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # identical statistics on every rank
    assert np.array_equal(res[0][0], res[1][0])
    allv = np.concatenate(shards)
    np.testing.assert_allclose(res[0][0][:3], [allv.size, allv.sum(), (allv * allv).sum()], rtol=1e-12)
    assert res[0][0][3] == pytest.approx(0.5 * 97 + 1.0 * 203) and res[0][0][5] == 2.0
    o = Oracle(threads=1)
    ref = o.whiten_apply(allv, o.whiten_partials(allv))
    np.testing.assert_allclose(np.concatenate([res[0][1], res[1][1]]), ref, rtol=1e-10, atol=1e-12)
