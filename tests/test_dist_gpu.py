"""Two ranks running the whole experience step (ExperienceMaker, mixed mode)
on their shards of the prompts, with the single collective carrying the
whitening / metric partials: the global statistics are bit-identical on both
ranks and match one rank running the union of the prompts.

* same GPU, gloo through the host callback (runs on any one-GPU box);
* one GPU per rank, NCCL through the library's own communicator
  (ppoexp_comm_*; needs two GPUs)."""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CFG = (1024, 128, 2, 4, 512, 128)
N_NEW = 16


def _models(px, ctx, o, cfg):
    from tests.golden_util import bf16_round
    pc = px.ModelConfig(*CFG)
    w = [bf16_round(o.init_params(cfg, 1)), bf16_round(o.init_params(cfg, 2)),
         bf16_round(o.init_params(cfg, 3, head=True, head_seed=4))]
    eng = px.Engine(px.DeviceModel(ctx, pc, w[0], px.MIXED))
    return eng, px.DeviceModel(ctx, pc, w[1], px.MIXED), px.DeviceModel(ctx, pc.with_head(), w[2], px.MIXED)


def _worker(rank, world, port, mode, q):
    import torch
    import torch.distributed as dist

    from oracle.oracle import ModelCfg, Oracle, synthetic_prompts
    from paper_2405_01481_b200 import ppoexp as px
    from paper_2405_01481_b200.dist import allgather_sum_fn
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = 0 if mode == "gloo" else rank
    torch.cuda.set_device(dev)
    o = Oracle(threads=1)
    cfg = ModelCfg(*CFG)
    ctx = px.Context(dev)
    eng, ref, crit = _models(px, ctx, o, cfg)
    prompts = synthetic_prompts(7, 8, 9, ragged_lengths=True)
    mine = prompts[rank * 4:(rank + 1) * 4]
    comm = None
    if mode == "gloo":
        xm = px.ExperienceMaker(eng, ref, crit, scripted_target=ord("e"),
                                allreduce=allgather_sum_fn(device=torch.device("cuda", dev), stage_on_host=True))
    else:
        uid = [px.Communicator.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)  # the side channel that ships the NCCL id
        comm = px.Communicator(ctx, uid[0], rank, world)
        xm = px.ExperienceMaker(eng, ref, crit, scripted_target=ord("e"), comm=comm)
    sp = px.SamplingSpec.temperature_spec(1.0, 0, 0, 0.9)
    batch, st = xm.run(mine, max_new=N_NEW, sampling=sp, seed=11, step_index=3, gidx0=rank * 4)
    one = None
    if rank == 0:  # the same step on one rank over all prompts
        solo = px.ExperienceMaker(eng, ref, crit, scripted_target=ord("e"))
        b1, s1 = solo.run(prompts, max_new=N_NEW, sampling=sp, seed=11, step_index=3, gidx0=0)
        one = ([x.response for x in b1], [x.whitened_advantages for x in b1],
               [s1.kl_sum, s1.kl_count, s1.reward_sum, s1.n_seqs, s1.adv_mean, s1.adv_std])
    q.put((rank, [st.kl_sum, st.kl_count, st.reward_sum, st.n_seqs, st.adv_mean, st.adv_std],
           [x.response for x in batch], [x.whitened_advantages for x in batch], one))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def _run(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000 + (50 if mode == "nccl" else 0)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=600)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    st0, st1 = res[0][1], res[1][1]
    assert st0 == st1, "global statistics differ between ranks"
    toks = res[0][2] + res[1][2]
    wh = res[0][3] + res[1][3]
    one_toks, one_wh, one_st = res[0][4]
    # sampling streams are keyed by the global prompt index: identical rollouts
    for a, b in zip(toks, one_toks):
        assert np.array_equal(a, b)
    assert st0[3] == 8.0 and st0[1] == one_st[1]
    # a different batch composition takes other GEMM tilings (fp32-grade, not
    # bitwise batch-invariant): agreement to fp32 rounding
    np.testing.assert_allclose(st0, one_st, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(np.concatenate(wh), np.concatenate(one_wh), rtol=1e-4, atol=1e-4)


def test_two_ranks_one_gpu_gloo():
    _run("gloo")


def test_two_ranks_nccl_in_library():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (one NCCL rank per GPU)")
    _run("nccl")
