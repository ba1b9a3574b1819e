"""The train side against the reference itself: the
unmodified reference sources compiled in place (oracle/_ref, its tape autodiff
and AdamW) run the same update on the same fp32-rounded weights.  Losses of
every step and the weights after the steps must agree within 1e-3 abs + 1e-3
rel (north_star).  GPU only; needs oracle/_ref (built by oracle/Makefile)."""
import os

import numpy as np
import pytest

from oracle.oracle import REF_SO, ModelCfg, synthetic_prompts
from tests.golden_util import to_px_cfg

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")]

CFG = ModelCfg(V=1024, d=128, L=2, H=4, f=512, S=128)  # C1 (BASELINE config 1)
ADAM = (0.9, 0.999, 1e-8, 0.01)
TOL = 1e-3


def close(a, b, atol=TOL, rtol=TOL):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    err = np.abs(a - b) - (atol + rtol * np.abs(b))
    assert (err <= 0).all(), f"max excess {err.max():.3e}, max abs diff {np.abs(a - b).max():.3e}"
    return float(np.abs(a - b).max())


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import RefLib
    return RefLib()


@pytest.fixture(scope="module")
def px():
    from paper_2405_01481_b200 import ppoexp
    return ppoexp


def f32(w):
    return np.asarray(w, np.float32).astype(np.float64)


def rollout(oracle, seed, n=6):
    prompts = synthetic_prompts(seed, n, 9, ragged_lengths=True)
    rng = np.random.default_rng(seed)
    seqs = [np.concatenate([p, rng.integers(0, 256, 5 + 3 * i)]).astype(np.int32) for i, p in enumerate(prompts)]
    return seqs, [len(p) for p in prompts]


def test_ppo_actor_step_matches_reference(px, ctx, oracle, ref):
    w = f32(ref.init_params(CFG, 5))
    seqs, rs = rollout(oracle, 3)
    lps = oracle.sequence_logprobs(CFG, w, seqs)
    rng = np.random.default_rng(1)
    # old log-probs a little off the current ones: some ratios fall outside the clip range
    old = [lp[r:] + rng.normal(0, 0.15, len(lp) - r) for lp, r in zip(lps, rs)]
    adv = [rng.normal(0, 1, len(lp) - r) for lp, r in zip(lps, rs)]
    lr, steps = 3e-4, 3
    w_ref, l_ref = ref.ppo_actor_step(CFG, w, seqs, rs, np.concatenate(old), np.concatenate(adv), 0.2, lr,
                                      adam=ADAM, n_steps=steps)
    tr = px.Trainer(ctx, to_px_cfg(CFG), w, adamw=px.AdamWOptions(*ADAM))
    losses = [tr.ppo_actor_step(seqs, rs, old, adv, clip_eps=0.2, lr=lr) for _ in range(steps)]
    close(losses, l_ref)
    close(tr.flat(), w_ref)
    assert np.abs(w_ref - w).max() > lr  # the weights moved


def test_critic_step_matches_reference(px, ctx, oracle, ref):
    cfg = CFG
    w = f32(ref.init_params(cfg, 6, head=True))
    w[-cfg.d:] = f32(np.random.default_rng(2).normal(0, 0.1, cfg.d))  # a non-zero scalar head
    seqs, rs = rollout(oracle, 4)
    rng = np.random.default_rng(3)
    n = [len(s) - r for s, r in zip(seqs, rs)]
    old_v = [rng.normal(0, 0.5, k) for k in n]
    rets = [rng.normal(0, 1, k) for k in n]
    lr, steps = 3e-4, 3
    w_ref, l_ref = ref.critic_step(cfg, w, seqs, rs, np.concatenate(old_v), np.concatenate(rets), 0.2, lr, adam=ADAM,
                                   n_steps=steps)
    tr = px.Trainer(ctx, to_px_cfg(cfg, True), w, adamw=px.AdamWOptions(*ADAM))
    losses = [tr.critic_step(seqs, rs, old_v, rets, value_clip=0.2, lr=lr) for _ in range(steps)]
    close(losses, l_ref)
    close(tr.flat(), w_ref)


@pytest.mark.parametrize("variant", ["dpo", "ipo", "cdpo", "kto"])
def test_dpo_step_matches_reference(px, ctx, oracle, ref, variant):
    w_pol = f32(ref.init_params(CFG, 7))
    w_ref = f32(ref.init_params(CFG, 8))
    rng = np.random.default_rng(4)
    pc = to_px_cfg(CFG)
    pairs = []
    for i in range(4):
        prompt = rng.integers(0, 256, 6 + i).tolist()
        c, rc = px.build_sft_sequence(pc, prompt, rng.integers(0, 256, 7 + i).tolist())
        r, rr = px.build_sft_sequence(pc, prompt, rng.integers(0, 256, 5 + 2 * i).tolist())
        pairs.append((c, r, rc, rr))
    lr, steps, beta, eps = 3e-4, 2, 0.5, 0.1
    var = {"dpo": 0, "ipo": 1, "cdpo": 2, "kto": 3}[variant]
    w_out, l_ref = ref.dpo_step(CFG, w_pol, w_ref, pairs, var, beta, eps, lr, adam=ADAM, n_steps=steps)
    frozen = px.DeviceModel(ctx, pc, w_ref, px.F32)
    tr = px.Trainer(ctx, pc, w_pol, adamw=px.AdamWOptions(*ADAM))
    losses = [tr.dpo_step(frozen, pairs, variant, beta, eps, lr)[0] for _ in range(steps)]
    close(losses, l_ref)
    close(tr.flat(), w_out)


def test_trainer_refit_updates_the_engine(px, ctx, oracle, ref):
    """After an actor update, refit pushes the weights into the serving engine
    in place: the generation counter advances and the engine's snapshot is the
    trainer's weights (Engine::refit, src/engine.cpp:60-90)."""
    w = f32(ref.init_params(CFG, 9))
    pc = to_px_cfg(CFG)
    eng = px.Engine(px.DeviceModel(ctx, pc, w, px.F32))
    tr = px.Trainer(ctx, pc, w, serving=eng.model)
    seqs, rs = rollout(oracle, 5, n=3)
    lps = oracle.sequence_logprobs(CFG, w, seqs)
    old = [lp[r:] for lp, r in zip(lps, rs)]
    adv = [np.ones(len(o)) for o in old]
    tr.ppo_actor_step(seqs, rs, old, adv, lr=1e-3)
    g0 = eng.generation_counter
    tr.refit()
    assert eng.generation_counter == g0 + 1
    snap = eng.model.snapshot()
    got = tr.get()
    for k in ("tok_embed.weight", "layers.1.attn.q_proj.weight", "layers.0.ffn.down_proj.weight", "final_norm.bias"):
        assert np.array_equal(snap[k], got[k]), k
    # the refitted engine generates what a freshly built engine on those weights generates
    flat = tr.flat()
    fresh = px.Engine(px.DeviceModel(ctx, pc, flat, px.F32))
    task = [px.GenTask(list(seqs[0][:rs[0]]), 8)]
    a, b = eng.generate_batch(task)[0], fresh.generate_batch(task)[0]
    assert np.array_equal(a.tokens, b.tokens) and np.array_equal(a.logprobs, b.logprobs)


def test_spin_make_pairs_matches_reference_generation(px, ctx, oracle, ref):
    """spin_make_pairs (src/losses.cpp:277-295) on the device engine: the
    rejected side is the reference model's greedy generation (equal to the
    oracle's), degenerate pairs (rejected == response) are dropped and counted."""
    w = f32(ref.init_params(CFG, 12))
    eng = px.Engine(px.DeviceModel(ctx, to_px_cfg(CFG), w, px.F32))
    prompts = synthetic_prompts(13, 5, 7, ragged_lengths=True)
    t_o, _ = oracle.generate(CFG, w, prompts, 6)
    rng = np.random.default_rng(2)
    examples = [(p, rng.integers(0, 256, 6)) for p in prompts]
    examples[2] = (prompts[2], t_o[2])  # the reference would generate exactly the response: dropped
    sp = px.spin_make_pairs(eng, examples, 6)
    assert sp.dropped == 1 and len(sp.pairs) == 4
    kept = [i for i in range(5) if i != 2]
    for (p, c, r), i in zip(sp.pairs, kept):
        assert np.array_equal(r, t_o[i]) and np.array_equal(c, examples[i][1])



def test_ppo_iterations_match_reference(px, ctx, oracle, ref):
    """Three full PPO iterations (ppo_step, src/ppo.cpp:302-441): greedy
    experience → actor update → critic update → refit of the serving engine and
    the critic → the next experience on the refitted models, against the same
    loop run by the reference itself (its tape autodiff and persistent AdamW;
    oracle/ref_shim.cpp ref_ppo_loop).  Rollouts identical, experience and
    losses within the bar in every iteration, final weights within the bar."""
    cfg = ModelCfg(V=258, d=32, L=2, H=2, f=64, S=48)
    pc = to_px_cfg(cfg)
    w_pol = f32(ref.init_params(cfg, 21))
    w_ref = f32(ref.init_params(cfg, 22))
    w_crit = f32(ref.init_params(cfg, 23, head=True))
    w_crit[-cfg.d:] = f32(np.random.default_rng(5).normal(0, 0.1, cfg.d))
    prompts = synthetic_prompts(31, 4, 6, ragged_lengths=True)
    N, lr, kl, iters = 8, 3e-4, 0.01, 3
    ref_iters, w_pol_ref, w_crit_ref = ref.ppo_loop(cfg, w_pol, w_ref, w_crit, prompts, max_new=N, n_iters=iters,
                                                     kl_coef=kl, lr=lr, scripted_target=ord("e"), adam=ADAM)
    eng = px.Engine(px.DeviceModel(ctx, pc, w_pol, px.F32))
    refm = px.DeviceModel(ctx, pc, w_ref, px.F32)
    crit = px.DeviceModel(ctx, pc.with_head(), w_crit, px.F32)
    actor = px.Trainer(ctx, pc, w_pol, serving=eng.model, adamw=px.AdamWOptions(*ADAM))
    critic = px.Trainer(ctx, pc.with_head(), w_crit, serving=crit, adamw=px.AdamWOptions(*ADAM))
    xm = px.ExperienceMaker(eng, refm, crit, scripted_target=ord("e"), hyper=px.PpoHyper(kl, 1.0, 0.95))
    for it, r in enumerate(ref_iters):
        batch, _ = xm.run(prompts, max_new=N, sampling=px.SamplingSpec.greedy_spec(), seed=7, step_index=it)
        for i, s in enumerate(batch):
            assert np.array_equal(s.response, r["tokens"][i]), f"iteration {it}: rollout {i} differs"
            close(s.actor_logprobs, r["actor_logprobs"][i])
            close(s.values, r["values"][i])
            close(s.advantages, r["advantages"][i])
        seqs = [np.concatenate([p, s.response]).astype(np.int32) for p, s in zip(prompts, batch)]
        rs = [len(p) for p in prompts]
        la = actor.ppo_actor_step(seqs, rs, [s.actor_logprobs for s in batch], [s.advantages for s in batch],
                                  clip_eps=0.2, lr=lr)
        lc = critic.critic_step(seqs, rs, [s.values for s in batch], [s.returns for s in batch], value_clip=0.2,
                                lr=lr)
        close([la, lc], [r["actor_loss"], r["critic_loss"]])
        actor.refit()
        critic.refit()
    close(actor.flat(), w_pol_ref)
    close(critic.flat(), w_crit_ref)
