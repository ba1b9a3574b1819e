"""Parity of the CUDA path (through the C ABI) against the reference's golden
vectors and the oracle.  GPU only.

Tolerances (BASELINE.json north_star): greedy tokens, argmax indices and
sample counts bit-exact; log-probs / KL / values / advantages within
1e-3 abs + 1e-3 rel (|x - ref| <= 1e-3 + 1e-3*|ref|).
Parity mode (F32) carries the bit-exact claims; perf mode (BF16) is checked by
teacher-forced properties on the same bf16-rounded weights."""
import numpy as np
import pytest

from oracle.oracle import EOT, ModelCfg, Oracle, synthetic_prompts
from tests.golden_util import bf16_round, load, rows, to_px_cfg

pytestmark = pytest.mark.gpu

ATOL, RTOL = 1e-3, 1e-3


def close(a, b, atol=ATOL, rtol=RTOL):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    err = np.abs(a - b) - (atol + rtol * np.abs(b))
    assert a.shape == b.shape, (a.shape, b.shape)
    assert (err <= 0).all(), f"max excess {err.max():.3e}, max abs diff {np.abs(a - b).max():.3e}"
    return float(np.abs(a - b).max()) if a.size else 0.0


@pytest.fixture(scope="module")
def px():
    from paper_2405_01481_b200 import ppoexp
    ppoexp.lib()
    return ppoexp


def engine(px, ctx, cfg, w, dtype, **opts):
    return px.Engine(px.DeviceModel(ctx, to_px_cfg(cfg), w, dtype), px.EngineOptions(**opts))


# ----------------------------------------------------------------- golden (parity mode)
@pytest.mark.parametrize("name", ["c1", "toy"])
@pytest.mark.parametrize("graphs", [True, False])
def test_golden_greedy_bitexact(px, ctx, oracle, name, graphs):
    z, cfg, W, prompts = load(name, oracle)
    N = int(z["N"])
    eng = engine(px, ctx, cfg, W["pol"], px.F32, use_graphs=graphs)
    res = eng.generate_batch([px.GenTask(p, N, px.SamplingSpec.greedy_spec()) for p in prompts])
    for r, t, l in zip(res, rows(z["greedy_tokens"], z["greedy_lens"]), rows(z["greedy_lps"], z["greedy_lens"])):
        assert np.array_equal(r.tokens, t)  # argmax indices and sample counts
        close(r.logprobs, l)


@pytest.mark.parametrize("name", ["c1", "toy"])
def test_golden_sampled_tokens_exact(px, ctx, oracle, name):
    z, cfg, W, prompts = load(name, oracle)
    N, seed, step = int(z["N"]), int(z["seed"]), int(z["step_index"])
    eng = engine(px, ctx, cfg, W["pol"], px.F32)
    tasks = [px.GenTask(p, N, px.SamplingSpec.temperature_spec(0.7, oracle.mix_seed(seed, step * 1000003 + i)))
             for i, p in enumerate(prompts)]
    res = eng.generate_batch(tasks)
    for r, t, l in zip(res, rows(z["samp_tokens"], z["samp_lens"]), rows(z["samp_lps"], z["samp_lens"])):
        assert np.array_equal(r.tokens, t)
        close(r.logprobs, l)


@pytest.mark.parametrize("name", ["c1", "toy"])
@pytest.mark.parametrize("tag", ["xs", "xr"])
def test_golden_experience(px, ctx, oracle, name, tag):
    z, cfg, W, prompts = load(name, oracle)
    N = int(z["N"])
    pc = to_px_cfg(cfg)
    eng = px.Engine(px.DeviceModel(ctx, pc, W["pol"], px.F32))
    ref = px.DeviceModel(ctx, pc, W["ref"], px.F32)
    crit = px.DeviceModel(ctx, pc.with_head(), W["crit"], px.F32)
    rm = px.DeviceModel(ctx, pc.with_head(), W["rm"], px.F32) if tag == "xr" else None
    xm = px.ExperienceMaker(eng, ref, crit, rm, scripted_target=int(z["scripted_target"]),
                            hyper=px.PpoHyper(float(z["kl_coef"]), 1.0, 0.95))
    batch, st = xm.run(prompts, max_new=N, sampling=px.SamplingSpec.temperature_spec(1.0, 0),
                       seed=int(z["seed"]), step_index=int(z["step_index"]))
    lens = z[f"{tag}_lens"]
    for i, s in enumerate(batch):
        assert np.array_equal(s.response, z[f"{tag}_tokens"][i, :lens[i]])
        close(s.actor_logprobs, z[f"{tag}_actor_logprobs"][i, :lens[i]])
        close(s.ref_logprobs, z[f"{tag}_ref_logprobs"][i, :lens[i]])
        close(s.values, z[f"{tag}_values"][i, :lens[i]])
        close(s.advantages, z[f"{tag}_advantages"][i, :lens[i]])
        close(s.returns, z[f"{tag}_returns"][i, :lens[i]])
        close(s.actor_logprobs - s.ref_logprobs,
              z[f"{tag}_actor_logprobs"][i, :lens[i]] - z[f"{tag}_ref_logprobs"][i, :lens[i]])
    close([s.reward for s in batch], z[f"{tag}_rewards"])
    # kl_mean / reward_mean (src/ppo.cpp:389-392, :438-441)
    a = np.concatenate([z[f"{tag}_actor_logprobs"][i, :lens[i]] - z[f"{tag}_ref_logprobs"][i, :lens[i]]
                        for i in range(len(lens))])
    close(st.kl_mean, a.mean())
    close(st.reward_mean, z[f"{tag}_rewards"].mean())
    # whitening over all tokens: population mean 0 / std 1 (north-star convention)
    w = np.concatenate([s.whitened_advantages for s in batch])
    adv = np.concatenate([s.advantages for s in batch])
    close(w, (adv - adv.mean()) / np.sqrt(adv.var() + 1e-8), atol=1e-9, rtol=1e-9)


@pytest.mark.parametrize("name", ["c1", "toy"])
def test_golden_scoring(px, ctx, oracle, name):
    z, cfg, W, prompts = load(name, oracle)
    lens = z["full_lens"]
    offs = np.concatenate([[0], np.cumsum(lens)])
    full = [z["full_tokens"][offs[i]:offs[i + 1]] for i in range(len(lens))]
    pc = to_px_cfg(cfg)
    ref = px.DeviceModel(ctx, pc, W["ref"], px.F32)
    close(np.concatenate(px.sequence_logprobs(ref, full)), z["slp_ref"])
    crit = px.DeviceModel(ctx, pc.with_head(), W["crit"], px.F32)
    close(np.concatenate(px.value_estimates(crit, full, [len(p) for p in prompts])), z["values_crit"])
    rm = px.DeviceModel(ctx, pc.with_head(), W["rm"], px.F32)
    close(px.reward_head(rm, full), z["reward_rm"])


@pytest.mark.parametrize("name", ["c1", "toy"])
def test_golden_response_logprob_sums(px, ctx, oracle, name):
    """frozen_response_logprob_sum (src/trainers.cpp:24-29): the per-sequence sum
    of the reference-pinned sequence log-probs over the response positions."""
    z, cfg, W, prompts = load(name, oracle)
    lens = z["full_lens"]
    offs = np.concatenate([[0], np.cumsum(lens)])
    full = [z["full_tokens"][offs[i]:offs[i + 1]] for i in range(len(lens))]
    rs = [len(p) for p in prompts]
    ref = px.DeviceModel(ctx, to_px_cfg(cfg), W["ref"], px.F32)
    got = px.response_logprob_sums(ref, full, rs)
    want = []
    for i in range(len(lens)):
        acc = 0.0
        for v in z["slp_ref"][offs[i] + rs[i]:offs[i + 1]]:  # position order, as the reference accumulates
            acc += float(v)
        want.append(acc)
    close(got, want)


def test_response_logprob_sums_dpo_layout(px, ctx, oracle):
    """DPO scoring over build_sft_sequence layouts (chosen / rejected share a
    prompt; one is truncated at max_seq_len) equals the oracle's teacher-forced
    sums, and response_start outside [1, T) is a ContractError."""
    cfg = ModelCfg(V=300, d=64, L=2, H=4, f=128, S=40)
    w = oracle.init_params(cfg, 61).astype(np.float32).astype(np.float64)
    pc = to_px_cfg(cfg)
    m = px.DeviceModel(ctx, pc, w, px.F32)
    rng = np.random.default_rng(5)
    seqs, rs = [], []
    for i in range(6):
        prompt = rng.integers(0, 256, 5 + i).tolist()
        for resp_len in (3 + i, 30):  # the second overflows max_seq_len = 40 for the longer prompts
            full, r = px.build_sft_sequence(pc, prompt, rng.integers(0, 256, resp_len).tolist())
            seqs.append(full)
            rs.append(r)
    got = px.response_logprob_sums(m, seqs, rs)
    lps = oracle.sequence_logprobs(cfg, w, seqs)
    want = [float(sum(lp[r:])) for lp, r in zip(lps, rs)]
    close(got, want)
    with pytest.raises(px.ContractError, match="nonempty prompt and response"):
        px.response_logprob_sums(m, [seqs[0]], [len(seqs[0])])
    with pytest.raises(px.ContractError, match="nonempty prompt and response"):
        px.response_logprob_sums(m, [seqs[0]], [0])


# ----------------------------------------------------------------- engine semantics
def test_batch_composition_invariance(px, ctx, oracle):
    # results are index-aligned and independent of batching (tests/test_engine.cpp:213-243)
    z, cfg, W, prompts = load("c1", oracle)
    eng = engine(px, ctx, cfg, W["pol"], px.F32)
    tasks = [px.GenTask(p, 24, px.SamplingSpec.temperature_spec(1.0, 100 + i)) for i, p in enumerate(prompts)]
    together = eng.generate_batch(tasks)
    alone = [eng.generate_batch([t])[0] for t in tasks]
    for a, b in zip(together, alone):
        assert np.array_equal(a.tokens, b.tokens)
        assert np.array_equal(a.logprobs, b.logprobs)
    rev = eng.generate_batch(tasks[::-1])[::-1]
    for a, b in zip(together, rev):
        assert np.array_equal(a.tokens, b.tokens)


def test_refit_semantics(px, ctx, oracle):
    # tests/test_engine.cpp:151-211
    cfg = ModelCfg(258, 32, 2, 2, 64, 48)
    w = oracle.init_params(cfg, 43).astype(np.float32).astype(np.float64)
    eng = engine(px, ctx, cfg, w, px.F32)
    task = [px.GenTask([4, 5], 5)]
    before = eng.generate_batch(task)
    eng.refit(w)
    assert eng.generation_counter == 1
    assert np.array_equal(eng.generate_batch(task)[0].tokens, before[0].tokens)
    w2 = w.copy()
    params = px.flat_to_params(to_px_cfg(cfg), w2)
    params["layers.0.ffn.up_proj.weight"][:] += 0.01
    eng.refit(w2)
    assert eng.generation_counter == 2
    fresh = engine(px, ctx, cfg, w2, px.F32).generate_batch(task)
    got = eng.generate_batch(task)
    assert np.array_equal(got[0].tokens, fresh[0].tokens) and np.array_equal(got[0].logprobs, fresh[0].logprobs)
    t_o, l_o = oracle.generate(cfg, w2, [[4, 5]], 5)
    assert np.array_equal(got[0].tokens, t_o[0])
    # name/shape mismatch: RefitError mentioning "rebuild", engine untouched
    bad = dict(params)
    bad["layers.0.ffn.up_proj.weight"] = np.zeros((32, 32))
    with pytest.raises(px.RefitError, match="rebuild"):
        eng.refit(bad)
    missing = dict(params)
    missing.pop("final_norm.bias")
    with pytest.raises(px.RefitError, match="rebuild"):
        eng.refit(missing)
    assert eng.generation_counter == 2
    assert np.array_equal(eng.generate_batch(task)[0].tokens, got[0].tokens)


def test_contract_errors(px, ctx, oracle):
    cfg = ModelCfg(258, 32, 1, 2, 64, 16)
    w = oracle.init_params(cfg, 1)
    eng = engine(px, ctx, cfg, w, px.F32)
    with pytest.raises(px.ContractError, match="nonempty"):
        eng.generate_batch([px.GenTask([], 4)])
    with pytest.raises(px.IndexError_, match="out of range"):
        eng.generate_batch([px.GenTask([1, 999], 4)])
    with pytest.raises(px.ContractError, match="max_seq_len"):
        eng.generate_batch([px.GenTask(list(range(17)), 4)])
    assert eng.generate_batch([]) == []
    # budget = min(max_new, S - P) (src/model.cpp:447-448); greedy runs to the budget unless EOT
    r = eng.generate_batch([px.GenTask(list(range(10)), 100)])[0]
    t_o, _ = oracle.generate(cfg, w.astype(np.float32).astype(np.float64), [list(range(10))], 100)
    assert len(r.tokens) == len(t_o[0]) <= 6
    with pytest.raises(px.ContractError):
        px.value_estimates(px.DeviceModel(ctx, to_px_cfg(cfg, True), oracle.init_params(cfg, 1, head=True), px.F32),
                           [[1, 2, 3]], [3])
    bad_cfg = px.ModelConfig(258, 30, 1, 4, 64, 16)
    with pytest.raises(px.ContractError, match="divisible"):
        px.DeviceModel(ctx, bad_cfg, np.zeros(10), px.F32)


def test_eot_stops_and_is_kept(px, ctx, oracle):
    cfg = ModelCfg(258, 16, 1, 1, 32, 24)
    w = oracle.init_params(cfg, 9)
    d = cfg.d
    w[-2 * d:-d] = 0.0
    w[-d:] = 1.0
    w[EOT * d:(EOT + 1) * d] = 1.0
    eng = engine(px, ctx, cfg, w, px.F32)
    r = eng.generate_batch([px.GenTask([1, 2], 10), px.GenTask([3], 10, px.SamplingSpec.temperature_spec(0.01, 3))])
    assert list(r[0].tokens) == [EOT] and list(r[1].tokens) == [EOT]


@pytest.mark.parametrize("top_k,top_p", [(0, 0.9), (40, 1.0), (40, 0.8), (1, 1.0)])
def test_topk_topp_matches_oracle(px, ctx, oracle, top_k, top_p):
    z, cfg, W, prompts = load("c1", oracle)
    N = 32
    eng = engine(px, ctx, cfg, W["pol"], px.F32)
    seeds = [oracle.mix_seed(11, i) for i in range(len(prompts))]
    res = eng.generate_batch([px.GenTask(p, N, px.SamplingSpec.temperature_spec(1.3, s, top_k, top_p))
                              for p, s in zip(prompts, seeds)])
    u = np.stack([oracle.uniforms(s, N) for s in seeds])
    t_o, l_o = oracle.generate(cfg, W["pol"], prompts, N, greedy=False, temperature=1.3, top_k=top_k, top_p=top_p,
                               uniforms=u)
    for r, t, l in zip(res, t_o, l_o):
        assert np.array_equal(r.tokens, t)
        close(r.logprobs, l)


@pytest.mark.parametrize("top_k,top_p", [(0, 0.9), (50, 0.95), (0, 1.0)])
def test_large_vocab_sampler_matches_oracle(px, ctx, oracle, top_k, top_p):
    """A vocabulary above the per-CTA logit cache (the 128k-vocab configs take
    this path): the uncached CTA-pair sampler, token-exact against the oracle."""
    cfg = ModelCfg(V=70000, d=32, L=1, H=2, f=64, S=48)
    w = oracle.init_params(cfg, 17).astype(np.float32).astype(np.float64)
    w[:cfg.V * cfg.d] *= 40.0  # spread the logits so top-k / top-p cut inside the row
    prompts = synthetic_prompts(19, 6, 8, ragged_lengths=True)
    N = 6
    eng = engine(px, ctx, cfg, w, px.F32)
    seeds = [oracle.mix_seed(23, i) for i in range(len(prompts))]
    res = eng.generate_batch([px.GenTask(p, N, px.SamplingSpec.temperature_spec(1.0, s, top_k, top_p))
                              for p, s in zip(prompts, seeds)])
    u = np.stack([oracle.uniforms(s, N) for s in seeds])
    t_o, l_o = oracle.generate(cfg, w, prompts, N, greedy=False, top_k=top_k, top_p=top_p, uniforms=u)
    for r, t, l in zip(res, t_o, l_o):
        assert np.array_equal(r.tokens, t)
        close(r.logprobs, l)


# ----------------------------------------------------------------- perf mode (bf16)
def test_bf16_teacher_forced_parity(px, ctx, oracle):
    """bf16 weights/activations: generation log-probs must match the oracle's
    teacher-forced log-probs of the SAME tokens on the same bf16-rounded
    weights, and every greedy token must be the oracle argmax up to a near-tie."""
    z, cfg, W, prompts = load("c1", oracle)
    wb = bf16_round(W["pol"])
    eng = engine(px, ctx, cfg, wb, px.BF16)
    N = 48
    res = eng.generate_batch([px.GenTask(p, N) for p in prompts])
    full = [np.concatenate([p, r.tokens]) for p, r in zip(prompts, res)]
    slp = oracle.sequence_logprobs(cfg, wb, full)
    worst = 0.0
    for p, r, s, f in zip(prompts, res, slp, full):
        worst = max(worst, close(r.logprobs, s[len(p):], atol=2e-2, rtol=2e-3))
        logits = oracle.forward_logits(cfg, wb, f[:-1])[len(p) - 1:]
        for t, row in zip(r.tokens, logits):
            assert row[t] >= row.max() - 2e-2  # argmax up to a bf16 near-tie
    # scoring path (prefill GEMMs + K9) vs oracle on the same tokens
    m = px.DeviceModel(ctx, to_px_cfg(cfg), wb, px.BF16)
    got = px.sequence_logprobs(m, full)
    for g, s in zip(got, slp):
        close(g, s, atol=2e-2, rtol=2e-3)


def test_bf16_experience_c2_width(px, ctx, oracle):
    """Full experience step at the C2 width / vocab (125M shape, 2 layers to
    keep the fp64 oracle fast) in perf mode, checked teacher-forced."""
    cfg = ModelCfg(V=50257, d=768, L=2, H=12, f=3072, S=512)
    wp = bf16_round(oracle.init_params(cfg, 1))
    wr = bf16_round(oracle.init_params(cfg, 2))
    wc = bf16_round(oracle.init_params(cfg, 3, head=True, head_seed=4))
    prompts = synthetic_prompts(5, 4, 16, ragged_lengths=True)
    pc = to_px_cfg(cfg)
    eng = px.Engine(px.DeviceModel(ctx, pc, wp, px.BF16))
    ref = px.DeviceModel(ctx, pc, wr, px.BF16)
    crit = px.DeviceModel(ctx, pc.with_head(), wc, px.BF16)
    xm = px.ExperienceMaker(eng, ref, crit, scripted_target=ord("e"))
    batch, st = xm.run(prompts, max_new=12, sampling=px.SamplingSpec.temperature_spec(1.0, 0, 0, 0.9), seed=3)
    full = [np.concatenate([s.prompt, s.response]) for s in batch]
    rs = [len(s.prompt) for s in batch]
    a = oracle.sequence_logprobs(cfg, wp, full)
    r = oracle.sequence_logprobs(cfg, wr, full)
    v = oracle.value_estimates(cfg, wc, full, rs)
    for s, ai, ri, vi, p in zip(batch, a, r, v, rs):
        assert len(s.response) == 12
        close(s.actor_logprobs, ai[p:], atol=3e-2, rtol=3e-3)
        close(s.ref_logprobs, ri[p:], atol=3e-2, rtol=3e-3)
        close(s.values, vi, atol=3e-2, rtol=3e-2)
        shaped = oracle.kl_penalized_rewards(s.reward, s.actor_logprobs, s.ref_logprobs, 0.003)
        adv, ret = oracle.gae(shaped, s.values, 1.0, 0.95)
        close(s.advantages, adv, atol=1e-9, rtol=1e-9)  # shaping/GAE exact given the same inputs
        close(s.returns, ret, atol=1e-9, rtol=1e-9)


# ----------------------------------------------------------------- shaping kernels
def test_shape_gae_kernel_vs_oracle(px, ctx, oracle):
    rng = np.random.default_rng(0)
    B = 37
    lens = rng.integers(1, 300, size=B)
    a = [rng.normal(size=n) for n in lens]
    r = [rng.normal(size=n) for n in lens]
    v = [rng.normal(size=n) for n in lens]
    R = rng.normal(size=B)
    sh, adv, ret = px.shape_gae(ctx, R, a, r, v, 0.05, 0.99, 0.95)
    for i in range(B):
        s_o = oracle.kl_penalized_rewards(R[i], a[i], r[i], 0.05)
        a_o, r_o = oracle.gae(s_o, v[i], 0.99, 0.95)
        np.testing.assert_allclose(sh[i], s_o, rtol=0, atol=1e-13)
        np.testing.assert_allclose(adv[i], a_o, rtol=1e-12, atol=1e-11)
        np.testing.assert_allclose(ret[i], r_o, rtol=1e-12, atol=1e-11)


def test_kernel_launches_counted(px, ctx):
    assert ctx.launch_count > 0


@pytest.mark.parametrize("top_k,top_p", [(5, 1.0), (0, 0.3), (7, 0.5)])
def test_sampler_massive_ties(px, ctx, oracle, top_k, top_p):
    """All-equal logits (zero tok_embed): the crossing bucket holds the whole
    vocabulary, exercising the exact tie path; ties resolve to lower indices."""
    cfg = ModelCfg(2048, 32, 1, 2, 64, 32)
    w = oracle.init_params(cfg, 3).astype(np.float32).astype(np.float64)
    w[:cfg.V * cfg.d] = 0.0  # tied head → every logit is 0
    eng = engine(px, ctx, cfg, w, px.F32)
    seeds = [oracle.mix_seed(2, i) for i in range(4)]
    prompts = [[1, 2, 3], [4], [5, 6], [7, 8, 9, 10]]
    res = eng.generate_batch([px.GenTask(p, 6, px.SamplingSpec.temperature_spec(1.0, s, top_k, top_p))
                              for p, s in zip(prompts, seeds)])
    u = np.stack([oracle.uniforms(s, 6) for s in seeds])
    t_o, _ = oracle.generate(cfg, w, prompts, 6, greedy=False, top_k=top_k, top_p=top_p, uniforms=u)
    for r, t in zip(res, t_o):
        assert np.array_equal(r.tokens, t)


def test_bf16_fused_layernorm_matches_unfused(px, ctx, oracle, monkeypatch):
    """The decode path's fused LayerNorm (fixed-point row statistics accumulated
    by the residual producers + on-the-fly normalisation in the consumer GEMMs)
    against the standalone LN kernels."""
    cfg = ModelCfg(V=4096, d=256, L=3, H=4, f=1024, S=128)
    wb = bf16_round(oracle.init_params(cfg, 21))
    prompts = synthetic_prompts(8, 16, 12, ragged_lengths=True)
    outs = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("PPOEXP_FUSE_LN", flag)
        eng = engine(px, ctx, cfg, wb, px.BF16)
        outs[flag] = eng.generate_batch([px.GenTask(p, 40) for p in prompts])
    same = 0
    for a, b, p in zip(outs["0"], outs["1"], prompts):
        n = 0
        while n < min(len(a.tokens), len(b.tokens)) and a.tokens[n] == b.tokens[n]:
            n += 1
        same += n == len(a.tokens)
        close(b.logprobs[:n], a.logprobs[:n], atol=2e-2, rtol=2e-3)
        # and the fused run is itself consistent with the oracle, teacher-forced
        full = np.concatenate([p, b.tokens])
        lp = oracle.sequence_logprobs(cfg, wb, [full])[0][len(p):]
        close(b.logprobs, lp, atol=3e-2, rtol=3e-3)
    assert same >= len(prompts) // 2


def test_bf16_decode_batch_above_fused_ln_limit(px, ctx, oracle):
    """Decode batches above 64 take the standalone-LayerNorm path (the fused
    LayerNorm is the default only up to 64 rows): teacher-forced against the
    oracle, and the first 64 rows agree with a 64-row batch of the same tasks."""
    cfg = ModelCfg(V=2048, d=256, L=2, H=4, f=1024, S=96)
    wb = bf16_round(oracle.init_params(cfg, 71))
    prompts = synthetic_prompts(43, 100, 10, ragged_lengths=True)
    tasks = [px.GenTask(p, 24) for p in prompts]
    eng = engine(px, ctx, cfg, wb, px.BF16)
    big = eng.generate_batch(tasks)
    for r, p in zip(big[::7], prompts[::7]):
        full = np.concatenate([p, r.tokens])
        lp = oracle.sequence_logprobs(cfg, wb, [full])[0][len(p):]
        close(r.logprobs, lp, atol=3e-2, rtol=3e-3)
    small = eng.generate_batch(tasks[:64])
    same = sum(int(np.array_equal(a.tokens, b.tokens)) for a, b in zip(big[:64], small))
    assert same >= 32


@pytest.mark.parametrize("fuse_ln", ["0", "1"])
def test_bf16_decode_is_deterministic(px, ctx, oracle, monkeypatch, fuse_ln):
    """bf16 decode (split-K decode GEMMs with the direct DSMEM push reduction and
    no exit barrier; optionally the fused LayerNorm with atomically accumulated
    fixed-point row statistics) is bitwise reproducible: a lost, late or
    reordered partial would show up as run-to-run differences in tokens or log-probs."""
    monkeypatch.setenv("PPOEXP_FUSE_LN", fuse_ln)
    cfg = ModelCfg(V=4096, d=768, L=2, H=12, f=3072, S=128)
    wb = bf16_round(oracle.init_params(cfg, 29))
    prompts = synthetic_prompts(31, 64, 16, ragged_lengths=True)
    tasks = [px.GenTask(p, 40, px.SamplingSpec.temperature_spec(1.0, 1000 + i, 0, 0.9)) for i, p in enumerate(prompts)]
    runs = []
    for _ in range(3):
        eng = engine(px, ctx, cfg, wb, px.BF16)
        runs.append(eng.generate_batch(tasks))
    for r in runs[1:]:
        for a, b in zip(runs[0], r):
            assert np.array_equal(a.tokens, b.tokens)
            assert np.array_equal(a.logprobs, b.logprobs)


# ----------------------------------------------------------------- mixed mode (the parity-grade fast path)
# bf16 weights (the same bf16-rounded weights on both sides: "identical weights"),
# fp32 activations / KV, tensor-core products on a two-term bf16 split of every
# activation.  Held to the north_star bar exactly: greedy / sampled tokens and
# sample counts bit-exact, log-probs / KL / values / advantages within
# 1e-3 abs + 1e-3 rel (ATOL, RTOL above).

def _mixed_experience_check(px, ctx, oracle, cfg, prompts, N, seed=3, kl=0.003, tol_scale=1.0):
    wp = bf16_round(oracle.init_params(cfg, seed))
    wr = bf16_round(oracle.init_params(cfg, seed + 1))
    wc = bf16_round(oracle.init_params(cfg, seed + 2, head=True, head_seed=seed + 3))
    pc = to_px_cfg(cfg)
    eng = px.Engine(px.DeviceModel(ctx, pc, wp, px.MIXED))
    ref = px.DeviceModel(ctx, pc, wr, px.MIXED)
    crit = px.DeviceModel(ctx, pc.with_head(), wc, px.MIXED)
    xm = px.ExperienceMaker(eng, ref, crit, scripted_target=ord("e"), hyper=px.PpoHyper(kl, 1.0, 0.95))
    batch, st = xm.run(prompts, max_new=N, sampling=px.SamplingSpec.greedy_spec(), seed=seed)
    exp = oracle.experience(cfg, wp, wr, wc, prompts, max_new=N, greedy=True, kl_coef=kl, scripted_target=ord("e"))
    worst = {}
    for i, s in enumerate(batch):
        assert np.array_equal(s.response, exp["tokens"][i]), f"greedy rollout {i} differs from the oracle"
        for k, got, want in (("actor_lp", s.actor_logprobs, exp["actor_logprobs"][i]),
                             ("ref_lp", s.ref_logprobs, exp["ref_logprobs"][i]),
                             ("kl", s.actor_logprobs - s.ref_logprobs,
                              exp["actor_logprobs"][i] - exp["ref_logprobs"][i]),
                             ("values", s.values, exp["values"][i]), ("advantages", s.advantages, exp["advantages"][i]),
                             ("returns", s.returns, exp["returns"][i]), ("whitened", s.whitened_advantages,
                                                                         exp["whitened"][i])):
            worst[k] = max(worst.get(k, 0.0), close(got, want, ATOL * tol_scale, RTOL * tol_scale))
    close([s.reward for s in batch], exp["rewards"], 0, 0)  # scripted counts: exact
    close(st.kl_mean, exp["kl_mean"])
    close(st.reward_mean, exp["reward_mean"], 0, 0)
    eng.close()
    return worst


@pytest.mark.parametrize("lanes", ["1", "2"])
def test_mixed_experience_c1(px, ctx, oracle, monkeypatch, lanes):
    # lanes=2: the 8 prompts decode as two 4-sequence lanes on separate streams
    monkeypatch.setenv("PPOEXP_LANES", lanes)
    monkeypatch.setenv("PPOEXP_LANE_MIN_B", "2")
    cfg = ModelCfg(V=1024, d=128, L=2, H=4, f=512, S=128)
    _mixed_experience_check(px, ctx, oracle, cfg, synthetic_prompts(7, 8, 9, ragged_lengths=True), 64)


def test_mixed_experience_c2_full_depth(px, ctx, oracle):
    """The benchmarked C2 shape at full depth (12 layers, d 768, vocab 50257)."""
    cfg = ModelCfg(V=50257, d=768, L=12, H=12, f=3072, S=512)
    w = _mixed_experience_check(px, ctx, oracle, cfg, synthetic_prompts(5, 4, 16, ragged_lengths=True), 24)
    print("c2 worst abs errors", w)


@pytest.mark.parametrize("shape", ["c3", "c4"])
def test_mixed_experience_wide(px, ctx, oracle, shape):
    """C3 width (d 2048, vocab 32000) and C4 width (d 4096, vocab 128256, the
    uncached large-vocab sampler), one layer to keep the fp64 oracle short."""
    cfg = (ModelCfg(V=32000, d=2048, L=1, H=16, f=8192, S=1024) if shape == "c3"
           else ModelCfg(V=128256, d=4096, L=1, H=32, f=14336, S=2048))
    n_new = 8 if shape == "c3" else 4  # the fp64 oracle at d 4096 / vocab 128k dominates the test time
    _mixed_experience_check(px, ctx, oracle, cfg, synthetic_prompts(9, 2, 8 if shape == "c3" else 6,
                                                                    ragged_lengths=True), n_new)


@pytest.mark.parametrize("top_k,top_p,tau", [(0, 1.0, 0.7), (0, 0.9, 1.0), (40, 0.95, 1.3)])
def test_mixed_sampled_tokens_exact(px, ctx, oracle, top_k, top_p, tau):
    """Temperature / top-k / top-p sampling (one mt19937_64 uniform per token):
    tokens and sample counts bit-exact against the oracle on the same weights."""
    cfg = ModelCfg(V=1024, d=128, L=2, H=4, f=512, S=128)
    w = bf16_round(oracle.init_params(cfg, 13))
    w[:cfg.V * cfg.d] *= 20.0  # sharpen the distribution so the filters cut inside the row
    w = bf16_round(w)
    prompts = synthetic_prompts(17, 8, 9, ragged_lengths=True)
    N = 40
    eng = engine(px, ctx, cfg, w, px.MIXED)
    seeds = [oracle.mix_seed(29, i) for i in range(len(prompts))]
    res = eng.generate_batch([px.GenTask(p, N, px.SamplingSpec.temperature_spec(tau, s, top_k, top_p))
                              for p, s in zip(prompts, seeds)])
    u = np.stack([oracle.uniforms(s, N) for s in seeds])
    t_o, l_o = oracle.generate(cfg, w, prompts, N, greedy=False, temperature=tau, top_k=top_k, top_p=top_p,
                               uniforms=u)
    for r, t, l in zip(res, t_o, l_o):
        assert np.array_equal(r.tokens, t)
        close(r.logprobs, l)


def test_mixed_response_logprob_sums(px, ctx, oracle):
    """DPO scoring sums (frozen_response_logprob_sum, src/trainers.cpp:24-29) at
    the C2 width / vocab through the fused LM-head + LSE epilogue."""
    cfg = ModelCfg(V=50257, d=768, L=2, H=12, f=3072, S=512)
    w = bf16_round(oracle.init_params(cfg, 31))
    m = px.DeviceModel(ctx, to_px_cfg(cfg), w, px.MIXED)
    rng = np.random.default_rng(3)
    seqs, rs = [], []
    for i in range(6):
        full, r = px.build_sft_sequence(to_px_cfg(cfg), rng.integers(0, 256, 5 + 3 * i).tolist(),
                                        rng.integers(0, 256, 4 + 5 * i).tolist())
        seqs.append(full)
        rs.append(r)
    got = px.response_logprob_sums(m, seqs, rs)
    lps = oracle.sequence_logprobs(cfg, w, seqs)
    close(got, [float(sum(lp[r:])) for lp, r in zip(lps, rs)])
    close(np.concatenate(px.sequence_logprobs(m, seqs)), np.concatenate(lps))


@pytest.mark.parametrize("d,H", [(768, 12), (1024, 8), (2048, 16)])
def test_mixed_scoring_many_rows(px, ctx, oracle, d, H):
    """Scoring batches of >= 1024 packed rows take the warp-per-row split
    LayerNorm and the persistent planes GEMM (every epilogue: fp32 store,
    residual reduce-add, GELU planes, LSE): log-probs at the bar against the
    oracle (small vocab keeps the fp64 oracle fast)."""
    cfg = ModelCfg(V=1031, d=d, L=2, H=H, f=4 * d, S=256)
    w = bf16_round(oracle.init_params(cfg, 7 + d))
    m = px.DeviceModel(ctx, to_px_cfg(cfg), w, px.MIXED)
    rng = np.random.default_rng(d)
    seqs = [rng.integers(0, 1031, int(n)).astype(np.int32) for n in rng.integers(60, 140, 14)]
    assert sum(len(q) for q in seqs) >= 1024
    close(np.concatenate(px.sequence_logprobs(m, seqs)), np.concatenate(oracle.sequence_logprobs(cfg, w, seqs)))


@pytest.mark.parametrize("dtype", ["mixed", "bf16"])
def test_fused_ln_statistics_with_outliers(px, ctx, oracle, dtype):
    """1e3-magnitude outlier features at d = 4096 (massive activations): the
    fused-LayerNorm fixed-point row statistics stay in range and the decode
    matches the oracle teacher-forced (mixed: within the north_star bar)."""
    cfg = ModelCfg(V=2048, d=4096, L=1, H=32, f=1024, S=64)
    w = oracle.init_params(cfg, 37)
    pos0 = cfg.V * cfg.d
    for p_ in range(cfg.S):  # 8 outlier features of magnitude ~1e3 in every position
        w[pos0 + p_ * cfg.d + np.arange(0, 4096, 512)] = 1000.0 * (1 + 0.01 * p_)
    w = bf16_round(w)
    prompts = synthetic_prompts(41, 4, 6, ragged_lengths=True)
    eng = engine(px, ctx, cfg, w, px.MIXED if dtype == "mixed" else px.BF16)
    res = eng.generate_batch([px.GenTask(p, 12) for p in prompts])
    for r, p in zip(res, prompts):
        lp = oracle.sequence_logprobs(cfg, w, [np.concatenate([p, r.tokens])])[0][len(p):]
        if dtype == "mixed":
            close(r.logprobs, lp)
        else:
            close(r.logprobs, lp, atol=5e-2, rtol=5e-3)


def test_fused_ln_statistics_overflow_is_an_error(px, ctx, oracle):
    """A residual stream beyond the fixed-point range fails loudly (no silent clamp)."""
    cfg = ModelCfg(V=512, d=256, L=1, H=4, f=512, S=32)
    w = oracle.init_params(cfg, 43)
    pos0 = cfg.V * cfg.d
    w[pos0:pos0 + cfg.S * cfg.d] = 3.0e5
    eng = engine(px, ctx, cfg, bf16_round(w), px.BF16)
    with pytest.raises(px.ContractError, match="statistics range"):
        eng.generate_batch([px.GenTask([1, 2, 3], 4)])


def test_large_vocab_uncached_sampler_branch(px, ctx, oracle):
    """Vocab 128256 > 2 x the per-CTA logit cache: the uncached CTA-pair sampler
    (sampler_kernel<false, 2>, the config-4 path), token-exact vs the oracle."""
    cfg = ModelCfg(V=128256, d=32, L=1, H=2, f=64, S=48)
    w = oracle.init_params(cfg, 17).astype(np.float32).astype(np.float64)
    w[:cfg.V * cfg.d] *= 40.0
    prompts = synthetic_prompts(19, 6, 8, ragged_lengths=True)
    N = 6
    import ctypes
    f = px.lib().ppoexp_testing_variant_count
    f.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p]
    n0 = ctypes.c_int64()
    px._check(f(ctx.h, b"sampler:pair_uncached", ctypes.byref(n0)))
    eng = engine(px, ctx, cfg, w, px.F32)
    for top_k, top_p in ((0, 0.9), (50, 0.95), (0, 1.0)):
        seeds = [oracle.mix_seed(23 + top_k, i) for i in range(len(prompts))]
        res = eng.generate_batch([px.GenTask(p, N, px.SamplingSpec.temperature_spec(1.0, s, top_k, top_p))
                                  for p, s in zip(prompts, seeds)])
        u = np.stack([oracle.uniforms(s, N) for s in seeds])
        t_o, l_o = oracle.generate(cfg, w, prompts, N, greedy=False, top_k=top_k, top_p=top_p, uniforms=u)
        for r, t, l in zip(res, t_o, l_o):
            assert np.array_equal(r.tokens, t)
            close(r.logprobs, l)
    n1 = ctypes.c_int64()
    px._check(f(ctx.h, b"sampler:pair_uncached", ctypes.byref(n1)))
    assert n1.value > n0.value, "the uncached CTA-pair sampler branch did not run"


def test_device_token_ids_are_validated(px, ctx, oracle):
    """Out-of-range ids in DEVICE-resident inputs raise IndexError (a device
    validation kernel) instead of reading out of bounds (the reference throws
    IndexError, src/model.cpp:284-287)."""
    import torch
    cfg = ModelCfg(258, 32, 1, 2, 64, 32)
    m = px.DeviceModel(ctx, to_px_cfg(cfg), oracle.init_params(cfg, 5), px.BF16)
    toks = torch.tensor([1, 2, 3, 300, 4], dtype=torch.int32, device="cuda")
    offs = torch.tensor([0, 5], dtype=torch.int64, device="cuda")
    out = torch.zeros(5, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    rc = px.lib().ppoexp_sequence_logprobs(m.h, 1, toks.data_ptr(), offs.data_ptr(), out.data_ptr(), px.DEVICE)
    with pytest.raises(px.IndexError_, match="position 3"):
        px._check(rc)
    # the context stays usable
    assert len(px.sequence_logprobs(m, [[1, 2, 3]])[0]) == 3


@pytest.mark.parametrize("dtype", ["bf16", "mixed"])
def test_dpo_sums_c5_width(px, ctx, oracle, dtype):
    """DPO chosen / rejected sums at the C5 width and vocab (d 4096, V 128256),
    one layer: both compute modes within 1e-3 + 1e-3 |sum| of the oracle
    (the sums are what the DPO loss consumes, src/trainers.cpp:54-80)."""
    cfg = ModelCfg(V=128256, d=4096, L=1, H=32, f=14336, S=64)
    w = bf16_round(oracle.init_params(cfg, 47))
    m = px.DeviceModel(ctx, to_px_cfg(cfg), w, px.MIXED if dtype == "mixed" else px.BF16)
    rng = np.random.default_rng(8)
    seqs, rs = [], []
    for i in range(1):
        prompt = rng.integers(0, 256, 10).tolist()
        for _ in range(2):  # chosen, rejected
            full, r = px.build_sft_sequence(to_px_cfg(cfg), prompt, rng.integers(0, 256, 14).tolist())
            seqs.append(full)
            rs.append(r)
    got = px.response_logprob_sums(m, seqs, rs)
    lps = oracle.sequence_logprobs(cfg, w, seqs)
    close(got, [float(sum(lp[r:])) for lp, r in zip(lps, rs)])


@pytest.mark.parametrize("planes", ["0", "1"])
def test_mixed_decode_activation_paths(px, ctx, oracle, monkeypatch, planes):
    """Mixed decode with the LayerNorm fused into the consumer GEMMs (planes=0,
    the narrow-model default) and with split LayerNorm / attention / GELU
    producers writing bf16 hi|lo planes that the GEMMs TMA (planes=1, the
    wide-model default): both meet the bar at the C2 width."""
    monkeypatch.setenv("PPOEXP_MIXED_PLANES", planes)
    cfg = ModelCfg(V=50257, d=768, L=2, H=12, f=3072, S=512)
    _mixed_experience_check(px, ctx, oracle, cfg, synthetic_prompts(3, 4, 12, ragged_lengths=True), 16)


@pytest.mark.parametrize("dtype", ["MIXED"])
@pytest.mark.parametrize("graphs", [True, False])
def test_decode_lanes_match_single_lane(px, ctx, oracle, monkeypatch, dtype, graphs):
    """The two-lane decode (half batches on two streams, pages from one pool)
    gives exactly the tokens / log-probs / lengths of the single-lane engine
    (mixed mode: batch-composition invariant; bf16 activations are not, and
    its sampled tokens may flip on rounding-level differences):
    ragged prompts, mixed budgets (chunks of max_batch=24 over 41 tasks), greedy
    and top-p rows, EOT stops."""
    cfg = ModelCfg(V=1031, d=256, L=2, H=4, f=1024, S=160)
    w = oracle.init_params(cfg, 11)
    prompts = synthetic_prompts(21, 41, 24, ragged_lengths=True)
    tasks = []
    for i, p in enumerate(prompts):
        sp = (px.SamplingSpec.greedy_spec() if i % 3 == 0
              else px.SamplingSpec.temperature_spec(1.3, 500 + i, 0, 0.95))
        tasks.append(px.GenTask(p, [40, 7, 23, 1, 64][i % 5], sp))
    res = {}
    monkeypatch.setenv("PPOEXP_LANE_MIN_B", "8")
    for lanes in ("1", "2"):
        monkeypatch.setenv("PPOEXP_LANES", lanes)
        eng = engine(px, ctx, cfg, w, getattr(px, dtype), use_graphs=graphs, max_batch=24)
        res[lanes] = eng.generate_batch(tasks)
        eng.close()
    for a, b in zip(res["1"], res["2"]):
        assert np.array_equal(a.tokens, b.tokens)
        assert np.array_equal(a.logprobs, b.logprobs)
