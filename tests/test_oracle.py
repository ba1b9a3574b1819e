"""The oracle restatement against the reference's golden vectors and its own
known-answer tests (CPU only).  Mirrors the reference's test pins:
tests/test_model.cpp:137-195, tests/test_losses.cpp:127-185, :248-290,
tests/acceptance.cpp:199-225."""
import numpy as np
import pytest

from oracle.oracle import EOT, ModelCfg, Oracle
from tests.golden_util import load, rows


@pytest.mark.parametrize("name", ["c1", "toy"])
def test_golden_generation_exact(oracle: Oracle, name):
    z, cfg, W, prompts = load(name, oracle)
    N = int(z["N"])
    toks, lps = oracle.generate(cfg, W["pol"], prompts, N, greedy=True)
    for t, l, gt, gl in zip(toks, lps, rows(z["greedy_tokens"], z["greedy_lens"]),
                            rows(z["greedy_lps"], z["greedy_lens"])):
        assert np.array_equal(t, gt)
        assert np.array_equal(l, gl)  # the restatement is bit-exact
    seed, step = int(z["seed"]), int(z["step_index"])
    u = np.stack([oracle.uniforms(oracle.mix_seed(seed, step * 1000003 + i), N) for i in range(len(prompts))])
    toks, lps = oracle.generate(cfg, W["pol"], prompts, N, greedy=False, temperature=0.7, uniforms=u)
    for t, l, gt, gl in zip(toks, lps, rows(z["samp_tokens"], z["samp_lens"]), rows(z["samp_lps"], z["samp_lens"])):
        assert np.array_equal(t, gt)
        assert np.array_equal(l, gl)


@pytest.mark.parametrize("name", ["c1", "toy"])
@pytest.mark.parametrize("tag", ["xs", "xr"])
def test_golden_experience(oracle: Oracle, name, tag):
    z, cfg, W, prompts = load(name, oracle)
    e = oracle.experience(cfg, W["pol"], W["ref"], W["crit"], prompts, max_new=int(z["N"]), greedy=False,
                          temperature=1.0, seed=int(z["seed"]), step_index=int(z["step_index"]),
                          kl_coef=float(z["kl_coef"]), scripted_target=int(z["scripted_target"]),
                          w_rm=W["rm"] if tag == "xr" else None)
    lens = z[f"{tag}_lens"]
    for a, b in zip(e["tokens"], rows(z[f"{tag}_tokens"], lens)):
        assert np.array_equal(a, b)
    for k in ("actor_logprobs", "ref_logprobs", "values", "advantages", "returns"):
        for a, b in zip(e[k], rows(z[f"{tag}_{k}"], lens)):
            np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)
    np.testing.assert_allclose(e["rewards"], z[f"{tag}_rewards"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", ["c1", "toy"])
def test_golden_scoring(oracle: Oracle, name):
    z, cfg, W, prompts = load(name, oracle)
    lens = z["full_lens"]
    offs = np.concatenate([[0], np.cumsum(lens)])
    full = [z["full_tokens"][offs[i]:offs[i + 1]] for i in range(len(lens))]
    slp = np.concatenate(oracle.sequence_logprobs(cfg, W["ref"], full))
    np.testing.assert_array_equal(slp, z["slp_ref"])
    vals = np.concatenate(oracle.value_estimates(cfg, W["crit"], full, [len(p) for p in prompts]))
    np.testing.assert_allclose(vals, z["values_crit"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.reward_head(cfg, W["rm"], full), z["reward_rm"], rtol=0, atol=1e-12)


def test_kv_decode_matches_full_forward(oracle: Oracle):
    # tests/test_model.cpp:137-156: every chosen log-prob equals a full forward's
    cfg = ModelCfg(258, 32, 2, 4, 64, 40)
    w = oracle.init_params(cfg, 55)
    prompt = [1, 2, 3, 4]
    toks, lps = oracle.generate(cfg, w, [prompt], 8)
    seq = list(prompt)
    for t, l in zip(toks[0], lps[0]):
        logits = oracle.forward_logits(cfg, w, seq)[-1]
        m = logits.max()
        lse = m + np.log(np.exp(logits - m).sum())
        assert abs(logits[t] - lse - l) < 1e-9
        seq.append(int(t))


def test_sequence_logprobs_vs_teacher_forced(oracle: Oracle):
    # tests/test_model.cpp:183-195
    cfg = ModelCfg(258, 32, 2, 4, 64, 40)
    w = oracle.init_params(cfg, 77)
    tokens = np.array([5, 9, 200, 17, 3, 99, 4], np.int32)
    lps = oracle.sequence_logprobs(cfg, w, [tokens])[0]
    assert lps[0] == 0.0
    logits = oracle.forward_logits(cfg, w, tokens)
    for t in range(1, len(tokens)):
        row = logits[t - 1]
        m = row.max()
        assert abs(lps[t] - (row[tokens[t]] - m - np.log(np.exp(row - m).sum()))) < 1e-9


def test_tiny_temperature_is_greedy(oracle: Oracle):
    # tests/test_model.cpp:158-165
    cfg = ModelCfg(258, 32, 2, 4, 64, 40)
    w = oracle.init_params(cfg, 55)
    g, _ = oracle.generate(cfg, w, [[5, 6, 7]], 6)
    c, _ = oracle.generate(cfg, w, [[5, 6, 7]], 6, greedy=False, temperature=1e-9, uniforms=oracle.uniforms(1234, 6))
    assert np.array_equal(g[0], c[0])


def test_gae_known_answers(oracle: Oracle):
    # tests/test_losses.cpp:248-271, tests/acceptance.cpp:199-225
    a, r = oracle.gae([1.0], [0.5], 1.0, 1.0)
    assert a[0] == pytest.approx(0.5, abs=1e-12) and r[0] == pytest.approx(1.0, abs=1e-12)
    a, _ = oracle.gae(np.zeros(5), np.zeros(5), 0.9, 0.8)
    assert np.all(a == 0)
    rng = np.random.default_rng(717)
    for _ in range(100):
        n = int(rng.integers(1, 33))
        rw, v = rng.normal(size=n), rng.normal(size=n)
        g, lam = 0.5 + 0.5 * rng.random(), 0.5 + 0.5 * rng.random()
        adv, ret = oracle.gae(rw, v, g, lam)
        delta = rw + g * np.append(v[1:], 0.0) - v
        for t in range(n):
            brute = sum((g * lam) ** (k - t) * delta[k] for k in range(t, n))
            assert abs(adv[t] - brute) <= 1e-12
            assert abs(ret[t] - (brute + v[t])) <= 1e-12


def test_kl_shaping_signs(oracle: Oracle):
    # tests/test_losses.cpp:273-290
    r = oracle.kl_penalized_rewards(3.0, [-1.0, -2.0, -0.5], [-1.0, -2.0, -0.5], 0.1)
    assert r[0] == 0.0 and r[1] == 0.0 and r[2] == pytest.approx(3.0)
    r2 = oracle.kl_penalized_rewards(0.0, [-0.5, -2.0], [-1.0, -1.5], 0.2)
    assert r2[0] < 0 and r2[1] > 0
    r3 = oracle.kl_penalized_rewards(1.5, [-0.5, -2.0], [-1.0, -1.5], 0.0)
    assert r3[0] == 0.0 and r3[1] == pytest.approx(1.5)


def test_topk_topp_filter_convention(oracle: Oracle):
    rng = np.random.default_rng(3)
    q = np.exp(rng.normal(size=300))
    assert oracle.filter_topk_topp(q, 0, 1.0).all()
    k1 = oracle.filter_topk_topp(q, 1, 1.0)
    assert k1.sum() == 1 and k1[np.argmax(q)]
    keep = oracle.filter_topk_topp(q, 0, 0.5)
    order = np.argsort(-q, kind="stable")
    csum = np.cumsum(q[order])
    n = int(np.searchsorted(csum, 0.5 * q.sum()) + 1)
    assert keep.sum() == n and keep[order[:n]].all()
    both = oracle.filter_topk_topp(q, 20, 0.9)
    top20 = order[:20]
    c20 = np.cumsum(q[top20])
    n = int(np.searchsorted(c20, 0.9 * c20[-1]) + 1)
    assert both.sum() == n and both[top20[:n]].all()
    # ties go to the lower index
    qt = np.array([1.0, 2.0, 2.0, 2.0, 0.5])
    assert list(np.nonzero(oracle.filter_topk_topp(qt, 2, 1.0))[0]) == [1, 2]


def test_sampler_reference_equivalence(oracle: Oracle):
    # k = 0, p = 1 must be the reference's inverse CDF; greedy is argmax, first index on ties
    rng = np.random.default_rng(5)
    logits = rng.normal(size=64)
    assert oracle.sample(logits, True, 1.0, 0, 1.0, 0.0) == int(np.argmax(logits))
    tie = np.array([0.0, 3.0, 3.0, 1.0])
    assert oracle.sample(tie, True, 1.0, 0, 1.0, 0.0) == 1
    p = np.exp(logits - logits.max())
    for u in (0.0, 0.1, 0.5, 0.999):
        j = int(np.argmax(u * p.sum() < np.cumsum(p)))
        assert oracle.sample(logits, False, 1.0, 0, 1.0, u) == j


def test_whitening_convention(oracle: Oracle):
    rng = np.random.default_rng(1)
    a = rng.normal(3.0, 2.0, size=1000)
    p = oracle.whiten_partials(a)
    assert p[0] == 1000 and p[1] == pytest.approx(a.sum()) and p[2] == pytest.approx((a * a).sum())
    w = oracle.whiten_apply(a, p)
    assert abs(w.mean()) < 1e-12 and w.std() == pytest.approx(1.0, rel=1e-6)
    # partials compose over shards (the cross-rank reduction)
    p2 = oracle.whiten_partials(a[:400]) + oracle.whiten_partials(a[400:])
    np.testing.assert_allclose(oracle.whiten_apply(a, p2), w, rtol=0, atol=1e-12)


def test_eot_stops_generation(oracle: Oracle):
    # generation stops after EOT and keeps it (src/model.cpp:476-478): force EOT
    # by a logit bias built into a tiny model (tok_embed row of EOT = hidden dir)
    cfg = ModelCfg(258, 16, 1, 2, 32, 24)
    w = oracle.init_params(cfg, 9)
    # make EOT the argmax everywhere: scale its embedding row strongly along
    # the final-norm bias direction
    d = cfg.d
    w[-2 * d:-d] = 0.0     # final_norm.weight = 0 -> hidden = bias
    w[-d:] = 1.0           # final_norm.bias = 1 -> hidden = ones
    w[EOT * d:(EOT + 1) * d] = 1.0
    toks, _ = oracle.generate(cfg, w, [[1, 2]], 10)
    assert list(toks[0]) == [EOT]
