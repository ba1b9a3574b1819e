"""Generates tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref/libaligner_ref.so,
compiled in place from /root/reference/proj/src by oracle/Makefile).

    make -C oracle && python tests/golden/make_golden.py

The reference ships no golden vectors, so these fixtures are
the reference's own outputs on seeded inputs.  Weights are init_params(cfg,
seed) (src/model.cpp:156-184) rounded to fp32 (parity mode) — the fixture
stores seeds plus a sha256 of the reference's unrounded init so a consumer can
regenerate identical weights with the oracle restatement and prove it did.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import ModelCfg, RefLib, synthetic_prompts  # noqa: E402

SEED = 20240809  # configs/ppo-toy.cfg:1
C1 = ModelCfg(V=1024, d=128, L=2, H=4, f=512, S=128)  # BASELINE config 1
TOY = ModelCfg(V=258, d=64, L=2, H=4, f=128, S=48)     # configs/ppo-toy.cfg model.*


def f32(w):
    return w.astype(np.float32).astype(np.float64)


def models(ref: RefLib, cfg: ModelCfg, seed: int):
    pol = ref.init_params(cfg, seed)
    refm = ref.init_params(cfg, seed + 1)
    crit = ref.init_params(cfg, seed + 101, head=True)
    rm = ref.init_params(cfg, seed + 303, head=True)
    shas = {k: sha(w) for k, w in dict(pol=pol, ref=refm, crit=crit, rm=rm).items()}
    # heads re-drawn N(0, 0.1) as the PPO rig does (tests/test_ppo.cpp:40-44)
    from oracle.oracle import Oracle
    o = Oracle(threads=1)
    crit_o = o.init_params(cfg, seed + 101, head=True, head_seed=seed + 202)
    rm_o = o.init_params(cfg, seed + 303, head=True, head_seed=seed + 404)
    assert np.array_equal(crit[:-cfg.d], crit_o[:-cfg.d]) and np.array_equal(rm[:-cfg.d], rm_o[:-cfg.d])
    crit[-cfg.d:] = crit_o[-cfg.d:]
    rm[-cfg.d:] = rm_o[-cfg.d:]
    return pol, refm, crit, rm, shas


def sha(w):
    return hashlib.sha256(np.ascontiguousarray(w, np.float64).tobytes()).hexdigest()


def pad(seqs, n, dtype):
    out = np.zeros((len(seqs), n), dtype)
    for i, s in enumerate(seqs):
        out[i, :len(s)] = s
    return out


def make(cfg: ModelCfg, name: str, B: int, P: int, N: int, step_index: int = 3, kl_coef: float = 0.01,
         scripted_target: int = 122):
    ref = RefLib()
    pol, refm, crit, rm, shas = models(ref, cfg, SEED)
    prompts = synthetic_prompts(SEED, B, P, ragged_lengths=True)
    plens = np.array([len(p) for p in prompts], np.int64)
    pflat = np.concatenate(prompts).astype(np.int32)
    W = dict(pol=f32(pol), ref=f32(refm), crit=f32(crit), rm=f32(rm))
    out = dict(cfg=np.array([cfg.V, cfg.d, cfg.L, cfg.H, cfg.f, cfg.S], np.int64), seed=np.int64(SEED),
               prompts=pflat, plens=plens, N=np.int64(N), step_index=np.int64(step_index),
               kl_coef=np.float64(kl_coef), scripted_target=np.int64(scripted_target))
    for k, h in shas.items():
        out[f"sha_{k}"] = np.array(h)
    # generation: greedy + temperature (tau 0.7, per-task mix_seed seeds)
    toks, lps, _ = ref.generate_batch(cfg, W["pol"], prompts, N, greedy=True)
    out["greedy_tokens"], out["greedy_lps"] = pad(toks, N, np.int32), pad(lps, N, np.float64)
    out["greedy_lens"] = np.array([len(t) for t in toks], np.int64)
    seeds = [ref.mix_seed(SEED, step_index * 1000003 + i) for i in range(B)]
    toks, lps, _ = ref.generate_batch(cfg, W["pol"], prompts, N, greedy=False, temperature=0.7, seeds=seeds)
    out["samp_tokens"], out["samp_lps"] = pad(toks, N, np.int32), pad(lps, N, np.float64)
    out["samp_lens"] = np.array([len(t) for t in toks], np.int64)
    # full experience (ppo_step's experience half), sampled tau = 1, scripted and RM rewards
    for tag, w_rm in (("xs", None), ("xr", W["rm"])):
        e = ref.experience(cfg, W["pol"], W["ref"], W["crit"], prompts, max_new=N, greedy=False, temperature=1.0,
                           seed=SEED, step_index=step_index, kl_coef=kl_coef, scripted_target=scripted_target,
                           w_rm=w_rm)
        out[f"{tag}_lens"] = np.array([len(t) for t in e["tokens"]], np.int64)
        out[f"{tag}_tokens"] = pad(e["tokens"], N, np.int32)
        for k in ("actor_logprobs", "ref_logprobs", "values", "advantages", "returns"):
            out[f"{tag}_{k}"] = pad(e[k], N, np.float64)
        out[f"{tag}_rewards"] = e["rewards"]
    # standalone scoring on the greedy sequences
    full = [np.concatenate([p, t]) for p, t in zip(prompts, [out["greedy_tokens"][i, :out["greedy_lens"][i]]
                                                              for i in range(B)])]
    flens = np.array([len(f) for f in full], np.int64)
    out["full_tokens"] = np.concatenate(full).astype(np.int32)
    out["full_lens"] = flens
    out["slp_ref"] = np.concatenate([ref.sequence_logprobs(cfg, W["ref"], f) for f in full])
    out["values_crit"] = np.concatenate([ref.value_estimates(cfg, W["crit"], f, len(p)) for f, p in zip(full, prompts)])
    out["reward_rm"] = np.array([ref.reward_head(cfg, W["rm"], f) for f in full])
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    make(C1, "c1", B=8, P=9, N=64)
    make(TOY, "toy", B=6, P=8, N=12, kl_coef=0.01, scripted_target=ord("e"))
