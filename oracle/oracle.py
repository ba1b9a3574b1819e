"""ctypes front-end for the CPU checkers.  TEST INFRASTRUCTURE ONLY.

* ``Oracle`` wraps ``oracle/libppoexp_oracle.so`` — the C restatement of the
  reference's experience path (oracle/ppoexp_oracle.c).
* ``RefLib`` wraps ``oracle/_ref/libaligner_ref.so`` — the UNMODIFIED
  reference sources compiled in place (oracle/Makefile + oracle/ref_shim.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference
arm may import this module; the product package never does.

All model weights are numpy float64 arrays in the "flat canonical" layout
(``ModelParams::expected_names`` order, /root/reference/proj/src/model.cpp:66-90).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libppoexp_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libaligner_ref.so")

PAD, EOT = 256, 257  # include/aligner/model.hpp:17-18


@dataclass(frozen=True)
class ModelCfg:
    V: int
    d: int
    L: int
    H: int
    f: int
    S: int

    def as6(self):
        return (C.c_int64 * 6)(self.V, self.d, self.L, self.H, self.f, self.S)


class _OrcCfg(C.Structure):
    _fields_ = [("V", C.c_int64), ("d", C.c_int64), ("L", C.c_int64), ("H", C.c_int64),
                ("f", C.c_int64), ("S", C.c_int64), ("scalar_head", C.c_int32)]


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


D = C.c_double
I32 = C.c_int32
I64 = C.c_int64


def ensure_built():
    if not os.path.exists(ORACLE_SO):
        subprocess.check_call(["make", "-s", "-C", HERE, os.path.join(HERE, "libppoexp_oracle.so")])


def ragged(seqs):
    """list of int sequences -> (int32 flat, int64 offsets[B+1])"""
    offs = np.zeros(len(seqs) + 1, np.int64)
    offs[1:] = np.cumsum([len(s) for s in seqs])
    flat = np.concatenate([np.asarray(s, np.int32) for s in seqs]) if seqs else np.zeros(0, np.int32)
    return np.ascontiguousarray(flat, np.int32), offs


class Oracle:
    def __init__(self, threads: int | None = None):
        ensure_built()
        self.lib = C.CDLL(ORACLE_SO)
        L = self.lib
        L.orc_param_count.restype = I64
        L.orc_mix_seed.restype = C.c_uint64
        L.orc_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_uniforms.argtypes = [C.c_uint64, I64, C.POINTER(D)]
        L.orc_init_params.argtypes = [C.POINTER(_OrcCfg), C.c_uint64, C.POINTER(D)]
        L.orc_redraw_head.argtypes = [C.POINTER(_OrcCfg), C.POINTER(D), C.c_uint64, D]
        L.orc_generate.restype = I64
        L.orc_sample.restype = I64
        L.orc_sample.argtypes = [C.POINTER(D), I64, C.c_int, D, I64, D, D]
        L.orc_filter_topk_topp.argtypes = [C.POINTER(D), I64, I64, D, C.POINTER(C.c_ubyte)]
        L.orc_scripted_reward.restype = D
        L.orc_scripted_reward.argtypes = [C.POINTER(I32), I64, I64, I32]
        L.orc_kl_penalized_rewards.argtypes = [D, C.POINTER(D), C.POINTER(D), I64, D, C.POINTER(D)]
        L.orc_gae.argtypes = [C.POINTER(D), C.POINTER(D), I64, D, D, C.POINTER(D), C.POINTER(D)]
        L.orc_batch_generate.argtypes = [C.POINTER(_OrcCfg), C.POINTER(D), C.POINTER(I32), C.POINTER(I64),
                                         I64, I64, C.c_int, D, I64, D, C.POINTER(D), C.POINTER(I32),
                                         C.POINTER(D), C.POINTER(I64)]
        L.orc_batch_sequence_logprobs.argtypes = [C.POINTER(_OrcCfg), C.POINTER(D), C.POINTER(I32),
                                                  C.POINTER(I64), I64, C.POINTER(D)]
        L.orc_batch_value_estimates.argtypes = [C.POINTER(_OrcCfg), C.POINTER(D), C.POINTER(D), C.POINTER(I32),
                                                C.POINTER(I64), C.POINTER(I64), I64, C.POINTER(I64), C.POINTER(D)]
        L.orc_batch_reward_head.argtypes = [C.POINTER(_OrcCfg), C.POINTER(D), C.POINTER(D), C.POINTER(I32),
                                            C.POINTER(I64), I64, C.POINTER(D)]
        L.orc_forward_hidden.argtypes = [C.POINTER(_OrcCfg), C.POINTER(D), C.POINTER(I32), I64, C.POINTER(D)]
        L.orc_forward_logits.argtypes = [C.POINTER(_OrcCfg), C.POINTER(D), C.POINTER(I32), I64, C.POINTER(D)]
        L.orc_set_threads.argtypes = [C.c_int]
        L.orc_whiten_partials.argtypes = [C.POINTER(D), I64, C.POINTER(D)]
        L.orc_whiten_apply.argtypes = [C.POINTER(D), I64, C.POINTER(D), C.POINTER(D)]
        L.orc_set_threads(threads or os.cpu_count() or 1)

    @staticmethod
    def _cfg(cfg: ModelCfg, head: bool):
        return C.byref(_OrcCfg(cfg.V, cfg.d, cfg.L, cfg.H, cfg.f, cfg.S, 1 if head else 0))

    def param_count(self, cfg: ModelCfg, head=False) -> int:
        return self.lib.orc_param_count(self._cfg(cfg, head))

    def init_params(self, cfg: ModelCfg, seed: int, head=False, head_seed=None, head_sigma=0.1):
        w = np.empty(self.param_count(cfg, head), np.float64)
        self.lib.orc_init_params(self._cfg(cfg, head), seed, _p(w, D))
        if head and head_seed is not None:
            self.lib.orc_redraw_head(self._cfg(cfg, head), _p(w, D), head_seed, head_sigma)
        return w

    def mix_seed(self, a, b):
        return int(self.lib.orc_mix_seed(a, b))

    def uniforms(self, seed, n):
        out = np.empty(n, np.float64)
        self.lib.orc_uniforms(seed, n, _p(out, D))
        return out

    def generate(self, cfg, w, prompts, max_new, greedy=True, temperature=1.0, top_k=0, top_p=1.0,
                 uniforms=None):
        """Batched generate(); returns (tokens list, logprob list)."""
        flat, offs = ragged(prompts)
        B = len(prompts)
        toks = np.zeros((B, max_new), np.int32)
        lps = np.zeros((B, max_new), np.float64)
        n = np.zeros(B, np.int64)
        u = None
        if not greedy:
            u = np.ascontiguousarray(uniforms, np.float64).reshape(B, max_new)
        rc = self.lib.orc_batch_generate(self._cfg(cfg, False), _p(w, D), _p(flat, I32), _p(offs, I64), B, max_new,
                                         1 if greedy else 0, temperature, top_k, top_p,
                                         _p(u, D) if u is not None else None, _p(toks, I32), _p(lps, D),
                                         _p(n, I64))
        if rc:
            raise RuntimeError("oracle generate failed")
        return [toks[b, :n[b]].copy() for b in range(B)], [lps[b, :n[b]].copy() for b in range(B)]

    def sequence_logprobs(self, cfg, w, seqs):
        flat, offs = ragged(seqs)
        out = np.zeros(len(flat), np.float64)
        if self.lib.orc_batch_sequence_logprobs(self._cfg(cfg, False), _p(w, D), _p(flat, I32), _p(offs, I64),
                                                len(seqs), _p(out, D)):
            raise RuntimeError("oracle sequence_logprobs failed")
        return [out[offs[b]:offs[b + 1]].copy() for b in range(len(seqs))]

    def value_estimates(self, cfg, w, seqs, response_starts):
        flat, offs = ragged(seqs)
        rs = np.asarray(response_starts, np.int64)
        lens = np.array([len(s) for s in seqs], np.int64) - rs
        oo = np.zeros(len(seqs) + 1, np.int64)
        oo[1:] = np.cumsum(lens)
        out = np.zeros(int(oo[-1]), np.float64)
        head = np.ascontiguousarray(w[-cfg.d:])
        if self.lib.orc_batch_value_estimates(self._cfg(cfg, True), _p(w, D), _p(head, D), _p(flat, I32),
                                              _p(offs, I64), _p(rs, I64), len(seqs), _p(oo, I64), _p(out, D)):
            raise RuntimeError("oracle value_estimates failed")
        return [out[oo[b]:oo[b + 1]].copy() for b in range(len(seqs))]

    def reward_head(self, cfg, w, seqs):
        flat, offs = ragged(seqs)
        out = np.zeros(len(seqs), np.float64)
        head = np.ascontiguousarray(w[-cfg.d:])
        if self.lib.orc_batch_reward_head(self._cfg(cfg, True), _p(w, D), _p(head, D), _p(flat, I32),
                                          _p(offs, I64), len(seqs), _p(out, D)):
            raise RuntimeError("oracle reward_head failed")
        return out

    def forward_hidden(self, cfg, w, tokens, head=False):
        t = np.asarray(tokens, np.int32)
        out = np.zeros((len(t), cfg.d), np.float64)
        if self.lib.orc_forward_hidden(self._cfg(cfg, head), _p(w, D), _p(t, I32), len(t), _p(out, D)):
            raise RuntimeError("oracle forward failed")
        return out

    def forward_logits(self, cfg, w, tokens):
        t = np.asarray(tokens, np.int32)
        out = np.zeros((len(t), cfg.V), np.float64)
        if self.lib.orc_forward_logits(self._cfg(cfg, False), _p(w, D), _p(t, I32), len(t), _p(out, D)):
            raise RuntimeError("oracle forward failed")
        return out

    def sample(self, logits, greedy, temperature, top_k, top_p, u):
        l = np.ascontiguousarray(logits, np.float64)
        return int(self.lib.orc_sample(_p(l, D), len(l), 1 if greedy else 0, temperature, top_k, top_p, u))

    def filter_topk_topp(self, q, top_k, top_p):
        q = np.ascontiguousarray(q, np.float64)
        keep = np.zeros(len(q), np.uint8)
        self.lib.orc_filter_topk_topp(_p(q, D), len(q), top_k, top_p, _p(keep, C.c_ubyte))
        return keep.astype(bool)

    def scripted_reward(self, tokens, rs, target):
        t = np.asarray(tokens, np.int32)
        return float(self.lib.orc_scripted_reward(_p(t, I32), len(t), rs, target))

    def kl_penalized_rewards(self, rm, a, r, coef):
        a = np.ascontiguousarray(a, np.float64)
        r = np.ascontiguousarray(r, np.float64)
        out = np.zeros(len(a), np.float64)
        if self.lib.orc_kl_penalized_rewards(rm, _p(a, D), _p(r, D), len(a), coef, _p(out, D)):
            raise RuntimeError("kl_penalized_rewards: empty")
        return out

    def gae(self, rw, v, gamma, lam):
        rw = np.ascontiguousarray(rw, np.float64)
        v = np.ascontiguousarray(v, np.float64)
        adv = np.zeros(len(rw), np.float64)
        ret = np.zeros(len(rw), np.float64)
        self.lib.orc_gae(_p(rw, D), _p(v, D), len(rw), gamma, lam, _p(adv, D), _p(ret, D))
        return adv, ret

    def whiten_partials(self, adv):
        a = np.ascontiguousarray(adv, np.float64)
        p = np.zeros(3, np.float64)
        self.lib.orc_whiten_partials(_p(a, D), len(a), _p(p, D))
        return p

    def whiten_apply(self, adv, part3):
        a = np.ascontiguousarray(adv, np.float64)
        p = np.ascontiguousarray(part3, np.float64)
        out = np.zeros(len(a), np.float64)
        self.lib.orc_whiten_apply(_p(a, D), len(a), _p(p, D), _p(out, D))
        return out

    # ---------------------------------------------------------------- PPO
    def experience(self, cfg, w_policy, w_ref, w_critic, prompts, *, max_new, greedy, temperature=1.0,
                   top_k=0, top_p=1.0, seed=0, step_index=0, gidx0=0, kl_coef=0.003, gamma=1.0, lam=0.95,
                   scripted_target=122, w_rm=None):
        """The experience part of ppo_step (src/ppo.cpp:302-393) plus whitening."""
        B = len(prompts)
        u = None
        if not greedy:
            u = np.stack([self.uniforms(self.mix_seed(seed, step_index * 1000003 + gidx0 + i), max_new)
                          for i in range(B)])
        toks, gen_lps = self.generate(cfg, w_policy, prompts, max_new, greedy, temperature, top_k, top_p, u)
        full = [np.concatenate([np.asarray(p, np.int32), t]) for p, t in zip(prompts, toks)]
        rs = [len(p) for p in prompts]
        a_all = self.sequence_logprobs(cfg, w_policy, full)
        r_all = self.sequence_logprobs(cfg, w_ref, full)
        actor = [a[s:] for a, s in zip(a_all, rs)]
        ref = [r[s:] for r, s in zip(r_all, rs)]
        values = self.value_estimates(cfg, w_critic, full, rs)
        if w_rm is None:
            rewards = np.array([self.scripted_reward(f, s, scripted_target) for f, s in zip(full, rs)])
        else:
            rewards = self.reward_head(cfg, w_rm, full)
        adv, ret = [], []
        for i in range(B):
            shaped = self.kl_penalized_rewards(rewards[i], actor[i], ref[i], kl_coef)
            a, r = self.gae(shaped, values[i], gamma, lam)
            adv.append(a)
            ret.append(r)
        flat_adv = np.concatenate(adv)
        part = self.whiten_partials(flat_adv)
        wflat = self.whiten_apply(flat_adv, part)
        offs = np.cumsum([0] + [len(a) for a in adv])
        whitened = [wflat[offs[i]:offs[i + 1]] for i in range(B)]
        kl = np.concatenate([a - r for a, r in zip(actor, ref)])
        return dict(tokens=toks, gen_logprobs=gen_lps, actor_logprobs=actor, ref_logprobs=ref, values=values,
                    rewards=rewards, advantages=adv, returns=ret, whitened=whitened, whiten_partials=part,
                    kl_mean=float(kl.mean()), reward_mean=float(rewards.mean()))


class RefLib:
    """The reference itself (compiled in place).  Present only where
    /root/reference was available at build time or the .so travelled."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        self.lib = C.CDLL(REF_SO)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_param_count.restype = I64
        L.ref_param_count.argtypes = [C.POINTER(I64), I32]
        L.ref_init_params.argtypes = [C.POINTER(I64), I32, C.c_uint64, C.POINTER(D)]
        L.ref_mix_seed.restype = C.c_uint64
        L.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_uniforms.argtypes = [C.c_uint64, I64, C.POINTER(D)]
        L.ref_generate_batch.argtypes = [C.POINTER(I64), C.POINTER(D), C.POINTER(I32), C.POINTER(I64), I64, I64,
                                         I32, D, C.POINTER(C.c_uint64), I64, C.POINTER(I32), C.POINTER(D),
                                         C.POINTER(I64), C.POINTER(D)]
        L.ref_sequence_logprobs.argtypes = [C.POINTER(I64), C.POINTER(D), C.POINTER(I32), I64, C.POINTER(D)]
        L.ref_forward_hidden.argtypes = [C.POINTER(I64), I32, C.POINTER(D), C.POINTER(I32), I64, C.POINTER(D)]
        L.ref_value_estimates.argtypes = [C.POINTER(I64), C.POINTER(D), C.POINTER(I32), I64, I64, C.POINTER(D)]
        L.ref_reward_head.argtypes = [C.POINTER(I64), C.POINTER(D), C.POINTER(I32), I64, C.POINTER(D)]
        L.ref_kl_penalized_rewards.argtypes = [D, C.POINTER(D), C.POINTER(D), I64, D, C.POINTER(D)]
        L.ref_gae.argtypes = [C.POINTER(D), C.POINTER(D), I64, D, D, C.POINTER(D), C.POINTER(D)]
        L.ref_ppo_actor_step.argtypes = [C.POINTER(I64), C.POINTER(D), I64, C.POINTER(I32), C.POINTER(I64),
                                         C.POINTER(I64), C.POINTER(D), C.POINTER(D), D, D, C.POINTER(D), I64,
                                         C.POINTER(D)]
        L.ref_critic_step.argtypes = [C.POINTER(I64), C.POINTER(D), I64, C.POINTER(I32), C.POINTER(I64),
                                      C.POINTER(I64), C.POINTER(D), C.POINTER(D), D, D, C.POINTER(D), I64,
                                      C.POINTER(D)]
        L.ref_dpo_step.argtypes = [C.POINTER(I64), C.POINTER(D), C.POINTER(D), I64, C.POINTER(I32), C.POINTER(I64),
                                   C.POINTER(I64), I32, D, D, D, C.POINTER(D), I64, C.POINTER(D)]
        L.ref_ppo_loop.argtypes = [C.POINTER(I64), C.POINTER(D), C.POINTER(D), C.POINTER(D), I32, C.POINTER(I32),
                                   C.POINTER(I64), I64, I64, C.c_uint64, D, D, D, D, D, D, C.POINTER(D), I64,
                                   C.POINTER(I32), C.POINTER(I64), C.POINTER(D), C.POINTER(D), C.POINTER(D),
                                   C.POINTER(D)]
        L.ref_experience.argtypes = [C.POINTER(I64), C.POINTER(D), C.POINTER(D), C.POINTER(D), C.POINTER(D), I32,
                                     C.POINTER(I32), C.POINTER(I64), I64, I64, I64, I32, D, C.c_uint64, I64, D, D,
                                     D, I64, C.POINTER(I32), C.POINTER(I64), C.POINTER(D), C.POINTER(D),
                                     C.POINTER(D), C.POINTER(D), C.POINTER(D), C.POINTER(D), C.POINTER(D)]

    def _chk(self, rc):
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def init_params(self, cfg: ModelCfg, seed, head=False):
        n = self.lib.ref_param_count(cfg.as6(), 1 if head else 0)
        w = np.empty(n, np.float64)
        self._chk(self.lib.ref_init_params(cfg.as6(), 1 if head else 0, seed, _p(w, D)))
        return w

    def mix_seed(self, a, b):
        return int(self.lib.ref_mix_seed(a, b))

    def uniforms(self, seed, n):
        out = np.empty(n, np.float64)
        self.lib.ref_uniforms(seed, n, _p(out, D))
        return out

    def generate_batch(self, cfg, w, prompts, max_new, greedy=True, temperature=1.0, seeds=None, n_workers=1):
        flat, offs = ragged(prompts)
        B = len(prompts)
        sd = np.asarray(seeds if seeds is not None else [0] * B, np.uint64)
        toks = np.zeros((B, max_new), np.int32)
        lps = np.zeros((B, max_new), np.float64)
        n = np.zeros(B, np.int64)
        secs = np.zeros(1, np.float64)
        self._chk(self.lib.ref_generate_batch(cfg.as6(), _p(w, D), _p(flat, I32), _p(offs, I64), B, max_new,
                                              1 if greedy else 0, temperature, _p(sd, C.c_uint64), n_workers,
                                              _p(toks, I32), _p(lps, D), _p(n, I64), _p(secs, D)))
        return [toks[b, :n[b]].copy() for b in range(B)], [lps[b, :n[b]].copy() for b in range(B)], float(secs[0])

    def sequence_logprobs(self, cfg, w, tokens):
        t = np.asarray(tokens, np.int32)
        out = np.zeros(len(t), np.float64)
        self._chk(self.lib.ref_sequence_logprobs(cfg.as6(), _p(w, D), _p(t, I32), len(t), _p(out, D)))
        return out

    def forward_hidden(self, cfg, w, tokens, head=False):
        t = np.asarray(tokens, np.int32)
        out = np.zeros((len(t), cfg.d), np.float64)
        self._chk(self.lib.ref_forward_hidden(cfg.as6(), 1 if head else 0, _p(w, D), _p(t, I32), len(t), _p(out, D)))
        return out

    def value_estimates(self, cfg, w, tokens, rs):
        t = np.asarray(tokens, np.int32)
        out = np.zeros(len(t) - rs, np.float64)
        self._chk(self.lib.ref_value_estimates(cfg.as6(), _p(w, D), _p(t, I32), len(t), rs, _p(out, D)))
        return out

    def reward_head(self, cfg, w, tokens):
        t = np.asarray(tokens, np.int32)
        out = np.zeros(1, np.float64)
        self._chk(self.lib.ref_reward_head(cfg.as6(), _p(w, D), _p(t, I32), len(t), _p(out, D)))
        return float(out[0])

    def kl_penalized_rewards(self, rm, a, r, coef):
        a = np.ascontiguousarray(a, np.float64)
        r = np.ascontiguousarray(r, np.float64)
        out = np.zeros(len(a), np.float64)
        self._chk(self.lib.ref_kl_penalized_rewards(rm, _p(a, D), _p(r, D), len(a), coef, _p(out, D)))
        return out

    def gae(self, rw, v, gamma, lam):
        rw = np.ascontiguousarray(rw, np.float64)
        v = np.ascontiguousarray(v, np.float64)
        adv = np.zeros(len(rw), np.float64)
        ret = np.zeros(len(rw), np.float64)
        self._chk(self.lib.ref_gae(_p(rw, D), _p(v, D), len(rw), gamma, lam, _p(adv, D), _p(ret, D)))
        return adv, ret

    # ---- train-side steps on the reference's tape + AdamW (checkers for the GPU trainer)
    def ppo_actor_step(self, cfg, w, seqs, rs, old_lp, adv, clip_eps, lr, adam=(0.9, 0.999, 1e-8, 0.0), n_steps=1):
        flat, offs = ragged(seqs)
        w = np.array(w, np.float64)
        rs = np.asarray(rs, np.int64)
        old_lp, adv = np.ascontiguousarray(old_lp, np.float64), np.ascontiguousarray(adv, np.float64)
        a4 = np.asarray(adam, np.float64)
        losses = np.zeros(n_steps, np.float64)
        self._chk(self.lib.ref_ppo_actor_step(cfg.as6(), _p(w, D), len(seqs), _p(flat, I32), _p(offs, I64), _p(rs, I64),
                                              _p(old_lp, D), _p(adv, D), clip_eps, lr, _p(a4, D), n_steps,
                                              _p(losses, D)))
        return w, losses

    def critic_step(self, cfg, w, seqs, rs, old_values, returns, value_clip, lr, adam=(0.9, 0.999, 1e-8, 0.0),
                    n_steps=1):
        flat, offs = ragged(seqs)
        w = np.array(w, np.float64)
        rs = np.asarray(rs, np.int64)
        ov, rt = np.ascontiguousarray(old_values, np.float64), np.ascontiguousarray(returns, np.float64)
        a4 = np.asarray(adam, np.float64)
        losses = np.zeros(n_steps, np.float64)
        self._chk(self.lib.ref_critic_step(cfg.as6(), _p(w, D), len(seqs), _p(flat, I32), _p(offs, I64), _p(rs, I64),
                                           _p(ov, D), _p(rt, D), value_clip, lr, _p(a4, D), n_steps, _p(losses, D)))
        return w, losses

    def dpo_step(self, cfg, w_policy, w_ref, pairs, variant, beta, cdpo_eps, lr, adam=(0.9, 0.999, 1e-8, 0.0),
                 n_steps=1):
        """pairs: list of (chosen_full, rejected_full, response_start_chosen, response_start_rejected)."""
        seqs, rs = [], []
        for c, r, rc, rr in pairs:
            seqs += [c, r]
            rs += [rc, rr]
        flat, offs = ragged(seqs)
        w = np.array(w_policy, np.float64)
        wr = np.ascontiguousarray(w_ref, np.float64)
        rs = np.asarray(rs, np.int64)
        a4 = np.asarray(adam, np.float64)
        losses = np.zeros(n_steps, np.float64)
        self._chk(self.lib.ref_dpo_step(cfg.as6(), _p(w, D), _p(wr, D), len(pairs), _p(flat, I32), _p(offs, I64),
                                        _p(rs, I64), variant, beta, cdpo_eps, lr, _p(a4, D), n_steps, _p(losses, D)))
        return w, losses

    def ppo_loop(self, cfg, w_policy, w_ref, w_critic, prompts, *, max_new, n_iters, kl_coef, lr, clip_eps=0.2,
                 value_clip=0.2, gamma=1.0, lam=0.95, scripted_target=122, adam=(0.9, 0.999, 1e-8, 0.0)):
        """n_iters greedy PPO iterations on the reference (experience, actor and
        critic updates with persistent AdamW, engine refit)."""
        flat, offs = ragged(prompts)
        B = len(prompts)
        wp, wc = np.array(w_policy, np.float64), np.array(w_critic, np.float64)
        wr = np.ascontiguousarray(w_ref, np.float64)
        shp = (n_iters, B, max_new)
        toks = np.zeros(shp, np.int32)
        n = np.zeros((n_iters, B), np.int64)
        a, v, adv = (np.zeros(shp, np.float64) for _ in range(3))
        losses = np.zeros((n_iters, 2), np.float64)
        a4 = np.asarray(adam, np.float64)
        self._chk(self.lib.ref_ppo_loop(cfg.as6(), _p(wp, D), _p(wr, D), _p(wc, D), scripted_target, _p(flat, I32),
                                        _p(offs, I64), B, max_new, 0, kl_coef, gamma, lam, clip_eps, value_clip, lr,
                                        _p(a4, D), n_iters, _p(toks, I32), _p(n, I64), _p(a, D), _p(v, D), _p(adv, D),
                                        _p(losses, D)))
        cut = lambda m, it: [m[it, b, :n[it, b]].copy() for b in range(B)]
        iters = [dict(tokens=cut(toks, it), actor_logprobs=cut(a, it), values=cut(v, it), advantages=cut(adv, it),
                      actor_loss=losses[it, 0], critic_loss=losses[it, 1]) for it in range(n_iters)]
        return iters, wp, wc

    def experience(self, cfg, w_policy, w_ref, w_critic, prompts, *, max_new, greedy, temperature=1.0, seed=0,
                   step_index=0, gidx0=0, kl_coef=0.003, gamma=1.0, lam=0.95, scripted_target=122, w_rm=None,
                   n_workers=1):
        flat, offs = ragged(prompts)
        B = len(prompts)
        shp = (B, max_new)
        toks = np.zeros(shp, np.int32)
        n = np.zeros(B, np.int64)
        a, r, v, adv, ret = (np.zeros(shp, np.float64) for _ in range(5))
        rw = np.zeros(B, np.float64)
        ph = np.zeros(3, np.float64)
        w_rm_p = _p(w_rm, D) if w_rm is not None else None
        self._chk(self.lib.ref_experience(cfg.as6(), _p(w_policy, D), _p(w_ref, D), _p(w_critic, D), w_rm_p,
                                          0 if w_rm is not None else scripted_target, _p(flat, I32), _p(offs, I64),
                                          B, gidx0, max_new, 1 if greedy else 0, temperature, seed, step_index,
                                          kl_coef, gamma, lam, n_workers, _p(toks, I32), _p(n, I64), _p(a, D),
                                          _p(r, D), _p(v, D), _p(rw, D), _p(adv, D), _p(ret, D), _p(ph, D)))
        cut = lambda m: [m[b, :n[b]].copy() for b in range(B)]
        return dict(tokens=cut(toks), actor_logprobs=cut(a), ref_logprobs=cut(r), values=cut(v), rewards=rw,
                    advantages=cut(adv), returns=cut(ret), phase_seconds=ph)


def synthetic_prompts(seed, B, P, ragged_lengths=False, gidx0=0):
    """Prompt i: ids Rng(mix_seed(seed, i)).uniform_int(256);
    ragged_lengths varies P_i in [max(1, P//2), P]."""
    o = Oracle.__dict__.get("_shared")
    if o is None:
        o = Oracle(threads=1)
        Oracle._shared = o
    out = []
    lib = o.lib
    lib.orc_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
    lib.orc_rng_uniform_int.restype = C.c_uint64
    lib.orc_rng_uniform_int.argtypes = [C.c_void_p, C.c_uint64]
    state = C.create_string_buffer(8 * 313)
    for i in range(gidx0, gidx0 + B):
        lib.orc_rng_seed(state, o.mix_seed(seed, i))
        n = P
        if ragged_lengths:
            lo = max(1, P // 2)
            n = lo + int(lib.orc_rng_uniform_int(state, P - lo + 1))
        out.append(np.array([lib.orc_rng_uniform_int(state, 256) for _ in range(n)], np.int32))
    return out
