"""Loads a golden fixture and rebuilds its weights with the oracle restatement
(after proving the restated init equals the reference's by sha256)."""
import hashlib
import os

import numpy as np

from oracle.oracle import ModelCfg, Oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(w):
    return hashlib.sha256(np.ascontiguousarray(w, np.float64).tobytes()).hexdigest()


def load(name, oracle: Oracle):
    z = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    cfg = ModelCfg(*[int(x) for x in z["cfg"]])
    seed = int(z["seed"])
    raw = dict(pol=oracle.init_params(cfg, seed), ref=oracle.init_params(cfg, seed + 1),
               crit=oracle.init_params(cfg, seed + 101, head=True), rm=oracle.init_params(cfg, seed + 303, head=True))
    for k, w in raw.items():
        assert sha(w) == str(z[f"sha_{k}"]), f"oracle init_params({k}) differs from the reference's"
    raw["crit"] = oracle.init_params(cfg, seed + 101, head=True, head_seed=seed + 202)
    raw["rm"] = oracle.init_params(cfg, seed + 303, head=True, head_seed=seed + 404)
    W = {k: w.astype(np.float32).astype(np.float64) for k, w in raw.items()}
    plens = z["plens"]
    offs = np.concatenate([[0], np.cumsum(plens)])
    prompts = [z["prompts"][offs[i]:offs[i + 1]] for i in range(len(plens))]
    return z, cfg, W, prompts


def rows(mat, lens):
    return [mat[i, :lens[i]] for i in range(len(lens))]


def bf16_round(w):
    """fp64 -> nearest-even bf16 (via fp32), returned as fp64 (exactly representable)."""
    x = np.ascontiguousarray(w, np.float32).view(np.uint32).astype(np.uint64)
    x = (x + 0x7FFF + ((x >> 16) & 1)) & 0xFFFF0000
    return x.astype(np.uint32).view(np.float32).astype(np.float64)


def to_px_cfg(cfg: ModelCfg, head=False):
    from paper_2405_01481_b200 import ppoexp as px
    return px.ModelConfig(cfg.V, cfg.d, cfg.L, cfg.H, cfg.f, cfg.S, head)
