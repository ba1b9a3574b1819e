"""bf16 perf-mode error budget against the oracle (teacher-forced), reported as
max |err| / (1e-3 + 1e-3*|ref|) per quantity (north_star tolerance; <= 1 passes).

    python tools/parity_probe.py [--layers 2,12] [--prompts 4] [--new 24]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import ModelCfg, Oracle, synthetic_prompts  # noqa: E402
from tests.golden_util import bf16_round  # noqa: E402


def ratio(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float((np.abs(a - b) / (1e-3 + 1e-3 * np.abs(b))).max()), float(np.abs(a - b).max())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfgs", default="c1,c2w2,c2")
    ap.add_argument("--prompts", type=int, default=4)
    ap.add_argument("--new", type=int, default=24)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "mixed"])
    args = ap.parse_args()
    from paper_2405_01481_b200 import ppoexp as px
    DT = px.BF16 if args.dtype == "bf16" else px.MIXED
    o = Oracle()
    ctx = px.Context(0)
    shapes = {"c1": ModelCfg(1024, 128, 2, 4, 512, 128), "c2w2": ModelCfg(50257, 768, 2, 12, 3072, 512),
              "c2": ModelCfg(50257, 768, 12, 12, 3072, 512), "c3w2": ModelCfg(32000, 2048, 2, 16, 8192, 1024),
              "c4w2": ModelCfg(128256, 4096, 2, 32, 14336, 2048), "c4w1": ModelCfg(128256, 4096, 1, 32, 14336, 2048),
              "c3w1": ModelCfg(32000, 2048, 1, 16, 8192, 1024)}
    for name in args.cfgs.split(","):
        cfg = shapes[name]
        t0 = time.time()
        wp = bf16_round(o.init_params(cfg, 1))
        wr = bf16_round(o.init_params(cfg, 2))
        wc = bf16_round(o.init_params(cfg, 3, head=True, head_seed=4))
        prompts = synthetic_prompts(5, args.prompts, 16, ragged_lengths=True)
        pc = px.ModelConfig(cfg.V, cfg.d, cfg.L, cfg.H, cfg.f, cfg.S)
        eng = px.Engine(px.DeviceModel(ctx, pc, wp, DT))
        ref = px.DeviceModel(ctx, pc, wr, DT)
        crit = px.DeviceModel(ctx, pc.with_head(), wc, DT)
        xm = px.ExperienceMaker(eng, ref, crit, scripted_target=ord("e"))
        # greedy experience: tokens comparable with the oracle's own greedy rollout
        batch, st = xm.run(prompts, max_new=args.new, sampling=px.SamplingSpec.greedy_spec(), seed=3)
        full = [np.concatenate([s.prompt, s.response]) for s in batch]
        rs = [len(s.prompt) for s in batch]
        a = o.sequence_logprobs(cfg, wp, full)
        r = o.sequence_logprobs(cfg, wr, full)
        v = o.value_estimates(cfg, wc, full, rs)
        t_o, l_o = o.generate(cfg, wp, prompts, args.new)
        res = {"actor_lp": [], "ref_lp": [], "values": [], "adv": [], "gen_lp": []}
        tok_same = 0
        for s, ai, ri, vi, p, to in zip(batch, a, r, v, rs, t_o):
            res["actor_lp"].append(ratio(s.actor_logprobs, ai[p:]))
            res["ref_lp"].append(ratio(s.ref_logprobs, ri[p:]))
            res["values"].append(ratio(s.values, vi))
            shaped = o.kl_penalized_rewards(s.reward, ai[p:], ri[p:], 0.003)
            adv, _ = o.gae(shaped, vi, 1.0, 0.95)
            res["adv"].append(ratio(s.advantages, adv))
            tok_same += int(np.array_equal(s.response, to))
        gen = eng.generate_batch([px.GenTask(p, args.new) for p in prompts])
        for g, p, ai in zip(gen, prompts, o.sequence_logprobs(cfg, wp, [np.concatenate([p, g.tokens]) for p, g in
                                                                         zip(prompts, gen)])):
            res["gen_lp"].append(ratio(g.logprobs, ai[len(p):]))
        summ = {k: (max(x[0] for x in v_), max(x[1] for x in v_)) for k, v_ in res.items()}
        print(f"{name} L={cfg.L} d={cfg.d} V={cfg.V}: greedy rollouts identical {tok_same}/{len(prompts)}; "
              + "; ".join(f"{k} ratio {r_:.3f} (abs {e:.2e})" for k, (r_, e) in summ.items())
              + f"  [{time.time() - t0:.0f} s]", flush=True)
        eng.close()
        eng.model.close()
        ref.close()
        crit.close()
    ctx.close()


if __name__ == "__main__":
    main()
