"""Focused workload for ncu: C2-shaped engine, one warm generate, then one
profiled generate (64 prompts x 64 prompt tokens x `--new` tokens)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2405_01481_b200 import ppoexp as px  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--new", type=int, default=24)
ap.add_argument("--graphs", type=int, default=1)
ap.add_argument("--score", type=int, default=0)
ap.add_argument("--dtype", default="mixed", choices=["mixed", "bf16"])
a = ap.parse_args()
V, d, L, H, f, S, B, P, N, samp, _ = bench.CONFIGS[a.config]
cfg = px.ModelConfig(V, d, L, H, f, S)
ctx = px.Context(0)
dev = torch.device("cuda", 0)
m = px.DeviceModel(ctx, cfg, bench.init_weights(cfg, 1, dev), px.MIXED if a.dtype == "mixed" else px.BF16)
eng = px.Engine(m, px.EngineOptions(max_batch=B, use_graphs=bool(a.graphs)))
prompts = bench.prompts_for(0, B, P, V, 1)
tasks = [px.GenTask(p, a.new, px.SamplingSpec.temperature_spec(1.0, i, 0, 0.9)) for i, p in enumerate(prompts)]
eng.generate_batch(tasks)
torch.cuda.synchronize()
res = eng.generate_batch(tasks)
print("gen ms", eng.last_ms, "tokens", sum(len(r.tokens) for r in res))
if a.score:
    full = [np.concatenate([p, r.tokens]) for p, r in zip(prompts, res)]
    px.sequence_logprobs(m, full)
    px.sequence_logprobs(m, full)
