import sys, os
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import bench
from paper_2405_01481_b200 import ppoexp as px
V, d, L, H, f, S, B, P, N, samp, _ = bench.CONFIGS['c2']
cfg = px.ModelConfig(V, d, L, H, f, S)
ctx = px.Context(0)
m = px.DeviceModel(ctx, cfg, bench.init_weights(cfg, 1, torch.device('cuda', 0)), px.MIXED)
eng = px.Engine(m, px.EngineOptions(max_batch=64))
prompts = bench.prompts_for(0, 64, 64, V, 1)
tasks = [px.GenTask(p, 256, px.SamplingSpec.temperature_spec(1.0, i, 0, 0.9)) for i, p in enumerate(prompts)]
eng.generate_batch(tasks)
n0 = ctx.launch_count
res = eng.generate_batch(tasks)
print("launches per generate", ctx.launch_count - n0, "tokens", sum(len(r.tokens) for r in res))
