"""CUPTI (torch.profiler) breakdown of one whole C2 experience step
(ExperienceMaker.run_device: generate + policy/reference scoring + critic +
shaping + whitening), aggregated per kernel, decode and scoring separated by
the last sampler launch.

    python tools/timeline_experience.py
"""
import collections
import os
import re
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2405_01481_b200 import ppoexp as px  # noqa: E402

V, d, L, H, f, S, B, P, N, samp, _ = bench.CONFIGS["c2"]
cfg = px.ModelConfig(V, d, L, H, f, S)
ctx = px.Context(0)
dev = torch.device("cuda", 0)
pol = px.DeviceModel(ctx, cfg, bench.init_weights(cfg, bench.SEED, dev), px.BF16)
ref = px.DeviceModel(ctx, cfg, bench.init_weights(cfg, bench.SEED + 1, dev), px.BF16)
crit = px.DeviceModel(ctx, cfg.with_head(), bench.init_weights(cfg, bench.SEED + 101, dev, head=True), px.BF16)
eng = px.Engine(pol, px.EngineOptions(max_batch=B, page_size=64, max_total_tokens=B * (-(-(P + N) // 64)) * 64))
xm = px.ExperienceMaker(eng, ref, crit, scripted_target=ord("e"), hyper=px.PpoHyper(0.003, 1.0, 0.95))
sampling = px.SamplingSpec.temperature_spec(1.0, 0, 0, bench.TOP_P)
prompts = bench.prompts_for(0, B, P, V, bench.SEED)
import numpy as np  # noqa: E402

flat = torch.from_numpy(np.concatenate(prompts).astype(np.int32)).to(dev)
offs = torch.from_numpy(np.concatenate([[0], np.cumsum([len(p) for p in prompts])]).astype(np.int64)).to(dev)
out = px.ExperienceMaker.alloc_device_outputs(B, N, dev)
for i in range(2):
    xm.run_device(flat, offs, out, max_new=N, sampling=sampling, seed=bench.SEED, step_index=i, gidx0=0)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    xm.run_device(flat, offs, out, max_new=N, sampling=sampling, seed=bench.SEED, step_index=2, gidx0=0)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)


def short(n):
    n = n.replace("(anonymous namespace)::", "").replace("ppx::", "").replace("void ", "")
    return re.sub(r"\(.*", "", n)[:60]


last_s = max(i for i, e in enumerate(ev) if "sampler_kernel" in e.name)
first = ev[0].time_range.start
print(f"step span {(ev[-1].time_range.end - first) / 1e3:.2f} ms; decode ends at "
      f"{(ev[last_s].time_range.end - first) / 1e3:.2f} ms")
for name, part in (("after the last decode step (scoring, shaping, whitening)", ev[last_s + 1:]),):
    span = (part[-1].time_range.end - part[0].time_range.start) / 1e3
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in part:
        a = agg[short(e.name)]
        a[0] += 1
        a[1] += e.time_range.end - e.time_range.start
    print(f"\n{name}: {span:.2f} ms wall, {len(part)} kernels")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
        print(f"  {k:62s} {n:5d} x {t / n:8.1f} us = {t / 1e3:7.2f} ms")
