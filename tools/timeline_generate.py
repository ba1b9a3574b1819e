"""Where the generation phase's time goes outside steady-state decode steps:
prefill, per-call setup, and idle gaps on the GPU between kernels (e.g.
between CUDA-graph replays while the host polls).  CUPTI via torch.profiler.

    python tools/timeline_generate.py [--new 256]
"""
import argparse
import collections
import os
import re
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2405_01481_b200 import ppoexp as px  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--new", type=int, default=256)
a = ap.parse_args()
V, d, L, H, f, S, B, P, N, samp, _ = bench.CONFIGS["c2"]
cfg = px.ModelConfig(V, d, L, H, f, S)
ctx = px.Context(0)
dev = torch.device("cuda", 0)
m = px.DeviceModel(ctx, cfg, bench.init_weights(cfg, 1, dev), px.BF16)
eng = px.Engine(m, px.EngineOptions(max_batch=B, page_size=64, max_total_tokens=B * (-(-(P + a.new) // 64)) * 64))
prompts = bench.prompts_for(0, B, P, V, 1)
tasks = [px.GenTask(p, a.new, px.SamplingSpec.temperature_spec(1.0, i, 0, 0.9)) for i, p in enumerate(prompts)]
eng.generate_batch(tasks)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eng.generate_batch(tasks)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)


def short(n):
    n = n.replace("(anonymous namespace)::", "").replace("ppx::", "").replace("void ", "")
    return re.sub(r"\(.*", "", n)[:50]


t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
first_s = min(i for i, e in enumerate(ev) if "sampler_kernel" in e.name)
print(f"generate: {(t1 - t0) / 1e3:.2f} ms device span, {len(ev)} kernels/copies, device-reported {eng.last_ms:.2f} ms")
pre = ev[:first_s + 1]
agg = collections.defaultdict(lambda: [0, 0.0])
for e in pre:
    x = agg[short(e.name)]
    x[0] += 1
    x[1] += e.time_range.end - e.time_range.start
print(f"up to the first sampler (prefill + first token): {(pre[-1].time_range.end - t0) / 1e3:.2f} ms")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:10]:
    print(f"  {k:52s} {n:4d} x {t / n:8.1f} us")
# idle gaps: intervals where no kernel is resident
gaps, end = [], ev[0].time_range.end
for e in ev[1:]:
    if e.time_range.start > end:
        gaps.append((e.time_range.start - end, short(e.name)))
    end = max(end, e.time_range.end)
gaps.sort(reverse=True)
tot = sum(g for g, _ in gaps)
print(f"idle gaps: {len(gaps)} totalling {tot / 1e3:.2f} ms; largest:")
for g, n in gaps[:8]:
    print(f"  {g:8.1f} us before {n}")
big = [g for g, _ in gaps if g > 5]
print(f"gaps > 5 us: {len(big)} totalling {sum(big) / 1e3:.2f} ms")
