"""In-graph kernel timeline of the decode step (CUPTI via torch.profiler).

Runs the C2 engine (as tools/profile_decode.py), profiles one generate call
and prints, for a window of consecutive decode steps in steady state, each
kernel's duration and the gap since the previous kernel ended (negative =
overlap through programmatic dependent launch), aggregated per kernel class.

    python tools/timeline.py [--new 88]
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
ap.add_argument("--new", type=int, default=88)
ap.add_argument("--steps", type=int, default=8, help="decode steps to aggregate (from the middle)")
ap.add_argument("--config", default="c2")
ap.add_argument("--batch", type=int, default=0)
a = ap.parse_args()
V, d, L, H, f, S, B, P, N, samp, _ = bench.CONFIGS[a.config]
B = a.batch or B
cfg = px.ModelConfig(V, d, L, H, f, S)
ctx = px.Context(0)
dev = torch.device("cuda", 0)
m = px.DeviceModel(ctx, cfg, bench.init_weights(cfg, 1, dev), px.BF16)
eng = px.Engine(m, px.EngineOptions(max_batch=B))
prompts = bench.prompts_for(0, B, P, V, 1)
tasks = [px.GenTask(p, a.new, px.SamplingSpec.temperature_spec(1.0, i, 0, 0.9)) for i, p in enumerate(prompts)]
eng.generate_batch(tasks)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    eng.generate_batch(tasks)
    torch.cuda.synchronize()
print("gen ms", eng.last_ms)

ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "Memcpy" not in e.name
      and "Memset" not in e.name]
ev.sort(key=lambda e: e.time_range.start)


def short(n):
    n = n.replace("(anonymous namespace)::", "").replace("ppx::", "").replace("void ", "")
    return re.sub(r"\(.*", "", n)[:60]


# a decode step ends with the sampler kernel
ends = [i for i, e in enumerate(ev) if "sampler_kernel" in e.name]
print("sampler launches:", len(ends))
mid = len(ends) // 2
lo, hi = ends[max(0, mid - a.steps)], ends[mid]
win = ev[lo + 1:hi + 1]
span = (win[-1].time_range.end - win[0].time_range.start) / a.steps
agg = collections.OrderedDict()
prev_end = ev[lo].time_range.end
for e in win:
    k = short(e.name)
    dur = e.time_range.end - e.time_range.start
    contrib = max(0.0, e.time_range.end - prev_end)  # how much this kernel extends the step
    s_ = agg.setdefault(k, [0, 0.0, 0.0])
    s_[0] += 1
    s_[1] += dur
    s_[2] += contrib
    prev_end = max(prev_end, e.time_range.end)
print(f"steady-state decode step: {span:.1f} us over {a.steps} steps ({len(win) / a.steps:.0f} kernels/step)")
print(f"{'kernel':62s} {'n/step':>6s} {'resident us':>11s} {'critical us':>11s} {'us/step':>8s}")
tot = 0.0
for k, (n, dsum, csum) in sorted(agg.items(), key=lambda x: -x[1][2]):
    print(f"{k:62s} {n / a.steps:6.1f} {dsum / n:11.2f} {csum / n:11.2f} {csum / a.steps:8.1f}")
    tot += csum
print(f"critical-path sum {tot / a.steps:.1f} us/step (resident = start..end incl. PDL early start; "
      f"critical = end minus the previous latest end)")
