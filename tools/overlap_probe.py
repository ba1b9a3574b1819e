"""Probe: do two independent decode chains (two contexts / streams, half the
batch each) overlap on one B200?  C2 policy, 64 prompts x 256 sampled tokens."""
import sys, os, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2405_01481_b200 import ppoexp as px

dt = {"mixed": px.MIXED, "bf16": px.BF16}[sys.argv[1] if len(sys.argv) > 1 else "mixed"]
V, d, L, H, f, S, Bc, P, N, samp, desc = bench.CONFIGS["c2"]
cfg = px.ModelConfig(V, d, L, H, f, S)
dev = torch.device("cuda", 0)
w = bench.init_weights(cfg, bench.SEED, dev)
prompts = bench.prompts_for(0, 64, P, V, bench.SEED)
sp = px.SamplingSpec.temperature_spec(1.0, 0, 0, 0.9)


def mk(B):
    ctx = px.Context(0)
    m = px.DeviceModel(ctx, cfg, w, dt)
    e = px.Engine(m, px.EngineOptions(max_batch=B, page_size=64, max_total_tokens=B * 320))
    return ctx, m, e


def tasks(lo, hi):
    return [px.GenTask(prompts[i], N, px.SamplingSpec(False, 1.0, 1000 + i, 0, 0.9)) for i in range(lo, hi)]


one = mk(64)
a, b = mk(32), mk(32)
for _ in range(2):
    one[2].generate_batch(tasks(0, 64))
    a[2].generate_batch(tasks(0, 32)); b[2].generate_batch(tasks(32, 64))
torch.cuda.synchronize()
for rep in range(3):
    t = time.perf_counter(); r1 = one[2].generate_batch(tasks(0, 64)); t1 = time.perf_counter() - t
    t = time.perf_counter(); a[2].generate_batch(tasks(0, 32)); b[2].generate_batch(tasks(32, 64)); t2 = time.perf_counter() - t
    res = {}
    def run(k, e, lo, hi):
        res[k] = e.generate_batch(tasks(lo, hi))
    th = [threading.Thread(target=run, args=(0, a[2], 0, 32)), threading.Thread(target=run, args=(1, b[2], 32, 64))]
    t = time.perf_counter()
    for x in th: x.start()
    for x in th: x.join()
    t3 = time.perf_counter() - t
    same = all(np.array_equal(r1[i].tokens, (res[0] + res[1])[i].tokens) for i in range(64))
    print(f"one 64: {t1*1e3:.1f} ms  ({64*N/t1:.0f} tok/s) | 2x32 serial {t2*1e3:.1f} | 2x32 concurrent {t3*1e3:.1f} ms "
          f"({64*N/t3:.0f} tok/s)  tokens equal: {same}", flush=True)
