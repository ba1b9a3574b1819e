"""Probe: do two independent half-batch decode chains on separate streams
overlap on the GPU?  Compares one engine generating 64 sequences with two
engines (separate contexts = separate streams) generating 32 each from two
host threads (ctypes releases the GIL during the library call).

    python tools/concurrency_probe.py [--new 88]
"""
import argparse
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2405_01481_b200 import ppoexp as px  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--new", type=int, default=88)
a = ap.parse_args()
V, d, L, H, f, S, B, P, N, samp, _ = bench.CONFIGS["c2"]
cfg = px.ModelConfig(V, d, L, H, f, S)
dev = torch.device("cuda", 0)
w = bench.init_weights(cfg, 1, dev)
prompts = bench.prompts_for(0, B, P, V, 1)
tasks = [px.GenTask(p, a.new, px.SamplingSpec.temperature_spec(1.0, i, 0, 0.9)) for i, p in enumerate(prompts)]


def make(nb):
    ctx = px.Context(0)
    m = px.DeviceModel(ctx, cfg, w, px.BF16)
    return ctx, m, px.Engine(m, px.EngineOptions(max_batch=nb))


one = make(B)
one[2].generate_batch(tasks)
torch.cuda.synchronize()
t = time.perf_counter()
one[2].generate_batch(tasks)
t1 = time.perf_counter() - t
print(f"one engine x {B}: {t1 * 1e3:.1f} ms wall, {one[2].last_ms:.1f} ms device")

halves = [make(B // 2), make(B // 2)]
parts = [tasks[: B // 2], tasks[B // 2:]]
for h, p in zip(halves, parts):
    h[2].generate_batch(p)
torch.cuda.synchronize()
res = [None, None]


def run(i):
    res[i] = halves[i][2].generate_batch(parts[i])


th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
t = time.perf_counter()
for x in th:
    x.start()
for x in th:
    x.join()
t2 = time.perf_counter() - t
print(f"two engines x {B // 2} (concurrent): {t2 * 1e3:.1f} ms wall "
      f"({halves[0][2].last_ms:.1f} / {halves[1][2].last_ms:.1f} ms device each)  speedup {t1 / t2:.2f}x")
