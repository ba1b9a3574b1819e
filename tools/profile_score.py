"""Scoring-only workload at the C2 experience shape (64 sequences x 320
tokens through one 125M model): times sequence_logprobs with CUDA events, and
gives ncu a short, clean launch list (the second call)."""
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
ap.add_argument("--dtype", default="mixed", choices=["mixed", "bf16"])
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
V, d, L, H, f, S, B, P, N, samp, _ = bench.CONFIGS[a.config]
cfg = px.ModelConfig(V, d, L, H, f, S)
ctx = px.Context(0)
dev = torch.device("cuda", 0)
m = px.DeviceModel(ctx, cfg, bench.init_weights(cfg, 1, dev), px.MIXED if a.dtype == "mixed" else px.BF16)
rng = np.random.default_rng(0)
seqs = [rng.integers(0, V, size=P + N).astype(np.int32) for _ in range(B)]
st = torch.cuda.ExternalStream(ctx.stream)
for i in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    px.sequence_logprobs(m, seqs)
    e1.record(st)
    e1.synchronize()
    print(f"sequence_logprobs {B} x {P + N}: {e0.elapsed_time(e1):.2f} ms (incl. host staging)", flush=True)
