"""Focused workload for ncu: one causal prefill attention launch (C5 shape:
4096 tokens, 32 heads, head_dim 128) through the testing entry point."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_01481_b200 import ppoexp as px  # noqa: E402

path = int(sys.argv[1]) if len(sys.argv) > 1 else 0
T, H, DH, B = 4096, 32, 128, 2
ctx = px.Context(0)
f = px.lib().ppoexp_testing_attention_prefill
f.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
              C.c_int32]
d = H * DH
qkv = torch.randn(B * T, 3 * d, device="cuda").to(torch.bfloat16)
offs = torch.tensor([0, T, 2 * T], dtype=torch.int64, device="cuda")
out = torch.zeros(B * T, d, dtype=torch.bfloat16, device="cuda")
torch.cuda.synchronize()
for _ in range(3):
    px._check(f(ctx.h, qkv.data_ptr(), offs.data_ptr(), B, T, H, DH, B * T, out.data_ptr(), path))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    px._check(f(ctx.h, qkv.data_ptr(), offs.data_ptr(), B, T, H, DH, B * T, out.data_ptr(), path))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
flops = 2 * 2 * B * H * T * T / 2 * DH
print(f"path {path}: {ms:.3f} ms per launch, {flops / ms / 1e9:.0f} TFLOP/s")
