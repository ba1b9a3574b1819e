"""Which MN-major smem-descriptor assignment is right (tcgen05 P.V operand)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_01481_b200 import ppoexp as px  # noqa: E402

ctx = px.Context(0)
f = px.lib().ppoexp_testing_umma_probe
f.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32]
f.restype = C.c_int32
for N in (64, 128):
    A = torch.randn(128, 64, device="cuda").to(torch.bfloat16)
    B = torch.randn(64, N, device="cuda").to(torch.bfloat16)
    ref = A.float() @ B.float()
    for v in (0,):
        out = torch.zeros(128, N, device="cuda")
        torch.cuda.synchronize()
        rc = f(ctx.h, A.data_ptr(), B.data_ptr(), N, out.data_ptr(), v)
        err = (out - ref).abs().max().item() if rc == 0 else None
        print(f"N={N} variant={v} rc={rc} max err={err}")
