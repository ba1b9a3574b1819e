"""Time the mixed-mode scoring GEMM variants at the C2 scoring shapes
(M = 64 x 320 rows): in-kernel split (gemm_mixed), activation planes
(gemm_planes), and the plain bf16 GEMM for reference."""
import ctypes as C
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_01481_b200 import ppoexp as px

ctx = px.Context(0)
L = px.lib()
fm = L.ppoexp_testing_gemm_mixed
fm.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_void_p, C.c_int64]
fp = L.ppoexp_testing_gemm_planes
fp.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_void_p, C.c_int64]
fb = L.ppoexp_testing_gemm_bf16
fb.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_void_p, C.c_int64, C.c_int32]
st = torch.cuda.ExternalStream(ctx.stream)
M = int(sys.argv[1]) if len(sys.argv) > 1 else 20480
for (N, K, epi) in [(2304, 768, 3), (768, 768, 2), (3072, 768, 5), (768, 3072, 2)]:
    A = torch.randn(M, K, device="cuda")
    P = torch.cat([A.to(torch.bfloat16), (A - A.to(torch.bfloat16).float()).to(torch.bfloat16)], 1).contiguous()
    W = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
    Cf = torch.zeros(M, N, device="cuda")
    Cp = torch.zeros(M, 2 * N, dtype=torch.bfloat16, device="cuda")
    Ab = A.to(torch.bfloat16)
    torch.cuda.synchronize()
    def run(kind):
        if kind == "mixed":
            px._check(fm(ctx.h, A.data_ptr(), K, W.data_ptr(), K, M, N, K, epi, Cf.data_ptr(), N))
        elif kind == "planes":
            e = 6 if epi == 5 else epi
            px._check(fp(ctx.h, P.data_ptr(), W.data_ptr(), M, N, K, e, (Cp if e == 6 else Cf).data_ptr(), 2 * N if e == 6 else N))
        else:
            px._check(fb(ctx.h, Ab.data_ptr(), K, W.data_ptr(), K, M, N, K, 3, Cf.data_ptr(), N, 0))
    res = {}
    for kind in ("mixed", "planes", "bf16"):
        for _ in range(3):
            run(kind)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(20):
            run(kind)
        e1.record(st)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        res[kind] = ms
    fl = 2.0 * M * N * K
    print(f"M={M} N={N} K={K} epi={epi}: " + "  ".join(f"{k} {v*1e3:.1f} us ({fl/v/1e9:.0f} TF/s alg)" for k, v in res.items()), flush=True)
