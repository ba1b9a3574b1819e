"""Kernel-level numerics against a plain PyTorch fp32 reference of the same op
(GPU only): the tcgen05 GEMM (all epilogues, ragged M/N/K, decode-sized M)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def glib():
    from paper_2405_01481_b200 import ppoexp as px
    L = px.lib()
    f = L.ppoexp_testing_gemm_bf16
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                  C.c_int32, C.c_void_p, C.c_int64, C.c_int32]
    f.restype = C.c_int32
    return px, f


SHAPES = [(64, 2304, 768), (64, 768, 3072), (256, 2048, 8192), (256, 2048, 2048), (300, 1000, 768), (2048, 50257, 768), (4096, 3072, 768), (128, 256, 64),
          (17, 96, 16), (1024, 1024, 4096), (640, 768, 3072)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("epi", [0, 1, 2, 3])
@pytest.mark.parametrize("path", [0, 1])
def test_gemm_vs_torch(glib, ctx, M, N, K, epi, path):
    import torch
    px, f = glib
    if path == 1 and M * N * K > 2e10:
        pytest.skip("SIMT path too slow for this size")
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    ref = A.float() @ B.float().T
    ldc = (N + 63) // 64 * 64
    if epi in (0, 1):
        Cm = torch.zeros(M, ldc, dtype=torch.bfloat16, device="cuda")
    else:
        Cm = torch.randn(M, ldc, generator=g, device="cuda") if epi == 2 else torch.zeros(M, ldc, device="cuda")
    base = Cm.clone()
    torch.cuda.synchronize()
    px._check(f(ctx.h, A.data_ptr(), K, B.data_ptr(), K, M, N, K, epi, Cm.data_ptr(), ldc, path))
    out = Cm[:, :N].float()
    if epi == 1:
        ref = torch.nn.functional.gelu(ref, approximate="tanh")
    if epi == 2:
        ref = ref + base[:, :N]
    tol = 2e-2 if epi in (0, 1) else 2e-3
    err = (out - ref).abs() - tol * (1 + ref.abs())
    assert err.max().item() <= 0, f"max abs err {(out - ref).abs().max().item():.3e}"
    if epi in (0, 1):  # untouched padding
        assert torch.all(Cm[:, N:] == 0)


@pytest.fixture(scope="module")
def lmlib():
    from paper_2405_01481_b200 import ppoexp as px
    f = px.lib().ppoexp_testing_lm_head_logprobs
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                  C.c_void_p, C.c_int32]
    f.restype = C.c_int32
    return px, f


@pytest.mark.parametrize("R,V,K", [(300, 1000, 128), (1024, 50257, 768), (130, 128256, 256), (4096, 32000, 2048),
                                   (1, 258, 64)])
@pytest.mark.parametrize("path", [0, 1])
def test_lm_head_logprobs_vs_torch(lmlib, ctx, R, V, K, path):
    """Scoring log-probs (src/tensor.cpp:428-456 log_softmax + :491-519 gather)
    from bf16 hidden rows and the tied bf16 LM head: the fused tcgen05 LM head
    with the online-LSE epilogue (path 0) and fp32 logits + K9 (path 1)
    against torch on the same bf16 operands, fp32 products, fp64 softmax."""
    import torch
    px, f = lmlib
    g = torch.Generator(device="cuda").manual_seed(R + V + K)
    H = torch.randn(R, K, generator=g, device="cuda").to(torch.bfloat16)
    W = (torch.randn(V, K, generator=g, device="cuda") * (2.0 / K ** 0.5)).to(torch.bfloat16)
    tgt = torch.randint(0, V, (R,), generator=g, device="cuda", dtype=torch.int32)
    tgt[::7] = V - 1  # the ragged last column tile
    out = torch.zeros(R, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()  # the library runs on its own stream
    px._check(f(ctx.h, H.data_ptr(), W.data_ptr(), R, V, K, 0, tgt.data_ptr(), out.data_ptr(), path))
    logits = (H.double() @ W.double().T)
    ref = torch.log_softmax(logits, dim=-1).gather(1, tgt.long()[:, None])[:, 0]
    err = (out - ref).abs()
    assert (err <= 1e-4 * (1 + ref.abs())).all(), f"max abs err {err.max().item():.3e}"


def test_k9_on_fp32_logits_vs_torch(lmlib, ctx):
    import torch
    px, f = lmlib
    R, V, ld = 513, 50257, 50304
    g = torch.Generator(device="cuda").manual_seed(3)
    L = torch.randn(R, ld, generator=g, device="cuda") * 4
    tgt = torch.randint(0, V, (R,), generator=g, device="cuda", dtype=torch.int32)
    out = torch.zeros(R, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    px._check(f(ctx.h, L.data_ptr(), None, R, V, 0, ld, tgt.data_ptr(), out.data_ptr(), 2))
    ref = torch.log_softmax(L[:, :V].double(), dim=-1).gather(1, tgt.long()[:, None])[:, 0]
    assert (out - ref).abs().max().item() < 1e-4


MIXED_SHAPES = [(64, 2304, 768), (64, 768, 3072), (200, 50257, 768), (17, 96, 16), (300, 1000, 768),
                (2048, 3072, 768), (4096, 768, 3072), (1000, 4096, 4096)]


@pytest.mark.parametrize("M,N,K", MIXED_SHAPES)
@pytest.mark.parametrize("epi", [2, 3, 5])
def test_gemm_mixed_vs_torch(ctx, M, N, K, epi):
    """Mixed mode: fp32 activations x bf16 weights on the tensor cores with the
    two-term activation split must match fp64 products of the same operands to
    fp32-grade accuracy (bound below, ~1e-6 relative for these shapes)."""
    import torch
    from paper_2405_01481_b200 import ppoexp as px
    f = px.lib().ppoexp_testing_gemm_mixed
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                  C.c_int32, C.c_void_p, C.c_int64]
    f.restype = C.c_int32
    g = torch.Generator(device="cuda").manual_seed(M + 3 * N + 7 * K + epi)
    A = torch.randn(M, K, generator=g, device="cuda")
    W = (torch.randn(N, K, generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    ldc = (N + 63) // 64 * 64
    Cm = torch.randn(M, ldc, generator=g, device="cuda") if epi == 2 else torch.zeros(M, ldc, device="cuda")
    base = Cm.double().clone()
    torch.cuda.synchronize()
    px._check(f(ctx.h, A.data_ptr(), K, W.data_ptr(), K, M, N, K, epi, Cm.data_ptr(), ldc))
    ref = A.double() @ W.double().T
    if epi == 5:
        ref = torch.nn.functional.gelu(ref, approximate="tanh")
    if epi == 2:
        ref = ref + base[:, :N]
    # the split represents every activation to 2^-18 relative (|a - hi - lo|),
    # plus fp32 accumulation: bound the error by 2^-16 sum_k |a_k w_k| + fp32 ulps
    mag = A.double().abs() @ W.double().abs().T
    if epi == 5:
        mag = mag * 1.2  # |gelu'| <= 1.13
    err = (Cm[:, :N].double() - ref).abs()
    bound = 2.0 ** -16 * mag + 2e-7 * (1 + ref.abs())
    assert (err <= bound).all(), f"max abs err {err.max().item():.3e}, max err/bound {(err / bound).max().item():.3f}"


@pytest.mark.parametrize("DH,H,lens", [(64, 12, [320, 37, 1, 129, 64]), (128, 4, [4096]), (128, 8, [200, 513, 7]),
                                       (64, 2, [2048, 2048])])
@pytest.mark.parametrize("path", [0, 1])
def test_attention_prefill_vs_torch(ctx, DH, H, lens, path):
    """Causal prefill attention over packed ragged sequences (src/model.cpp:230-236):
    the tcgen05 flash attention (path 0: TMA K/V, S and O in TMEM, V as the
    MN-major operand) and the mma.sync kernel (path 1) against torch fp32."""
    import torch
    from paper_2405_01481_b200 import ppoexp as px
    f = px.lib().ppoexp_testing_attention_prefill
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                  C.c_void_p, C.c_int32]
    f.restype = C.c_int32
    d = H * DH
    M = sum(lens)
    g = torch.Generator(device="cuda").manual_seed(M + DH)
    qkv = (torch.randn(M, 3 * d, generator=g, device="cuda") * 1.5).to(torch.bfloat16)
    offs = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int64, device="cuda")
    out = torch.zeros(M, d, dtype=torch.bfloat16, device="cuda")
    torch.cuda.synchronize()
    px._check(f(ctx.h, qkv.data_ptr(), offs.data_ptr(), len(lens), max(lens), H, DH, M, out.data_ptr(), path))
    ref = torch.empty(M, d, device="cuda")
    q, k, v = qkv.float().split(d, dim=1)
    o = 0
    for T in lens:
        qs = q[o:o + T].view(T, H, DH).transpose(0, 1)
        ks = k[o:o + T].view(T, H, DH).transpose(0, 1)
        vs = v[o:o + T].view(T, H, DH).transpose(0, 1)
        s = qs @ ks.transpose(1, 2) / DH ** 0.5
        s = s.masked_fill(torch.triu(torch.ones(T, T, dtype=torch.bool, device="cuda"), 1), float("-inf"))
        ref[o:o + T] = (torch.softmax(s, -1) @ vs).transpose(0, 1).reshape(T, d)
        o += T
    err = (out.float() - ref).abs()
    assert err.max().item() < 2e-2, f"max abs err {err.max().item():.3e}"


@pytest.mark.parametrize("DH,H,lens", [(64, 12, [320, 37, 1, 129, 64]), (64, 4, [700]), (64, 2, [128, 128, 255]),
                                       (128, 4, [513, 7, 200]), (128, 2, [1024])])
def test_attention_prefill_split_tc_vs_fp64(ctx, DH, H, lens):
    """Mixed-mode scoring attention on tcgen05 (q / k / v as hi | lo planes, each
    product as three MMAs, P split the same way, output planes): fp32-grade
    against fp64 attention over the reconstructed (hi + lo) operands."""
    import torch
    from paper_2405_01481_b200 import ppoexp as px
    f = px.lib().ppoexp_testing_attention_prefill
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                  C.c_void_p, C.c_int32]
    f.restype = C.c_int32
    d = H * DH
    M = sum(lens)
    g = torch.Generator(device="cuda").manual_seed(M + H)
    qkv = torch.randn(M, 3 * d, generator=g, device="cuda") * 1.5
    hi = qkv.to(torch.bfloat16)
    lo = (qkv - hi.float()).to(torch.bfloat16)
    planes = torch.cat([hi, lo], dim=1).contiguous()
    offs = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int64, device="cuda")
    out = torch.zeros(M, 2 * d, dtype=torch.bfloat16, device="cuda")
    torch.cuda.synchronize()
    px._check(f(ctx.h, planes.data_ptr(), offs.data_ptr(), len(lens), max(lens), H, DH, M, out.data_ptr(), 2))
    got = out[:, :d].double() + out[:, d:].double()
    x = hi.double() + lo.double()
    q, k, v = x.split(d, dim=1)
    ref = torch.empty(M, d, dtype=torch.float64, device="cuda")
    o = 0
    for T in lens:
        qs = q[o:o + T].view(T, H, DH).transpose(0, 1)
        ks = k[o:o + T].view(T, H, DH).transpose(0, 1)
        vs = v[o:o + T].view(T, H, DH).transpose(0, 1)
        s = qs @ ks.transpose(1, 2) / DH ** 0.5
        s = s.masked_fill(torch.triu(torch.ones(T, T, dtype=torch.bool, device="cuda"), 1), float("-inf"))
        ref[o:o + T] = (torch.softmax(s, -1) @ vs).transpose(0, 1).reshape(T, d)
        o += T
    err = (got - ref).abs()
    # the omitted lo*lo terms leave ~2^-18 |q||k| per product in the scores
    # (~5e-5 at |x| ~ 1.5, dh 64; sqrt(2) more at dh 128), as in the mma.sync split kernel
    assert err.max().item() < 4e-4 and err.mean().item() < 2e-5, \
        f"max abs err {err.max().item():.3e}, mean {err.mean().item():.3e}"


@pytest.mark.parametrize("M,N,K", [(300, 2304, 768), (2048, 768, 3072), (129, 3072, 768), (64, 768, 768),
                                   (1000, 1000, 256),
                                   # wide decode-sized launches (config-4 shapes, the multi-wave LM head, ragged M / N)
                                   (64, 8192, 2048), (48, 6144, 4096), (7, 50257, 768), (64, 4096, 14336)])
@pytest.mark.parametrize("epi", [2, 3, 6])
def test_gemm_planes_vs_torch(ctx, M, N, K, epi):
    """Mixed mode with the activation as hi | lo bf16 planes (TMA'd, two MMAs per
    k-step; M <= 128 takes the decode kernel): fp32-grade against fp64 products."""
    import torch
    from paper_2405_01481_b200 import ppoexp as px
    f = px.lib().ppoexp_testing_gemm_planes
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_void_p,
                  C.c_int64]
    f.restype = C.c_int32
    g = torch.Generator(device="cuda").manual_seed(M + N + K + epi)
    A = torch.randn(M, K, generator=g, device="cuda")
    hi = A.to(torch.bfloat16)
    lo = (A - hi.float()).to(torch.bfloat16)
    planes = torch.cat([hi, lo], dim=1).contiguous()
    W = (torch.randn(N, K, generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    ref = (hi.double() + lo.double()) @ W.double().T
    if epi == 6:
        Cm = torch.zeros(M, 2 * N, dtype=torch.bfloat16, device="cuda")
        ldc = 2 * N
    else:
        Cm = torch.randn(M, N, generator=g, device="cuda") if epi == 2 else torch.zeros(M, N, device="cuda")
        ldc = N
    base = Cm.double().clone()
    torch.cuda.synchronize()
    px._check(f(ctx.h, planes.data_ptr(), W.data_ptr(), M, N, K, epi, Cm.data_ptr(), ldc))
    mag = (hi.double().abs() + lo.double().abs()) @ W.double().abs().T
    if epi == 6:
        ref = torch.nn.functional.gelu(ref, approximate="tanh")
        got = Cm[:, :N].double() + Cm[:, N:].double()
        mag = mag * 1.2
    else:
        got = Cm.double()
        if epi == 2:
            ref = ref + base
    err = (got - ref).abs()
    bound = 2.0 ** -16 * mag + 2e-7 * (1 + ref.abs())
    assert (err <= bound).all(), f"max abs err {err.max().item():.3e}, max err/bound {(err / bound).max().item():.3f}"
