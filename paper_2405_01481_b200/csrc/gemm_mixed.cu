// gemm_mixed.cu — K3 in mixed mode: C = A · W^T with A fp32 [M, K] (the
// activation) and W bf16 [N, K] (the weights, K-major), on the tcgen05 tensor
// cores with fp32-grade products.  The weights are exactly bf16 (both sides of
// the parity check use the same bf16-rounded weights), so only the activation
// has to be represented more finely than one bf16: each fp32 element is split
// into hi = bf16(a) and lo = bf16(a - hi) (|a - hi - lo| <= 2^-17 |a|) and the
// tile is issued as two MMAs into the same TMEM accumulator.
//
//   warp 0      : TMA producer of the weight tiles (128B swizzle);
//   warp 1      : TMEM allocator + MMA issuer (2 x 4 UMMA_K steps per k-block);
//   warps 2..5  : activation producers during the main loop (fp32 global ->
//                 registers, one k-block ahead -> hi / lo bf16 tiles written in
//                 the UMMA 128B-swizzled K-major layout), then the epilogue
//                 (fp32 store, GELU, residual add, or LM head + online LSE).
// One 128 x 256 tile per CTA, 3-stage ring (64 KB per stage), one CTA per SM.
#include <cuda.h>

#include "kernels.hpp"

namespace ppx {

CUtensorMap make_map(const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);  // gemm_tc.cu

namespace {

constexpr int BM = 128, BN = 256, BK = 64, kStages = 3, kThreads = 192;
constexpr int kTileA = BM * BK * 2;  // 16 KB (one bf16 term)
constexpr int kTileB = BN * BK * 2;  // 32 KB
constexpr int kStage = 2 * kTileA + kTileB;
constexpr int kSmem = kStages * kStage + 1024 + 256;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\nWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}" ::"r"(
          su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ uint64_t desc_sw128(const void* p) {
  const uint64_t a = su32(p);
  return ((a >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 8 chunks of 8 fp32 per producer thread per k-block: chunk q = et + 128 c
// covers row q >> 3, columns 8 (q & 7) .. +7 (8 threads read one 256-byte row).
struct AChunks {
  float4 v[8][2];
};

__device__ __forceinline__ void load_a(AChunks& a, const float* __restrict__ A, int64_t lda, int M, int K, int m0,
                                       int kb, int et) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int q = et + c * 128, row = m0 + (q >> 3), col = kb * BK + (q & 7) * 8;
    if (row < M && col < K) {
      const float4* p = reinterpret_cast<const float4*>(A + int64_t(row) * lda + col);
      a.v[c][0] = __ldg(p);
      a.v[c][1] = __ldg(p + 1);
    } else {
      a.v[c][0] = a.v[c][1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

__device__ __forceinline__ void store_split(const AChunks& a, uint8_t* hi, uint8_t* lo, int et) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int q = et + c * 128, r = q >> 3, c8 = q & 7;
    const float x[8] = {a.v[c][0].x, a.v[c][0].y, a.v[c][0].z, a.v[c][0].w,
                        a.v[c][1].x, a.v[c][1].y, a.v[c][1].z, a.v[c][1].w};
    uint32_t h[4], l[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {  // packed cvt.rn.bf16x2.f32: one conversion per pair
      const __nv_bfloat162 hp = __floats2bfloat162_rn(x[2 * e], x[2 * e + 1]);
      const float2 hf = __bfloat1622float2(hp);
      const __nv_bfloat162 lp = __floats2bfloat162_rn(x[2 * e] - hf.x, x[2 * e + 1] - hf.y);
      h[e] = *reinterpret_cast<const uint32_t*>(&hp);
      l[e] = *reinterpret_cast<const uint32_t*>(&lp);
    }
    const int off = r * 128 + ((c8 ^ (r & 7)) << 4);
    *reinterpret_cast<uint4*>(hi + off) = make_uint4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<uint4*>(lo + off) = make_uint4(l[0], l[1], l[2], l[3]);
  }
}

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_mixed_kernel(const float* __restrict__ A, int64_t lda, const __grid_constant__ CUtensorMap tmB, int M, int N,
                      int K, void* __restrict__ Cv, int64_t ldc, int group_m, LseEpi lse) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStage);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  auto sAh = [&](int s) { return smem + s * kStage; };
  auto sAl = [&](int s) { return smem + s * kStage + kTileA; };
  auto sB = [&](int s) { return smem + s * kStage + 2 * kTileA; };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
  const int t = blockIdx.x, per_group = group_m * num_n;
  const int g = t / per_group, first_m = g * group_m;
  const int gm = min(num_m - first_m, group_m);
  const int m_blk = first_m + (t % per_group) % gm, n_blk = (t % per_group) / gm;
  const int m0 = m_blk * BM, n0 = n_blk * BN;
  const int nk = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1 + 128);  // the TMA arrival (+ bytes) and the 128 producer threads
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)), "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0)
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kStages, r = kb / kStages;
        if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
        mbar_expect_tx(&full[s], kTileB);
        tma_2d(&tmB, &full[s], sB(s), kb * BK, n0);
      }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(BM, BN);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kStages, r = kb / kStages;
        mbar_wait(&full[s], r & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t dh = desc_sw128(sAh(s)), dl = desc_sw128(sAl(s)), db = desc_sw128(sB(s));
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          mma(tmem, dh + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          mma(tmem, dl + 2 * k, db + 2 * k, idesc, 1);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(tmem_full);
    }
    __syncwarp();
  } else {
    const int et = threadIdx.x - 64;
    // ---- activation producers: k-block kb+1 is in flight while kb is split
    {
      AChunks a0, a1;
      if (nk > 0) load_a(a0, A, lda, M, K, m0, 0, et);
      for (int kb = 0; kb < nk; kb += 2) {
        if (kb + 1 < nk) load_a(a1, A, lda, M, K, m0, kb + 1, et);
        {
          const int s = kb % kStages, r = kb / kStages;
          if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
          store_split(a0, sAh(s), sAl(s), et);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&full[s]);
        }
        if (kb + 1 >= nk) break;
        if (kb + 2 < nk) load_a(a0, A, lda, M, K, m0, kb + 2, et);
        {
          const int s = (kb + 1) % kStages, r = (kb + 1) / kStages;
          if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
          store_split(a1, sAh(s), sAl(s), et);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&full[s]);
        }
      }
    }
    // ---- epilogue: TMEM lane quarter = warp % 4 → rows m0 + 32 q + lane
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
    constexpr float kLog2e = 1.4426950408889634f;
    const int tgt = (EPI == int(Epi::kLse) && row < M) ? lse.target[row] : -1;
    float lm = -INFINITY, ls = 0.f, tv = 0.f;
    bool has_t = false;
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t v[32];
      tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(c), v);
      const int col = n0 + c;
      if (col >= N) break;
      const int nv = min(32, N - col);
      if constexpr (EPI == int(Epi::kLse)) {
        float cm = -INFINITY;
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (e < nv) cm = fmaxf(cm, __uint_as_float(v[e]));
        if (cm > lm) {
          ls *= exp2f((lm - cm) * kLog2e);
          lm = cm;
        }
        const float mb = lm * kLog2e;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float f = __uint_as_float(v[e]);
          if (e < nv) ls += exp2f(fmaf(f, kLog2e, -mb));
          if (col + e == tgt) {
            tv = f;
            has_t = true;
          }
        }
      } else {
        if (row >= M) continue;
        float* dst = static_cast<float*>(Cv) + int64_t(row) * ldc + col;
        if (nv == 32 && (ldc & 3) == 0) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 o = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                                   __uint_as_float(v[j + 3]));
            if constexpr (EPI == int(Epi::kAddResidual)) {
              const float4 x = *reinterpret_cast<const float4*>(dst + j);
              o.x += x.x;
              o.y += x.y;
              o.z += x.z;
              o.w += x.w;
            } else if constexpr (EPI == int(Epi::kGeluF32)) {
              o = make_float4(gelu_fast(o.x), gelu_fast(o.y), gelu_fast(o.z), gelu_fast(o.w));
            }
            *reinterpret_cast<float4*>(dst + j) = o;
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            if (e < nv) {
              const float a = __uint_as_float(v[e]);
              if constexpr (EPI == int(Epi::kAddResidual))
                dst[e] += a;
              else if constexpr (EPI == int(Epi::kGeluF32))
                dst[e] = gelu_fast(a);
              else
                dst[e] = a;
            }
          }
        }
      }
    }
    if constexpr (EPI == int(Epi::kLse)) {
      if (row < M) {
        lse.part[int64_t(row) * lse.ldp + n_blk] = make_float2(lm, ls);
        if (has_t) lse.tgt_logit[row] = tv;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
  }
}

template <int EPI>
void launch_mixed(Ctx& c, const float* A, int64_t lda, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
                  void* C, int64_t ldc, const LseEpi& lse) {
  const CUtensorMap tb = make_map(W, N, K, ldw, BN);
  auto k = gemm_mixed_kernel<EPI>;
  static bool attr = false;
  if (!attr) {
    PPOEXP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr = true;
  }
  const int num_m = int(ceil_div(M, BM)), num_n = int(ceil_div(N, BN));
  const int group_m = num_m < 16 ? num_m : 16;
  const double flops = 2.0 * M * N * K;  // algorithmic (the split issues twice as many MMAs)
  const double out_bytes = EPI == int(Epi::kLse) ? double(M) * (num_n * 8 + 8) : double(M) * N * 4;
  const double bytes = 4.0 * M * K + 2.0 * N * K + out_bytes;
  c.launch(EPI == int(Epi::kLse) ? "lm_head_lse" : "gemm_mixed", bytes, flops, [&] {
    launch_kernel(c, k, dim3(num_m * num_n), dim3(kThreads), kSmem, 1, A, lda, tb, int(M), int(N), int(K), C, ldc,
                  group_m, lse);
  });
}

}  // namespace

void gemm_mixed(Ctx& c, const float* A, int64_t lda, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
                Epi epi, void* C, int64_t ldc, const LseEpi* lse) {
  if (M <= 0 || N <= 0 || K <= 0) return;
  if (K % 8 || lda % 4 || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(W) & 15) || (ldw * 2) % 16)
    throw ContractError("gemm (mixed): K % 8, 16-byte aligned rows required");
  if (epi == Epi::kLse) {
    if (!lse || lse->ldp < lse_tiles(N)) throw ContractError("gemm (mixed): LSE outputs missing");
    return launch_mixed<int(Epi::kLse)>(c, A, lda, W, ldw, M, N, K, nullptr, 0, *lse);
  }
  // decode-sized M on the swap-AB split-K kernel (its split-activation ring holds
  // one stage at M > 128, so larger prefill batches use the 128 x 256 tiles)
  if (M <= 128) return gemm_decode_mixed(c, A, lda, W, ldw, M, N, K, epi, C, ldc, nullptr, nullptr);
  switch (epi) {
    case Epi::kStoreF32: return launch_mixed<int(Epi::kStoreF32)>(c, A, lda, W, ldw, M, N, K, C, ldc, LseEpi{});
    case Epi::kGeluF32: return launch_mixed<int(Epi::kGeluF32)>(c, A, lda, W, ldw, M, N, K, C, ldc, LseEpi{});
    case Epi::kAddResidual: return launch_mixed<int(Epi::kAddResidual)>(c, A, lda, W, ldw, M, N, K, C, ldc, LseEpi{});
    default: throw ContractError("gemm (mixed): fp32 epilogues only");
  }
}

}  // namespace ppx
