// gemm_decode.cu — K3 for decode-sized GEMMs (M = active sequences <= 256):
// C[M, N] = X[M, K] · W[N, K]^T computed as D^T = W · X^T ("swap-AB"), so the
// weight rows fill the 128-row tcgen05 M dimension and the batch is the MMA N
// (16..256).  The weight stream is split along K over a thread-block CLUSTER
// of S CTAs (S <= 8): every CTA accumulates its K-slice in TMEM, parks the
// fp32 partial in its own shared memory, and after a cluster barrier each CTA
// reduces 1/S of the feature rows by reading the S partials through DSMEM in
// rank order (deterministic, no global workspace, one launch), then applies
// the fused epilogue.  This turns a weight-bandwidth-bound GEMV into
// (N/128) x S CTAs each streaming a slice, instead of N/128 long K loops.
#include <cooperative_groups.h>
#include <cuda.h>

#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace ppx {

CUtensorMap make_map(const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);  // gemm_tc.cu

namespace {

constexpr int BMW = 128, BK = 64, kThreads = 192, kStages = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  const uint64_t addr = smem_u32(p);
  return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int NB>
struct DecLayout {
  static constexpr int kW = BMW * BK * 2;  // 16 KB weight tile
  static constexpr int kX = NB * BK * 2;   // activation tile
  static constexpr int kStage = kW + kX;
  static constexpr int kPart = NB * BMW * 4;  // fp32 partial [NB][128], feature-contiguous
  static constexpr int kPipe = kStages * kStage;
  static constexpr int kBody = kPipe > kPart ? kPipe : kPart;
  static constexpr int kBytes = kBody + 1024 + 256;
  static constexpr int kTmemCols = NB < 32 ? 32 : (NB <= 32 ? 32 : (NB <= 64 ? 64 : (NB <= 128 ? 128 : 256)));
};

template <int NB, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_decode_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, int Mrows,
                       int N, int K, void* __restrict__ Cv, int64_t ldc, int S) {
  using L = DecLayout<NB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sX = smem + kStages * L::kW;
  float* part = reinterpret_cast<float*>(smem);  // reused after the MMA loop
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBody);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  cg::cluster_group cluster = cg::this_cluster();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BMW;
  const int r = blockIdx.y;  // K-split rank == cluster rank (cluster spans y)
  const int nk = (K + BK - 1) / BK;
  const int kb0 = int((int64_t(r) * nk) / S), kb1 = int((int64_t(r + 1) * nk) / S);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(L::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // The weights are constant across the graph: stream the first stages of
      // them BEFORE waiting on the predecessor grid (PDL), so their HBM latency
      // overlaps the previous kernel.  Activations are loaded after the wait.
      const int pre = min(kStages, kb1 - kb0);
      for (int it = 0; it < pre; ++it) {
        mbar_expect_tx(&full[it], L::kStage);
        tma_load_2d(&tmW, &full[it], sW + it * L::kW, (kb0 + it) * BK, n0);
      }
      pdl_wait();
      pdl_trigger();
      for (int it = 0; it < pre; ++it) tma_load_2d(&tmX, &full[it], sX + it * L::kX, (kb0 + it) * BK, 0);
      for (int kb = kb0 + pre; kb < kb1; ++kb) {
        const int it = kb - kb0, s = it % kStages, u = it / kStages;
        if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
        mbar_expect_tx(&full[s], L::kStage);
        tma_load_2d(&tmW, &full[s], sW + s * L::kW, kb * BK, n0);
        tma_load_2d(&tmX, &full[s], sX + s * L::kX, kb * BK, 0);
      }
    } else {
      pdl_wait();
    }
  } else if (warp == 1) {
    pdl_wait();
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(BMW, NB);
      for (int kb = kb0; kb < kb1; ++kb) {
        const int it = kb - kb0, s = it % kStages, u = it / kStages;
        mbar_wait(&full[s], u & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t dw = smem_desc_sw128(sW + s * L::kW);
        const uint64_t dx = smem_desc_sw128(sX + s * L::kX);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) mma_bf16(tmem, dw + 2 * k, dx + 2 * k, idesc, (it | k) != 0);
        mma_commit(&empty[s]);
      }
      mma_commit(tmem_full);
    }
    __syncwarp();
  } else {
    pdl_wait();  // the epilogue reads/writes C, produced upstream
    // TMEM (feature rows x batch cols) → smem partial
    const int q = warp & 3;
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int f = q * 32 + lane;
#pragma unroll 1
    for (int c = 0; c < NB; c += 16) {
      uint32_t v[16];
      tmem_ld16(tmem + (uint32_t(q * 32) << 16) + uint32_t(c), v);
#pragma unroll
      for (int e = 0; e < 16; ++e) part[(c + e) * BMW + f] = __uint_as_float(v[e]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster.sync();  // all partials of the cluster are parked in smem
  // reduce feature rows [f0, f1) of this CTA over the S partials, in rank
  // order: float4 DSMEM loads, all S issued before the adds
  const int rows_per = ((BMW / S) + 3) & ~3;  // multiple of 4 features
  const int f0 = r * rows_per, f1 = min(BMW, f0 + rows_per);
  const int nf4 = (f1 - f0) / 4;
  const int ncols = min(Mrows, NB);
  const float4* parts[8];
  for (int k = 0; k < 8; ++k) parts[k] = reinterpret_cast<const float4*>(cluster.map_shared_rank(part, k < S ? k : 0));
  for (int e = threadIdx.x; e < nf4 * ncols; e += kThreads) {
    const int fl = f0 + 4 * (e % nf4), bcol = e / nf4;
    const int idx = (bcol * BMW + fl) >> 2;
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < S) v[k] = parts[k][idx];
    float4 acc = v[0];
#pragma unroll
    for (int k = 1; k < 8; ++k)
      if (k < S) {
        acc.x += v[k].x;
        acc.y += v[k].y;
        acc.z += v[k].z;
        acc.w += v[k].w;
      }
    const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + fl + j;
      if (n >= N) break;
      const float a = a4[j];
      const int64_t o = int64_t(bcol) * ldc + n;
      if constexpr (EPI == int(Epi::kStore)) {
        static_cast<bf16*>(Cv)[o] = __float2bfloat16_rn(a);
      } else if constexpr (EPI == int(Epi::kGelu)) {
        static_cast<bf16*>(Cv)[o] = __float2bfloat16_rn(gelu_tanh(a));
      } else if constexpr (EPI == int(Epi::kAddResidual)) {
        static_cast<float*>(Cv)[o] += a;
      } else {
        static_cast<float*>(Cv)[o] = a;
      }
    }
  }
  cluster.sync();  // keep our smem alive until every peer has read it
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L::kTmemCols));
  }
}

template <int NB, int EPI>
void launch_dec(Ctx& c, const bf16* X, int64_t ldx, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
                void* C, int64_t ldc) {
  using L = DecLayout<NB>;
  const CUtensorMap tw = make_map(W, N, K, ldw, BMW);
  const CUtensorMap tx = make_map(X, M, K, ldx, NB);
  auto k = gemm_decode_kernel<NB, EPI>;
  static bool attr = false;
  if (!attr) {
    PPOEXP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes));
    PPOEXP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  const int tiles = int(ceil_div(N, BMW));
  const int nk = int(ceil_div(K, BK));
  // K-split: aim for >= ~148 CTAs, at most 8 (portable cluster), >= 2 k-blocks each
  static const int smax = [] {
    const char* e = getenv("PPOEXP_DECODE_SPLIT_MAX");
    return e ? atoi(e) : 4;
  }();
  static const int target = [] {
    const char* e = getenv("PPOEXP_DECODE_CTA_TARGET");
    return e ? atoi(e) : 148;
  }();
  int S = 1;
  while (S < smax && tiles * S < target && nk >= 2 * S) S *= 2;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(tiles, S, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = L::kBytes;
  cfg.stream = c.stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 1;
  attrs[0].val.clusterDim.y = S;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  const double flops = 2.0 * M * N * K;
  const double bytes = 2.0 * (N * K + M * K) + double(M) * N * ((EPI == 0 || EPI == 1) ? 2 : 4);
  c.launch("gemm_decode", bytes, flops, [&] {
    PPOEXP_CUDA(cudaLaunchKernelEx(&cfg, k, tw, tx, int(M), int(N), int(K), C, ldc, S));
  });
}

template <int NB>
void dispatch(Ctx& c, const bf16* X, int64_t ldx, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
              Epi epi, void* C, int64_t ldc) {
  switch (epi) {
    case Epi::kStore: return launch_dec<NB, 0>(c, X, ldx, W, ldw, M, N, K, C, ldc);
    case Epi::kGelu: return launch_dec<NB, 1>(c, X, ldx, W, ldw, M, N, K, C, ldc);
    case Epi::kAddResidual: return launch_dec<NB, 2>(c, X, ldx, W, ldw, M, N, K, C, ldc);
    case Epi::kStoreF32: return launch_dec<NB, 3>(c, X, ldx, W, ldw, M, N, K, C, ldc);
  }
}

}  // namespace

// Decode-sized GEMM (M <= 256).  Returns false if not eligible.
bool gemm_decode_bf16(Ctx& c, const bf16* A, int64_t lda, const bf16* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                      Epi epi, void* C, int64_t ldc) {
  if (M > 256 || M <= 0) return false;
  if (M <= 32) return dispatch<32>(c, A, lda, B, ldb, M, N, K, epi, C, ldc), true;
  if (M <= 64) return dispatch<64>(c, A, lda, B, ldb, M, N, K, epi, C, ldc), true;
  if (M <= 128) return dispatch<128>(c, A, lda, B, ldb, M, N, K, epi, C, ldc), true;
  return dispatch<256>(c, A, lda, B, ldb, M, N, K, epi, C, ldc), true;
}

}  // namespace ppx
