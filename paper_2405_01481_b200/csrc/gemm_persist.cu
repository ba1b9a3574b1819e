// gemm_persist.cu — K3p: persistent tcgen05 GEMM for the prefill / scoring
// forwards.  C = A · W^T with W bf16 [N, K] (K-major weights) and A either
// one bf16 operand [M, K] or, in mixed mode, the activation's two bf16 terms
// as planes [M, 2K] (hi | lo, written by the producer: split LayerNorm,
// attention output, GELU epilogue) issued as two MMAs into one accumulator.
//
// One CTA per SM walks the 128 x 256 output tiles (grouped-M order, stride =
// grid).  Warp 0 streams A / W k-blocks through a 3-stage (planes) or 4-stage
// 128B-swizzled TMA ring; warp 1 issues the MMAs into one of two TMEM
// accumulators (2 x 256 columns = all of TMEM), so the epilogue of tile i
// runs while the tensor cores work on tile i + 1; warps 2-5 drain the
// accumulator (tcgen05.ld), apply the epilogue and write through per-warp
// swizzled smem boxes with TMA bulk stores (fp32 residual add as a TMA
// reduce-add: one add per element, the same fp32 rounding as x + v).
#include <cuda.h>

#include "kernels.hpp"

namespace ppx {

CUtensorMap make_map(const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);  // gemm_tc.cu
CUtensorMap make_map_2d(const void* ptr, int esz, int64_t rows, int64_t cols, int64_t ld, int box_cols, int box_rows);

namespace {

constexpr int BM = 128, BN = 256, BK = 64, kThreads = 192;

template <bool SPLIT>
struct PL {
  static constexpr int kAT = BM * BK * 2;  // 16 KB: one bf16 A tile
  static constexpr int kA = kAT * (SPLIT ? 2 : 1);
  static constexpr int kB = BN * BK * 2;   // 32 KB
  static constexpr int kStage = kA + kB;
  static constexpr int kStages = SPLIT ? 3 : 4;  // 192 KB of ring
  static constexpr int kEpiWarp = 8192;          // per epilogue warp: two 4 KB store boxes
  static constexpr int kBytes = kStages * kStage + 4 * kEpiWarp + 1024 + 256;
};

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
__device__ __forceinline__ void tma_load(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(su32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_add(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(su32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
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
// 16 bytes into row `r` (128 B) of a 128B-swizzled box at 16-byte chunk j
__device__ __forceinline__ void st_sw(uint8_t* box, int r, int j, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(su32(box + r * 128 + ((j ^ (r & 7)) << 4))), "r"(a),
               "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

template <int EPI, bool SPLIT>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_pp_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmA2,
                   const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmC,
                   const __grid_constant__ CUtensorMap tmC2, int M, int N, int K, int group_m, LseEpi lse) {
  using L = PL<SPLIT>;
  constexpr int S = L::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_smem = smem + S * L::kStage;  // 1024-aligned (kStage is a multiple of 16 KB)
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + 4 * L::kEpiWarp);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN, tiles = num_m * num_n;
  const int nk = (K + BK - 1) / BK;
  const int per_group = group_m * num_n;
  auto tile_mn = [&](int t, int& m_blk, int& n_blk) {
    const int g = t / per_group, first_m = g * group_m;
    const int gm = min(num_m - first_m, group_m);
    m_blk = first_m + (t % per_group) % gm;
    n_blk = (t % per_group) / gm;
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int m_blk, n_blk;
        tile_mn(t, m_blk, n_blk);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % S, r = it / S;
          if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
          uint8_t* st = smem + s * L::kStage;
          mbar_expect_tx(&full[s], L::kStage);
          tma_load(&tmA, &full[s], st, kb * BK, m_blk * BM);
          if constexpr (SPLIT) tma_load(&tmA2, &full[s], st + L::kAT, kb * BK, m_blk * BM);
          tma_load(&tmB, &full[s], st + L::kA, kb * BK, n_blk * BN);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(BM, BN);
      int it = 0, lt = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++lt) {
        const int acc = lt & 1, use = lt >> 1;
        if (use > 0) mbar_wait(&acc_empty[acc], (use - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + uint32_t(acc * BN);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % S, r = it / S;
          mbar_wait(&full[s], r & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          uint8_t* st = smem + s * L::kStage;
          const uint64_t da = desc_sw128(st), db = desc_sw128(st + L::kA);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) mma(d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          if constexpr (SPLIT) {
            const uint64_t dl = desc_sw128(st + L::kAT);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) mma(d, dl + 2 * k, db + 2 * k, idesc, 1);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&acc_full[acc]);
      }
    }
    __syncwarp();
  } else {
    // epilogue: warp w drains TMEM lanes 32 (w % 4) .. +31 = rows m0 + 32 q + lane
    const int q = warp & 3;
    uint8_t* box0 = epi_smem + (warp - 2) * L::kEpiWarp;
    int lt = 0, nbox = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++lt) {
      int m_blk, n_blk;
      tile_mn(t, m_blk, n_blk);
      const int acc = lt & 1, use = lt >> 1;
      const int m0 = m_blk * BM, n0 = n_blk * BN, r0 = m0 + q * 32, row = r0 + lane;
      mbar_wait(&acc_full[acc], use & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tbase = tmem + (uint32_t(q * 32) << 16) + uint32_t(acc * BN);
      if constexpr (EPI == int(Epi::kLse)) {
        constexpr float kLog2e = 1.4426950408889634f;
        const int tgt = row < M ? lse.target[row] : -1;
        float lm = -INFINITY, ls = 0.f, tv = 0.f;
        bool has_t = false;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          if (n0 + c >= N) break;
          uint32_t v[32];
          tmem_ld32(tbase + uint32_t(c), v);
          const int col = n0 + c, nv = min(32, N - col);
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
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[acc]);
        if (row < M) {
          lse.part[int64_t(row) * lse.ldp + n_blk] = make_float2(lm, ls);
          if (has_t) lse.tgt_logit[row] = tv;
        }
      } else if constexpr (EPI == int(Epi::kStoreF32) || EPI == int(Epi::kAddResidual) ||
                           EPI == int(Epi::kGeluF32)) {
        // 32-column fp32 boxes [32 rows x 128 B], two per warp in flight
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          if (n0 + c >= N) break;
          uint32_t v[32];
          tmem_ld32(tbase + uint32_t(c), v);
          if (c + 32 >= BN || n0 + c + 32 >= N) {  // the accumulator is free once the last columns are read
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[acc]);
          }
          if constexpr (EPI == int(Epi::kGeluF32)) {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(gelu_fast(__uint_as_float(v[e])));
          }
          uint8_t* box = box0 + (nbox & 1) * 4096;
          if (lane == 0) bulk_wait_read<1>();  // the store issued from this box two boxes ago has read it
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j) st_sw(box, lane, j, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if constexpr (EPI == int(Epi::kAddResidual))
              tma_add(&tmC, box, n0 + c, r0);
            else
              tma_store(&tmC, box, n0 + c, r0);
            bulk_commit();
          }
          ++nbox;
        }
      } else {
        // bf16 outputs, 64-column boxes [32 rows x 128 B]: kStore / kGelu (one
        // plane, double-buffered) or kGeluSplit (hi and lo planes, one box each)
#pragma unroll 1
        for (int c = 0; c < BN; c += 64) {
          if (n0 + c >= N) break;
          uint32_t v[32], w[32];
          tmem_ld32(tbase + uint32_t(c), v);
          const bool second = n0 + c + 32 < N;
          if (second) tmem_ld32(tbase + uint32_t(c + 32), w);
          if (c + 64 >= BN || n0 + c + 64 >= N) {
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[acc]);
          }
          constexpr bool kSplitOut = EPI == int(Epi::kGeluSplit) || EPI == int(Epi::kStoreSplit);
          uint8_t* box = box0 + (kSplitOut ? 0 : (nbox & 1) * 4096);
          if (lane == 0) {
            if constexpr (kSplitOut)
              bulk_wait_read<0>();
            else
              bulk_wait_read<1>();
          }
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float g[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int k = 8 * j + e;
              float x = __uint_as_float(k < 32 ? v[k] : (second ? w[k - 32] : 0u));
              if constexpr (EPI == int(Epi::kGelu) || EPI == int(Epi::kGeluSplit)) x = gelu_fast(x);
              g[e] = x;
            }
            uint32_t h[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) h[e] = pack_bf16(g[2 * e], g[2 * e + 1]);
            st_sw(box, lane, j, h[0], h[1], h[2], h[3]);
            if constexpr (kSplitOut) {
              uint32_t l[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const __nv_bfloat162 hh = *reinterpret_cast<const __nv_bfloat162*>(&h[e]);
                const float2 hf = __bfloat1622float2(hh);
                l[e] = pack_bf16(g[2 * e] - hf.x, g[2 * e + 1] - hf.y);
              }
              st_sw(box + 4096, lane, j, l[0], l[1], l[2], l[3]);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store(&tmC, box, n0 + c, r0);
            if constexpr (kSplitOut) tma_store(&tmC2, box + 4096, n0 + c, r0);
            bulk_commit();
          }
          ++nbox;
        }
      }
    }
    if (lane == 0) bulk_wait_read<0>();  // smem stays valid until every store has read it
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

int num_sms() {
  static const int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <int EPI, bool SPLIT>
void launch_pp(Ctx& c, const bf16* A, int64_t lda, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
               void* C, int64_t ldc, const LseEpi& lse) {
  using L = PL<SPLIT>;
  const CUtensorMap ta = make_map(A, M, K, lda, BM);
  const CUtensorMap ta2 = SPLIT ? make_map(A + K, M, K, lda, BM) : ta;
  const CUtensorMap tb = make_map(W, N, K, ldw, BN);
  CUtensorMap tc = tb, tc2 = tb;
  if constexpr (EPI == int(Epi::kStoreF32) || EPI == int(Epi::kAddResidual) || EPI == int(Epi::kGeluF32)) {
    tc = make_map_2d(C, 4, M, N, ldc, 32, 32);
  } else if constexpr (EPI == int(Epi::kStore) || EPI == int(Epi::kGelu)) {
    tc = make_map_2d(C, 2, M, N, ldc, 64, 32);
  } else if constexpr (EPI == int(Epi::kGeluSplit) || EPI == int(Epi::kStoreSplit)) {
    tc = make_map_2d(C, 2, M, N, ldc, 64, 32);  // hi plane: columns [0, N)
    tc2 = make_map_2d(static_cast<const bf16*>(C) + N, 2, M, N, ldc, 64, 32);  // lo plane: [N, 2N)
  }
  auto k = gemm_pp_kernel<EPI, SPLIT>;
  static bool attr = false;
  if (!attr) {
    PPOEXP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes));
    attr = true;
  }
  const int num_m = int(ceil_div(M, BM)), num_n = int(ceil_div(N, BN));
  const int group_m = num_m < 16 ? num_m : 16;
  const int grid = std::min(num_m * num_n, num_sms());
  const double flops = 2.0 * M * N * K;  // algorithmic (planes issue twice as many MMAs)
  const double a_bytes = double(M) * K * (SPLIT ? 4 : 2);
  double out_bytes = double(M) * N * 4;
  if (EPI == int(Epi::kLse)) out_bytes = double(M) * (num_n * 8 + 8);
  if (EPI == int(Epi::kStore) || EPI == int(Epi::kGelu)) out_bytes = double(M) * N * 2;
  if (EPI == int(Epi::kAddResidual)) out_bytes = double(M) * N * 8;
  if (EPI == int(Epi::kGeluSplit) || EPI == int(Epi::kStoreSplit)) out_bytes = double(M) * N * 4;
  const char* cls = EPI == int(Epi::kLse) ? "lm_head_lse" : (SPLIT ? "gemm_mixed" : "gemm_tc");
  c.launch(cls, a_bytes + 2.0 * N * K + out_bytes, flops, [&] {
    launch_kernel(c, k, dim3(grid), dim3(kThreads), L::kBytes, 1, ta, ta2, tb, tc, tc2, int(M), int(N), int(K),
                  group_m, lse);
  });
}

}  // namespace

bool gemm_pp_enabled() {
  static const bool on = [] {
    const char* e = getenv("PPOEXP_GEMM_PERSIST");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Persistent GEMM over a bf16 activation (SPLIT = false) or hi | lo planes
// (SPLIT = true, A = [M, 2K] with row stride lda).  Output alignment: 16-byte
// rows (TMA); the caller checks eligibility.
void gemm_persist(Ctx& c, const bf16* A, int64_t lda, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
                  Epi epi, void* C, int64_t ldc, bool split, const LseEpi* lse) {
  if (M <= 0 || N <= 0 || K <= 0) return;
  const LseEpi le = lse ? *lse : LseEpi{};
  if (split) {
    switch (epi) {
      case Epi::kStoreF32: return launch_pp<int(Epi::kStoreF32), true>(c, A, lda, W, ldw, M, N, K, C, ldc, le);
      case Epi::kAddResidual: return launch_pp<int(Epi::kAddResidual), true>(c, A, lda, W, ldw, M, N, K, C, ldc, le);
      case Epi::kGeluSplit: return launch_pp<int(Epi::kGeluSplit), true>(c, A, lda, W, ldw, M, N, K, C, ldc, le);
      case Epi::kStoreSplit: return launch_pp<int(Epi::kStoreSplit), true>(c, A, lda, W, ldw, M, N, K, C, ldc, le);
      case Epi::kGeluF32: return launch_pp<int(Epi::kGeluF32), true>(c, A, lda, W, ldw, M, N, K, C, ldc, le);
      case Epi::kLse: return launch_pp<int(Epi::kLse), true>(c, A, lda, W, ldw, M, N, K, C, ldc, le);
      default: throw ContractError("gemm (persistent planes): unsupported epilogue");
    }
  }
  switch (epi) {
    case Epi::kStore: return launch_pp<int(Epi::kStore), false>(c, A, lda, W, ldw, M, N, K, C, ldc, le);
    case Epi::kGelu: return launch_pp<int(Epi::kGelu), false>(c, A, lda, W, ldw, M, N, K, C, ldc, le);
    case Epi::kStoreF32: return launch_pp<int(Epi::kStoreF32), false>(c, A, lda, W, ldw, M, N, K, C, ldc, le);
    case Epi::kAddResidual: return launch_pp<int(Epi::kAddResidual), false>(c, A, lda, W, ldw, M, N, K, C, ldc, le);
    case Epi::kLse: return launch_pp<int(Epi::kLse), false>(c, A, lda, W, ldw, M, N, K, C, ldc, le);
    default: throw ContractError("gemm (persistent): unsupported epilogue");
  }
}

}  // namespace ppx
