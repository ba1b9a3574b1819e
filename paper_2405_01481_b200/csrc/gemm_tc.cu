// gemm_tc.cu — K3 on the 5th-generation tensor cores: C = A · B^T with
// A [M, K] and B [N, K] bf16 K-major, fp32 accumulation in TMEM.
//
//   warp 0      : TMA producer (one elected lane), cp.async.bulk.tensor into a
//                 STAGES-deep ring of 128B-swizzled smem tiles, mbarrier
//                 full/empty handshakes;
//   warp 1      : TMEM allocator + MMA issuer (one lane issues
//                 tcgen05.mma.cta_group::1.kind::f16, tcgen05.commit frees
//                 the smem stage);
//   warps 2..5  : epilogue (tcgen05.ld 32x32b → registers → fused epilogue →
//                 global): bf16 store, GELU (src/model.cpp:358-361), fp32
//                 residual add (src/model.cpp:335, :341) or fp32 store (logits).
// Tiles are visited in grouped-M order so the weight (B) tile of a column
// block is reused from L2 by consecutive CTAs.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <map>
#include <mutex>
#include <tuple>

#include "kernels.hpp"

namespace ppx {

namespace {

constexpr int BM = 128, BK = 64;
constexpr int kThreads = 192;

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
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Shared-memory matrix descriptor: K-major, 128B swizzle, 8-row atoms
// 1024 B apart (SBO = 64 x 16 B), LBO = 1, version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= 1ull << 16;               // LBO (ignored for swizzled K-major)
  d |= 64ull << 32;              // SBO = 1024 B
  d |= 1ull << 46;               // version
  d |= 2ull << 61;               // SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::f16: D f32, A/B bf16, both K-major.
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

template <int BN, bool SPLIT = false>
struct SmemLayout {
  static constexpr int kAT = BM * BK * 2;  // 16 KB: one bf16 A tile
  static constexpr int kA = kAT * (SPLIT ? 2 : 1);  // mixed mode: hi and lo planes of the activation
  static constexpr int kB = BN * BK * 2;
  static constexpr int kStage = kA + kB;
  // ~110 KB of stages: two CTAs share an SM (TMEM: 2 x BN <= 512 columns), so
  // one CTA's epilogue (TMEM -> registers -> global, fp32 residual RMW)
  // overlaps the other's TMA/MMA main loop.  Split 128 x 256 tiles (the LM
  // head's LSE) take one CTA per SM with three 64 KB stages instead.
  static constexpr int kBudget = (SPLIT && BN == 256) ? 200 * 1024 : 110 * 1024;
  static constexpr int kStages = kBudget / kStage > 8 ? 8 : kBudget / kStage;
  static constexpr int kBytes = kStages * kStage + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int kTmemCols = BN < 32 ? 32 : BN;
};

template <int BN, int EPI, bool SPLIT = false>
__global__ void __launch_bounds__(kThreads, 2)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmA2,
                   const __grid_constant__ CUtensorMap tmB, int M, int N, int K, void* __restrict__ Cv, int64_t ldc,
                   int group_m, LseEpi lse) {
  using L = SmemLayout<BN, SPLIT>;
  constexpr int S = L::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * L::kA;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * L::kStage);
  uint64_t* empty = full + S;
  uint64_t* tmem_full = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grouped-M tile order
  const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
  const int t = blockIdx.x;
  const int per_group = group_m * num_n;
  const int g = t / per_group, first_m = g * group_m;
  const int gm = min(num_m - first_m, group_m);
  const int m_blk = first_m + (t % per_group) % gm;
  const int n_blk = (t % per_group) / gm;
  const int m0 = m_blk * BM, n0 = n_blk * BN;
  const int nk = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
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
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % S, r = kb / S;
        if (r > 0) mbar_wait(&empty[s], (r - 1) & 1);
        mbar_expect_tx(&full[s], L::kStage);
        tma_load_2d(&tmA, &full[s], sA + s * L::kA, kb * BK, m0);
        if constexpr (SPLIT) tma_load_2d(&tmA2, &full[s], sA + s * L::kA + L::kAT, kb * BK, m0);
        tma_load_2d(&tmB, &full[s], sB + s * L::kB, kb * BK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(BM, BN);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % S, r = kb / S;
        mbar_wait(&full[s], r & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t da = smem_desc_sw128(sA + s * L::kA);
        const uint64_t db = smem_desc_sw128(sB + s * L::kB);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)  // UMMA_K = 16 (32 bytes): +2 in the >>4 address field
          mma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
        if constexpr (SPLIT) {  // the activation's low-order bf16 term into the same accumulator
          const uint64_t dal = smem_desc_sw128(sA + s * L::kA + L::kAT);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) mma_bf16(tmem, dal + 2 * k, db + 2 * k, idesc, 1);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(tmem_full);
    }
    __syncwarp();
  } else {
    // epilogue warps 2..5 → TMEM lane quarter = warp % 4
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
    if constexpr (EPI == int(Epi::kLse)) {
      // LM head + online log-sum-exp + target gather: the fp32 logits of this
      // row's BN columns never leave registers.  Each tile writes its (max,
      // sum exp(l - max)) partial; the tile holding the row's target also
      // writes the target logit (src/tensor.cpp:428-456, :491-519).
      constexpr float kLog2e = 1.4426950408889634f;
      const int tgt = row < M ? lse.target[row] : -1;
      mbar_wait(tmem_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float m = -INFINITY, s = 0.f, tv = 0.f;
      bool has_t = false;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(c), v);
        const int col = n0 + c;
        if (col >= N) break;
        const int nv = min(32, N - col);
        float cm = -INFINITY;
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (e < nv) cm = fmaxf(cm, __uint_as_float(v[e]));
        if (cm > m) {
          s *= exp2f((m - cm) * kLog2e);
          m = cm;
        }
        const float mb = m * kLog2e;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float f = __uint_as_float(v[e]);
          if (e < nv) s += exp2f(fmaf(f, kLog2e, -mb));
          if (col + e == tgt) {
            tv = f;
            has_t = true;
          }
        }
      }
      if (row < M) {
        lse.part[int64_t(row) * lse.ldp + n_blk] = make_float2(m, s);
        if (has_t) lse.tgt_logit[row] = tv;
      }
    } else {
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t v[32];
      tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(c), v);
      const int col = n0 + c;
      if (row >= M || col >= N) continue;
      const bool full_cols = col + 32 <= N;
      if constexpr (EPI == int(Epi::kGeluSplit)) {
        // GELU output as two bf16 planes: hi at [row, col], lo at [row, N + col]
        bf16* dst = static_cast<bf16*>(Cv) + int64_t(row) * ldc + col;
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          if (col + e + 1 < N || full_cols) {
            const float g0 = gelu_fast(__uint_as_float(v[e])), g1 = gelu_fast(__uint_as_float(v[e + 1]));
            const __nv_bfloat162 h = __floats2bfloat162_rn(g0, g1);
            const float2 hf = __bfloat1622float2(h);
            *reinterpret_cast<__nv_bfloat162*>(dst + e) = h;
            *reinterpret_cast<__nv_bfloat162*>(dst + N + e) = __floats2bfloat162_rn(g0 - hf.x, g1 - hf.y);
          } else if (col + e < N) {
            const float g0 = gelu_fast(__uint_as_float(v[e]));
            const bf16 h = __float2bfloat16_rn(g0);
            dst[e] = h;
            dst[N + e] = __float2bfloat16_rn(g0 - __bfloat162float(h));
          }
        }
      } else if constexpr (EPI == int(Epi::kStore) || EPI == int(Epi::kGelu)) {
        bf16* dst = static_cast<bf16*>(Cv) + int64_t(row) * ldc + col;
        if (full_cols) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            Vec16<bf16> o;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              float f = __uint_as_float(v[j + e]);
              if constexpr (EPI == int(Epi::kGelu)) f = gelu_fast(f);
              o.v[e] = __float2bfloat16_rn(f);
            }
            *reinterpret_cast<uint4*>(dst + j) = o.u;
          }
        } else {  // ragged last column block (unrolled + predicated: v stays in registers)
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            if (col + e < N) {
              float f = __uint_as_float(v[e]);
              if constexpr (EPI == int(Epi::kGelu)) f = gelu_fast(f);
              dst[e] = __float2bfloat16_rn(f);
            }
          }
        }
      } else {
        float* dst = static_cast<float*>(Cv) + int64_t(row) * ldc + col;
        if (full_cols) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 o;
            if constexpr (EPI == int(Epi::kAddResidual)) {
              o = *reinterpret_cast<const float4*>(dst + j);
              o.x += __uint_as_float(v[j]);
              o.y += __uint_as_float(v[j + 1]);
              o.z += __uint_as_float(v[j + 2]);
              o.w += __uint_as_float(v[j + 3]);
            } else {
              o = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                              __uint_as_float(v[j + 3]));
            }
            *reinterpret_cast<float4*>(dst + j) = o;
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            if (col + e < N) {
              if constexpr (EPI == int(Epi::kAddResidual))
                dst[e] += __uint_as_float(v[e]);
              else
                dst[e] = __uint_as_float(v[e]);
            }
          }
        }
      }
    }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L::kTmemCols));
  }
}

}  // namespace

// ------------------------------------------------------------------ host
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 2-D K-major bf16 tensor [rows, cols] with leading dimension ld (elements).
CUtensorMap make_map(const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int64_t, int64_t, int64_t, int>, CUtensorMap> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(ptr, rows, cols, ld, box_rows);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(ld * 2)};
  const cuuint32_t box[2] = {BK, cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  auto fn = encode_fn();
  if (!fn) throw Error(6, "cuda: cuTensorMapEncodeTiled unavailable");
  const CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(6, "cuda: cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  cache.emplace(key, m);
  return m;
}

// General 2-D tensor map (128B swizzle) over [rows, cols] elements of `esz`
// bytes (2: bf16, 4: fp32) with row stride ld elements, box {box_cols, box_rows}.
CUtensorMap make_map_2d(const void* ptr, int esz, int64_t rows, int64_t cols, int64_t ld, int box_cols, int box_rows) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int64_t, int64_t, int64_t, int, int>, CUtensorMap> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(ptr, esz, rows, cols, ld, box_cols, box_rows);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(ld * esz)};
  const cuuint32_t box[2] = {cuuint32_t(box_cols), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  auto fn = encode_fn();
  if (!fn) throw Error(6, "cuda: cuTensorMapEncodeTiled unavailable");
  const CUresult r = fn(&m, esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                        const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(6, "cuda: cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  cache.emplace(key, m);
  return m;
}

namespace {

template <int BN, int EPI, bool SPLIT = false>
void launch_tc(Ctx& c, const bf16* A, int64_t lda, const bf16* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
               void* C, int64_t ldc, const LseEpi& lse = LseEpi{}) {
  using L = SmemLayout<BN, SPLIT>;
  const CUtensorMap ta = make_map(A, M, K, lda, BM);
  // split planes: the activation is [M, 2K] (hi | lo) with row stride lda
  const CUtensorMap ta2 = SPLIT ? make_map(A + K, M, K, lda, BM) : ta;
  const CUtensorMap tb = make_map(B, N, K, ldb, BN);
  auto k = gemm_tc_kernel<BN, EPI, SPLIT>;
  static bool attr = false;
  if (!attr) {
    PPOEXP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes));
    attr = true;
  }
  const int num_m = int(ceil_div(M, BM)), num_n = int(ceil_div(N, BN));
  const int group_m = num_m < 16 ? num_m : 16;
  const double flops = 2.0 * M * N * K;
  const double out_bytes = EPI == int(Epi::kLse) ? double(M) * (num_n * 8 + 8)
                                                 : double(M) * N * ((EPI == 0 || EPI == 1) ? 2 : 4);
  const double bytes = 2.0 * ((SPLIT ? 2 : 1) * M * K + N * K) + out_bytes;
  c.launch(EPI == int(Epi::kLse) ? "lm_head_lse" : (SPLIT ? "gemm_mixed" : "gemm_tc"), bytes, flops, [&] {
    launch_kernel(c, k, dim3(num_m * num_n), dim3(kThreads), L::kBytes, 1, ta, ta2, tb, int(M), int(N), int(K), C,
                  ldc, group_m, lse);
  });
}

template <int BN>
void dispatch_epi(Ctx& c, const bf16* A, int64_t lda, const bf16* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                  Epi epi, void* C, int64_t ldc) {
  switch (epi) {
    case Epi::kStore: return launch_tc<BN, 0>(c, A, lda, B, ldb, M, N, K, C, ldc);
    case Epi::kGelu: return launch_tc<BN, 1>(c, A, lda, B, ldb, M, N, K, C, ldc);
    case Epi::kAddResidual: return launch_tc<BN, 2>(c, A, lda, B, ldb, M, N, K, C, ldc);
    case Epi::kStoreF32: return launch_tc<BN, 3>(c, A, lda, B, ldb, M, N, K, C, ldc);
    case Epi::kLse: throw ContractError("gemm: the LSE epilogue goes through gemm_tc_lse");
    default: throw ContractError("gemm: fp32-activation epilogues go through the mixed-mode GEMMs");
  }
}

}  // namespace

bool gemm_decode_bf16(Ctx& c, const bf16* A, int64_t lda, const bf16* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                      Epi epi, void* C, int64_t ldc);

bool tc_disabled() {
  static const bool off = [] {
    const char* e = getenv("PPOEXP_DISABLE_TC");
    return e && e[0] == '1';
  }();
  return off;
}

// Returns false when the shape is not eligible (the caller then uses the SIMT path).
bool gemm_tc_bf16(Ctx& c, const bf16* A, int64_t lda, const bf16* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                  Epi epi, void* C, int64_t ldc) {
  if (tc_disabled()) return false;
  // TMA: 16-byte aligned base and row stride; K must be a multiple of 8 (16 B).
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) return false;
  if ((lda * 2) % 16 || (ldb * 2) % 16 || K % 8 || ldc % 8) return false;
  if (M <= 0 || N <= 0 || K <= 0) return true;
  // decode-sized M: swap-AB + cluster split-K kernel (gemm_decode.cu)
  if (gemm_decode_bf16(c, A, lda, B, ldb, M, N, K, epi, C, ldc)) return true;
  if (gemm_pp_enabled() && !(reinterpret_cast<uintptr_t>(C) & 15) && epi != Epi::kLse)
    return gemm_persist(c, A, lda, B, ldb, M, N, K, epi, C, ldc, false, nullptr), true;
  const int64_t num_m = ceil_div(M, BM);
  static const int bn_env = [] {
    const char* e = getenv("PPOEXP_TC_BN");
    return e ? atoi(e) : 256;
  }();
  if (bn_env == 256 && num_m * ceil_div(N, 256) >= 148)
    return dispatch_epi<256>(c, A, lda, B, ldb, M, N, K, epi, C, ldc), true;
  return dispatch_epi<128>(c, A, lda, B, ldb, M, N, K, epi, C, ldc), true;
}

// Fused LM head + online LSE + target gather (scoring, bf16 perf mode).
// part[M, ldp] gets one (max, sum exp) pair per 256-column tile.
int lse_tiles(int64_t N) { return int(ceil_div(N, 256)); }

// Mixed mode with the activation as two bf16 planes A[M, 2K] (hi | lo, row
// stride lda >= 2K, written by the producer: split LayerNorm / attention /
// GELU epilogue): both TMA'd, two MMAs per k16 step; 128 x 128 tiles (two
// CTAs per SM), the LSE epilogue on 128 x 256 tiles.
void gemm_tc_planes(Ctx& c, const bf16* A, int64_t lda, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
                    Epi epi, void* C, int64_t ldc, const LseEpi* lse) {
  if (M <= 0 || N <= 0 || K <= 0) return;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(W)) & 15 || (lda * 2) % 16 || (ldw * 2) % 16 ||
      K % 8 || lda < 2 * K)
    throw ContractError("gemm (planes): 16-byte aligned rows, K % 8 and a [M, 2K] activation required");
  if (epi == Epi::kLse) {
    if (!lse || lse->ldp < lse_tiles(N)) throw ContractError("gemm (planes): LSE outputs missing");
    if (gemm_pp_enabled()) return gemm_persist(c, A, lda, W, ldw, M, N, K, epi, nullptr, 0, true, lse);
    return launch_tc<256, int(Epi::kLse), true>(c, A, lda, W, ldw, M, N, K, nullptr, 0, *lse);
  }
  if (M <= 128) return gemm_decode_planes(c, A, lda, W, ldw, M, N, K, epi, C, ldc, nullptr);
  if (gemm_pp_enabled() && !(reinterpret_cast<uintptr_t>(C) & 15) && ldc % 8 == 0)
    return gemm_persist(c, A, lda, W, ldw, M, N, K, epi, C, ldc, true, nullptr);
  static const int bn = [] {  // 256: one CTA per SM, three 64 KB stages; 128: two CTAs per SM
    const char* e = getenv("PPOEXP_PLANES_BN");
    return e ? atoi(e) : 256;
  }();
  if (bn == 128) {
    switch (epi) {
      case Epi::kStoreF32: return launch_tc<128, int(Epi::kStoreF32), true>(c, A, lda, W, ldw, M, N, K, C, ldc);
      case Epi::kAddResidual: return launch_tc<128, int(Epi::kAddResidual), true>(c, A, lda, W, ldw, M, N, K, C, ldc);
      case Epi::kGeluSplit: return launch_tc<128, int(Epi::kGeluSplit), true>(c, A, lda, W, ldw, M, N, K, C, ldc);
      default: throw ContractError("gemm (planes): unsupported epilogue");
    }
  }
  switch (epi) {
    case Epi::kStoreF32: return launch_tc<256, int(Epi::kStoreF32), true>(c, A, lda, W, ldw, M, N, K, C, ldc);
    case Epi::kAddResidual: return launch_tc<256, int(Epi::kAddResidual), true>(c, A, lda, W, ldw, M, N, K, C, ldc);
    case Epi::kGeluSplit: return launch_tc<256, int(Epi::kGeluSplit), true>(c, A, lda, W, ldw, M, N, K, C, ldc);
    default: throw ContractError("gemm (planes): unsupported epilogue");
  }
}

bool gemm_tc_lse(Ctx& c, const bf16* A, int64_t lda, const bf16* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                 const LseEpi& e) {
  if (tc_disabled()) return false;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) return false;
  if ((lda * 2) % 16 || (ldb * 2) % 16 || K % 8) return false;
  if (e.ldp < lse_tiles(N)) throw ContractError("gemm_tc_lse: partial row stride too small");
  if (M <= 0 || N <= 0 || K <= 0) return true;
  if (gemm_pp_enabled()) return gemm_persist(c, A, lda, B, ldb, M, N, K, Epi::kLse, nullptr, 0, false, &e), true;
  launch_tc<256, int(Epi::kLse)>(c, A, lda, B, ldb, M, N, K, nullptr, 0, e);
  return true;
}

}  // namespace ppx
