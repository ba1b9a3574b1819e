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

#include <algorithm>
#include <vector>

#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace ppx {

CUtensorMap make_map(const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);  // gemm_tc.cu

namespace {

constexpr int BMW = 128, BK = 64, kThreads = 192;
constexpr int kMaxS = 16;  // K-split ranks per cluster (16 = non-portable cluster size)

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

// Shared memory: a ring of `wst` 16 KB weight tiles (all of this CTA's K
// slice when it fits → fetched entirely before the grid-dependency wait), an
// XST-deep ring of activation tiles, then barriers.  The fp32 partial used by
// the split-K reduction reuses the weight ring after the MMAs complete.
// Activation operand modes (XM): 0 = bf16 tile by TMA; 1 = LayerNorm fused
// (fp32 x + row statistics normalised by the epilogue threads into bf16);
// 2 = fp32 activation split by the epilogue threads into two bf16 terms
// (hi = bf16(a), lo = bf16(a - hi)) issued as two MMAs into one accumulator
// (mixed mode: bf16 weights, fp32-grade activations); 3 = LayerNorm fused + split;
// 4 = split terms that arrive as two bf16 planes [rows, 2K] (hi | lo, written
// by the producer kernel), both TMA'd.
template <int XM>
struct XMode {
  static constexpr bool kLn = XM == 1 || XM == 3;
  static constexpr bool kSplit = XM >= 2;
  static constexpr bool kProduced = XM == 1 || XM == 2 || XM == 3;  // the epilogue threads write the X tiles
};

template <int NB, bool SPLIT = false>
struct DecLayout {
  static constexpr int kW = BMW * BK * 2;  // 16 KB weight tile
  static constexpr int kXT = NB * BK * 2;  // one bf16 activation tile
  static constexpr int kX = kXT * (SPLIT ? 2 : 1);  // ring stage: the tile (+ its low-order term)
  // (split at NB = 256: 64 KB per stage next to the 128 KB partial → one stage)
  static constexpr int XST = NB <= 64 ? 4 : (SPLIT && NB > 128 ? 1 : 2);
  static constexpr int kPart = NB * BMW * 4;  // fp32 partial [NB][128], feature-contiguous
  // 227 KB opt-in minus the static LayerNorm scratch (2 x NB floats) and slack
  static constexpr int kSmemMax = 232448 - 2 * NB * 4 - 256;
  static constexpr int kFixed = XST * kX + 1024 /*align*/ + 1024 /*barriers*/;
  static constexpr int kWcap = (kSmemMax - kFixed) / kW;
  // split activations at NB <= 128: the hi and lo tiles are adjacent rows of one
  // N = 2 NB operand — ONE MMA per k16 step reads the weight tile once (two
  // N = NB MMAs read it twice: the smem-bandwidth-bound part of a decode MMA),
  // the epilogue adds the two accumulator halves
  static constexpr bool kComb = SPLIT && NB <= 128;
  static constexpr int kAccCols = kComb ? 2 * NB : NB;
  static constexpr int kTmemCols = kAccCols <= 32 ? 32 : (kAccCols <= 64 ? 64 : (kAccCols <= 128 ? 128 : 256));
  static int bytes(int wst) {
    const int body = wst * kW > kPart ? wst * kW : kPart;
    return body + XST * kX + 1024 + 1024;
  }
};

template <int NB, int EPI, int XM>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_decode_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                       const __grid_constant__ CUtensorMap tmX2, int Mrows,
                       int N, int K, void* __restrict__ Cv, int64_t ldc, int S, int wst, LnIn ln, RowStats so,
                       int push, uint64_t* dbg) {
  // debug timeline (PPOEXP_GEMM_TRACE): CTA (0, 0) stamps clock64 at each stage
  const bool trace = dbg != nullptr && blockIdx.x == 0 && blockIdx.y == 0;
  auto stamp = [&](int k) {
    if (trace) {
      dbg[k] = clock64();  // one CTA, one SM: cycle counts are comparable
    }
  };
  if (threadIdx.x == 0) stamp(0);
  constexpr bool LNIN = XMode<XM>::kLn, SPLIT = XMode<XM>::kSplit, PROD = XMode<XM>::kProduced;
  using L = DecLayout<NB, SPLIT>;
  constexpr int XST = L::XST;
  __shared__ float ln_mu[NB], ln_rs[NB];
  constexpr int kGB = LNIN ? 512 : 1;  // LN mode: gamma / beta of the first 8 k-blocks, staged before the PDL wait
  __shared__ float ln_g[kGB], ln_b[kGB];
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int body = wst * L::kW > L::kPart ? wst * L::kW : L::kPart;
  uint8_t* sW = smem;
  uint8_t* sX = smem + body;
  float* part = reinterpret_cast<float*>(smem);  // reused after the MMA loop
  // push mode (S > 1): a receive area for the peers' partial slices follows the X ring
  float* recv = reinterpret_cast<float*>(sX + XST * L::kX);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sX + XST * L::kX + (push ? L::kPart : 0));
  uint64_t* xfull = bars;
  uint64_t* xempty = xfull + XST;
  uint64_t* tmem_full = xempty + XST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  uint64_t* wfull = tmem_full + 2;   // [wst]
  uint64_t* wempty = wfull + wst;    // [wst]
  uint64_t* rfull = wempty + wst;    // push mode: peers' slices landed
  const int rows_per = S > 1 ? ((BMW / S) + 3) & ~3 : BMW;
  const uint32_t slice_bytes = uint32_t(NB) * rows_per * 4;
  cg::cluster_group cluster = cg::this_cluster();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BMW;
  const int r = blockIdx.y;  // K-split rank == cluster rank (cluster spans y)
  const int nk = (K + BK - 1) / BK;
  const int kb0 = int((int64_t(r) * nk) / S), kb1 = int((int64_t(r + 1) * nk) / S);
  const int nkl = kb1 - kb0;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < XST; ++i) {
      mbar_init(&xfull[i], PROD ? 128 : 1);  // LN / split modes: the 128 epilogue threads produce X
      mbar_init(&xempty[i], 1);
    }
    for (int i = 0; i < wst; ++i) {
      mbar_init(&wfull[i], 1);
      mbar_init(&wempty[i], 1);
    }
    mbar_init(tmem_full, 1);
    if (push) mbar_init(rfull, push == 2 ? 128 : 1);  // direct: one arrival per feature row of the slice
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (push == 1) mbar_expect_tx(rfull, uint32_t(S - 1) * slice_bytes);  // the single arrival + the peers' bytes
    // The weights are constant across the graph: fetch this CTA's weight slice
    // (up to the ring size) BEFORE waiting on the predecessor grid (PDL), so
    // the HBM stream overlaps the previous kernel.
    const int pre = min(wst, nkl);
    for (int it = 0; it < pre; ++it) {
      mbar_expect_tx(&wfull[it], L::kW);
      tma_load_2d(&tmW, &wfull[it], sW + it * L::kW, (kb0 + it) * BK, n0);
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(L::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // push mode: publish this CTA's initialised rfull to the cluster; the
  // matching wait happens just before the first remote push, long after
  if (push) asm volatile("barrier.cluster.arrive.aligned;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) stamp(1);
  if constexpr (LNIN) {
    if (threadIdx.x >= 64)  // LayerNorm parameters are not produced upstream
      for (int i = threadIdx.x - 64; i < min(nkl, kGB / BK) * BK; i += 128) {
        const int col = kb0 * BK + i;
        ln_g[i] = col < K ? ln.g[col] : 0.f;
        ln_b[i] = col < K ? ln.b[col] : 0.f;
      }
  }
  pdl_wait();  // upstream activations are valid from here on
  if (threadIdx.x == 0) stamp(2);
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      if (!PROD)
        for (int it = 0; it < nkl; ++it) {
          const int kb = kb0 + it;
          // activation tile (L2-resident, produced upstream)
          const int xs = it % XST, xu = it / XST;
          if (xu > 0) mbar_wait(&xempty[xs], (xu - 1) & 1);
          mbar_expect_tx(&xfull[xs], L::kX);
          tma_load_2d(&tmX, &xfull[xs], sX + xs * L::kX, kb * BK, 0);
          if constexpr (SPLIT) tma_load_2d(&tmX2, &xfull[xs], sX + xs * L::kX + L::kXT, kb * BK, 0);
        }
    } else if (lane == 1) {
      // refill the weight ring for slices larger than the ring
      for (int it = wst; it < nkl; ++it) {
        const int ws = it % wst, wu = it / wst;
        mbar_wait(&wempty[ws], (wu - 1) & 1);
        mbar_expect_tx(&wfull[ws], L::kW);
        tma_load_2d(&tmW, &wfull[ws], sW + ws * L::kW, (kb0 + it) * BK, n0);
      }
    }
    __syncwarp();  // reconverge before any block-wide barrier
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(BMW, L::kAccCols);
      for (int it = 0; it < nkl; ++it) {
        const int ws = it % wst, wu = it / wst;
        const int xs = it % XST, xu = it / XST;
        mbar_wait(&wfull[ws], wu & 1);
        mbar_wait(&xfull[xs], xu & 1);
        if (it == 0) stamp(3);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t dw = smem_desc_sw128(sW + ws * L::kW);
        const uint64_t dx = smem_desc_sw128(sX + xs * L::kX);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) mma_bf16(tmem, dw + 2 * k, dx + 2 * k, idesc, (it | k) != 0);
        if constexpr (SPLIT && !L::kComb) {  // the low-order activation term into the same accumulator
          const uint64_t dxl = smem_desc_sw128(sX + xs * L::kX + L::kXT);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) mma_bf16(tmem, dw + 2 * k, dxl + 2 * k, idesc, 1);
        }
        mma_commit(&xempty[xs]);
        mma_commit(&wempty[ws]);
      }
      mma_commit(tmem_full);
    }
    __syncwarp();
  } else {
    const int et = threadIdx.x - 64;  // 0..127
    if constexpr (PROD) {
      // ---- fused LayerNorm producer: every independent load first (the row
      // statistics and the x chunks of the first PF k-blocks), then row mean /
      // rstd, then LN(x) -> bf16 in the 128B-swizzled K-major layout UMMA reads.
      // Thread et owns chunks et + 128 c (c < CPT) of every k-block: always the
      // same 8-column group c8.
      constexpr int CPT = NB * 8 / 128;
      constexpr int PF = CPT >= 8 ? 1 : (CPT >= 4 ? 3 : 4);
      const int c8 = et & 7;
      unsigned long long sa[2][2] = {{0ull, 0ull}, {0ull, 0ull}};
      if constexpr (LNIN) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int rr = et + u * 128;
          if (rr < NB && rr < Mrows) {
            sa[u][0] = __ldcg(ln.acc + rr * kStatStride);
            sa[u][1] = __ldcg(ln.acc + rr * kStatStride + 1);
          }
        }
      }
      auto load_kb = [&](int it, float4 (&xa)[CPT][2]) {
        const int col = (kb0 + it) * BK + c8 * 8;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const int rr = (et + c * 128) >> 3;
          if (col < K && rr < Mrows) {
            const float4* xr = reinterpret_cast<const float4*>(ln.x + int64_t(rr) * ln.ldx + col);
            xa[c][0] = __ldcg(xr);
            xa[c][1] = __ldcg(xr + 1);
          } else {
            xa[c][0] = xa[c][1] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      };
      float4 xpf[PF][CPT][2];
#pragma unroll
      for (int p = 0; p < PF; ++p)
        if (p < nkl) load_kb(p, xpf[p]);
      if constexpr (LNIN) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int rr = et + u * 128;
          if (rr < NB) {
            float mu = 0.f, rs = 0.f;
            if (rr < Mrows) {
              const double inv_d = 1.0 / ln.d;
              const double mean = stat_of(sa[u][0]) * inv_d;
              const double var = fmax(stat_of(sa[u][1]) * inv_d - mean * mean, 0.0);
              mu = float(mean);
              // split mode keeps fp32-grade statistics (1 / sqrt in fp64)
              rs = SPLIT ? float(1.0 / sqrt(var + 1e-5)) : rsqrtf(float(var) + 1e-5f);
            }
            ln_mu[rr] = mu;
            ln_rs[rr] = rs;
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");  // mu / rstd and the staged gamma / beta
      }
      auto emit_kb = [&](int it, const float4 (&xa)[CPT][2]) {
        const int xs = it % XST, xu = it / XST;
        const int col = (kb0 + it) * BK + c8 * 8;
        float gv[8], bv[8];
        if constexpr (!LNIN) {
        } else if (it < kGB / BK) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            gv[e] = ln_g[it * BK + c8 * 8 + e];
            bv[e] = ln_b[it * BK + c8 * 8 + e];
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            gv[e] = col + e < K ? __ldg(ln.g + col + e) : 0.f;
            bv[e] = col + e < K ? __ldg(ln.b + col + e) : 0.f;
          }
        }
        if (xu > 0) mbar_wait(&xempty[xs], (xu - 1) & 1);
        uint8_t* tile = sX + xs * L::kX;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const int rr = (et + c * 128) >> 3;
          Vec16<bf16> o, ol;
          if (col < K && rr < Mrows) {
            const float xv[8] = {xa[c][0].x, xa[c][0].y, xa[c][0].z, xa[c][0].w,
                                 xa[c][1].x, xa[c][1].y, xa[c][1].z, xa[c][1].w};
            float yv[8];
            if constexpr (LNIN) {
              const float mu = ln_mu[rr], rs = ln_rs[rr];
#pragma unroll
              for (int e = 0; e < 8; ++e) yv[e] = gv[e] * ((xv[e] - mu) * rs) + bv[e];
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) yv[e] = xv[e];
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              o.v[e] = __float2bfloat16_rn(yv[e]);
              if constexpr (SPLIT) ol.v[e] = __float2bfloat16_rn(yv[e] - __bfloat162float(o.v[e]));
            }
          } else {
            o.u = make_uint4(0u, 0u, 0u, 0u);
            ol.u = o.u;
          }
          *reinterpret_cast<uint4*>(tile + rr * 128 + ((c8 ^ (rr & 7)) << 4)) = o.u;
          if constexpr (SPLIT) *reinterpret_cast<uint4*>(tile + L::kXT + rr * 128 + ((c8 ^ (rr & 7)) << 4)) = ol.u;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&xfull[xs])) : "memory");
      };
#pragma unroll
      for (int p = 0; p < PF; ++p)
        if (p < nkl) emit_kb(p, xpf[p]);
      for (int it = PF; it < nkl; ++it) {
        float4 xa[CPT][2];
        load_kb(it, xa);
        emit_kb(it, xa);
      }
    }
    // TMEM (feature rows x batch cols) → registers → (S == 1) epilogue straight
    // to global, or (S > 1) fp32 partial in smem for the cluster reduction
    const int q = warp & 3;
    mbar_wait(tmem_full, 0);
    if (threadIdx.x == 64) stamp(4);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int f = q * 32 + lane;
    const int n = n0 + f;
    const int ncols = min(Mrows, NB);
    // direct push (push == 2): this thread's feature row goes straight from
    // registers into the owner rank's receive area, [sender][bcol][f % rows_per]
    uint32_t rdst = 0;
    if (S > 1 && push == 2) {
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // every rank's rfull is initialised
      const uint32_t loc = smem_u32(recv) + uint32_t((r * NB * rows_per + (f % rows_per)) * 4);
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(loc), "r"(f / rows_per));
    }
#pragma unroll 1
    for (int c = 0; c < NB; c += 16) {
      uint32_t v[16];
      tmem_ld16(tmem + (uint32_t(q * 32) << 16) + uint32_t(c), v);
      if constexpr (L::kComb) {  // + the lo-term half of the accumulator
        uint32_t vl[16];
        tmem_ld16(tmem + (uint32_t(q * 32) << 16) + uint32_t(NB + c), vl);
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) + __uint_as_float(vl[e]));
      }
      if (S > 1 && push == 2) {
#pragma unroll
        for (int e = 0; e < 16; ++e)
          asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(rdst + uint32_t((c + e) * rows_per * 4)), "r"(v[e])
                       : "memory");
      } else if (S > 1 && push) {
        // slice-major [k][bcol][f % rows_per]: the slice for rank k is one
        // contiguous block, pushed with a single bulk copy
        float* ps = part + (f / rows_per) * (NB * rows_per) + (f % rows_per);
#pragma unroll
        for (int e = 0; e < 16; ++e) ps[(c + e) * rows_per] = __uint_as_float(v[e]);
      } else if (S > 1) {
#pragma unroll
        for (int e = 0; e < 16; ++e) part[(c + e) * BMW + f] = __uint_as_float(v[e]);
      } else if (n < N) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int bcol = c + e;
          if (bcol >= ncols) break;
          const float a = __uint_as_float(v[e]);
          const int64_t o = int64_t(bcol) * ldc + n;
          if constexpr (EPI == int(Epi::kStore)) {
            static_cast<bf16*>(Cv)[o] = __float2bfloat16_rn(a);
          } else if constexpr (EPI == int(Epi::kGelu)) {
            static_cast<bf16*>(Cv)[o] = __float2bfloat16_rn(gelu_fast(a));
          } else if constexpr (EPI == int(Epi::kAddResidual)) {
            static_cast<float*>(Cv)[o] += a;
          } else if constexpr (EPI == int(Epi::kGeluF32)) {
            static_cast<float*>(Cv)[o] = gelu_fast(a);
          } else if constexpr (EPI == int(Epi::kGeluSplit)) {
            const float gv = gelu_fast(a);
            const bf16 hi = __float2bfloat16_rn(gv);
            static_cast<bf16*>(Cv)[o] = hi;
            static_cast<bf16*>(Cv)[o + N] = __float2bfloat16_rn(gv - __bfloat162float(hi));
          } else {
            static_cast<float*>(Cv)[o] = a;
          }
        }
      }
      if (EPI == int(Epi::kAddResidual) && S == 1 && so.acc) {
        // per-row partial statistics of the updated residual over this tile's
        // 128 features: warp reduce, 4 warp partials parked in smem (sX is free)
        float* wred = reinterpret_cast<float*>(sX);  // [4][NB][2]
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int bcol = c + e;
          float xv = 0.f;
          if (n < N && bcol < ncols) xv = static_cast<const float*>(Cv)[int64_t(bcol) * ldc + n];
          const float s1 = warp_sum(xv), s2 = warp_sum(xv * xv);
          if (lane == 0) {
            wred[(q * NB + bcol) * 2] = s1;
            wred[(q * NB + bcol) * 2 + 1] = s2;
          }
        }
      }
    }
    if (S > 1 && push == 2) {  // release this row's stores to the owner rank
      uint32_t rbar;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(rfull)), "r"(f / rows_per));
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
    }
    if (EPI == int(Epi::kAddResidual) && S == 1 && so.acc) {
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const float* wred = reinterpret_cast<const float*>(sX);
      for (int bcol = threadIdx.x - 64; bcol < ncols; bcol += 128) {
        double s1 = 0.0, s2 = 0.0;
        for (int w4 = 0; w4 < 4; ++w4) {
          s1 += wred[(w4 * NB + bcol) * 2];
          s2 += wred[(w4 * NB + bcol) * 2 + 1];
        }
        atomicAdd(&so.acc[bcol * kStatStride], stat_fix(s1, so.ovf));
        atomicAdd(&so.acc[bcol * kStatStride + 1], stat_fix(s2, so.ovf));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (S > 1) {
    // reduce feature rows [f0, f1) of this CTA over the S partials, in rank
    // order.  push: every CTA bulk-copies slice k of its partial into rank k's
    // receive area (TMA engine, completion on rank k's rfull), then reduces
    // from local smem.  pull (fallback when smem is short): cluster barrier,
    // then float4 DSMEM loads from every peer.
    const int f0 = r * rows_per, f1 = min(BMW, f0 + rows_per);
    const int nf4 = (f1 - f0) / 4;
    const int ncols = min(Mrows, NB);
    float4 xpre[4];
    if (push == 2) {
      if constexpr (EPI == int(Epi::kAddResidual)) {
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int e = threadIdx.x + it * kThreads;
          xpre[it] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (e < nf4 * ncols) {
            const int fl = f0 + 4 * (e % nf4), bcol = e / nf4;
            const int64_t o = int64_t(bcol) * ldc + n0 + fl;
            if (n0 + fl + 3 < N && (o & 3) == 0) xpre[it] = __ldcg(reinterpret_cast<const float4*>(static_cast<float*>(Cv) + o));
          }
        }
      }
      if (threadIdx.x == 0) stamp(5);
      asm volatile(  // acquire the peers' releases (cluster scope)
          "{\n .reg .pred p;\n WAITC_%=:\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], 0;\n @!p bra WAITC_%=;\n}" ::"r"(
              smem_u32(rfull))
          : "memory");
      if (threadIdx.x == 0) stamp(6);
    } else if (push) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // parked partial -> bulk-copy reads
      if (threadIdx.x == 64) stamp(9);
      __syncthreads();
      if (threadIdx.x == 0) stamp(10);
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // every peer's rfull is initialised
      if (threadIdx.x == 0) stamp(11);
      if (threadIdx.x == 0) {
        for (int k = 0; k < S; ++k) {
          if (k == r) continue;
          uint32_t dst, bar;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(smem_u32(recv) + r * slice_bytes), "r"(k));
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(bar) : "r"(smem_u32(rfull)), "r"(k));
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
              "r"(smem_u32(part) + k * slice_bytes), "r"(slice_bytes), "r"(bar)
              : "memory");
        }
      }
      // residual epilogue: the x values this thread updates are loaded while
      // the peers' slices are in flight (after the proxy fence, which would
      // otherwise wait for these loads)
      if constexpr (EPI == int(Epi::kAddResidual)) {
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int e = threadIdx.x + it * kThreads;
          xpre[it] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (e < nf4 * ncols) {
            const int fl = f0 + 4 * (e % nf4), bcol = e / nf4;
            const int64_t o = int64_t(bcol) * ldc + n0 + fl;
            if (n0 + fl + 3 < N && (o & 3) == 0) xpre[it] = __ldcg(reinterpret_cast<const float4*>(static_cast<float*>(Cv) + o));
          }
        }
      }
      if (threadIdx.x == 0) stamp(5);
      mbar_wait(rfull, 0);
      if (threadIdx.x == 0) stamp(6);

    } else {
      if constexpr (EPI == int(Epi::kAddResidual)) {
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int e = threadIdx.x + it * kThreads;
          xpre[it] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (e < nf4 * ncols) {
            const int fl = f0 + 4 * (e % nf4), bcol = e / nf4;
            const int64_t o = int64_t(bcol) * ldc + n0 + fl;
            if (n0 + fl + 3 < N && (o & 3) == 0) xpre[it] = __ldcg(reinterpret_cast<const float4*>(static_cast<float*>(Cv) + o));
          }
        }
      }
      cluster.sync();  // all partials of the cluster are parked in smem

    }
    int it = 0;
    // rank k's partial: push -> own slice (k == r) or the receive area; pull -> DSMEM of rank k
    auto part_of = [&](int k) -> const float4* {
      if (push == 2) return reinterpret_cast<const float4*>(recv + size_t(k) * NB * rows_per);
      if (push)
        return reinterpret_cast<const float4*>(k == r ? part + size_t(r) * NB * rows_per
                                                      : recv + size_t(k) * NB * rows_per);
      return reinterpret_cast<const float4*>(cluster.map_shared_rank(part, k));
    };
    for (int e = threadIdx.x; e < nf4 * ncols; e += kThreads, ++it) {
      const int fl = f0 + 4 * (e % nf4), bcol = e / nf4;
      const int idx = push ? ((bcol * rows_per + (fl - f0)) >> 2) : ((bcol * BMW + fl) >> 2);
      // rank order, 8 partials in flight at a time
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int k0 = 0; k0 < S; k0 += 8) {
        float4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k0 + k < S) v[k] = part_of(k0 + k)[idx];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k0 + k < S) {
            if (k0 + k == 0) {
              acc = v[0];
            } else {
              acc.x += v[k].x;
              acc.y += v[k].y;
              acc.z += v[k].z;
              acc.w += v[k].w;
            }
          }
      }
      const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
      double ps = 0.0, pq = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int nn = n0 + fl + j;
        if (nn >= N) break;
        const float a = a4[j];
        const int64_t o = int64_t(bcol) * ldc + nn;
        if constexpr (EPI == int(Epi::kStore)) {
          static_cast<bf16*>(Cv)[o] = __float2bfloat16_rn(a);
        } else if constexpr (EPI == int(Epi::kGelu)) {
          static_cast<bf16*>(Cv)[o] = __float2bfloat16_rn(gelu_fast(a));
        } else if constexpr (EPI == int(Epi::kAddResidual)) {
          float* xp = static_cast<float*>(Cv) + o;
          const int64_t o4 = int64_t(bcol) * ldc + n0 + fl;
          const bool pre = it < 4 && n0 + fl + 3 < N && (o4 & 3) == 0;
          const float xo = pre ? (j == 0 ? xpre[it & 3].x : j == 1 ? xpre[it & 3].y : j == 2 ? xpre[it & 3].z : xpre[it & 3].w)
                               : *xp;
          const float nv = xo + a;
          *xp = nv;
          ps += double(nv);
          pq += double(nv) * double(nv);
        } else if constexpr (EPI == int(Epi::kGeluF32)) {
          static_cast<float*>(Cv)[o] = gelu_fast(a);
        } else if constexpr (EPI == int(Epi::kGeluSplit)) {
          const float gv = gelu_fast(a);
          const bf16 hi = __float2bfloat16_rn(gv);
          static_cast<bf16*>(Cv)[o] = hi;
          static_cast<bf16*>(Cv)[o + N] = __float2bfloat16_rn(gv - __bfloat162float(hi));
        } else {
          static_cast<float*>(Cv)[o] = a;
        }
      }
      if (EPI == int(Epi::kAddResidual) && so.acc) {
        double2* red = reinterpret_cast<double2*>(sX);  // [ncols][nf4], the X ring is idle now
        red[bcol * nf4 + (e % nf4)] = make_double2(ps, pq);
      }
    }
    if (EPI == int(Epi::kAddResidual) && so.acc) {
      __syncthreads();
      const double2* red = reinterpret_cast<const double2*>(sX);
      for (int bcol = threadIdx.x; bcol < ncols; bcol += kThreads) {
        double s1 = 0.0, s2 = 0.0;
        for (int g4 = 0; g4 < nf4; ++g4) {
          s1 += red[bcol * nf4 + g4].x;
          s2 += red[bcol * nf4 + g4].y;
        }
        atomicAdd(&so.acc[bcol * kStatStride], stat_fix(s1, so.ovf));
        atomicAdd(&so.acc[bcol * kStatStride + 1], stat_fix(s2, so.ovf));
      }
    }
    if (push == 2) {
      // nothing reads this CTA's shared memory remotely, and every rank waits for all
      // stores into its own receive area before it exits: no exit barrier
    } else if (push) {  // every peer's incoming copies (including ours) have landed before anyone exits
      if (threadIdx.x == 0) stamp(7);
      asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
      if (threadIdx.x == 0) stamp(8);
    } else {
      cluster.sync();  // keep our smem alive until every peer has read it
    }
  } else {
    __syncthreads();
  }
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L::kTmemCols));
  }
}

template <int NB, int EPI, int XM>
void launch_dec(Ctx& c, const bf16* X, int64_t ldx, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
               void* C, int64_t ldc, const LnIn* ln, const RowStats* so) {
  constexpr bool LNIN = XMode<XM>::kLn;
  using L = DecLayout<NB, XMode<XM>::kSplit>;
  const CUtensorMap tw = make_map(W, N, K, ldw, BMW);
  // produced-X modes never read X through TMA; any valid map will do.  Planes
  // (XM 4): hi = X[:, 0:K), lo = X[:, K:2K) with row stride ldx (= 2K)
  const CUtensorMap tx = XMode<XM>::kProduced ? tw : make_map(X, M, K, ldx, NB);
  const CUtensorMap tx2 = XM == 4 ? make_map(X + K, M, K, ldx, NB) : tx;
  auto k = gemm_decode_kernel<NB, EPI, XM>;
  const int smem_max = L::kSmemMax - (LNIN ? 2 * 512 * 4 : 0);  // LN mode: static gamma / beta staging
  static bool attr = false;
  if (!attr) {
    PPOEXP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
    PPOEXP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  const int tiles = int(ceil_div(N, BMW));
  const int nk = int(ceil_div(K, BK));
  // K-split over a cluster: enough CTAs to stream the weights in parallel
  // (~148 target, <= 4 ranks: measured best on B200), >= 2 k-blocks each, and
  // always enough that a CTA's slice fits the smem weight ring.
  static const int smax = [] {
    const char* e = getenv("PPOEXP_DECODE_SPLIT_MAX");
    return e ? atoi(e) : 4;
  }();
  static const int smax_small = [] {  // narrow outputs (N <= 1024: O / down projections)
    const char* e = getenv("PPOEXP_DECODE_SPLIT_SMALLN");
    return std::min(e ? atoi(e) : 8, kMaxS);  // 8: measured best with the direct push exchange
  }();
  const int cap = tiles <= 8 ? smax_small : smax;
  int S = 1;
  static const int fit_env = [] {  // 1: double only while the doubled grid still fits one wave
    const char* e = getenv("PPOEXP_DECODE_SPLIT_FIT");
    return e ? atoi(e) : -1;
  }();
  // auto: the one-wave rule for wide batches (each CTA re-reads a 256-row
  // activation: measured best at config 3, batch 256) and for the mixed-mode
  // planes (twice the activation bytes per k-block: config 4 mixed 5.0k -> 5.5k
  // tok/s); bf16 small batches keep doubling while the grid is under one CTA
  // per SM — more weight streams in flight (config 4 bf16, batch 64: 6.4k ->
  // 7.5k tok/s; config 2 picks the same S either way)
  const bool fit = fit_env >= 0 ? fit_env != 0 : (NB > 64 || XM == 4);
  while (S < cap && (fit ? tiles * S * 2 <= 148 : tiles * S < 148) && nk >= 2 * S) S *= 2;
  // a slice larger than the weight ring cycles it (warp 0 lane 1 refills); only
  // split further for that while the launch stays one wave (1 CTA/SM at batch > 64)
  static const int onewave = [] {
    const char* e = getenv("PPOEXP_DECODE_ONEWAVE");
    return e ? atoi(e) : 1;
  }();
  while (S < kMaxS && ceil_div(nk, S) > L::kWcap && (!onewave || tiles * S * 2 <= 148)) S *= 2;
  static const int wring = [] {
    const char* e = getenv("PPOEXP_DECODE_WRING");
    return e ? atoi(e) : 8;
  }();
  // K-split launches hold their whole slice (one wave, the ring is filled
  // before the PDL wait); multi-wave launches (tiles > #SMs, e.g. the LM
  // head) keep a 2-deep ring so three CTAs share an SM
  static const int wring_wide = [] {
    const char* e = getenv("PPOEXP_DECODE_WRING_WIDE");  // 2: three CTAs per SM (the LM head fits one wave)
    return e ? atoi(e) : 2;
  }();
  const int ring = tiles * S > 148 ? std::min(wring, wring_wide) : wring;
  const int wst = int(std::min<int64_t>(std::min<int64_t>(L::kWcap, ring), ceil_div(nk, S)));
  static const int push_env = [] {
    // 2 = direct register -> remote-smem stores (default), 1 = park + bulk copy, 0 = pull
    const char* e = getenv("PPOEXP_DECODE_PUSH");
    return e ? atoi(e) : 2;
  }();
  const int push = (push_env && S > 1 && L::bytes(wst) + wst * 16 + L::kPart <= smem_max) ? push_env : 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(tiles, S, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = L::bytes(wst) + wst * 16 + (push ? L::kPart : 0);
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
  const LnIn lnv = ln ? *ln : LnIn{};
  const RowStats sov = (so && EPI == int(Epi::kAddResidual)) ? *so : RowStats{};
  const double flops = 2.0 * M * N * K;
  const double bytes = 2.0 * N * K + double(M) * K * (XM ? 4 : 2) + double(M) * N * ((EPI == 0 || EPI == 1) ? 2 : 4);
  c.launch("gemm_decode", bytes, flops, [&] {
    uint64_t* dbg = nullptr;
    static const bool gtrace = getenv("PPOEXP_GEMM_TRACE") != nullptr;
    if (gtrace) {  // debug: slot per launch (graph nodes keep their slot)
      auto* buf = static_cast<uint64_t*>(c.workspace("gemm_decode.trace", size_t(4096) * 16 * 8));
      const int64_t slot = int64_t(c.gemm_trace_meta.size()) % 4096;
      c.gemm_trace_meta.push_back({int(N), int(K), EPI, S});
      dbg = buf + slot * 16;
    }
    const cudaError_t e =
        cudaLaunchKernelEx(&cfg, k, tw, tx, tx2, int(M), int(N), int(K), C, ldc, S, wst, lnv, sov, push, dbg);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      throw Error(6, std::string("cuda: decode GEMM launch failed (") + cudaGetErrorString(e) + ") NB=" +
                         std::to_string(NB) + " EPI=" + std::to_string(EPI) + " XM=" + std::to_string(XM) +
                         " M=" + std::to_string(M) + " N=" + std::to_string(N) + " K=" + std::to_string(K) +
                         " S=" + std::to_string(S) + " wst=" + std::to_string(wst) + " smem=" +
                         std::to_string(cfg.dynamicSmemBytes) + " max=" + std::to_string(smem_max));
    }
  });
}

template <int NB, int XM>
void dispatch(Ctx& c, const bf16* X, int64_t ldx, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K, Epi epi,
             void* C, int64_t ldc, const LnIn* ln, const RowStats* so) {
  if constexpr (XMode<XM>::kSplit) {  // mixed mode: fp32 outputs only
    switch (epi) {
      case Epi::kAddResidual: return launch_dec<NB, 2, XM>(c, X, ldx, W, ldw, M, N, K, C, ldc, ln, so);
      case Epi::kStoreF32: return launch_dec<NB, 3, XM>(c, X, ldx, W, ldw, M, N, K, C, ldc, ln, so);
      case Epi::kGeluF32: return launch_dec<NB, 5, XM>(c, X, ldx, W, ldw, M, N, K, C, ldc, ln, so);
      case Epi::kGeluSplit: return launch_dec<NB, 6, XM>(c, X, ldx, W, ldw, M, N, K, C, ldc, ln, so);
      default: throw ContractError("decode GEMM: split activations need an fp32 epilogue");
    }
  } else {
    switch (epi) {
      case Epi::kStore: return launch_dec<NB, 0, XM>(c, X, ldx, W, ldw, M, N, K, C, ldc, ln, so);
      case Epi::kGelu: return launch_dec<NB, 1, XM>(c, X, ldx, W, ldw, M, N, K, C, ldc, ln, so);
      case Epi::kAddResidual: return launch_dec<NB, 2, XM>(c, X, ldx, W, ldw, M, N, K, C, ldc, ln, so);
      case Epi::kStoreF32: return launch_dec<NB, 3, XM>(c, X, ldx, W, ldw, M, N, K, C, ldc, ln, so);
      default: throw ContractError("decode GEMM: unsupported epilogue");
    }
  }
}

template <int XM>
void dispatch_nb(Ctx& c, const bf16* X, int64_t ldx, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
                Epi epi, void* C, int64_t ldc, const LnIn* ln, const RowStats* so) {
  if (M <= 32) return dispatch<32, XM>(c, X, ldx, W, ldw, M, N, K, epi, C, ldc, ln, so);
  if (M <= 64) return dispatch<64, XM>(c, X, ldx, W, ldw, M, N, K, epi, C, ldc, ln, so);
  if (M <= 128) return dispatch<128, XM>(c, X, ldx, W, ldw, M, N, K, epi, C, ldc, ln, so);
  return dispatch<256, XM>(c, X, ldx, W, ldw, M, N, K, epi, C, ldc, ln, so);
}

}  // namespace

// Debug (PPOEXP_GEMM_TRACE): write the per-launch stage stamps + {N, K, epi, S}
// of every traced decode-GEMM launch to `path` (binary: n, meta[n][4] int32,
// stamps[n][16] u64).
void dump_gemm_trace(Ctx& c, const char* path) {
  const int64_t n = std::min<int64_t>(int64_t(c.gemm_trace_meta.size()), 4096);
  if (n == 0) return;
  std::vector<uint64_t> h(size_t(n) * 16);
  PPOEXP_CUDA(cudaMemcpy(h.data(), c.workspace("gemm_decode.trace", size_t(4096) * 16 * 8), h.size() * 8,
                         cudaMemcpyDeviceToHost));
  if (FILE* fp = fopen(path, "wb")) {
    const int32_t nn = int32_t(n);
    fwrite(&nn, 4, 1, fp);
    for (int64_t i = 0; i < n; ++i) fwrite(c.gemm_trace_meta[i].data(), 4, 4, fp);
    fwrite(h.data(), 8, h.size(), fp);
    fclose(fp);
  }
}

// Decode-sized GEMM (M <= 256).  Returns false if not eligible.
bool gemm_decode_bf16(Ctx& c, const bf16* A, int64_t lda, const bf16* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                      Epi epi, void* C, int64_t ldc) {
  if (M > 256 || M <= 0) return false;
  dispatch_nb<0>(c, A, lda, B, ldb, M, N, K, epi, C, ldc, nullptr, nullptr);
  return true;
}

void gemm_decode_fused(Ctx& c, const bf16* X, int64_t ldx, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
                      Epi epi, void* C, int64_t ldc, const LnIn* ln, const RowStats* so) {
  if (M > 256 || M <= 0) throw ContractError("decode GEMM: batch above 256");
  if (ln) {
    if (K % 8 || ln->d != K) throw ContractError("decode GEMM: fused LayerNorm needs K == d_model, K % 8 == 0");
    return dispatch_nb<1>(c, X, ldx, W, ldw, M, N, K, epi, C, ldc, ln, so);
  }
  return dispatch_nb<0>(c, X, ldx, W, ldw, M, N, K, epi, C, ldc, ln, so);
}

// Mixed mode, activation as two bf16 planes [M, 2K] (hi | lo) from the producer
// kernel (split LayerNorm / attention / GELU epilogue): both TMA'd, two MMAs.
void gemm_decode_planes(Ctx& c, const bf16* X, int64_t ldx, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
                        Epi epi, void* C, int64_t ldc, const RowStats* so) {
  if (M > 256 || M <= 0) throw ContractError("decode GEMM: batch above 256");
  if (K % 8 || ldx % 8 || ldx < 2 * K) throw ContractError("decode GEMM (planes): K % 8 and a [M, 2K] operand required");
  return dispatch_nb<4>(c, X, ldx, W, ldw, M, N, K, epi, C, ldc, nullptr, so);
}

// Mixed mode (bf16 weights, fp32 activations): the fp32 activation (or the
// LayerNorm of x when ln != null) is split into two bf16 terms in-kernel.
void gemm_decode_mixed(Ctx& c, const float* X, int64_t ldx, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
                       Epi epi, void* C, int64_t ldc, const LnIn* ln, const RowStats* so) {
  if (M > 256 || M <= 0) throw ContractError("decode GEMM: batch above 256");
  if (K % 8 || ldx % 4) throw ContractError("decode GEMM (mixed): K and the activation stride must be multiples of 8 / 4");
  if (ln) {
    if (ln->d != K) throw ContractError("decode GEMM: fused LayerNorm needs K == d_model");
    return dispatch_nb<3>(c, nullptr, 0, W, ldw, M, N, K, epi, C, ldc, ln, so);
  }
  const LnIn xin{X, ldx, nullptr, nullptr, nullptr, int(K)};
  return dispatch_nb<2>(c, nullptr, 0, W, ldw, M, N, K, epi, C, ldc, &xin, so);
}

}  // namespace ppx
