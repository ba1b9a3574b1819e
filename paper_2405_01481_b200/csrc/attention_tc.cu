// attention_tc.cu — K5a on the 5th-generation tensor cores: causal flash
// attention over packed ragged sequences (bf16 scoring / critic / RM forwards
// and the engine's batched prefill; src/model.cpp:230-236 semantics: scores
// scaled by 1/sqrt(dh) before the max, causal, exp(s - max) / sum).
//
// CTA = QT tiles of 128 queries of one (sequence, head), 2 + 4 QT warps:
//   warp 0    : TMA producer — the Q tile(s) once, then K / V tiles of 64 keys
//               (128B-swizzled boxes of the packed qkv buffer) into a 2-3-stage ring;
//   warp 1    : TMEM allocator + MMA issuer — S_j = Q K_j^T into one of two TMEM
//               score buffers (issued one tile ahead), O += P_j V_j into the TMEM
//               output accumulator (V is the MN-major B operand, straight from TMA);
//   warps 2-5 (+ 6-9 for the second Q tile) : softmax — thread r owns query row r
//               (TMEM lane r of its tile's columns): tcgen05.ld of
//               the score row, mask, online max / sum in the log2 domain, the
//               O-row rescale in TMEM when the max moves, P_j (bf16) written in
//               the UMMA K-major swizzle; epilogue O / l -> global.
#include <cuda.h>

#include <cfloat>

#include "kernels.hpp"

namespace ppx {

CUtensorMap make_map(const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);  // gemm_tc.cu

namespace {

constexpr int BQ = 128, BKV = 64;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\nWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}" ::"r"(
          su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma2d(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// K-major, 128B swizzle, 8-row atoms 1024 B apart
__device__ __forceinline__ uint64_t desc_k(const void* p) {
  const uint64_t a = su32(p);
  return ((a >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// MN-major, 128B swizzle: 8 K-rows x 128 B atoms, 1024 B apart along K; the next
// 64 N-elements (the next TMA box of 64 rows x 128 B) 8192 B further (pinned by
// tools/umma_probe.py / umma_probe.cu)
__device__ __forceinline__ uint64_t desc_mn(const void* p) {
  const uint64_t a = su32(p);
  return ((a >> 4) & 0x3FFFull) | ((8192ull >> 4) << 16) | ((1024ull >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
constexpr uint32_t idesc(int M, int N, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (b_mn ? (1u << 16) : 0u) | (uint32_t(N >> 3) << 17) |
         (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void tld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tst32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// SPLIT (mixed mode): q / k / v arrive as bf16 hi | lo planes of the packed
// [M, 3d] projection (hi in columns [0, 3d), lo in [3d, 6d)); every operand
// tile is held as both terms and each product is issued as three MMAs
// (hi·hi + hi·lo + lo·hi, fp32-grade), P split the same way; the output is
// written as hi | lo planes [M, 2d] for the O projection.
template <int DH, bool SPLIT, int QT>
struct FaSmem {
  static constexpr int kT = SPLIT ? 2 : 1;
  static constexpr int kQ1 = BQ * DH * 2;     // one Q term: DH/64 boxes of 128 rows x 128 B
  static constexpr int kQ = kQ1 * kT;         // one Q tile (both terms)
  static constexpr int kKV1 = BKV * DH * 2;   // one term of a K (or V) tile: DH/64 boxes of 64 rows x 128 B
  static constexpr int kKV = kKV1 * kT;
  static constexpr int kP1 = BQ * BKV * 2;    // one term of the P tile: 128 rows x 128 B
  static constexpr int kP = kP1 * kT;
  // the P tile of step j is written only after P_{j-1} V_{j-1} completed (the
  // softmax waits for it before the O rescale), so one P buffer suffices; the
  // split head_dim-128 tiles use it (and a 2-stage K / V ring) to fit 227 KB,
  // and so do two Q tiles per CTA
  static constexpr bool kBig = SPLIT && DH == 128;
  static constexpr int kNst = kBig ? 2 : 3;
  static constexpr int kPB = (kBig || QT == 2) ? 1 : 2;
  static constexpr int kBytes = QT * kQ + kNst * 2 * kKV + QT * kPB * kP + 1024 /*align*/ + 512 /*barriers*/;
  static constexpr int kTmem = 256 * QT;      // per Q tile: S0 (64) | S1 (64) | O (DH <= 128)
  static constexpr int kThreads = 64 + 128 * QT;
};

// QT = 2: two 128-query tiles of the same (sequence, head) share each K / V
// tile, with one softmax warpgroup per Q tile: while one group computes its
// exponentials the tensor core runs the other group's S = Q K^T / O += P V,
// and the SMs' schedulers have two softmax warps each to interleave.
template <int DH, bool SPLIT, int QT>
__global__ void __launch_bounds__(FaSmem<DH, SPLIT, QT>::kThreads, 1)
    attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tkv,
                           const int64_t* __restrict__ seq_offsets, int H, bf16* __restrict__ out) {
  using L = FaSmem<DH, SPLIT, QT>;
  constexpr int NB = DH / 64;  // 64-column boxes per row
  constexpr int NST = L::kNst, PB = L::kPB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto sQ = [&](int g) { return sm + g * L::kQ; };
  auto sK = [&](int s) { return sm + QT * L::kQ + s * 2 * L::kKV; };
  auto sV = [&](int s) { return sm + QT * L::kQ + s * 2 * L::kKV + L::kKV; };
  auto sP = [&](int g, int bb) { return sm + QT * L::kQ + NST * 2 * L::kKV + (g * PB + bb) * L::kP; };
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + QT * L::kQ + NST * 2 * L::kKV + QT * PB * L::kP);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;         // [NST]
  uint64_t* kv_empty = kv_full + NST;   // [NST]
  // per Q tile g: s_full[2] | s_free[2] | p_full[2] | o_done
  auto s_full = [&](int g) { return kv_empty + NST + g * 8; };
  auto s_free = [&](int g) { return kv_empty + NST + g * 8 + 2; };
  auto p_full = [&](int g) { return kv_empty + NST + g * 8 + 4; };
  auto o_done = [&](int g) { return kv_empty + NST + g * 8 + 6; };
  uint32_t* tslot = reinterpret_cast<uint32_t*>(kv_empty + NST + QT * 8);

  PDL_ENTRY();
  const int64_t b = blockIdx.z;
  const int h = blockIdx.y;
  const int64_t q0 = int64_t(blockIdx.x) * BQ * QT;
  const int64_t start = seq_offsets[b], len = seq_offsets[b + 1] - start;
  if (q0 >= len) return;
  const int64_t d = int64_t(H) * DH;
  const int ntile = (QT == 2 && q0 + BQ < len) ? 2 : 1;  // Q tiles holding queries of this sequence
  // K / V tiles each Q tile needs (causal): keys < min(len, q0 + (g + 1) BQ)
  auto nt_of = [&](int g) { return int((min(len, q0 + int64_t(g + 1) * BQ) + BKV - 1) / BKV); };
  const int nt_all = nt_of(ntile - 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    bar_init(q_full, 1);
    for (int s = 0; s < NST; ++s) {
      bar_init(&kv_full[s], 1);
      bar_init(&kv_empty[s], 1);
    }
    for (int g = 0; g < QT; ++g) {
      for (int i = 0; i < 2; ++i) {
        bar_init(&s_full(g)[i], 1);
        bar_init(&s_free(g)[i], 128);
        bar_init(&p_full(g)[i], 128);
      }
      bar_init(o_done(g), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tq)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tkv)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "r"(L::kTmem));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  auto tS = [&](int g) { return tmem + uint32_t(g * 256); };
  auto tO = [&](int g) { return tmem + uint32_t(g * 256 + 128); };

  if (warp == 0) {
    if (lane == 0) {
      bar_expect(q_full, ntile * L::kQ);
      for (int g = 0; g < ntile; ++g)
        for (int c = 0; c < NB; ++c) {
          const int row = int(start + q0 + g * BQ);
          tma2d(&tq, q_full, sQ(g) + c * (BQ * 128), int(h * DH + c * 64), row);
          if constexpr (SPLIT)
            tma2d(&tq, q_full, sQ(g) + L::kQ1 + c * (BQ * 128), int(3 * d + h * DH + c * 64), row);
        }
      for (int j = 0; j < nt_all; ++j) {
        const int s = j % NST, r = j / NST;
        if (r > 0) bar_wait(&kv_empty[s], (r - 1) & 1);
        bar_expect(&kv_full[s], 2 * L::kKV);
        const int row = int(start + int64_t(j) * BKV);
        for (int c = 0; c < NB; ++c) {
          tma2d(&tkv, &kv_full[s], sK(s) + c * (BKV * 128), int(d + h * DH + c * 64), row);
          tma2d(&tkv, &kv_full[s], sV(s) + c * (BKV * 128), int(2 * d + h * DH + c * 64), row);
          if constexpr (SPLIT) {
            tma2d(&tkv, &kv_full[s], sK(s) + L::kKV1 + c * (BKV * 128), int(4 * d + h * DH + c * 64), row);
            tma2d(&tkv, &kv_full[s], sV(s) + L::kKV1 + c * (BKV * 128), int(5 * d + h * DH + c * 64), row);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = idesc(BQ, BKV, false), id_o = idesc(BQ, DH, true);
      auto issue_s = [&](int g, int j) {
        const int s = j % NST, bf = j & 1;
        bar_wait(&kv_full[s], (j / NST) & 1);
        if (j >= 2) bar_wait(&s_free(g)[bf], ((j >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint64_t a = desc_k(sQ(g) + (kk >> 2) * (BQ * 128)) + 2 * (kk & 3);
          const uint64_t bb = desc_k(sK(s) + (kk >> 2) * (BKV * 128)) + 2 * (kk & 3);
          mma(tS(g) + bf * 64, a, bb, id_s, kk > 0);
          if constexpr (SPLIT) {  // + q_hi k_lo + q_lo k_hi
            const uint64_t al = desc_k(sQ(g) + L::kQ1 + (kk >> 2) * (BQ * 128)) + 2 * (kk & 3);
            const uint64_t bl = desc_k(sK(s) + L::kKV1 + (kk >> 2) * (BKV * 128)) + 2 * (kk & 3);
            mma(tS(g) + bf * 64, a, bl, id_s, 1);
            mma(tS(g) + bf * 64, al, bb, id_s, 1);
          }
        }
        commit(&s_full(g)[bf]);
      };
      bar_wait(q_full, 0);
      for (int g = 0; g < ntile; ++g) issue_s(g, 0);
      for (int j = 0; j < nt_all; ++j) {
        for (int g = 0; g < ntile; ++g)
          if (j + 1 < nt_of(g)) issue_s(g, j + 1);
        const int s = j % NST, pb = j % PB;
        for (int g = 0; g < ntile; ++g) {
          if (j >= nt_of(g)) continue;
          bar_wait(&p_full(g)[pb], (j / PB) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk) {
            const uint64_t a = desc_k(sP(g, pb)) + 2 * kk;
            const uint64_t bb = desc_mn(sV(s)) + ((2048 * kk) >> 4);
            mma(tO(g), a, bb, id_o, (j | kk) != 0);
            if constexpr (SPLIT) {  // + p_hi v_lo + p_lo v_hi
              const uint64_t al = desc_k(sP(g, pb) + L::kP1) + 2 * kk;
              const uint64_t bl = desc_mn(sV(s) + L::kKV1) + ((2048 * kk) >> 4);
              mma(tO(g), a, bl, id_o, 1);
              mma(tO(g), al, bb, id_o, 1);
            }
          }
          commit(o_done(g));
        }
        commit(&kv_empty[s]);
      }
    }
    __syncwarp();
  } else {
    // ---- softmax: warpgroup g = Q tile g; thread r <-> query q0 + g BQ + r <-> TMEM lane r
    const int g = (warp - 2) >> 2;
    const int q = warp & 3, r = q * 32 + lane;
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    const int64_t qg = q0 + int64_t(g) * BQ, qi = qg + r;
    const int nt = g < ntile ? nt_of(g) : 0;
    const float scale = 1.4426950408889634f / sqrtf(float(DH));  // log2 domain
    float m = -FLT_MAX, l = 0.f;
    for (int j = 0; j < nt; ++j) {
      const int bf = j & 1;
      bar_wait(&s_full(g)[bf], (j >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t sa[32], sb[32];
      tld32(tS(g) + lane_off + bf * 64, sa);
      tld32(tS(g) + lane_off + bf * 64 + 32, sb);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      bar_arrive(&s_free(g)[bf]);
      const int k0 = j * BKV;
      float sv[64];
      float mx = -FLT_MAX;
      // masks only on tiles that reach the diagonal or the end of the sequence
      // (block-uniform test): the others are raw scaled scores
      if (k0 + BKV - 1 <= int(qg) && k0 + BKV <= int(len)) {
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          sv[c] = __uint_as_float(c < 32 ? sa[c] : sb[c - 32]) * scale;
          mx = fmaxf(mx, sv[c]);
        }
      } else {
        const int lim = min(int(qi), int(len) - 1) - k0;  // keys k0 + c with c <= lim are visible
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          const float v = c <= lim ? __uint_as_float(c < 32 ? sa[c] : sb[c - 32]) * scale : -FLT_MAX;
          sv[c] = v;
          mx = fmaxf(mx, v);
        }
      }
      // lazy rescale (log2 domain): keep the running max unless some row of the
      // warp grew by more than 2^8 — p <= 256 stays exact in fp32 / bf16 and the
      // final O / l uses the same max, so the result is unchanged
      const bool grow = __any_sync(0xffffffffu, m == -FLT_MAX || mx > m + 8.f);
      const float mn = grow ? fmaxf(m, mx) : m;
      const float corr = m == -FLT_MAX ? 0.f : exp2f(m - mn);
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < 64; ++c) {  // masked scores (-FLT_MAX) underflow to exactly 0
        const float p = exp2f(sv[c] - mn);
        sv[c] = p;
        rs += p;
      }
      l = l * corr + rs;
      if (j > 0) {
        // O holds P_{j-1} V_{j-1}: wait for it, then rescale rows whose max moved
        bar_wait(o_done(g), (j - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (grow) {
#pragma unroll 1
          for (int c = 0; c < DH; c += 32) {
            uint32_t o[32];
            tld32(tO(g) + lane_off + c, o);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
            tst32(tO(g) + lane_off + c, o);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
      }
      m = mn;
      // P_j row (bf16) in the K-major 128B swizzle: row r at r * 128, chunk c ^ (r & 7)
      uint8_t* prow = sP(g, j % PB) + r * 128;
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8) {
        uint32_t w4[4], l4[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p0 = sv[c8 * 8 + 2 * e], p1 = sv[c8 * 8 + 2 * e + 1];
          const __nv_bfloat162 p2 = __floats2bfloat162_rn(p0, p1);
          w4[e] = *reinterpret_cast<const uint32_t*>(&p2);
          if constexpr (SPLIT) {
            const float2 hf = __bfloat1622float2(p2);
            const __nv_bfloat162 q2 = __floats2bfloat162_rn(p0 - hf.x, p1 - hf.y);
            l4[e] = *reinterpret_cast<const uint32_t*>(&q2);
          }
        }
        *reinterpret_cast<uint4*>(prow + ((c8 ^ (r & 7)) << 4)) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        if constexpr (SPLIT)
          *reinterpret_cast<uint4*>(prow + L::kP1 + ((c8 ^ (r & 7)) << 4)) = make_uint4(l4[0], l4[1], l4[2], l4[3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      bar_arrive(&p_full(g)[j % PB]);
    }
    // ---- epilogue: O / l
    if (nt > 0) {
      bar_wait(o_done(g), (nt - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const float inv = 1.0f / l;
#pragma unroll 1
      for (int c = 0; c < DH; c += 32) {
        uint32_t o[32];
        tld32(tO(g) + lane_off + c, o);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (qi < len) {
          bf16* dst = out + (start + qi) * (SPLIT ? 2 * d : d) + h * DH + c;
#pragma unroll
          for (int e8 = 0; e8 < 32; e8 += 8) {
            Vec16<bf16> ov, ol;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float y = __uint_as_float(o[e8 + e]) * inv;
              ov.v[e] = __float2bfloat16_rn(y);
              if constexpr (SPLIT) ol.v[e] = __float2bfloat16_rn(y - __bfloat162float(ov.v[e]));
            }
            *reinterpret_cast<uint4*>(dst + e8) = ov.u;
            if constexpr (SPLIT) *reinterpret_cast<uint4*>(dst + d + e8) = ol.u;  // lo plane
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L::kTmem));
  }
}

// Q tiles per CTA (PPOEXP_ATTN_QT forces 1 or 2).  Measured on B200: two help
// the mixed-mode split kernel at head_dim 64 (C2 scoring pass 10.05 -> 9.83 ms)
// but slow the bf16 kernel (C5 shape 0.49 -> 0.59 ms per launch: half the CTAs,
// a longer causal tail), so bf16 keeps one; the split head_dim-128 tiles would
// not fit shared memory twice.
int attn_qt(bool split) {
  static const int qt = [] {
    const char* e = getenv("PPOEXP_ATTN_QT");
    return e ? atoi(e) : 0;
  }();
  return qt ? qt : (split ? 2 : 1);
}

template <int DH, bool SPLIT, int QT>
void launch_fa_qt(Ctx& c, const bf16* qkv, const int64_t* seq_offsets, int64_t B, int64_t max_len, int64_t H,
                  int64_t M_total, bf16* out) {
  using L = FaSmem<DH, SPLIT, QT>;
  const int64_t d = H * DH, w = (SPLIT ? 6 : 3) * d;
  const CUtensorMap tq = make_map(qkv, M_total, w, w, BQ);
  const CUtensorMap tkv = make_map(qkv, M_total, w, w, BKV);
  auto k = attn_prefill_tc_kernel<DH, SPLIT, QT>;
  static bool attr = false;
  if (!attr) {
    PPOEXP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes));
    attr = true;
  }
  dim3 grid(unsigned(ceil_div(max_len, BQ * QT)), unsigned(H), unsigned(B));
  const double flops = 2.0 * 2.0 * B * H * double(max_len) * max_len / 2 * DH;
  c.launch("attention_prefill", 0, flops, [&] {
    launch_kernel(c, k, grid, dim3(L::kThreads), L::kBytes, 1, tq, tkv, seq_offsets, int(H), out);
  });
}

template <int DH, bool SPLIT = false>
void launch_fa(Ctx& c, const bf16* qkv, const int64_t* seq_offsets, int64_t B, int64_t max_len, int64_t H,
               int64_t M_total, bf16* out) {
  if constexpr (!(SPLIT && DH == 128)) {
    if (attn_qt(SPLIT) == 2) return launch_fa_qt<DH, SPLIT, 2>(c, qkv, seq_offsets, B, max_len, H, M_total, out);
  }
  launch_fa_qt<DH, SPLIT, 1>(c, qkv, seq_offsets, B, max_len, H, M_total, out);
}

}  // namespace

// bf16 prefill attention on tcgen05; false when the shape is not supported
// (head_dim 64 / 128, 16-byte aligned qkv rows).
bool attention_prefill_tc(Ctx& c, const bf16* qkv, const int64_t* seq_offsets, int64_t B, int64_t max_len, int64_t H,
                          int64_t DH, int64_t M_total, bf16* out, bool force) {
  // PPOEXP_ATTN_TC=0 falls back to the mma.sync kernel (measured slower: C2 scoring
  // 3.94 vs 3.17 ms per step, C5 shape 1.44 vs 0.50 ms per launch)
  static const int mode = [] {
    const char* e = getenv("PPOEXP_ATTN_TC");
    return e ? atoi(e) : 1;
  }();
  if (!force && mode == 0) return false;
  if (M_total <= 0 || (reinterpret_cast<uintptr_t>(qkv) & 15)) return false;
  switch (DH) {
    case 64: return launch_fa<64>(c, qkv, seq_offsets, B, max_len, H, M_total, out), true;
    case 128: return launch_fa<128>(c, qkv, seq_offsets, B, max_len, H, M_total, out), true;
    default: return false;
  }
}

// Mixed mode: qkv as hi | lo planes [M, 6d], output planes [M, 2d]; head_dim
// 64 or 128.  False when not eligible (PPOEXP_ATTN_TC=0 also disables it).
bool attention_prefill_tc_split(Ctx& c, const bf16* qkv_planes, const int64_t* seq_offsets, int64_t B,
                                int64_t max_len, int64_t H, int64_t DH, int64_t M_total, bf16* out_planes) {
  static const int mode = [] {
    const char* e = getenv("PPOEXP_ATTN_TC");
    return e ? atoi(e) : 1;
  }();
  if (mode == 0 || (DH != 64 && DH != 128) || M_total <= 0 || (reinterpret_cast<uintptr_t>(qkv_planes) & 15))
    return false;
  if (DH == 64)
    launch_fa<64, true>(c, qkv_planes, seq_offsets, B, max_len, H, M_total, out_planes);
  else
    launch_fa<128, true>(c, qkv_planes, seq_offsets, B, max_len, H, M_total, out_planes);
  return true;
}

}  // namespace ppx
