// decode_mega.cu — the body of one bf16 decode step as ONE persistent,
// cooperative kernel (one 256-thread CTA per SM, grid-wide barriers between
// phases).
//
// Launched one kernel per op, a decode step (KvSession::step,
// src/model.cpp:279-355) is ~85 small dependent kernels whose HBM work is a
// few microseconds each; the chain is bound by launch / drain / ramp latency.
// Here it runs inside one kernel:
//
//   per layer:  [R]  x += Σ_s part_s (or embed), LN1 → h     CTA per row
//               [G]  part_s = h · Wqkv^T                      tcgen05, split-K
//               [A]  qkv = Σ_s part_s; append K/V; attention   warp per (seq, head)
//               [G]  part_s = att · Wo^T
//               [R]  x += Σ_s part_s, LN2 → h
//               [G]  part_s = h · Wup^T
//               [U]  up = gelu(Σ_s part_s)                     elementwise
//               [G]  part_s = up · Wdown^T
//   then        [R]  x += Σ_s part_s, LN_f → h   (the LM head + sampler follow)
//
// GEMM phases are swap-AB tcgen05 MMAs: a CTA owns one 128-feature weight
// tile (UMMA M = 128) × the batch (UMMA N = 64) × one K-slice of <= 256,
// operands staged by TMA (128B swizzle) and accumulated in TMEM.  The K
// split is chosen so tiles × splits <= #SMs, so every CTA ingests only its
// K-slice of the activations (per-SM L2 ingest, ~64 B/clk, is the limit a
// "full-K per CTA" decomposition hits).  Split-K partials go to one fp32
// buffer [S][B][N] and are reduced by the consuming phase in split order:
// every output is a fixed-order sum (deterministic, no atomics).  A CTA's
// weight tile for the next GEMM phase is issued between its barrier arrival
// and the barrier wait, and layer l+1's weights are prefetched into L2 during
// layer l.
#include <cuda.h>

#include <cfloat>

#include "attn_core.cuh"
#include "kernels.hpp"

namespace ppx {

CUtensorMap make_map(const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);  // gemm_tc.cu

namespace {

constexpr int kThreads = 256, kWarps = 8, kNB = 64, kBM = 128, kBK = 64, kMaxCh = 4, kTT = 32;
constexpr int kWTile = kBM * kBK * 2;  // 16 KB weight chunk
constexpr int kXTile = kNB * kBK * 2;  // 8 KB activation chunk
constexpr int kTmemCols = 64;
constexpr int kMaxSplit = 32;  // K splits per GEMM

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  const uint64_t addr = su32(p);
  return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
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
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// This CTA's 1/gridDim slice of [p, p + bytes) into L2.
__device__ __forceinline__ void prefetch_slice(const void* p, size_t bytes) {
  const size_t per = ((bytes + gridDim.x - 1) / gridDim.x + 15) & ~size_t(15);
  const size_t off = per * blockIdx.x;
  if (off >= bytes) return;
  size_t n = bytes - off < per ? bytes - off : per;
  const uint8_t* q = static_cast<const uint8_t*>(p) + off;
  while (n > 0) {
    const uint32_t c = n > (size_t(1) << 20) ? (1u << 20) : uint32_t(n);
    prefetch_l2(q, c);
    q += c;
    n -= c;
  }
}
__device__ __forceinline__ void prefetch_layer(const MegaLayer& ly, int d, int f) {
  if (threadIdx.x != 0) return;
  prefetch_slice(ly.wqkv, size_t(3) * d * d * 2);
  prefetch_slice(ly.wo, size_t(d) * d * 2);
  prefetch_slice(ly.wup, size_t(f) * d * 2);
  prefetch_slice(ly.wdown, size_t(d) * f * 2);
}

// ------------------------------------------------------------------ grid barrier
// Counting barrier over co-resident CTAs on a monotonically increasing 64-bit
// arrival counter bar[0]: barrier k of this launch completes when the counter
// reaches base + (k+1)·G, base = bar[1] = the counter value the previous
// launch ended at (stored by CTA 0 at exit; launches are stream-ordered).
// arrive(): CTA sync, then thread 0 adds 1 with a fire-and-forget RELEASE
// reduction (no return trip, no reset, no separate generation word).
// wait(): thread 0 spins with RELAXED loads and acquires once.  Independent
// work (the next phase's weight TMA) goes between the two.
// Optional trace (PPOEXP_MEGA_TRACE): per barrier k and CTA, {arrive, depart}.
__device__ __forceinline__ void grid_arrive(unsigned long long* bar, uint64_t* trace, int k) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (trace) trace[(size_t(k) * gridDim.x + blockIdx.x) * 2] = gtimer();
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
  }
}
__device__ __forceinline__ void grid_wait(unsigned long long* bar, unsigned long long target, uint64_t* trace, int k) {
  if (threadIdx.x == 0) {
    unsigned long long v;
    do {
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
    } while (v < target);
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
    if (trace) trace[(size_t(k) * gridDim.x + blockIdx.x) * 2 + 1] = gtimer();
  }
  __syncthreads();
}
// Writes that a later phase reads through TMA (h, att, up) are made visible
// to the async proxy by their writers before the barrier.
__device__ __forceinline__ void fence_for_tma() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// ------------------------------------------------------------------ CTA state
struct Ctl {
  uint64_t wfull, xfull, done;  // mbarriers (one completion per GEMM item)
  uint32_t tmem;                // TMEM base (kTmemCols fp32 columns x 128 lanes)
  float red[kWarps];
};

// ------------------------------------------------------------------ row phase
// x[b] <- embed(b) (mode 0) or x[b] + Σ_s part[s][b] (mode 1, split order);
// h[b] <- LN(x[b]) (src/model.cpp:387-400: mean, centred variance / d, eps
// 1e-5).  float4 per thread (d <= 4096); a row's partial loads are issued in
// groups of 8 before the adds.
__device__ __noinline__ void row_phase(const MegaArgs& a, int mode, int nsplit, const float* __restrict__ g,
                                       const float* __restrict__ bb, float* red) {
  const int d = a.d, d4 = d >> 2, tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
    float4 v[4];
    float s = 0.f;
    const int t = mode == 0 ? a.next_tok[b] : 0, p = mode == 0 ? a.pos[b] : 0;
    float4* xr = reinterpret_cast<float4*>(a.x + int64_t(b) * d);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j4 = tid + i * kThreads;
      v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (j4 < d4) {
        if (mode == 0) {
          const uint2 tu = *reinterpret_cast<const uint2*>(a.tok + int64_t(t) * d + j4 * 4);
          const uint2 pu = *reinterpret_cast<const uint2*>(a.posemb + int64_t(p) * d + j4 * 4);
          const float2 t0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&tu.x));
          const float2 t1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&tu.y));
          const float2 p0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pu.x));
          const float2 p1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pu.y));
          v[i] = make_float4(t0.x + p0.x, t0.y + p0.y, t1.x + p1.x, t1.y + p1.y);
        } else {
          float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
          const float4* pp = reinterpret_cast<const float4*>(a.part + int64_t(b) * d) + j4;
          const int64_t sstride = int64_t(a.B) * d4;
          for (int s0 = 0; s0 < nsplit; s0 += 8) {
            float4 pt[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (s0 + k < nsplit) pt[k] = __ldcg(pp + (s0 + k) * sstride);
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (s0 + k < nsplit) {
                r.x += pt[k].x;
                r.y += pt[k].y;
                r.z += pt[k].z;
                r.w += pt[k].w;
              }
          }
          v[i] = __ldcg(xr + j4);
          v[i].x += r.x;
          v[i].y += r.y;
          v[i].z += r.z;
          v[i].w += r.w;
        }
        xr[j4] = v[i];
        s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
      }
    }
    s = warp_sum(s);
    if (lane == 0) red[w] = s;
    __syncthreads();
    float mu = 0.f;
#pragma unroll
    for (int k = 0; k < kWarps; ++k) mu += red[k];
    mu /= float(d);
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (tid + i * kThreads < d4) {
        const float c0 = v[i].x - mu, c1 = v[i].y - mu, c2 = v[i].z - mu, c3 = v[i].w - mu;
        q += (c0 * c0 + c1 * c1) + (c2 * c2 + c3 * c3);
      }
    q = warp_sum(q);
    __syncthreads();
    if (lane == 0) red[w] = q;
    __syncthreads();
    float var = 0.f;
#pragma unroll
    for (int k = 0; k < kWarps; ++k) var += red[k];
    const float is = 1.0f / sqrtf(var / float(d) + 1e-5f);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j4 = tid + i * kThreads;
      if (j4 < d4) {
        const float4 gg = reinterpret_cast<const float4*>(g)[j4], b4 = reinterpret_cast<const float4*>(bb)[j4];
        __nv_bfloat162 lo = __floats2bfloat162_rn(gg.x * ((v[i].x - mu) * is) + b4.x, gg.y * ((v[i].y - mu) * is) + b4.y);
        __nv_bfloat162 hi = __floats2bfloat162_rn(gg.z * ((v[i].z - mu) * is) + b4.z, gg.w * ((v[i].w - mu) * is) + b4.w);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&lo);
        u.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(a.h + int64_t(b) * d + j4 * 4) = u;
      }
    }
    __syncthreads();
  }
  fence_for_tma();
}

// ------------------------------------------------------------------ GELU reduce
// up[b][n] = bf16(gelu(Σ_s part[s][b][n])) over the whole [B, f] block, each
// CTA a contiguous float4 range.
__device__ __noinline__ void gelu_phase(const MegaArgs& a, int nsplit) {
  const int64_t n4 = int64_t(a.B) * a.f / 4;
  const int64_t per = (n4 + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = per * blockIdx.x, e1 = e0 + per < n4 ? e0 + per : n4;
  const float4* pp = reinterpret_cast<const float4*>(a.part);
  for (int64_t e = e0 + threadIdx.x; e < e1; e += kThreads) {
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < nsplit; s0 += 8) {
      float4 pt[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (s0 + k < nsplit) pt[k] = __ldcg(pp + (s0 + k) * n4 + e);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (s0 + k < nsplit) {
          r.x += pt[k].x;
          r.y += pt[k].y;
          r.z += pt[k].z;
          r.w += pt[k].w;
        }
    }
    __nv_bfloat162 lo = __floats2bfloat162_rn(gelu_tanh(r.x), gelu_tanh(r.y));
    __nv_bfloat162 hi = __floats2bfloat162_rn(gelu_tanh(r.z), gelu_tanh(r.w));
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&lo);
    u.y = *reinterpret_cast<uint32_t*>(&hi);
    reinterpret_cast<uint2*>(a.up)[e] = u;
  }
  fence_for_tma();
}

// ------------------------------------------------------------------ GEMM phase
struct GemmJob {
  const CUtensorMap* tw;  // weights [N, K] (K-major), box 128 x 64
  const CUtensorMap* tx;  // activations [rows, K], box 64 x 64
  int N, K, S;
};

// This CTA's item: 128-feature tile m0, K-slice [k0, k0 + nch*64), split s.
__device__ __forceinline__ bool gemm_item(const GemmJob& j, int& m0, int& k0, int& nch, int& s) {
  const int T = j.N / kBM;
  if (int(blockIdx.x) >= T * j.S) return false;
  s = blockIdx.x / T;
  m0 = (blockIdx.x % T) * kBM;
  const int Kr = j.K / j.S;
  k0 = s * Kr;
  nch = Kr / kBK;
  return true;
}

// One thread: TMA the weight chunks of this CTA's item into smem.
__device__ __forceinline__ void issue_w(uint8_t* sm, Ctl& c, const GemmJob& j, int m0, int k0, int nch) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect(&c.wfull, uint32_t(nch) * kWTile);
  for (int ch = 0; ch < nch; ++ch) tma_load_2d(j.tw, &c.wfull, sm + ch * kWTile, k0 + ch * kBK, m0);
}

// Between barrier arrive and wait: this CTA's weight tile for job j.
__device__ __forceinline__ bool prefetch_w(uint8_t* sm, Ctl& c, const GemmJob& j) {
  int m0, k0, nch, s;
  if (!gemm_item(j, m0, k0, nch, s)) return false;
  if (threadIdx.x == 0) issue_w(sm, c, j, m0, k0, nch);
  return true;
}

// part[s][b][m0 + i] = Σ_{k in slice} W[m0 + i][k] · X[b][k]   (b < B)
__device__ __noinline__ void gemm_phase(uint8_t* sm, Ctl& c, const GemmJob& j, int B, float* __restrict__ part,
                                        bool prefetched, uint32_t& cnt) {
  int m0, k0, nch, s;
  if (!gemm_item(j, m0, k0, nch, s)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t par = cnt & 1u;
  ++cnt;
  uint8_t* sW = sm;
  uint8_t* sX = sm + kMaxCh * kWTile;
  if (threadIdx.x == 0) {
    if (!prefetched) issue_w(sm, c, j, m0, k0, nch);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect(&c.xfull, uint32_t(nch) * kXTile);
    for (int ch = 0; ch < nch; ++ch) tma_load_2d(j.tx, &c.xfull, sX + ch * kXTile, k0 + ch * kBK, 0);
  } else if (threadIdx.x == 32) {
    mbar_wait(&c.wfull, par);
    mbar_wait(&c.xfull, par);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    constexpr uint32_t idesc = idesc_bf16(kBM, kNB);
    for (int ch = 0; ch < nch; ++ch) {
      const uint64_t dw = smem_desc_sw128(sW + ch * kWTile);
      const uint64_t dx = smem_desc_sw128(sX + ch * kXTile);
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k) umma_bf16(c.tmem, dw + 2 * k, dx + 2 * k, idesc, (ch | k) != 0);
    }
    umma_commit(&c.done);
  }
  if (warp >= 4) {
    mbar_wait(&c.done, par);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3;
    const int n = m0 + q * 32 + lane;
    float* out = part + int64_t(s) * B * j.N + n;
#pragma unroll 1
    for (int cb = 0; cb < kNB; cb += 16) {
      if (cb >= B) break;
      uint32_t v[16];
      tmem_ld16(c.tmem + (uint32_t(q * 32) << 16) + uint32_t(cb), v);
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if (cb + e < B) out[int64_t(cb + e) * j.N] = __uint_as_float(v[e]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
}

// ------------------------------------------------------------------ attention
// Warp per (sequence, head).  q/k/v = Σ_s QKV partials (split order); K/V
// are appended at pos in bf16 (src/model.cpp:305-308), then the paged cache
// is streamed in 32-token tiles through a 3-stage cp.async ring into the
// lane-per-token WarpAttn core (attn_core.cuh).  The partial loads are issued
// first, together with the sequence's state and block-table row.
constexpr int kStages = 3;
template <int DH>
__device__ __noinline__ void attn_phase(const MegaArgs& a, int layer, int nsplit, uint8_t* smr) {
  constexpr int ROWB = DH * 2, LDB = ROWB + 16, CPR = ROWB / 16, DPL = DH / 32;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* st = (a.trace && lane == 0) ? a.trace + size_t(8 * a.L) * gridDim.x * 2 +
                                              ((size_t(layer) * gridDim.x + blockIdx.x) * kWarps + w) * 4
                                        : nullptr;
  if (st) st[0] = st[1] = st[2] = st[3] = 0;
  uint8_t* wsm = smr + size_t(w) * kStages * 2 * kTT * LDB;
  float* qs = reinterpret_cast<float*>(smr + size_t(kWarps) * kStages * 2 * kTT * LDB) + w * DH;
  auto tile_ptr = [&](int stg, int which) { return wsm + (stg * 2 + which) * kTT * LDB; };
  const int d = int(a.g.H) * DH, PS = int(a.g.page_size), d3 = 3 * d;
  const float scale = 1.0f / sqrtf(float(DH));
  const int64_t pstride = int64_t(a.B) * d3;
  for (int item = blockIdx.x * kWarps + w; item < a.B * a.g.H; item += gridDim.x * kWarps) {
    const int b = item / int(a.g.H), h = item % int(a.g.H);
    if (st) st[0] = clock64();
    // everything independent first: QKV partials, state, block-table row
    float tq[8][DPL], tk[8][DPL], tv[8][DPL];
    const float* pp = a.part + int64_t(b) * d3 + h * DH + lane * DPL;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < nsplit) {
        const float* ps = pp + k * pstride;
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
          tq[k][i] = __ldcg(ps + i);
          tk[k][i] = __ldcg(ps + d + i);
          tv[k][i] = __ldcg(ps + 2 * d + i);
        }
      }
    const int isdone = a.done[b];
    const int p = a.pos[b], ctx = p + 1;
    const int32_t my_page = lane < a.g.max_pages_per_seq ? a.block_table[int64_t(b) * a.g.max_pages_per_seq + lane] : 0;
    if (isdone) continue;
    const int64_t lbase = ((int64_t)layer * a.g.n_pages) * 2;
    auto base = [&](int tk_, int which) -> bf16* {
      const int64_t page = __shfl_sync(0xffffffffu, my_page, tk_ / PS);
      return a.kv + (((lbase + page * 2) + which) * a.g.H + h) * PS * DH + (tk_ % PS) * DH;
    };
    auto issue = [&](int t) {  // tile t (tokens [32t, 32t+32)) into stage t % kStages
      const int t0 = t * kTT, n = (ctx - t0) < kTT ? (ctx - t0) : kTT, stg = t % kStages;
      const uint8_t* k0 = reinterpret_cast<const uint8_t*>(base(t0, 0));
      const uint8_t* v0 = reinterpret_cast<const uint8_t*>(base(t0, 1));
      for (int e = lane; e < kTT * CPR; e += 32) {
        const int r = e / CPR, cc = e % CPR;
        if (r < n) {
          cp16(tile_ptr(stg, 0) + r * LDB + cc * 16, k0 + r * ROWB + cc * 16);
          cp16(tile_ptr(stg, 1) + r * LDB + cc * 16, v0 + r * ROWB + cc * 16);
        }
      }
    };
    const int ntiles = (ctx + kTT - 1) / kTT;
    // remaining partials (nsplit > 8), then the sums in split order
    float qv[DPL], kv[DPL], vv[DPL];
#pragma unroll
    for (int i = 0; i < DPL; ++i) qv[i] = kv[i] = vv[i] = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < nsplit)
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
          qv[i] += tq[k][i];
          kv[i] += tk[k][i];
          vv[i] += tv[k][i];
        }
    for (int k = 8; k < nsplit; ++k) {
      const float* ps = pp + k * pstride;
#pragma unroll
      for (int i = 0; i < DPL; ++i) {
        qv[i] += __ldcg(ps + i);
        kv[i] += __ldcg(ps + d + i);
        vv[i] += __ldcg(ps + 2 * d + i);
      }
    }
    bf16* const kdst = base(p, 0);
    bf16* const vdst = base(p, 1);
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      kdst[lane * DPL + i] = from_f<bf16>(kv[i]);
      vdst[lane * DPL + i] = from_f<bf16>(vv[i]);
      qs[lane * DPL + i] = qv[i];
    }
    __syncwarp();
    float q[DH];
#pragma unroll
    for (int i = 0; i < DH; ++i) q[i] = qs[i];
    if (st) st[1] = clock64();
    // group g carries tile g: two tiles in flight ahead of the one consumed
    issue(0);
    cp_commit();
    if (1 < ntiles) issue(1);
    cp_commit();
    WarpAttn<DH> wa;
    wa.init();
    for (int t = 0; t < ntiles; ++t) {
      if (t + 2 < ntiles) issue(t + 2);
      cp_commit();
      asm volatile("cp.async.wait_group 2;" ::: "memory");
      __syncwarp();
      const int t0 = t * kTT, stg = t % kStages;
      wa.tile(q, tile_ptr(stg, 0), tile_ptr(stg, 1), LDB, (ctx - t0) < kTT ? (ctx - t0) : kTT, scale);
      __syncwarp();  // stage stg is refilled three tiles from now
    }
    cp_wait_all();
    const float inv = 1.0f / wa.finish();
    if (st) {
      st[2] = clock64();
      st[3] = ntiles;
    }
#pragma unroll
    for (int i = 0; i < DPL; ++i) a.att[int64_t(b) * d + h * DH + lane * DPL + i] = from_f<bf16>(wa.acc[i] * inv);
    __syncwarp();  // qs is rewritten by the next item
  }
  fence_for_tma();
}

template <int DH>
constexpr size_t attn_smem() {
  return size_t(kWarps) * kStages * 2 * kTT * (DH * 2 + 16) + size_t(kWarps) * DH * 4;
}
constexpr size_t gemm_smem() { return size_t(kMaxCh) * (kWTile + kXTile); }
template <int DH>
constexpr size_t mega_smem() {
  return (attn_smem<DH>() > gemm_smem() ? attn_smem<DH>() : gemm_smem()) + 1024;  // + 1 KB alignment slack
}

// ------------------------------------------------------------------ the kernel
template <int DH>
__global__ void __launch_bounds__(kThreads, 1) decode_mega_kernel(const __grid_constant__ MegaArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ Ctl c;
  if (threadIdx.x == 0) {
    mbar_init(&c.wfull, 1);
    mbar_init(&c.xfull, 1);
    mbar_init(&c.done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&c.tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(a.bar);
  const unsigned long long base = bar[1];  // counter value at the end of the previous launch
  const unsigned long long G = gridDim.x;
  uint32_t cnt = 0;
  int kb = 0;
  const int d = a.d, f = a.f;
  if (a.prefetch) prefetch_layer(a.layers[0], d, f);
#define BARRIER_THEN(pre)                                 \
  grid_arrive(bar, a.trace, kb);                          \
  pre;                                                    \
  grid_wait(bar, base + (kb + 1) * G, a.trace, kb);       \
  ++kb;
  for (int l = 0; l < a.L; ++l) {
    const MegaLayer ly = a.layers[l];
    if (a.prefetch && l + 1 < a.L) prefetch_layer(a.layers[l + 1], d, f);
    const CUtensorMap* wm = a.wmaps + 4 * l;
    const GemmJob jq{wm + 0, &a.tm_h, 3 * d, d, a.split[0]};
    const GemmJob jo{wm + 1, &a.tm_att, d, d, a.split[1]};
    const GemmJob ju{wm + 2, &a.tm_h, f, d, a.split[2]};
    const GemmJob jd{wm + 3, &a.tm_up, d, f, a.split[3]};
    bool pf;
    row_phase(a, l == 0 ? 0 : 1, a.split[3], ly.ln1w, ly.ln1b, c.red);
    BARRIER_THEN(pf = prefetch_w(sm, c, jq))
    gemm_phase(sm, c, jq, a.B, a.part, pf, cnt);
    BARRIER_THEN((void)0)
    attn_phase<DH>(a, l, a.split[0], sm);
    BARRIER_THEN(pf = prefetch_w(sm, c, jo))
    gemm_phase(sm, c, jo, a.B, a.part, pf, cnt);
    BARRIER_THEN((void)0)
    row_phase(a, 1, a.split[1], ly.ln2w, ly.ln2b, c.red);
    BARRIER_THEN(pf = prefetch_w(sm, c, ju))
    gemm_phase(sm, c, ju, a.B, a.part, pf, cnt);
    BARRIER_THEN((void)0)
    gelu_phase(a, a.split[2]);
    BARRIER_THEN(pf = prefetch_w(sm, c, jd))
    gemm_phase(sm, c, jd, a.B, a.part, pf, cnt);
    BARRIER_THEN((void)0)
  }
#undef BARRIER_THEN
  row_phase(a, 1, a.split[3], a.lnfw, a.lnfb, c.red);
  // every CTA has passed the last barrier, so all kb·G arrivals are in
  if (blockIdx.x == 0 && threadIdx.x == 0) bar[1] = base + (unsigned long long)kb * G;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(c.tmem), "r"(kTmemCols));
}

// Largest tiles x splits <= grid with a K-slice of 1..kMaxCh 64-wide chunks.
int pick_split(int N, int K, int grid) {
  const int T = N / kBM, nk = K / kBK;
  int best = 0;
  for (int S = 1; S <= nk; ++S) {
    if (nk % S || nk / S > kMaxCh || T * S > grid || S > kMaxSplit) continue;
    if (best == 0 || S > best) best = S;
  }
  return best;
}

int sm_count() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <int DH>
void launch_impl(Ctx& c, const MegaArgs& a, double bytes) {
  auto k = decode_mega_kernel<DH>;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = mega_smem<DH>();
  cfg.stream = c.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  c.launch("decode_step", bytes, 0, [&] { PPOEXP_CUDA(cudaLaunchKernelEx(&cfg, k, a)); });
}

}  // namespace

size_t decode_mega_part_bytes() { return size_t(sm_count()) * kBM * kNB * 4; }

bool decode_mega_plan(MegaArgs& a) {
  const int DH = int(a.g.DH);
  if (a.B < 1 || a.B > kNB || a.d % kBM || a.f % kBM || a.d > 4096 || a.g.page_size % kTT) return false;
  if (DH != 32 && DH != 64) return false;
  if (a.g.max_pages_per_seq > 32) return false;
  a.grid = sm_count();
  a.split[0] = pick_split(3 * a.d, a.d, a.grid);
  a.split[1] = pick_split(a.d, a.d, a.grid);
  a.split[2] = pick_split(a.f, a.d, a.grid);
  a.split[3] = pick_split(a.d, a.f, a.grid);
  for (int i = 0; i < 4; ++i)
    if (a.split[i] < 1) return false;
  const size_t smem = DH == 32 ? mega_smem<32>() : mega_smem<64>();
  int per_sm = 0;
  auto occ = [&](auto k) {
    PPOEXP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    PPOEXP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, smem));
  };
  if (DH == 32)
    occ(decode_mega_kernel<32>);
  else
    occ(decode_mega_kernel<64>);
  return per_sm >= 1;
}

void decode_mega_act_maps(MegaArgs& a, int64_t rows) {
  a.tm_h = make_map(a.h, rows, a.d, a.d, kNB);
  a.tm_att = make_map(a.att, rows, a.d, a.d, kNB);
  a.tm_up = make_map(a.up, rows, a.f, a.f, kNB);
}

void decode_mega_weight_maps(const MegaLayer* layers_host, int L, int d, int f, CUtensorMap* out) {
  for (int l = 0; l < L; ++l) {
    const MegaLayer& ly = layers_host[l];
    out[4 * l + 0] = make_map(ly.wqkv, 3 * d, d, d, kBM);
    out[4 * l + 1] = make_map(ly.wo, d, d, d, kBM);
    out[4 * l + 2] = make_map(ly.wup, f, d, d, kBM);
    out[4 * l + 3] = make_map(ly.wdown, d, f, f, kBM);
  }
}

void launch_decode_mega(Ctx& c, const MegaArgs& a, double bytes) {
  if (a.g.DH == 32)
    launch_impl<32>(c, a, bytes);
  else
    launch_impl<64>(c, a, bytes);
}

}  // namespace ppx
