// attention.cu — K5 attention kernels.
//
//  * attn_prefill: causal multi-head attention over packed ragged sequences
//    (scoring / critic / RM forwards and the engine's batched prefill).  The
//    reference computes softmax(q·k^T/sqrt(dh) + mask)·v per head
//    (src/model.cpp:230-236); masked scores are exp(-1e30) = 0, so a causal
//    online softmax is the same arithmetic up to fp32 rounding.
//  * attn_decode: one query per sequence against the PAGED KV cache (flash
//    decode).  It appends this step's K/V row first (KvSession::step,
//    src/model.cpp:305-308), then attends over positions 0..pos
//    (src/model.cpp:313-333): scale by 1/sqrt(dh) before the max, exp(s-max),
//    normalise, weighted V sum.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "kernels.hpp"

namespace ppx {

namespace {

// ---------------------------------------------------------------- prefill
// CTA = (64 queries) x (one head) x (one sequence).  TPQ threads per query,
// each owning 16 of the DH dims; K/V tiles of 64 keys staged in smem (fp32).
template <class T, int DH>
__global__ void __launch_bounds__(64 * (DH / 16)) attn_prefill_kernel(const T* __restrict__ qkv,
                                                                      const int64_t* __restrict__ seq_offsets,
                                                                      int64_t H, T* __restrict__ out) {
  PDL_ENTRY();
  constexpr int TPQ = DH / 16, QT = 64, KT = 64, NT = QT * TPQ, LD = DH + 4;
  extern __shared__ __align__(16) float sm[];
  float* Ks = sm;
  float* Vs = sm + KT * LD;
  const int64_t b = blockIdx.z, h = blockIdx.y, q0 = int64_t(blockIdx.x) * QT;
  const int64_t start = seq_offsets[b], len = seq_offsets[b + 1] - start;
  if (q0 >= len) return;
  const int64_t d = H * DH, ld3 = 3 * d;
  const int tid = threadIdx.x, ql = tid / TPQ, part = tid % TPQ;
  const int64_t qi = q0 + ql;
  const bool valid = qi < len;
  float q[16], acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    q[i] = valid ? to_f(qkv[(start + qi) * ld3 + h * DH + part * 16 + i]) : 0.f;
    acc[i] = 0.f;
  }
  const float inv_sqrt_dh = 1.0f / sqrtf(float(DH));
  float m = -FLT_MAX, l = 0.f;
  const int64_t kend = min(len, q0 + QT);
  for (int64_t k0 = 0; k0 < kend; k0 += KT) {
    for (int e = tid; e < KT * DH; e += NT) {
      const int j = e / DH, i = e % DH;
      const int64_t kj = k0 + j;
      float kv = 0.f, vv = 0.f;
      if (kj < len) {
        kv = to_f(qkv[(start + kj) * ld3 + d + h * DH + i]);
        vv = to_f(qkv[(start + kj) * ld3 + 2 * d + h * DH + i]);
      }
      Ks[j * LD + i] = kv;
      Vs[j * LD + i] = vv;
    }
    __syncthreads();
    const int jn = int((kend - k0) < KT ? (kend - k0) : KT);
    for (int j = 0; j < jn; ++j) {
      const float* kr = Ks + j * LD + part * 16;
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < 16; ++i) s = fmaf(q[i], kr[i], s);
#pragma unroll
      for (int o = TPQ / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      s *= inv_sqrt_dh;
      if (valid && k0 + j <= qi) {
        if (s > m) {
          const float corr = m > -FLT_MAX ? expf(m - s) : 0.f;
          l *= corr;
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[i] *= corr;
          m = s;
        }
        const float p = expf(s - m);
        l += p;
        const float* vr = Vs + j * LD + part * 16;
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fmaf(p, vr[i], acc[i]);
      }
    }
    __syncthreads();
  }
  if (valid) {
    const float inv = 1.0f / l;
#pragma unroll
    for (int i = 0; i < 16; ++i) out[(start + qi) * d + h * DH + part * 16 + i] = from_f<T>(acc[i] * inv);
  }
}

// ---------------------------------------------------------------- decode
// CTA per (sequence, head); each of the 4 warps streams its own 32-token
// tiles of the paged K/V cache into shared memory with coalesced,
// double-buffered cp.async (a tile never straddles a page: page_size % 32 == 0).
// Q·K: lane-per-token dot products out of padded smem rows (no per-token
// shuffles).  Online softmax per tile.  P·V: lane-per-dim with the tile's
// probabilities broadcast by shuffle.  The warps' (max, sum, acc) are merged
// through shared memory at the end.
__device__ __forceinline__ void cp_async16_dec(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}

__device__ __forceinline__ uint32_t dec_su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// NS: K/V tile stages per warp, TT: tokens per tile.  (NS, TT) = (2, 16) keeps the
// (1, 32) footprint (32 KB per CTA for dh 64 bf16: 6 CTAs/SM) but double-buffers.
// Rows of a multiple of 128 bytes arrive by TMA: the pool is a 2-D tensor
// [rows, DH] (one row = one (layer, page, K|V, head, slot)), boxes of 128 bytes x
// TT rows with the 128B swizzle, one elected lane per warp issuing them against
// a per-warp mbarrier; other row sizes use cp.async.
template <class T, int DH, int NS, int TT>
__global__ void __launch_bounds__(128, 6) attn_decode_kernel(const T* __restrict__ qkv, const int32_t* __restrict__ pos,
                                                          const int32_t* __restrict__ done,
                                                          const int32_t* __restrict__ block_table, int layer,
                                                          KvGeom g, T* __restrict__ kv, T* __restrict__ out,
                                                          unsigned long long* dbg, bf16* __restrict__ split_out,
                                                          const __grid_constant__ CUtensorMap tmkv) {
  // debug (PPOEXP_ATTN_TRACE): CTA (0, 0) thread 0 stage clocks
  auto stamp = [&](int k) {
    if (dbg && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) dbg[k] = clock64();
  };
  stamp(0);
  // Programmatic dependent launch: only this step's q/k/v (the immediately
  // preceding QKV GEMM) is produced by the predecessor grid.  Every earlier
  // kernel has completed when this grid starts (each kernel triggers its
  // dependents only after its own griddepcontrol.wait), so the sequence
  // state, the block table and the cached K/V rows < pos are read BEFORE the
  // wait: the first tile's HBM latency overlaps the QKV GEMM's tail.
  constexpr int NW = 4;
  constexpr int ROWB = DH * int(sizeof(T));   // bytes per K/V row
  // 128-byte rows (bf16, dh 64) are stored unpadded with the 16-byte chunks
  // XOR-swizzled by (row & 7): conflict-free for lane-per-token K reads and
  // per-row V reads, and 32 KB of tiles per CTA (6 CTAs/SM: one wave of 768).
  // Other row sizes keep a 16-byte pad.
  constexpr bool TMAK = ROWB % 128 == 0;      // TMA-fed tiles: dense [box][TT][128 B], 128B swizzle
  constexpr bool SWZ = ROWB == 128;
  constexpr int LDB = (SWZ || TMAK) ? ROWB : ROWB + 16;  // smem bytes per row (per tile: TT * LDB)
  constexpr int NBOX = ROWB / 128;
  constexpr int CPR = ROWB / 16;              // 16-byte chunks per row
  constexpr int EPT = DH;                     // lane-per-token: whole row
  constexpr int DPL = DH >= 32 ? DH / 32 : 1; // dims per lane (P·V)
  constexpr int DLANES = DH / DPL;
  constexpr bool HALF = TT == 16 && sizeof(T) == 4 && CPR % 2 == 0;  // fp32 KV: 16-token tiles, half rows per lane
  extern __shared__ __align__(1024) uint8_t smem_dec[];
  __shared__ __align__(8) uint64_t tbar[NW][NS];  // TMA completion per warp and stage
  __shared__ float sm_m[NW], sm_l[NW];
  __shared__ float sm_acc[NW][DH];
  __shared__ __align__(16) float sm_q[DH];  // the query (lane-uniform reads: broadcast)
  const int64_t b = blockIdx.y, h = blockIdx.x;
  if (done[b]) return;  // (implicit trigger at exit)
  const int64_t p = pos[b], ctx = p + 1;
  const int64_t d = g.H * DH, PS = g.page_size;
  const T* row = qkv + b * 3 * d;
  const int32_t* bt = block_table + b * g.max_pages_per_seq;
  auto base = [&](int64_t t, int which) -> T* {
    const int64_t page = bt[t / PS];
    return kv + ((((int64_t)layer * g.n_pages + page) * 2 + which) * g.H + h) * PS * DH + (t % PS) * DH;
  };
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  // per-warp tiles: [stage][K|V][TT rows][LDB bytes] (TMA: 1024-byte aligned swizzle atoms)
  uint8_t* sbase = smem_dec;
  if constexpr (TMAK)
    sbase = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dec) + 1023) & ~uintptr_t(1023));
  uint8_t* wsm = sbase + size_t(w) * NS * 2 * TT * LDB;
  auto tile_ptr = [&](int buf, int which) { return wsm + (buf * 2 + which) * TT * LDB; };
  auto chunk = [](int r, int c) {
    if constexpr (TMAK) return (c >> 3) * (TT * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4);
    return r * LDB + ((SWZ ? (c ^ (r & 7)) : c) << 4);
  };
  if constexpr (TMAK) {
    if (lane == 0) {
      for (int s = 0; s < NS; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(dec_su32(&tbar[w][s])));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  uint32_t tphase = 0;  // bit s: parity of the next completion of stage s
  auto issue = [&](int64_t t0, int buf) {
    if constexpr (TMAK) {
      if (lane == 0) {
        const int64_t page = bt[t0 / PS];
        const int64_t rk = ((((int64_t)layer * g.n_pages + page) * 2 + 0) * g.H + h) * PS + (t0 % PS);
        const int64_t rv = rk + g.H * PS;  // the V rows of the same page / head
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(dec_su32(&tbar[w][buf])),
                     "r"(2 * TT * ROWB)
                     : "memory");
#pragma unroll
        for (int bx = 0; bx < NBOX; ++bx) {
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                  dec_su32(tile_ptr(buf, 0) + bx * TT * 128)),
              "l"(reinterpret_cast<uint64_t>(&tmkv)), "r"(dec_su32(&tbar[w][buf])), "r"(bx * (128 / int(sizeof(T)))),
              "r"(int(rk))
              : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                  dec_su32(tile_ptr(buf, 1) + bx * TT * 128)),
              "l"(reinterpret_cast<uint64_t>(&tmkv)), "r"(dec_su32(&tbar[w][buf])), "r"(bx * (128 / int(sizeof(T)))),
              "r"(int(rv))
              : "memory");
        }
      }
      return;
    }
    const int64_t n = (ctx - t0) < TT ? (ctx - t0) : TT;
    const T* k0 = base(t0, 0);  // contiguous within the page
    const T* v0 = base(t0, 1);
    for (int e = lane; e < TT * CPR; e += 32) {
      const int r = e / CPR, c = e % CPR;
      if (r < n) {
        cp_async16_dec(tile_ptr(buf, 0) + chunk(r, c), reinterpret_cast<const uint8_t*>(k0) + r * ROWB + c * 16);
        cp_async16_dec(tile_ptr(buf, 1) + chunk(r, c), reinterpret_cast<const uint8_t*>(v0) + r * ROWB + c * 16);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const float* q = sm_q;
  const float inv_sqrt_dh = 1.0f / sqrtf(float(DH));
  float m = -FLT_MAX, l = 0.f, acc[DPL];
#pragma unroll
  for (int i = 0; i < DPL; ++i) acc[i] = 0.f;
  const int dl = lane < DLANES ? lane : 0;
  int64_t t0 = int64_t(w) * TT;
  auto holds_p = [&](int64_t t) { return p >= t && p < t + TT; };
  // this warp's first tile (and second, when double-buffered), unless it
  // holds the new position (appended below)
  const bool early0 = t0 < ctx && !holds_p(t0);
  const int64_t t1 = t0 + int64_t(NW) * TT;
  const bool early1 = NS == 2 && t1 < ctx && !holds_p(t1);
  if (early0) issue(t0, 0);
  if (early1) issue(t1, 1);
  stamp(1);
  pdl_wait();  // this step's q/k/v are valid from here on
  pdl_trigger();
  stamp(2);
  // append this step's K/V row (KvSession::step, src/model.cpp:305-308)
  for (int i = tid; i < DH; i += 128) {
    base(p, 0)[i] = row[d + h * DH + i];
    base(p, 1)[i] = row[2 * d + h * DH + i];
  }
  for (int i = tid; i < DH; i += 128) sm_q[i] = to_f(row[h * DH + i]);
  // the appended row is read back by TMA (the async proxy) below
  if constexpr (TMAK) asm volatile("fence.proxy.async.global;" ::: "memory");
  __syncthreads();  // the appended row and the query are visible to the whole CTA
  stamp(3);
  bool nxt_issued = early1;          // tile it+1 already committed
  bool zero_last = false;            // tile 0 committed after tile 1: wait for everything
  if (t0 < ctx && !early0) {
    issue(t0, 0);
    zero_last = early1;
  }
  int it = 0;
  for (; t0 < ctx; t0 += int64_t(NW) * TT, ++it) {
    const int64_t tn = t0 + int64_t(NW) * TT;
    const int buf = NS == 2 ? (it & 1) : 0;
    if constexpr (TMAK) {
      if (NS == 2 && !nxt_issued && tn < ctx) {
        issue(tn, buf ^ 1);
        nxt_issued = true;
      }
      const uint32_t par = (tphase >> buf) & 1u;
      asm volatile(
          "{\n\t.reg .pred P1;\nTW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra TW_%=;\n\t}" ::"r"(
              dec_su32(&tbar[w][buf])),
          "r"(par)
          : "memory");
      tphase ^= 1u << buf;
    } else if (NS == 2) {
      if (!nxt_issued && tn < ctx) {
        issue(tn, buf ^ 1);
        nxt_issued = true;
      }
      if (nxt_issued && !zero_last && tn < ctx)
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      else
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    const int nt = int((ctx - t0) < TT ? (ctx - t0) : TT);
    // ---- scores: lane = token (HALF: 16-token fp32 tiles, lanes 0-15 and
    // 16-31 take the two halves of the same token's row, one shuffle joins them)
    float s = -FLT_MAX;
    if constexpr (HALF) {
      const int tk = lane & 15, hv = lane >> 4;
      float dot = 0.f;
      if (tk < nt) {
        const uint8_t* kt = tile_ptr(buf, 0);
#pragma unroll
        for (int c = hv * (CPR / 2); c < (hv + 1) * (CPR / 2); ++c) {
          Vec16<T> v4;
          v4.u = *reinterpret_cast<const uint4*>(kt + chunk(tk, c));
#pragma unroll
          for (int e = 0; e < Vec16<T>::N; ++e) dot = fmaf(to_f(v4.v[e]), q[c * Vec16<T>::N + e], dot);
        }
      }
      dot += __shfl_xor_sync(0xffffffffu, dot, 16);
      if (lane < nt) s = dot * inv_sqrt_dh;
    } else if (lane < nt) {
      const uint8_t* kt = tile_ptr(buf, 0);
      float dot = 0.f;
#pragma unroll
      for (int c = 0; c < CPR; ++c) {
        Vec16<T> v4;
        v4.u = *reinterpret_cast<const uint4*>(kt + chunk(lane, c));
#pragma unroll
        for (int e = 0; e < Vec16<T>::N; ++e) dot = fmaf(to_f(v4.v[e]), q[c * Vec16<T>::N + e], dot);
      }
      s = dot * inv_sqrt_dh;
    }
    float tm = s;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, o));
    const float mnew = fmaxf(m, tm);
    const float corr = m == -FLT_MAX ? 0.f : expf(m - mnew);
    const float pr = lane < nt ? expf(s - mnew) : 0.f;
    float ps = pr;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
    l = l * corr + ps;
    m = mnew;
#pragma unroll
    for (int i = 0; i < DPL; ++i) acc[i] *= corr;
    // ---- P·V: lane = dims
    const uint8_t* vt = tile_ptr(buf, 1);
    const int vb = dl * DPL * int(sizeof(T));  // byte offset of this lane's dims in an unswizzled row
    for (int j = 0; j < nt; ++j) {
      const float pj = __shfl_sync(0xffffffffu, pr, j);
      const T* vr = reinterpret_cast<const T*>(vt + chunk(j, vb >> 4) + (vb & 15));
#pragma unroll
      for (int i = 0; i < DPL; ++i) acc[i] = fmaf(pj, to_f(vr[i]), acc[i]);
    }
    __syncwarp();  // this buffer is refilled next (NS == 1) or two tiles from now
    if (NS == 1 && tn < ctx) issue(tn, 0);
    nxt_issued = false;
    zero_last = false;
  }
  stamp(4);
  // ---- merge the warps
  if (lane == 0) {
    sm_m[w] = m;
    sm_l[w] = l;
  }
  if (lane < DLANES)
#pragma unroll
    for (int i = 0; i < DPL; ++i) sm_acc[w][lane * DPL + i] = acc[i];
  __syncthreads();
  float M = sm_m[0];
#pragma unroll
  for (int k = 1; k < NW; ++k) M = fmaxf(M, sm_m[k]);
  float L = 0.f, sc[NW];
#pragma unroll
  for (int k = 0; k < NW; ++k) {
    sc[k] = sm_m[k] == -FLT_MAX ? 0.f : expf(sm_m[k] - M);
    L += sm_l[k] * sc[k];
  }
  const float inv = 1.0f / L;
  for (int i = tid; i < DH; i += 128) {
    float o = 0.f;
#pragma unroll
    for (int k = 0; k < NW; ++k) o += sm_acc[k][i] * sc[k];
    if (split_out) {  // mixed decode: the O projection TMAs the two bf16 terms
      const float v = o * inv;
      const bf16 hi = __float2bfloat16_rn(v);
      split_out[b * 2 * d + h * DH + i] = hi;
      split_out[b * 2 * d + d + h * DH + i] = __float2bfloat16_rn(v - __bfloat162float(hi));
    } else {
      out[b * d + h * DH + i] = from_f<T>(o * inv);
    }
  }
  stamp(5);
  if (dbg && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) dbg[6] = ctx;
}

template <class T, int DH>
void prefill_impl(Ctx& c, const T* qkv, const int64_t* seq_offsets, int64_t B, int64_t max_len, int64_t H, T* out) {
  constexpr int TPQ = DH / 16, LD = DH + 4;
  const size_t smem = 2 * 64 * LD * sizeof(float);
  auto k = attn_prefill_kernel<T, DH>;
  PPOEXP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  dim3 grid(ceil_div(max_len, 64), H, B);
  const double flops = 2.0 * 2.0 * B * H * double(max_len) * max_len / 2 * DH;
  c.launch("attention_prefill", 0, flops, [&] { launch_kernel(c, k, dim3(grid), dim3(64 * TPQ), smem, 1, qkv, seq_offsets, H, out); });
}

// 2-D view of the paged KV pool for TMA: rows of DH elements, boxes of 128 bytes
// x TT rows, 128B swizzle (cached per pool / shape).
template <class T>
CUtensorMap kv_map(const T* kv, const KvGeom& g, int tt) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int64_t, int64_t, int>, CUtensorMap> cache;
  const int64_t rows = g.n_layers * g.n_pages * 2 * g.H * g.page_size;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(static_cast<const void*>(kv), rows, g.DH, tt);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  if (!fn) throw Error(6, "cuda: cuTensorMapEncodeTiled unavailable");
  if (rows >= (int64_t(1) << 31)) throw ContractError("decode attention: KV pool above 2^31 rows");
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(g.DH), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(g.DH * sizeof(T))};
  const cuuint32_t box[2] = {cuuint32_t(128 / sizeof(T)), cuuint32_t(tt)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(&m, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                        const_cast<T*>(kv), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(6, "cuda: cuTensorMapEncodeTiled (KV pool) failed (" + std::to_string(int(r)) + ")");
  cache.emplace(key, m);
  return m;
}

template <class T, int DH, int NS, int TT>
void decode_launch(Ctx& c, const T* qkv, int64_t B, const int32_t* pos, const int32_t* done,
                   const int32_t* block_table, int layer, const KvGeom& g, T* kv, T* out, double bytes,
                   bf16* split_out) {
  auto k = attn_decode_kernel<T, DH, NS, TT>;
  constexpr bool tmak = (DH * sizeof(T)) % 128 == 0;
  const size_t row = tmak ? DH * sizeof(T) : (DH * sizeof(T) == 128 ? 128 : DH * sizeof(T) + 16);  // kernel's LDB
  const size_t smem = size_t(4) * NS * 2 * TT * row + (tmak ? 1024 : 0);  // 4 warps x NS x (K, V) x TT rows
  CUtensorMap tm{};
  if (tmak) tm = kv_map(kv, g, TT);
  static bool attr = false;
  if (!attr) {
    PPOEXP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
    if (getenv("PPOEXP_DEBUG_ATTN")) {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 128, smem);
      fprintf(stderr, "attn_decode<%d,%d,%d,%d>: dynamic smem %zu, %d CTAs/SM\n", int(sizeof(T)), DH, NS, TT, smem,
              per_sm);
    }
  }
  dim3 grid(g.H, B);
  unsigned long long* dbg = nullptr;
  if (getenv("PPOEXP_ATTN_TRACE"))  // debug: stamps of the last launch
    dbg = static_cast<unsigned long long*>(c.workspace("attn.trace", 16 * 8));
  c.launch("decode_attention", bytes, 0, [&] { launch_kernel(c, k, grid, dim3(128), smem, 1, qkv, pos, done,
                                                              block_table, layer, g, kv, out, dbg, split_out, tm); });
}

template <class T, int DH>
void decode_impl(Ctx& c, const T* qkv, int64_t B, const int32_t* pos, const int32_t* done, const int32_t* block_table,
                 int layer, const KvGeom& g, T* kv, T* out, double bytes, bf16* split_out) {
  if (g.page_size % 32) throw ContractError("engine: page_size must be a multiple of 32");
  // single-stage tiles halve the CTA's shared memory (6 resident CTAs/SM for dh 64 bf16: one wave of
  // 768 (sequence, head) CTAs at C2); other warps on the SM hide each warp's tile latency
  // 32-token tiles, single stage (default), or 16-token tiles double buffered:
  // both 32 KB per CTA for dh 64 bf16 (6 CTAs/SM: one wave of 768 (sequence,
  // head) CTAs at C2).  Measured: the tile loop streams KV at the HBM roofline
  // (9.1 us for 61.5 MB at context 313), and 16-token tiles are ~3% slower.
  static const int tile = [] {
    const char* e = getenv("PPOEXP_ATTN_TILE");
    return e ? atoi(e) : 32;
  }();
  // fp32 KV (mixed / F32 modes): a 32-token fp32 tile set is 64 KB per CTA (3 CTAs/SM, 1.7 waves at
  // C2); 16-token tiles with two lanes per token row keep 6 CTAs/SM (one wave)
  static const int f32_tile = [] {
    const char* e = getenv("PPOEXP_ATTN_TILE_F32");
    return e ? atoi(e) : 16;
  }();
  if (tile == 16 && DH * sizeof(T) == 128)
    decode_launch<T, DH, 2, 16>(c, qkv, B, pos, done, block_table, layer, g, kv, out, bytes, split_out);
  else if (sizeof(T) == 4 && f32_tile == 16 && DH >= 32)
    decode_launch<T, DH, 1, 16>(c, qkv, B, pos, done, block_table, layer, g, kv, out, bytes, split_out);
  else
    decode_launch<T, DH, 1, 32>(c, qkv, B, pos, done, block_table, layer, g, kv, out, bytes, split_out);
}

}  // namespace

bool attention_prefill_mma(Ctx& c, const bf16* qkv, const int64_t* seq_offsets, int64_t B, int64_t max_len,
                           int64_t H, int64_t DH, bf16* out);

template <class T>
void launch_attention_prefill(Ctx& c, const T* qkv, const int64_t* seq_offsets, int64_t B, int64_t max_len,
                              int64_t H, int64_t DH, T* out) {
  if (B <= 0 || max_len <= 0) return;
  if constexpr (std::is_same_v<T, bf16>) {
    if (attention_prefill_mma(c, qkv, seq_offsets, B, max_len, H, DH, out)) return;
  }
  switch (DH) {
    case 16: return prefill_impl<T, 16>(c, qkv, seq_offsets, B, max_len, H, out);
    case 32: return prefill_impl<T, 32>(c, qkv, seq_offsets, B, max_len, H, out);
    case 64: return prefill_impl<T, 64>(c, qkv, seq_offsets, B, max_len, H, out);
    case 128: return prefill_impl<T, 128>(c, qkv, seq_offsets, B, max_len, H, out);
    default: throw ContractError("attention: head_dim " + std::to_string(DH) + " unsupported (16/32/64/128)");
  }
}

template <class T>
void launch_attention_decode(Ctx& c, const T* qkv, int64_t B, const int32_t* pos, const int32_t* done,
                             const int32_t* block_table, int layer, const KvGeom& g, T* kv, T* out,
                             double algorithmic_bytes, bf16* split_out) {
  if (B <= 0) return;
  const double ab = algorithmic_bytes;
  switch (g.DH) {
    case 16: return decode_impl<T, 16>(c, qkv, B, pos, done, block_table, layer, g, kv, out, ab, split_out);
    case 32: return decode_impl<T, 32>(c, qkv, B, pos, done, block_table, layer, g, kv, out, ab, split_out);
    case 64: return decode_impl<T, 64>(c, qkv, B, pos, done, block_table, layer, g, kv, out, ab, split_out);
    case 128: return decode_impl<T, 128>(c, qkv, B, pos, done, block_table, layer, g, kv, out, ab, split_out);
    default: throw ContractError("attention: head_dim " + std::to_string(g.DH) + " unsupported (16/32/64/128)");
  }
}

template void launch_attention_prefill<float>(Ctx&, const float*, const int64_t*, int64_t, int64_t, int64_t, int64_t,
                                              float*);
template void launch_attention_prefill<bf16>(Ctx&, const bf16*, const int64_t*, int64_t, int64_t, int64_t, int64_t,
                                             bf16*);
template void launch_attention_decode<float>(Ctx&, const float*, int64_t, const int32_t*, const int32_t*,
                                             const int32_t*, int, const KvGeom&, float*, float*, double, bf16*);
template void launch_attention_decode<bf16>(Ctx&, const bf16*, int64_t, const int32_t*, const int32_t*,
                                            const int32_t*, int, const KvGeom&, bf16*, bf16*, double, bf16*);

}  // namespace ppx
