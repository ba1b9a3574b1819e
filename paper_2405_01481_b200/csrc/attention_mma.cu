// attention_mma.cu — K5a on tensor cores for the bf16 path: causal
// multi-head attention over packed ragged sequences (scoring / critic / RM
// forwards and the engine's batched prefill).  FlashAttention-2 structure:
//   CTA = 64 queries (4 warps x 16 rows) of one head of one sequence;
//   K/V tiles of 64 keys double-buffered in smem with cp.async;
//   S = Q K^T and O += P V on mma.sync m16n8k16 (bf16 in, fp32 accumulate),
//   fragments fed by ldmatrix (V through ldmatrix.trans);
//   online softmax in registers, P re-used as the A operand without a trip
//   through shared memory.
// Semantics are the reference's (src/model.cpp:230-236): scores scaled by
// 1/sqrt(dh) before the max, causal, exp(s - max) / sum.
#include <cfloat>

#include "kernels.hpp"

namespace ppx {

namespace {

constexpr int QT = 64, KT = 64, NWARP = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool pred) {
  const int n = pred ? 16 : 0;  // zero-fill when out of range
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_u32(p)));
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int DH>
__global__ void __launch_bounds__(128) attn_prefill_mma_kernel(const bf16* __restrict__ qkv,
                                                               const int64_t* __restrict__ seq_offsets, int64_t H,
                                                               bf16* __restrict__ out) {
  PDL_ENTRY();
  constexpr int LD = DH + 8;        // padded smem row (bank-conflict-free ldmatrix)
  constexpr int KC = DH / 16;       // k16 chunks over the head dim
  constexpr int NO = DH / 8;        // n8 tiles of the output
  constexpr int CH = DH / 8;        // 16-byte chunks per row
  extern __shared__ __align__(128) uint8_t smem_raw[];
  bf16* sQ = reinterpret_cast<bf16*>(smem_raw);
  // double-buffered K / V tiles (pointer arithmetic: a runtime-indexed pointer
  // array would live on the stack)
  auto sK = [&](int bf) { return sQ + QT * LD + bf * KT * LD; };
  auto sV = [&](int bf) { return sQ + QT * LD + (2 + bf) * KT * LD; };
  const int64_t b = blockIdx.z, h = blockIdx.y, q0 = int64_t(blockIdx.x) * QT;
  const int64_t start = seq_offsets[b], len = seq_offsets[b + 1] - start;
  if (q0 >= len) return;
  const int64_t d = H * DH, ld3 = 3 * d;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;

  auto load_rows = [&](bf16* dst, int64_t row0, int64_t col0) {
    for (int e = tid; e < KT * CH; e += 128) {
      const int r = e / CH, c = e % CH;
      const int64_t rr = row0 + r;
      const bool ok = rr < len;
      const bf16* src = qkv + (start + (ok ? rr : 0)) * ld3 + col0 + c * 8;
      cp_async16(dst + r * LD + c * 8, src, ok);
    }
  };
  // Q tile + first K/V tile
  load_rows(sQ, q0, h * DH);
  const int64_t kend = min(len, q0 + QT);  // causal: keys < last query + 1
  const int ntiles = int((kend + KT - 1) / KT);
  load_rows(sK(0), 0, d + h * DH);
  load_rows(sV(0), 0, 2 * d + h * DH);
  cp_async_commit();

  uint32_t qf[KC][4];
  float o[NO][4];
#pragma unroll
  for (int i = 0; i < NO; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-FLT_MAX, -FLT_MAX}, l_r[2] = {0.f, 0.f};
  // softmax in the log2 domain: exp(x - m) == exp2(x * log2e - m * log2e), one MUFU.EX2 per score
  const float scale = 1.4426950408889634f / sqrtf(float(DH));
  const int64_t qrow0 = q0 + warp * 16 + g, qrow1 = qrow0 + 8;

  for (int it = 0; it < ntiles; ++it) {
    const int buf = it & 1;
    if (it + 1 < ntiles) {
      load_rows(sK(buf ^ 1), int64_t(it + 1) * KT, d + h * DH);
      load_rows(sV(buf ^ 1), int64_t(it + 1) * KT, 2 * d + h * DH);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (it == 0) {
      // Q fragments (A operand, row-major): ldmatrix.x4 per k16 chunk
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        const int r = warp * 16 + (lane & 15), c = kc * 16 + (lane >> 4) * 8;
        ldsm_x4(qf[kc][0], qf[kc][1], qf[kc][2], qf[kc][3], sQ + r * LD + c);
      }
    }
    const int64_t k0 = int64_t(it) * KT;
    // ---- S = Q K^T (16 x 64 per warp)
    float s[KT / 8][4];
#pragma unroll
    for (int j = 0; j < KT / 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
    const bf16* K = sK(buf);
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
#pragma unroll
      for (int j = 0; j < KT / 8; j += 2) {
        // two n8 tiles (keys j*8.., (j+1)*8..) x one k16 chunk
        uint32_t b0, b1, b2, b3;
        const int r = j * 8 + (lane & 7) + ((lane >> 4) << 3), c = kc * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(b0, b1, b2, b3, K + r * LD + c);
        mma16816(s[j], qf[kc], b0, b1);
        mma16816(s[j + 1], qf[kc], b2, b3);
      }
    }
    // ---- scale, causal / length mask, online softmax
    float mx[2] = {-FLT_MAX, -FLT_MAX};
#pragma unroll
    for (int j = 0; j < KT / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t key = k0 + j * 8 + 2 * t4 + (e & 1);
        const int64_t qr = e < 2 ? qrow0 : qrow1;
        float v = s[j][e] * scale;
        if (key > qr || key >= len) v = -FLT_MAX;
        s[j][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float mn = fmaxf(m_r[r], mx[r]);
      corr[r] = m_r[r] == -FLT_MAX ? 0.f : exp2f(m_r[r] - mn);
      m_r[r] = mn;
    }
    float rs[2] = {0.f, 0.f};
#pragma unroll
    for (int j = 0; j < KT / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = e >> 1;
        const float p = s[j][e] == -FLT_MAX ? 0.f : exp2f(s[j][e] - m_r[r]);
        s[j][e] = p;
        rs[r] += p;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 1);
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 2);
      l_r[r] = l_r[r] * corr[r] + rs[r];
    }
#pragma unroll
    for (int i = 0; i < NO; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
    // ---- O += P V: P (16 x 64) as A fragments straight from the S accumulators
    const bf16* Vt = sV(buf);
#pragma unroll
    for (int kk = 0; kk < KT / 16; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int i = 0; i < NO; i += 2) {
        uint32_t b0, b1, b2, b3;
        const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, c = i * 8 + (lane >> 4) * 8;
        ldsm_x4_t(b0, b1, b2, b3, Vt + r * LD + c);
        mma16816(o[i], pa, b0, b1);
        mma16816(o[i + 1], pa, b2, b3);
      }
    }
    __syncthreads();  // the buffer is refilled next iteration
  }
  // ---- normalise and store
  const float inv0 = 1.0f / l_r[0], inv1 = 1.0f / l_r[1];
#pragma unroll
  for (int i = 0; i < NO; ++i) {
    const int64_t col = h * DH + i * 8 + 2 * t4;
    if (qrow0 < len)
      *reinterpret_cast<uint32_t*>(out + (start + qrow0) * d + col) = pack_bf16(o[i][0] * inv0, o[i][1] * inv0);
    if (qrow1 < len)
      *reinterpret_cast<uint32_t*>(out + (start + qrow1) * d + col) = pack_bf16(o[i][2] * inv1, o[i][3] * inv1);
  }
}

// ---------------------------------------------------------------- mixed mode
// The same FlashAttention-2 structure with fp32-grade products for mixed mode:
// q, k, v arrive in fp32; each tile is split into two bf16 terms (x = hi + lo,
// |x - hi - lo| <= 2^-18 |x|) and every product takes three MMAs
// (hi*hi + hi*lo + lo*hi; the lo*lo term is below fp32 rounding): S = Q K^T and
// O += P V with P split the same way after the fp32 online softmax.  K / V
// tiles are staged as fp32 by cp.async one tile ahead and split in shared memory.
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
  const float2 hf = __bfloat1622float2(h);
  const __nv_bfloat162 l = __floats2bfloat162_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

template <int DH>
struct SplitSmem {
  static constexpr int LD = DH + 8;                 // bf16 row (conflict-free ldmatrix)
  static constexpr int kTile = 64 * LD;             // elements of one 64-row bf16 tile
  static constexpr int kStage = 64 * DH;            // fp32 elements of one staged 64-row tile
  // bf16: Qh Ql Kh Kl Vh Vl; fp32 staging: K, V
  static constexpr size_t kBytes = size_t(6) * kTile * 2 + size_t(2) * kStage * 4;
};

template <int DH>
__global__ void __launch_bounds__(128) attn_prefill_split_kernel(const float* __restrict__ qkv,
                                                                 const int64_t* __restrict__ seq_offsets, int64_t H,
                                                                 float* __restrict__ out, bf16* __restrict__ planes) {
  PDL_ENTRY();
  using SL = SplitSmem<DH>;
  constexpr int LD = SL::LD, KC = DH / 16, NO = DH / 8, CH4 = DH / 4;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  bf16* sb = reinterpret_cast<bf16*>(smem_raw);
  bf16 *sQh = sb, *sQl = sb + SL::kTile, *sKh = sb + 2 * SL::kTile, *sKl = sb + 3 * SL::kTile;
  bf16 *sVh = sb + 4 * SL::kTile, *sVl = sb + 5 * SL::kTile;
  float* stK = reinterpret_cast<float*>(sb + 6 * SL::kTile);
  float* stV = stK + SL::kStage;
  const int64_t b = blockIdx.z, h = blockIdx.y, q0 = int64_t(blockIdx.x) * QT;
  const int64_t start = seq_offsets[b], len = seq_offsets[b + 1] - start;
  if (q0 >= len) return;
  const int64_t d = H * DH, ld3 = 3 * d;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;

  // fp32 rows -> staging (cp.async, zero-filled past the end)
  auto stage_rows = [&](float* dst, int64_t row0, int64_t col0) {
    for (int e = tid; e < 64 * CH4; e += 128) {
      const int r = e / CH4, c = e % CH4;
      const int64_t rr = row0 + r;
      const bool ok = rr < len;
      cp_async16(dst + r * DH + c * 4, qkv + (start + (ok ? rr : 0)) * ld3 + col0 + c * 4, ok);
    }
  };
  // staging (or registers for Q) -> hi / lo bf16 tiles
  auto split_tile = [&](const float* src, bf16* hi, bf16* lo) {
    for (int e = tid; e < 64 * CH4; e += 128) {
      const int r = e / CH4, c = e % CH4;
      const float4 v = *reinterpret_cast<const float4*>(src + r * DH + c * 4);
      uint32_t h0, l0, h1, l1;
      split2(v.x, v.y, h0, l0);
      split2(v.z, v.w, h1, l1);
      *reinterpret_cast<uint2*>(hi + r * LD + c * 4) = make_uint2(h0, h1);
      *reinterpret_cast<uint2*>(lo + r * LD + c * 4) = make_uint2(l0, l1);
    }
  };
  const int64_t kend = min(len, q0 + QT);
  const int ntiles = int((kend + KT - 1) / KT);
  // Q through the K staging buffer, then the first K / V tile
  stage_rows(stK, q0, h * DH);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  split_tile(stK, sQh, sQl);
  __syncthreads();
  stage_rows(stK, 0, d + h * DH);
  stage_rows(stV, 0, 2 * d + h * DH);
  cp_async_commit();

  uint32_t qh[KC][4], ql[KC][4];
  float o[NO][4];
#pragma unroll
  for (int i = 0; i < NO; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-FLT_MAX, -FLT_MAX}, l_r[2] = {0.f, 0.f};
  const float scale = 1.0f / sqrtf(float(DH));
  const int64_t qrow0 = q0 + warp * 16 + g, qrow1 = qrow0 + 8;
#pragma unroll
  for (int kc = 0; kc < KC; ++kc) {
    const int r = warp * 16 + (lane & 15), c = kc * 16 + (lane >> 4) * 8;
    ldsm_x4(qh[kc][0], qh[kc][1], qh[kc][2], qh[kc][3], sQh + r * LD + c);
    ldsm_x4(ql[kc][0], ql[kc][1], ql[kc][2], ql[kc][3], sQl + r * LD + c);
  }

  for (int it = 0; it < ntiles; ++it) {
    cp_async_wait<0>();
    __syncthreads();  // staged tile landed; the previous tile's MMAs are done with the split tiles
    split_tile(stK, sKh, sKl);
    split_tile(stV, sVh, sVl);
    __syncthreads();  // split tiles visible; staging free
    if (it + 1 < ntiles) {
      stage_rows(stK, int64_t(it + 1) * KT, d + h * DH);
      stage_rows(stV, int64_t(it + 1) * KT, 2 * d + h * DH);
      cp_async_commit();
    }
    const int64_t k0 = int64_t(it) * KT;
    float s[KT / 8][4];
#pragma unroll
    for (int j = 0; j < KT / 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
#pragma unroll
      for (int j = 0; j < KT / 8; j += 2) {
        uint32_t b0, b1, b2, b3, c0, c1, c2, c3;
        const int r = j * 8 + (lane & 7) + ((lane >> 4) << 3), c = kc * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(b0, b1, b2, b3, sKh + r * LD + c);
        ldsm_x4(c0, c1, c2, c3, sKl + r * LD + c);
        mma16816(s[j], ql[kc], b0, b1);  // small terms first
        mma16816(s[j + 1], ql[kc], b2, b3);
        mma16816(s[j], qh[kc], c0, c1);
        mma16816(s[j + 1], qh[kc], c2, c3);
        mma16816(s[j], qh[kc], b0, b1);
        mma16816(s[j + 1], qh[kc], b2, b3);
      }
    }
    // scale, causal / length mask, online softmax (fp32, exp in the natural domain)
    float mx[2] = {-FLT_MAX, -FLT_MAX};
#pragma unroll
    for (int j = 0; j < KT / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t key = k0 + j * 8 + 2 * t4 + (e & 1);
        const int64_t qr = e < 2 ? qrow0 : qrow1;
        float v = s[j][e] * scale;
        if (key > qr || key >= len) v = -FLT_MAX;
        s[j][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float mn = fmaxf(m_r[r], mx[r]);
      corr[r] = m_r[r] == -FLT_MAX ? 0.f : expf(m_r[r] - mn);
      m_r[r] = mn;
    }
    float rs[2] = {0.f, 0.f};
#pragma unroll
    for (int j = 0; j < KT / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = e >> 1;
        const float p = s[j][e] == -FLT_MAX ? 0.f : expf(s[j][e] - m_r[r]);
        s[j][e] = p;
        rs[r] += p;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 1);
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 2);
      l_r[r] = l_r[r] * corr[r] + rs[r];
    }
#pragma unroll
    for (int i = 0; i < NO; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
#pragma unroll
    for (int kk = 0; kk < KT / 16; ++kk) {
      uint32_t ph[4], pl[4];
      split2(s[2 * kk][0], s[2 * kk][1], ph[0], pl[0]);
      split2(s[2 * kk][2], s[2 * kk][3], ph[1], pl[1]);
      split2(s[2 * kk + 1][0], s[2 * kk + 1][1], ph[2], pl[2]);
      split2(s[2 * kk + 1][2], s[2 * kk + 1][3], ph[3], pl[3]);
#pragma unroll
      for (int i = 0; i < NO; i += 2) {
        uint32_t b0, b1, b2, b3, c0, c1, c2, c3;
        const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, c = i * 8 + (lane >> 4) * 8;
        ldsm_x4_t(b0, b1, b2, b3, sVh + r * LD + c);
        ldsm_x4_t(c0, c1, c2, c3, sVl + r * LD + c);
        mma16816(o[i], pl, b0, b1);
        mma16816(o[i + 1], pl, b2, b3);
        mma16816(o[i], ph, c0, c1);
        mma16816(o[i + 1], ph, c2, c3);
        mma16816(o[i], ph, b0, b1);
        mma16816(o[i + 1], ph, b2, b3);
      }
    }
  }
  const float inv0 = 1.0f / l_r[0], inv1 = 1.0f / l_r[1];
#pragma unroll
  for (int i = 0; i < NO; ++i) {
    const int64_t col = h * DH + i * 8 + 2 * t4;
    if (planes) {  // the O projection reads the output as hi | lo bf16 planes [M, 2d]
      uint32_t h, l;
      if (qrow0 < len) {
        split2(o[i][0] * inv0, o[i][1] * inv0, h, l);
        *reinterpret_cast<uint32_t*>(planes + (start + qrow0) * 2 * d + col) = h;
        *reinterpret_cast<uint32_t*>(planes + (start + qrow0) * 2 * d + d + col) = l;
      }
      if (qrow1 < len) {
        split2(o[i][2] * inv1, o[i][3] * inv1, h, l);
        *reinterpret_cast<uint32_t*>(planes + (start + qrow1) * 2 * d + col) = h;
        *reinterpret_cast<uint32_t*>(planes + (start + qrow1) * 2 * d + d + col) = l;
      }
      continue;
    }
    if (qrow0 < len) *reinterpret_cast<float2*>(out + (start + qrow0) * d + col) = make_float2(o[i][0] * inv0, o[i][1] * inv0);
    if (qrow1 < len) *reinterpret_cast<float2*>(out + (start + qrow1) * d + col) = make_float2(o[i][2] * inv1, o[i][3] * inv1);
  }
}

template <int DH>
void launch_split(Ctx& c, const float* qkv, const int64_t* seq_offsets, int64_t B, int64_t max_len, int64_t H,
                  float* out, bf16* planes) {
  constexpr size_t smem = SplitSmem<DH>::kBytes;
  static bool attr = false;
  if (!attr) {
    PPOEXP_CUDA(cudaFuncSetAttribute(attn_prefill_split_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smem)));
    attr = true;
  }
  dim3 grid(ceil_div(max_len, QT), H, B);
  const double flops = 2.0 * 2.0 * B * H * double(max_len) * max_len / 2 * DH;
  c.launch("attention_prefill", 0, flops, [&] {
    launch_kernel(c, attn_prefill_split_kernel<DH>, grid, dim3(128), smem, 1, qkv, seq_offsets, H, out, planes);
  });
}

// bf16 prefill attention on tensor cores; false if the head size is unsupported.
template <int DH>
void launch_mma(Ctx& c, const bf16* qkv, const int64_t* seq_offsets, int64_t B, int64_t max_len, int64_t H,
                bf16* out) {
  constexpr size_t smem = size_t(QT + 4 * KT) * (DH + 8) * sizeof(bf16);
  static bool attr = false;
  if (!attr) {
    PPOEXP_CUDA(cudaFuncSetAttribute(attn_prefill_mma_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smem)));
    attr = true;
  }
  dim3 grid(ceil_div(max_len, QT), H, B);
  const double flops = 2.0 * 2.0 * B * H * double(max_len) * max_len / 2 * DH;
  c.launch("attention_prefill", 0, flops, [&] {
    launch_kernel(c, attn_prefill_mma_kernel<DH>, grid, dim3(128), smem, 1, qkv, seq_offsets, H, out);
  });
}

}  // namespace

// Mixed-mode prefill attention (fp32 q/k/v/out, split-bf16 tensor-core products).
void attention_prefill_split(Ctx& c, const float* qkv, const int64_t* seq_offsets, int64_t B, int64_t max_len,
                             int64_t H, int64_t DH, float* out, bf16* planes) {
  if (B <= 0 || max_len <= 0) return;
  switch (DH) {
    case 16: return launch_split<16>(c, qkv, seq_offsets, B, max_len, H, out, planes);
    case 32: return launch_split<32>(c, qkv, seq_offsets, B, max_len, H, out, planes);
    case 64: return launch_split<64>(c, qkv, seq_offsets, B, max_len, H, out, planes);
    case 128: return launch_split<128>(c, qkv, seq_offsets, B, max_len, H, out, planes);
    default: throw ContractError("attention: head_dim " + std::to_string(DH) + " unsupported (16/32/64/128)");
  }
}

// bf16 prefill attention on tensor cores; false if the head size is unsupported.
bool attention_prefill_mma(Ctx& c, const bf16* qkv, const int64_t* seq_offsets, int64_t B, int64_t max_len,
                           int64_t H, int64_t DH, bf16* out) {
  switch (DH) {
    case 32: return launch_mma<32>(c, qkv, seq_offsets, B, max_len, H, out), true;
    case 64: return launch_mma<64>(c, qkv, seq_offsets, B, max_len, H, out), true;
    case 128: return launch_mma<128>(c, qkv, seq_offsets, B, max_len, H, out), true;
    default: return false;
  }
}

}  // namespace ppx
