// attn_core.cuh — per-warp decode-attention core over shared-memory K/V tiles
// (one query against a run of cached positions; src/model.cpp:313-333:
// scores scaled by 1/sqrt(dh) before the max, exp(s - max), normalised,
// weighted V sum).
//
// Lane-per-token for BOTH products: lane t scores token t of a 32-token tile
// (Q·K over its own K row, 4 independent partial sums) and accumulates
// p_t · V_t into a lane-private DH-float accumulator.  The running max is
// warp-uniform (one 5-step shuffle max per tile); the running sum stays
// lane-private.  No per-token shuffles; one butterfly reduce-scatter at the
// end (DH-2 shuffles) leaves each lane DH/32 finished dims.
#pragma once

#include <cfloat>

#include "common.cuh"

namespace ppx {

template <int DH>
struct WarpAttn {
  static constexpr int DPL = DH / 32;  // dims per lane after finish()
  float acc[DH];
  float m, l;

  __device__ __forceinline__ void init() {
    m = -FLT_MAX;
    l = 0.f;
#pragma unroll
    for (int i = 0; i < DH; ++i) acc[i] = 0.f;
  }

  // One tile of nt (<= 32) tokens; lane < nt owns K/V row `lane` (bf16, rows
  // ldb bytes apart).  q holds the full query in fp32.
  __device__ __forceinline__ void tile(const float (&q)[DH], const uint8_t* ktile, const uint8_t* vtile, int ldb,
                                       int nt, float scale) {
    const int lane = threadIdx.x & 31;
    float s = -FLT_MAX;
    if (lane < nt) {
      const uint8_t* kr = ktile + lane * ldb;
      float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < DH / 8; ++c) {
        const uint4 u = *reinterpret_cast<const uint4*>(kr + c * 16);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
          d[e] = fmaf(f.x, q[c * 8 + 2 * e], d[e]);
          d[e] = fmaf(f.y, q[c * 8 + 2 * e + 1], d[e]);
        }
      }
      s = ((d[0] + d[1]) + (d[2] + d[3])) * scale;
    }
    float tm = s;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tm = fmaxf(tm, __shfl_xor_sync(0xffffffffu, tm, o));
    if (tm > m) {  // warp-uniform
      const float corr = m == -FLT_MAX ? 0.f : expf(m - tm);
      l *= corr;
#pragma unroll
      for (int i = 0; i < DH; ++i) acc[i] *= corr;
      m = tm;
    }
    if (lane < nt) {
      const float p = expf(s - m);
      l += p;
      const uint8_t* vr = vtile + lane * ldb;
#pragma unroll
      for (int c = 0; c < DH / 8; ++c) {
        const uint4 u = *reinterpret_cast<const uint4*>(vr + c * 16);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
          acc[c * 8 + 2 * e] = fmaf(p, f.x, acc[c * 8 + 2 * e]);
          acc[c * 8 + 2 * e + 1] = fmaf(p, f.y, acc[c * 8 + 2 * e + 1]);
        }
      }
    }
  }

  // Butterfly reduce-scatter: afterwards acc[0 .. DPL) of lane t holds the
  // warp sums of dims [t*DPL, t*DPL + DPL); returns the warp sum of l.
  __device__ __forceinline__ float finish() {
    const int lane = threadIdx.x & 31;
    level<DH>(lane, 16);
    level<DH / 2>(lane, 8);
    level<DH / 4>(lane, 4);
    level<DH / 8>(lane, 2);
    level<DH / 16>(lane, 1);
    return warp_sum(l);
  }

 private:
  template <int N>
  __device__ __forceinline__ void level(int lane, int o) {
    constexpr int H = N / 2;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const float send = up ? acc[i] : acc[i + H];
      const float keep = up ? acc[i + H] : acc[i];
      acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
};

}  // namespace ppx
