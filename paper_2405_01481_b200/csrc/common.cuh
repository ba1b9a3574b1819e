// common.cuh — shared helpers for the ppoexp sm_100a kernels and host runtime.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace ppx {

using bf16 = __nv_bfloat16;

// ------------------------------------------------------------ errors
// Typed errors mirror the reference's exception set
// (include/aligner/tensor.hpp:17-25, engine.hpp:19-21, ppo.hpp:22-24).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
inline Error ContractError(const std::string& m) { return Error(1, m); }
inline Error IndexError(const std::string& m) { return Error(2, m); }
inline Error ShapeError(const std::string& m) { return Error(3, m); }
inline Error RefitError(const std::string& m) { return Error(4, m); }
inline Error PpoError(const std::string& m) { return Error(5, m); }

#define PPOEXP_CUDA(expr)                                                                        \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess) {                                                                    \
      (void)cudaGetLastError();                                                                 \
      throw ::ppx::Error(e_ == cudaErrorMemoryAllocation ? 7 : 6,                            \
                            std::string("cuda: ") + cudaGetErrorString(e_) + " at " #expr);     \
    }                                                                                           \
  } while (0)

// ------------------------------------------------------------ device math
template <class T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<bf16>(bf16 x) { return __bfloat162float(x); }

template <class T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

// GELU-tanh, reference src/model.cpp:358-361 (fp32 here).
__device__ __forceinline__ float gelu_tanh(float x) {
  const float kC = 0.7978845608028654f;
  return 0.5f * x * (1.0f + tanhf(kC * (x + 0.044715f * x * x * x)));
}
// The same GELU as x * sigmoid(2u) (1 + tanh(u) = 2 / (1 + e^{-2u})): no
// cancellation, one ex2.approx (2^-22 relative) and one fast division —
// a third of the instructions of tanhf, within ~5e-7 relative of gelu_tanh
// (tensor-core epilogues; the F32 parity mode keeps gelu_tanh)
__device__ __forceinline__ float gelu_fast(float x) {
  const float kC2 = -2.0f * 0.7978845608028654f * 1.4426950408889634f;  // -2 kC log2(e)
  const float t = kC2 * fmaf(0.044715f * x, x * x, x);
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(t));
  return __fdividef(x, 1.0f + e);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// 16-byte vector of T.
template <class T>
struct Vec16 {
  static constexpr int N = 16 / sizeof(T);
  union {
    uint4 u;
    T v[N];
  };
};

// Programmatic dependent launch (PDL): every kernel is launched with
// programmatic stream serialization, so it may start while its predecessor
// drains.  pdl_wait() blocks until the predecessor grid has completed and its
// writes are visible; nothing produced upstream may be touched before it.
// pdl_trigger() lets the successor grid begin its own prologue early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Small single-wave grids (decode: a CTA per sequence) release their dependent
// before waiting on their own predecessor, so the next kernel (a decode GEMM)
// runs its setup and weight prefetch while this one is still queued.  Only
// safe for a grid that is resident in one wave: early-launched dependents could
// otherwise hold the SM slots its remaining CTAs need.
__device__ __forceinline__ void pdl_entry_small_grid() {
  if (gridDim.x * gridDim.y * gridDim.z <= 256) {
    pdl_trigger();
    pdl_wait();
  } else {
    pdl_wait();
    pdl_trigger();
  }
}
#define PDL_ENTRY() \
  do {              \
    pdl_wait();     \
    pdl_trigger();  \
  } while (0)

constexpr int kPadToken = 256;  // include/aligner/model.hpp:17
constexpr int kEotToken = 257;  // include/aligner/model.hpp:18

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace ppx
