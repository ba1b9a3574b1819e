// kernels_basic.cu — embedding, LayerNorm (+ fused value/reward head), KV
// scatter, weight conversion and small helpers; plus the Ctx runtime.
#include <cstring>

#include <type_traits>

#include "kernels.hpp"

namespace ppx {

// ===================================================================== runtime
Ctx::Ctx(int dev) : device(dev) {
  int n = 0;
  PPOEXP_CUDA(cudaGetDeviceCount(&n));
  if (dev < 0 || dev >= n) throw Error(6, "cuda: device " + std::to_string(dev) + " not present");
  DeviceGuard g(dev);
  PPOEXP_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
}

Ctx::~Ctx() {
  DeviceGuard g(device, true);
  cudaStreamSynchronize(stream);
  for (auto& t : pending) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (auto e : event_pool) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    if (aux[i]) {
      cudaStreamSynchronize(aux[i]);
      cudaStreamDestroy(aux[i]);
    }
    if (join_ev[i]) cudaEventDestroy(join_ev[i]);
  }
  if (fork_ev) cudaEventDestroy(fork_ev);
  ws.clear();
  if (pinned) cudaFreeHost(pinned);
  cudaStreamDestroy(stream);
}

cudaEvent_t Ctx::new_event() {
  if (!event_pool.empty()) {
    auto e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  PPOEXP_CUDA(cudaEventCreate(&e));
  return e;
}

void Ctx::harvest_list(const std::vector<TimedLaunch>& evs, bool release) {
  for (const auto& t : evs) {
    PPOEXP_CUDA(cudaEventSynchronize(t.b));
    float ms = 0.f;
    PPOEXP_CUDA(cudaEventElapsedTime(&ms, t.a, t.b));
    auto& s = stats[t.cls];
    s.ms += ms;
    s.launches += 1;
    s.bytes += t.bytes;
    s.flops += t.flops;
    if (release) {
      release_event(t.a);
      release_event(t.b);
    }
  }
}

void Ctx::harvest() {
  harvest_list(pending, true);
  pending.clear();
}

void* Ctx::pinned_staging(size_t bytes) {
  PPOEXP_CUDA(cudaStreamSynchronize(stream));
  if (bytes > pinned_bytes) {
    if (pinned) PPOEXP_CUDA(cudaFreeHost(pinned));
    pinned = nullptr;
    pinned_bytes = 0;
    PPOEXP_CUDA(cudaMallocHost(&pinned, bytes));
    pinned_bytes = bytes;
  }
  return pinned;
}

void copy_in(Ctx& c, void* dst_dev, const void* src, size_t bytes, int where) {
  if (!bytes) return;
  PPOEXP_CUDA(cudaMemcpyAsync(dst_dev, src, bytes, where ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                              c.stream));
}

void copy_out(Ctx& c, void* dst, const void* src_dev, size_t bytes, int where) {
  if (!bytes) return;
  PPOEXP_CUDA(cudaMemcpyAsync(dst, src_dev, bytes, where ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                              c.stream));
}

// ===================================================================== kernels
template <class T>
__global__ void embed_kernel(const int32_t* __restrict__ tokens, const int32_t* __restrict__ positions,
                             int64_t rows, int64_t d, const T* __restrict__ tok, const T* __restrict__ pos,
                             float* __restrict__ x) {
  pdl_entry_small_grid();
  const int64_t r = blockIdx.x;
  if (r >= rows) return;
  const int64_t t = tokens[r], p = positions[r];
  for (int64_t j = threadIdx.x; j < d; j += blockDim.x)
    x[r * d + j] = to_f(tok[t * d + j]) + to_f(pos[p * d + j]);
}

template <class T>
void launch_embed(Ctx& c, const int32_t* tokens, const int32_t* positions, int64_t rows, int64_t d, const T* tok,
                  const T* pos, float* x) {
  if (rows <= 0) return;
  c.launch("embed", double(rows) * d * (2 * sizeof(T) + 4), 0, [&] {
    launch_kernel(c, embed_kernel<T>, dim3(rows), dim3(256), 0, 1, tokens, positions, rows, d, tok, pos, x);
  });
}

template <class T>
__global__ void __launch_bounds__(256) embed_stats_kernel(const int32_t* __restrict__ tokens,
                                                          const int32_t* __restrict__ positions, int64_t rows,
                                                          int64_t d, const T* __restrict__ tok,
                                                          const T* __restrict__ pos, float* __restrict__ x,
                                                          RowStats so) {
  PDL_ENTRY();
  __shared__ double red[2][8];
  const int64_t r = blockIdx.x;
  if (r >= rows) return;
  const int64_t t = tokens[r], p = positions[r];
  double s = 0.0, q = 0.0;
  for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
    const float v = to_f(tok[t * d + j]) + to_f(pos[p * d + j]);
    x[r * d + j] = v;
    s += double(v);
    q += double(v) * double(v);
  }
  s = warp_sum_d(s);
  q = warp_sum_d(q);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[0][w] = s;
    red[1][w] = q;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, c = 0.0;
    for (int k = 0; k < 8; ++k) {
      a += red[0][k];
      c += red[1][k];
    }
    so.acc[r * kStatStride] = stat_fix(a, so.ovf);  // the sole producer of these accumulators
    so.acc[r * kStatStride + 1] = stat_fix(c, so.ovf);
  }
  // clear this step's downstream accumulators (the previous step's readers
  // have completed: PDL_ENTRY waited for the predecessor grid)
  for (int64_t k = r * blockDim.x + threadIdx.x; k < so.zero_n; k += rows * blockDim.x) {
    so.zero[k * kStatStride] = 0ull;
    so.zero[k * kStatStride + 1] = 0ull;
  }
}

template <class T>
void launch_embed_stats(Ctx& c, const int32_t* tokens, const int32_t* positions, int64_t rows, int64_t d,
                        const T* tok, const T* pos, float* x, RowStats so) {
  if (rows <= 0) return;
  c.launch("embed", double(rows) * d * (2 * sizeof(T) + 4), 0, [&] {
    launch_kernel(c, embed_stats_kernel<T>, dim3(rows), dim3(256), 0, 1, tokens, positions, rows, d, tok, pos, x, so);
  });
}

template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  if (w == 0) {
    t = l < NT / 32 ? red[l] : 0.f;
    t = warp_sum(t);
    if (l == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// One CTA per row; the row is cached in registers (d <= 256 * 32).
template <class T>
__global__ void __launch_bounds__(256) layernorm_kernel(const float* __restrict__ x, int64_t rows, int64_t d,
                                                        const float* __restrict__ g, const float* __restrict__ b,
                                                        T* __restrict__ y, const int32_t* __restrict__ gather,
                                                        const float* __restrict__ head, float* __restrict__ head_out) {
  PDL_ENTRY();
  __shared__ float red[32];
  const int64_t r = blockIdx.x;
  const int64_t src = gather ? gather[r] : r;
  const float* xr = x + src * d;
  constexpr int MAXV = 32;
  float v[MAXV];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int64_t j = threadIdx.x + int64_t(i) * 256;
    v[i] = j < d ? xr[j] : 0.f;
    s += v[i];
  }
  const float mu = block_sum<256>(s, red) / float(d);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int64_t j = threadIdx.x + int64_t(i) * 256;
    if (j < d) q += (v[i] - mu) * (v[i] - mu);
  }
  const float var = block_sum<256>(q, red) / float(d);
  const float is = 1.0f / sqrtf(var + 1e-5f);
  float hd = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int64_t j = threadIdx.x + int64_t(i) * 256;
    if (j < d) {
      const float o = g[j] * ((v[i] - mu) * is) + b[j];
      if (y) y[r * d + j] = from_f<T>(o);
      if (head) hd += o * head[j];
    }
  }
  if (head) {
    hd = block_sum<256>(hd, red);
    if (threadIdx.x == 0) head_out[r] = hd;
  }
}

// Warp-per-row variant for d <= 1024 (8 rows per 256-thread CTA): the
// decode step's LayerNorms are 64-row launches where a CTA per row wastes
// three block barriers per row.
// Warp per row, float4 (d % 4 == 0, d <= 1024: up to 8 float4 per lane, all
// loads issued before the reductions); 8-byte stores of 4 T values.
template <class T>
__global__ void __launch_bounds__(256) layernorm_warp4_kernel(const float* __restrict__ x, int64_t rows, int64_t d,
                                                              const float* __restrict__ g, const float* __restrict__ b,
                                                              T* __restrict__ y, const int32_t* __restrict__ gather,
                                                              const float* __restrict__ head,
                                                              float* __restrict__ head_out) {
  // gamma / beta / head are shared by the CTA's 8 rows: staged in shared memory
  // while the row loads are in flight (they would otherwise be a dependent
  // L2 round trip after the reductions)
  __shared__ float4 sg[256], sb[256], sh4[256];
  const int d4 = int(d >> 2);
  for (int k = threadIdx.x; k < d4; k += 256) {  // parameters: not produced upstream
    sg[k] = reinterpret_cast<const float4*>(g)[k];
    sb[k] = reinterpret_cast<const float4*>(b)[k];
    if (head) sh4[k] = reinterpret_cast<const float4*>(head)[k];
  }
  PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t r = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const bool live = r < rows;
  const int64_t src = live ? (gather ? gather[r] : r) : 0;
  const float4* xr = reinterpret_cast<const float4*>(x + src * d);
  float4 v[8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int j4 = lane + i * 32;
    v[i] = (live && j4 < d4) ? xr[j4] : make_float4(0.f, 0.f, 0.f, 0.f);
    s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
  __syncthreads();  // staged parameters visible
  if (!live) return;
  const float mu = warp_sum(s) / float(d);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (lane + i * 32 < d4) {
      const float c0 = v[i].x - mu, c1 = v[i].y - mu, c2 = v[i].z - mu, c3 = v[i].w - mu;
      q += (c0 * c0 + c1 * c1) + (c2 * c2 + c3 * c3);
    }
  const float is = 1.0f / sqrtf(warp_sum(q) / float(d) + 1e-5f);
  float hd = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int j4 = lane + i * 32;
    if (j4 < d4) {
      const float4 gg = sg[j4], bb = sb[j4];
      const float o0 = gg.x * ((v[i].x - mu) * is) + bb.x, o1 = gg.y * ((v[i].y - mu) * is) + bb.y;
      const float o2 = gg.z * ((v[i].z - mu) * is) + bb.z, o3 = gg.w * ((v[i].w - mu) * is) + bb.w;
      if (y) {
        if constexpr (std::is_same_v<T, bf16>) {
          __nv_bfloat162 lo = __floats2bfloat162_rn(o0, o1), hi = __floats2bfloat162_rn(o2, o3);
          uint2 u;
          u.x = *reinterpret_cast<uint32_t*>(&lo);
          u.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(y + r * d + 4 * j4) = u;
        } else {
          *reinterpret_cast<float4*>(y + r * d + 4 * j4) = make_float4(o0, o1, o2, o3);
        }
      }
      if (head) {
        const float4 hh = sh4[j4];
        hd += (o0 * hh.x + o1 * hh.y) + (o2 * hh.z + o3 * hh.w);
      }
    }
  }
  if (head) {
    hd = warp_sum(hd);
    if (lane == 0) head_out[r] = hd;
  }
}

template <class T>
__global__ void __launch_bounds__(256) layernorm_warp_kernel(const float* __restrict__ x, int64_t rows, int64_t d,
                                                             const float* __restrict__ g, const float* __restrict__ b,
                                                             T* __restrict__ y, const int32_t* __restrict__ gather,
                                                             const float* __restrict__ head,
                                                             float* __restrict__ head_out) {
  PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int64_t r = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int64_t src = gather ? gather[r] : r;
  const float* xr = x + src * d;
  constexpr int MAXV = 32;
  float v[MAXV];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int64_t j = lane + int64_t(i) * 32;
    v[i] = j < d ? xr[j] : 0.f;
    s += v[i];
  }
  const float mu = warp_sum(s) / float(d);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int64_t j = lane + int64_t(i) * 32;
    if (j < d) q += (v[i] - mu) * (v[i] - mu);
  }
  const float var = warp_sum(q) / float(d);
  const float is = 1.0f / sqrtf(var + 1e-5f);
  float hd = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int64_t j = lane + int64_t(i) * 32;
    if (j < d) {
      const float o = g[j] * ((v[i] - mu) * is) + b[j];
      if (y) y[r * d + j] = from_f<T>(o);
      if (head) hd += o * head[j];
    }
  }
  if (head) {
    hd = warp_sum(hd);
    if (lane == 0) head_out[r] = hd;
  }
}

// Wide rows (1024 < d <= 8192, d % 1024 == 0 via VPT float4 per thread): CTA
// of 256 threads per row, every load issued before the first reduction,
// two-pass statistics from registers, 8- / 16-byte stores.
template <class T, int VPT>
__global__ void __launch_bounds__(256) layernorm_wide_kernel(const float* __restrict__ x, int64_t d,
                                                             const float* __restrict__ g, const float* __restrict__ b,
                                                             T* __restrict__ y, const int32_t* __restrict__ gather,
                                                             const float* __restrict__ head,
                                                             float* __restrict__ head_out) {
  PDL_ENTRY();
  __shared__ float red[32];
  const int64_t r = blockIdx.x;
  const int64_t src = gather ? gather[r] : r;
  const float4* xr = reinterpret_cast<const float4*>(x + src * d);
  float4 v[VPT];
#pragma unroll
  for (int i = 0; i < VPT; ++i) v[i] = __ldg(xr + threadIdx.x + i * 256);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  const float mu = block_sum<256>(s, red) / float(d);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const float a = v[i].x - mu, bq = v[i].y - mu, c = v[i].z - mu, e = v[i].w - mu;
    q += (a * a + bq * bq) + (c * c + e * e);
  }
  const float is = 1.0f / sqrtf(block_sum<256>(q, red) / float(d) + 1e-5f);
  float hd = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int j = (threadIdx.x + i * 256) * 4;
    const float4 gg = __ldg(reinterpret_cast<const float4*>(g + j)), bb = __ldg(reinterpret_cast<const float4*>(b + j));
    const float o0 = gg.x * ((v[i].x - mu) * is) + bb.x, o1 = gg.y * ((v[i].y - mu) * is) + bb.y;
    const float o2 = gg.z * ((v[i].z - mu) * is) + bb.z, o3 = gg.w * ((v[i].w - mu) * is) + bb.w;
    if (y) {
      if constexpr (sizeof(T) == 2) {
        __nv_bfloat162 p0 = __floats2bfloat162_rn(o0, o1), p1 = __floats2bfloat162_rn(o2, o3);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&p0);
        u.y = *reinterpret_cast<uint32_t*>(&p1);
        *reinterpret_cast<uint2*>(y + r * d + j) = u;
      } else {
        *reinterpret_cast<float4*>(y + r * d + j) = make_float4(o0, o1, o2, o3);
      }
    }
    if (head) {
      const float4 hh = __ldg(reinterpret_cast<const float4*>(head + j));
      hd += o0 * hh.x + o1 * hh.y + o2 * hh.z + o3 * hh.w;
    }
  }
  if (head) {
    hd = block_sum<256>(hd, red);
    if (threadIdx.x == 0) head_out[r] = hd;
  }
}

// Mixed decode: LayerNorm of a row (fp32, two-pass statistics in fp64) written as
// two bf16 planes, y[r, j] = hi, y[r, d + j] = lo (the consumer GEMM TMAs both).
// EmbedIn (decode step start): x[r] = tok_embed[tokens[r]] + pos_embed[positions[r]] is
// computed here and written out, then normalised — one launch instead of embed + LayerNorm.
struct EmbedIn {
  const int32_t* tokens = nullptr;
  const int32_t* positions = nullptr;
  const bf16* tok = nullptr;
  const bf16* pos = nullptr;
};

__global__ void layernorm_split_kernel(const float* __restrict__ x, int64_t d, const float* __restrict__ g,
                                       const float* __restrict__ b, bf16* __restrict__ y,
                                       const int32_t* __restrict__ gather, EmbedIn em) {
  pdl_entry_small_grid();
  __shared__ double red[32];
  const int64_t r = blockIdx.x;
  const int64_t src = gather ? gather[r] : r;
  const int nw = (blockDim.x + 31) >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = threadIdx.x * 4;
  const bool act = j < d;
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (em.tokens) {
    if (act) {
      const int64_t t = em.tokens[r], p = em.positions[r];
      const uint2 a = *reinterpret_cast<const uint2*>(em.tok + t * d + j);
      const uint2 c = *reinterpret_cast<const uint2*>(em.pos + p * d + j);
      const float2 a0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&a.x));
      const float2 a1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&a.y));
      const float2 c0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&c.x));
      const float2 c1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&c.y));
      v = make_float4(a0.x + c0.x, a0.y + c0.y, a1.x + c1.x, a1.y + c1.y);
      *reinterpret_cast<float4*>(const_cast<float*>(x) + r * d + j) = v;
    }
  } else if (act) {
    v = *reinterpret_cast<const float4*>(x + src * d + j);
  }
  double s = warp_sum_d(double(v.x) + v.y + v.z + v.w);
  if (lane == 0) red[w] = s;
  __syncthreads();
  double mu = 0.0;
  for (int k = 0; k < nw; ++k) mu += red[k];
  mu /= double(d);
  __syncthreads();
  const double c0 = v.x - mu, c1 = v.y - mu, c2 = v.z - mu, c3 = v.w - mu;
  double q = warp_sum_d(act ? c0 * c0 + c1 * c1 + c2 * c2 + c3 * c3 : 0.0);
  if (lane == 0) red[w] = q;
  __syncthreads();
  double var = 0.0;
  for (int k = 0; k < nw; ++k) var += red[k];
  const double is = 1.0 / sqrt(var / double(d) + 1e-5);
  if (!act) return;
  const float4 gg = *reinterpret_cast<const float4*>(g + j), bb = *reinterpret_cast<const float4*>(b + j);
  const float o[4] = {float(gg.x * (c0 * is) + bb.x), float(gg.y * (c1 * is) + bb.y), float(gg.z * (c2 * is) + bb.z),
                      float(gg.w * (c3 * is) + bb.w)};
  bf16 hi[4], lo[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    hi[e] = __float2bfloat16_rn(o[e]);
    lo[e] = __float2bfloat16_rn(o[e] - __bfloat162float(hi[e]));
  }
  *reinterpret_cast<uint2*>(y + r * 2 * d + j) = *reinterpret_cast<const uint2*>(hi);
  *reinterpret_cast<uint2*>(y + r * 2 * d + d + j) = *reinterpret_cast<const uint2*>(lo);
}

// Many rows (prefill / scoring): a warp per row, the row's NV float4 per lane
// loaded up front, shuffle-only fp64 reductions (the same two-pass statistics).
template <int NV>
__global__ void __launch_bounds__(256) layernorm_split_warp_kernel(const float* __restrict__ x, int64_t rows, int64_t d,
                                                                   const float* __restrict__ g,
                                                                   const float* __restrict__ b, bf16* __restrict__ y,
                                                                   const int32_t* __restrict__ gather) {
  pdl_entry_small_grid();
  const int lane = threadIdx.x & 31;
  const int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int64_t src = gather ? gather[r] : r;
  const float4* xr = reinterpret_cast<const float4*>(x + src * d);
  float4 v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = __ldcs(xr + lane + 32 * k);  // read once: streaming
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < NV; ++k) s += double(v[k].x) + v[k].y + v[k].z + v[k].w;
  const double mu = warp_sum_d(s) / double(d);
  double q = 0.0;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double c0 = v[k].x - mu, c1 = v[k].y - mu, c2 = v[k].z - mu, c3 = v[k].w - mu;
    q += c0 * c0 + c1 * c1 + c2 * c2 + c3 * c3;
  }
  const double is = 1.0 / sqrt(warp_sum_d(q) / double(d) + 1e-5);
  bf16* yr = y + r * 2 * d;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int j = 4 * (lane + 32 * k);
    const float4 gg = __ldg(reinterpret_cast<const float4*>(g + j)), bb = __ldg(reinterpret_cast<const float4*>(b + j));
    const float o[4] = {float(gg.x * ((v[k].x - mu) * is) + bb.x), float(gg.y * ((v[k].y - mu) * is) + bb.y),
                        float(gg.z * ((v[k].z - mu) * is) + bb.z), float(gg.w * ((v[k].w - mu) * is) + bb.w)};
    bf16 hi[4], lo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      hi[e] = __float2bfloat16_rn(o[e]);
      lo[e] = __float2bfloat16_rn(o[e] - __bfloat162float(hi[e]));
    }
    *reinterpret_cast<uint2*>(yr + j) = *reinterpret_cast<const uint2*>(hi);
    *reinterpret_cast<uint2*>(yr + d + j) = *reinterpret_cast<const uint2*>(lo);
  }
}

void launch_layernorm_split(Ctx& c, const float* x, int64_t rows, int64_t d, const float* g, const float* b, bf16* y,
                            const int32_t* gather) {
  if (rows <= 0) return;
  if (d % 4 || d > 4096) throw ContractError("layernorm (split planes): d % 4 == 0 and d <= 4096 required");
  // (decode batches keep the CTA-per-row kernel: its 4-element fp64 chains are
  // shorter — a warp per row measured 61 -> 102 us per C2 decode step)
  if (rows >= 1024 && (d == 768 || d == 1024 || d == 2048)) {
    auto k = d == 768    ? layernorm_split_warp_kernel<6>
             : d == 1024 ? layernorm_split_warp_kernel<8>
                         : layernorm_split_warp_kernel<16>;
    const int wpb = 8;
    c.launch("layernorm", double(rows) * d * 8, 0, [&] {
      launch_kernel(c, k, dim3(unsigned(ceil_div(rows, wpb))), dim3(32 * wpb), 0, 1, x, rows, d, g, b, y, gather);
    });
    return;
  }
  const int th = int((d / 4 + 31) / 32 * 32);
  c.launch("layernorm", double(rows) * d * 8, 0, [&] {
    launch_kernel(c, layernorm_split_kernel, dim3(rows), dim3(th), 0, 1, x, d, g, b, y, gather, EmbedIn{});
  });
}

// Decode step start (mixed planes): embedding sum written to x and its split
// LayerNorm planes in one launch (embed_kernel's arithmetic: bf16 -> fp32, one add).
void launch_embed_layernorm_split(Ctx& c, const int32_t* tokens, const int32_t* positions, int64_t rows, int64_t d,
                                  const bf16* tok, const bf16* pos, float* x, const float* g, const float* b, bf16* y) {
  if (rows <= 0) return;
  if (d % 4 || d > 4096) throw ContractError("embed + layernorm (split planes): d % 4 == 0 and d <= 4096 required");
  const int th = int((d / 4 + 31) / 32 * 32);
  EmbedIn em;
  em.tokens = tokens;
  em.positions = positions;
  em.tok = tok;
  em.pos = pos;
  c.launch("layernorm", double(rows) * d * 12, 0, [&] {
    launch_kernel(c, layernorm_split_kernel, dim3(rows), dim3(th), 0, 1, x, d, g, b, y, nullptr, em);
  });
}

// CTA-per-row float4 variant for few rows (decode): one float4 per thread,
// two barrier-reductions — short dependency chains on many SMs.
template <class T>
__global__ void layernorm_vec_kernel(const float* __restrict__ x, int64_t d, const float* __restrict__ g,
                                     const float* __restrict__ b, T* __restrict__ y,
                                     const int32_t* __restrict__ gather, const float* __restrict__ head,
                                     float* __restrict__ head_out) {
  PDL_ENTRY();
  __shared__ float red[2][32];
  const int64_t r = blockIdx.x;
  const int64_t src = gather ? gather[r] : r;
  const int j = threadIdx.x * 4;
  const bool act = j < d;
  float4 v = act ? *reinterpret_cast<const float4*>(x + src * d + j) : make_float4(0.f, 0.f, 0.f, 0.f);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
  float s = warp_sum(v.x + v.y + v.z + v.w);
  if (lane == 0) red[0][w] = s;
  __syncthreads();
  float mu = 0.f;
  for (int k = 0; k < nw; ++k) mu += red[0][k];
  mu /= float(d);
  const float4 c = make_float4(v.x - mu, v.y - mu, v.z - mu, v.w - mu);
  float q = act ? c.x * c.x + c.y * c.y + c.z * c.z + c.w * c.w : 0.f;
  q = warp_sum(q);
  if (lane == 0) red[1][w] = q;
  __syncthreads();
  float var = 0.f;
  for (int k = 0; k < nw; ++k) var += red[1][k];
  const float is = 1.0f / sqrtf(var / float(d) + 1e-5f);
  if (act) {
    const float4 gg = *reinterpret_cast<const float4*>(g + j), bb = *reinterpret_cast<const float4*>(b + j);
    const float o0 = gg.x * (c.x * is) + bb.x, o1 = gg.y * (c.y * is) + bb.y, o2 = gg.z * (c.z * is) + bb.z,
                o3 = gg.w * (c.w * is) + bb.w;
    if (y) {
      T* yr = y + r * d + j;
      yr[0] = from_f<T>(o0);
      yr[1] = from_f<T>(o1);
      yr[2] = from_f<T>(o2);
      yr[3] = from_f<T>(o3);
    }
    if (head) {
      const float4 hh = *reinterpret_cast<const float4*>(head + j);
      s = o0 * hh.x + o1 * hh.y + o2 * hh.z + o3 * hh.w;
    }
  } else {
    s = 0.f;
  }
  if (head) {
    __syncthreads();
    s = warp_sum(s);
    if (lane == 0) red[0][w] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int k = 0; k < nw; ++k) t += red[0][k];
      head_out[r] = t;
    }
  }
}

// Decode-step head: x[r] = tok[tokens[r]] + pos[positions[r]] (src/model.cpp:290-295)
// and y[r] = LN1(x[r]) (src/model.cpp:387-400) in one CTA-per-row float4 pass.
template <class T>
__global__ void embed_layernorm_kernel(const int32_t* __restrict__ tokens, const int32_t* __restrict__ positions,
                                       int64_t d, const T* __restrict__ tok, const T* __restrict__ pos,
                                       float* __restrict__ x, const float* __restrict__ g, const float* __restrict__ b,
                                       T* __restrict__ y) {
  PDL_ENTRY();
  __shared__ float red[2][32];
  const int64_t r = blockIdx.x;
  const int64_t t = tokens[r], p = positions[r];
  const int j = threadIdx.x * 4;
  const bool act = j < d;
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (act) {
    v = make_float4(to_f(tok[t * d + j]) + to_f(pos[p * d + j]), to_f(tok[t * d + j + 1]) + to_f(pos[p * d + j + 1]),
                    to_f(tok[t * d + j + 2]) + to_f(pos[p * d + j + 2]),
                    to_f(tok[t * d + j + 3]) + to_f(pos[p * d + j + 3]));
    *reinterpret_cast<float4*>(x + r * d + j) = v;
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
  float s = warp_sum(v.x + v.y + v.z + v.w);
  if (lane == 0) red[0][w] = s;
  __syncthreads();
  float mu = 0.f;
  for (int k = 0; k < nw; ++k) mu += red[0][k];
  mu /= float(d);
  const float4 c = make_float4(v.x - mu, v.y - mu, v.z - mu, v.w - mu);
  float q = act ? c.x * c.x + c.y * c.y + c.z * c.z + c.w * c.w : 0.f;
  q = warp_sum(q);
  if (lane == 0) red[1][w] = q;
  __syncthreads();
  float var = 0.f;
  for (int k = 0; k < nw; ++k) var += red[1][k];
  const float is = 1.0f / sqrtf(var / float(d) + 1e-5f);
  if (act) {
    const float4 gg = *reinterpret_cast<const float4*>(g + j), bb = *reinterpret_cast<const float4*>(b + j);
    T* yr = y + r * d + j;
    yr[0] = from_f<T>(gg.x * (c.x * is) + bb.x);
    yr[1] = from_f<T>(gg.y * (c.y * is) + bb.y);
    yr[2] = from_f<T>(gg.z * (c.z * is) + bb.z);
    yr[3] = from_f<T>(gg.w * (c.w * is) + bb.w);
  }
}

template <class T>
bool launch_embed_layernorm(Ctx& c, const int32_t* tokens, const int32_t* positions, int64_t rows, int64_t d,
                            const T* tok, const T* pos, float* x, const float* g, const float* b, T* y) {
  if (rows <= 0) return true;
  if (d % 4 || d > 4096) return false;
  const int th = int((d / 4 + 31) / 32 * 32);
  c.launch("layernorm", double(rows) * d * (2 * sizeof(T) + 4 + sizeof(T)), 0, [&] {
    launch_kernel(c, embed_layernorm_kernel<T>, dim3(rows), dim3(th), 0, 1, tokens, positions, d, tok, pos, x, g, b,
                  y);
  });
  return true;
}

template <class T>
void launch_layernorm(Ctx& c, const float* x, int64_t rows, int64_t d, const float* g, const float* b, T* y,
                      const int32_t* gather, const float* head, float* head_out) {
  if (rows <= 0) return;
  if (d > 256 * 32) throw ContractError("layernorm: d_model above 8192 unsupported");
  c.launch("layernorm", double(rows) * d * (4 + (y ? sizeof(T) : 0)), 0, [&] {
    if (d % 4 == 0 && d <= 4096 && rows <= 1024) {
      const int th = int((d / 4 + 31) / 32 * 32);
      launch_kernel(c, layernorm_vec_kernel<T>, dim3(rows), dim3(th), 0, 1, x, d, g, b, y, gather, head, head_out);
    } else if (d <= 1024) {
      if (d % 4 == 0) {
        launch_kernel(c, layernorm_warp4_kernel<T>, dim3(ceil_div(rows, 8)), dim3(256), 0, 1, x, rows, d, g, b, y,
                      gather, head, head_out);
      } else {
        launch_kernel(c, layernorm_warp_kernel<T>, dim3(ceil_div(rows, 8)), dim3(256), 0, 1, x, rows, d, g, b, y,
                      gather, head, head_out);
      }
    } else if (d % 1024 == 0 && d <= 8192) {
      auto go = [&](auto kern) {
        launch_kernel(c, kern, dim3(rows), dim3(256), 0, 1, x, d, g, b, y, gather, head, head_out);
      };
      switch (d / 1024) {
        case 2: go(layernorm_wide_kernel<T, 2>); break;
        case 3: go(layernorm_wide_kernel<T, 3>); break;
        case 4: go(layernorm_wide_kernel<T, 4>); break;
        case 5: go(layernorm_wide_kernel<T, 5>); break;
        case 6: go(layernorm_wide_kernel<T, 6>); break;
        case 7: go(layernorm_wide_kernel<T, 7>); break;
        default: go(layernorm_wide_kernel<T, 8>); break;
      }
    } else {
      launch_kernel(c, layernorm_kernel<T>, dim3(rows), dim3(256), 0, 1, x, rows, d, g, b, y, gather, head, head_out);
    }
  });
}

template <class T>
__global__ void kv_scatter_kernel(const T* __restrict__ qkv, int64_t rows, int64_t d,
                                  const int32_t* __restrict__ seq_of_row, const int32_t* __restrict__ pos_of_row,
                                  const int32_t* __restrict__ block_table, int layer, KvGeom g, T* __restrict__ kv) {
  PDL_ENTRY();
  const int64_t r = blockIdx.x;
  if (r >= rows) return;
  const int64_t s = seq_of_row[r], p = pos_of_row[r];
  const int64_t page = block_table[s * g.max_pages_per_seq + p / g.page_size];
  const int64_t slot = p % g.page_size;
  constexpr int E = 16 / int(sizeof(T));  // elements per 16-byte chunk
  if (g.DH % E == 0 && d % E == 0) {
    // 16-byte chunks: a head's K (or V) row is DH contiguous elements in both layouts
    const int dc = int(d / E), hc = int(g.DH / E);
    const uint4* src = reinterpret_cast<const uint4*>(qkv + r * 3 * d + d);
    for (int j = threadIdx.x; j < 2 * dc; j += blockDim.x) {
      const int which = j / dc, cc = j - which * dc, h = cc / hc, i = cc - h * hc;
      const int64_t dst = ((((int64_t)layer * g.n_pages + page) * 2 + which) * g.H + h) * g.page_size * g.DH +
                          slot * g.DH + int64_t(i) * E;
      *reinterpret_cast<uint4*>(kv + dst) = src[j];
    }
    return;
  }
  for (int64_t j = threadIdx.x; j < 2 * d; j += blockDim.x) {
    const int64_t which = j / d, col = j % d, h = col / g.DH, i = col % g.DH;
    const int64_t dst = ((((int64_t)layer * g.n_pages + page) * 2 + which) * g.H + h) * g.page_size * g.DH +
                        slot * g.DH + i;
    kv[dst] = qkv[r * 3 * d + d + j];
  }
}

template <class T>
void launch_kv_scatter(Ctx& c, const T* qkv, int64_t rows, int64_t d, const int32_t* seq_of_row,
                       const int32_t* pos_of_row, const int32_t* block_table, int layer, const KvGeom& g, T* kv) {
  if (rows <= 0) return;
  c.launch("kv_scatter", double(rows) * 2 * d * sizeof(T) * 2, 0, [&] {
    launch_kernel(c, kv_scatter_kernel<T>, dim3(rows), dim3(256), 0, 1, qkv, rows, d, seq_of_row, pos_of_row, block_table, layer, g,
                                                     kv);
  });
}

__device__ __forceinline__ float load_any(const void* p, int dt, int64_t i) {
  if (dt == 0) return static_cast<const float*>(p)[i];
  if (dt == 1) return __bfloat162float(static_cast<const bf16*>(p)[i]);
  return float(static_cast<const double*>(p)[i]);
}

__global__ void convert_kernel(const void* src, int sdt, void* dst, int ddt, int64_t rows, int64_t cols,
                               bool transpose, int64_t dst_ld, int64_t dst_row0) {
  PDL_ENTRY();
  const int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    // e indexes the destination in [dst_rows, dst_cols] order.
    int64_t dr, dc, si;
    if (transpose) {  // dst [cols, rows]
      dr = e / rows;
      dc = e % rows;
      si = dc * cols + dr;
    } else {
      dr = e / cols;
      dc = e % cols;
      si = e;
    }
    const float v = load_any(src, sdt, si);
    const int64_t di = (dst_row0 + dr) * dst_ld + dc;
    if (ddt == 0)
      static_cast<float*>(dst)[di] = v;
    else
      static_cast<bf16*>(dst)[di] = __float2bfloat16_rn(v);
  }
}

// IndexError check for device-resident token ids: the first position whose id is
// outside [0, V) (atomicMin over positions; n when all are valid).
__global__ void validate_tokens_kernel(const int32_t* __restrict__ t, int64_t n, int64_t V,
                                       unsigned long long* __restrict__ first_bad) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    if (t[i] < 0 || t[i] >= V) atomicMin(first_bad, static_cast<unsigned long long>(i));
}

void check_tokens(Ctx& c, const int32_t* tokens, int64_t n, int64_t V, int where, const char* what) {
  auto fail = [&](int64_t i, int32_t v) {
    throw IndexError(std::string(what) + ": token id " + std::to_string(v) + " at position " + std::to_string(i) +
                     " out of range [0," + std::to_string(V) + ")");
  };
  if (n <= 0) return;
  if (where == 0) {
    for (int64_t i = 0; i < n; ++i)
      if (tokens[i] < 0 || tokens[i] >= V) fail(i, tokens[i]);
    return;
  }
  auto* fb = static_cast<unsigned long long*>(c.workspace("validate.first_bad", 16));
  const unsigned long long init = static_cast<unsigned long long>(n);
  PPOEXP_CUDA(cudaMemcpyAsync(fb, &init, 8, cudaMemcpyHostToDevice, c.stream));
  c.launch("validate", 4.0 * n, 0, [&] {
    launch_kernel(c, validate_tokens_kernel, dim3(std::min<int64_t>(ceil_div(n, 256), 592)), dim3(256), 0, 1, tokens, n,
                  V, fb);
  });
  unsigned long long first = 0;
  PPOEXP_CUDA(cudaMemcpyAsync(&first, fb, 8, cudaMemcpyDeviceToHost, c.stream));
  PPOEXP_CUDA(cudaStreamSynchronize(c.stream));
  if (first < init) {
    int32_t v = 0;
    PPOEXP_CUDA(cudaMemcpy(&v, tokens + first, 4, cudaMemcpyDeviceToHost));
    fail(int64_t(first), v);
  }
}

void launch_convert(Ctx& c, const void* src, int src_dtype, void* dst, int dst_dtype, int64_t rows, int64_t cols,
                    bool transpose, int64_t dst_ld, int64_t dst_row0) {
  if (rows * cols <= 0) return;
  const int64_t blocks = std::min<int64_t>(ceil_div(rows * cols, 256), 148 * 16);
  c.launch("convert", 0, 0, [&] {
    launch_kernel(c, convert_kernel, dim3(blocks), dim3(256), 0, 1, src, src_dtype, dst, dst_dtype, rows, cols, transpose, dst_ld,
                                                 dst_row0);
  });
}

__global__ void scripted_reward_kernel(int64_t B, int64_t stride, const int32_t* tokens, const int64_t* lengths,
                                       int32_t target, double* out) {
  PDL_ENTRY();
  const int64_t b = blockIdx.x;
  if (b >= B) return;
  int n = 0;
  for (int64_t t = threadIdx.x; t < lengths[b]; t += blockDim.x) n += tokens[b * stride + t] == target;
  n = __reduce_add_sync(0xffffffffu, n);
  if (threadIdx.x == 0) out[b] = double(n);
}

// CriticJob::scripted_reward_for, src/ppo.cpp:109-115 (count over the response).
void launch_scripted_reward(Ctx& c, int64_t B, int64_t stride, const int32_t* tokens, const int64_t* lengths,
                            int32_t target, double* out) {
  if (B <= 0) return;
  c.launch("scripted_reward", 0, 0, [&] {
    launch_kernel(c, scripted_reward_kernel, dim3(B), dim3(32), 0, 1, B, stride, tokens, lengths, target, out);
  });
}

__global__ void f32_to_f64_kernel(const float* src, int64_t n, double* dst) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = double(src[i]);
}

void launch_f32_to_f64(Ctx& c, const float* src, int64_t n, double* dst) {
  if (n <= 0) return;
  c.launch("convert", 12.0 * n, 0, [&] {
    launch_kernel(c, f32_to_f64_kernel, dim3(std::min<int64_t>(ceil_div(n, 256), 1184)), dim3(256), 0, 1, src, n, dst);
  });
}

__global__ void fill_i32_kernel(int32_t* dst, int64_t n, int32_t v) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = v;
}

void launch_fill_i32(Ctx& c, int32_t* dst, int64_t n, int32_t v) {
  if (n <= 0) return;
  c.launch("fill", 4.0 * n, 0, [&] {
    launch_kernel(c, fill_i32_kernel, dim3(std::min<int64_t>(ceil_div(n, 256), 1184)), dim3(256), 0, 1, dst, n, v);
  });
}

#define INST(T)                                                                                                   \
  template void launch_embed_stats<T>(Ctx&, const int32_t*, const int32_t*, int64_t, int64_t, const T*, const T*, \
                                      float*, RowStats);                                                         \
  template void launch_embed<T>(Ctx&, const int32_t*, const int32_t*, int64_t, int64_t, const T*, const T*,      \
                                float*);                                                                        \
  template bool launch_embed_layernorm<T>(Ctx&, const int32_t*, const int32_t*, int64_t, int64_t, const T*,      \
                                         const T*, float*, const float*, const float*, T*);                      \
  template void launch_layernorm<T>(Ctx&, const float*, int64_t, int64_t, const float*, const float*, T*,       \
                                    const int32_t*, const float*, float*);                                      \
  template void launch_kv_scatter<T>(Ctx&, const T*, int64_t, int64_t, const int32_t*, const int32_t*,          \
                                     const int32_t*, int, const KvGeom&, T*);
INST(float)
INST(bf16)
#undef INST

}  // namespace ppx
