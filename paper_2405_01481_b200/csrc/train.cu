// train.cu — the train side that consumes the experience (SURVEY.md §8f rows
// 2-4): one device trainer per model with fp32 master weights in the
// reference layout, a recorded fp32 forward (embedding, LayerNorm, GELU,
// causal attention, tied LM head / scalar head), its exact backward, and
// AdamW (src/optim.cpp:32-55).  The losses are the reference's:
//   PPO actor   ppo_actor_loss  (src/losses.cpp:201-214; src/ppo.cpp:395-424)
//   critic      ppo_critic_loss (src/losses.cpp:216-231; src/ppo.cpp:195-231)
//   DPO family  dpo_family_loss (src/losses.cpp:129-166; src/trainers.cpp:54-80)
// computed in fp64 on the host from the device log-probs / values (a few
// numbers per sequence); their gradients flow back through the device graph.
//
// GEMMs are plain row-major fp32 library GEMMs (cuBLAS, pedantic fp32 math:
// no TF32), the rest are kernels here.  After a step, refit() copies the
// master weights into the serving model in place (Engine::refit semantics,
// src/engine.cpp:60-90: same buffers, captured graphs stay valid).
#include <cublas_v2.h>

#include <cmath>
#include <cstring>

#include "train.hpp"

namespace ppx {

namespace {

void blas_check(cublasStatus_t s, const char* what) {
  if (s != CUBLAS_STATUS_SUCCESS) throw Error(6, std::string("cublas: ") + what + " failed (" + std::to_string(int(s)) + ")");
}

// ---------------------------------------------------------------- kernels
__global__ void t_embed_fwd(const int32_t* __restrict__ tok, const int32_t* __restrict__ pos, int64_t M, int64_t d,
                            const float* __restrict__ E, const float* __restrict__ P, float* __restrict__ x) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M * d; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / d, j = i % d;
    x[i] = E[int64_t(tok[r]) * d + j] + P[int64_t(pos[r]) * d + j];
  }
}

__global__ void t_embed_bwd(const int32_t* __restrict__ tok, const int32_t* __restrict__ pos, int64_t M, int64_t d,
                            const float* __restrict__ dx, float* __restrict__ dE, float* __restrict__ dP) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < M * d; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / d, j = i % d;
    atomicAdd(dE + int64_t(tok[r]) * d + j, dx[i]);
    atomicAdd(dP + int64_t(pos[r]) * d + j, dx[i]);
  }
}

// LayerNorm (src/tensor.cpp:594-624): two-pass mean / variance in fp64, eps 1e-5
__global__ void t_ln_fwd(const float* __restrict__ x, int64_t d, const float* __restrict__ g,
                         const float* __restrict__ b, float* __restrict__ y, float* __restrict__ mu_out,
                         float* __restrict__ rs_out) {
  __shared__ double red[32];
  const int64_t r = blockIdx.x;
  const float* xr = x + r * d;
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < d; j += blockDim.x) s += xr[j];
  s = warp_sum_d(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    t = warp_sum_d(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const double mu = red[0] / double(d);
  __syncthreads();
  double q = 0.0;
  for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
    const double c = xr[j] - mu;
    q += c * c;
  }
  q = warp_sum_d(q);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = q;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    t = warp_sum_d(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const double rs = 1.0 / sqrt(red[0] / double(d) + 1e-5);
  for (int64_t j = threadIdx.x; j < d; j += blockDim.x) y[r * d + j] = float(g[j] * ((xr[j] - mu) * rs) + b[j]);
  if (threadIdx.x == 0) {
    mu_out[r] = float(mu);
    rs_out[r] = float(rs);
  }
}

// dx += rs (dh - mean(dh) - xhat mean(dh xhat)), dh = dy * gamma (src/tensor.cpp:627-655)
__global__ void t_ln_bwd_x(const float* __restrict__ x, const float* __restrict__ dy, int64_t d,
                           const float* __restrict__ g, const float* __restrict__ mu, const float* __restrict__ rs,
                           float* __restrict__ dx) {
  __shared__ double red[2][32];
  const int64_t r = blockIdx.x;
  const float m = mu[r], s = rs[r];
  double m1 = 0.0, m2 = 0.0;
  for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
    const double dh = double(dy[r * d + j]) * g[j];
    const double xh = (double(x[r * d + j]) - m) * s;
    m1 += dh;
    m2 += dh * xh;
  }
  m1 = warp_sum_d(m1);
  m2 = warp_sum_d(m2);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = m1;
    red[1][threadIdx.x >> 5] = m2;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    double a = threadIdx.x < blockDim.x / 32 ? red[0][threadIdx.x] : 0.0;
    double c = threadIdx.x < blockDim.x / 32 ? red[1][threadIdx.x] : 0.0;
    a = warp_sum_d(a);
    c = warp_sum_d(c);
    if (threadIdx.x == 0) {
      red[0][0] = a;
      red[1][0] = c;
    }
  }
  __syncthreads();
  m1 = red[0][0] / double(d);
  m2 = red[1][0] / double(d);
  for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
    const double dh = double(dy[r * d + j]) * g[j];
    const double xh = (double(x[r * d + j]) - m) * s;
    dx[r * d + j] += float(s * (dh - m1 - xh * m2));
  }
}

// dgamma += sum_r dy xhat, dbeta += sum_r dy: one thread per column, rows in order
__global__ void t_ln_bwd_params(const float* __restrict__ x, const float* __restrict__ dy, int64_t M, int64_t d,
                                const float* __restrict__ mu, const float* __restrict__ rs, float* __restrict__ dg,
                                float* __restrict__ db) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j >= d) return;
  double a = 0.0, c = 0.0;
  for (int64_t r = 0; r < M; ++r) {
    const double g = dy[r * d + j];
    a += g * ((double(x[r * d + j]) - mu[r]) * rs[r]);
    c += g;
  }
  dg[j] += float(a);
  db[j] += float(c);
}

__device__ __forceinline__ double gelu_d(double x) {  // src/model.cpp:358-361 and its derivative
  const double kC = 0.7978845608028654, u = kC * (x + 0.044715 * x * x * x);
  const double t = tanh(u);
  return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * kC * (1.0 + 3.0 * 0.044715 * x * x);
}
__device__ __forceinline__ double gelu_v(double x) {
  const double kC = 0.7978845608028654;
  return 0.5 * x * (1.0 + tanh(kC * (x + 0.044715 * x * x * x)));
}

__global__ void t_gelu_fwd(const float* __restrict__ u, int64_t n, float* __restrict__ g) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    g[i] = float(gelu_v(u[i]));
}
__global__ void t_gelu_bwd(const float* __restrict__ u, int64_t n, float* __restrict__ dg) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dg[i] = float(dg[i] * gelu_d(u[i]));
}

__global__ void t_add(float* __restrict__ y, const float* __restrict__ a, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] += a[i];
}

// causal softmax of S[h, i, j] (scale, -1e30 mask above the diagonal; src/model.cpp:198-236), in place
__global__ void t_softmax_causal(float* __restrict__ S, int64_t T, float scale) {
  const int64_t row = blockIdx.x;  // h * T + i
  const int64_t i = row % T;
  float* s = S + row * T;
  __shared__ float red[32];
  float mx = -INFINITY;
  for (int64_t j = threadIdx.x; j <= i; j += blockDim.x) mx = fmaxf(mx, s[j] * scale);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : -INFINITY;
    t = warp_max(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  mx = red[0];
  __syncthreads();
  double sum = 0.0;
  for (int64_t j = threadIdx.x; j <= i; j += blockDim.x) sum += exp(double(s[j] * scale) - double(mx));
  sum = warp_sum_d(sum);
  __shared__ double rd[32];
  if ((threadIdx.x & 31) == 0) rd[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < blockDim.x / 32 ? rd[threadIdx.x] : 0.0;
    t = warp_sum_d(t);
    if (threadIdx.x == 0) rd[0] = t;
  }
  __syncthreads();
  const double inv = 1.0 / rd[0];
  for (int64_t j = threadIdx.x; j < T; j += blockDim.x)
    s[j] = j <= i ? float(exp(double(s[j] * scale) - double(mx)) * inv) : 0.f;
}

// dS = P (dP - sum_k dP P) * scale, in place over dP
__global__ void t_softmax_bwd(const float* __restrict__ P, float* __restrict__ dP, int64_t T, float scale) {
  const int64_t row = blockIdx.x;
  const float* p = P + row * T;
  float* g = dP + row * T;
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < T; j += blockDim.x) s += double(g[j]) * p[j];
  s = warp_sum_d(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    t = warp_sum_d(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const double dot = red[0];
  for (int64_t j = threadIdx.x; j < T; j += blockDim.x) g[j] = float(double(p[j]) * (double(g[j]) - dot) * scale);
}

__global__ void t_gather_rows(const float* __restrict__ src, const int32_t* __restrict__ idx, int64_t R, int64_t d,
                              float* __restrict__ dst) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < R * d; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[int64_t(idx[i / d]) * d + i % d];
}
__global__ void t_scatter_add_rows(const float* __restrict__ src, const int32_t* __restrict__ idx, int64_t R, int64_t d,
                                   float* __restrict__ dst) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < R * d; i += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(dst + int64_t(idx[i / d]) * d + i % d, src[i]);
}

// log_softmax + gather per row (fp64 LSE): lp[r] = l[t] - lse; with dlp != null
// the row becomes dlogits = dlp (onehot(t) - softmax) in place
__global__ void t_lm_rows(float* __restrict__ L, int64_t V, const int32_t* __restrict__ tgt,
                          const double* __restrict__ dlp, double* __restrict__ lp_out) {
  const int64_t r = blockIdx.x;
  float* l = L + r * V;
  __shared__ double red[32];
  __shared__ float fr[32];
  float mx = -INFINITY;
  for (int64_t j = threadIdx.x; j < V; j += blockDim.x) mx = fmaxf(mx, l[j]);
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) fr[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < blockDim.x / 32 ? fr[threadIdx.x] : -INFINITY;
    t = warp_max(t);
    if (threadIdx.x == 0) fr[0] = t;
  }
  __syncthreads();
  mx = fr[0];
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < V; j += blockDim.x) s += exp(double(l[j]) - mx);
  s = warp_sum_d(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    t = warp_sum_d(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const double lse = double(mx) + log(red[0]);
  const int t = tgt[r];
  if (!dlp) {
    if (threadIdx.x == 0) lp_out[r] = double(l[t]) - lse;
    return;
  }
  const double g = dlp[r];
  __syncthreads();
  for (int64_t j = threadIdx.x; j < V; j += blockDim.x) {
    const double p = exp(double(l[j]) - lse);
    l[j] = float(g * ((j == t ? 1.0 : 0.0) - p));
  }
}

// value head: v[r] = hf[idx[r]] . head (fp64 accumulation)
__global__ void t_value_fwd(const float* __restrict__ hf, const int32_t* __restrict__ idx, int64_t d,
                            const float* __restrict__ head, double* __restrict__ v) {
  const int64_t r = blockIdx.x;
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < d; j += blockDim.x) s += double(hf[int64_t(idx[r]) * d + j]) * head[j];
  s = warp_sum_d(s);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < int(blockDim.x / 32); ++k) t += red[k];
    v[r] = t;
  }
}
// dhf[idx[r]] += dv[r] head; dhead[j] += sum_r dv[r] hf[idx[r], j] (one thread per j, rows in order)
__global__ void t_value_bwd_h(const double* __restrict__ dv, const int32_t* __restrict__ idx, int64_t R, int64_t d,
                              const float* __restrict__ head, float* __restrict__ dhf) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < R * d; i += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(dhf + int64_t(idx[i / d]) * d + i % d, float(dv[i / d] * head[i % d]));
}
__global__ void t_value_bwd_head(const double* __restrict__ dv, const int32_t* __restrict__ idx, int64_t R, int64_t d,
                                 const float* __restrict__ hf, float* __restrict__ dhead) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j >= d) return;
  double s = 0.0;
  for (int64_t r = 0; r < R; ++r) s += dv[r] * hf[int64_t(idx[r]) * d + j];
  dhead[j] += float(s);
}

// AdamW (src/optim.cpp:32-55), fp64 arithmetic per element
__global__ void t_adamw(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ m,
                        float* __restrict__ v, int64_t n, double lr, double b1, double b2, double eps, double wd,
                        double bc1, double bc2) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double gi = g[i];
    const double mi = b1 * m[i] + (1.0 - b1) * gi;
    const double vi = b2 * v[i] + (1.0 - b2) * gi * gi;
    m[i] = float(mi);
    v[i] = float(vi);
    const double wi = w[i];
    w[i] = float(wi - lr * ((mi / bc1) / (sqrt(vi / bc2) + eps) + wd * wi));
  }
}

dim3 grid_for(int64_t n) { return dim3(unsigned(std::min<int64_t>(std::max<int64_t>(ceil_div(n, 256), 1), 148 * 8))); }

}  // namespace

// ------------------------------------------------------------------ Trainer
Trainer::Trainer(Ctx* ctx, const ppoexp_model_config& config, const ppoexp_tensor_view* views, int64_t n,
                 Model* target, const AdamOpts& o)
    : c(ctx), cfg(config), model(target), opts(o) {
  if (target && (target->cfg.vocab_size != cfg.vocab_size || target->cfg.d_model != cfg.d_model ||
                 target->cfg.n_layers != cfg.n_layers || target->cfg.scalar_head != cfg.scalar_head))
    throw ContractError("trainer: model config differs from the trainer's");
  DeviceGuard gd(c->device);
  const auto exp = Model::expected(cfg);
  std::map<std::string, const ppoexp_tensor_view*> by;
  for (int64_t i = 0; i < n; ++i) {
    if (!views[i].name) throw ContractError("tensor view without a name");
    by[views[i].name] = &views[i];
  }
  if (int64_t(by.size()) != int64_t(exp.size()) || n != int64_t(exp.size()))
    throw ContractError("trainer: parameter count mismatch");
  size_t off = 0;
  for (const auto& [name, shape] : exp) {
    int64_t k = 1;
    for (auto s : shape) k *= s;
    params.push_back({name, shape, k, off});
    off += size_t((k + 63) / 64 * 64);
  }
  total = off;
  W.ensure(total * 4);
  G.ensure(total * 4);
  Mo.ensure(total * 4);
  Vo.ensure(total * 4);
  PPOEXP_CUDA(cudaMemsetAsync(W.ptr, 0, total * 4, c->stream));
  PPOEXP_CUDA(cudaMemsetAsync(Mo.ptr, 0, total * 4, c->stream));
  PPOEXP_CUDA(cudaMemsetAsync(Vo.ptr, 0, total * 4, c->stream));
  for (const auto& p : params) {
    auto it = by.find(p.name);
    if (it == by.end()) throw ContractError("trainer: missing parameter " + p.name);
    const auto* v = it->second;
    const size_t esz = v->dtype == PPOEXP_F64 ? 8 : (v->dtype == PPOEXP_F32 ? 4 : 2);
    const void* src = v->data;
    if (v->where == PPOEXP_HOST) {
      void* st = c->workspace("train.staging", p.numel * esz);
      PPOEXP_CUDA(cudaMemcpyAsync(st, v->data, p.numel * esz, cudaMemcpyHostToDevice, c->stream));
      src = st;
    }
    launch_convert(*c, src, v->dtype, w(p.name), PPOEXP_F32, 1, p.numel, false, p.numel, 0);
    if (v->where == PPOEXP_HOST) PPOEXP_CUDA(cudaStreamSynchronize(c->stream));
  }
  blas_check(cublasCreate(reinterpret_cast<cublasHandle_t*>(&blas)), "create");
  blas_check(cublasSetMathMode(static_cast<cublasHandle_t>(blas), CUBLAS_PEDANTIC_MATH), "math mode");
  PPOEXP_CUDA(cudaStreamSynchronize(c->stream));
}

Trainer::~Trainer() {
  if (blas) cublasDestroy(static_cast<cublasHandle_t>(blas));
}

const Trainer::Param& Trainer::param(const std::string& name) const {
  for (const auto& p : params)
    if (p.name == name) return p;
  throw ContractError("trainer: unknown parameter " + name);
}
float* Trainer::w(const std::string& n) { return W.as<float>() + param(n).off; }
float* Trainer::g(const std::string& n) { return G.as<float>() + param(n).off; }

// C[M,N] = alpha op(A) op(B) + beta C, all row-major fp32
void Trainer::mm(bool ta, bool tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* B,
                 int64_t ldb, float beta, float* C, int64_t ldc, float alpha) {
  auto h = static_cast<cublasHandle_t>(blas);
  blas_check(cublasSetStream(h, c->stream), "stream");
  blas_check(cublasSgemm(h, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, int(N), int(M), int(K),
                         &alpha, B, int(ldb), A, int(lda), &beta, C, int(ldc)),
             "sgemm");
}
void Trainer::mm_batched(bool ta, bool tb, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, int64_t sa,
                         const float* B, int64_t ldb, int64_t sb, float beta, float* C, int64_t ldc, int64_t sc,
                         int64_t batch, float alpha) {
  auto h = static_cast<cublasHandle_t>(blas);
  blas_check(cublasSetStream(h, c->stream), "stream");
  blas_check(cublasSgemmStridedBatched(h, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, int(N),
                                       int(M), int(K), &alpha, B, int(ldb), sb, A, int(lda), sa, &beta, C, int(ldc),
                                       sc, int(batch)),
             "sgemm batched");
}

// Recorded forward over a packed ragged batch; leaves hf (final LayerNorm output).
void Trainer::forward(const Packed& p) {
  Ctx& cc = *c;
  const int64_t M = p.M, d = cfg.d_model, f = cfg.d_ff, L = cfg.n_layers, H = cfg.n_heads, dh = d / H;
  rows = M;
  pk = p;
  auto ws = [&](const char* nm, size_t n) { return static_cast<float*>(cc.workspace(std::string("train.") + nm, n * 4)); };
  const size_t per_layer = layer_floats();
  act = ws("act", per_layer * L + size_t(M) * (2 * d) + 2 * size_t(M) + 64);
  int64_t pbytes = 0;
  for (int64_t b = 0; b < p.B; ++b) {
    const int64_t T = p.offsets[b + 1] - p.offsets[b];
    pbytes += H * T * T;
  }
  pstride = pbytes;
  probs = ws("probs", size_t(std::max<int64_t>(pbytes, 1)) * L);
  float* x = act + per_layer * L;  // running residual, then x_L
  t_embed_fwd<<<grid_for(M * d), 256, 0, cc.stream>>>(p.tokens_d, p.positions_d, M, d, w("tok_embed.weight"),
                                                      w("pos_embed.weight"), x);
  const float scale = 1.0f / std::sqrt(float(dh));
  for (int64_t l = 0; l < L; ++l) {
    LayerAct a = layer_act(l);
    const std::string base = "layers." + std::to_string(l) + ".";
    PPOEXP_CUDA(cudaMemcpyAsync(a.x, x, size_t(M) * d * 4, cudaMemcpyDeviceToDevice, cc.stream));
    t_ln_fwd<<<unsigned(M), 256, 0, cc.stream>>>(a.x, d, w(base + "attn_norm.weight"), w(base + "attn_norm.bias"), a.h1,
                                                 a.mu1, a.rs1);
    const char* qkvn[3] = {"attn.q_proj.weight", "attn.k_proj.weight", "attn.v_proj.weight"};
    for (int k = 0; k < 3; ++k) mm(false, false, M, d, d, a.h1, d, w(base + qkvn[k]), d, 0.f, a.qkv + k * d, 3 * d);
    float* P = probs + size_t(pstride) * l;
    int64_t po = 0;
    for (int64_t b = 0; b < p.B; ++b) {
      const int64_t o = p.offsets[b], T = p.offsets[b + 1] - o;
      if (T == 0) continue;
      // S_h = Q_h K_h^T over all heads (stride dh between heads inside a qkv row)
      mm_batched(false, true, T, T, dh, a.qkv + o * 3 * d, 3 * d, dh, a.qkv + o * 3 * d + d, 3 * d, dh, 0.f, P + po, T,
                 T * T, H);
      t_softmax_causal<<<unsigned(H * T), 128, 0, cc.stream>>>(P + po, T, scale);
      mm_batched(false, false, T, dh, T, P + po, T, T * T, a.qkv + o * 3 * d + 2 * d, 3 * d, dh, 0.f, a.att + o * d, d,
                 dh, H);
      po += H * T * T;
    }
    PPOEXP_CUDA(cudaMemcpyAsync(a.xm, a.x, size_t(M) * d * 4, cudaMemcpyDeviceToDevice, cc.stream));
    mm(false, false, M, d, d, a.att, d, w(base + "attn.o_proj.weight"), d, 1.f, a.xm, d);
    t_ln_fwd<<<unsigned(M), 256, 0, cc.stream>>>(a.xm, d, w(base + "ffn_norm.weight"), w(base + "ffn_norm.bias"), a.h2,
                                                 a.mu2, a.rs2);
    mm(false, false, M, f, d, a.h2, d, w(base + "ffn.up_proj.weight"), f, 0.f, a.u, f);
    t_gelu_fwd<<<grid_for(M * f), 256, 0, cc.stream>>>(a.u, M * f, a.gu);
    PPOEXP_CUDA(cudaMemcpyAsync(x, a.xm, size_t(M) * d * 4, cudaMemcpyDeviceToDevice, cc.stream));
    mm(false, false, M, d, f, a.gu, f, w(base + "ffn.down_proj.weight"), d, 1.f, x, d);
  }
  float* hf = x + size_t(M) * d;
  float* muf = hf + size_t(M) * d;
  t_ln_fwd<<<unsigned(M), 256, 0, cc.stream>>>(x, d, w("final_norm.weight"), w("final_norm.bias"), hf, muf, muf + M);
  PPOEXP_CUDA(cudaGetLastError());
}

// per layer, per row: x | h1 | qkv (3d) | att | xm | h2 (8 d) | u | gelu(u) (2 f) | mu1 rs1 mu2 rs2
size_t Trainer::layer_floats() const {
  return size_t(rows) * (8 * cfg.d_model + 2 * cfg.d_ff) + 4 * size_t(rows);
}

Trainer::LayerAct Trainer::layer_act(int64_t l) {
  const int64_t M = rows, d = cfg.d_model, f = cfg.d_ff;
  float* b = act + layer_floats() * l;
  LayerAct a;
  a.x = b;
  a.h1 = a.x + M * d;
  a.qkv = a.h1 + M * d;
  a.att = a.qkv + 3 * M * d;
  a.xm = a.att + M * d;
  a.h2 = a.xm + M * d;
  a.u = a.h2 + M * d;
  a.gu = a.u + M * f;
  a.mu1 = a.gu + M * f;
  a.rs1 = a.mu1 + M;
  a.mu2 = a.rs1 + M;
  a.rs2 = a.mu2 + M;
  return a;
}

float* Trainer::hf() { return act + layer_floats() * cfg.n_layers + size_t(rows) * cfg.d_model; }

// Response-row log-probs through the tied LM head: lp[r] = log p(tgt[r] | hf[idx[r]]).
void Trainer::lm_logprobs(const int32_t* idx, const int32_t* tgt, int64_t R, double* lp) {
  Ctx& cc = *c;
  const int64_t d = cfg.d_model, V = cfg.vocab_size;
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(R, (int64_t(1) << 28) / V));
  float* hg = static_cast<float*>(cc.workspace("train.hg", size_t(chunk) * d * 4));
  float* lg = static_cast<float*>(cc.workspace("train.logits", size_t(chunk) * V * 4));
  for (int64_t r0 = 0; r0 < R; r0 += chunk) {
    const int64_t n = std::min(chunk, R - r0);
    t_gather_rows<<<grid_for(n * d), 256, 0, cc.stream>>>(hf(), idx + r0, n, d, hg);
    mm(false, true, n, V, d, hg, d, w("tok_embed.weight"), d, 0.f, lg, V);
    t_lm_rows<<<unsigned(n), 256, 0, cc.stream>>>(lg, V, tgt + r0, nullptr, lp + r0);
  }
  PPOEXP_CUDA(cudaGetLastError());
}

// Backward of the LM-head rows given dlp: accumulates dtok (tied head) and dhf.
void Trainer::lm_backward(const int32_t* idx, const int32_t* tgt, int64_t R, const double* dlp, float* dhf) {
  Ctx& cc = *c;
  const int64_t d = cfg.d_model, V = cfg.vocab_size;
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(R, (int64_t(1) << 28) / V));
  float* hg = static_cast<float*>(cc.workspace("train.hg", size_t(chunk) * d * 4));
  float* lg = static_cast<float*>(cc.workspace("train.logits", size_t(chunk) * V * 4));
  float* dhg = static_cast<float*>(cc.workspace("train.dhg", size_t(chunk) * d * 4));
  for (int64_t r0 = 0; r0 < R; r0 += chunk) {
    const int64_t n = std::min(chunk, R - r0);
    t_gather_rows<<<grid_for(n * d), 256, 0, cc.stream>>>(hf(), idx + r0, n, d, hg);
    mm(false, true, n, V, d, hg, d, w("tok_embed.weight"), d, 0.f, lg, V);
    t_lm_rows<<<unsigned(n), 256, 0, cc.stream>>>(lg, V, tgt + r0, dlp + r0, nullptr);  // lg := dlogits
    mm(false, false, n, d, V, lg, V, w("tok_embed.weight"), d, 0.f, dhg, d);           // dhg = dlogits E
    mm(true, false, V, d, n, lg, V, hg, d, 1.f, g("tok_embed.weight"), d);             // dE += dlogits^T hg
    t_scatter_add_rows<<<grid_for(n * d), 256, 0, cc.stream>>>(dhg, idx + r0, n, d, dhf);
  }
  PPOEXP_CUDA(cudaGetLastError());
}

void Trainer::values(const int32_t* idx, int64_t R, double* v) {
  t_value_fwd<<<unsigned(R), 128, 0, c->stream>>>(hf(), idx, cfg.d_model, w("scalar_head.weight"), v);
  PPOEXP_CUDA(cudaGetLastError());
}

void Trainer::value_backward(const int32_t* idx, int64_t R, const double* dv, float* dhf) {
  const int64_t d = cfg.d_model;
  t_value_bwd_h<<<grid_for(R * d), 256, 0, c->stream>>>(dv, idx, R, d, w("scalar_head.weight"), dhf);
  t_value_bwd_head<<<unsigned(ceil_div(d, 128)), 128, 0, c->stream>>>(dv, idx, R, d, hf(), g("scalar_head.weight"));
  PPOEXP_CUDA(cudaGetLastError());
}

// Backward from dhf (the final LayerNorm output) through every layer into G.
void Trainer::backward(float* dhf) {
  Ctx& cc = *c;
  const int64_t M = rows, d = cfg.d_model, f = cfg.d_ff, L = cfg.n_layers, H = cfg.n_heads, dh = d / H;
  const Packed& p = pk;
  auto ws = [&](const char* nm, size_t n) { return static_cast<float*>(cc.workspace(std::string("train.") + nm, n * 4)); };
  float* xL = hf() - size_t(M) * d;
  float* muf = hf() + size_t(M) * d;
  float* dx = ws("dx", size_t(M) * d);
  float* dt = ws("dtmp", size_t(M) * std::max(f, 3 * d));
  float* dt2 = ws("dtmp2", size_t(M) * d);
  float* dP = ws("dP", size_t(std::max<int64_t>(pstride, 1)));
  PPOEXP_CUDA(cudaMemsetAsync(dx, 0, size_t(M) * d * 4, cc.stream));
  t_ln_bwd_x<<<unsigned(M), 256, 0, cc.stream>>>(xL, dhf, d, w("final_norm.weight"), muf, muf + M, dx);
  t_ln_bwd_params<<<unsigned(ceil_div(d, 128)), 128, 0, cc.stream>>>(xL, dhf, M, d, muf, muf + M,
                                                                    g("final_norm.weight"), g("final_norm.bias"));
  const float scale = 1.0f / std::sqrt(float(dh));
  for (int64_t l = L - 1; l >= 0; --l) {
    LayerAct a = layer_act(l);
    const std::string base = "layers." + std::to_string(l) + ".";
    // x_{l+1} = xm + gelu(u) Wdown
    mm(false, true, M, f, d, dx, d, w(base + "ffn.down_proj.weight"), d, 0.f, dt, f);  // d gelu(u)
    mm(true, false, f, d, M, a.gu, f, dx, d, 1.f, g(base + "ffn.down_proj.weight"), d);
    t_gelu_bwd<<<grid_for(M * f), 256, 0, cc.stream>>>(a.u, M * f, dt);               // du
    mm(false, true, M, d, f, dt, f, w(base + "ffn.up_proj.weight"), f, 0.f, dt2, d);   // dh2
    mm(true, false, d, f, M, a.h2, d, dt, f, 1.f, g(base + "ffn.up_proj.weight"), f);
    // xm = x + att Wo;  dx (now d xm) += LN2 backward
    t_ln_bwd_x<<<unsigned(M), 256, 0, cc.stream>>>(a.xm, dt2, d, w(base + "ffn_norm.weight"), a.mu2, a.rs2, dx);
    t_ln_bwd_params<<<unsigned(ceil_div(d, 128)), 128, 0, cc.stream>>>(a.xm, dt2, M, d, a.mu2, a.rs2,
                                                                      g(base + "ffn_norm.weight"), g(base + "ffn_norm.bias"));
    float* datt = dt2;
    mm(false, true, M, d, d, dx, d, w(base + "attn.o_proj.weight"), d, 0.f, datt, d);
    mm(true, false, d, d, M, a.att, d, dx, d, 1.f, g(base + "attn.o_proj.weight"), d);
    // attention backward per sequence, all heads batched → dqkv (dt, [M, 3d])
    float* dqkv = dt;
    const float* P = probs + size_t(pstride) * l;
    int64_t po = 0;
    for (int64_t b = 0; b < p.B; ++b) {
      const int64_t o = p.offsets[b], T = p.offsets[b + 1] - o;
      if (T == 0) continue;
      const float* q = a.qkv + o * 3 * d;
      float* dq = dqkv + o * 3 * d;
      // dP = dO V^T ; dV = P^T dO
      mm_batched(false, true, T, T, dh, datt + o * d, d, dh, q + 2 * d, 3 * d, dh, 0.f, dP + po, T, T * T, H);
      mm_batched(true, false, T, dh, T, P + po, T, T * T, datt + o * d, d, dh, 0.f, dq + 2 * d, 3 * d, dh, H);
      t_softmax_bwd<<<unsigned(H * T), 128, 0, cc.stream>>>(P + po, dP + po, T, scale);  // dS (scaled)
      // dQ = dS K ; dK = dS^T Q
      mm_batched(false, false, T, dh, T, dP + po, T, T * T, q + d, 3 * d, dh, 0.f, dq, 3 * d, dh, H);
      mm_batched(true, false, T, dh, T, dP + po, T, T * T, q, 3 * d, dh, 0.f, dq + d, 3 * d, dh, H);
      po += H * T * T;
    }
    // q|k|v = h1 W;  dh1 = sum dq W^T
    float* dh1 = dt2;
    const char* qkvn[3] = {"attn.q_proj.weight", "attn.k_proj.weight", "attn.v_proj.weight"};
    for (int k = 0; k < 3; ++k) {
      mm(false, true, M, d, d, dqkv + k * d, 3 * d, w(base + qkvn[k]), d, k ? 1.f : 0.f, dh1, d);
      mm(true, false, d, d, M, a.h1, d, dqkv + k * d, 3 * d, 1.f, g(base + qkvn[k]), d);
    }
    t_ln_bwd_x<<<unsigned(M), 256, 0, cc.stream>>>(a.x, dh1, d, w(base + "attn_norm.weight"), a.mu1, a.rs1, dx);
    t_ln_bwd_params<<<unsigned(ceil_div(d, 128)), 128, 0, cc.stream>>>(a.x, dh1, M, d, a.mu1, a.rs1,
                                                                      g(base + "attn_norm.weight"), g(base + "attn_norm.bias"));
  }
  t_embed_bwd<<<grid_for(M * d), 256, 0, cc.stream>>>(p.tokens_d, p.positions_d, M, d, dx, g("tok_embed.weight"),
                                                      g("pos_embed.weight"));
  PPOEXP_CUDA(cudaGetLastError());
}

void Trainer::zero_grad() { PPOEXP_CUDA(cudaMemsetAsync(G.ptr, 0, total * 4, c->stream)); }

void Trainer::adamw_step(double lr) {
  ++t;
  const double bc1 = 1.0 - std::pow(opts.beta1, double(t)), bc2 = 1.0 - std::pow(opts.beta2, double(t));
  t_adamw<<<grid_for(int64_t(total)), 256, 0, c->stream>>>(W.as<float>(), G.as<float>(), Mo.as<float>(), Vo.as<float>(),
                                                           int64_t(total), lr, opts.beta1, opts.beta2, opts.eps,
                                                           opts.weight_decay, bc1, bc2);
  PPOEXP_CUDA(cudaGetLastError());
}

void Trainer::refit() {
  if (!model) throw ContractError("trainer: no serving model to refit");
  std::vector<ppoexp_tensor_view> v;
  for (const auto& p : params) {
    ppoexp_tensor_view x{};
    x.name = p.name.c_str();
    x.rank = int32_t(p.shape.size());
    x.dtype = PPOEXP_F32;
    x.shape[0] = p.shape[0];
    x.shape[1] = p.shape.size() > 1 ? p.shape[1] : 0;
    x.data = W.as<float>() + p.off;
    x.where = PPOEXP_DEVICE;
    v.push_back(x);
  }
  PPOEXP_CUDA(cudaStreamSynchronize(c->stream));
  model->load(v.data(), int64_t(v.size()), true);
  ++model->generation;
}

void Trainer::get(const std::string& name, double* out, int64_t numel) {
  const Param& p = param(name);
  if (numel != p.numel) throw ShapeError("trainer: " + name + " has " + std::to_string(p.numel) + " elements");
  std::vector<float> h(p.numel);
  PPOEXP_CUDA(cudaStreamSynchronize(c->stream));
  PPOEXP_CUDA(cudaMemcpy(h.data(), W.as<float>() + p.off, p.numel * 4, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < p.numel; ++i) out[i] = h[i];
}


// ------------------------------------------------------------------ steps
namespace {

// response rows of a packed batch: row o+t-1 predicts token o+t for t >= rs
void response_rows(const std::vector<int64_t>& off, const std::vector<int64_t>& rs, const std::vector<int32_t>& tok,
                   std::vector<int32_t>& idx, std::vector<int32_t>& tgt, std::vector<int64_t>& seq_of) {
  const int64_t B = int64_t(off.size()) - 1;
  for (int64_t b = 0; b < B; ++b)
    for (int64_t t = rs[b]; t < off[b + 1] - off[b]; ++t) {
      idx.push_back(int32_t(off[b] + t - 1));
      tgt.push_back(tok[off[b] + t]);
      seq_of.push_back(b);
    }
}

double sigmoid(double x) { return x >= 0 ? 1.0 / (1.0 + std::exp(-x)) : std::exp(x) / (1.0 + std::exp(x)); }
double log_sigmoid(double x) { return x < 0.0 ? x - std::log1p(std::exp(x)) : -std::log1p(std::exp(-x)); }

}  // namespace

Trainer::Batch Trainer::prepare(int64_t B, const int32_t* tokens, const int64_t* offsets, const int64_t* rs_in,
                                int where) {
  Ctx& cc = *c;
  Batch bt;
  bt.off.assign(B + 1, 0);
  bt.rs.assign(B, 0);
  if (where == PPOEXP_HOST) {
    std::memcpy(bt.off.data(), offsets, (B + 1) * 8);
    std::memcpy(bt.rs.data(), rs_in, B * 8);
  } else {
    PPOEXP_CUDA(cudaMemcpy(bt.off.data(), offsets, (B + 1) * 8, cudaMemcpyDeviceToHost));
    PPOEXP_CUDA(cudaMemcpy(bt.rs.data(), rs_in, B * 8, cudaMemcpyDeviceToHost));
  }
  if (bt.off[0] != 0) throw ContractError("trainer: offsets[0] must be 0");
  for (int64_t b = 0; b < B; ++b) {
    const int64_t T = bt.off[b + 1] - bt.off[b];
    if (T > cfg.max_seq_len) throw ContractError("forward: sequence length exceeds max_seq_len");
    if (bt.rs[b] < 1 || bt.rs[b] >= T)
      throw ContractError("trainer: response_start must leave a nonempty prompt and response");
  }
  const int64_t M = bt.off[B];
  bt.tok.resize(M);
  if (where == PPOEXP_HOST)
    std::memcpy(bt.tok.data(), tokens, M * 4);
  else
    PPOEXP_CUDA(cudaMemcpy(bt.tok.data(), tokens, M * 4, cudaMemcpyDeviceToHost));
  check_tokens(cc, bt.tok.data(), M, cfg.vocab_size, PPOEXP_HOST, "trainer");
  response_rows(bt.off, bt.rs, bt.tok, bt.idx, bt.tgt, bt.seq_of);
  Packed p;
  p.offsets = bt.off;
  p.tokens_d = static_cast<int32_t*>(cc.workspace("train.tokens", std::max<int64_t>(M, 1) * 4));
  PPOEXP_CUDA(cudaMemcpyAsync(p.tokens_d, bt.tok.data(), M * 4, cudaMemcpyHostToDevice, cc.stream));
  pack_metadata(cc, p, "train");
  bt.R = int64_t(bt.idx.size());
  bt.idx_d = static_cast<int32_t*>(cc.workspace("train.idx", std::max<int64_t>(bt.R, 1) * 4));
  bt.tgt_d = static_cast<int32_t*>(cc.workspace("train.tgt", std::max<int64_t>(bt.R, 1) * 4));
  PPOEXP_CUDA(cudaMemcpyAsync(bt.idx_d, bt.idx.data(), bt.R * 4, cudaMemcpyHostToDevice, cc.stream));
  PPOEXP_CUDA(cudaMemcpyAsync(bt.tgt_d, bt.tgt.data(), bt.R * 4, cudaMemcpyHostToDevice, cc.stream));
  forward(p);
  return bt;
}

std::vector<double> Trainer::to_host_d(const double* d, int64_t n) {
  std::vector<double> h(n);
  PPOEXP_CUDA(cudaMemcpyAsync(h.data(), d, n * 8, cudaMemcpyDeviceToHost, c->stream));
  PPOEXP_CUDA(cudaStreamSynchronize(c->stream));
  return h;
}

double* Trainer::to_dev_d(const std::vector<double>& h, const char* name) {
  double* d = static_cast<double*>(c->workspace(name, std::max<size_t>(h.size(), 1) * 8));
  PPOEXP_CUDA(cudaMemcpyAsync(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice, c->stream));
  return d;
}

void Trainer::backprop_lm(const Batch& bt, const std::vector<double>& dlp) {
  const int64_t d = cfg.d_model;
  float* dhf = static_cast<float*>(c->workspace("train.dhf", size_t(rows) * d * 4));
  PPOEXP_CUDA(cudaMemsetAsync(dhf, 0, size_t(rows) * d * 4, c->stream));
  zero_grad();
  lm_backward(bt.idx_d, bt.tgt_d, bt.R, to_dev_d(dlp, "train.dlp"), dhf);
  backward(dhf);
}

// PPO actor update (src/ppo.cpp:395-424): new log-probs of the response tokens
// under the current weights, ppo_actor_loss (src/losses.cpp:201-214), backward,
// AdamW.  Gradient of -masked_mean(min(r A, clamp(r) A)): ties route to the
// unclipped term, clamp passes gradient strictly inside (1-eps, 1+eps)
// (src/tensor.cpp:229-270).
double Trainer::ppo_actor_step(int64_t B, const int32_t* tokens, const int64_t* offsets, const int64_t* rs,
                               const double* old_lp, const double* adv, const double* mask, double clip_eps, double lr,
                               int where) {
  Batch bt = prepare(B, tokens, offsets, rs, where);
  const int64_t R = bt.R;
  double* lp_d = static_cast<double*>(c->workspace("train.lp", std::max<int64_t>(R, 1) * 8));
  lm_logprobs(bt.idx_d, bt.tgt_d, R, lp_d);
  const auto lp = to_host_d(lp_d, R);
  auto host = [&](const double* p) {
    std::vector<double> v(R, 1.0);
    if (!p) return v;
    if (where == PPOEXP_HOST)
      std::memcpy(v.data(), p, R * 8);
    else
      PPOEXP_CUDA(cudaMemcpy(v.data(), p, R * 8, cudaMemcpyDeviceToHost));
    return v;
  };
  const auto old = host(old_lp), A = host(adv), mk = host(mask);
  double denom = 0.0;
  for (double m : mk) denom += m;
  if (denom == 0.0) throw ContractError("masked_mean: mask selects no elements");
  double loss = 0.0;
  std::vector<double> dlp(R, 0.0);
  for (int64_t r = 0; r < R; ++r) {
    const double ratio = std::exp(lp[r] - old[r]);
    const double u = ratio * A[r];
    const double cl = std::min(std::max(ratio, 1.0 - clip_eps), 1.0 + clip_eps) * A[r];
    loss += (u <= cl ? u : cl) * mk[r];
    const double dmin = u <= cl ? A[r] : ((ratio > 1.0 - clip_eps && ratio < 1.0 + clip_eps) ? A[r] : 0.0);
    dlp[r] = -(mk[r] / denom) * dmin * ratio;
  }
  loss = -loss / denom;
  backprop_lm(bt, dlp);
  adamw_step(lr);
  return loss;
}

// Critic update (CriticJob::handle_train, src/ppo.cpp:195-231): per sequence
// ppo_critic_loss (src/losses.cpp:216-231) over its response values, mean over
// the sequences; maximum routes ties to the unclipped term.
double Trainer::critic_step(int64_t B, const int32_t* tokens, const int64_t* offsets, const int64_t* rs,
                            const double* old_values, const double* returns, double value_clip, double lr, int where) {
  if (!cfg.scalar_head) throw PpoError("critic job: critic model needs a scalar head");
  Batch bt = prepare(B, tokens, offsets, rs, where);
  const int64_t R = bt.R, d = cfg.d_model;
  double* v_d = static_cast<double*>(c->workspace("train.v", std::max<int64_t>(R, 1) * 8));
  values(bt.idx_d, R, v_d);
  const auto v = to_host_d(v_d, R);
  std::vector<double> ov(R), rt(R);
  if (where == PPOEXP_HOST) {
    std::memcpy(ov.data(), old_values, R * 8);
    std::memcpy(rt.data(), returns, R * 8);
  } else {
    PPOEXP_CUDA(cudaMemcpy(ov.data(), old_values, R * 8, cudaMemcpyDeviceToHost));
    PPOEXP_CUDA(cudaMemcpy(rt.data(), returns, R * 8, cudaMemcpyDeviceToHost));
  }
  std::vector<double> dv(R, 0.0), seq_loss(B, 0.0);
  std::vector<int64_t> n_b(B, 0);
  for (int64_t r = 0; r < R; ++r) ++n_b[bt.seq_of[r]];
  for (int64_t r = 0; r < R; ++r) {
    const int64_t b = bt.seq_of[r];
    const double e = v[r] - rt[r], sq = e * e;
    const double dvc = v[r] - ov[r];
    const double vc = std::min(std::max(dvc, -value_clip), value_clip) + ov[r];
    const double ec = vc - rt[r], sqc = ec * ec;
    const double w = 1.0 / (double(n_b[b]) * double(B));
    seq_loss[b] += (sq >= sqc ? sq : sqc) / double(n_b[b]);
    dv[r] = w * (sq >= sqc ? 2.0 * e : 2.0 * ec * ((dvc > -value_clip && dvc < value_clip) ? 1.0 : 0.0));
  }
  double loss = 0.0;
  for (int64_t b = 0; b < B; ++b) loss += seq_loss[b];
  loss /= double(B);
  float* dhf = static_cast<float*>(c->workspace("train.dhf", size_t(rows) * d * 4));
  PPOEXP_CUDA(cudaMemsetAsync(dhf, 0, size_t(rows) * d * 4, c->stream));
  zero_grad();
  value_backward(bt.idx_d, R, to_dev_d(dv, "train.dv"), dhf);
  backward(dhf);
  adamw_step(lr);
  return loss;
}

// DPO family update (src/trainers.cpp:54-80): policy response sums through
// this trainer's graph, frozen reference sums from `ref_sums`, dpo_family_loss
// (src/losses.cpp:129-166) and its gradient in fp64 on the host.
double Trainer::dpo_step(int64_t n_pairs, const int32_t* tokens, const int64_t* offsets, const int64_t* rs,
                         const std::vector<double>& ref_sums, int variant, double beta, double cdpo_eps, double lr,
                         int where, double* margin_out) {
  if (!(beta > 0.0)) throw ContractError("dpo hyper: beta must be positive");
  if (variant < 0 || variant > 3) throw ContractError("dpo hyper: unknown variant");
  const int64_t B = 2 * n_pairs, n = n_pairs;
  if (n == 0) throw ContractError("dpo_family_loss: mismatched sequence counts");
  Batch bt = prepare(B, tokens, offsets, rs, where);
  const int64_t R = bt.R;
  double* lp_d = static_cast<double*>(c->workspace("train.lp", std::max<int64_t>(R, 1) * 8));
  lm_logprobs(bt.idx_d, bt.tgt_d, R, lp_d);
  const auto lp = to_host_d(lp_d, R);
  std::vector<double> sums(B, 0.0);
  for (int64_t r = 0; r < R; ++r) sums[bt.seq_of[r]] += lp[r];  // position order within each sequence
  std::vector<double> cr(n), rr(n), dcr(n, 0.0), drr(n, 0.0);
  double margin_sum = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    cr[i] = sums[2 * i] - ref_sums[2 * i];
    rr[i] = sums[2 * i + 1] - ref_sums[2 * i + 1];
    margin_sum += cr[i] - rr[i];
  }
  if (margin_out) *margin_out = beta * margin_sum / double(n);
  double loss = 0.0;
  const double inv_n = 1.0 / double(n);
  if (variant == 3) {  // kto: paired Kahneman-Tversky, zero-floored class means
    double mc = 0.0, mr = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      mc += cr[i] * inv_n;
      mr += rr[i] * inv_n;
    }
    const double zc = std::min(std::max(mc, 0.0), 1e300), zr = std::min(std::max(mr, 0.0), 1e300);
    const double gzc = (mc > 0.0 && mc < 1e300) ? 1.0 : 0.0, gzr = (mr > 0.0 && mr < 1e300) ? 1.0 : 0.0;
    double sc = 0.0, sr = 0.0, dzr = 0.0, dzc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double a = sigmoid(beta * (cr[i] - zr)), b2 = sigmoid(beta * (zc - rr[i]));
      sc += 1.0 - a;
      sr += 1.0 - b2;
      // d/d(cr_i) of 0.5 mean(1 - a) ; the z terms collect the cross terms
      dcr[i] += -0.5 * inv_n * beta * a * (1.0 - a);
      dzr += 0.5 * inv_n * beta * a * (1.0 - a);
      drr[i] += 0.5 * inv_n * beta * b2 * (1.0 - b2);
      dzc += -0.5 * inv_n * beta * b2 * (1.0 - b2);
    }
    for (int64_t i = 0; i < n; ++i) {
      dcr[i] += dzc * gzc * inv_n;
      drr[i] += dzr * gzr * inv_n;
    }
    loss = 0.5 * (sc * inv_n + sr * inv_n);
  } else {
    for (int64_t i = 0; i < n; ++i) {
      const double m = cr[i] - rr[i];
      double gm = 0.0;
      if (variant == 0) {  // dpo: mean(-log sigmoid(beta m))
        loss += -log_sigmoid(beta * m) * inv_n;
        gm = -beta * (1.0 - sigmoid(beta * m));
      } else if (variant == 1) {  // ipo: mean((m - 1/(2 beta))^2)
        const double dl = m - 1.0 / (2.0 * beta);
        loss += dl * dl * inv_n;
        gm = 2.0 * dl;
      } else {  // cdpo: label-smoothed
        const double s = beta * m;
        loss += ((1.0 - cdpo_eps) * -log_sigmoid(s) + cdpo_eps * -log_sigmoid(-s)) * inv_n;
        gm = beta * (-(1.0 - cdpo_eps) * (1.0 - sigmoid(s)) + cdpo_eps * sigmoid(s));
      }
      dcr[i] = gm * inv_n;
      drr[i] = -gm * inv_n;
    }
  }
  std::vector<double> dlp(R);
  for (int64_t r = 0; r < R; ++r) {
    const int64_t sq = bt.seq_of[r];
    dlp[r] = (sq & 1) ? drr[sq / 2] : dcr[sq / 2];
  }
  backprop_lm(bt, dlp);
  adamw_step(lr);
  return loss;
}

}  // namespace ppx
