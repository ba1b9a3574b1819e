// logprob_shaping.cu — K9 fused log-softmax + gather, K11 KL shaping + GAE,
// K12 whitening statistics.
#include <cfloat>

#include "kernels.hpp"

namespace ppx {

namespace {

// ------------------------------------------------------------------- K9
// One CTA per logits row; a single streaming pass with an online
// (max, sum exp) per thread, 16-byte vector loads, then the gather of the
// target logit: lp = l[target] - (max + log(sum)).  This is
// gather_token_logprobs(log_softmax(logits)) (src/tensor.cpp:428-456,
// :491-519) and KvSession's log_softmax_vec(...)[tok] (src/model.cpp:417-426,
// :490-491) without materialising the [V] log-prob row.
template <class T, int NTH>
__global__ void __launch_bounds__(NTH) logprob_gather_kernel(const T* __restrict__ logits, int64_t ld, int64_t rows,
                                                             int64_t V, const int32_t* __restrict__ target,
                                                             const int64_t* __restrict__ out_index,
                                                             double* __restrict__ out) {
  PDL_ENTRY();
  constexpr int N = 16 / sizeof(T);
  constexpr float kLog2e = 1.4426950408889634f;
  __shared__ float sm_m[NTH / 32], sm_s[NTH / 32];
  const int64_t r = blockIdx.x;
  const int tgt = target[r];
  if (tgt < 0) return;
  const T* row = logits + r * ld;
  float m = -INFINITY, s = 0.f;  // s is scaled by 2^(-m*log2e)
  const int64_t nvec = V / N;
  const uint4* rv = reinterpret_cast<const uint4*>(row);
  constexpr int U = 4;
  int64_t v0 = threadIdx.x;
  for (; v0 + (U - 1) * NTH < nvec; v0 += U * NTH) {
    Vec16<T> x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u].u = __ldcs(rv + v0 + u * NTH);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float lm = to_f(x[u].v[0]);
#pragma unroll
      for (int k = 1; k < N; ++k) lm = fmaxf(lm, to_f(x[u].v[k]));
      if (lm > m) {
        s *= exp2f((m - lm) * kLog2e);
        m = lm;
      }
      const float mb = m * kLog2e;
#pragma unroll
      for (int k = 0; k < N; ++k) s += exp2f(fmaf(to_f(x[u].v[k]), kLog2e, -mb));
    }
  }
  for (; v0 < nvec; v0 += NTH) {
    Vec16<T> x;
    x.u = __ldcs(rv + v0);
    float lm = to_f(x.v[0]);
#pragma unroll
    for (int k = 1; k < N; ++k) lm = fmaxf(lm, to_f(x.v[k]));
    if (lm > m) {
      s *= exp2f((m - lm) * kLog2e);
      m = lm;
    }
#pragma unroll
    for (int k = 0; k < N; ++k) s += exp2f((to_f(x.v[k]) - m) * kLog2e);
  }
  for (int64_t j = nvec * N + threadIdx.x; j < V; j += NTH) {
    const float v = to_f(row[j]);
    if (v > m) {
      s *= exp2f((m - v) * kLog2e);
      m = v;
    }
    s += exp2f((v - m) * kLog2e);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float M = fmaxf(m, m2);
    s = (m == -INFINITY ? 0.f : s * exp2f((m - M) * kLog2e)) + (m2 == -INFINITY ? 0.f : s2 * exp2f((m2 - M) * kLog2e));
    m = M;
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sm_m[w] = m;
    sm_s[w] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = sm_m[0];
    for (int k = 1; k < NTH / 32; ++k) M = fmaxf(M, sm_m[k]);
    float S = 0.f;
    for (int k = 0; k < NTH / 32; ++k) S += sm_m[k] == -INFINITY ? 0.f : sm_s[k] * exp2f((sm_m[k] - M) * kLog2e);
    out[out_index[r]] = double(to_f(row[tgt]) - (M + logf(S)));
  }
}

// K9f combine: the fused LM-head GEMM (Epi::kLse) leaves one (max, sum exp)
// pair per 256-column tile; a warp per row merges them in fp64 and gathers:
// lp = l[target] - (M + log sum_j s_j exp(m_j - M)).
__global__ void lse_combine_kernel(const float2* __restrict__ part, int ldp, int ntiles,
                                   const float* __restrict__ tgt_logit, const int32_t* __restrict__ target,
                                   int64_t rows, const int64_t* __restrict__ out_index, double* __restrict__ out) {
  PDL_ENTRY();
  const int64_t r = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows || target[r] < 0) return;
  const float2* p = part + r * ldp;
  float M = -INFINITY;
  for (int j = lane; j < ntiles; j += 32) M = fmaxf(M, p[j].x);
  M = warp_max(M);
  double S = 0.0;
  for (int j = lane; j < ntiles; j += 32) S += double(p[j].y) * exp(double(p[j].x) - double(M));
  S = warp_sum_d(S);
  if (lane == 0) out[out_index[r]] = double(tgt_logit[r]) - (double(M) + log(S));
}

// ------------------------------------------------------------------ K11
// One warp per sequence.  Shaping (kl_penalized_rewards, src/losses.cpp:188-199):
//   r_t = -kl_coef * (a_t - ref_t);  r_{n-1} += R
// GAE (src/losses.cpp:168-186), V_n = 0:
//   delta_t = r_t + gamma * V_{t+1} - V_t;  A_t = delta_t + gamma*lam*A_{t+1};  R_t = A_t + V_t
// The reverse recurrence runs as 32-wide chunks from the end: a weighted
// suffix scan with shuffles inside the chunk plus the carried A of the chunk
// to the right.  fp64 throughout.
__global__ void shape_gae_kernel(int64_t B, int64_t stride, const int64_t* __restrict__ lengths,
                                 const double* __restrict__ rm_reward, const double* __restrict__ actor,
                                 const double* __restrict__ ref, const double* __restrict__ values, double kl_coef,
                                 double gamma, double lam, double* __restrict__ shaped, double* __restrict__ adv,
                                 double* __restrict__ ret, double* __restrict__ part) {
  PDL_ENTRY();
  const int64_t b = blockIdx.x;
  if (b >= B) return;
  const int lane = threadIdx.x;
  const int64_t n = lengths[b], base = b * stride;
  const double R = rm_reward[b];
  const double c = gamma * lam;
  const double cpow_tail = pow(c, double(32 - lane));  // c^(chunk_end - t)
  double carry = 0.0, kl = 0.0, as = 0.0, aq = 0.0;
  for (int64_t end = n; end > 0; end -= 32) {
    const int64_t t = end - 32 + lane;
    const bool valid = t >= 0;
    double a_t = 0, r_t = 0, v_t = 0, v_next = 0, rw = 0, delta = 0;
    if (valid) {
      a_t = actor[base + t];
      r_t = ref[base + t];
      v_t = values[base + t];
      v_next = (t + 1 < n) ? values[base + t + 1] : 0.0;
      rw = -kl_coef * (a_t - r_t);
      if (t == n - 1) rw += R;
      delta = rw + gamma * v_next - v_t;
    }
    double S = delta, cp = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double other = __shfl_down_sync(0xffffffffu, S, o);
      if (lane + o < 32) S += cp * other;
      cp *= cp;
    }
    const double A = S + cpow_tail * carry;
    if (valid) {
      shaped[base + t] = rw;
      adv[base + t] = A;
      ret[base + t] = A + v_t;
      kl += a_t - r_t;
      as += A;
      aq += A * A;
    }
    carry = __shfl_sync(0xffffffffu, A, 0);
  }
  kl = warp_sum_d(kl);
  as = warp_sum_d(as);
  aq = warp_sum_d(aq);
  if (lane == 0) {
    part[b * 5 + 0] = kl;
    part[b * 5 + 1] = double(n);
    part[b * 5 + 2] = R;
    part[b * 5 + 3] = as;
    part[b * 5 + 4] = aq;
  }
}

// Fixed-order (deterministic) reduction of the per-sequence partials.
__global__ void reduce_partials_kernel(int64_t B, const double* __restrict__ part, double* __restrict__ out5) {
  PDL_ENTRY();
  __shared__ double sm[5][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;  // 5 warps, one per field
  if (w >= 5) return;
  double s = 0.0;
  for (int64_t b = lane; b < B; b += 32) s += part[b * 5 + w];
  sm[w][lane] = s;
  __syncwarp();
  if (lane == 0) {
    double t = 0.0;
    for (int k = 0; k < 32; ++k) t += sm[w][k];
    out5[w] = t;
  }
}

// w = (a - mean) / sqrt(var + 1e-8); stats3 = (n, sum a, sum a^2) over all ranks.
__global__ void whiten_apply_kernel(int64_t B, int64_t stride, const int64_t* __restrict__ lengths,
                                    const double* __restrict__ adv, const double* __restrict__ st,
                                    double* __restrict__ out) {
  PDL_ENTRY();
  const double cnt = st[0] > 0 ? st[0] : 1.0;
  const double mean = st[1] / cnt;
  double var = st[2] / cnt - mean * mean;
  if (var < 0) var = 0;
  const double inv = 1.0 / sqrt(var + 1e-8);
  const int64_t b = blockIdx.x;
  for (int64_t t = threadIdx.x; t < lengths[b]; t += blockDim.x) out[b * stride + t] = (adv[b * stride + t] - mean) * inv;
}

}  // namespace

template <class T>
void launch_logprob_gather(Ctx& c, const T* logits, int64_t ld, int64_t rows, int64_t V, const int32_t* target,
                           const int64_t* out_index, double* out) {
  if (rows <= 0) return;
  if ((ld * sizeof(T)) % 16) throw ContractError("logprob_gather: row stride must be 16-byte aligned");
  c.launch("logprob_gather", double(rows) * V * sizeof(T) + rows * 20.0, 0, [&] {
    launch_kernel(c, logprob_gather_kernel<T, 256>, dim3(rows), dim3(256), 0, 1, logits, ld, rows, V, target, out_index, out);
  });
}

void launch_lse_combine(Ctx& c, const float2* part, int ldp, int ntiles, const float* tgt_logit,
                        const int32_t* target, int64_t rows, const int64_t* out_index, double* out) {
  if (rows <= 0) return;
  c.launch("lse_combine", double(rows) * (ntiles * 8.0 + 20.0), 0, [&] {
    launch_kernel(c, lse_combine_kernel, dim3(ceil_div(rows, 8)), dim3(256), 0, 1, part, ldp, ntiles, tgt_logit, target,
                  rows, out_index, out);
  });
}

void launch_shape_gae(Ctx& c, int64_t B, int64_t stride, const int64_t* lengths, const double* rm_reward,
                      const double* actor_lp, const double* ref_lp, const double* values, double kl_coef,
                      double gamma, double lam, double* shaped, double* adv, double* ret, double* part) {
  if (B <= 0) return;
  c.launch("shape_gae", double(B) * stride * 8 * 7, 0, [&] {
    launch_kernel(c, shape_gae_kernel, dim3(B), dim3(32), 0, 1, B, stride, lengths, rm_reward, actor_lp, ref_lp, values, kl_coef, gamma,
                                             lam, shaped, adv, ret, part);
  });
}

void launch_reduce_partials(Ctx& c, int64_t B, const double* part, double* out5) {
  c.launch("reduce_partials", double(B) * 40, 0,
           [&] { launch_kernel(c, reduce_partials_kernel, dim3(1), dim3(160), 0, 1, B, part, out5); });
}

void launch_whiten_apply(Ctx& c, int64_t B, int64_t stride, const int64_t* lengths, const double* adv,
                         const double* stats3, double* out) {
  if (B <= 0) return;
  c.launch("whiten", double(B) * stride * 16, 0,
           [&] { launch_kernel(c, whiten_apply_kernel, dim3(B), dim3(128), 0, 1, B, stride, lengths, adv, stats3, out); });
}

template void launch_logprob_gather<float>(Ctx&, const float*, int64_t, int64_t, int64_t, const int32_t*,
                                           const int64_t*, double*);
template void launch_logprob_gather<bf16>(Ctx&, const bf16*, int64_t, int64_t, int64_t, const int32_t*,
                                          const int64_t*, double*);

}  // namespace ppx
