// sampler.cu — K8: fused per-row sampler over the decode logits.
//
// Reference semantics (src/model.cpp:450-478):
//   lp(tok) = log_softmax(logits)[tok] (untempered, recorded for every token)
//   greedy : argmax, first index wins on ties (argmax_index, :428-434)
//   sampled: q_j = exp((l_j - max)/max(tau,1e-12)); u = uniform()*sum(q);
//            first j with u < cumsum_j (index order), fallback V-1 (:455-473)
// North-star extension (oracle/ppoexp_oracle.c orc_filter_topk_topp): top-k
// then top-p filtering of q before the inverse CDF; with k = 0 and p >= 1 the
// kernel is exactly the reference sampler.
//
// One 1024-thread CTA per sequence.  Thresholds for top-k / top-p come from a
// 4-pass radix select over the fp32 bit patterns of q (positive floats sort
// like their bits), with 256-bin (count, fp64 sum) histograms in smem; the
// inverse CDF runs over warp-contiguous index ranges with warp shuffles, so
// every pass reads the row coalesced.
#include <cfloat>

#include "kernels.hpp"

namespace ppoexp {

namespace {
constexpr int NT = 1024, NW = NT / 32;

struct Shared {
  float fm[NW];
  int fi[NW];
  float fs[NW];
  double dsum[NW];
  int icount[NW];
  unsigned cnt[256];
  double hs[256];
  double zsum;
  unsigned prefix, mask;
  double s_above;
  unsigned c_above;
  int chosen_bin;
  int result;
};

__device__ __forceinline__ float qval(const float* row, int64_t j, float M, float inv_tau) {
  return expf((row[j] - M) * inv_tau);
}

// mode 0: select by count (top-k: want k), mode 1: select by sum (top-p: want target).
// On exit: sh.prefix = threshold bits t; sh.c_above = #(q > t); sh.s_above = sum(q > t);
// returns #(q == t) via sh.cnt[chosen_bin] of the last pass.
__device__ void radix_select(const float* row, int64_t V, float M, float inv_tau, int mode, double want, Shared& sh,
                             unsigned& eq_count) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    sh.prefix = 0;
    sh.mask = 0;
    sh.s_above = 0.0;
    sh.c_above = 0;
  }
  __syncthreads();
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int i = tid; i < 256; i += NT) {
      sh.cnt[i] = 0;
      sh.hs[i] = 0.0;
    }
    __syncthreads();
    const unsigned prefix = sh.prefix, mask = sh.mask;
    for (int64_t j = tid; j < V; j += NT) {
      const float q = qval(row, j, M, inv_tau);
      const unsigned bits = __float_as_uint(q);
      if ((bits & mask) == prefix) {
        const int bin = (bits >> shift) & 255;
        atomicAdd(&sh.cnt[bin], 1u);
        if (mode == 1) atomicAdd(&sh.hs[bin], double(q));
      }
    }
    __syncthreads();
    if (tid == 0) {
      // Walk bins from the largest q down; stop at the first bin whose
      // inclusion reaches `want`.  c_above / s_above exclude the chosen bin.
      unsigned ca = sh.c_above;
      double sa = sh.s_above;
      int chosen = -1, lowest = -1;
      for (int bin = 255; bin >= 0; --bin) {
        if (sh.cnt[bin] == 0) continue;
        lowest = bin;
        const bool hit = mode == 0 ? double(ca + sh.cnt[bin]) >= want : sa + sh.hs[bin] >= want;
        if (hit) {
          chosen = bin;
          break;
        }
        ca += sh.cnt[bin];
        sa += sh.hs[bin];
      }
      if (chosen < 0) {  // rounding: nothing reached `want`; keep down to the lowest bin
        chosen = lowest < 0 ? 0 : lowest;
        ca -= sh.cnt[chosen];
        sa -= sh.hs[chosen];
      }
      sh.chosen_bin = chosen;
      sh.c_above = ca;
      sh.s_above = sa;
      sh.prefix = prefix | (unsigned(chosen) << shift);
      sh.mask = mask | (255u << shift);
    }
    __syncthreads();
  }
  eq_count = sh.cnt[sh.chosen_bin];
  __syncthreads();
}

__global__ void __launch_bounds__(NT) sampler_kernel(const float* __restrict__ logits, int64_t ld, int64_t V,
                                                     SamplerState s) {
  __shared__ Shared sh;
  const int64_t b = blockIdx.x;
  const SampleParams prm = s.params[b];
  const int greedy = prm.greedy;
  const float temperature = prm.temperature;
  const int64_t top_k = prm.top_k;
  const double top_p = prm.top_p;
  if (s.done[b]) return;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const float* row = logits + b * ld;
  const int i = s.n_gen[b];

  // pass 1: max, first argmax, online sum of exp(l - max)
  float m = -INFINITY, se = 0.f;
  int am = 0x7fffffff;
  for (int64_t j = tid; j < V; j += NT) {
    const float v = row[j];
    if (v > m) {
      se = se * expf(m - v) + 1.f;
      m = v;
      am = int(j);
    } else {
      se += expf(v - m);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const int a2 = __shfl_xor_sync(0xffffffffu, am, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, se, o);
    const float M = fmaxf(m, m2);
    const float sc = (m == -INFINITY ? 0.f : se * expf(m - M)) + (m2 == -INFINITY ? 0.f : s2 * expf(m2 - M));
    am = m > m2 ? am : (m2 > m ? a2 : min(am, a2));
    m = M;
    se = sc;
  }
  if (lane == 0) {
    sh.fm[w] = m;
    sh.fi[w] = am;
    sh.fs[w] = se;
  }
  __syncthreads();
  float M = sh.fm[0];
  int AM = sh.fi[0];
  for (int k = 1; k < NW; ++k) {
    if (sh.fm[k] > M || (sh.fm[k] == M && sh.fi[k] < AM)) AM = sh.fm[k] > M ? sh.fi[k] : min(AM, sh.fi[k]);
    M = fmaxf(M, sh.fm[k]);
  }
  float SE = 0.f;
  for (int k = 0; k < NW; ++k) SE += sh.fm[k] == -INFINITY ? 0.f : sh.fs[k] * expf(sh.fm[k] - M);
  const float lse = M + logf(SE);

  int chosen = AM;
  if (!greedy) {
    const float tau = fmaxf(temperature, 1e-12f);
    const float inv_tau = 1.0f / tau;
    const bool filt_k = top_k > 0 && top_k < V;
    const bool filt_p = top_p < 1.0;
    // kept(j): q > t_final, or q == t_final and tie-rank(j) < c_final
    unsigned t_final = 0;      // bits; 0 with c_final = ~0 keeps everything
    unsigned c_final = 0xffffffffu;
    bool filtering = filt_k || filt_p;
    if (filtering) {
      unsigned eq = 0, tk = 0, ck = 0xffffffffu;
      double zk = 0.0;
      if (filt_k) {
        radix_select(row, V, M, inv_tau, 0, double(top_k), sh, eq);
        tk = sh.prefix;
        ck = unsigned(top_k) - sh.c_above;
        zk = sh.s_above + double(ck) * double(__uint_as_float(tk));
        // s_above for mode 0 was not accumulated; recompute sum(q > tk) directly
        double part = 0.0;
        for (int64_t j = tid; j < V; j += NT) {
          const float q = qval(row, j, M, inv_tau);
          if (__float_as_uint(q) > tk) part += double(q);
        }
        part = warp_sum_d(part);
        if (lane == 0) sh.dsum[w] = part;
        __syncthreads();
        double sa = 0.0;
        for (int k = 0; k < NW; ++k) sa += sh.dsum[k];
        __syncthreads();
        zk = sa + double(ck) * double(__uint_as_float(tk));
        t_final = tk;
        c_final = ck;
      }
      if (filt_p) {
        if (!filt_k) {
          double part = 0.0;
          for (int64_t j = tid; j < V; j += NT) part += double(qval(row, j, M, inv_tau));
          part = warp_sum_d(part);
          if (lane == 0) sh.dsum[w] = part;
          __syncthreads();
          zk = 0.0;
          for (int k = 0; k < NW; ++k) zk += sh.dsum[k];
          __syncthreads();
        }
        const double target = top_p * zk;
        radix_select(row, V, M, inv_tau, 1, target, sh, eq);
        unsigned tp = sh.prefix;
        const double tq = double(__uint_as_float(tp));
        double need = tq > 0.0 ? ceil((target - sh.s_above) / tq) : double(eq);
        if (need < 1.0) need = 1.0;
        if (need > double(eq)) need = double(eq);
        unsigned cp = unsigned(need);
        if (filt_k) {
          if (tp < tk) {
            tp = tk;
            cp = ck;
          } else if (tp == tk) {
            cp = min(cp, ck);
          }
        }
        t_final = tp;
        c_final = cp;
      }
    }
    // ---- inverse CDF over warp-contiguous ranges
    const int64_t CW = ((V + NW - 1) / NW + 31) / 32 * 32;  // elements per warp, multiple of 32
    const int64_t w0 = int64_t(w) * CW, w1 = (V < w0 + CW ? V : w0 + CW);
    // tie counts per warp (only needed when ties are partially kept)
    int tie_base = 0;
    if (filtering) {
      int ties = 0;
      for (int64_t j = w0 + lane; j < w1; j += 32)
        ties += __float_as_uint(qval(row, j, M, inv_tau)) == t_final;
      ties = __reduce_add_sync(0xffffffffu, ties);
      if (lane == 0) sh.icount[w] = ties;
      __syncthreads();
      for (int k = 0; k < w; ++k) tie_base += sh.icount[k];
    }
    auto kept_step = [&](int64_t j, int& tie_run, float& q) -> bool {
      // all 32 lanes call this together for j = base + lane
      q = j < w1 ? qval(row, j, M, inv_tau) : 0.f;
      if (!filtering) return j < w1;
      const unsigned bits = __float_as_uint(q);
      const bool tie = j < w1 && bits == t_final;
      const unsigned tb = __ballot_sync(0xffffffffu, tie);
      const int rank = tie_run + __popc(tb & ((1u << lane) - 1u));
      tie_run += __popc(tb);
      return j < w1 && (bits > t_final || (tie && unsigned(rank) < c_final));
    };
    double wsum = 0.0;
    int last_kept = -1;
    {
      int tie_run = tie_base;
      for (int64_t base = w0; base < w1; base += 32) {
        float q;
        const bool k = kept_step(base + lane, tie_run, q);
        if (k) {
          wsum += double(q);
          last_kept = int(base + lane);
        }
      }
    }
    wsum = warp_sum_d(wsum);
    int lk = last_kept;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lk = max(lk, __shfl_xor_sync(0xffffffffu, lk, o));
    if (lane == 0) {
      sh.dsum[w] = wsum;
      sh.fi[w] = lk;
    }
    if (tid == 0) sh.result = 0x7fffffff;
    __syncthreads();
    double prefix = 0.0, total = 0.0;
    int fallback = -1;
    for (int k = 0; k < NW; ++k) {
      if (k < w) prefix += sh.dsum[k];
      total += sh.dsum[k];
      fallback = max(fallback, sh.fi[k]);
    }
    const double u = s.uniforms[b * s.ustride + i];
    const double target = u * total;
    // the crossing can only be in a warp whose [prefix, prefix + wsum] brackets target
    if (prefix <= target && target < prefix + sh.dsum[w] * (1.0 + 1e-12) + 1e-300) {
      int tie_run = tie_base;
      double acc = prefix;
      for (int64_t base = w0; base < w1; base += 32) {
        float q;
        const bool k = kept_step(base + lane, tie_run, q);
        // inclusive warp scan of kept q (index order)
        double v = k ? double(q) : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double t = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += t;
        }
        const double cum = acc + v;
        const unsigned hit = __ballot_sync(0xffffffffu, k && target < cum);
        if (hit) {
          if (lane == 0) atomicMin(&sh.result, int(base + __ffs(hit) - 1));
          break;
        }
        acc += __shfl_sync(0xffffffffu, v, 31);
      }
    }
    __syncthreads();
    chosen = sh.result != 0x7fffffff ? sh.result : (fallback >= 0 ? fallback : int(V - 1));
  }
  if (tid == 0) {
    if (i > 0) s.pos[b] += 1;
    s.out_tokens[b * s.ostride + i] = chosen;
    s.out_lps[b * s.ostride + i] = row[chosen] - lse;
    s.next_tok[b] = chosen;
    s.n_gen[b] = i + 1;
    if (chosen == kEotToken || i + 1 >= s.budget[b]) {
      s.done[b] = 1;
      atomicSub(s.n_active, 1);
    }
  }
}
}  // namespace

void launch_sampler(Ctx& c, const float* logits, int64_t ld, int64_t B, int64_t V, const SamplerState& s) {
  if (B <= 0) return;
  c.launch("sampler", double(B) * V * 4, 0, [&] { sampler_kernel<<<B, NT, 0, c.stream>>>(logits, ld, V, s); });
}

}  // namespace ppoexp
