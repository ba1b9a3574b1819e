// sampler.cu — K8: fused per-row sampler over the decode logits.
//
// Reference semantics (src/model.cpp:450-478):
//   lp(tok) = log_softmax(logits)[tok] (untempered, recorded for every token)
//   greedy : argmax, first index wins on ties (argmax_index, :428-434)
//   sampled: q_j = exp((l_j - max)/max(tau,1e-12)); u = uniform()*sum(q);
//            first j with u < cumsum_j (index order), fallback V-1 (:455-473)
// North-star extension (convention in oracle/ppoexp_oracle.c,
// orc_filter_topk_topp): top-k then top-p over q sorted by (q desc, index
// asc); the inverse CDF then runs in index order over the kept tokens.  With
// k = 0 and p >= 1 this is exactly the reference sampler.
//
// One 1024-thread CTA per sequence.  Sampled rows cache q in shared memory
// (V <= 52k) so every pass after the first is on-chip.  Thresholds: a
// 1024-bucket histogram keyed by the fp32 bit pattern of q (monotone in q and
// log-spaced, so flat and peaked rows both spread), a block scan to find the
// crossing bucket, and an exact (q desc, index asc) bitonic sort of that
// bucket alone.  The kept set is {q > t} ∪ {q == t, index <= cut}.  The
// inverse CDF runs over warp-contiguous index ranges with warp scans.
#include <cooperative_groups.h>

#include <cfloat>

#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace ppx {

namespace {
constexpr int NT = 1024, NW = NT / 32, NB = 1024, LIST = 1024;
constexpr int64_t kCacheMaxV = 50600;
constexpr double kFix = 1.0 / 65536.0;  // 2^-16 (V * 2^16 < 2^32: no overflow)

struct Shared {
  unsigned hcnt[NB];
  unsigned hsum[NB];  // approximate bucket sums, fixed point q * 2^16 (native 32-bit smem atomics)
  unsigned long long list[LIST];
  unsigned long long list2[256];  // rank-sort output for small crossing buckets
  float fm[NW], fmn[NW], fs[NW];
  int fi[NW];
  double dsum[NW];
  unsigned uwarp[NW + 1];
  double dwarp[NW + 1];
  int lk[NW];
  int list_n;
  int result;
  // selection state
  int bk, bp;
  unsigned c_above;
  double s_above, zk, zk_bucket;
  unsigned t_final;
  int idx_cut;
  int overflow;
  // CTA-pair exchange slots (two, alternating)
  float xf[2][4];
  int xi[2][4];
  unsigned xu[2][4];
  double xd[2][4];
};

__device__ __forceinline__ unsigned qbits_of(float q) { return __float_as_uint(q); }

// bucket 0 = largest q (bits of 1.0), NB-1 = smallest:
//   b = floor((top - bits) * scale / 2^32),  scale = floor(2^32 * NB / span).
// Integer multiply-high only (no conversions: they are quarter-rate); monotone
// in the bits, so equal q map to equal buckets and larger q to lower ones.
__device__ __forceinline__ int bucket_of(unsigned bits, unsigned top, unsigned scale) {
  const int b = int(__umulhi(top - bits, scale));  // bits <= top
  return b >= NB ? NB - 1 : b;
}

template <class T>
__device__ T block_excl_scan(T v, T* wtot, T& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) wtot[w] = inc;
  __syncthreads();
  if (w == 0) {
    T x = wtot[lane];
    T xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T t = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += t;
    }
    wtot[lane] = xi - x;  // exclusive warp prefix
    if (lane == 31) wtot[NW] = xi;
  }
  __syncthreads();
  const T res = wtot[w] + inc - v;
  total = wtot[NW];
  __syncthreads();
  return res;
}

__device__ double block_sum_d(double v, Shared& sh) {
  v = warp_sum_d(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh.dsum[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int k = 0; k < NW; ++k) t += sh.dsum[k];  // fixed order
  __syncthreads();
  return t;
}

// sort a[0..n) ascending (padded to a power of two with ~0 keys)
__device__ void bitonic_sort(unsigned long long* a, int n) {
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = n + threadIdx.x; i < m; i += NT) a[i] = ~0ull;
  __syncthreads();
  for (int k = 2; k <= m; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < m; i += NT) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const unsigned long long x = a[i], y = a[l];
          if ((x > y) == up) {
            a[i] = y;
            a[l] = x;
          }
        }
      }
      __syncthreads();
    }
}

// sort sh.list[0..n) ascending: small lists (the usual crossing bucket) by
// rank counting (keys are unique: the index is part of the key), one pass and
// one barrier; larger ones by the bitonic network
template <class S>
__device__ void sort_list(S& sh, int n) {
  if (n <= 256) {
    if (threadIdx.x < n) {
      const unsigned long long key = sh.list[threadIdx.x];
      int rank = 0;
      for (int k = 0; k < n; ++k) rank += sh.list[k] < key;
      sh.list2[rank] = key;
    }
    __syncthreads();
    if (threadIdx.x < n) sh.list[threadIdx.x] = sh.list2[threadIdx.x];
    __syncthreads();
  } else {
    bitonic_sort(sh.list, n);
  }
}

// key = (q desc, index asc) ascending
__device__ __forceinline__ unsigned long long sort_key(unsigned qb, int idx) {
  return ((unsigned long long)(~qb) << 32) | unsigned(idx);
}
__device__ __forceinline__ float key_q(unsigned long long e) { return __uint_as_float(~unsigned(e >> 32)); }

// Cluster helpers (CL = 2: a row split over a CTA pair).  A row-global value
// is combined by writing this CTA's part to a shared slot, one cluster
// barrier, and reading the partner's slot through DSMEM; parts are combined in
// rank order, so both CTAs hold identical, deterministic results.
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
template <class T>
__device__ __forceinline__ const T* peer_ptr(const T* p, unsigned rank) {
  return static_cast<const T*>(cg::this_cluster().map_shared_rank(const_cast<T*>(p), rank));
}

template <bool CACHED, int CL>
__global__ void __launch_bounds__(NT) sampler_kernel(const float* __restrict__ logits, int64_t ld, int64_t V,
                                                     SamplerState s) {
  PDL_ENTRY();
  extern __shared__ __align__(16) float qcache[];  // CACHED: this CTA's part of the row (logits, then q)
  __shared__ Shared sh;
  const unsigned r = CL > 1 ? cl_rank() : 0u, pr = r ^ 1u;
  const int64_t b = blockIdx.x / CL;
  if (s.done[b]) return;  // both CTAs of a row return together
  // this CTA's index range [jlo, jhi): halves rounded to 16 bytes
  const int64_t half = CL > 1 ? (V + 7) / 8 * 4 : V;
  const int64_t jlo = int64_t(r) * half, jhi = V < jlo + half ? V : jlo + half;
  const SampleParams prm = s.params[b];
  auto stamp = [&](int k) {
    if (s.dbg && b == 0 && r == 0 && threadIdx.x == 0) s.dbg[k] = clock64();
  };
  stamp(0);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const float* row = logits + b * ld;
  const int i = s.n_gen[b];
  int xs = 0;  // exchange slot (alternates: a slot is rewritten only two barriers later)

  // ---- pass 1: max, min, first argmax over [jlo, jhi) (16-byte loads;
  // ascending index per thread keeps "first index wins" exact); the logits
  // are cached in shared memory on the way
  float m = -INFINITY, mn = INFINITY;
  int am = 0x7fffffff;
  auto visit = [&](float v, int j) {
    if (v > m) {
      m = v;
      am = j;
    }
    mn = fminf(mn, v);
  };
  {
    const int64_t nv = (jhi - jlo) / 4;
    const float4* r4 = reinterpret_cast<const float4*>(row + jlo);
    float4* c4 = reinterpret_cast<float4*>(qcache);
    // up to 8 float4 per thread in flight before the first compare
    for (int64_t k0 = tid; k0 < nv; k0 += 8 * NT) {
      float4 a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (k0 + u * NT < nv) a[u] = r4[k0 + u * NT];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t k = k0 + u * NT;
        if (k < nv) {
          if constexpr (CACHED) c4[k] = a[u];
          const int j0 = int(jlo + 4 * k);
          visit(a[u].x, j0); visit(a[u].y, j0 + 1); visit(a[u].z, j0 + 2); visit(a[u].w, j0 + 3);
        }
      }
    }
    for (int64_t j = jlo + nv * 4 + tid; j < jhi; j += NT) {
      const float v = row[j];
      if constexpr (CACHED) qcache[j - jlo] = v;
      visit(v, int(j));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const int a2 = __shfl_xor_sync(0xffffffffu, am, o);
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    am = m > m2 ? am : (m2 > m ? a2 : min(am, a2));
    m = fmaxf(m, m2);
  }
  if (lane == 0) {
    sh.fm[w] = m;
    sh.fi[w] = am;
    sh.fmn[w] = mn;
  }
  __syncthreads();
  float M = sh.fm[0], MN = sh.fmn[0];
  int AM = sh.fi[0];
  for (int k = 1; k < NW; ++k) {
    if (sh.fm[k] > M || (sh.fm[k] == M && sh.fi[k] < AM)) AM = sh.fm[k] > M ? sh.fi[k] : min(AM, sh.fi[k]);
    M = fmaxf(M, sh.fm[k]);
    MN = fminf(MN, sh.fmn[k]);
  }
  if constexpr (CL > 1) {
    if (tid == 0) {
      sh.xf[xs][0] = M;
      sh.xf[xs][1] = MN;
      sh.xi[xs][0] = AM;
    }
    cl_sync();
    const float M2 = peer_ptr(&sh.xf[xs][0], pr)[0], MN2 = peer_ptr(&sh.xf[xs][0], pr)[1];
    const int AM2 = peer_ptr(&sh.xi[xs][0], pr)[0];
    AM = M > M2 ? AM : (M2 > M ? AM2 : min(AM, AM2));
    M = fmaxf(M, M2);
    MN = fminf(MN, MN2);
    xs ^= 1;
  }
  stamp(1);
  // row-global float sum of per-CTA block totals, in rank order
  auto row_sum_f = [&](float v) -> float {
    if constexpr (CL > 1) {
      if (tid == 0) sh.xf[xs][2] = v;
      cl_sync();
      const float o = peer_ptr(&sh.xf[xs][0], pr)[2];
      xs ^= 1;
      return r == 0 ? v + o : o + v;
    } else {
      return v;
    }
  };
  auto row_sum_d2 = [&](double& a, double& c) {  // two fp64 block totals, rank order
    if constexpr (CL > 1) {
      if (tid == 0) {
        sh.xd[xs][0] = a;
        sh.xd[xs][1] = c;
      }
      cl_sync();
      const double* o = peer_ptr(&sh.xd[xs][0], pr);
      const double oa = o[0], oc = o[1];
      a = r == 0 ? a + oa : oa + a;
      c = r == 0 ? c + oc : oc + c;
      xs ^= 1;
    }
  };
  // sum exp(l - M) for the untempered log-prob (src/model.cpp:450); when the
  // row is sampled at tau == 1 it is folded into pass 2 (q == exp(l - M))
  const bool fold = !prm.greedy && prm.temperature == 1.0f;
  float lse = 0.f;
  if (!fold) {
    float se = 0.f;
    for (int64_t j = jlo + tid; j < jhi; j += NT) se += expf(row[j] - M);
    se = warp_sum(se);
    __syncthreads();
    if (lane == 0) sh.fs[w] = se;
    __syncthreads();
    float SE = 0.f;
    for (int k = 0; k < NW; ++k) SE += sh.fs[k];
    lse = M + logf(row_sum_f(SE));
  }

  int chosen = AM;
  if (!prm.greedy) {
    const float tau = fmaxf(prm.temperature, 1e-12f);
    const float inv_tau = 1.0f / tau;
    const bool filt_k = prm.top_k > 0 && prm.top_k < V;
    const bool filt_p = prm.top_p < 1.0;
    const bool filtering = filt_k || filt_p;
    auto Q = [&](int64_t j) -> float {  // j in [jlo, jhi)
      if constexpr (CACHED) return qcache[j - jlo];
      else return expf((row[j] - M) * inv_tau);
    };
    // any j (the overflow path, run by rank 0 alone): the partner's part through DSMEM
    const float* pq = CL > 1 ? peer_ptr(qcache, pr) : qcache;
    auto Qall = [&](int64_t j) -> float {
      if constexpr (CACHED) {
        if (j >= jlo && j < jhi) return qcache[j - jlo];
        return pq[j - int64_t(pr) * half];
      } else {
        return expf((row[j] - M) * inv_tau);
      }
    };
    // bucket span: bits(1.0) .. bits(q_min); q is monotone in the logit
    const unsigned top = qbits_of(1.0f);
    const unsigned botb = qbits_of(expf((MN - M) * inv_tau));
    const unsigned long long span = (unsigned long long)(top - botb) + 1ull;
    const unsigned scale = unsigned(((unsigned long long)NB << 32) / span);  // (span - 1) * scale < NB * 2^32
    // ---- pass 2: q (cached), histogram
    if (filtering)
      for (int k = tid; k < NB; k += NT) {
        sh.hcnt[k] = 0;
        sh.hsum[k] = 0u;
      }
    __syncthreads();
    double zloc = 0.0;
    float fsum = 0.f;
    auto pass2 = [&](float q) {
      fsum += q;
      if (filtering) {
        zloc += double(q);
        const int bk = bucket_of(qbits_of(q), top, scale);
        atomicAdd(&sh.hcnt[bk], 1u);
        atomicAdd(&sh.hsum[bk], __float2uint_rn(q * 65536.0f));
      }
    };
    if constexpr (CACHED) {
      // the logits are in shared memory (pass 1): float4 in-place transform
      float4* c4 = reinterpret_cast<float4*>(qcache);
      const int nloc = int(jhi - jlo), nv = nloc / 4;
      for (int k4 = tid; k4 < nv; k4 += NT) {
        float4 l = c4[k4];
        l.x = expf((l.x - M) * inv_tau);
        l.y = expf((l.y - M) * inv_tau);
        l.z = expf((l.z - M) * inv_tau);
        l.w = expf((l.w - M) * inv_tau);
        c4[k4] = l;
        pass2(l.x);
        pass2(l.y);
        pass2(l.z);
        pass2(l.w);
      }
      for (int j = nv * 4 + tid; j < nloc; j += NT) {
        const float q = expf((qcache[j] - M) * inv_tau);
        qcache[j] = q;
        pass2(q);
      }
    } else {
      for (int64_t j = jlo + tid; j < jhi; j += NT) pass2(expf((row[j] - M) * inv_tau));
    }
    if (fold) {  // lse from the same exp pass (tau == 1)
      fsum = warp_sum(fsum);
      if (lane == 0) sh.fs[w] = fsum;
      __syncthreads();
      float SE = 0.f;
      for (int k = 0; k < NW; ++k) SE += sh.fs[k];
      lse = M + logf(row_sum_f(SE));
    }
    __syncthreads();
    stamp(2);
    unsigned t_final = 0;
    int idx_cut = int(V);  // keep everything
    if (filtering) {
      double Z = block_sum_d(zloc, sh), unused = 0.0;
      if constexpr (CL > 1) {
        // the pair's histograms are merged into hcnt/hsum of both CTAs: partner
        // values are read into registers first, then (after a barrier that keeps
        // the partner from reading half-updated bins) added in rank order
        row_sum_d2(Z, unused);  // (the barrier here also publishes the histograms)
        unsigned pc = 0, psum = 0;
        if (tid < NB) {
          pc = peer_ptr(sh.hcnt, pr)[tid];
          psum = peer_ptr(sh.hsum, pr)[tid];
        }
        cl_sync();
        if (tid < NB) {
          sh.hcnt[tid] += pc;  // integer sums: order-independent
          sh.hsum[tid] += psum;
        }
        __syncthreads();
      }
      stamp(3);
      if (tid == 0) {
        sh.overflow = 0;
        sh.bk = NB;  // top-k bucket (NB = no top-k)
        sh.zk = Z;
        sh.zk_bucket = 0.0;
      }
      __syncthreads();
      // union of the pair's collected lists: own entries first, then the
      // partner's (both CTAs end with the same multiset; sorting makes it canonical)
      auto merge_lists = [&]() {
        if constexpr (CL > 1) {
          const int n_own = sh.list_n;
          if (tid == 0) sh.xi[xs][1] = n_own;
          cl_sync();
          const int n_p = peer_ptr(&sh.xi[xs][0], pr)[1];
          const unsigned long long* plist = peer_ptr(sh.list, pr);
          const bool fits = n_own <= LIST && n_p <= LIST && n_own + n_p <= LIST;
          if (fits)
            for (int k = tid; k < n_p; k += NT) sh.list[n_own + k] = plist[k];
          cl_sync();  // the partner has copied our entries before either list is permuted
          if (tid == 0) sh.list_n = fits ? n_own + n_p : LIST + 1;
          xs ^= 1;
          __syncthreads();
        }
      };
      // collect the members of bucket `bkt` into sh.list and sort them
      auto collect_sort = [&](int bkt) {
        if constexpr (CL > 1) cl_sync();  // the previous union has been consumed by both CTAs
        if (tid == 0) sh.list_n = 0;
        __syncthreads();
        for (int64_t j = jlo + tid; j < jhi; j += NT) {
          const unsigned qb = qbits_of(Q(j));
          if (bucket_of(qb, top, scale) == bkt) {
            const int slot = atomicAdd(&sh.list_n, 1);
            if (slot < LIST) sh.list[slot] = sort_key(qb, int(j));
          }
        }
        __syncthreads();
        merge_lists();
        const int n = sh.list_n;
        if (n > LIST) {
          if (tid == 0) sh.overflow = 1;
          __syncthreads();
          return;
        }
        sort_list(sh, n);
      };
      unsigned k_t = 0;
      int k_cut = int(V), k_take = 0;
      if (filt_k) {
        const unsigned c = sh.hcnt[tid];
        unsigned tot;
        const unsigned ex = block_excl_scan<unsigned>(c, sh.uwarp, tot);
        if (c > 0 && ex < unsigned(prm.top_k) && unsigned(prm.top_k) <= ex + c) {
          sh.bk = tid;
          sh.c_above = ex;
        }
        double dtot;
        const double sex = block_excl_scan<double>(double(sh.hsum[tid]) * kFix, sh.dwarp, dtot);
        if (tid == sh.bk) sh.s_above = sex;
        __syncthreads();
        collect_sort(sh.bk);
        if (!sh.overflow) {
          k_take = int(unsigned(prm.top_k) - sh.c_above);
          if (tid == 0) {
            double zb = 0.0;
            for (int rr = 0; rr < k_take; ++rr) zb += double(key_q(sh.list[rr]));
            sh.zk_bucket = zb;
            sh.zk = sh.s_above + zb;
            const unsigned long long e = sh.list[k_take - 1];
            sh.t_final = ~unsigned(e >> 32);
            sh.idx_cut = int(e & 0xffffffffu);
          }
          __syncthreads();
          k_t = sh.t_final;
          k_cut = sh.idx_cut;
        }
      }
      if (!sh.overflow && filt_p) {
        const double target = prm.top_p * sh.zk;
        const int bk = sh.bk;
        // effective bucket sums: beyond the top-k bucket nothing is kept
        const double hs = tid < bk ? double(sh.hsum[tid]) * kFix : (tid == bk ? sh.zk_bucket : 0.0);
        double dtot;
        const double ex = block_excl_scan<double>(hs, sh.dwarp, dtot);
        if (tid == 0) sh.bp = -1;
        __syncthreads();
        if (hs > 0.0 && ex < target && target <= ex + hs) sh.bp = tid;
        __syncthreads();
        if (sh.bp < 0) {  // rounding: the crossing is the last kept bucket
          if (hs > 0.0) atomicMax(&sh.bp, tid);
          __syncthreads();
        }
        // the fixed-point histogram only locates the crossing approximately:
        // confirm it with exact fp64 sums (no atomics) and step to a neighbour
        // bucket if rounding put it one off; the same pass collects the
        // members of the crossing bucket
        int bp = sh.bp;
        bool listed = false;  // sh.list holds the members of bucket bp
        for (int guard = 0; guard < NB; ++guard) {
          const bool col = bp != bk;  // bp == bk reuses the top-k sorted list
          if (col) {
            if constexpr (CL > 1) cl_sync();  // the previous union has been consumed by both CTAs
            if (tid == 0) sh.list_n = 0;
            __syncthreads();
          }
          double lt = 0.0, eq = 0.0;
          auto one = [&](float q, int j) {
            const unsigned qb = qbits_of(q);
            const int bj = bucket_of(qb, top, scale);
            const bool inK = bj < bk || (bj == bk && (qb > k_t || (qb == k_t && j <= k_cut)));
            if (!inK) return;
            if (bj < bp) {
              lt += double(q);
            } else if (bj == bp) {
              eq += double(q);
              if (col) {
                const int slot = atomicAdd(&sh.list_n, 1);
                if (slot < LIST) sh.list[slot] = sort_key(qb, j);
              }
            }
          };
          if constexpr (CACHED) {
            const float4* c4 = reinterpret_cast<const float4*>(qcache);
            const int nloc = int(jhi - jlo), nv = nloc / 4;
            for (int k4 = tid; k4 < nv; k4 += NT) {
              const float4 q4 = c4[k4];
              const int j0 = int(jlo) + 4 * k4;
              one(q4.x, j0);
              one(q4.y, j0 + 1);
              one(q4.z, j0 + 2);
              one(q4.w, j0 + 3);
            }
            for (int j = nv * 4 + tid; j < nloc; j += NT) one(qcache[j], int(jlo) + j);
          } else {
            for (int64_t j = jlo + tid; j < jhi; j += NT) one(Q(j), int(j));
          }
          lt = block_sum_d(lt, sh);
          eq = block_sum_d(eq, sh);
          row_sum_d2(lt, eq);
          if (col) merge_lists();
          if (target <= lt && bp > 0) {
            --bp;
          } else if (target > lt + eq && bp < min(bk, NB - 1) && eq >= 0.0 && lt + eq < target) {
            ++bp;
          } else {
            if (tid == 0) sh.s_above = lt;
            listed = col;
            break;
          }
        }
        __syncthreads();
        stamp(4);
        if (bp != bk) {
          if (listed) {  // members already collected (and merged): sort them
            const int n = sh.list_n;
            if (n > LIST) {
              if (tid == 0) sh.overflow = 1;
              __syncthreads();
            } else {
              sort_list(sh, n);
            }
          } else {
            collect_sort(bp);
          }
        }
        stamp(5);
        if (s.dbg && b == 0 && r == 0 && threadIdx.x == 0) s.dbg[8] = sh.list_n;
        if (!sh.overflow) {
          // first sorted member r with s_above + sum_{<=r} q >= target, as a block scan
          const int limit = bp == bk ? k_take : min(sh.list_n, LIST);
          const double qv = tid < limit ? double(key_q(sh.list[tid])) : 0.0;
          double tot;
          const double ex = block_excl_scan<double>(qv, sh.dwarp, tot);
          if (tid == 0) sh.result = 0x7fffffff;
          __syncthreads();
          if (tid < limit && sh.s_above + ex + qv >= target) atomicMin(&sh.result, tid);
          __syncthreads();
          if (tid == 0) {
            const int rr = sh.result != 0x7fffffff ? sh.result : limit - 1;
            const unsigned long long e = sh.list[rr];
            sh.t_final = ~unsigned(e >> 32);
            sh.idx_cut = int(e & 0xffffffffu);
          }
        }
        __syncthreads();
        k_t = sh.t_final;
        k_cut = sh.idx_cut;
      }
      if (sh.overflow) {
        // exact but slow path (a crossing bucket with > LIST members, i.e.
        // massive ties): binary search on the threshold bits with block
        // reductions, ties resolved by index.  With a CTA pair, rank 0 runs it
        // over the whole row (the partner's part through DSMEM) and shares the
        // threshold.
        unsigned tk = botb, tp = botb;
        int cutk = int(V), cutp = int(V);
        if (r == 0) {
          if (filt_k) {
            unsigned lo = botb, hi = top;
            while (lo < hi) {
              const unsigned mid = lo + (hi - lo + 1) / 2;
              double c = 0;
              for (int64_t j = tid; j < V; j += NT) c += qbits_of(Qall(j)) >= mid;
              c = block_sum_d(c, sh);
              if (c >= double(prm.top_k)) lo = mid; else hi = mid - 1;
            }
            tk = lo;
            double above = 0;
            for (int64_t j = tid; j < V; j += NT) above += qbits_of(Qall(j)) > tk;
            above = block_sum_d(above, sh);
            const int need = int(prm.top_k - int64_t(above));
            if (tid == 0) {
              int cnt = 0;
              for (int64_t j = 0; j < V; ++j)
                if (qbits_of(Qall(j)) == tk && ++cnt == need) {
                  sh.idx_cut = int(j);
                  break;
                }
            }
            __syncthreads();
            cutk = sh.idx_cut;
          }
          auto keptk = [&](int64_t j) {
            const unsigned qb = qbits_of(Qall(j));
            return !filt_k || qb > tk || (qb == tk && j <= cutk);
          };
          double zk = 0;
          for (int64_t j = tid; j < V; j += NT)
            if (keptk(j)) zk += double(Qall(j));
          zk = block_sum_d(zk, sh);
          tp = tk;
          cutp = cutk;
          if (filt_p) {
            const double target = prm.top_p * zk;
            unsigned lo = tk, hi = top;
            while (lo < hi) {
              const unsigned mid = lo + (hi - lo + 1) / 2;
              double sacc = 0;
              for (int64_t j = tid; j < V; j += NT)
                if (keptk(j) && qbits_of(Qall(j)) >= mid) sacc += double(Qall(j));
              sacc = block_sum_d(sacc, sh);
              if (sacc >= target) lo = mid; else hi = mid - 1;
            }
            tp = lo;
            double above = 0;
            for (int64_t j = tid; j < V; j += NT)
              if (keptk(j) && qbits_of(Qall(j)) > tp) above += double(Qall(j));
            above = block_sum_d(above, sh);
            if (tid == 0) {
              double acc = above;
              int cut = -1;
              for (int64_t j = 0; j < V; ++j)
                if (keptk(j) && qbits_of(Qall(j)) == tp) {
                  acc += double(Qall(j));
                  cut = int(j);
                  if (acc >= target) break;
                }
              sh.idx_cut = cut;
            }
            __syncthreads();
            cutp = sh.idx_cut;
          }
        }
        if constexpr (CL > 1) {  // share rank 0's threshold
          if (tid == 0) {
            sh.xu[xs][0] = tp;
            sh.xi[xs][2] = cutp;
          }
          cl_sync();
          if (r == 1) {
            tp = peer_ptr(&sh.xu[xs][0], 0u)[0];
            cutp = peer_ptr(&sh.xi[xs][0], 0u)[2];
          }
          xs ^= 1;
        }
        k_t = tp;
        k_cut = cutp;
        __syncthreads();
      }
      t_final = k_t;
      idx_cut = k_cut;
    }
    stamp(6);
    // ---- inverse CDF in index order over the kept tokens: every thread owns a
    // contiguous chunk of this CTA's range (sequential fp64 sums), one block
    // scan, rank 0's total ahead of rank 1's, and the thread whose chunk
    // brackets u*Z walks it (src/model.cpp:464-473 semantics)
    auto kept = [&](int64_t j, float& q) -> bool {
      q = Q(j);
      if (!filtering) return true;
      const unsigned qb = qbits_of(q);
      return qb > t_final || (qb == t_final && j <= idx_cut);
    };
    const int64_t nloc = jhi - jlo;
    const int64_t CH = (nloc + NT - 1) / NT;
    const int64_t c0 = jlo + int64_t(tid) * CH, c1 = (jhi < c0 + CH ? jhi : c0 + CH);
    double csum = 0.0;
    int last = -1;
    for (int64_t j = c0; j < c1; ++j) {
      float q;
      if (kept(j, q)) {
        csum += double(q);
        last = int(j);
      }
    }
    double total;
    double prefix = block_excl_scan<double>(csum, sh.dwarp, total);
    int lk = last;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lk = max(lk, __shfl_xor_sync(0xffffffffu, lk, o));
    if (lane == 0) sh.lk[w] = lk;
    if (tid == 0) sh.result = 0x7fffffff;
    __syncthreads();
    int fallback = -1;
    for (int k = 0; k < NW; ++k) fallback = max(fallback, sh.lk[k]);
    if constexpr (CL > 1) {
      if (tid == 0) {
        sh.xd[xs][2] = total;
        sh.xi[xs][3] = fallback;
      }
      cl_sync();
      const double ot = peer_ptr(&sh.xd[xs][0], pr)[2];
      fallback = max(fallback, peer_ptr(&sh.xi[xs][0], pr)[3]);
      if (r == 1) prefix += ot;
      total = r == 0 ? total + ot : ot + total;
      xs ^= 1;
    }
    const double u = s.uniforms[b * s.ustride + i];
    const double target = u * total;
    if (csum > 0.0 && prefix <= target && target < prefix + csum * (1.0 + 1e-12)) {
      double acc = prefix;
      for (int64_t j = c0; j < c1; ++j) {
        float q;
        if (kept(j, q)) {
          acc += double(q);
          if (target < acc) {
            atomicMin(&sh.result, int(j));
            break;
          }
        }
      }
    }
    __syncthreads();
    int res = sh.result;
    if constexpr (CL > 1) {
      if (tid == 0) sh.xi[xs][0] = res;
      cl_sync();
      res = min(res, peer_ptr(&sh.xi[xs][0], pr)[0]);
      xs ^= 1;
    }
    chosen = res != 0x7fffffff ? res : (fallback >= 0 ? fallback : int(V - 1));
    stamp(7);
  }
  if (r == 0 && tid == 0) {
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
  if constexpr (CL > 1) cl_sync();  // the partner may still read this CTA's shared memory
}
}  // namespace

void launch_sampler(Ctx& c, const float* logits, int64_t ld, int64_t B, int64_t V, const SamplerState& s) {
  if (B <= 0) return;
  // a CTA pair per row while the pairs fit one wave (rows <= #SMs / 2); each
  // CTA caches half the row
  static const int cl_env = [] {
    const char* e = getenv("PPOEXP_SAMPLER_CL");
    return e ? atoi(e) : 2;
  }();
  int sms = 0;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const bool pair_ok = cl_env == 2 && 2 * B <= sms && V >= 64 && (ld % 4) == 0;
  const bool pair = pair_ok && (V + 7) / 8 * 4 <= kCacheMaxV;
  if (pair_ok && !pair) {
    // vocabularies too large for the per-CTA logit cache (e.g. 128k): still a
    // CTA pair per row, each streaming its half of the row from L2 every pass
    ++c.variants["sampler:pair_uncached"];
    c.launch("sampler", double(B) * V * 4, 0, [&] {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(unsigned(2 * B));
      cfg.blockDim = dim3(NT);
      cfg.dynamicSmemBytes = 0;
      cfg.stream = c.stream;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      PPOEXP_CUDA(cudaLaunchKernelEx(&cfg, sampler_kernel<false, 2>, logits, ld, V, s));
    });
  } else if (pair) {
    ++c.variants["sampler:pair_cached"];
    const int64_t half = (V + 7) / 8 * 4;
    const size_t smem = size_t(half) * sizeof(float);
    static bool attr = false;
    if (!attr) {
      PPOEXP_CUDA(cudaFuncSetAttribute(sampler_kernel<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kCacheMaxV * sizeof(float))));
      attr = true;
    }
    c.launch("sampler", double(B) * V * 4, 0, [&] {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(unsigned(2 * B));
      cfg.blockDim = dim3(NT);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = c.stream;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      PPOEXP_CUDA(cudaLaunchKernelEx(&cfg, sampler_kernel<true, 2>, logits, ld, V, s));
    });
  } else if (V <= kCacheMaxV) {
    ++c.variants["sampler:single_cached"];
    const size_t smem = size_t(V) * sizeof(float);
    static bool attr = false;
    if (!attr) {
      PPOEXP_CUDA(cudaFuncSetAttribute(sampler_kernel<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kCacheMaxV * sizeof(float))));
      attr = true;
    }
    c.launch("sampler", double(B) * V * 4, 0,
             [&] { launch_kernel(c, sampler_kernel<true, 1>, dim3(B), dim3(NT), smem, 1, logits, ld, V, s); });
  } else {
    ++c.variants["sampler:single_uncached"];
    c.launch("sampler", double(B) * V * 4, 0,
             [&] { launch_kernel(c, sampler_kernel<false, 1>, dim3(B), dim3(NT), 0, 1, logits, ld, V, s); });
  }
}

}  // namespace ppx
