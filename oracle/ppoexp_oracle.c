/*
 * ppoexp_oracle.c — CPU restatement (fp64) of the reference's PPO
 * experience-making path.  TEST INFRASTRUCTURE ONLY: this file is the
 * checker.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it.  The product path (paper_2405_01481_b200/) never links or
 * calls it.
 *
 * Parity pin: every function here is checked against the reference itself,
 * compiled from /root/reference/proj/src by oracle/Makefile into
 * oracle/_ref/libaligner_ref.so (see tests/test_oracle_vs_reference.py), and
 * against the golden fixtures under tests/golden/ generated from that build
 * (tests/golden/make_golden.py).
 *
 * Citations are relative to /root/reference/proj.
 *
 * Weight layout ("flat canonical"): the tensors of
 * ModelParams::expected_names (src/model.cpp:66-90) concatenated in that
 * order, each in the reference's row-major layout (projections are x·W with
 * W [in, out], src/model.cpp:363-374; the LM head is tied to tok_embed [V, d],
 * src/model.cpp:346-352).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t V, d, L, H, f, S;
  int32_t scalar_head;
} orc_cfg;

/* ------------------------------------------------------------------ rng */
/* std::mt19937_64 restated (include/aligner/rng.hpp:14-48 wraps it). */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_rng;

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

uint64_t orc_rng_next(orc_rng* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* Rng::uniform, include/aligner/rng.hpp:21-23 */
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

/* Rng::normal (Box-Muller), include/aligner/rng.hpp:28-33 */
double orc_rng_normal(orc_rng* r) {
  double u1 = orc_rng_uniform(r);
  while (u1 <= 0.0) u1 = orc_rng_uniform(r);
  const double u2 = orc_rng_uniform(r);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* Rng::uniform_int, include/aligner/rng.hpp:38-44 */
uint64_t orc_rng_uniform_int(orc_rng* r, uint64_t n) {
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t x = orc_rng_next(r);
  while (x >= limit) x = orc_rng_next(r);
  return x % n;
}

/* mix_seed, include/aligner/rng.hpp:51-56 */
uint64_t orc_mix_seed(uint64_t a, uint64_t b) {
  uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* Fills out[n] with the first n uniforms of Rng(seed) — the per-task sampling
 * stream of generate() (src/model.cpp:445, :464). */
void orc_uniforms(uint64_t seed, int64_t n, double* out) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = orc_rng_uniform(&r);
}

/* ------------------------------------------------------------ params */
typedef struct {
  const double *tok, *pos;
  const double *ln1_w, *ln1_b, *wq, *wk, *wv, *wo, *ln2_w, *ln2_b, *wup, *wdown;
  const double *lnf_w, *lnf_b, *head;
} orc_layer_view;

int64_t orc_param_count(const orc_cfg* c) {
  const int64_t d = c->d, per_layer = 2 * d + 4 * d * d + 2 * d + d * c->f + c->f * d;
  return c->V * d + c->S * d + c->L * per_layer + 2 * d + (c->scalar_head ? d : 0);
}

/* Offsets follow ModelParams::expected_names (src/model.cpp:66-90). */
static const double* layer_base(const orc_cfg* c, const double* w, int64_t l) {
  const int64_t d = c->d, per_layer = 2 * d + 4 * d * d + 2 * d + d * c->f + c->f * d;
  return w + c->V * d + c->S * d + l * per_layer;
}

typedef struct {
  const double *ln1_w, *ln1_b, *wq, *wk, *wv, *wo, *ln2_w, *ln2_b, *wup, *wdown;
} orc_layer;

static orc_layer get_layer(const orc_cfg* c, const double* w, int64_t l) {
  const int64_t d = c->d;
  const double* p = layer_base(c, w, l);
  orc_layer y;
  y.ln1_w = p; p += d;
  y.ln1_b = p; p += d;
  y.wq = p; p += d * d;
  y.wk = p; p += d * d;
  y.wv = p; p += d * d;
  y.wo = p; p += d * d;
  y.ln2_w = p; p += d;
  y.ln2_b = p; p += d;
  y.wup = p; p += d * c->f;
  y.wdown = p;
  return y;
}

static const double* final_norm_w(const orc_cfg* c, const double* w) { return layer_base(c, w, c->L); }
static const double* final_norm_b(const orc_cfg* c, const double* w) { return layer_base(c, w, c->L) + c->d; }
const double* orc_scalar_head(const orc_cfg* c, const double* w) {
  return c->scalar_head ? layer_base(c, w, c->L) + 2 * c->d : NULL;
}

/* init_params, src/model.cpp:156-184: one Rng(seed) walks the tensors in
 * canonical order; norm weights 1, norm biases and the scalar head 0, all
 * others N(0, 0.02). */
void orc_init_params(const orc_cfg* c, uint64_t seed, double* w) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  const int64_t d = c->d;
  double* p = w;
  for (int64_t i = 0; i < c->V * d + c->S * d; ++i) *p++ = 0.0 + 0.02 * orc_rng_normal(&r);
  for (int64_t l = 0; l < c->L; ++l) {
    for (int64_t i = 0; i < d; ++i) *p++ = 1.0;
    for (int64_t i = 0; i < d; ++i) *p++ = 0.0;
    for (int64_t i = 0; i < 4 * d * d; ++i) *p++ = 0.0 + 0.02 * orc_rng_normal(&r);
    for (int64_t i = 0; i < d; ++i) *p++ = 1.0;
    for (int64_t i = 0; i < d; ++i) *p++ = 0.0;
    for (int64_t i = 0; i < 2 * d * c->f; ++i) *p++ = 0.0 + 0.02 * orc_rng_normal(&r);
  }
  for (int64_t i = 0; i < d; ++i) *p++ = 1.0;
  for (int64_t i = 0; i < d; ++i) *p++ = 0.0;
  if (c->scalar_head)
    for (int64_t i = 0; i < d; ++i) *p++ = 0.0;
}

/* Re-draws the scalar head N(mu, sigma) from Rng(seed), as the reference's
 * PPO rig does (tests/test_ppo.cpp:40-44). */
void orc_redraw_head(const orc_cfg* c, double* w, uint64_t seed, double sigma) {
  orc_rng r;
  orc_rng_seed(&r, seed);
  double* h = (double*)orc_scalar_head(c, w);
  if (!h) return;
  for (int64_t i = 0; i < c->d; ++i) h[i] = 0.0 + sigma * orc_rng_normal(&r);
}

/* ------------------------------------------------------------ kernels */
/* KvSession::layer_norm_core, src/model.cpp:387-400 (eps 1e-5, population
 * variance, two passes). */
static void layer_norm(const double* x, const double* g, const double* b, int64_t d, double* y) {
  double mu = 0.0;
  for (int64_t j = 0; j < d; ++j) mu += x[j];
  mu /= (double)d;
  double var = 0.0;
  for (int64_t j = 0; j < d; ++j) var += (x[j] - mu) * (x[j] - mu);
  var /= (double)d;
  const double is = 1.0 / sqrt(var + 1e-5);
  for (int64_t j = 0; j < d; ++j) y[j] = g[j] * ((x[j] - mu) * is) + b[j];
}

/* KvSession::matvec, src/model.cpp:363-374: y = x·W, W [in, out]. */
static void matvec(const double* x, const double* w, int64_t in, int64_t out, double* y) {
  for (int64_t j = 0; j < out; ++j) y[j] = 0.0;
  for (int64_t i = 0; i < in; ++i) {
    const double xi = x[i];
    if (xi == 0.0) continue;
    const double* row = w + i * out;
    for (int64_t j = 0; j < out; ++j) y[j] += xi * row[j];
  }
}

/* GELU-tanh, src/model.cpp:358-361 */
static double gelu(double x) {
  const double kC = 0.7978845608028654;
  return 0.5 * x * (1.0 + tanh(kC * (x + 0.044715 * x * x * x)));
}

typedef struct {
  const orc_cfg* c;
  const double* w;
  int64_t n_fed;
  double* kc; /* [L][S][d] */
  double* vc;
  double *x, *h, *q, *k, *v, *att, *o, *up, *scores;
} kv_session;

static void kv_open(kv_session* s, const orc_cfg* c, const double* w) {
  s->c = c;
  s->w = w;
  s->n_fed = 0;
  const int64_t d = c->d;
  s->kc = (double*)malloc(sizeof(double) * c->L * c->S * d);
  s->vc = (double*)malloc(sizeof(double) * c->L * c->S * d);
  s->x = (double*)malloc(sizeof(double) * d);
  s->h = (double*)malloc(sizeof(double) * d);
  s->q = (double*)malloc(sizeof(double) * d);
  s->k = (double*)malloc(sizeof(double) * d);
  s->v = (double*)malloc(sizeof(double) * d);
  s->att = (double*)malloc(sizeof(double) * d);
  s->o = (double*)malloc(sizeof(double) * d);
  s->up = (double*)malloc(sizeof(double) * (c->f > c->d ? c->f : c->d));
  s->scores = (double*)malloc(sizeof(double) * c->S);
}

static void kv_close(kv_session* s) {
  free(s->kc); free(s->vc); free(s->x); free(s->h); free(s->q); free(s->k); free(s->v);
  free(s->att); free(s->o); free(s->up); free(s->scores);
}

/* KvSession::step, src/model.cpp:279-355.  Returns 0, or -1 when the
 * position exceeds max_seq_len (:281-284), -2 for an out-of-range token
 * (:285-288).  logits[V] receives the tied-head logits. */
static int kv_step(kv_session* s, int32_t token, double* logits) {
  const orc_cfg* c = s->c;
  const int64_t pos = s->n_fed, d = c->d, dh = c->d / c->H;
  if (pos >= c->S) return -1;
  if (token < 0 || token >= c->V) return -2;
  const double* tok = s->w;
  const double* pe = s->w + c->V * d;
  for (int64_t j = 0; j < d; ++j) s->x[j] = tok[token * d + j] + pe[pos * d + j];
  const double inv_sqrt_dh = 1.0 / sqrt((double)dh);
  for (int64_t l = 0; l < c->L; ++l) {
    orc_layer ly = get_layer(c, s->w, l);
    layer_norm(s->x, ly.ln1_w, ly.ln1_b, d, s->h);
    matvec(s->h, ly.wq, d, d, s->q);
    matvec(s->h, ly.wk, d, d, s->k);
    matvec(s->h, ly.wv, d, d, s->v);
    double* kc = s->kc + l * c->S * d;
    double* vc = s->vc + l * c->S * d;
    memcpy(kc + pos * d, s->k, sizeof(double) * d);
    memcpy(vc + pos * d, s->v, sizeof(double) * d);
    const int64_t t_len = pos + 1;
    for (int64_t j = 0; j < d; ++j) s->att[j] = 0.0;
    for (int64_t hd = 0; hd < c->H; ++hd) {
      const int64_t off = hd * dh;
      double mx = -1e300;
      for (int64_t t = 0; t < t_len; ++t) {
        double acc = 0.0;
        const double* krow = kc + t * d + off;
        for (int64_t j = 0; j < dh; ++j) acc += s->q[off + j] * krow[j];
        s->scores[t] = acc * inv_sqrt_dh;
        if (s->scores[t] > mx) mx = s->scores[t];
      }
      double se = 0.0;
      for (int64_t t = 0; t < t_len; ++t) {
        s->scores[t] = exp(s->scores[t] - mx);
        se += s->scores[t];
      }
      for (int64_t t = 0; t < t_len; ++t) {
        const double wgt = s->scores[t] / se;
        const double* vrow = vc + t * d + off;
        for (int64_t j = 0; j < dh; ++j) s->att[off + j] += wgt * vrow[j];
      }
    }
    matvec(s->att, ly.wo, d, d, s->o);
    for (int64_t j = 0; j < d; ++j) s->x[j] += s->o[j];
    layer_norm(s->x, ly.ln2_w, ly.ln2_b, d, s->h);
    matvec(s->h, ly.wup, d, c->f, s->up);
    for (int64_t j = 0; j < c->f; ++j) s->up[j] = gelu(s->up[j]);
    matvec(s->up, ly.wdown, c->f, d, s->o);
    for (int64_t j = 0; j < d; ++j) s->x[j] += s->o[j];
  }
  layer_norm(s->x, final_norm_w(c, s->w), final_norm_b(c, s->w), d, s->h);
  for (int64_t vv = 0; vv < c->V; ++vv) {
    const double* row = tok + vv * d;
    double acc = 0.0;
    for (int64_t j = 0; j < d; ++j) acc += s->h[j] * row[j];
    logits[vv] = acc;
  }
  ++s->n_fed;
  return 0;
}

/* log_softmax_vec, src/model.cpp:417-426: returns lse. */
static double log_sum_exp(const double* l, int64_t n) {
  double mx = l[0];
  for (int64_t i = 0; i < n; ++i) mx = l[i] > mx ? l[i] : mx;
  double se = 0.0;
  for (int64_t i = 0; i < n; ++i) se += exp(l[i] - mx);
  return mx + log(se);
}

/* argmax_index, src/model.cpp:428-434: first strictly-greater wins. */
static int64_t argmax_first(const double* l, int64_t n) {
  int64_t best = 0;
  for (int64_t i = 1; i < n; ++i)
    if (l[i] > l[best]) best = i;
  return best;
}

/* ---------------------------------------------------------- top-k/top-p */
/* NOT IN THE REFERENCE (north-star extension).  The
 * convention, fixed here and mirrored by the CUDA sampler:
 *   q_j = exp((l_j - max)/tau)  (the reference's tempered weights,
 *                                src/model.cpp:456-463)
 *   top-k (k > 0 and k < V): keep the k largest q_j, ties to the lower index;
 *   top-p (p < 1): of the survivors, keep tokens with q_j > t plus, among the
 *   tokens with q_j == t, the lowest indices, where t is chosen so the kept
 *   set is the shortest prefix of the survivors sorted by (q desc, index asc)
 *   whose sum reaches p * (sum of survivors' q);
 *   then the reference's inverse CDF (src/model.cpp:464-473) runs in index
 *   order over the kept tokens only; fallback = last kept index.
 * With k = 0 and p >= 1 this is exactly the reference sampler. */
typedef struct {
  double q;
  int64_t i;
} qi_pair;

static int cmp_qi(const void* a, const void* b) {
  const qi_pair* x = (const qi_pair*)a;
  const qi_pair* y = (const qi_pair*)b;
  if (x->q > y->q) return -1;
  if (x->q < y->q) return 1;
  return x->i < y->i ? -1 : (x->i > y->i ? 1 : 0);
}

/* keep[V] <- 1 for kept tokens; q[V] holds the tempered weights. */
void orc_filter_topk_topp(const double* q, int64_t V, int64_t top_k, double top_p, unsigned char* keep) {
  const int filt_k = top_k > 0 && top_k < V;
  const int filt_p = top_p < 1.0;
  if (!filt_k && !filt_p) {
    for (int64_t j = 0; j < V; ++j) keep[j] = 1;
    return;
  }
  qi_pair* s = (qi_pair*)malloc(sizeof(qi_pair) * V);
  for (int64_t j = 0; j < V; ++j) { s[j].q = q[j]; s[j].i = j; }
  qsort(s, (size_t)V, sizeof(qi_pair), cmp_qi);
  int64_t n = filt_k ? top_k : V;
  if (filt_p) {
    double tot = 0.0;
    for (int64_t r = 0; r < n; ++r) tot += s[r].q;
    const double target = top_p * tot;
    double acc = 0.0;
    int64_t r = 0;
    for (; r < n; ++r) {
      acc += s[r].q;
      if (acc >= target) break;
    }
    n = r < n ? r + 1 : n;
  }
  for (int64_t j = 0; j < V; ++j) keep[j] = 0;
  for (int64_t r = 0; r < n; ++r) keep[s[r].i] = 1;
  free(s);
}

/* One sampling decision over logits[V] given the uniform u; returns the
 * chosen index (src/model.cpp:452-474 plus the filter above). */
int64_t orc_sample(const double* logits, int64_t V, int greedy, double temperature, int64_t top_k,
                   double top_p, double u) {
  if (greedy) return argmax_first(logits, V);
  const double tau = temperature > 1e-12 ? temperature : 1e-12;
  double mx = logits[0];
  for (int64_t j = 0; j < V; ++j) mx = logits[j] > mx ? logits[j] : mx;
  double* probs = (double*)malloc(sizeof(double) * V);
  unsigned char* keep = (unsigned char*)malloc((size_t)V);
  for (int64_t j = 0; j < V; ++j) probs[j] = exp((logits[j] - mx) / tau);
  orc_filter_topk_topp(probs, V, top_k, top_p, keep);
  double se = 0.0;
  int64_t last = V - 1;
  for (int64_t j = 0; j < V; ++j)
    if (keep[j]) { se += probs[j]; last = j; }
  const double target = u * se;
  double acc = 0.0;
  int64_t chosen = last;
  for (int64_t j = 0; j < V; ++j) {
    if (!keep[j]) continue;
    acc += probs[j];
    if (target < acc) { chosen = j; break; }
  }
  free(probs);
  free(keep);
  return chosen;
}

/* ------------------------------------------------------------ generate */
/* generate(), src/model.cpp:438-482.  uniforms: per sampled token, in order
 * (the Rng(seed) stream; see orc_uniforms); ignored when greedy.
 * Returns the number of tokens written (<= budget), or a negative error. */
int64_t orc_generate(const orc_cfg* c, const double* w, const int32_t* prompt, int64_t P,
                     int64_t max_new, int greedy, double temperature, int64_t top_k, double top_p,
                     const double* uniforms, int32_t* out_tokens, double* out_lps) {
  if (P <= 0) return -3;
  kv_session s;
  kv_open(&s, c, w);
  double* logits = (double*)malloc(sizeof(double) * c->V);
  int rc = 0;
  for (int64_t i = 0; i < P && rc == 0; ++i) rc = kv_step(&s, prompt[i], logits);
  int64_t n = 0;
  if (rc == 0) {
    const int64_t pc = P < c->S ? P : c->S;
    const int64_t budget = max_new < c->S - pc ? max_new : c->S - pc;
    for (int64_t i = 0; i < budget; ++i) {
      const double lse = log_sum_exp(logits, c->V);
      const int64_t chosen =
          orc_sample(logits, c->V, greedy, temperature, top_k, top_p, greedy ? 0.0 : uniforms[i]);
      out_tokens[n] = (int32_t)chosen;
      out_lps[n] = logits[chosen] - lse;
      ++n;
      if (chosen == 257) break; /* kEotToken, include/aligner/model.hpp:18 */
      if (i + 1 < budget) {
        rc = kv_step(&s, (int32_t)chosen, logits);
        if (rc) break;
      }
    }
  }
  free(logits);
  kv_close(&s);
  return rc ? rc : n;
}

/* sequence_logprobs, src/model.cpp:484-495: out[0] = 0, out[t] = log p(t_t | t_<t). */
int orc_sequence_logprobs(const orc_cfg* c, const double* w, const int32_t* tokens, int64_t T,
                          double* out) {
  if (T == 0) return 0;
  kv_session s;
  kv_open(&s, c, w);
  double* logits = (double*)malloc(sizeof(double) * c->V);
  int rc = kv_step(&s, tokens[0], logits);
  out[0] = 0.0;
  for (int64_t t = 1; t < T && rc == 0; ++t) {
    const double lse = log_sum_exp(logits, c->V);
    out[t] = logits[tokens[t]] - lse;
    rc = kv_step(&s, tokens[t], logits);
  }
  free(logits);
  kv_close(&s);
  return rc;
}

/* transformer_hidden (full-sequence causal forward), src/model.cpp:205-245.
 * hidden[T, d] = final-LN output.  The tape path's mask adds -1e30 above the
 * diagonal (src/model.cpp:198-203); exp underflows those to exactly 0, so the
 * causal softmax below is the same arithmetic. */
int orc_forward_hidden(const orc_cfg* c, const double* w, const int32_t* tokens, int64_t T,
                       double* hidden) {
  if (T == 0) return -3;
  if (T > c->S) return -1;
  const int64_t d = c->d, dh = c->d / c->H, f = c->f;
  for (int64_t t = 0; t < T; ++t)
    if (tokens[t] < 0 || tokens[t] >= c->V) return -2;
  double* x = (double*)malloc(sizeof(double) * T * d);
  double* h = (double*)malloc(sizeof(double) * T * d);
  double* q = (double*)malloc(sizeof(double) * T * d);
  double* k = (double*)malloc(sizeof(double) * T * d);
  double* v = (double*)malloc(sizeof(double) * T * d);
  double* a = (double*)malloc(sizeof(double) * T * d);
  double* o = (double*)malloc(sizeof(double) * T * d);
  double* up = (double*)malloc(sizeof(double) * T * f);
  double* sc = (double*)malloc(sizeof(double) * T);
  const double* tok = w;
  const double* pe = w + c->V * d;
  for (int64_t t = 0; t < T; ++t)
    for (int64_t j = 0; j < d; ++j) x[t * d + j] = tok[tokens[t] * d + j] + pe[t * d + j];
  const double inv_sqrt_dh = 1.0 / sqrt((double)dh);
  for (int64_t l = 0; l < c->L; ++l) {
    orc_layer ly = get_layer(c, w, l);
    for (int64_t t = 0; t < T; ++t) {
      layer_norm(x + t * d, ly.ln1_w, ly.ln1_b, d, h + t * d);
      matvec(h + t * d, ly.wq, d, d, q + t * d);
      matvec(h + t * d, ly.wk, d, d, k + t * d);
      matvec(h + t * d, ly.wv, d, d, v + t * d);
    }
    for (int64_t i = 0; i < T * d; ++i) a[i] = 0.0;
    for (int64_t hd = 0; hd < c->H; ++hd) {
      const int64_t off = hd * dh;
      for (int64_t i = 0; i < T; ++i) {
        double mx = -1e300;
        for (int64_t t = 0; t <= i; ++t) {
          double acc = 0.0;
          for (int64_t j = 0; j < dh; ++j) acc += q[i * d + off + j] * k[t * d + off + j];
          sc[t] = acc * inv_sqrt_dh;
          if (sc[t] > mx) mx = sc[t];
        }
        double se = 0.0;
        for (int64_t t = 0; t <= i; ++t) {
          sc[t] = exp(sc[t] - mx);
          se += sc[t];
        }
        for (int64_t t = 0; t <= i; ++t) {
          const double wgt = sc[t] / se;
          for (int64_t j = 0; j < dh; ++j) a[i * d + off + j] += wgt * v[t * d + off + j];
        }
      }
    }
    for (int64_t t = 0; t < T; ++t) {
      matvec(a + t * d, ly.wo, d, d, o + t * d);
      for (int64_t j = 0; j < d; ++j) x[t * d + j] += o[t * d + j];
      layer_norm(x + t * d, ly.ln2_w, ly.ln2_b, d, h + t * d);
      matvec(h + t * d, ly.wup, d, f, up + t * f);
      for (int64_t j = 0; j < f; ++j) up[t * f + j] = gelu(up[t * f + j]);
      matvec(up + t * f, ly.wdown, f, d, o + t * d);
      for (int64_t j = 0; j < d; ++j) x[t * d + j] += o[t * d + j];
    }
  }
  for (int64_t t = 0; t < T; ++t)
    layer_norm(x + t * d, final_norm_w(c, w), final_norm_b(c, w), d, hidden + t * d);
  free(x); free(h); free(q); free(k); free(v); free(a); free(o); free(up); free(sc);
  return 0;
}

/* forward_one logits (tied head), src/model.cpp:253-256: logits[T, V]. */
int orc_forward_logits(const orc_cfg* c, const double* w, const int32_t* tokens, int64_t T,
                       double* logits) {
  double* hid = (double*)malloc(sizeof(double) * T * c->d);
  int rc = orc_forward_hidden(c, w, tokens, T, hid);
  if (rc == 0) {
    for (int64_t t = 0; t < T; ++t)
      for (int64_t vv = 0; vv < c->V; ++vv) {
        double acc = 0.0;
        for (int64_t j = 0; j < c->d; ++j) acc += hid[t * c->d + j] * w[vv * c->d + j];
        logits[t * c->V + vv] = acc;
      }
  }
  free(hid);
  return rc;
}

/* value_estimates, src/losses.cpp:117-127: V_t = h[rs-1+t] · head, t < T-rs. */
int orc_value_estimates(const orc_cfg* c, const double* w, const double* head, const int32_t* tokens,
                        int64_t T, int64_t rs, double* out) {
  if (rs == 0 || rs >= T) return -3;
  double* hid = (double*)malloc(sizeof(double) * T * c->d);
  int rc = orc_forward_hidden(c, w, tokens, T, hid);
  if (rc == 0) {
    for (int64_t t = 0; t < T - rs; ++t) {
      const double* row = hid + (rs - 1 + t) * c->d;
      double acc = 0.0;
      for (int64_t j = 0; j < c->d; ++j) acc += row[j] * head[j];
      out[t] = acc;
    }
  }
  free(hid);
  return rc;
}

/* last_content_index, src/losses.cpp:97-103 (PAD = 256). */
int64_t orc_last_content_index(const int32_t* tokens, int64_t T) {
  for (int64_t i = T; i-- > 0;)
    if (tokens[i] != 256) return i;
  return -1;
}

/* reward_head, src/losses.cpp:105-115. */
int orc_reward_head(const orc_cfg* c, const double* w, const double* head, const int32_t* tokens,
                    int64_t T, double* out) {
  const int64_t last = orc_last_content_index(tokens, T);
  if (last < 0) return -3;
  double* hid = (double*)malloc(sizeof(double) * T * c->d);
  int rc = orc_forward_hidden(c, w, tokens, T, hid);
  if (rc == 0) {
    double acc = 0.0;
    for (int64_t j = 0; j < c->d; ++j) acc += hid[last * c->d + j] * head[j];
    *out = acc;
  }
  free(hid);
  return rc;
}

/* CriticJob::scripted_reward_for, src/ppo.cpp:109-115. */
double orc_scripted_reward(const int32_t* tokens, int64_t T, int64_t rs, int32_t target) {
  double n = 0.0;
  for (int64_t t = rs; t < T; ++t)
    if (tokens[t] == target) n += 1.0;
  return n;
}

/* kl_penalized_rewards, src/losses.cpp:188-199. */
int orc_kl_penalized_rewards(double rm, const double* a, const double* r, int64_t n, double kl_coef,
                             double* out) {
  if (n == 0) return -3;
  for (int64_t t = 0; t < n; ++t) out[t] = -kl_coef * (a[t] - r[t]);
  out[n - 1] += rm;
  return 0;
}

/* gae, src/losses.cpp:168-186 (V beyond the last token = 0). */
void orc_gae(const double* rw, const double* v, int64_t n, double gamma, double lam, double* adv,
             double* ret) {
  double running = 0.0;
  for (int64_t t = n; t-- > 0;) {
    const double next = (t + 1 < n) ? v[t + 1] : 0.0;
    const double delta = rw[t] + gamma * next - v[t];
    running = delta + gamma * lam * running;
    adv[t] = running;
    ret[t] = running + v[t];
  }
}

/* Advantage whitening — NOT IN THE REFERENCE (advantages go
 * straight from gae into the loss, src/ppo.cpp:382-393).  Convention (the
 * survey's recommendation, §8 a18): statistics over every valid response
 * token of every rank, population variance, eps = 1e-8, mean shifted:
 *   w = (a - mean) / sqrt(var + 1e-8).
 * Partials are (n, sum a, sum a^2); var = E[a^2] - mean^2 computed in fp64. */
void orc_whiten_partials(const double* adv, int64_t n, double* part3) {
  double s = 0.0, s2 = 0.0;
  for (int64_t i = 0; i < n; ++i) { s += adv[i]; s2 += adv[i] * adv[i]; }
  part3[0] = (double)n;
  part3[1] = s;
  part3[2] = s2;
}

void orc_whiten_apply(const double* adv, int64_t n, const double* part3, double* out) {
  const double cnt = part3[0] > 0 ? part3[0] : 1.0;
  const double mean = part3[1] / cnt;
  double var = part3[2] / cnt - mean * mean;
  if (var < 0) var = 0;
  const double inv = 1.0 / sqrt(var + 1e-8);
  for (int64_t i = 0; i < n; ++i) out[i] = (adv[i] - mean) * inv;
}

/* ------------------------------------------------------ batched helpers */
/* Ragged batch versions (offsets[B+1]) for the Python test harness; the
 * per-sequence work is independent, so a small pthread pool spreads it over
 * cores (orc_set_threads; default 1). */
#include <pthread.h>

static int g_threads = 1;
void orc_set_threads(int n) { g_threads = n > 0 ? n : 1; }

typedef struct {
  void (*fn)(void*, int64_t);
  void* ctx;
  int64_t n;
  int64_t next;
  pthread_mutex_t mu;
} par_job;

static void* par_worker(void* arg) {
  par_job* j = (par_job*)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    const int64_t i = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (i >= j->n) break;
    j->fn(j->ctx, i);
  }
  return NULL;
}

static void par_for(int64_t n, void (*fn)(void*, int64_t), void* ctx) {
  par_job j;
  j.fn = fn; j.ctx = ctx; j.n = n; j.next = 0;
  pthread_mutex_init(&j.mu, NULL);
  int nt = g_threads < n ? g_threads : (int)n;
  if (nt <= 1) {
    par_worker(&j);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nt);
    for (int t = 0; t < nt; ++t) pthread_create(&th[t], NULL, par_worker, &j);
    for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    free(th);
  }
  pthread_mutex_destroy(&j.mu);
}

typedef struct {
  const orc_cfg* c;
  const double* w;
  const double* head;
  const int32_t* tokens;
  const int64_t* offsets;
  const int64_t* rs;
  const int64_t* out_offsets;
  double* out;
  int64_t max_new;
  int greedy;
  double temperature;
  int64_t top_k;
  double top_p;
  const double* uniforms;
  int32_t* out_tokens;
  int64_t* out_n;
  volatile int rc;
} batch_ctx;

static void do_lp(void* p, int64_t b) {
  batch_ctx* x = (batch_ctx*)p;
  if (orc_sequence_logprobs(x->c, x->w, x->tokens + x->offsets[b], x->offsets[b + 1] - x->offsets[b],
                            x->out + x->offsets[b]))
    x->rc = 1;
}

int orc_batch_sequence_logprobs(const orc_cfg* c, const double* w, const int32_t* tokens,
                                const int64_t* offsets, int64_t B, double* out) {
  batch_ctx x;
  memset(&x, 0, sizeof x);
  x.c = c; x.w = w; x.tokens = tokens; x.offsets = offsets; x.out = out;
  par_for(B, do_lp, &x);
  return x.rc;
}

static void do_val(void* p, int64_t b) {
  batch_ctx* x = (batch_ctx*)p;
  if (orc_value_estimates(x->c, x->w, x->head, x->tokens + x->offsets[b], x->offsets[b + 1] - x->offsets[b],
                          x->rs[b], x->out + x->out_offsets[b]))
    x->rc = 1;
}

int orc_batch_value_estimates(const orc_cfg* c, const double* w, const double* head,
                              const int32_t* tokens, const int64_t* offsets, const int64_t* rs,
                              int64_t B, const int64_t* out_offsets, double* out) {
  batch_ctx x;
  memset(&x, 0, sizeof x);
  x.c = c; x.w = w; x.head = head; x.tokens = tokens; x.offsets = offsets; x.rs = rs;
  x.out_offsets = out_offsets; x.out = out;
  par_for(B, do_val, &x);
  return x.rc;
}

static void do_rw(void* p, int64_t b) {
  batch_ctx* x = (batch_ctx*)p;
  if (orc_reward_head(x->c, x->w, x->head, x->tokens + x->offsets[b], x->offsets[b + 1] - x->offsets[b],
                      x->out + b))
    x->rc = 1;
}

int orc_batch_reward_head(const orc_cfg* c, const double* w, const double* head, const int32_t* tokens,
                          const int64_t* offsets, int64_t B, double* out) {
  batch_ctx x;
  memset(&x, 0, sizeof x);
  x.c = c; x.w = w; x.head = head; x.tokens = tokens; x.offsets = offsets; x.out = out;
  par_for(B, do_rw, &x);
  return x.rc;
}

static void do_gen(void* p, int64_t b) {
  batch_ctx* x = (batch_ctx*)p;
  const int64_t n = orc_generate(x->c, x->w, x->tokens + x->offsets[b], x->offsets[b + 1] - x->offsets[b],
                                 x->max_new, x->greedy, x->temperature, x->top_k, x->top_p,
                                 x->uniforms ? x->uniforms + b * x->max_new : NULL,
                                 x->out_tokens + b * x->max_new, x->out + b * x->max_new);
  x->out_n[b] = n;
  if (n < 0) x->rc = 1;
}

/* uniforms: [B, max_new] row-major; out_tokens/out_lps: [B, max_new];
 * out_n[B] the per-sequence lengths. */
int orc_batch_generate(const orc_cfg* c, const double* w, const int32_t* prompts, const int64_t* offsets,
                       int64_t B, int64_t max_new, int greedy, double temperature, int64_t top_k,
                       double top_p, const double* uniforms, int32_t* out_tokens, double* out_lps,
                       int64_t* out_n) {
  batch_ctx x;
  memset(&x, 0, sizeof x);
  x.c = c; x.w = w; x.tokens = prompts; x.offsets = offsets; x.max_new = max_new; x.greedy = greedy;
  x.temperature = temperature; x.top_k = top_k; x.top_p = top_p; x.uniforms = uniforms;
  x.out_tokens = out_tokens; x.out = out_lps; x.out_n = out_n;
  par_for(B, do_gen, &x);
  return x.rc;
}
