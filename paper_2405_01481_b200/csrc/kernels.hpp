// kernels.hpp — host launchers for the sm_100a kernels of the experience path.
// T is the compute/storage type of weights and GEMM operands: float (parity
// mode) or bf16 (perf mode).  The residual stream is always fp32.
#pragma once

#include <cuda.h>

#include <cstdint>

#include "runtime.hpp"

namespace ppx {

// Paged KV cache geometry.  Pool layout (elements of T):
//   kv[(((layer * n_pages + page) * 2 + kv) * H + h) * page_size * DH + slot * DH + i]
struct KvGeom {
  int64_t n_layers, n_pages, page_size, H, DH, max_pages_per_seq;
};

// K1: x[r] = tok[tokens[r]] + pos[positions[r]] (src/model.cpp:290-295).
template <class T>
void launch_embed(Ctx& c, const int32_t* tokens, const int32_t* positions, int64_t rows, int64_t d,
                  const T* tok, const T* pos, float* x);

// K1 + K2 for the decode step: embedding and the first LayerNorm in one pass
// (false when d % 4 != 0 or d > 4096: use launch_embed + launch_layernorm).
template <class T>
bool launch_embed_layernorm(Ctx& c, const int32_t* tokens, const int32_t* positions, int64_t rows, int64_t d,
                            const T* tok, const T* pos, float* x, const float* g, const float* b, T* y);

// K2: LayerNorm (src/model.cpp:387-400), fp32 in, T out.  gather (nullable)
// selects input rows; head (nullable) additionally writes head_out[r] =
// dot(LN(x_row), head) in fp32 (K10: value / reward head) and, when y is
// null, skips the T output.
template <class T>
void launch_layernorm(Ctx& c, const float* x, int64_t rows, int64_t d, const float* g, const float* b, T* y,
                      const int32_t* gather, const float* head, float* head_out);

// K3: C[M,N] = A[M,K] · B[N,K]^T with epilogue.
// kGeluSplit: GELU output written as two bf16 planes (hi at [row, col], lo at [row, N + col]; ldc >= 2N)
enum class Epi : int { kStore = 0, kGelu = 1, kAddResidual = 2, kStoreF32 = 3, kLse = 4, kGeluF32 = 5, kGeluSplit = 6, kStoreSplit = 7 };
// Epilogue outputs of the fused LM-head + log-sum-exp + gather GEMM (Epi::kLse).
struct LseEpi {
  const int32_t* target = nullptr;  // [M] target column per row (< 0: none)
  float* tgt_logit = nullptr;       // [M] fp32 logit of the target
  float2* part = nullptr;           // [M, ldp] (max, sum exp(l - max)) per 256-column tile
  int ldp = 0;
};
int lse_tiles(int64_t N);
bool gemm_tc_lse(Ctx& c, const bf16* A, int64_t lda, const bf16* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                 const LseEpi& e);
// lp[r] = tgt_logit[r] - LSE(part[r, :ntiles]) → out[out_index[r]] (fp64 combine).
void launch_lse_combine(Ctx& c, const float2* part, int ldp, int ntiles, const float* tgt_logit,
                        const int32_t* target, int64_t rows, const int64_t* out_index, double* out);
template <class T>
void launch_gemm(Ctx& c, const T* A, int64_t lda, const T* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                 Epi epi, void* C, int64_t ldc);

// ---- decode-path LayerNorm fusion (bf16 engine) ----
// Row statistics of the fp32 residual x travel as one pair of fixed-point
// accumulators per row: acc[row * kStatStride + {0, 1}] = {sum x, sum x^2} in units of
// 2^-kStatShift (two's complement in u64).  Residual-producing decode GEMMs add
// their per-CTA partials with integer atomics (order-independent, so the
// statistics are bit-reproducible); consumer GEMMs normalise their activation
// K-slice on the fly (LN = src/model.cpp:387-400, one-pass mean / variance).
// Range: every producer adds one partial per row (a 128-feature slice of x, or
// the whole row at the embedding); a partial must stay below kStatMax so that up
// to 64 of them cannot overflow 2^63 (|x| rms up to ~2.3e4 per element).  A
// partial beyond that sets *ovf and the engine fails loudly (no silent clamp).
constexpr int kStatShift = 20;
constexpr int kStatStride = 16;  // u64 per row: one 128-byte line each, so the producers' atomics spread over L2 slices
constexpr double kStatMax = 9.2233720368547758e18 / 64.0 / double(1ll << kStatShift);
__device__ __forceinline__ unsigned long long stat_fix(double v, unsigned* ovf) {
  if (!(fabs(v) < kStatMax)) {
    if (ovf) atomicOr(ovf, 1u);
    v = 0.0;
  }
  return static_cast<unsigned long long>(__double2ll_rn(v * double(1ll << kStatShift)));
}
__device__ __forceinline__ double stat_of(unsigned long long a) {
  return double(static_cast<long long>(a)) * (1.0 / double(1ll << kStatShift));
}
struct RowStats {
  unsigned long long* acc;            // [rows][kStatStride] (first two used), zero before the first add
  unsigned* ovf = nullptr;            // set to 1 when a partial is outside the fixed-point range
  unsigned long long* zero = nullptr;  // (embedding only) accumulator rows to clear for this step
  int64_t zero_n = 0;                  // ... their number
};
struct LnIn {
  const float* x;                  // fp32 residual stream [rows, d]
  int64_t ldx;
  const unsigned long long* acc;   // RowStats of x
  const float* g;
  const float* b;
  int d;
};
// Decode GEMM with optional fused LN on the activation operand (ln != null:
// X is ignored) and optional row statistics of the updated residual (so != null,
// Epi::kAddResidual only).
void gemm_decode_fused(Ctx& c, const bf16* X, int64_t ldx, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
                      Epi epi, void* C, int64_t ldc, const LnIn* ln, const RowStats* so);
// Mixed mode (bf16 weights, fp32 activations): X fp32 (or LN(x) when ln != null)
// split into hi + lo bf16 terms in-kernel, two MMAs per k-step; fp32 epilogues.
void gemm_decode_mixed(Ctx& c, const float* X, int64_t ldx, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
                       Epi epi, void* C, int64_t ldc, const LnIn* ln, const RowStats* so);
void gemm_decode_planes(Ctx& c, const bf16* X, int64_t ldx, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
                        Epi epi, void* C, int64_t ldc, const RowStats* so);
// LayerNorm written as two bf16 planes y[r, 0:d) = hi, y[r, d:2d) = lo (mixed decode).
void launch_embed_layernorm_split(Ctx& c, const int32_t* tokens, const int32_t* positions, int64_t rows, int64_t d,
                                  const bf16* tok, const bf16* pos, float* x, const float* g, const float* b, bf16* y);
void launch_layernorm_split(Ctx& c, const float* x, int64_t rows, int64_t d, const float* g, const float* b, bf16* y,
                            const int32_t* gather = nullptr);
// Mixed-mode GEMM over a [M, 2K] hi|lo bf16 plane activation (tcgen05, both planes TMA'd).
// Persistent tcgen05 GEMM (gemm_persist.cu): one CTA per SM over 128 x 256
// tiles, double-buffered TMEM accumulators, TMA-store epilogues; A bf16
// [M, K] or hi | lo planes [M, 2K] (split).  PPOEXP_GEMM_PERSIST=0 disables.
bool gemm_pp_enabled();
void gemm_persist(Ctx& c, const bf16* A, int64_t lda, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
                  Epi epi, void* C, int64_t ldc, bool split, const LseEpi* lse);
void gemm_tc_planes(Ctx& c, const bf16* A, int64_t lda, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
                    Epi epi, void* C, int64_t ldc, const LseEpi* lse = nullptr);
// Mixed-mode GEMM for any M (decode-sized M goes to gemm_decode_mixed).
void gemm_mixed(Ctx& c, const float* A, int64_t lda, const bf16* W, int64_t ldw, int64_t M, int64_t N, int64_t K,
                Epi epi, void* C, int64_t ldc, const LseEpi* lse = nullptr);
// Embedding that also writes the row statistics of x and clears so.zero's first zero_n rows.
template <class T>
void launch_embed_stats(Ctx& c, const int32_t* tokens, const int32_t* positions, int64_t rows, int64_t d,
                        const T* tok, const T* pos, float* x, RowStats so);

// K4: scatter the K/V columns of packed qkv rows into the paged pool
// (prefill).  seq_of_row / pos_of_row per packed row; block_table [B, max_pages].
template <class T>
void launch_kv_scatter(Ctx& c, const T* qkv, int64_t rows, int64_t d, const int32_t* seq_of_row,
                       const int32_t* pos_of_row, const int32_t* block_table, int layer, const KvGeom& g, T* kv);

// K5a: causal self-attention over packed ragged sequences (prefill/scoring),
// src/model.cpp:205-245 (tape path) == :313-333 (KvSession).
template <class T>
void launch_attention_prefill(Ctx& c, const T* qkv, const int64_t* seq_offsets, int64_t B, int64_t max_len,
                              int64_t H, int64_t DH, T* out);

// K5a on tcgen05 (bf16, head_dim 64 / 128): false when not eligible.
bool attention_prefill_tc_split(Ctx& c, const bf16* qkv_planes, const int64_t* seq_offsets, int64_t B,
                                int64_t max_len, int64_t H, int64_t DH, int64_t M_total, bf16* out_planes);
bool attention_prefill_tc(Ctx& c, const bf16* qkv, const int64_t* seq_offsets, int64_t B, int64_t max_len, int64_t H,
                          int64_t DH, int64_t M_total, bf16* out, bool force = false);
// K5a in mixed mode: fp32 q/k/v in, fp32 out, tensor-core products on the
// two-term bf16 split (three MMAs per product).
// planes (nullable): write the output as hi | lo bf16 planes [M, 2d] instead of `out`.
void attention_prefill_split(Ctx& c, const float* qkv, const int64_t* seq_offsets, int64_t B, int64_t max_len,
                             int64_t H, int64_t DH, float* out, bf16* planes = nullptr);

// K5b: one decode step: append this step's K/V (row b of qkv at position
// pos[b]) to the paged pool, then attend over positions 0..pos[b].
// Sequences with done[b] != 0 are skipped.
// split_out (fp32 KV only, nullable): the output as two bf16 planes [B, 2d] instead of `out`.
template <class T>
void launch_attention_decode(Ctx& c, const T* qkv, int64_t B, const int32_t* pos, const int32_t* done,
                             const int32_t* block_table, int layer, const KvGeom& g, T* kv, T* out,
                             double algorithmic_bytes, bf16* split_out = nullptr);

// K8: fused sampler over logits [B, ld] fp32 (src/model.cpp:450-477 + top-k/p).
struct SampleParams {
  int32_t greedy;
  float temperature;
  int64_t top_k;
  double top_p;
};
struct SamplerState {
  const SampleParams* params;  // device, [B] (one spec per task)
  int32_t* next_tok;    // [B] token fed at the next decode step
  int32_t* pos;         // [B] position the next fed token occupies
  int32_t* n_gen;       // [B]
  int32_t* done;        // [B]
  const int32_t* budget;  // [B]
  const double* uniforms;  // [B, ustride]
  int64_t ustride;
  int32_t* out_tokens;  // [B, ostride]
  float* out_lps;       // [B, ostride]
  int64_t ostride;
  int32_t* n_active;    // [1] sequences still running after this step
  unsigned long long* dbg = nullptr;  // debug (PPOEXP_SAMPLER_TRACE): row-0 stage clocks
};
void launch_sampler(Ctx& c, const float* logits, int64_t ld, int64_t B, int64_t V, const SamplerState& s);

// K9: fused log-softmax + gather: lp[r] = logits[r, target[r]] - LSE(row r),
// written to out[out_index[r]] (double).  Rows with target < 0 are skipped.
template <class T>
void launch_logprob_gather(Ctx& c, const T* logits, int64_t ld, int64_t rows, int64_t V, const int32_t* target,
                           const int64_t* out_index, double* out);

// K11: KL-shaped rewards + reverse GAE scan per sequence, plus per-sequence
// partial sums {kl_sum, n, reward, adv_sum, adv_sq_sum} into part[B][5].
void launch_shape_gae(Ctx& c, int64_t B, int64_t stride, const int64_t* lengths, const double* rm_reward,
                      const double* actor_lp, const double* ref_lp, const double* values, double kl_coef,
                      double gamma, double lam, double* shaped, double* adv, double* ret, double* part);
// K12: fixed-order reduction of part[B][5] → out[5] (deterministic).
void launch_reduce_partials(Ctx& c, int64_t B, const double* part, double* out5);
void launch_whiten_apply(Ctx& c, int64_t B, int64_t stride, const int64_t* lengths, const double* adv,
                         const double* stats3, double* out);


// misc
// IndexError (the reference's wording, src/model.cpp:284-287) for any id outside
// [0, V): a host scan (where = 0) or a device validation kernel (where = 1).
void check_tokens(Ctx& c, const int32_t* tokens, int64_t n, int64_t V, int where, const char* what);
void launch_convert(Ctx& c, const void* src, int src_dtype, void* dst, int dst_dtype, int64_t rows, int64_t cols,
                    bool transpose, int64_t dst_ld, int64_t dst_row0);
void launch_scripted_reward(Ctx& c, int64_t B, int64_t stride, const int32_t* tokens, const int64_t* lengths,
                            int32_t target, double* out);
void launch_f32_to_f64(Ctx& c, const float* src, int64_t n, double* dst);
void launch_fill_i32(Ctx& c, int32_t* dst, int64_t n, int32_t v);

}  // namespace ppx
