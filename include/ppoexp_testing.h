/*
 * ppoexp_testing.h — internal entry points exported for the parity tests only
 * (not part of the reference-facing boundary in ppoexp.h).
 */
#ifndef PPOEXP_TESTING_H_
#define PPOEXP_TESTING_H_

#include "ppoexp.h"

#ifdef __cplusplus
extern "C" {
#endif

/* C[M,N] (+)= A[M,K] · B[N,K]^T on device pointers (bf16 A/B).
 * epi: 0 store bf16, 1 GELU→bf16, 2 fp32 residual add, 3 store fp32.
 * path: 0 = dispatcher (tcgen05 when eligible), 1 = force SIMT. */
PPOEXP_API ppoexp_status ppoexp_testing_gemm_bf16(ppoexp_ctx ctx, const void* A, int64_t lda, const void* B, int64_t ldb,
                                       int64_t M, int64_t N, int64_t K, int32_t epi, void* C, int64_t ldc,
                                       int32_t path);

/* How often the host chose kernel variant `name` on this context (e.g.
 * "sampler:pair_uncached"); graph-captured launches count once per capture. */
PPOEXP_API ppoexp_status ppoexp_testing_variant_count(ppoexp_ctx ctx, const char* name, int64_t* out);

/* Causal prefill attention over packed ragged sequences (bf16 qkv [M, 3 d],
 * out [M, d]); path 0 = tcgen05 flash attention, 1 = mma.sync, 2 = the mixed-mode
 * split tcgen05 kernel (qkv as hi | lo planes [M, 6 d], out planes [M, 2 d]; dh 64). */
PPOEXP_API ppoexp_status ppoexp_testing_attention_prefill(ppoexp_ctx ctx, const void* qkv, const int64_t* offsets,
                                               int64_t B, int64_t max_len, int64_t H, int64_t DH, int64_t M,
                                               void* out, int32_t path);

/* D[128, N] = A[128, 64] (K-major) x B[64, N] (row-major: MN-major operand), one
 * tcgen05 MMA chain; pins the MN-major 128B-swizzle descriptor (variant 0 / 1). */
PPOEXP_API ppoexp_status ppoexp_testing_umma_probe(ppoexp_ctx ctx, const void* A, const void* B, int32_t N, float* out,
                                        int32_t variant);

/* Mixed-mode GEMM over activation planes A[M, 2K] (hi | lo bf16): epi 2 residual add,
 * 3 store fp32, 6 GELU -> hi | lo planes (C [M, 2N] bf16, ldc = row stride). */
PPOEXP_API ppoexp_status ppoexp_testing_gemm_planes(ppoexp_ctx ctx, const void* A, const void* W, int64_t M, int64_t N,
                                         int64_t K, int32_t epi, void* C, int64_t ldc);

/* Mixed-mode GEMM: C[M,N] (+)= A[M,K] (fp32) · W[N,K]^T (bf16), activations
 * split into two bf16 terms in-kernel.  epi: 2 fp32 residual add, 3 store fp32,
 * 5 GELU -> fp32.  M <= 256 takes the decode (swap-AB, cluster split-K) kernel. */
PPOEXP_API ppoexp_status ppoexp_testing_gemm_mixed(ppoexp_ctx ctx, const void* A, int64_t lda, const void* W, int64_t ldw,
                                        int64_t M, int64_t N, int64_t K, int32_t epi, void* C, int64_t ldc);

/* lp[r] = log_softmax(H[r] · W^T)[target[r]] on device pointers: H [R, K] bf16,
 * W [V, K] bf16 (the tied LM head), out[R] double.
 * path: 0 = fused tcgen05 LM head + online LSE + gather (Epi::kLse) + combine,
 *       1 = fp32 logits (tcgen05 GEMM) + K9 log-softmax/gather,
 *       2 = K9 only over caller fp32 logits (H = logits [R, ldl] fp32, W unused). */
PPOEXP_API ppoexp_status ppoexp_testing_lm_head_logprobs(ppoexp_ctx ctx, const void* H, const void* W, int64_t R,
                                              int64_t V, int64_t K, int64_t ldl, const int32_t* target,
                                              double* out, int32_t path);

#ifdef __cplusplus
}
#endif
#endif
