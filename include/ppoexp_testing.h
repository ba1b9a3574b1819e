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

#ifdef __cplusplus
}
#endif
#endif
