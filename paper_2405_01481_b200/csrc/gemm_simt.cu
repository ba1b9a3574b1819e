// gemm_simt.cu — K3 fallback GEMM on the CUDA cores: C = A·B^T, fp32 FMA,
// k accumulated strictly in ascending order per output (deterministic; the
// parity-mode path that keeps fp32 greedy argmaxes equal to the fp64
// reference).  bf16 GEMMs on the hot path go to gemm_tc.cu (tcgen05).
#include "kernels.hpp"

namespace ppx {

namespace {
constexpr int BM = 64, BN = 64, BK = 16;

template <class T, int EPI>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const T* __restrict__ A, int64_t lda,
                                                         const T* __restrict__ B, int64_t ldb, int64_t M,
                                                         int64_t N, int64_t K, void* __restrict__ Cv,
                                                         int64_t ldc) {
  PDL_ENTRY();
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = int64_t(blockIdx.y) * BM, n0 = int64_t(blockIdx.x) * BN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  const int lrow = tid >> 2, lk = (tid & 3) * 4;
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t kk = k0 + lk + i;
      const int64_t ma = m0 + lrow, nb = n0 + lrow;
      As[lk + i][lrow] = (ma < M && kk < K) ? to_f(A[ma * lda + kk]) : 0.f;
      Bs[lk + i][lrow] = (nb < N && kk < K) ? to_f(B[nb * ldb + kk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a4 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float a[4] = {a4.x, a4.y, a4.z, a4.w};
      const float b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      if (n >= N) continue;
      const float v = acc[i][j];
      if constexpr (EPI == int(Epi::kStore)) {
        static_cast<T*>(Cv)[m * ldc + n] = from_f<T>(v);
      } else if constexpr (EPI == int(Epi::kGelu)) {
        static_cast<T*>(Cv)[m * ldc + n] = from_f<T>(gelu_tanh(v));
      } else if constexpr (EPI == int(Epi::kAddResidual)) {
        static_cast<float*>(Cv)[m * ldc + n] += v;
      } else {
        static_cast<float*>(Cv)[m * ldc + n] = v;
      }
    }
  }
}
}  // namespace

template <class T>
void launch_gemm_simt(Ctx& c, const T* A, int64_t lda, const T* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                      Epi epi, void* C, int64_t ldc) {
  if (M <= 0 || N <= 0) return;
  dim3 grid(ceil_div(N, BN), ceil_div(M, BM));
  const double flops = 2.0 * M * N * K;
  const double bytes = double(M) * K * sizeof(T) + double(N) * K * sizeof(T) +
                       double(M) * N * ((epi == Epi::kStore || epi == Epi::kGelu) ? sizeof(T) : 4);
  c.launch("gemm_simt", bytes, flops, [&] {
    switch (epi) {
      case Epi::kStore:
        launch_kernel(c, gemm_simt_kernel<T, 0>, dim3(grid), dim3(256), 0, 1, A, lda, B, ldb, M, N, K, C, ldc);
        break;
      case Epi::kGelu:
        launch_kernel(c, gemm_simt_kernel<T, 1>, dim3(grid), dim3(256), 0, 1, A, lda, B, ldb, M, N, K, C, ldc);
        break;
      case Epi::kAddResidual:
        launch_kernel(c, gemm_simt_kernel<T, 2>, dim3(grid), dim3(256), 0, 1, A, lda, B, ldb, M, N, K, C, ldc);
        break;
      case Epi::kStoreF32:
        launch_kernel(c, gemm_simt_kernel<T, 3>, dim3(grid), dim3(256), 0, 1, A, lda, B, ldb, M, N, K, C, ldc);
        break;
      case Epi::kLse:
        throw ContractError("gemm_simt: no LSE epilogue");
    }
  });
}

template void launch_gemm_simt<float>(Ctx&, const float*, int64_t, const float*, int64_t, int64_t, int64_t, int64_t,
                                      Epi, void*, int64_t);
template void launch_gemm_simt<bf16>(Ctx&, const bf16*, int64_t, const bf16*, int64_t, int64_t, int64_t, int64_t,
                                     Epi, void*, int64_t);

}  // namespace ppx
