// Microbenchmark: HBM weight streaming as the decode GEMM does it, without
// the math.  W is [N, K] bf16 (K-major, 8 KB rows at K = 4096).  Each CTA
// streams whole 128-row tiles, k-block by k-block, through an ST-stage ring:
//   mode 0: TMA 2-D boxes of 128 rows x 64 columns (128 B per row, rows 8 KB apart)
//   mode 1: the same tiles pre-packed tile-major (16 KB contiguous per k-block), 1-D bulk copies
// optionally (+2) with an L2-resident 16 KB activation chunk per k-block (the planes' re-read).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ws weight_stream.cu -lcuda && ./ws
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

constexpr int TILE = 16384;

__global__ void __launch_bounds__(32, 1) stream(const __grid_constant__ CUtensorMap tw, const uint8_t* packed,
                                                const uint8_t* xbuf, int tiles, int nk, int ST, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const bool withx = mode & 2;
  const int stride = withx ? 2 * TILE : TILE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(ring + ST * stride);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < ST; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint32_t bytes = withx ? 2 * TILE : TILE;
  int it = 0;
  auto issue = [&](int t, int kb, int s) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(bytes) : "memory");
    uint8_t* dst = ring + s * stride;
    if (mode & 1) {
      const uint8_t* src = packed + (size_t(t) * nk + kb) * TILE;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(dst)),
                   "l"(src), "r"(TILE), "r"(su32(&bar[s]))
                   : "memory");
    } else {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              su32(dst)),
          "l"(reinterpret_cast<uint64_t>(&tw)), "r"(su32(&bar[s])), "r"(kb * 64), "r"(t * 128)
          : "memory");
    }
    if (withx)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(dst + TILE)),
                   "l"(xbuf + size_t(kb) * TILE), "r"(TILE), "r"(su32(&bar[s]))
                   : "memory");
  };
  // units of this CTA: an equal contiguous range of the tiles x k-blocks units
  const long long U = (long long)tiles * nk;
  const long long u0 = blockIdx.x * U / gridDim.x, u1 = (blockIdx.x + 1) * U / gridDim.x;
  const int total = int(u1 - u0);
  int issued = 0;
  auto next = [&]() {
    const long long u = u0 + issued;
    issue(int(u / nk), int(u % nk), issued % ST);
    ++issued;
  };
  while (issued < total && issued < ST) next();
  for (it = 0; it < total; ++it) {
    const int s = it % ST;
    asm volatile(
        "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(
            su32(&bar[s])),
        "r"((it / ST) & 1)
        : "memory");
    if (issued < total) next();
  }
}

int main() {
  const int N = 12288, K = 4096, tiles = N / 128, nk = K / 64;
  uint8_t *w, *packed, *x;
  cudaMalloc(&w, size_t(N) * K * 2);
  cudaMalloc(&packed, size_t(N) * K * 2);
  cudaMalloc(&x, size_t(nk) * TILE);
  cudaMemset(w, 1, size_t(N) * K * 2);
  cudaMemset(packed, 1, size_t(N) * K * 2);
  cudaMemset(x, 1, size_t(nk) * TILE);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  CUtensorMap tw;
  const cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(N)};
  const cuuint64_t strides[1] = {cuuint64_t(K) * 2};
  const cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  uint8_t* flush;
  cudaMalloc(&flush, 512u << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* mname[4] = {"tma2d", "packed1d", "tma2d+x", "packed1d+x"};
  for (int mode = 0; mode < 4; ++mode)
    for (int G : {96, 148})
      for (int ST : {4, 8, 12}) {
        const size_t smem = size_t(ST) * ((mode & 2) ? 2 : 1) * TILE + 1024 + 256;
        if (smem > 232448) continue;
        cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        float best = 1e9f;
        for (int rep = 0; rep < 5; ++rep) {
          cudaMemset(flush, rep, 512u << 20);  // cold L2 for the weights
          cudaEventRecord(a);
          stream<<<G, 32, smem>>>(tw, packed, x, tiles, nk, ST, mode);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (rep) best = ms < best ? ms : best;
        }
        const cudaError_t e = cudaGetLastError();
        printf("%-11s G=%3d ST=%2d: %7.1f us  %5.2f TB/s weights%s\n", mname[mode], G, ST, best * 1e3,
               double(N) * K * 2 / (best * 1e-3) / 1e12, e ? cudaGetErrorString(e) : "");
      }
  return 0;
}
