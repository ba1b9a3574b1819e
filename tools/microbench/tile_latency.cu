// Microbenchmark: latency of loading one 24 KB weight tile (16 rows x 1.5 KB)
// into shared memory, one CTA per SM, by mechanism:
//   0 = cp.async.bulk rows + mbarrier, 1 = cp.async 16 B (8 warps), 2 = ld.global.v4
// Each CTA reads its own tile of a large buffer (cold: fresh region each
// rep; warm: same region as the previous rep).  Prints median cycles.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tl tile_latency.cu && ./tl
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(256, 1) tile_kernel(const uint8_t* buf, size_t region, int mode, int rep_stride,
                                                     long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t mb;
  __shared__ uint32_t ph;
  const int tid = threadIdx.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    ph = 0;
  }
  __syncthreads();
  for (int rep = 0; rep < 8; ++rep) {
    const uint8_t* src = buf + (size_t(rep / rep_stride) * gridDim.x + blockIdx.x) * 24576 % region;
    __syncthreads();
    long long t0 = clock64();
    if (mode == 0) {
      if (tid < 32) {
        if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mb)), "r"(24576));
        __syncwarp();
        if (tid < 16)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1536, [%2];" ::"r"(
                           su32(sm + tid * 1552)),
                       "l"(src + tid * 1536), "r"(su32(&mb))
                       : "memory");
      }
      const uint32_t p = ph;
      asm volatile(
          "{\n .reg .pred q;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n @!q bra W_%=;\n}" ::"r"(
              su32(&mb)),
          "r"(p)
          : "memory");
      __syncthreads();
      if (tid == 0) ph ^= 1u;
    } else if (mode == 1) {
      for (int e = tid; e < 1536; e += 256) {
        const int r = e / 96, c = e % 96;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(sm + r * 1552 + c * 16)),
                     "l"(src + r * 1536 + c * 16)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      __syncthreads();
    } else {
      uint4 v[6];
#pragma unroll
      for (int i = 0; i < 6; ++i) v[i] = __ldcg(reinterpret_cast<const uint4*>(src) + tid + i * 256);
#pragma unroll
      for (int i = 0; i < 6; ++i) reinterpret_cast<uint4*>(sm)[tid + i * 256] = v[i];
      __syncthreads();
    }
    long long t1 = clock64();
    if (tid == 0) out[rep * gridDim.x + blockIdx.x] = t1 - t0;
  }
}

int main() {
  const size_t region = size_t(1) << 30;  // 1 GiB (>> L2)
  uint8_t* buf;
  cudaMalloc(&buf, region);
  cudaMemset(buf, 1, region);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* out;
  cudaMalloc(&out, 8 * sms * 8);
  cudaFuncSetAttribute(tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const char* names[3] = {"bulk", "cp.async", "ld.v4"};
  for (int grid : {1, sms})
    for (int mode = 0; mode < 3; ++mode)
      for (int warm = 0; warm < 2; ++warm) {
        // flush L2 by touching a different 256 MB region
        cudaMemset(buf + (size_t(768) << 20), 2, size_t(256) << 20);
        tile_kernel<<<grid, 256, 64 * 1024>>>(buf, region, mode, warm ? 8 : 1, out);
        cudaDeviceSynchronize();
        std::vector<long long> h(8 * grid);
        cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
        std::vector<long long> r(h.begin() + grid, h.end());  // skip rep 0 (first touch of code/TLB)
        std::sort(r.begin(), r.end());
        printf("grid %3d %-8s %-4s  median %6lld cyc  max %6lld  first-rep median %6lld\n", grid, names[mode],
               warm ? "warm" : "cold", r[r.size() / 2], r.back(), h[grid / 2]);
      }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
