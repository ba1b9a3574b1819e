// Microbenchmark: per-SM L2 -> shared-memory ingress bandwidth.
// Each CTA (one per SM) streams `bytes` from global into a 64 KB smem ring,
// either from the SAME buffer for all CTAs (broadcast hot-spot, like the
// decode GEMM's activation tile) or from a distinct buffer per CTA.
// Mechanisms: cp.async.bulk (one warp, 4 KB chunks), cp.async 16 B (all warps).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2i l2_ingress.cu && ./l2i
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(256, 1) ingress(const uint8_t* buf, size_t bytes, int distinct, int mode,
                                                 long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t mb;
  const int tid = threadIdx.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint8_t* src = buf + (distinct ? size_t(blockIdx.x) * bytes : 0);
  // warm L2 with one pass
  for (size_t o = tid * 16; o < bytes; o += 256 * 16) (void)__ldcg(reinterpret_cast<const uint4*>(src + o));
  __syncthreads();
  long long t0 = clock64();
  if (mode == 0) {
    uint32_t ph = 0;
    const size_t chunk = 4096;
    for (size_t o = 0; o < bytes; o += 16 * chunk) {  // 64 KB per round
      const size_t n = (16 * chunk < bytes - o ? 16 * chunk : bytes - o);
      if (tid < 32) {
        if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mb)), "r"(uint32_t(n)));
        __syncwarp();
        if (tid < int(n / chunk))
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           su32(sm + tid * chunk)),
                       "l"(src + o + tid * chunk), "r"(uint32_t(chunk)), "r"(su32(&mb))
                       : "memory");
      }
      asm volatile(
          "{\n .reg .pred q;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n @!q bra W_%=;\n}" ::"r"(
              su32(&mb)),
          "r"(ph)
          : "memory");
      ph ^= 1;
      __syncthreads();
    }
  } else {
    for (size_t o = 0; o < bytes; o += 65536) {
      for (int e = tid; e < 4096; e += 256)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(sm + e * 16)), "l"(src + o + e * 16) : "memory");
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      __syncthreads();
    }
  }
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = size_t(1) << 20;  // 1 MB per CTA
  uint8_t* buf;
  cudaMalloc(&buf, bytes * sms);
  cudaMemset(buf, 1, bytes * sms);
  long long* out;
  cudaMalloc(&out, sms * 8);
  cudaFuncSetAttribute(ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const char* mn[2] = {"bulk", "cp.async"};
  for (int grid : {1, 8, sms})
    for (int distinct = 0; distinct < 2; ++distinct)
      for (int mode = 0; mode < 2; ++mode) {
        ingress<<<grid, 256, 65536>>>(buf, bytes, distinct, mode, out);
        ingress<<<grid, 256, 65536>>>(buf, bytes, distinct, mode, out);
        cudaDeviceSynchronize();
        std::vector<long long> h(grid);
        cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost);
        std::sort(h.begin(), h.end());
        const double med = double(h[grid / 2]);
        printf("grid %3d %-8s %-9s  %.1f B/clk/SM (median), aggregate %.2f TB/s @1.965GHz\n", grid, mn[mode],
               distinct ? "distinct" : "same-data", bytes / med, bytes / med * grid * 1.965e9 / 1e12);
      }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
