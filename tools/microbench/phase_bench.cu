// Microbenchmark: the persistent decode kernel's GEMM phase (QKV shape,
// B=64, d=768) run as a standalone kernel, one CTA per SM, so its intrinsic
// cost can be compared with the in-kernel trace (tools/mega_trace.py).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I include -o tools/microbench/pb tools/microbench/phase_bench.cu
#include "../../paper_2405_01481_b200/csrc/decode_mega.cu"

cudaEvent_t ppx::Ctx::new_event() { return nullptr; }  // unused by this harness

namespace ppx {
namespace {
__global__ void __launch_bounds__(kThreads, 1) phase_kernel(const bf16* X, const bf16* W, bf16* out, int d, int prefetch,
                                                            uint64_t* st) {
  extern __shared__ __align__(128) uint8_t smem_pb[];
  __shared__ __align__(8) uint64_t mbars[3];
  __shared__ uint32_t phases[3];
  const int KCW = 1024;
  Sm sm{reinterpret_cast<bf16*>(smem_pb), KCW, smem_pb + size_t(2) * kTileN * (KCW + 8) * 2, mbars, phases};
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) {
      mbar_init(&mbars[i], 1);
      phases[i] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const GemmJob jq{X, d, W, 3 * d, d, 1};
  uint64_t* my = st + blockIdx.x * 8;
  const uint64_t t0 = clock64();
  bool pf = false;
  if (prefetch) {
    pf = prefetch_w(sm, jq, nullptr);
    // wait long enough for the weights to land
    const uint64_t tw = clock64();
    while (clock64() - tw < 20000) {
    }
    __syncthreads();
  }
  const uint64_t t1 = clock64();
  gemm_phase<0>(sm, jq, 64, out, 3 * d, pf, my);
  const uint64_t t2 = clock64();
  if (threadIdx.x == 0) {
    my[4] = t1;
    my[5] = t2;
    my[6] = t0;
  }
}
}  // namespace
}  // namespace ppx

int main() {
  using namespace ppx;
  const int d = 768;
  bf16 *X, *W, *out;
  cudaMalloc(&X, 64 * d * 2);
  cudaMalloc(&W, size_t(3) * d * d * 2);
  cudaMalloc(&out, 64 * 3 * d * 2);
  cudaMemset(X, 0, 64 * d * 2);
  cudaMemset(W, 0, size_t(3) * d * d * 2);
  uint64_t* st;
  cudaMalloc(&st, 148 * 8 * 8);
  const size_t smem = mega_smem<64>(1024);
  cudaFuncSetAttribute(phase_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  for (int pf = 0; pf < 2; ++pf)
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(st, 0, 148 * 64);
      phase_kernel<<<148, kThreads, smem>>>(X, W, out, d, pf, st);
      cudaDeviceSynchronize();
      uint64_t h[148 * 8];
      cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
      // median over CTAs with work (first stamp set)
      std::vector<double> wr, xr, mm, ep, tot;
      for (int c = 0; c < 148; ++c) {
        const uint64_t* m = h + c * 8;
        if (!m[0]) continue;
        wr.push_back(double(m[3] - m[4]));
        xr.push_back(double(m[0] - m[4]));
        mm.push_back(double(m[1] - m[4]));
        ep.push_back(double(m[2] - m[4]));
        tot.push_back(double(m[5] - m[4]));
      }
      auto med = [](std::vector<double> v) {
        std::sort(v.begin(), v.end());
        return v[v.size() / 2];
      };
      printf("prefetch %d rep %d: cycles after phase start  W rdy %6.0f  X rdy %6.0f  mma %6.0f  epi %6.0f  end %6.0f\n",
             pf, rep, med(wr), med(xr), med(mm), med(ep), med(tot));
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
