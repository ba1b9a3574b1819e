// Microbenchmark: critical-path cost per kernel of a dependent chain captured
// in a CUDA graph, with and without programmatic dependent launch (PDL), for
// (a) empty kernels (launch + dependency floor) and (b) kernels that read a
// 16 KB slice from L2 and write 512 B (a minimal "real" step).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdl pdl_chain.cu && ./pdl
#include <cstdio>

__global__ void k_empty(int pdl) {
  if (pdl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
}

__global__ void k_touch(const float4* __restrict__ in, float* __restrict__ out, int pdl) {
  if (pdl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  // each CTA reads 16 KB (4 float4 per thread x 256 threads) and writes one float per warp
  const float4* p = in + size_t(blockIdx.x) * 1024;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float4 v = __ldcg(p + threadIdx.x + i * 256);
    s += v.x + v.y + v.z + v.w;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 8 + (threadIdx.x >> 5)] = s;
}

int main() {
  cudaStream_t st;
  cudaStreamCreate(&st);
  float4* in;
  float* out;
  cudaMalloc(&in, size_t(148) * 1024 * 16);
  cudaMalloc(&out, 148 * 8 * 4);
  cudaMemset(in, 0, size_t(148) * 1024 * 16);
  const int n = 200;
  for (int kind = 0; kind < 2; ++kind)
    for (int pdl = 0; pdl < 2; ++pdl)
      for (int grid : {1, 148}) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < n; ++i) {
          cudaLaunchConfig_t cfg{};
          cfg.gridDim = dim3(grid);
          cfg.blockDim = dim3(256);
          cfg.stream = st;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = pdl;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          if (kind == 0)
            cudaLaunchKernelEx(&cfg, k_empty, pdl);
          else
            cudaLaunchKernelEx(&cfg, k_touch, (const float4*)in, out, pdl);
        }
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st);
        cudaStreamSynchronize(st);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, st);
        for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-6s pdl=%d grid=%3d: %.2f us per kernel\n", kind ? "touch" : "empty", pdl, grid, ms * 1e3 / (5 * n));
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
      }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
