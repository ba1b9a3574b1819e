// umma_probe.cu — test-only: D[128, N] = A[128, 64] · B[64, N] with A K-major
// and B MN-major (N contiguous, as a row-major [keys, dh] V tile arrives from
// TMA), one CTA, to pin the MN-major 128B-swizzled shared-memory descriptor
// that the tcgen05 attention's P·V product uses.  `variant` selects the
// (leading, stride) byte-offset assignment.
#include <cuda.h>

#include "kernels.hpp"

namespace ppx {

CUtensorMap make_map(const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);  // gemm_tc.cu

namespace {

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int N>
__global__ void umma_probe_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                                  float* out, int variant) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;                 // 128 x 64 bf16 = 16 KB
  uint8_t* sB = sm + 16384;         // N/64 boxes of [64 rows x 64 cols] = 8 KB each
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 16384 + (N / 64) * 8192);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(slot)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[0])),
                 "r"(16384 + (N / 64) * 8192)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            su32(sA)),
        "l"(reinterpret_cast<uint64_t>(&tA)), "r"(su32(&bar[0])), "r"(0), "r"(0)
        : "memory");
    for (int nb = 0; nb < N / 64; ++nb)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              su32(sB + nb * 8192)),
          "l"(reinterpret_cast<uint64_t>(&tB)), "r"(su32(&bar[0])), "r"(nb * 64), "r"(0)
          : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\nW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W1;\n\t}" ::"r"(
            su32(&bar[0]))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint64_t a0 = su32(sA);
    const uint64_t da = ((a0 >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
    const uint64_t b0 = su32(sB);
    // MN-major SW128: one atom = 8 K-rows x 128 B (64 N elements); atoms repeat
    // along K every 1024 B and along N every 8192 B (the next TMA box)
    const uint64_t lbo = variant == 0 ? 8192 : 1024, sbo = variant == 0 ? 1024 : 8192;
    const uint64_t db = ((b0 >> 4) & 0x3FFFull) | (((lbo >> 4) & 0x3FFFull) << 16) | (((sbo >> 4) & 0x3FFFull) << 32) |
                        (1ull << 46) | (2ull << 61);
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    for (int k = 0; k < 4; ++k) {
      // A: +32 B per k16 inside the 128-B row; B (MN-major): +16 K-rows = 2 atoms = 2048 B
      const uint64_t ak = da + 2 * k, bk = db + ((2048 * k) >> 4);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(
              tmem),
          "l"(ak), "l"(bk), "r"(idesc), "r"(k));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[1]))
                 : "memory");
  }
  __syncwarp();
  asm volatile(
      "{\n\t.reg .pred P1;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W2;\n\t}" ::"r"(
          su32(&bar[1]))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int q = warp & 3, lane = threadIdx.x & 31, row = q * 32 + lane;
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + (uint32_t(q * 32) << 16) + uint32_t(c)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int e = 0; e < 8; ++e) out[row * N + c + e] = __uint_as_float(v[e]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

}  // namespace

void umma_probe(Ctx& c, const bf16* A, const bf16* B, int N, float* out, int variant) {
  const CUtensorMap ta = make_map(A, 128, 64, 64, 128);
  const CUtensorMap tb = make_map(B, 64, N, N, 64);  // rows = K (keys), cols = N, box 64 x 64
  const int smem = 16384 + (N / 64) * 8192 + 2048;
  auto k = N == 64 ? umma_probe_kernel<64> : umma_probe_kernel<128>;
  PPOEXP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k<<<1, 128, smem, c.stream>>>(ta, tb, out, variant);
  PPOEXP_CUDA(cudaGetLastError());
}

}  // namespace ppx
