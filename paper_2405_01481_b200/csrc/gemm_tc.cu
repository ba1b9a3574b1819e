// gemm_tc.cu — K3 on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
#include "kernels.hpp"

namespace ppoexp {

bool gemm_tc_bf16(Ctx&, const bf16*, int64_t, const bf16*, int64_t, int64_t, int64_t, int64_t, Epi, void*, int64_t) {
  return false;
}

}  // namespace ppoexp
