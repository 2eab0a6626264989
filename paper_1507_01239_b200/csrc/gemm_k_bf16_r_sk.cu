// GEMM kernel instantiations: bf16, transposed epilogue false, split-K CTA pairs exchanging partial
// tiles through distributed shared memory (see gemm_pick.cuh).
#include "gemm_pick.cuh"

namespace pnb {
PNB_GEMM_PICK(bf16_r_sk, __nv_bfloat16, false, false, 3)
}  // namespace pnb
