// GEMM kernel instantiations: bf16, transposed epilogue true, split-K CTA pairs exchanging partial
// tiles through distributed shared memory (see gemm_pick.cuh).
#include "gemm_pick.cuh"

namespace pnb {
PNB_GEMM_PICK(bf16_t_sk, __nv_bfloat16, false, true, 3)
}  // namespace pnb
