// GEMM kernel instantiations: bf16, transposed epilogue true, CTA pairs with 2-SM MMAs
// (see gemm_pick.cuh).
#include "gemm_pick.cuh"

namespace pnb {
PNB_GEMM_PICK(bf16_t_mc, __nv_bfloat16, false, true, 2)
}  // namespace pnb
