// GEMM kernel instantiations: bf16, transposed epilogue false, CTA pairs with 2-SM MMAs
// (see gemm_pick.cuh).
#include "gemm_pick.cuh"

namespace pnb {
PNB_GEMM_PICK(bf16_r_mc, __nv_bfloat16, false, false, 2)
}  // namespace pnb
