// GEMM kernel instantiations: __nv_bfloat16, 3xTF32 split false, transposed epilogue true (see gemm_pick.cuh).
#include "gemm_pick.cuh"

namespace pnb {
PNB_GEMM_PICK(bf16_t, __nv_bfloat16, false, true, 1)
}  // namespace pnb
