// GEMM kernel instantiations: __nv_bfloat16, 3xTF32 split false, transposed epilogue false (see gemm_pick.cuh).
#include "gemm_pick.cuh"

namespace pnb {
PNB_GEMM_PICK(bf16_r, __nv_bfloat16, false, false, 1)
}  // namespace pnb
