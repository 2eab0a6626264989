// GEMM kernel instantiations: float, 3xTF32 split false, transposed epilogue true (see gemm_pick.cuh).
#include "gemm_pick.cuh"

namespace pnb {
PNB_GEMM_PICK(f32_t, float, false, true, 1)
}  // namespace pnb
