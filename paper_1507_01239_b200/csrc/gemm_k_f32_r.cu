// GEMM kernel instantiations: float, 3xTF32 split false, transposed epilogue false (see gemm_pick.cuh).
#include "gemm_pick.cuh"

namespace pnb {
PNB_GEMM_PICK(f32_r, float, false, false, 1)
}  // namespace pnb
