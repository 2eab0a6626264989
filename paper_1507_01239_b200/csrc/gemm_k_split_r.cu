// GEMM kernel instantiations: float, 3xTF32 split true, transposed epilogue false (see gemm_pick.cuh).
#include "gemm_pick.cuh"

namespace pnb {
PNB_GEMM_PICK(split_r, float, true, false, 1)
}  // namespace pnb
