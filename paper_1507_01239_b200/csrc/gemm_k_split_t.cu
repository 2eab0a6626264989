// GEMM kernel instantiations: float, 3xTF32 split true, transposed epilogue true (see gemm_pick.cuh).
#include "gemm_pick.cuh"

namespace pnb {
PNB_GEMM_PICK(split_t, float, true, true, 1)
}  // namespace pnb
