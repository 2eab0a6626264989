// Grouped GEMM instantiation (see gemm_pick.cuh / gemm.cuh NP > 1): every
// layer's dW GEMM of a step in one persistent launch.
#include "gemm_pick.cuh"

namespace pnb {
GroupKernelFn gemm_pick_group_dw(int* smem) {
    constexpr int ST = gemm_pick_detail::stages_for<256, false>();
    *smem = GemmSmem<256, ST, __nv_bfloat16, false, true>::kBytes;
    auto k = &gemm_tc_kernel<__nv_bfloat16, 256, ST, true, true, false, true, 1, kGroupMax>;
    ensure_smem_attr(reinterpret_cast<const void*>(k), *smem);
    return k;
}
}  // namespace pnb
