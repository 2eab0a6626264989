// Kernel instantiation + launch-attribute setup for one operand type /
// epilogue style. The GEMM kernels are instantiated in six translation units
// (gemm_k_*.cu: {bf16, tf32, 3xTF32} x {row-wise, transposed epilogue}, plus
// the bf16 CTA-pair kernels with 2-SM MMAs) so
// they compile in parallel; gemm.cu picks among them at plan time.
#pragma once
#include <stdexcept>

#include "gemm.cuh"
#include "runtime.h"

namespace pnb {

using KernelFn = void (*)(GemmParams<1>);
using GroupKernelFn = void (*)(GemmParams<kGroupMax>);

namespace gemm_pick_detail {

template <int BN, bool SPLIT>
constexpr int stages_for() {
    if (SPLIT) return BN == 256 ? 2 : (BN == 128 ? 3 : 4);
    return BN == 256 ? 4 : (BN == 128 ? 6 : 8);
}

template <typename T, int BN, bool AMN, bool BMN, bool SPLIT, bool TE, int MC>
KernelFn kernel_ptr(int* smem) {
    constexpr int ST = stages_for<BN, SPLIT>();
    *smem = GemmSmem<BN, ST, T, SPLIT, TE>::kBytes;
    auto k = &gemm_tc_kernel<T, BN, ST, AMN, BMN, SPLIT, TE, MC, 1>;
    ensure_smem_attr(reinterpret_cast<const void*>(k), *smem);
    return reinterpret_cast<KernelFn>(k);
}

template <typename T, int BN, bool SPLIT, bool TE, int MC>
KernelFn pick_major(bool amn, bool bmn, int* smem) {
    if (!amn && !bmn) return kernel_ptr<T, BN, false, false, SPLIT, TE, MC>(smem);
    if (amn && bmn) return kernel_ptr<T, BN, true, true, SPLIT, TE, MC>(smem);
    if (!amn && bmn) return kernel_ptr<T, BN, false, true, SPLIT, TE, MC>(smem);
    return kernel_ptr<T, BN, true, false, SPLIT, TE, MC>(smem);
}

template <typename T, bool SPLIT, bool TE, int MC>
KernelFn pick(int bn, bool amn, bool bmn, int* smem) {
    if constexpr (MC != 1) {
        if (bn == 256) return pick_major<T, 256, SPLIT, TE, MC>(amn, bmn, smem);
        if (bn == 128) return pick_major<T, 128, SPLIT, TE, MC>(amn, bmn, smem);
        throw std::runtime_error("gemm: CTA-pair tiles need BN >= 128");
    } else {
        switch (bn) {
            case 256: return pick_major<T, 256, SPLIT, TE, MC>(amn, bmn, smem);
            case 128: return pick_major<T, 128, SPLIT, TE, MC>(amn, bmn, smem);
            default: return pick_major<T, 64, SPLIT, TE, MC>(amn, bmn, smem);
        }
    }
}

}  // namespace gemm_pick_detail

// one per gemm_k_*.cu
KernelFn gemm_pick_bf16_r(int bn, bool amn, bool bmn, int* smem);
KernelFn gemm_pick_bf16_t(int bn, bool amn, bool bmn, int* smem);
KernelFn gemm_pick_f32_r(int bn, bool amn, bool bmn, int* smem);
KernelFn gemm_pick_f32_t(int bn, bool amn, bool bmn, int* smem);
KernelFn gemm_pick_split_r(int bn, bool amn, bool bmn, int* smem);
KernelFn gemm_pick_split_t(int bn, bool amn, bool bmn, int* smem);
KernelFn gemm_pick_bf16_r_mc(int bn, bool amn, bool bmn, int* smem);  // CTA pairs, 2-SM MMA
KernelFn gemm_pick_bf16_t_mc(int bn, bool amn, bool bmn, int* smem);
KernelFn gemm_pick_bf16_r_sk(int bn, bool amn, bool bmn, int* smem);  // split-K CTA pairs (DSMEM exchange)
KernelFn gemm_pick_bf16_t_sk(int bn, bool amn, bool bmn, int* smem);
// grouped launches (gemm_k_group.cu): bf16, BN = 256, both operands MN-major,
// transposed epilogue, single-CTA tiles -- the trainer's dW GEMMs
GroupKernelFn gemm_pick_group_dw(int* smem);

#define PNB_GEMM_PICK(name, T, SPLIT, TE, MC)                                 \
    KernelFn gemm_pick_##name(int bn, bool amn, bool bmn, int* smem) {        \
        return gemm_pick_detail::pick<T, SPLIT, TE, MC>(bn, amn, bmn, smem);  \
    }

}  // namespace pnb
