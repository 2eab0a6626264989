// Host side of the tcgen05 GEMM: TMA tensor-map construction, tile-shape
// selection and launch. See gemm.cuh for the kernel.
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gemm.cuh"
#include "gemm_pick.cuh"
#include "runtime.h"

namespace pnb {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw std::runtime_error("gemm: cuTensorMapEncodeTiled unavailable");
    return fn;
}

// 2D row-major tensor [outer x inner] with row pitch ld (elements), box
// {box_inner, box_outer}, 128-B swizzle, zero OOB fill.
CUtensorMap make_tmap(const void* base, bool f32, uint64_t inner, uint64_t outer, uint64_t ld,
                      uint32_t box_inner, uint32_t box_outer, bool mn_major = false) {
    CUtensorMap m;
    const uint64_t esz = f32 ? 4 : 2;
    if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld * esz) & 15))
        throw std::runtime_error("gemm: TMA operand must be 16-byte aligned (base " +
                                 std::to_string(reinterpret_cast<uintptr_t>(base)) + ", ld " + std::to_string(ld) + ")");
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld * esz};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                              const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              (f32 && mn_major) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("gemm: cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return m;
}

}  // namespace

int choose_bn(int M, int N, int num_sms) {
    const int mt = (M + 127) / 128;
    for (int bn : {256, 128}) {
        const long tiles = long(mt) * ((N + bn - 1) / bn);
        if (tiles >= (num_sms * 3) / 4) return bn;
    }
    return 64;
}

void gemm_plan(GemmPlan& p, int prec, bool a_mn, const void* A, long lda, bool b_mn, const void* B, long ldb,
               int M, int N, int K, const GemmEpi& ep, int num_sms, int force_bn, int force_mc) {
    if (M <= 0 || N <= 0 || K <= 0) throw std::runtime_error("gemm: empty problem");
    const bool f32 = prec != 0, split = prec == 2;
    const int bn = force_bn ? force_bn : choose_bn(M, N, num_sms);
    const uint32_t atom = f32 ? 32 : 64;  // elements per 128-B row
    const uint32_t bk = atom;
    // split-K: round the factor so that every split owns >= 1 k-block
    const int nk = static_cast<int>((K + bk - 1) / bk);
    const int per = (nk + std::max(ep.ksplit, 1) - 1) / std::max(ep.ksplit, 1);
    const int ksplit = (nk + per - 1) / per;
    if (ksplit > 1 && ep.mode != EPI_PARTIAL) throw std::runtime_error("gemm: split-K needs EPI_PARTIAL");
    const int tiles_m = (M + 127) / 128, tiles_n = (N + bn - 1) / bn;
    // CTA pairs with 2-SM MMAs (256 x BN pair tiles, each SM loads its A rows and half
    // of B): opt-in (PARNN_GEMM_PAIRS=1). Measured on the trainer's shapes it is no
    // faster than single-CTA tiles (the mainloop is bound by MMA consumption, not by
    // operand delivery), so the default stays 1-SM.
    static const bool pairs_on = [] {
        const char* v = std::getenv("PARNN_GEMM_PAIRS");
        return v && v[0] == '1';
    }();
    p.mc = (!f32 && pairs_on && ksplit == 1 && !ep.lower && bn >= 128 && tiles_m >= 2) ? 2 : 1;
    // Split-K CTA pairs (mc = 3): a GEMM whose 128 x 256 tiles number at most half the
    // SMs runs each tile on a cluster of two CTAs, one per half of K, exchanging the
    // partial tiles through distributed shared memory. N = 256 MMAs run at ~95% of
    // the tensor peak where the N = 128 tiles that would otherwise fill the GPU
    // reach ~66%.
    static const bool sk_off = [] {
        const char* v = std::getenv("PARNN_GEMM_SK2");
        return v && v[0] == '0';
    }();
    int bn_eff = bn;
    if (force_mc) {
        if (force_mc == 2 && (f32 || ksplit != 1 || ep.lower || bn < 128 || tiles_m < 2))
            throw std::runtime_error("gemm: CTA pairs need bf16, no split-K / lower, BN >= 128 and >= 2 row tiles");
        if (force_mc == 3 && (f32 || ksplit != 1 || ep.lower || nk < 2))
            throw std::runtime_error("gemm: split-K CTA pairs need bf16, no split-K / lower and >= 2 k-blocks");
        p.mc = force_mc;
        if (force_mc == 3) bn_eff = 256;
    } else if (p.mc == 1 && !f32 && !sk_off && !force_bn && ksplit == 1 && !ep.lower && nk >= 8) {
        const long t256 = static_cast<long>(tiles_m) * ((N + 255) / 256);
        static const int min_frac = [] {  // tuning aid: pairs must fill >= 1/x of the SMs
            const char* v = std::getenv("PARNN_GEMM_SK2_FRAC");
            return v ? std::max(1, std::atoi(v)) : 2;
        }();
        if (2 * t256 <= num_sms && 2 * t256 >= num_sms / min_frac) {
            p.mc = 3;
            bn_eff = 256;
        }
    }
    // A(m,k): K-major buffer [M x K] or MN-major buffer [K x M].
    p.ta = a_mn ? make_tmap(A, f32, M, K, lda, atom, bk, true) : make_tmap(A, f32, K, M, lda, bk, 128);
    p.tb = b_mn ? make_tmap(B, f32, N, K, ldb, atom, bk, true)
                : make_tmap(B, f32, K, N, ldb, bk, p.mc == 2 ? bn_eff / 2 : bn_eff);
    p.M = M;
    p.N = N;
    p.K = K;
    p.prec = prec;
    p.a_mn = a_mn;
    p.b_mn = b_mn;
    p.ep = ep;
    p.ep.ksplit = ksplit;
    if (p.mc == 3) {
        const long t = static_cast<long>(tiles_m) * ((N + bn_eff - 1) / bn_eff);
        p.grid = dim3(static_cast<unsigned>(2 * t), 1, 1);  // one tile per cluster (the ring holds the exchange)
        p.tiles = static_cast<int>(t);
    } else if (p.mc == 2) {
        const long pairs = static_cast<long>((tiles_m + 1) / 2) * tiles_n;
        p.grid = dim3(static_cast<unsigned>(2 * std::min<long>(pairs, num_sms / 2)), 1, 1);
        p.tiles = static_cast<int>(2 * pairs);
    } else {
        const long tiles = static_cast<long>(tiles_n) * tiles_m * ksplit;
        p.grid = dim3(static_cast<unsigned>(std::min<long>(tiles, num_sms)), 1, 1);  // persistent
        p.tiles = static_cast<int>(tiles);
    }
    const bool te = gemm_epi_transposed(ep.mode);
    KernelFn fn;
    if (p.mc == 3)
        fn = te ? gemm_pick_bf16_t_sk(bn_eff, a_mn, b_mn, &p.smem) : gemm_pick_bf16_r_sk(bn_eff, a_mn, b_mn, &p.smem);
    else if (p.mc == 2)
        fn = te ? gemm_pick_bf16_t_mc(bn, a_mn, b_mn, &p.smem) : gemm_pick_bf16_r_mc(bn, a_mn, b_mn, &p.smem);
    else if (split)
        fn = te ? gemm_pick_split_t(bn, a_mn, b_mn, &p.smem) : gemm_pick_split_r(bn, a_mn, b_mn, &p.smem);
    else if (f32)
        fn = te ? gemm_pick_f32_t(bn, a_mn, b_mn, &p.smem) : gemm_pick_f32_r(bn, a_mn, b_mn, &p.smem);
    else
        fn = te ? gemm_pick_bf16_t(bn, a_mn, b_mn, &p.smem) : gemm_pick_bf16_r(bn, a_mn, b_mn, &p.smem);
    p.fn = reinterpret_cast<void*>(fn);
    p.bn = bn_eff;
    p.threads = split ? 448 : 320;  // GemmSmem::kThreads
}

namespace {
thread_local int g_grid_cap = 0;
}

void ensure_smem_attr(const void* fn, int bytes) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void*, int>, int>> done;  // (fn, device) -> bytes set
    int dev = 0;
    CUDA_THROW(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    for (auto& d : done)
        if (d.first.first == fn && d.first.second == dev && d.second >= bytes) return;
    CUDA_THROW(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.push_back({{fn, dev}, bytes});
}

void gemm_set_grid_cap(int cap) { g_grid_cap = cap; }
thread_local bool g_pdl_off = false;
void gemm_set_pdl(bool on) { g_pdl_off = !on; }

dim3 gemm_launch_grid(const GemmPlan& p) {
    // the persistent kernel covers every tile with any grid (tile = blockIdx + k * gridDim;
    // CTA pairs: pair = blockIdx / 2 + k * gridDim / 2, so the grid stays even)
    if (p.mc == 3) return p.grid;  // one tile per cluster: the grid cannot shrink
    if (g_grid_cap > 0 && static_cast<int>(p.grid.x) > g_grid_cap)
        return dim3(p.mc == 2 ? std::max(2, g_grid_cap & ~1) : g_grid_cap, 1, 1);
    return p.grid;
}

// Every GEMM is launched with programmatic stream serialization (PDL): the
// kernel may start while the previous kernel of its stream finishes; it runs
// its prologue (barriers, TMEM, descriptor prefetch) and then waits in
// griddepcontrol.wait until that kernel has completed and its writes are
// visible. The previous GEMM releases it once its own mainloop is done. Every
// grid here fits the GPU in one wave (persistent, <= #SMs CTAs), so an early
// dependent can only take SMs its predecessor does not hold.
// PARNN_NO_PDL=1 turns it off (A/B timing).
void gemm_launch(const GemmPlan& p, cudaStream_t s) {
    static const bool pdl = [] {
        const char* v = std::getenv("PARNN_NO_PDL");
        return !(v && v[0] == '1');
    }();
    auto fn = reinterpret_cast<KernelFn>(p.fn);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = gemm_launch_grid(p);
    cfg.blockDim = dim3(p.threads, 1, 1);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (p.mc != 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 2;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (pdl && !g_pdl_off) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    GemmParams<1> args;
    args.ta[0] = p.ta;
    args.tb[0] = p.tb;
    args.ep[0] = p.ep;
    args.M[0] = p.M;
    args.N[0] = p.N;
    args.K[0] = p.K;
    args.tile0[0] = 0;
    args.tile0[1] = p.tiles;
    args.np = 1;
    CUDA_THROW(cudaLaunchKernelEx(&cfg, fn, args));
    CUDA_THROW(cudaGetLastError());
}

bool gemm_groupable(const GemmPlan& p) {
    return p.prec == PREC_BF16 && p.a_mn && p.b_mn && p.bn == 256 && p.mc == 1 && p.ep.ksplit == 1 && !p.ep.lower &&
           p.ep.mode == EPI_GRAD_SGD && p.ep.out32;
}

void gemm_group_plan(GemmGroupPlan& g, const std::vector<const GemmPlan*>& parts, int num_sms) {
    if (parts.empty() || parts.size() > static_cast<size_t>(kGroupMax))
        throw std::runtime_error("gemm: a group holds 1.." + std::to_string(kGroupMax) + " problems");
    g.np = static_cast<int>(parts.size());
    int t = 0;
    for (int i = 0; i < g.np; ++i) {
        const GemmPlan& p = *parts[i];
        if (!gemm_groupable(p)) throw std::runtime_error("gemm: problem " + std::to_string(i) + " cannot be grouped");
        g.args.ta[i] = p.ta;
        g.args.tb[i] = p.tb;
        g.args.ep[i] = p.ep;
        g.args.M[i] = p.M;
        g.args.N[i] = p.N;
        g.args.K[i] = p.K;
        g.args.tile0[i] = t;
        t += ((p.M + 127) / 128) * ((p.N + 255) / 256);
    }
    g.args.tile0[g.np] = t;
    g.args.np = g.np;
    g.tiles = t;
    g.grid = dim3(static_cast<unsigned>(std::min(t, num_sms)), 1, 1);
    g.fn = reinterpret_cast<void*>(gemm_pick_group_dw(&g.smem));
    g.threads = 320;
}

void gemm_group_launch(const GemmGroupPlan& g, cudaStream_t s) {
    static const bool pdl = [] {
        const char* v = std::getenv("PARNN_NO_PDL");
        return !(v && v[0] == '1');
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = (g_grid_cap > 0 && static_cast<int>(g.grid.x) > g_grid_cap) ? dim3(g_grid_cap, 1, 1) : g.grid;
    cfg.blockDim = dim3(g.threads, 1, 1);
    cfg.dynamicSmemBytes = g.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    CUDA_THROW(cudaLaunchKernelEx(&cfg, reinterpret_cast<GroupKernelFn>(g.fn), g.args));
    CUDA_THROW(cudaGetLastError());
}

}  // namespace pnb
