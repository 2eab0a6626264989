// Test hook behind parnn_debug_gemm: ONE production GEMM plan (gemm_plan's
// tile / cluster selection, the same kernel instantiations and fused
// epilogues the trainer launches) on caller data, so the tests can check every
// path of the tcgen05 GEMM against an fp64 product at the trainer's real
// shapes: operand precisions (bf16, tf32, 3xTF32), operand majors (K / MN),
// cluster modes (1-SM tiles, 2-SM CTA pairs, split-K CTA pairs), split-K
// partials, ragged M / N / K and every epilogue mode.
#include <cstring>
#include <vector>

#include "runtime.h"

namespace pnb {

namespace {

// host fp32 rows [rows x cols] -> device operand buffer [rows x ld] (zero padded)
void* upload(const float* h, long rows, long cols, long ld, bool f32) {
    void* d = nullptr;
    const size_t es = f32 ? 4 : 2;
    CUDA_THROW(cudaMalloc(&d, static_cast<size_t>(rows * ld) * es + 256));
    zero(d, static_cast<size_t>(rows * ld) * es + 256);
    if (f32) {
        CUDA_THROW(cudaMemcpy2D(d, ld * 4, h, cols * 4, cols * 4, rows, cudaMemcpyHostToDevice));
        CUDA_THROW(cudaStreamSynchronize(cudaStreamLegacy));
    } else {
        std::vector<bf16> t(static_cast<size_t>(rows * ld), __float2bfloat16_rn(0.f));
        for (long r = 0; r < rows; ++r)
            for (long c = 0; c < cols; ++c) t[r * ld + c] = __float2bfloat16_rn(h[r * cols + c]);
        pnb::upload(d, t.data(), t.size() * 2);
    }
    return d;
}

void download(float* h, const void* d, long rows, long cols, long ld, bool f32) {
    const size_t es = f32 ? 4 : 2;
    std::vector<uint8_t> t(static_cast<size_t>(rows * ld) * es);
    CUDA_THROW(cudaMemcpy(t.data(), d, t.size(), cudaMemcpyDeviceToHost));
    for (long r = 0; r < rows; ++r)
        for (long c = 0; c < cols; ++c)
            h[r * cols + c] = f32 ? reinterpret_cast<const float*>(t.data())[r * ld + c]
                                  : __bfloat162float(reinterpret_cast<const bf16*>(t.data())[r * ld + c]);
}

}  // namespace

// info[6] = {cluster mode used, BN used, split-K factor used, non-finite flag bits, grid, threads}
void debug_gemm(int prec, bool a_mn, bool b_mn, int M, int N, int K, int mode, int act, int ksplit, int force_bn,
                int force_mc, int lower, int bias_col, float alpha, float beta, float lr, const float* a,
                const float* b, const float* bias, const float* aux, float* out, float* out2, double* sums,
                int* info) {
    if (M <= 0 || N <= 0 || K <= 0) throw std::runtime_error("gemm: empty problem");
    const bool f32 = prec != PREC_BF16;
    int dev = 0, sms = 148;
    CUDA_THROW(cudaGetDevice(&dev));
    CUDA_THROW(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // A(m, k): K-major [M x K] or MN-major [K x M]; B(n, k): [N x K] or [K x N]
    const long ar = a_mn ? K : M, ac = a_mn ? M : K, br = b_mn ? K : N, bc = b_mn ? N : K;
    const long lda = pad32(ac), ldb = pad32(bc), ldo = pad32(N);
    std::vector<void*> owned;
    auto keep = [&](void* p) {
        owned.push_back(p);
        return p;
    };
    struct Free {
        std::vector<void*>& v;
        ~Free() {
            for (void* p : v) cudaFree(p);
        }
    } fr{owned};
    void* dA = keep(upload(a, ar, ac, lda, f32));
    void* dB = keep(upload(b, br, bc, ldb, f32));
    GemmEpi e;
    e.mode = mode;
    e.act = act;
    e.alpha = alpha;
    e.beta = beta;
    e.lower = lower;
    e.ksplit = ksplit > 0 ? ksplit : 1;
    unsigned* dflags = static_cast<unsigned*>(keep(upload(std::vector<float>(4, 0.f).data(), 1, 4, 4, true)));
    e.flag = dflags;
    e.flag_bit = 0;
    // fp32 in/out buffer of the read-modify-write / fp32-output modes
    const bool o32 = mode == EPI_FWD_LINEAR || mode == EPI_GRAD || mode == EPI_GRAD_SGD || mode == EPI_EMA ||
                     mode == EPI_SUB || mode == EPI_AXPY;
    float* d32 = nullptr;
    void* dT = nullptr;
    bf16* dsh = nullptr;
    float* dlr = nullptr;
    float* dbias = nullptr;
    const long nsplit_cap = e.ksplit;
    if (mode == EPI_PARTIAL) {
        d32 = static_cast<float*>(keep(upload(std::vector<float>(static_cast<size_t>(M) * N * nsplit_cap, 0.f).data(),
                                              M * nsplit_cap, N, ldo, true)));
        e.out32 = d32;
        e.ld_out32 = ldo;
        e.split_stride = M * ldo;
    } else if (o32) {
        d32 = static_cast<float*>(keep(upload(out, M, N, ldo, true)));
        e.out32 = d32;
        e.ld_out32 = ldo;
    } else {
        dT = keep(upload(std::vector<float>(static_cast<size_t>(M) * N, 0.f).data(), M, N, ldo, f32));
        e.out = dT;
        e.ld_out = ldo;
    }
    if (mode == EPI_FWD_ACT || mode == EPI_FWD_LINEAR) {
        dbias = static_cast<float*>(keep(upload(bias, 1, N, pad32(N), true)));
        e.bias = dbias;
    }
    if (mode == EPI_ACTGRAD || mode == EPI_RESID) {
        e.aux = keep(upload(aux, M, N, ldo, f32));
        e.ld_aux = ldo;
    }
    double* dpart = nullptr;
    if (mode == EPI_RESID) {
        const long cap = 2 * 16384;  // floats: room for 16384 CTAs' {sum aux^2, sum out^2}
        dpart = static_cast<double*>(keep(upload(std::vector<float>(cap, 0.f).data(), 1, cap, cap, true)));
        e.part = dpart;
    }
    if (mode == EPI_GRAD_SGD || mode == EPI_AXPY) {
        if (!f32) {
            dsh = static_cast<bf16*>(keep(upload(std::vector<float>(static_cast<size_t>(M) * N, 0.f).data(), M, N,
                                                 ldo, false)));
            e.shadow = dsh;
            e.ld_shadow = ldo;
        }
        if (mode == EPI_GRAD_SGD) {
            dlr = static_cast<float*>(keep(upload(&lr, 1, 1, 4, true)));
            e.lr = dlr;
            e.step = nullptr;
            if (bias_col >= 0) {
                e.bias_col = bias_col;
                e.bias32 = static_cast<float*>(keep(upload(bias, 1, M, pad32(M), true)));
            }
        }
    }
    GemmPlan p;
    gemm_plan(p, prec, a_mn, dA, lda, b_mn, dB, ldb, M, N, K, e, sms, force_bn, force_mc);
    gemm_launch(p, 0);
    CUDA_THROW(cudaDeviceSynchronize());
    // outputs
    if (mode == EPI_PARTIAL) {
        std::vector<float> t(static_cast<size_t>(M) * N);
        std::fill(out, out + static_cast<size_t>(M) * N, 0.f);
        std::vector<double> acc(static_cast<size_t>(M) * N, 0.0);
        for (int ks = 0; ks < p.ep.ksplit; ++ks) {
            download(t.data(), d32 + static_cast<long>(ks) * M * ldo, M, N, ldo, true);
            for (size_t i = 0; i < t.size(); ++i) acc[i] += t[i];
        }
        for (size_t i = 0; i < t.size(); ++i) out[i] = static_cast<float>(acc[i]);
    } else if (o32) {
        download(out, d32, M, N, ldo, true);
    } else {
        download(out, dT, M, N, ldo, f32);
    }
    // out2: the updated bias (bias-column mode, M values) or else the bf16 operand copy (M x N)
    if (out2 && e.bias32)
        CUDA_THROW(cudaMemcpy(out2, e.bias32, M * 4, cudaMemcpyDeviceToHost));
    else if (out2 && dsh)
        download(out2, dsh, M, N, ldo, false);
    if (sums && dpart) {
        std::vector<double> pt(2 * static_cast<size_t>(gemm_launch_grid(p).x));
        CUDA_THROW(cudaMemcpy(pt.data(), dpart, pt.size() * 8, cudaMemcpyDeviceToHost));
        sums[0] = sums[1] = 0.0;
        for (size_t i = 0; i < pt.size(); i += 2) {
            sums[0] += pt[i];
            sums[1] += pt[i + 1];
        }
    }
    unsigned fl[4];
    CUDA_THROW(cudaMemcpy(fl, dflags, sizeof(fl), cudaMemcpyDeviceToHost));
    if (info) {
        info[0] = p.mc;
        info[1] = p.bn;
        info[2] = p.ep.ksplit;
        info[3] = static_cast<int>(fl[0]);
        info[4] = static_cast<int>(gemm_launch_grid(p).x);
        info[5] = p.threads;
    }
}

}  // namespace pnb
