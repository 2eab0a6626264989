// RBM CD-1 on device (pretrain.cpp:9-207).
//
// One update = 4 tcgen05 GEMMs + 3 small kernels:
//   pos   = sigmoid(X W^T + hb)                      -> PN[0:b)   (hidden_probs)
//   hs    = Bernoulli(pos)                           -> HS        (sample_bernoulli)
//   recon = hs W + vb  (sigmoid for bernoulli)       -> XR[b:2b)  (reconstruct_mean)
//   -neg  = -sigmoid(recon W^T + hb)                 -> PN[b:2b)
//   W    += lr/b * [pos; -neg]^T [X; recon]          one GEMM with K = 2b (cd1_apply)
//   hb   += lr/b * colsum(PN),  vb += lr/b * colsum(X - recon)
// Bernoulli draws: counter-based Philox4x32-10 keyed by (seed, element
// counter) in row-major draw order, or threshold_half, or injected uniforms
// (parity modes, pretrain.cpp:63-77).
#include <algorithm>
#include <cstring>

#include "host.h"
#include "rbm.h"

namespace pnb {

namespace {

template <typename T>
T* dalloc(size_t n) {
    void* p = nullptr;
    CUDA_THROW(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    CUDA_THROW(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T)));
    return static_cast<T*>(p);
}

__device__ __forceinline__ uint32_t mulhilo(uint32_t a, uint32_t b, uint32_t& hi) {
    const uint64_t p = static_cast<uint64_t>(a) * b;
    hi = static_cast<uint32_t>(p >> 32);
    return static_cast<uint32_t>(p);
}

// Philox4x32-10 (Salmon et al. 2011), first output word -> uniform in [0,1).
__device__ __forceinline__ float philox_uniform(uint64_t key, uint64_t ctr) {
    uint32_t c0 = static_cast<uint32_t>(ctr), c1 = static_cast<uint32_t>(ctr >> 32), c2 = 0x5EED, c3 = 0xC0FFEE;
    uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0, hi1;
        const uint32_t lo0 = mulhilo(0xD2511F53u, c0, hi0);
        const uint32_t lo1 = mulhilo(0xCD9E8D57u, c2, hi1);
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return static_cast<float>(c0 >> 8) * (1.0f / 16777216.0f);
}

template <typename T>
__device__ __forceinline__ float tf(T v) {
    return static_cast<float>(v);
}
template <>
__device__ __forceinline__ float tf<bf16>(bf16 v) {
    return __bfloat162float(v);
}

template <typename T>
__global__ void sample_kernel(const T* __restrict__ pos, long ldp, long b, long h, T* __restrict__ hs, long ldh,
                              int mode, uint64_t key, uint64_t counter, const double* __restrict__ u) {
    const long total = b * h;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const long r = i / h, c = i % h;
        const float p = tf<T>(pos[r * ldp + c]);
        bool on;
        if (mode == 1) on = p > 0.5f;
        else if (mode == 2) on = u[i] < static_cast<double>(p);
        else on = philox_uniform(key, counter + static_cast<uint64_t>(i)) < p;
        hs[r * ldh + c] = static_cast<T>(on ? 1.f : 0.f);
    }
}

// Bias updates of a CD-1 step (pretrain.cpp:106-119): hb += s * colsum(PN) over
// the 2b stacked rows [pos_h; -neg_h], vb += s * colsum(v - recon). A block is
// 32 columns x 16 row groups: each thread sums every 16th row of its column
// (independent loads in flight), then the 16 partials are added in a fixed order
// (deterministic). One thread per column summing all rows serially was
// latency-bound (80 us of a 2048 x 2048, b = 128 step).
template <typename T>
__global__ void __launch_bounds__(512) bias_update_kernel(const T* __restrict__ pn, long ldh, long b, long h,
                                                          float* __restrict__ hb, const T* __restrict__ xr, long ldv,
                                                          long v, float* __restrict__ vb, float s) {
    __shared__ float red[2][16][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const long j = blockIdx.x * 32L + tx;
    float ah = 0.f, av = 0.f;
    if (j < h) {
#pragma unroll 4
        for (long i = ty; i < 2 * b; i += 16) ah += tf<T>(pn[i * ldh + j]);
    }
    if (j < v) {
#pragma unroll 4
        for (long i = ty; i < b; i += 16) av += tf<T>(xr[i * ldv + j]) - tf<T>(xr[(b + i) * ldv + j]);
    }
    red[0][ty][tx] = ah;
    red[1][ty][tx] = av;
    __syncthreads();
    if (ty < 2) {  // ty 0: hidden bias, ty 1: visible bias
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += red[ty][k][tx];
        if (ty == 0 && j < h) hb[j] += s * acc;
        if (ty == 1 && j < v) vb[j] += s * acc;
    }
}

template <typename T>
__global__ void load_rows_kernel(const float* __restrict__ src, long lds, const uint32_t* __restrict__ rows, long b,
                                 long d, T* __restrict__ dst, long ldd) {
    const long total = b * ldd;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const long r = i / ldd, c = i % ldd;
        const long sr = rows ? rows[r] : r;
        dst[i] = static_cast<T>(c < d ? src[sr * lds + c] : 0.f);
    }
}

template <typename T>
__global__ void store_rows_kernel(const T* __restrict__ src, long lds, long b, long d, float* __restrict__ dst,
                                  long ldd) {
    const long total = b * ldd;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const long r = i / ldd, c = i % ldd;
        dst[i] = c < d ? tf<T>(src[r * lds + c]) : 0.f;
    }
}

template <typename T>
__global__ void sqerr_kernel(const T* __restrict__ xr, long ldv, long B, long b, long v, double* out) {
    __shared__ double sh[256];
    double acc = 0.0;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < b * v; i += (long)gridDim.x * blockDim.x) {
        const long r = i / v, c = i % v;
        const double d = static_cast<double>(tf<T>(xr[r * ldv + c])) - tf<T>(xr[(B + r) * ldv + c]);
        acc += d * d;
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] += sh[0];
}

template <typename T>
__global__ void copy_rows_kernel(const T* __restrict__ src, long lds, long b, long d, T* __restrict__ dst, long ldd) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < b * d; i += (long)gridDim.x * blockDim.x)
        dst[(i / d) * ldd + (i % d)] = src[(i / d) * lds + (i % d)];
}

int grid_of(long total) { return (int)std::max<long>(1, std::min<long>((total + 255) / 256, 148L * 8)); }

}  // namespace

RbmDevice::RbmDevice(Context* c, long visible, long hidden, bool g, long batch, Precision p)
    : ctx(c), v(visible), h(hidden), B(batch), gaussian(g), prec(p), ldv(pad32(visible)), ldh(pad32(hidden)) {
    if (v <= 0 || h <= 0)
        throw std::runtime_error("rbm_init: zero dimension (visible " + std::to_string(v) + ", hidden " +
                                 std::to_string(h) + ")");
    if (B <= 0) throw std::runtime_error("cd1_gibbs: empty batch");
    CUDA_THROW(cudaSetDevice(c->device));
    CUDA_THROW(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    const size_t es = f32() ? 4 : 2;
    W = dalloc<float>(h * ldv);
    if (!f32()) Ws = dalloc<bf16>(h * ldv);
    vb = dalloc<float>(ldv);
    hb = dalloc<float>(ldh);
    CUDA_THROW(cudaMalloc(&XR, 2 * B * ldv * es));
    CUDA_THROW(cudaMemset(XR, 0, 2 * B * ldv * es));
    CUDA_THROW(cudaMalloc(&PN, 2 * B * ldh * es));
    CUDA_THROW(cudaMemset(PN, 0, 2 * B * ldh * es));
    CUDA_THROW(cudaMalloc(&HS, B * ldh * es));
    CUDA_THROW(cudaMemset(HS, 0, B * ldh * es));
    u_dev = dalloc<double>(B * h);
    red = dalloc<double>(1024);
}

RbmDevice::~RbmDevice() {
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : {(void*)W, (void*)Ws, (void*)vb, (void*)hb, XR, PN, HS, (void*)u_dev, (void*)red})
        if (p) cudaFree(p);
    if (stream) cudaStreamDestroy(stream);
}

void RbmDevice::set_params(const double* p) {
    std::vector<float> w(h * ldv, 0.f), b1(ldv, 0.f), b2(ldh, 0.f);
    for (long r = 0; r < h; ++r)
        for (long c = 0; c < v; ++c) w[r * ldv + c] = static_cast<float>(p[r * v + c]);
    for (long j = 0; j < v; ++j) b1[j] = static_cast<float>(p[h * v + j]);
    for (long j = 0; j < h; ++j) b2[j] = static_cast<float>(p[h * v + v + j]);
    CUDA_THROW(cudaMemcpy(W, w.data(), w.size() * 4, cudaMemcpyHostToDevice));
    CUDA_THROW(cudaMemcpy(vb, b1.data(), b1.size() * 4, cudaMemcpyHostToDevice));
    CUDA_THROW(cudaMemcpy(hb, b2.data(), b2.size() * 4, cudaMemcpyHostToDevice));
    if (Ws) launch_f32_to_bf16_rows(W, ldv, h, v, Ws, stream);
    CUDA_THROW(cudaStreamSynchronize(stream));
}

void RbmDevice::get_params(double* p) {
    CUDA_THROW(cudaStreamSynchronize(stream));
    std::vector<float> w(h * ldv), b1(ldv), b2(ldh);
    CUDA_THROW(cudaMemcpy(w.data(), W, w.size() * 4, cudaMemcpyDeviceToHost));
    CUDA_THROW(cudaMemcpy(b1.data(), vb, b1.size() * 4, cudaMemcpyDeviceToHost));
    CUDA_THROW(cudaMemcpy(b2.data(), hb, b2.size() * 4, cudaMemcpyDeviceToHost));
    for (long r = 0; r < h; ++r)
        for (long c = 0; c < v; ++c) p[r * v + c] = w[r * ldv + c];
    for (long j = 0; j < v; ++j) p[h * v + j] = b1[j];
    for (long j = 0; j < h; ++j) p[h * v + v + j] = b2[j];
}

void RbmDevice::plan(long b) {
    if (b == planned_b) return;
    if (b > B) throw std::runtime_error("cd1_gibbs: batch larger than the RBM's buffers");
    const bool F = f32();
    const size_t es = F ? 4 : 2;
    const void* Wop = F ? static_cast<const void*>(W) : static_cast<const void*>(Ws);
    char* xr = static_cast<char*>(XR);
    char* pn = static_cast<char*>(PN);
    const int sms = ctx->num_sms;
    GemmEpi e;
    e.mode = EPI_FWD_ACT;
    e.act = 0;
    e.bias = hb;
    e.out = pn;
    e.ld_out = ldh;
    gemm_plan(g_pos, prec, false, xr, ldv, false, Wop, ldv, (int)b, (int)h, (int)v, e, sms);
    GemmEpi r;
    r.mode = EPI_FWD_ACT;
    r.act = gaussian ? 2 : 0;  // reconstruct_mean: linear for gaussian visibles
    r.bias = vb;
    r.out = xr + b * ldv * es;
    r.ld_out = ldv;
    gemm_plan(g_recon, prec, false, HS, ldh, true, Wop, ldv, (int)b, (int)v, (int)h, r, sms);
    GemmEpi n = e;
    n.out_scale = -1.f;
    n.out = pn + b * ldh * es;
    gemm_plan(g_neg, prec, false, xr + b * ldv * es, ldv, false, Wop, ldv, (int)b, (int)h, (int)v, n, sms);
    GemmEpi u;
    u.mode = EPI_AXPY;
    u.out32 = W;
    u.ld_out32 = ldv;
    u.shadow = Ws;
    u.ld_shadow = ldv;
    gemm_plan(g_upd, prec, true, pn, ldh, true, xr, ldv, (int)h, (int)v, (int)(2 * b), u, sms);
    planned_b = b;
}

void RbmDevice::cd1(long b, double lr, int sampling, uint64_t seed, uint64_t counter) {
    plan(b);
    cudaStream_t s = stream;
    const bool F = f32();
    gemm_launch(g_pos, s);
    if (F)
        sample_kernel<float><<<grid_of(b * h), 256, 0, s>>>(static_cast<float*>(PN), ldh, b, h, static_cast<float*>(HS),
                                                            ldh, sampling, seed, counter, u_dev);
    else
        sample_kernel<bf16><<<grid_of(b * h), 256, 0, s>>>(static_cast<bf16*>(PN), ldh, b, h, static_cast<bf16*>(HS),
                                                           ldh, sampling, seed, counter, u_dev);
    gemm_launch(g_recon, s);
    gemm_launch(g_neg, s);
    const float scale = static_cast<float>(lr / static_cast<double>(b));
    g_upd.ep.alpha = scale;
    gemm_launch(g_upd, s);
    const long wmax = std::max(v, h);
    const dim3 bgrid(static_cast<unsigned>((wmax + 31) / 32)), bblock(32, 16);
    if (F)
        bias_update_kernel<float><<<bgrid, bblock, 0, s>>>(static_cast<float*>(PN), ldh, b, h, hb,
                                                           static_cast<float*>(XR), ldv, v, vb, scale);
    else
        bias_update_kernel<bf16><<<bgrid, bblock, 0, s>>>(static_cast<bf16*>(PN), ldh, b, h, hb,
                                                          static_cast<bf16*>(XR), ldv, v, vb, scale);
    CUDA_THROW(cudaGetLastError());
}

namespace {
void upload_rows(RbmDevice& r, const double* x, long b, long d, long ld, void* dst) {
    std::vector<float> hbuf(b * ld, 0.f);
    for (long i = 0; i < b; ++i)
        for (long j = 0; j < d; ++j) hbuf[i * ld + j] = static_cast<float>(x[i * d + j]);
    float* tmp = nullptr;
    CUDA_THROW(cudaMalloc(&tmp, hbuf.size() * 4));
    CUDA_THROW(cudaMemcpyAsync(tmp, hbuf.data(), hbuf.size() * 4, cudaMemcpyHostToDevice, r.stream));
    if (r.f32())
        load_rows_kernel<float><<<grid_of(b * ld), 256, 0, r.stream>>>(tmp, ld, nullptr, b, d, static_cast<float*>(dst), ld);
    else
        load_rows_kernel<bf16><<<grid_of(b * ld), 256, 0, r.stream>>>(tmp, ld, nullptr, b, d, static_cast<bf16*>(dst), ld);
    CUDA_THROW(cudaStreamSynchronize(r.stream));
    cudaFree(tmp);
}
}  // namespace

void RbmDevice::cd1_host(const double* batch, long b, double lr, int sampling, uint64_t seed, uint64_t counter,
                         const double* u) {
    if (b <= 0) throw std::runtime_error("cd1_gibbs: empty batch");
    upload_rows(*this, batch, b, v, ldv, XR);
    if (sampling == 2) {
        if (!u) throw std::runtime_error("cd1: injected-uniform mode needs uniforms");
        CUDA_THROW(cudaMemcpyAsync(u_dev, u, b * h * 8, cudaMemcpyHostToDevice, stream));
    }
    cd1(b, lr, sampling, seed, counter);
    CUDA_THROW(cudaStreamSynchronize(stream));
}

void RbmDevice::hidden_probs_host(const double* x, long n, double* out) {
    const size_t es = f32() ? 4 : 2;
    std::vector<float> tmp(B * ldh);
    float* d32 = nullptr;
    CUDA_THROW(cudaMalloc(&d32, B * ldh * 4));
    for (long c0 = 0; c0 < n; c0 += B) {
        const long cb = std::min(B, n - c0);
        upload_rows(*this, x + c0 * v, cb, v, ldv, XR);
        plan(B);
        gemm_launch(g_pos, stream);
        if (f32())
            store_rows_kernel<float><<<grid_of(cb * ldh), 256, 0, stream>>>(static_cast<float*>(PN), ldh, cb, h, d32, ldh);
        else
            store_rows_kernel<bf16><<<grid_of(cb * ldh), 256, 0, stream>>>(static_cast<bf16*>(PN), ldh, cb, h, d32, ldh);
        CUDA_THROW(cudaMemcpyAsync(tmp.data(), d32, cb * ldh * 4, cudaMemcpyDeviceToHost, stream));
        CUDA_THROW(cudaStreamSynchronize(stream));
        for (long i = 0; i < cb; ++i)
            for (long j = 0; j < h; ++j) out[(c0 + i) * h + j] = tmp[i * ldh + j];
    }
    (void)es;
    cudaFree(d32);
}

double RbmDevice::reconstruction_error_host(const double* x, long n) {
    if (n <= 0) throw std::runtime_error("reconstruction_error: empty batch");
    CUDA_THROW(cudaMemsetAsync(red, 0, 8 * 64, stream));
    plan(B);
    for (long c0 = 0; c0 < n; c0 += B) {
        const long cb = std::min(B, n - c0);
        upload_rows(*this, x + c0 * v, cb, v, ldv, XR);
        gemm_launch(g_pos, stream);
        if (f32()) {
            copy_rows_kernel<float><<<grid_of(cb * h), 256, 0, stream>>>(static_cast<float*>(PN), ldh, cb, h,
                                                                         static_cast<float*>(HS), ldh);
            gemm_launch(g_recon, stream);
            sqerr_kernel<float><<<64, 256, 0, stream>>>(static_cast<float*>(XR), ldv, B, cb, v, red);
        } else {
            copy_rows_kernel<bf16><<<grid_of(cb * h), 256, 0, stream>>>(static_cast<bf16*>(PN), ldh, cb, h,
                                                                        static_cast<bf16*>(HS), ldh);
            gemm_launch(g_recon, stream);
            sqerr_kernel<bf16><<<64, 256, 0, stream>>>(static_cast<bf16*>(XR), ldv, B, cb, v, red);
        }
    }
    double parts[64];
    CUDA_THROW(cudaMemcpyAsync(parts, red, sizeof(parts), cudaMemcpyDeviceToHost, stream));
    CUDA_THROW(cudaStreamSynchronize(stream));
    double acc = 0.0;
    for (double p : parts) acc += p;
    return acc / static_cast<double>(n * v);
}

// greedy_pretrain (pretrain.cpp:162-207). The host Rng drives rbm_init, the
// per-epoch shuffles and the output-layer init in the reference's exact order;
// the b*h Bernoulli draws the reference takes from that same stream per batch
// are skipped with an xoshiro256** GF(2) jump, while the device draws its own
// counter-based Philox uniforms.
void greedy_pretrain(Context* ctx, const std::vector<long>& dims, const double* data, long n, uint64_t epochs,
                     double lr_g, double lr_b, long batch, host::Rng& rng, uint64_t philox_seed, Precision prec,
                     double* out) {
    if (dims.size() < 2) throw std::runtime_error("greedy_pretrain: need at least 2 dims");
    if (batch <= 0) throw std::runtime_error("greedy_pretrain: batch size must be >= 1");
    if (n <= 0) throw std::runtime_error("cd1_gibbs: empty batch");
    const long bs = std::min(batch, n);
    long d0 = dims[0], ld0 = pad32(d0);
    float* X = nullptr;
    {
        std::vector<float> hx(n * ld0, 0.f);
        for (long i = 0; i < n; ++i)
            for (long j = 0; j < d0; ++j) hx[i * ld0 + j] = static_cast<float>(data[i * d0 + j]);
        CUDA_THROW(cudaMalloc(&X, hx.size() * 4));
        CUDA_THROW(cudaMemcpy(X, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice));
    }
    uint32_t* d_idx = nullptr;
    CUDA_THROW(cudaMalloc(&d_idx, n * 4));
    long pos = 0;
    uint64_t counter = 0;
    const size_t L = dims.size() - 1;
    for (size_t l = 0; l + 1 < L; ++l) {
        const long v = dims[l], h = dims[l + 1];
        const bool gauss = l == 0;
        const double lr = gauss ? lr_g : lr_b;
        RbmDevice rbm(ctx, v, h, gauss, bs, prec);
        std::vector<double> p(h * v + v + h, 0.0);
        for (long i = 0; i < h * v; ++i) p[i] = rng.gaussian(0.0, 0.01);  // rbm_init (pretrain.cpp:9-21)
        rbm.set_params(p.data());
        const host::Jump skip = host::make_jump(static_cast<uint64_t>(bs) * static_cast<uint64_t>(h));
        const long ldx = pad32(v);
        std::vector<uint32_t> idx(n);
        for (uint64_t ep = 0; ep < epochs; ++ep) {
            std::vector<uint64_t> order(n);
            for (long i = 0; i < n; ++i) order[i] = static_cast<uint64_t>(i);
            rng.shuffle(order);  // feature_batches (pretrain.cpp:141-158)
            for (long i = 0; i < n; ++i) idx[i] = static_cast<uint32_t>(order[i]);
            CUDA_THROW(cudaMemcpyAsync(d_idx, idx.data(), n * 4, cudaMemcpyHostToDevice, rbm.stream));
            for (long b = 0; b < n / bs; ++b) {
                if (rbm.f32())
                    load_rows_kernel<float><<<grid_of(bs * ldx), 256, 0, rbm.stream>>>(
                        X, ldx, d_idx + b * bs, bs, v, static_cast<float*>(rbm.XR), ldx);
                else
                    load_rows_kernel<bf16><<<grid_of(bs * ldx), 256, 0, rbm.stream>>>(
                        X, ldx, d_idx + b * bs, bs, v, static_cast<bf16*>(rbm.XR), ldx);
                rbm.cd1(bs, lr, 0, philox_seed, counter);
                counter += static_cast<uint64_t>(bs) * static_cast<uint64_t>(h);
                rng.jump(skip);
            }
        }
        // next layer input: hidden probabilities over the whole data (pretrain.cpp:190)
        const long ldh = pad32(h);
        float* Xn = nullptr;
        CUDA_THROW(cudaMalloc(&Xn, n * ldh * 4));
        rbm.plan(bs);
        for (long c0 = 0; c0 < n; c0 += bs) {
            const long cb = std::min(bs, n - c0);
            if (rbm.f32())
                load_rows_kernel<float><<<grid_of(cb * ldx), 256, 0, rbm.stream>>>(X + c0 * ldx, ldx, nullptr, cb, v,
                                                                                static_cast<float*>(rbm.XR), ldx);
            else
                load_rows_kernel<bf16><<<grid_of(cb * ldx), 256, 0, rbm.stream>>>(X + c0 * ldx, ldx, nullptr, cb, v,
                                                                               static_cast<bf16*>(rbm.XR), ldx);
            gemm_launch(rbm.g_pos, rbm.stream);
            if (rbm.f32())
                store_rows_kernel<float><<<grid_of(cb * ldh), 256, 0, rbm.stream>>>(static_cast<float*>(rbm.PN), ldh, cb,
                                                                                 h, Xn + c0 * ldh, ldh);
            else
                store_rows_kernel<bf16><<<grid_of(cb * ldh), 256, 0, rbm.stream>>>(static_cast<bf16*>(rbm.PN), ldh, cb, h,
                                                                                Xn + c0 * ldh, ldh);
        }
        CUDA_THROW(cudaStreamSynchronize(rbm.stream));
        cudaFree(X);
        X = Xn;
        rbm.get_params(p.data());
        for (long i = 0; i < h * v; ++i) out[pos++] = p[i];                 // weights
        for (long j = 0; j < h; ++j) out[pos++] = p[h * v + v + j];         // h_bias
    }
    const long di = dims[L - 1], dout = dims[L];
    const double r = std::sqrt(6.0 / static_cast<double>(di + dout));
    for (long i = 0; i < di * dout; ++i) out[pos++] = rng.uniform(-r, r);
    for (long j = 0; j < dout; ++j) out[pos++] = 0.0;
    cudaFree(X);
    cudaFree(d_idx);
}

}  // namespace pnb
