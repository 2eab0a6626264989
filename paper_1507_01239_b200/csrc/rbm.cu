// RBM CD-1 on device (pretrain.cpp:9-207).
//
// One update = 4 tcgen05 GEMMs + 4 small kernels. The three M = b GEMMs run
// split-K (EPI_PARTIAL) and each is followed by one reduction kernel that sums
// the splits and applies the elementwise step:
//   pos   = sigmoid(X W^T + hb)                      -> PN[0:b)   (hidden_probs)
//   hs    = Bernoulli(pos)    (same kernel)          -> HS        (sample_bernoulli)
//   recon = hs W + vb  (sigmoid for bernoulli)       -> XR[b:2b)  (reconstruct_mean)
//   -neg  = -sigmoid(recon W^T + hb)                 -> PN[b:2b)
//   W    += lr/b * [pos; -neg]^T [X; recon]          one GEMM with K = 2b (cd1_apply)
//   hb   += lr/b * colsum(PN),  vb += lr/b * colsum(X - recon)  (column sums
//           taken by the reductions, folded by bias_finish_kernel)
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
    zero(p, std::max<size_t>(n, 1) * sizeof(T));
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

// Split-K reductions with the CD-1 epilogues fused (pretrain.cpp:37-121). The
// three M = b GEMMs of a step (b = 128 rows against a 2048-wide layer) have 8-16
// output tiles: each runs split-K over ~128 CTAs writing fp32 partial tiles
// (EPI_PARTIAL), and one of these kernels sums the splits and applies the
// step's elementwise work. Block = 32 columns x 8 row groups over one chunk of
// rows; its column sums go to colpart[chunk][col] (fixed order, deterministic)
// and bias_finish_kernel folds them into the biases once all chunks are done.
struct PartIn {
    const float* p;  // split ks at p + ks * stride, element (r, c) at r * ld + c
    long stride, ld;
    int ks;
};

// the splits are summed in split order; the loads are read-only (nc) so the
// unrolled batch of them is in flight together
__device__ __forceinline__ float part_sum(const PartIn& in, long r, long c) {
    const float* q = in.p + r * in.ld + c;
    float a = __ldg(q);
#pragma unroll 8
    for (int k = 1; k < in.ks; ++k) a += __ldg(q + k * in.stride);
    return a;
}

__device__ __forceinline__ float sigmoid_exact(float z) { return 1.f / (1.f + expf(-z)); }
__device__ __forceinline__ double sigmoid_d(float z) { return 1.0 / (1.0 + exp(-static_cast<double>(z))); }

struct Chunk {
    long r0, r1;  // rows of this block
    long j;       // column
};

__device__ __forceinline__ Chunk chunk_of(long b, long n) {
    const long per = 8;  // one row per thread (grid.y = ceil(b / 8))
    Chunk c;
    c.r0 = blockIdx.y * per;
    c.r1 = min(b, c.r0 + per);
    c.j = blockIdx.x * 32L + threadIdx.x;
    return c;
}

// column sum over the block's 8 row groups -> colpart[blockIdx.y][j]
__device__ __forceinline__ void block_colsum(double acc, long j, long n, double* colpart, long ldc) {
    __shared__ double red[8][33];
    red[threadIdx.y][threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.y == 0 && j < n) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) s += red[k][threadIdx.x];
        colpart[blockIdx.y * ldc + j] = s;
    }
}

// pos = sigmoid(sum + hb) -> PN rows [0, b) (and fp32 rows of out32 when given);
// hs = Bernoulli(pos) -> HS: mode 0 Philox keyed by (key, counter + r*h + c)
// (the reference's row-major draw order), 1 threshold_half, 2 injected
// uniforms, 3 hs = pos (mean-field pass of reconstruction_error), 4 no hs
// (hidden_probs).
template <typename T>
__global__ void __launch_bounds__(256) cd1_pos_kernel(PartIn in, long b, long h, const float* __restrict__ hb,
                                                      T* __restrict__ pn, long ldh, T* __restrict__ hs, int mode,
                                                      uint64_t key, uint64_t counter, const double* __restrict__ u,
                                                      float* __restrict__ zp, float* __restrict__ out32, long ld32,
                                                      const uint64_t* __restrict__ dctr, long koff) {
    grid_dep_wait();
    // graph-launched steps: counter = epoch base + step * b * h, step = graph base + koff
    // (dctr = {graph base step, counter base})
    if (dctr) counter = dctr[1] + (dctr[0] + koff) * static_cast<uint64_t>(b) * static_cast<uint64_t>(h);
    const Chunk c = chunk_of(b, h);
    if (c.j < h) {
        const float bias = hb[c.j];
        for (long r = c.r0 + threadIdx.y; r < c.r1; r += 8) {
            const float z = part_sum(in, r, c.j) + bias;
            if (zp) zp[r * ldh + c.j] = z;
            const T pv = static_cast<T>(sigmoid_exact(z));
            const float p = tf<T>(pv);
            pn[r * ldh + c.j] = pv;
            if (out32) out32[r * ld32 + c.j] = p;
            if (!hs) continue;
            const long i = r * h + c.j;
            float s;
            if (mode == 3) s = p;
            else if (mode == 1) s = p > 0.5f ? 1.f : 0.f;
            else if (mode == 2) s = u[i] < static_cast<double>(p) ? 1.f : 0.f;
            else s = philox_uniform(key, counter + static_cast<uint64_t>(i)) < p ? 1.f : 0.f;
            hs[r * ldh + c.j] = static_cast<T>(s);
        }
    }
}

// recon = act(sum + vb) -> xr rows [b, 2b) (act: sigmoid, or identity for
// Gaussian visibles); colpart <- column sums of (v - recon) over the block's rows.
template <typename T>
__global__ void __launch_bounds__(256) cd1_recon_kernel(PartIn in, long b, long v, const float* __restrict__ vb,
                                                        bool gaussian, T* __restrict__ xr, long ldv, T* __restrict__ rec,
                                                        double* __restrict__ colpart) {
    grid_dep_wait();
    const Chunk c = chunk_of(b, v);
    double acc = 0.0;
    if (c.j < v) {
        const float bias = vb[c.j];
        for (long r = c.r0 + threadIdx.y; r < c.r1; r += 8) {
            const float z = part_sum(in, r, c.j) + bias;
            const T x = static_cast<T>(gaussian ? z : sigmoid_exact(z));
            rec[r * ldv + c.j] = x;
            if (colpart) acc += static_cast<double>(tf<T>(xr[r * ldv + c.j])) - (gaussian ? z : sigmoid_d(z));
        }
    }
    grid_dep_launch();
    if (colpart) block_colsum(acc, c.j, v, colpart, ldv);
}

// -neg = -sigmoid(sum + hb) -> PN rows [b, 2b); colpart <- column sums of
// (pos - neg). pos and neg are close once the RBM reconstructs well, so their
// difference is taken in fp64 from the two pre-activations (zp: the pos pass's,
// kept by cd1_pos_kernel) rather than from the rounded probabilities.
template <typename T>
__global__ void __launch_bounds__(256) cd1_neg_kernel(PartIn in, long b, long h, const float* __restrict__ hb,
                                                      const float* __restrict__ zp, T* __restrict__ pn, long ldh,
                                                      double* __restrict__ colpart) {
    grid_dep_wait();
    const Chunk c = chunk_of(b, h);
    double acc = 0.0;
    if (c.j < h) {
        const float bias = hb[c.j];
        for (long r = c.r0 + threadIdx.y; r < c.r1; r += 8) {
            const float z = part_sum(in, r, c.j) + bias;
            pn[(b + r) * ldh + c.j] = static_cast<T>(-sigmoid_exact(z));
            acc += sigmoid_d(zp[r * ldh + c.j]) - sigmoid_d(z);
        }
    }
    grid_dep_launch();
    block_colsum(acc, c.j, h, colpart, ldh);
}

// hb += s * sum (pos - neg), vb += s * sum (v - recon)   (pretrain.cpp:106-119)
__global__ void bias_finish_kernel(const double* __restrict__ cpn, int chunks_h, long h, long ldh,
                                   float* __restrict__ hb, const double* __restrict__ cvis, int chunks_v, long v,
                                   long ldv, float* __restrict__ vb, double s, uint64_t* __restrict__ dctr,
                                   long inc) {
    grid_dep_wait();
    const long j = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (dctr && inc && j == 0) dctr[0] += inc;  // the graph's last step: advance the graph base step
    if (j < h) {
        double a = 0.0;
        for (int k = 0; k < chunks_h; ++k) a += cpn[k * ldh + j];
        hb[j] = static_cast<float>(hb[j] + s * a);
    }
    if (j < v) {
        double a = 0.0;
        for (int k = 0; k < chunks_v; ++k) a += cvis[k * ldv + j];
        vb[j] = static_cast<float>(vb[j] + s * a);
    }
}

template <typename T>
__global__ void load_rows_kernel(const float* __restrict__ src, long lds, const uint32_t* __restrict__ rows, long b,
                                 long d, T* __restrict__ dst, long ldd, const uint64_t* __restrict__ dstep,
                                 long koff) {
    grid_dep_wait();
    if (dstep) rows += (dstep[0] + koff) * b;  // graph-launched steps: this step's slice of the shuffled order
    const long total = b * ldd;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const long r = i / ldd, c = i % ldd;
        const long sr = rows ? rows[r] : r;
        dst[i] = static_cast<T>(c < d ? src[sr * lds + c] : 0.f);
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

int grid_of(long total) { return (int)std::max<long>(1, std::min<long>((total + 255) / 256, 148L * 8)); }

}  // namespace

RbmDevice::RbmDevice(Context* c, long visible, long hidden, bool g, long batch, Precision p)
    : ctx(c), v(visible), h(hidden), B(batch), gaussian(g), prec(p), ldv(pad32(visible)), ldh(pad32(hidden)) {
    if (v <= 0 || h <= 0)
        throw std::runtime_error("rbm_init: zero dimension (visible " + std::to_string(v) + ", hidden " +
                                 std::to_string(h) + ")");
    if (B <= 0) throw std::runtime_error("cd1_gibbs: empty batch");
    CUDA_THROW(cudaSetDevice(c->device));
    stream = make_stream(0);  // the CD-1 chain; the graphs' side stream (batch gathers, bias updates) is low
    const size_t es = f32() ? 4 : 2;
    W = dalloc<float>(h * ldv);
    if (!f32()) Ws = dalloc<bf16>(h * ldv);
    vb = dalloc<float>(ldv);
    hb = dalloc<float>(ldh);
    CUDA_THROW(cudaMalloc(&XR, 2 * B * ldv * es));
    zero(XR, 2 * B * ldv * es);
    CUDA_THROW(cudaMalloc(&XRs[1], 2 * B * ldv * es));
    zero(XRs[1], 2 * B * ldv * es);
    XRs[0] = XR;
    CUDA_THROW(cudaMalloc(&PN, 2 * B * ldh * es));
    zero(PN, 2 * B * ldh * es);
    CUDA_THROW(cudaMalloc(&HS, B * ldh * es));
    zero(HS, B * ldh * es);
    u_dev = dalloc<double>(B * h);
    red = dalloc<double>(1024);
    const long chunks = (B + 7) / 8;
    colp = dalloc<double>(chunks * (ldh + ldv));
    ZP = dalloc<float>(B * ldh);
    dctr = dalloc<uint64_t>(2);
}

RbmDevice::~RbmDevice() {
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : {(void*)W, (void*)Ws, (void*)vb, (void*)hb, XRs[0], XRs[1], PN, HS, (void*)u_dev, (void*)red,
                    (void*)part, (void*)colp, (void*)ZP, (void*)dctr})
        if (p) cudaFree(p);
    if (stream) cudaStreamDestroy(stream);
}

void RbmDevice::set_params(const double* p) {
    std::vector<float> w(h * ldv, 0.f), b1(ldv, 0.f), b2(ldh, 0.f);
    for (long r = 0; r < h; ++r)
        for (long c = 0; c < v; ++c) w[r * ldv + c] = static_cast<float>(p[r * v + c]);
    for (long j = 0; j < v; ++j) b1[j] = static_cast<float>(p[h * v + j]);
    for (long j = 0; j < h; ++j) b2[j] = static_cast<float>(p[h * v + v + j]);
    upload(W, w.data(), w.size() * 4);
    upload(vb, b1.data(), b1.size() * 4);
    upload(hb, b2.data(), b2.size() * 4);
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

namespace {
// split-K factor of an M = b CD-1 GEMM: about one CTA per SM,
// at least two k-blocks per split (gemm_plan rounds it so no split is empty)
// Tile width of the M = b split-K GEMMs: 64 (twice the tiles, half the splits and
// half the partial bytes for the reductions: 53.7 vs 56.3 us per 2048 x 2048 bf16
// step) except in fp32 mode, where the 3xTF32 mainloop favours 128 (83 vs 89 us).
// PARNN_CD1_BN: tuning aid.
int cd1_bn(int prec) {
    static const int forced = [] {
        const char* v = std::getenv("PARNN_CD1_BN");
        const int x = v ? std::atoi(v) : 0;
        return (x == 64 || x == 128 || x == 256) ? x : 0;
    }();
    return forced ? forced : (prec == PREC_FP32 ? 128 : 64);
}

int cd1_ksplit(int prec, long M, long N, long K, int sms) {
    const long tiles = ((M + 127) / 128) * ((N + cd1_bn(prec) - 1) / cd1_bn(prec));
    const long nk = (K + (prec ? 31 : 63)) / (prec ? 32 : 64);
    return static_cast<int>(std::max<long>(1, std::min<long>(sms / tiles, nk / 2)));
}

int row_chunks(long b) { return static_cast<int>((b + 7) / 8); }  // grid.y of the reductions: a row per thread

// Launch with programmatic stream serialization: the kernel is scheduled while
// its predecessor drains and waits for it in griddepcontrol.wait (every kernel
// launched this way starts with grid_dep_wait()).
template <typename... KArgs, typename... Args>
void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CUDA_THROW(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...));
}

PartIn part_of(const GemmPlan& g) { return PartIn{g.ep.out32, g.ep.split_stride, g.ep.ld_out32, g.ep.ksplit}; }
}  // namespace

void RbmDevice::plan(long b) {
    if (b == planned_b) return;
    if (b > B) throw std::runtime_error("cd1_gibbs: batch larger than the RBM's buffers");
    const bool F = f32();
    const size_t es = F ? 4 : 2;
    const void* Wop = F ? static_cast<const void*>(W) : static_cast<const void*>(Ws);
    // one plan set per XR buffer (graph-launched epochs alternate them)
    for (int sl = 1; sl >= 0; --sl) {
        XR = XRs[sl];
        char* xr = static_cast<char*>(XR);
        char* pn = static_cast<char*>(PN);
        const int sms = ctx->num_sms;
        const int kp = cd1_ksplit(prec, b, h, v, sms), kr = cd1_ksplit(prec, b, v, h, sms);
        const size_t need = std::max(static_cast<size_t>(kp) * b * ldh, static_cast<size_t>(kr) * b * ldv);
        if (need > part_n) {
            if (part) CUDA_THROW(cudaFree(part));
            CUDA_THROW(cudaMalloc(&part, need * 4));
            part_n = need;
        }
        auto split = [&](GemmPlan& g, bool b_mn, const void* A, long lda, int N, int K, int ks, long ld) {
            GemmEpi e;
            e.mode = EPI_PARTIAL;
            e.out32 = part;
            e.ld_out32 = ld;
            e.split_stride = b * ld;
            e.ksplit = ks;
            gemm_plan(g, prec, false, A, lda, b_mn, Wop, ldv, static_cast<int>(b), N, K, e, sms, cd1_bn(prec));
        };
        split(g_pos, false, xr, ldv, static_cast<int>(h), static_cast<int>(v), kp, ldh);             // X W^T
        split(g_recon, true, HS, ldh, static_cast<int>(v), static_cast<int>(h), kr, ldv);            // hs W
        split(g_neg, false, xr + b * ldv * es, ldv, static_cast<int>(h), static_cast<int>(v), kp, ldh);  // recon W^T
        GemmEpi u;
        u.mode = EPI_AXPY;
        u.out32 = W;
        u.ld_out32 = ldv;
        u.shadow = Ws;
        u.ld_shadow = ldv;
        gemm_plan(g_upd, prec, true, pn, ldh, true, xr, ldv, (int)h, (int)v, (int)(2 * b), u, sms);
        slot_plans[sl][0] = g_pos;
        slot_plans[sl][1] = g_recon;
        slot_plans[sl][2] = g_neg;
        slot_plans[sl][3] = g_upd;
    }
    ch_h = ch_v = row_chunks(b);
    planned_b = b;
}

void RbmDevice::use_slot(int sl) {
    XR = XRs[sl];
    g_pos = slot_plans[sl][0];
    g_recon = slot_plans[sl][1];
    g_neg = slot_plans[sl][2];
    g_upd = slot_plans[sl][3];
}

namespace {
template <typename T>
void launch_pos(RbmDevice& r, long rows, int mode, uint64_t seed, uint64_t counter, float* out32, long ld32,
                const uint64_t* dctr = nullptr, long koff = 0) {
    const dim3 grid(static_cast<unsigned>((r.h + 31) / 32), r.ch_h), block(32, 8);
    launch_pdl(cd1_pos_kernel<T>, grid, block, r.stream, part_of(r.g_pos), rows, r.h, r.hb, static_cast<T*>(r.PN),
               r.ldh, mode == 4 ? nullptr : static_cast<T*>(r.HS), mode, seed, counter, r.u_dev,
               mode < 3 ? r.ZP : nullptr, out32, ld32, dctr, koff);
}

template <typename T>
void launch_recon(RbmDevice& r, long rows, double* colpart) {
    const dim3 grid(static_cast<unsigned>((r.v + 31) / 32), r.ch_v), block(32, 8);
    T* xr = static_cast<T*>(r.XR);
    launch_pdl(cd1_recon_kernel<T>, grid, block, r.stream, part_of(r.g_recon), rows, r.v, r.vb, r.gaussian, xr, r.ldv,
               xr + r.planned_b * r.ldv, colpart);
}

// one CD-1 update (pretrain.cpp:79-121): 3 split-K GEMMs each followed by its
// fused reduction, the rank-2b weight update, the bias update
template <typename T>
// dctr: graph-captured step koff of a graph reads its Philox counter from {graph
// base step, counter base}; the graph's last step advances the base by inc
void run_cd1(RbmDevice& r, long b, double lr, int sampling, uint64_t seed, uint64_t counter,
             uint64_t* dctr = nullptr, long koff = 0, long inc = 0) {
    cudaStream_t s = r.stream;
    double* cpn = r.colp;
    double* cvis = cpn + r.ch_h * r.ldh;
    gemm_launch(r.g_pos, s);
    if (r.bias_side && r.bias_pending) {
        // the previous step's bias update (side stream) lands before this step reads hb
        CUDA_THROW(cudaStreamWaitEvent(s, r.ev_bias, 0));
        r.bias_pending = false;
    }
    launch_pos<T>(r, b, sampling, seed, counter, nullptr, 0, dctr, koff);
    gemm_launch(r.g_recon, s);
    launch_recon<T>(r, b, cvis);
    gemm_launch(r.g_neg, s);
    const dim3 grid(static_cast<unsigned>((r.h + 31) / 32), r.ch_h), block(32, 8);
    launch_pdl(cd1_neg_kernel<T>, grid, block, s, part_of(r.g_neg), b, r.h, r.hb, r.ZP, static_cast<T*>(r.PN), r.ldh,
               cpn);
    const double scale = lr / static_cast<double>(b);
    const long wmax = std::max(r.v, r.h);
    const dim3 bgrid(static_cast<unsigned>((wmax + 255) / 256)), bblock(256);
    if (r.bias_side) {
        // graph-launched steps: the bias update runs beside the weight update
        CUDA_THROW(cudaEventRecord(r.ev_neg, s));
        CUDA_THROW(cudaStreamWaitEvent(r.bias_side, r.ev_neg, 0));
        launch_pdl(bias_finish_kernel, bgrid, bblock, r.bias_side, cpn, r.ch_h, r.h, r.ldh, r.hb, cvis, r.ch_v, r.v,
                   r.ldv, r.vb, scale, dctr, inc);
        CUDA_THROW(cudaEventRecord(r.ev_bias, r.bias_side));
        r.bias_pending = true;
    }
    r.g_upd.ep.alpha = static_cast<float>(scale);
    gemm_launch(r.g_upd, s);
    if (!r.bias_side)
        launch_pdl(bias_finish_kernel, bgrid, bblock, s, cpn, r.ch_h, r.h, r.ldh, r.hb, cvis, r.ch_v, r.v, r.ldv, r.vb,
                   scale, dctr, inc);
    CUDA_THROW(cudaGetLastError());
}
}  // namespace

void RbmDevice::cd1(long b, double lr, int sampling, uint64_t seed, uint64_t counter) {
    plan(b);
    if (f32()) run_cd1<float>(*this, b, lr, sampling, seed, counter);
    else run_cd1<bf16>(*this, b, lr, sampling, seed, counter);
}

void RbmDevice::hidden_probs_rows(long rows, float* out32, long ld32) {
    gemm_launch(g_pos, stream);
    if (f32()) launch_pos<float>(*this, rows, 4, 0, 0, out32, ld32);
    else launch_pos<bf16>(*this, rows, 4, 0, 0, out32, ld32);
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
        load_rows_kernel<float><<<grid_of(b * ld), 256, 0, r.stream>>>(tmp, ld, nullptr, b, d, static_cast<float*>(dst), ld,
                                                                        nullptr, 0);
    else
        load_rows_kernel<bf16><<<grid_of(b * ld), 256, 0, r.stream>>>(tmp, ld, nullptr, b, d, static_cast<bf16*>(dst), ld,
                                                                       nullptr, 0);
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
    std::vector<float> tmp(B * ldh);
    float* d32 = nullptr;
    CUDA_THROW(cudaMalloc(&d32, B * ldh * 4));
    plan(B);
    for (long c0 = 0; c0 < n; c0 += B) {
        const long cb = std::min(B, n - c0);
        upload_rows(*this, x + c0 * v, cb, v, ldv, XR);
        hidden_probs_rows(cb, d32, ldh);
        CUDA_THROW(cudaMemcpyAsync(tmp.data(), d32, cb * ldh * 4, cudaMemcpyDeviceToHost, stream));
        CUDA_THROW(cudaStreamSynchronize(stream));
        for (long i = 0; i < cb; ++i)
            for (long j = 0; j < h; ++j) out[(c0 + i) * h + j] = tmp[i * ldh + j];
    }
    cudaFree(d32);
}

// pretrain.cpp:127-136: mean-field pass (hs = pos), squared error of the
// reconstruction over the first cb rows
double RbmDevice::reconstruction_error_host(const double* x, long n) {
    if (n <= 0) throw std::runtime_error("reconstruction_error: empty batch");
    CUDA_THROW(cudaMemsetAsync(red, 0, 8 * 64, stream));
    plan(B);
    for (long c0 = 0; c0 < n; c0 += B) {
        const long cb = std::min(B, n - c0);
        upload_rows(*this, x + c0 * v, cb, v, ldv, XR);
        gemm_launch(g_pos, stream);
        if (f32()) {
            launch_pos<float>(*this, cb, 3, 0, 0, nullptr, 0);
            gemm_launch(g_recon, stream);
            launch_recon<float>(*this, cb, nullptr);
            sqerr_kernel<float><<<64, 256, 0, stream>>>(static_cast<float*>(XR), ldv, B, cb, v, red);
        } else {
            launch_pos<bf16>(*this, cb, 3, 0, 0, nullptr, 0);
            gemm_launch(g_recon, stream);
            launch_recon<bf16>(*this, cb, nullptr);
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
thread_local PretrainStats g_pretrain_stats;

void greedy_pretrain(Context* ctx, const std::vector<long>& dims, const double* data, long n, uint64_t epochs,
                     double lr_g, double lr_b, long batch, host::Rng& rng, uint64_t philox_seed, Precision prec,
                     double* out) {
    g_pretrain_stats = PretrainStats();
    if (dims.size() < 2) throw std::runtime_error("greedy_pretrain: need at least 2 dims");
    if (batch <= 0) throw std::runtime_error("greedy_pretrain: batch size must be >= 1");
    if (n <= 0) throw std::runtime_error("cd1_gibbs: empty batch");
    const long bs = std::min(batch, n);
    long d0 = dims[0], ld0 = pad32(d0);
    // device buffers, streams, events and graphs are released on every exit path
    struct Owned {
        std::vector<void*> mem;
        std::vector<cudaStream_t> streams;
        std::vector<cudaEvent_t> events;
        std::vector<cudaGraphExec_t> graphs;
        ~Owned() {
            for (auto g : graphs) cudaGraphExecDestroy(g);
            for (auto e : events) cudaEventDestroy(e);
            for (auto st : streams) cudaStreamDestroy(st);
            for (void* m : mem) cudaFree(m);
        }
    } own;
    float* X = nullptr;
    {
        std::vector<float> hx(n * ld0, 0.f);
        for (long i = 0; i < n; ++i)
            for (long j = 0; j < d0; ++j) hx[i * ld0 + j] = static_cast<float>(data[i * d0 + j]);
        CUDA_THROW(cudaMalloc(&X, hx.size() * 4));
        own.mem.push_back(X);
        upload(X, hx.data(), hx.size() * 4);
    }
    uint32_t* d_idx = nullptr;
    CUDA_THROW(cudaMalloc(&d_idx, n * 4));
    own.mem.push_back(d_idx);
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
        // The epoch's CD-1 steps run as CUDA graphs of kGraphSteps steps (and
        // single-step graphs for the remainder): launched one kernel at a time the
        // step is bound by host launch submission (~3.7 us per launch against
        // ~0.6 us per graph node). The steps read their slice of the shuffled
        // order and their Philox counter from rbm.dctr = {step, base}.
        rbm.plan(bs);
        const long steps = n / bs;
        constexpr long kGraphSteps = 32;
        // Two XR buffers: step k gathers its batch into buffer k % 2 on a side stream,
        // so the gather overlaps step k-1 (it waits only for step k-2, the last reader
        // of that buffer) and leaves the step's dependent chain.
        cudaStream_t side = make_stream(2);
        own.streams.push_back(side);
        cudaEvent_t ev_begin, ev_load[2], ev_done[2], ev_side;
        for (cudaEvent_t* e : {&ev_begin, &ev_load[0], &ev_load[1], &ev_done[0], &ev_done[1], &ev_side}) {
            CUDA_THROW(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
            own.events.push_back(*e);
        }
        CUDA_THROW(cudaEventCreateWithFlags(&rbm.ev_neg, cudaEventDisableTiming));
        own.events.push_back(rbm.ev_neg);
        CUDA_THROW(cudaEventCreateWithFlags(&rbm.ev_bias, cudaEventDisableTiming));
        own.events.push_back(rbm.ev_bias);
        auto capture = [&](long nsteps) {
            cudaGraph_t g = nullptr;
            cudaGraphExec_t ge = nullptr;
            rbm.bias_side = side;  // the bias updates run on the side stream too
            rbm.bias_pending = false;
            CUDA_THROW(cudaStreamBeginCapture(rbm.stream, cudaStreamCaptureModeThreadLocal));
            CUDA_THROW(cudaEventRecord(ev_begin, rbm.stream));
            CUDA_THROW(cudaStreamWaitEvent(side, ev_begin, 0));
            for (long k = 0; k < nsteps; ++k) {
                const int slot = static_cast<int>(k & 1);
                if (k >= 2) CUDA_THROW(cudaStreamWaitEvent(side, ev_done[slot], 0));  // step k-2 read this buffer
                const dim3 gr(static_cast<unsigned>(grid_of(bs * ldx))), t(256);
                if (rbm.f32())
                    launch_pdl(load_rows_kernel<float>, gr, t, side, X, ldx, d_idx, bs, v,
                               static_cast<float*>(rbm.XRs[slot]), ldx, static_cast<const uint64_t*>(rbm.dctr), k);
                else
                    launch_pdl(load_rows_kernel<bf16>, gr, t, side, X, ldx, d_idx, bs, v,
                               static_cast<bf16*>(rbm.XRs[slot]), ldx, static_cast<const uint64_t*>(rbm.dctr), k);
                CUDA_THROW(cudaEventRecord(ev_load[slot], side));
                CUDA_THROW(cudaStreamWaitEvent(rbm.stream, ev_load[slot], 0));
                rbm.use_slot(slot);
                if (rbm.f32())
                    run_cd1<float>(rbm, bs, lr, 0, philox_seed, 0, rbm.dctr, k, k + 1 == nsteps ? nsteps : 0);
                else
                    run_cd1<bf16>(rbm, bs, lr, 0, philox_seed, 0, rbm.dctr, k, k + 1 == nsteps ? nsteps : 0);
                CUDA_THROW(cudaEventRecord(ev_done[slot], rbm.stream));
            }
            rbm.use_slot(0);
            rbm.bias_side = nullptr;
            rbm.bias_pending = false;
            CUDA_THROW(cudaEventRecord(ev_side, side));  // join the side stream back
            CUDA_THROW(cudaStreamWaitEvent(rbm.stream, ev_side, 0));
            CUDA_THROW(cudaStreamEndCapture(rbm.stream, &g));
            const cudaError_t ie = cudaGraphInstantiate(&ge, g, 0);
            cudaGraphDestroy(g);
            CUDA_THROW(ie);
            own.graphs.push_back(ge);
            return ge;
        };
        // PARNN_CD1_GRAPH=0: the same steps launched one kernel at a time on the chain
        // stream (test reference for the graphs; read per call)
        const char* gv = std::getenv("PARNN_CD1_GRAPH");
        const bool graphs = !(gv && gv[0] == '0');
        cudaGraphExec_t gbig = graphs && steps >= kGraphSteps ? capture(kGraphSteps) : nullptr;
        cudaGraphExec_t gone = graphs && steps % kGraphSteps ? capture(1) : nullptr;
        uint64_t hctr[2];
        cudaEvent_t t0, t1;
        CUDA_THROW(cudaEventCreate(&t0));
        CUDA_THROW(cudaEventCreate(&t1));
        CUDA_THROW(cudaEventRecord(t0, rbm.stream));
        for (uint64_t ep = 0; ep < epochs; ++ep) {
            std::vector<uint64_t> order(n);
            for (long i = 0; i < n; ++i) order[i] = static_cast<uint64_t>(i);
            rng.shuffle(order);  // feature_batches (pretrain.cpp:141-158)
            CUDA_THROW(cudaStreamSynchronize(rbm.stream));  // idx / hctr of the previous epoch are free
            for (long i = 0; i < n; ++i) idx[i] = static_cast<uint32_t>(order[i]);
            hctr[0] = 0;
            hctr[1] = counter;
            CUDA_THROW(cudaMemcpyAsync(d_idx, idx.data(), n * 4, cudaMemcpyHostToDevice, rbm.stream));
            CUDA_THROW(cudaMemcpyAsync(rbm.dctr, hctr, sizeof(hctr), cudaMemcpyHostToDevice, rbm.stream));
            if (graphs) {
                for (long k = 0; k + kGraphSteps <= steps; k += kGraphSteps)
                    CUDA_THROW(cudaGraphLaunch(gbig, rbm.stream));
                for (long k = 0; k < steps % kGraphSteps; ++k) CUDA_THROW(cudaGraphLaunch(gone, rbm.stream));
            } else {
                for (long k = 0; k < steps; ++k) {
                    const dim3 gr(static_cast<unsigned>(grid_of(bs * ldx))), t(256);
                    const uint64_t ck = counter + static_cast<uint64_t>(k) * bs * static_cast<uint64_t>(h);
                    if (rbm.f32()) {
                        launch_pdl(load_rows_kernel<float>, gr, t, rbm.stream, X, ldx, d_idx + k * bs, bs, v,
                                   static_cast<float*>(rbm.XR), ldx, static_cast<const uint64_t*>(nullptr), 0L);
                        run_cd1<float>(rbm, bs, lr, 0, philox_seed, ck);
                    } else {
                        launch_pdl(load_rows_kernel<bf16>, gr, t, rbm.stream, X, ldx, d_idx + k * bs, bs, v,
                                   static_cast<bf16*>(rbm.XR), ldx, static_cast<const uint64_t*>(nullptr), 0L);
                        run_cd1<bf16>(rbm, bs, lr, 0, philox_seed, ck);
                    }
                }
            }
            counter += static_cast<uint64_t>(steps) * static_cast<uint64_t>(bs) * static_cast<uint64_t>(h);
            for (long k = 0; k < steps; ++k) rng.jump(skip);  // the reference's b*h sample_bernoulli draws
        }
        CUDA_THROW(cudaEventRecord(t1, rbm.stream));
        CUDA_THROW(cudaStreamSynchronize(rbm.stream));
        float ms = 0.f;
        CUDA_THROW(cudaEventElapsedTime(&ms, t0, t1));  // device span of the epochs (host shuffles overlap it)
        g_pretrain_stats.cd1_seconds += ms * 1e-3;
        g_pretrain_stats.cd1_steps += static_cast<uint64_t>(steps) * epochs;
        g_pretrain_stats.cd1_flop += 10.0 * v * h * static_cast<double>(bs) * steps * epochs;
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
        rbm.ev_neg = rbm.ev_bias = nullptr;  // released with the other per-layer objects at exit
        // next layer input: hidden probabilities over the whole data (pretrain.cpp:190)
        const long ldh = pad32(h);
        float* Xn = nullptr;
        CUDA_THROW(cudaMalloc(&Xn, n * ldh * 4));
        own.mem.push_back(Xn);
        rbm.plan(bs);
        for (long c0 = 0; c0 < n; c0 += bs) {
            const long cb = std::min(bs, n - c0);
            if (rbm.f32())
                load_rows_kernel<float><<<grid_of(cb * ldx), 256, 0, rbm.stream>>>(X + c0 * ldx, ldx, nullptr, cb, v,
                                                                                static_cast<float*>(rbm.XR), ldx, nullptr, 0);
            else
                load_rows_kernel<bf16><<<grid_of(cb * ldx), 256, 0, rbm.stream>>>(X + c0 * ldx, ldx, nullptr, cb, v,
                                                                               static_cast<bf16*>(rbm.XR), ldx, nullptr, 0);
            rbm.hidden_probs_rows(cb, Xn + c0 * ldh, ldh);
        }
        CUDA_THROW(cudaStreamSynchronize(rbm.stream));
        // the previous layer's input is no longer needed (at config 4: 8 GB per layer)
        own.mem.erase(std::find(own.mem.begin(), own.mem.end(), static_cast<void*>(X)));
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
}

}  // namespace pnb
