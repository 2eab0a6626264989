// Data ingress on the device: generate_synthetic + split_cv +
// train-split feature_stats / standardize_in_place (data.cpp:124-242) straight
// into a DeviceDataset, for data sets too large to generate on the host
// (config 2 at 128 frames per class: 1.1 M frames x 440 = 5e8 gaussians).
//
// The reference draws every gaussian from ONE sequential Rng(seed) stream
// (rng.cpp:60-77, Marsaglia polar method with a cached spare): attempt a of
// the polar loop consumes u64 draws 2a and 2a+1 of xoshiro256**, and each
// accepted attempt yields two consecutive gaussians (u k, then the spare v k).
// So the gaussian stream is a function of the u64 stream alone:
//   1. segments of S attempts start at xoshiro states obtained by GF(2)
//      jump-ahead (the host squares T^2S repeatedly, each thread composes the
//      bits of its segment index: no sequential walk);
//   2. every segment counts its accepted attempts (u, v and s = u^2 + v^2 in
//      exact IEEE fp64 without contraction, so the accept decisions are the
//      reference's bit for bit); an exclusive scan places them;
//   3. the segments are replayed and write their gaussians in place.
// Class means (the first classes x dim gaussians) are rescaled to norm s; the
// features are mean + noise. The split permutation is the reference's own
// shuffled_indices (host Fisher-Yates, integer). Labels and row order are
// therefore bit-exact; features agree to fp64 libm ulps before the fp32 store
// (CUDA's log / sqrt vs glibc's), i.e. within fp32 rounding.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "host.h"
#include "runtime.h"

namespace pnb {

namespace {

constexpr int kSeg = 2048;  // polar attempts per segment (4096 u64 draws)
constexpr int kJumpLevels = 24;

struct JumpSet {  // T^(2 kSeg 2^i), i < kJumpLevels: [level][256 columns][4 words]
    uint64_t col[kJumpLevels][256][4];
};

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

__device__ __forceinline__ uint64_t xo_next(uint64_t (&s)[4]) {
    const uint64_t out = rotl64(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return out;
}

// xoshiro state of segment `seg`: the seeded state jumped by seg * 2 kSeg draws
__device__ void segment_state(const JumpSet* J, const uint64_t* s0, long seg, uint64_t (&s)[4]) {
    for (int w = 0; w < 4; ++w) s[w] = s0[w];
    for (int lv = 0; seg; ++lv, seg >>= 1) {
        if (!(seg & 1)) continue;
        uint64_t r[4] = {0, 0, 0, 0};
        for (int k = 0; k < 256; ++k)
            if ((s[k >> 6] >> (k & 63)) & 1)
                for (int w = 0; w < 4; ++w) r[w] ^= J->col[lv][k][w];
        for (int w = 0; w < 4; ++w) s[w] = r[w];
    }
}

// one polar attempt: u, v = uniform(-1, 1) (rng.cpp:43-49), s = u^2 + v^2, exact
// IEEE operations in the reference's order (no FMA contraction)
__device__ __forceinline__ bool polar_attempt(uint64_t (&st)[4], double& u, double& v, double& s) {
    const double x1 = __dmul_rn(static_cast<double>(xo_next(st) >> 11), 0x1.0p-53);
    const double x2 = __dmul_rn(static_cast<double>(xo_next(st) >> 11), 0x1.0p-53);
    u = __dadd_rn(-1.0, __dmul_rn(2.0, x1));
    v = __dadd_rn(-1.0, __dmul_rn(2.0, x2));
    s = __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v));
    return s < 1.0 && s != 0.0;
}

__global__ void polar_count_kernel(const JumpSet* J, const uint64_t* s0, long nseg, int* counts) {
    const long seg = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (seg >= nseg) return;
    uint64_t st[4];
    segment_state(J, s0, seg, st);
    int c = 0;
    double u, v, s;
    for (int a = 0; a < kSeg; ++a) c += polar_attempt(st, u, v, s);
    counts[seg] = c;
}

__global__ void polar_emit_kernel(const JumpSet* J, const uint64_t* s0, long nseg, const long* first,
                                  long ngauss, double* __restrict__ g) {
    const long seg = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (seg >= nseg) return;
    uint64_t st[4];
    segment_state(J, s0, seg, st);
    long m = first[seg];  // accepted attempts before this segment
    double u, v, s;
    for (int a = 0; a < kSeg && 2 * m < ngauss; ++a) {
        if (!polar_attempt(st, u, v, s)) continue;
        const double k = sqrt(-2.0 * log(s) / s);
        g[2 * m] = u * k;
        if (2 * m + 1 < ngauss) g[2 * m + 1] = v * k;
        ++m;
    }
}

// class means on the sphere of radius sep (data.cpp:135-145): one thread per class
__global__ void class_means_kernel(double* __restrict__ mu, long classes, long dim, double sep) {
    const long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= classes) return;
    double* row = mu + k * dim;
    double acc = 0.0;
    for (long j = 0; j < dim; ++j) acc += row[j] * row[j];
    const double scale = sep / sqrt(acc);
    for (long j = 0; j < dim; ++j) row[j] *= scale;
}

// per-column partial sums of the (unstandardized) split rows:
// pass 0 sum x, pass 1 sum (x - mean)^2; block (column group, row chunk)
__global__ void column_partials_kernel(const double* __restrict__ g, long kd, long dim, long per_class,
                                       const uint64_t* __restrict__ rows, long n, long chunk,
                                       const double* __restrict__ mean, double* __restrict__ part) {
    const long j = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (j >= dim) return;
    const long r0 = blockIdx.y * chunk, r1 = min(n, r0 + chunk);
    double acc = 0.0;
    for (long i = r0; i < r1; ++i) {
        const long r = static_cast<long>(rows[i]);
        const double x = g[(r / per_class) * dim + j] + g[kd + r * dim + j];
        if (mean) {
            const double c = x - mean[j];
            acc += c * c;
        } else {
            acc += x;
        }
    }
    part[blockIdx.y * dim + j] = acc;
}

// fixed-order sum of the partials -> mean (pass 0) or stddev (pass 1, < 1e-12 -> 1, data.cpp:226)
__global__ void column_finish_kernel(const double* __restrict__ part, long nchunk, long dim, long n, int pass,
                                     double* __restrict__ out) {
    const long j = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (j >= dim) return;
    double acc = 0.0;
    for (long c = 0; c < nchunk; ++c) acc += part[c * dim + j];
    double v = acc / static_cast<double>(n);
    if (pass == 1) {
        v = sqrt(v);
        if (v < 1e-12) v = 1.0;
    }
    out[j] = v;
}

// output rows i of a split (Dataset::select order): fp32 (standardized) features + label
__global__ void emit_rows_kernel(const double* __restrict__ g, long kd, long dim, long per_class,
                                 const uint64_t* __restrict__ rows, long n, const double* __restrict__ mean,
                                 const double* __restrict__ sd, float* __restrict__ x, long ld,
                                 int32_t* __restrict__ y) {
    const long i = blockIdx.x;
    if (i >= n) return;
    const long r = static_cast<long>(rows[i]);
    const long k = r / per_class;
    for (long j = threadIdx.x; j < dim; j += blockDim.x) {
        double v = g[k * dim + j] + g[kd + r * dim + j];
        if (mean) v = (v - mean[j]) / sd[j];
        x[i * ld + j] = static_cast<float>(v);
    }
    if (threadIdx.x == 0) y[i] = static_cast<int32_t>(k);
}

template <typename T>
T* dmalloc(size_t n) {
    void* p = nullptr;
    CUDA_THROW(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    return static_cast<T*>(p);
}

}  // namespace

void generate_device(Context* ctx, uint64_t classes, uint64_t dim, uint64_t per_class, double sep, uint64_t seed,
                     double cv_fraction, uint64_t split_seed, bool standardize, DeviceDataset** train,
                     DeviceDataset** cv) {
    if (classes == 0 || dim == 0 || per_class == 0)
        throw std::runtime_error("generate_synthetic: classes, dim and per_class must be >= 1");
    if (sep < 0.0) throw std::runtime_error("generate_synthetic: separation must be >= 0, got " + host::fmt_num(sep));
    if (cv_fraction <= 0.0 || cv_fraction >= 1.0)
        throw std::runtime_error("split_cv: cv_fraction must be in (0,1), got " + host::fmt_num(cv_fraction));
    const uint64_t n = classes * per_class;
    if (n < 10) throw std::runtime_error("split_cv: need at least 10 examples, got " + std::to_string(n));
    CUDA_THROW(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const long kd = static_cast<long>(classes * dim);
    const long ngauss = kd + static_cast<long>(n * dim);
    // attempts: the acceptance rate is pi/4; segments for 4/3 of the expected count,
    // more are added if the scan comes up short
    long nseg = (static_cast<long>(static_cast<double>(ngauss) / 2.0 / 0.785398 * 1.02) + kSeg) / kSeg + 1;
    // jump matrices T^(2 kSeg 2^i) and the seeded state
    std::vector<JumpSet> hj(1);
    {
        host::Jump j = host::make_jump(2ull * kSeg);
        for (int lv = 0; lv < kJumpLevels; ++lv) {
            std::memcpy(hj[0].col[lv], j.col, sizeof(j.col));
            if (lv + 1 < kJumpLevels) j = host::jump_square(j);
        }
    }
    if (nseg >= (1L << kJumpLevels)) throw std::runtime_error("generate_synthetic: data set too large");
    host::Rng rng0(seed);
    uint64_t s0[4];
    double spare;
    bool has;
    rng0.get_state(s0, &spare, &has);
    JumpSet* dJ = dmalloc<JumpSet>(1);
    uint64_t* ds0 = dmalloc<uint64_t>(4);
    CUDA_THROW(cudaMemcpyAsync(dJ, hj.data(), sizeof(JumpSet), cudaMemcpyHostToDevice, s));
    CUDA_THROW(cudaMemcpyAsync(ds0, s0, sizeof(s0), cudaMemcpyHostToDevice, s));
    int* dcount = nullptr;
    long* dfirst = nullptr;
    std::vector<int> counts;
    std::vector<long> first;
    for (;;) {
        dcount = dmalloc<int>(nseg);
        polar_count_kernel<<<static_cast<unsigned>((nseg + 127) / 128), 128, 0, s>>>(dJ, ds0, nseg, dcount);
        CUDA_THROW(cudaGetLastError());
        counts.resize(nseg);
        CUDA_THROW(cudaMemcpyAsync(counts.data(), dcount, nseg * sizeof(int), cudaMemcpyDeviceToHost, s));
        CUDA_THROW(cudaStreamSynchronize(s));
        first.assign(nseg, 0);
        long acc = 0;
        for (long i = 0; i < nseg; ++i) {
            first[i] = acc;
            acc += counts[i];
        }
        if (2 * acc >= ngauss) break;
        cudaFree(dcount);
        nseg = nseg + nseg / 8 + 1;  // (practically never) too few attempts: widen
    }
    dfirst = dmalloc<long>(nseg);
    CUDA_THROW(cudaMemcpyAsync(dfirst, first.data(), nseg * sizeof(long), cudaMemcpyHostToDevice, s));
    double* g = dmalloc<double>(ngauss);
    polar_emit_kernel<<<static_cast<unsigned>((nseg + 127) / 128), 128, 0, s>>>(dJ, ds0, nseg, dfirst, ngauss, g);
    class_means_kernel<<<static_cast<unsigned>((classes + 127) / 128), 128, 0, s>>>(g, static_cast<long>(classes),
                                                                                     static_cast<long>(dim), sep);
    CUDA_THROW(cudaGetLastError());
    // split_cv: shuffled_indices(n, split_seed) (integer stream, host), the first
    // ceil(f n) rows to CV (data.cpp:170-183)
    const std::vector<uint64_t> idx = host::shuffled_indices(n, split_seed);
    const uint64_t ncv = static_cast<uint64_t>(std::ceil(cv_fraction * static_cast<double>(n)));
    const uint64_t ntr = n - ncv;
    uint64_t* drows = dmalloc<uint64_t>(n);
    CUDA_THROW(cudaMemcpyAsync(drows, idx.data(), n * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    const uint64_t* cv_rows = drows;
    const uint64_t* tr_rows = drows + ncv;
    double *mean = nullptr, *sd = nullptr, *part = nullptr;
    if (standardize) {
        if (ntr == 0) throw std::runtime_error("feature_stats: empty dataset");
        const long chunk = 2048, nchunk = (static_cast<long>(ntr) + chunk - 1) / chunk;
        mean = dmalloc<double>(dim);
        sd = dmalloc<double>(dim);
        part = dmalloc<double>(static_cast<size_t>(nchunk) * dim);
        const dim3 grid(static_cast<unsigned>((dim + 127) / 128), static_cast<unsigned>(nchunk));
        const unsigned g1 = static_cast<unsigned>((dim + 127) / 128);
        column_partials_kernel<<<grid, 128, 0, s>>>(g, kd, dim, per_class, tr_rows, ntr, chunk, nullptr, part);
        column_finish_kernel<<<g1, 128, 0, s>>>(part, nchunk, dim, ntr, 0, mean);
        column_partials_kernel<<<grid, 128, 0, s>>>(g, kd, dim, per_class, tr_rows, ntr, chunk, mean, part);
        column_finish_kernel<<<g1, 128, 0, s>>>(part, nchunk, dim, ntr, 1, sd);
        CUDA_THROW(cudaGetLastError());
    }
    auto* tr = new DeviceDataset(ctx, static_cast<long>(ntr), static_cast<long>(dim), static_cast<long>(classes));
    auto* cvd = new DeviceDataset(ctx, static_cast<long>(ncv), static_cast<long>(dim), static_cast<long>(classes));
    if (ntr) emit_rows_kernel<<<static_cast<unsigned>(ntr), 128, 0, s>>>(g, kd, dim, per_class, tr_rows, ntr, mean, sd,
                                                                        tr->x32, tr->ld, tr->y);
    if (ncv) emit_rows_kernel<<<static_cast<unsigned>(ncv), 128, 0, s>>>(g, kd, dim, per_class, cv_rows, ncv, mean, sd,
                                                                        cvd->x32, cvd->ld, cvd->y);
    CUDA_THROW(cudaGetLastError());
    CUDA_THROW(cudaStreamSynchronize(s));
    for (void* p : {static_cast<void*>(dJ), static_cast<void*>(ds0), static_cast<void*>(dcount),
                    static_cast<void*>(dfirst), static_cast<void*>(g), static_cast<void*>(drows),
                    static_cast<void*>(mean), static_cast<void*>(sd), static_cast<void*>(part)})
        if (p) cudaFree(p);
    *train = tr;
    *cv = cvd;
}

}  // namespace pnb
