// In-kernel split-K reduction with the CD-1 epilogues (pretrain.cpp:37-121),
// for the three M = b GEMMs of an RBM step (rbm.cu).
//
// A split-K GEMM whose GemmEpi::coop points at a Cd1Epi runs one work item per
// CTA (tiles x ksplit <= SMs, all co-resident). Each CTA stores its fp32 partial
// tile (EPI_PARTIAL), then the ksplit CTAs of a tile meet on a per-tile arrival
// counter and each one finalises 1/ksplit of the tile's rows: it sums the
// partials in split order (deterministic, the same sum as the separate
// reduction kernels) and applies the step's elementwise work --
//   POS:   pos = sigmoid(z + hb) -> PN, z -> ZP, hs = draw(pos) -> HS
//   RECON: recon = act(z + vb) -> rec rows; column sums of (v - recon) in fp64
//   NEG:   -neg = -sigmoid(z + hb) -> PN rows [b, 2b); column sums of
//          (pos - neg) in fp64 from the two pre-activations
// -- so the step needs no separate reduction launches. Column sums go to
// colpart[row chunk][col] with row chunk = tile_m * ksplit + split.
#pragma once
#include <cuda_bf16.h>

#include <cstdint>

namespace pnb {

enum Cd1Kind : int { CD1_POS = 0, CD1_RECON = 1, CD1_NEG = 2 };

struct Cd1Epi {
    int kind = 0;
    int mode = 0;      // POS sampling: 0 Philox, 1 threshold_half, 2 injected uniforms, 3 hs = pos
    int gaussian = 0;  // RECON: identity (Gaussian visibles) instead of sigmoid
    long b = 0;        // rows of the step
    const float* bias = nullptr;  // hb (POS, NEG) or vb (RECON)
    void* pn = nullptr;  // T: PN rows [0, b) = pos, [b, 2b) = -neg
    void* hs = nullptr;  // T: POS samples
    long ldh = 0;
    float* zp = nullptr;  // POS writes, NEG reads: pos pre-activations [b x ldh]
    const void* x = nullptr;  // T: RECON visible rows (v)
    void* rec = nullptr;      // T: RECON output rows
    long ldv = 0;
    double* colpart = nullptr;  // RECON / NEG: [chunks][ldc]
    long ldc = 0;
    uint64_t key = 0, counter = 0;
    const uint64_t* dctr = nullptr;  // graph-launched steps: {step, counter base}
    const double* u = nullptr;       // injected uniforms [b x n]
    unsigned* ctr = nullptr;         // 2 per output tile: arrivals, departures
};

__device__ __forceinline__ uint32_t cd1_mulhilo(uint32_t a, uint32_t b, uint32_t& hi) {
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
        const uint32_t lo0 = cd1_mulhilo(0xD2511F53u, c0, hi0);
        const uint32_t lo1 = cd1_mulhilo(0xCD9E8D57u, c2, hi1);
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return static_cast<float>(c0 >> 8) * (1.0f / 16777216.0f);
}

__device__ __forceinline__ float cd1_sigmoid(float z) { return 1.f / (1.f + expf(-z)); }
__device__ __forceinline__ double cd1_sigmoid_d(float z) { return 1.0 / (1.0 + exp(-static_cast<double>(z))); }

template <typename T>
__device__ __forceinline__ float cd1_tf(T v) {
    return static_cast<float>(v);
}
template <>
__device__ __forceinline__ float cd1_tf<__nv_bfloat16>(__nv_bfloat16 v) {
    return __bfloat162float(v);
}

// The per-element CD-1 step for (row r, column j) of an output of width n with
// split-summed accumulator z; returns this element's column-sum term.
template <typename T>
__device__ __forceinline__ double cd1_element(const Cd1Epi& e, long r, long j, long n, float acc, uint64_t counter) {
    const float z = acc + e.bias[j];
    if (e.kind == CD1_POS) {
        const T pv = static_cast<T>(cd1_sigmoid(z));
        const float p = cd1_tf<T>(pv);
        static_cast<T*>(e.pn)[r * e.ldh + j] = pv;
        e.zp[r * e.ldh + j] = z;
        const long i = r * n + j;
        float s;
        if (e.mode == 3) s = p;
        else if (e.mode == 1) s = p > 0.5f ? 1.f : 0.f;
        else if (e.mode == 2) s = e.u[i] < static_cast<double>(p) ? 1.f : 0.f;
        else s = philox_uniform(e.key, counter + static_cast<uint64_t>(i)) < p ? 1.f : 0.f;
        static_cast<T*>(e.hs)[r * e.ldh + j] = static_cast<T>(s);
        return 0.0;
    }
    if (e.kind == CD1_RECON) {
        const T x = static_cast<T>(e.gaussian ? z : cd1_sigmoid(z));
        static_cast<T*>(e.rec)[r * e.ldv + j] = x;
        return static_cast<double>(cd1_tf<T>(static_cast<const T*>(e.x)[r * e.ldv + j])) -
               (e.gaussian ? static_cast<double>(z) : cd1_sigmoid_d(z));
    }
    static_cast<T*>(e.pn)[(e.b + r) * e.ldh + j] = static_cast<T>(-cd1_sigmoid(z));
    return cd1_sigmoid_d(e.zp[r * e.ldh + j]) - cd1_sigmoid_d(z);
}

// Epilogue-warp part of a cooperative split-K tile (256 threads = warps 2-9,
// t = their index). `scratch` is idle shared memory (the TMA ring) for 256
// doubles. Called once per CTA after its partial tile is stored.
template <typename T>
__device__ __noinline__ void cd1_coop_finish(const Cd1Epi* __restrict__ ep_, const float* __restrict__ part,
                                             long split_stride, long ldp, int ksplit, int M, int N, int BN, int m0,
                                             int n0, int ks, int tile_mn, int tile_m, int t, double* scratch) {
    const Cd1Epi& e = *ep_;
    asm volatile("bar.sync 1, 256;" ::: "memory");  // this CTA's partial tile is stored
    if (t == 0) {
        __threadfence();
        atomicAdd(&e.ctr[2 * tile_mn], 1u);
        unsigned seen;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(&e.ctr[2 * tile_mn]) : "memory");
            if (seen < static_cast<unsigned>(ksplit)) __nanosleep(64);
        } while (seen < static_cast<unsigned>(ksplit));
        __threadfence();
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");  // every split of the tile is stored
    const int rows_per = (128 + ksplit - 1) / ksplit;
    const int r_lo = m0 + ks * rows_per;
    const int r_hi = min(min(M, m0 + 128), r_lo + rows_per);
    const int nrg = 256 / BN;  // row groups
    const int cj = t % BN, rg = t / BN;
    const long j = n0 + cj;
    uint64_t counter = e.counter;
    if (e.kind == CD1_POS && e.dctr)
        counter = e.dctr[1] + e.dctr[0] * static_cast<uint64_t>(e.b) * static_cast<uint64_t>(N);
    double acc = 0.0;
    if (j < N) {
        for (int r = r_lo + rg; r < r_hi; r += nrg) {
            const float* q = part + static_cast<long>(r) * ldp + j;
            float a = __ldcg(q);
            for (int k = 1; k < ksplit; ++k) a += __ldcg(q + k * split_stride);
            acc += cd1_element<T>(e, r, j, N, a, counter);
        }
    }
    if (e.kind != CD1_POS) {
        scratch[t] = acc;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (rg == 0 && j < N) {
            double s = 0.0;
            for (int g = 0; g < nrg; ++g) s += scratch[g * BN + cj];
            e.colpart[(static_cast<long>(tile_m) * ksplit + ks) * e.ldc + j] = s;
        }
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");  // this CTA is done reading the partials
    if (t == 0) {
        // the last CTA out re-arms the tile's counters for the next launch
        if (atomicAdd(&e.ctr[2 * tile_mn + 1], 1u) == static_cast<unsigned>(ksplit) - 1) {
            e.ctr[2 * tile_mn] = 0u;
            e.ctr[2 * tile_mn + 1] = 0u;
        }
    }
}

}  // namespace pnb
