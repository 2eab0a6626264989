// NG-SGD, full Kronecker-factored variant (optimizer.cpp:108-157), on device.
//
// Per layer: S = R + lambda I with lambda = max(alpha tr(R)/n, 1e-8)
// (smoothed_factor), Cholesky of S_out and S_in (S_out factored ONCE; the
// reference re-factors it for the bias solve), Ghat = S_out^-1 [G | g_b],
// transpose, S_in^-1 on the weight part, transpose back, Frobenius rescale
// gamma and the fused SGD update (sgd_step_in_place) with the finite check.
//
// Blocked algorithms, 128-row blocks (NG_NB):
//   Cholesky (right-looking): per block j
//     chol_diag_kernel  — SIMT fp32, one CTA: L_jj = chol(A_jj) and L_jj^-1
//     panel  A_{>j,j} <- A_{>j,j} L_jj^-T           tcgen05 GEMM (in place)
//     trail  A_{>j,>j} -= A_{>j,j} A_{>j,j}^T       tcgen05 GEMM, lower tiles only
//   S^-1 X (X with c columns, in place):
//     forward  X_i <- L_ii^-1 X_i ; X_{>i} -= L_{>i,i} X_i
//     backward X_i <- L_ii^-T X_i ; X_{<i} -= L_{i,<i}^T X_i
// Every GEMM runs in fp32 mode (3xTF32 split, see gemm.cuh): the solves need
// fp32 accuracy at kappa(S) ~ 1e2, which TF32 alone does not give.
#include <cfloat>

#include "runtime.h"

namespace pnb {

namespace {

#ifndef PNB_CLK
#define PNB_CLK(i) \
    do {           \
    } while (0)
#endif

constexpr int NB = NG_NB;
constexpr int LDS = NB + 1;  // padded shared-memory row

float* dalloc_f(size_t n) {
    void* p = nullptr;
    CUDA_THROW(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(float)));
    zero(p, std::max<size_t>(n, 1) * sizeof(float));
    return static_cast<float*>(p);
}

__global__ void trace_lambda_kernel(const float* __restrict__ r, long n, long ld, double alpha,
                                    double* __restrict__ lam) {
    __shared__ double sh[256];
    double acc = 0.0;
    for (long i = threadIdx.x; i < n; i += blockDim.x) acc += r[i * ld + i];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double l = alpha * sh[0] / static_cast<double>(n);
        *lam = l < 1e-8 ? 1e-8 : l;
    }
}

// S = R + lambda I (Cholesky reads the lower triangle incl. the diagonal).
__global__ void shift_copy_kernel(const float* __restrict__ r, long n, long ld, const double* __restrict__ lam,
                                  float* __restrict__ s) {
    const long total = n * ld;
    const float l = static_cast<float>(*lam);
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const long row = i / ld, col = i % ld;
        float v = (col < n) ? r[i] : 0.f;
        if (row == col) v += l;
        s[i] = v;
    }
}

// Per-thread micro-tile product for the in-CTA block algebra of the diagonal
// kernel (256 threads as a 16 x 16 grid, thread tile TM x TN):
//   acc[i][q] = sum_{k<K} A(m0 + ty*TM + i, k) * B(n0 + tx*TN + q, k)
// A(m, k) = A[m*LDS + k]; B(n, k) = Bm[n*LDS + k] if BT, else Bm[k*LDS + n].
template <int TM, int TN, bool BT>
__device__ __forceinline__ void micro_mma(const float* A, const float* Bm, int K, int m0, int n0,
                                          float (&acc)[TM][TN]) {
    const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int q = 0; q < TN; ++q) acc[i][q] = 0.f;
    const float* ap = A + (m0 + ty * TM) * LDS;
#pragma unroll 4
    for (int k = 0; k < K; ++k) {
        float av[TM], bv[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) av[i] = ap[i * LDS + k];
#pragma unroll
        for (int q = 0; q < TN; ++q)
            bv[q] = BT ? Bm[(n0 + tx * TN + q) * LDS + k] : Bm[k * LDS + n0 + tx * TN + q];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int q = 0; q < TN; ++q) acc[i][q] = fmaf(av[i], bv[q], acc[i][q]);
    }
}

// Rows [r0, r0 + 16*TM) of the panel columns [c0, c0+32): P <- P * D^-T.
template <int TM>
__device__ __forceinline__ void panel_solve(float* S, const float* V, int c0) {
    const int r0 = c0 + 32;
    float acc[TM][2];
    micro_mma<TM, 2, true>(S + c0, V + c0 * LDS + c0, 32, r0, 0, acc);
    __syncthreads();
    const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int q = 0; q < 2; ++q) S[(r0 + ty * TM + i) * LDS + c0 + tx * 2 + q] = acc[i][q];
}

// Lower part of S[r0:, r0:] -= P P^T with P = S[r0:, c0:c0+32], r0 = c0 + 32.
template <int TM>
__device__ __forceinline__ void trailing_update(float* S, int c0) {
    const int r0 = c0 + 32;
    const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
    if (tx * TM > ty * TM + TM - 1) return;  // micro tile strictly above the diagonal
    float acc[TM][TM];
    micro_mma<TM, TM, true>(S + c0, S + c0, 32, r0, r0, acc);  // A(m,k) = B(m,k) = S[m][c0+k]
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int q = 0; q < TM; ++q) {
            const int r = r0 + ty * TM + i, c = r0 + tx * TM + q;
            if (c <= r) S[r * LDS + c] -= acc[i][q];
        }
}

// Diagonal block j: L = chol(A_jj) in place (zero upper part) and V = L^-1
// into linv (NB x NB, zero padded). Pivot failures are recorded with the
// reference's semantics (first non-positive / non-finite pivot, matrix.cpp:110-113).
//
// 256 threads; 4 panels of 32 columns. Per panel:
//   A. warp 0 factors the 32x32 diagonal sub-block D: lane i keeps row i in
//      registers, the 32 column steps fully unrolled; pivot and L[c][k]
//      arrive by warp shuffle;
//   B. rows below solve x D^T = a by forward substitution (one thread per row,
//      D broadcast from shared memory);
//   C. all 8 warps apply the rank-32 trailing update with register-tiled
//      micro products (6x6/4x4/2x2 per thread).
// Then 4 warps invert the 4 diagonal sub-blocks concurrently and the
// off-diagonal blocks of V follow by block forward substitution.
// Padding rows/columns (b < NB) hold the identity so every step is
// branch-free; only the b x b block is written back.
__global__ void __launch_bounds__(256) chol_diag_kernel(float* __restrict__ a, long ld, long j, int b,
                                                        float* __restrict__ linv, DevErr* err) {
    extern __shared__ float sm[];
    float* S = sm;                 // [NB][LDS]  A -> L
    float* V = sm + NB * LDS;      // [NB][LDS]  L^-1
    float* col = V + NB * LDS;     // [32] column broadcast of the 32x32 factorizations (16-byte aligned)
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    // PDL: the previous kernel of the chain (the look-ahead update of this block) is complete
    // and visible. (No early launch_dependents: the panel GEMM's CTAs would then hold SMs for
    // the whole factorization, 13.3 -> 14.4 ms per config-2 step.)
    grid_dep_wait();
    PNB_CLK(0);
    {
        // 16-byte loads, all issued before the shared stores (fewer memory requests: inside
        // the factorization chain, beside the bulk updates' traffic, that is what counts).
        // A warp covers 4 rows x 32 columns: lane -> row (lane >> 3), columns 4 (lane & 7) ..,
        // so each store instruction hits 32 distinct banks of the padded rows (bank r + c).
        float4 v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int tile = i * 8 + warp, r = 4 * (tile >> 2) + (lane >> 3), c = 32 * (tile & 3) + 4 * (lane & 7);
            v[i] = (r < b && c < b && c <= r) ? *reinterpret_cast<const float4*>(a + (j + r) * ld + j + c)
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int tile = i * 8 + warp, r = 4 * (tile >> 2) + (lane >> 3), c = 32 * (tile & 3) + 4 * (lane & 7);
            const float e[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int cc = c + q;
                S[r * LDS + cc] = (r >= b && r == cc) ? 1.f : ((cc <= r && cc < b) ? e[q] : 0.f);
            }
        }
        float4* v4 = reinterpret_cast<float4*>(V);  // 16-byte aligned: NB * LDS floats precede it
        for (int i = t; i < NB * LDS / 4; i += 256) v4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    PNB_CLK(1);
#pragma unroll 1
    for (int p = 0; p < NB / 32; ++p) {
        const int c0 = 32 * p;
        if (warp == 0) {
            // lane i holds row i of the block; the column steps are unrolled so
            // every register index is static, the pivot and L[c][k] come from the
            // owning lanes by shuffle (no shared-memory round trips on the chain)
            float d[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) d[c] = S[(c0 + lane) * LDS + c0 + c];
            // Software-pipelined: step k first finishes column k+1 and fetches the next
            // pivot, then applies its remaining column updates while that pivot's
            // shuffle / rsqrt latency runs (the same operations as the plain order).
            // The first failing pivot is remembered with warp-uniform selects and
            // recorded after the loop (a lane-0 branch per step cost a reconvergence).
            float piv = __shfl_sync(0xffffffffu, d[0], 0);
            int bad_k = -1;
            float bad_v = 0.f;
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const bool bad = c0 + k < b && (!(piv > 0.f) || !isfinite(piv));
                bad_v = (bad_k < 0 && bad) ? piv : bad_v;
                bad_k = (bad_k < 0 && bad) ? k : bad_k;
                const float rs = rsqrtf(piv);  // 1/L_kk
                const float lkk = piv * rs;
                const float lik = lane > k ? d[k] * rs : (lane == k ? lkk : 0.f);
                d[k] = lik;
                if (k + 1 < 32) {
                    // column k of L broadcast through shared memory (one store per lane,
                    // broadcast loads: the 31 - k shuffles per step were SHFL-throughput bound)
                    col[lane] = lik;
                    __syncwarp();
                    // rows c <= lane: a_ic -= L_ik L_ck (columns above the diagonal are dropped)
                    d[k + 1] = fmaf(-lik, col[k + 1], d[k + 1]);
                    piv = __shfl_sync(0xffffffffu, d[k + 1], k + 1);
#pragma unroll
                    for (int c = k + 2; c < 32; ++c) d[c] = fmaf(-lik, col[c], d[c]);
                    __syncwarp();  // every lane has read column k before the next step overwrites it
                }
            }
            if (lane == 0 && bad_k >= 0 && atomicCAS(&err->chol_failed, 0, 1) == 0) {
                err->chol_index = static_cast<int>(j + c0 + bad_k);
                err->chol_value = bad_v;
            }
#pragma unroll
            for (int c = 0; c < 32; ++c) S[(c0 + lane) * LDS + c0 + c] = c <= lane ? d[c] : 0.f;
        }
        __syncthreads();
        // B. rows below: x D^T = a (forward substitution, D rows broadcast)
        if (t < NB - c0 - 32) {
            const int r = c0 + 32 + t;
            float x[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) x[c] = S[r * LDS + c0 + c];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const float* dr = S + (c0 + c) * LDS + c0;
                float acc = x[c];
#pragma unroll
                for (int k = 0; k < c; ++k) acc -= x[k] * dr[k];
                x[c] = acc / dr[c];
            }
#pragma unroll
            for (int c = 0; c < 32; ++c) S[r * LDS + c0 + c] = x[c];
        }
        __syncthreads();
        PNB_CLK(2 + 2 * p);
        if (p == 0) trailing_update<6>(S, c0);
        else if (p == 1) trailing_update<4>(S, c0);
        else if (p == 2) trailing_update<2>(S, c0);
        __syncthreads();
        PNB_CLK(3 + 2 * p);
    }
    // D. inverses of the four 32x32 diagonal sub-blocks, one warp each:
    //    lane owns column `lane`; x_i = (e - sum_{q<i} D[i][q] x_q) / D[i][i]
    if (warp < NB / 32) {
        // right-looking: once x_i is known every later row's partial sum takes its
        // term (independent FMAs) instead of a serial dot product per row
        const int c0 = 32 * warp;
        float acc[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = (i == lane) ? 1.f : 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const float xi = acc[i] / S[(c0 + i) * LDS + c0 + i];
            acc[i] = xi;
#pragma unroll
            for (int r = i + 1; r < 32; ++r) acc[r] = fmaf(-S[(c0 + r) * LDS + c0 + i], xi, acc[r]);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) V[(c0 + i) * LDS + c0 + lane] = acc[i];
    }
    __syncthreads();
    PNB_CLK(10);
    // E. off-diagonal blocks of V = L^-1: V_{bi,q} = -D_bi^-1 sum_{k=q}^{bi-1} L_{bi,k} V_{k,q}
#pragma unroll 1
    for (int bi = 1; bi < NB / 32; ++bi) {
        const int r0 = 32 * bi;
        const int ty = t >> 4, tx = t & 15;
        // T = L[r0:r0+32, 0:r0] V[0:r0, 0:r0] -> staged in V[r0:r0+32, 0:r0] (still zero)
        if (bi == 1) {
            float acc[2][2];
            micro_mma<2, 2, false>(S, V, r0, r0, 0, acc);
            for (int i = 0; i < 2; ++i)
                for (int q = 0; q < 2; ++q) V[(r0 + ty * 2 + i) * LDS + tx * 2 + q] = acc[i][q];
        } else if (bi == 2) {
            float acc[2][4];
            micro_mma<2, 4, false>(S, V, r0, r0, 0, acc);
            for (int i = 0; i < 2; ++i)
                for (int q = 0; q < 4; ++q) V[(r0 + ty * 2 + i) * LDS + tx * 4 + q] = acc[i][q];
        } else {
            float acc[2][6];
            micro_mma<2, 6, false>(S, V, r0, r0, 0, acc);
            for (int i = 0; i < 2; ++i)
                for (int q = 0; q < 6; ++q) V[(r0 + ty * 2 + i) * LDS + tx * 6 + q] = acc[i][q];
        }
        __syncthreads();
        // V[r0:r0+32, 0:r0] = -D_bi^-1 T  (D_bi^-1 = V[r0:, r0:r0+32])
        if (bi == 1) {
            float acc[2][2];
            micro_mma<2, 2, false>(V + r0, V + r0 * LDS, 32, r0, 0, acc);
            __syncthreads();
            for (int i = 0; i < 2; ++i)
                for (int q = 0; q < 2; ++q) V[(r0 + ty * 2 + i) * LDS + tx * 2 + q] = -acc[i][q];
        } else if (bi == 2) {
            float acc[2][4];
            micro_mma<2, 4, false>(V + r0, V + r0 * LDS, 32, r0, 0, acc);
            __syncthreads();
            for (int i = 0; i < 2; ++i)
                for (int q = 0; q < 4; ++q) V[(r0 + ty * 2 + i) * LDS + tx * 4 + q] = -acc[i][q];
        } else {
            float acc[2][6];
            micro_mma<2, 6, false>(V + r0, V + r0 * LDS, 32, r0, 0, acc);
            __syncthreads();
            for (int i = 0; i < 2; ++i)
                for (int q = 0; q < 6; ++q) V[(r0 + ty * 2 + i) * LDS + tx * 6 + q] = -acc[i][q];
        }
        __syncthreads();
    }
    PNB_CLK(14);
    // 16-byte stores; a column group that straddles b (ragged last block) goes element-wise
#pragma unroll 4
    for (int i = 0; i < 16; ++i) {
        const int idx = t + 256 * i, r = idx >> 5, c = (idx & 31) * 4;
        float l4[4], v4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const bool in = r < b && c + q < b && c + q <= r;
            l4[q] = in ? S[r * LDS + c + q] : 0.f;
            v4[q] = in ? V[r * LDS + c + q] : 0.f;
        }
        *reinterpret_cast<float4*>(linv + r * NB + c) = make_float4(v4[0], v4[1], v4[2], v4[3]);
        if (r < b) {
            float* dst = a + (j + r) * ld + j + c;
            if (c + 4 <= b) {
                *reinterpret_cast<float4*>(dst) = make_float4(l4[0], l4[1], l4[2], l4[3]);
            } else {
                for (int q = 0; q < 4 && c + q < b; ++q) dst[q] = l4[q];
            }
        }
    }
    PNB_CLK(15);
}

__global__ void transpose_kernel(const float* __restrict__ src, long lds, long rows, long cols,
                                 float* __restrict__ dst, long ldd) {
    __shared__ float t[32][33];
    const long r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const long r = r0 + i, c = c0 + threadIdx.x;
        t[i][threadIdx.x] = (r < rows && c < cols) ? src[r * lds + c] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const long c = c0 + i, r = r0 + threadIdx.x;
        if (c < cols && r < rows) dst[c * ldd + r] = t[threadIdx.x][i];
    }
}

// [G | g_b] -> t (ld_t), for the joint S_out solve of weights and bias.
__global__ void pack_rhs_kernel(const float* __restrict__ g, long ldg, const float* __restrict__ gb, long rows,
                                long cols, float* __restrict__ t, long ldt) {
    const long total = rows * ldt;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const long r = i / ldt, c = i % ldt;
        t[i] = c < cols ? g[r * ldg + c] : (c == cols ? gb[r] : 0.f);
    }
}

// Deterministic sum of squares of a [rows x cols] region (two-level, fixed order).
__global__ void sumsq_partial_kernel(const float* __restrict__ x, long ld, long rows, long cols,
                                     double* __restrict__ part) {
    __shared__ double sh[256];
    double acc = 0.0;
    const long total = rows * cols;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const float v = x[(i / cols) * ld + (i % cols)];
        acc += static_cast<double>(v) * v;
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void sum_final_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
    __shared__ double sh[256];
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += part[i];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

// W -= lr * gamma * Ghat ; b -= lr * gamma_b * bhat (optimizer.cpp:142-154 + 29-34).
// scal: [0] |G|^2, [1] |g_b|^2, [2] |Ghat|^2, [3] |bhat|^2.
__global__ void ng_update_kernel(float* __restrict__ w, long ldw, float* __restrict__ bias, bf16* __restrict__ shadow,
                                 const float* __restrict__ gh, long ldgh, const float* __restrict__ bh, long ldbh,
                                 long dout, long din, const double* __restrict__ scal, const float* __restrict__ lr,
                                 const int* __restrict__ step, unsigned* __restrict__ flags, unsigned bit) {
    const double gamma = sqrt(scal[0]) / fmax(sqrt(scal[2]), 1e-20);
    const double gamma_b = sqrt(scal[1]) / fmax(sqrt(scal[3]), 1e-20);
    const float rate = lr[step ? *step : 0];
    const float gw = static_cast<float>(gamma), gbs = static_cast<float>(gamma_b);
    bool bad = false;
    const long total = dout * din;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const long r = i / din, c = i % din;
        const float g = gw * gh[r * ldgh + c];
        bad |= !isfinite(g);
        const float nw = w[r * ldw + c] - rate * g;
        w[r * ldw + c] = nw;
        if (shadow) shadow[r * ldw + c] = __float2bfloat16_rn(nw);
    }
    bool badb = false;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < dout; i += (long)gridDim.x * blockDim.x) {
        const float g = gbs * bh[i * ldbh];
        badb |= !isfinite(g);
        bias[i] -= rate * g;
    }
    if (bad) atomicOr(flags, 1u << bit);
    if (badb) atomicOr(flags, 1u << (bit + 1));
}

int grid_for(long total) { return (int)std::max<long>(1, std::min<long>((total + 255) / 256, 148L * 8)); }

constexpr int kDiagSmem = 2 * NB * LDS * 4 + 48 * 4;
// tuning aid: PARNN_NG_DIAG_SMEM=bytes requests more shared memory than the kernel uses (an SM of its own)
int diag_smem_req() {
    static const int v = std::getenv("PARNN_NG_DIAG_SMEM") ? std::atoi(std::getenv("PARNN_NG_DIAG_SMEM")) : 0;
    return v;
}

void ensure_diag_attr() {
    ensure_smem_attr(reinterpret_cast<const void*>(chol_diag_kernel), std::max(kDiagSmem, diag_smem_req()));
}

float* linv_blk(NgFactor& f, long j) { return f.linv + (j / NB) * NB * NB; }

// Trailing updates in super-blocks of G 128-column blocks: a block updates the next
// block column with every panel of its super-block so far (look-ahead, K = (pos+1)
// x 128); the super-block's last block also applies all G panels at once (K = 128 G)
// to the rest of the trailing matrix. 1/G as many bulk updates, each with G times
// the K: the fp32 read-modify-write of the trailing matrix (the early blocks'
// critical path) is paid once per super-block. PARNN_NG_SUPER=G (1 = per block).
int ng_super() {  // blocks per super-block (1 = one bulk update per block)
    static const int g = [] {
        const char* v = std::getenv("PARNN_NG_SUPER");
        return v ? std::max(1, std::atoi(v)) : 2;
    }();
    return g;
}

void build_factor(NgFactor& f, int sms) {
    f.panel.clear();
    f.col.clear();
    f.rest.clear();
    const int G = ng_super();
    const bool sup = G > 1;
    for (long j = 0; j < f.n; j += NB) {
        const long b = std::min<long>(NB, f.n - j), below = f.n - j - b;
        const int pos = static_cast<int>((j / NB) % G);  // position in the super-block
        const bool last = pos == G - 1;
        GemmPlan pp, cp, rp;
        if (below > 0 && sup) {
            float* a21 = f.a + (j + b) * f.ld + j;
            GemmEpi e;  // A21 <- A21 L_jj^-T, in place
            e.mode = EPI_GRAD;
            e.alpha = 1.f;
            e.out32 = a21;
            e.ld_out32 = f.ld;
            gemm_plan(pp, PREC_FP32, false, a21, f.ld, false, linv_blk(f, j), NB, (int)below, (int)b, (int)b, e, sms,
                      128);
            // the super-block's panels so far (columns j - pos*128 .. j + b): none of them has
            // reached block column j+1 yet, and at the super-block's end none has reached the rest
            const long k0 = j - pos * NB, kk = pos * NB + b;
            float* p21 = f.a + (j + b) * f.ld + k0;
            const long bn1 = std::min<long>(NB, below);
            GemmEpi c;
            c.mode = EPI_SUB;
            c.out32 = f.a + (j + b) * f.ld + (j + b);
            c.ld_out32 = f.ld;
            gemm_plan(cp, PREC_FP32, false, p21, f.ld, false, p21, f.ld, (int)below, (int)bn1, (int)kk, c, sms);
            const long rest = below - bn1;
            if (last && rest > 0) {
                float* p31 = p21 + bn1 * f.ld;
                GemmEpi u;
                u.mode = EPI_SUB;
                u.lower = 1;
                u.out32 = f.a + (j + b + bn1) * f.ld + (j + b + bn1);
                u.ld_out32 = f.ld;
                gemm_plan(rp, PREC_FP32, false, p31, f.ld, false, p31, f.ld, (int)rest, (int)rest, (int)kk, u, sms);
            }
        } else if (below > 0) {
            float* a21 = f.a + (j + b) * f.ld + j;
            GemmEpi e;  // A21 <- A21 L_jj^-T, in place (one N tile: BN = 128 >= b)
            e.mode = EPI_GRAD;
            e.alpha = 1.f;
            e.out32 = a21;
            e.ld_out32 = f.ld;
            gemm_plan(pp, PREC_FP32, false, a21, f.ld, false, linv_blk(f, j), NB, (int)below, (int)b, (int)b, e, sms,
                      128);
            // look-ahead: block column j+1 first (rows >= j+1) ...
            const long bn1 = std::min<long>(NB, below);
            GemmEpi c;
            c.mode = EPI_SUB;
            c.out32 = f.a + (j + b) * f.ld + (j + b);
            c.ld_out32 = f.ld;
            gemm_plan(cp, PREC_FP32, false, a21, f.ld, false, a21, f.ld, (int)below, (int)bn1, (int)b, c, sms);
            // ... then the rest of the trailing matrix (rows/cols >= j+2), lower tiles only
            const long rest = below - bn1;
            if (rest > 0) {
                float* a31 = a21 + bn1 * f.ld;
                GemmEpi u;
                u.mode = EPI_SUB;
                u.lower = 1;
                u.out32 = f.a + (j + b + bn1) * f.ld + (j + b + bn1);
                u.ld_out32 = f.ld;
                gemm_plan(rp, PREC_FP32, false, a31, f.ld, false, a31, f.ld, (int)rest, (int)rest, (int)b, u, sms);
            }
        }
        f.panel.push_back(pp);
        f.col.push_back(cp);
        f.rest.push_back(rp);
    }
}

void build_solve(NgFactor& f, NgSolve& sv, float* x, long ldx, long c, int sms) {
    sv.fdiag.clear();
    sv.fupd.clear();
    sv.bdiag.clear();
    sv.bupd.clear();
    sv.bnext.clear();
    sv.bpair.clear();
    sv.fnext.clear();
    sv.fpair.clear();
    for (long i0 = 0; i0 < f.n; i0 += NB) {
        const long b = std::min<long>(NB, f.n - i0), rest = f.n - i0 - b;
        float* xi = x + i0 * ldx;
        GemmEpi d;  // X_i <- Linv_ii X_i  (in place; single M tile)
        d.mode = EPI_GRAD;
        d.alpha = 1.f;
        d.out32 = xi;
        d.ld_out32 = ldx;
        GemmPlan fd, fu, bd, bu;
        gemm_plan(fd, PREC_FP32, false, linv_blk(f, i0), NB, true, xi, ldx, (int)b, (int)c, (int)b, d, sms);
        gemm_plan(bd, PREC_FP32, true, linv_blk(f, i0), NB, true, xi, ldx, (int)b, (int)c, (int)b, d, sms);
        if (rest > 0) {
            GemmEpi u;  // X_{>i} -= L_{>i,i} X_i
            u.mode = EPI_SUB;
            u.out32 = x + (i0 + b) * ldx;
            u.ld_out32 = ldx;
            gemm_plan(fu, PREC_FP32, false, f.a + (i0 + b) * f.ld + i0, f.ld, true, xi, ldx, (int)rest, (int)c,
                      (int)b, u, sms);
        }
        if (i0 > 0) {
            GemmEpi u;  // X_{<i} -= L_{i,<i}^T X_i
            u.mode = EPI_SUB;
            u.out32 = x;
            u.ld_out32 = ldx;
            gemm_plan(bu, PREC_FP32, true, f.a + i0 * f.ld, f.ld, true, xi, ldx, (int)i0, (int)c, (int)b, u, sms);
        }
        GemmPlan bn, bp;
        if (i0 >= NB) {
            GemmEpi u;  // X_{i-1} -= L_{i,i-1}^T X_i
            u.mode = EPI_SUB;
            u.out32 = x + (i0 - NB) * ldx;
            u.ld_out32 = ldx;
            gemm_plan(bn, PREC_FP32, true, f.a + i0 * f.ld + (i0 - NB), f.ld, true, xi, ldx, NB, (int)c, (int)b, u,
                      sms);
            if (i0 >= 2 * NB) {
                GemmEpi w;  // X_{<i-1} -= L_{{i-1,i},<i-1}^T [X_{i-1}; X_i]
                w.mode = EPI_SUB;
                w.out32 = x;
                w.ld_out32 = ldx;
                gemm_plan(bp, PREC_FP32, true, f.a + (i0 - NB) * f.ld, f.ld, true, x + (i0 - NB) * ldx, ldx,
                          (int)(i0 - NB), (int)c, (int)(NB + b), w, sms);
            }
        }
        sv.fdiag.push_back(fd);
        sv.fupd.push_back(fu);
        sv.bdiag.push_back(bd);
        sv.bupd.push_back(bu);
        sv.bnext.push_back(bn);
        sv.bpair.push_back(bp);
        GemmPlan fn, fp;
        if (rest > 0) {
            const long b1 = std::min<long>(NB, rest);
            GemmEpi u;  // X_{i+1} -= L_{i+1,i} X_i
            u.mode = EPI_SUB;
            u.out32 = x + (i0 + b) * ldx;
            u.ld_out32 = ldx;
            gemm_plan(fn, PREC_FP32, false, f.a + (i0 + b) * f.ld + i0, f.ld, true, xi, ldx, (int)b1, (int)c, (int)b,
                      u, sms);
            if (rest > b1) {
                GemmEpi w;  // X_{>i+1} -= L_{>i+1,{i,i+1}} [X_i; X_{i+1}]
                w.mode = EPI_SUB;
                w.out32 = x + (i0 + b + b1) * ldx;
                w.ld_out32 = ldx;
                gemm_plan(fp, PREC_FP32, false, f.a + (i0 + b + b1) * f.ld + i0, f.ld, true, xi, ldx,
                          (int)(rest - b1), (int)c, (int)(b + b1), w, sms);
            }
        }
        sv.fnext.push_back(fn);
        sv.fpair.push_back(fp);
    }
}

// Blocked Cholesky with look-ahead. fs carries the critical path
// diag(j) -> panel(j) -> col(j) [-> diag(j+1)]; the bulk rest(j) runs on ts
// concurrently with diag(j+1)/panel(j+1). col(j) must see rest(j-1) (both
// update block column j+1), so fs waits for it first. ev_panel[j] tells the
// forward solve that block column j of L is final.
void cholesky(Replica& r, int l, NgFactor& f, DevErr* err, cudaStream_t fs, cudaStream_t ts, bool conc) {
    size_t blk = 0;
    for (long j = 0; j < f.n; j += NB, ++blk) {
        const int b = (int)std::min<long>(NB, f.n - j);
        {
            static const bool pdl = !std::getenv("PARNN_NG_DIAG_PDL") || std::atoi(std::getenv("PARNN_NG_DIAG_PDL"));
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(1);
            cfg.blockDim = dim3(256);
            cfg.dynamicSmemBytes = std::max(kDiagSmem, diag_smem_req());
            cfg.stream = fs;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = pdl ? 1 : 0;
            float* lb = linv_blk(f, j);
            CUDA_THROW(cudaLaunchKernelEx(&cfg, chol_diag_kernel, f.a, f.ld, j, b, lb, err));
        }
        r.mark("ng_potrf_diag", l, static_cast<double>(b) * b * b / 3.0 * 2.0, fs);
        if (f.panel[blk].M > 0) {
            gemm_launch(f.panel[blk], fs);
            r.mark("ng_potrf_panel", l, 2.0 * f.panel[blk].M * f.panel[blk].N * f.panel[blk].K, fs);
        }
        if (conc) CUDA_THROW(cudaEventRecord(f.ev_panel[blk], fs));
        if (f.col[blk].M > 0) {
            if (conc && blk >= 1 && f.rest[blk - 1].M > 0) CUDA_THROW(cudaStreamWaitEvent(fs, f.ev_trail[blk - 1], 0));
            gemm_launch(f.col[blk], fs);
            r.mark("ng_potrf_trail", l, 2.0 * f.col[blk].M * f.col[blk].N * f.col[blk].K, fs);
        }
        if (f.rest[blk].M > 0) {
            if (conc) CUDA_THROW(cudaStreamWaitEvent(ts, f.ev_panel[blk], 0));
            // the bulk update's persistent grid leaves SMs free, so the chain's diag / panel /
            // look-ahead kernels never wait for one (13.39 -> 13.28 ms per config-2 step;
            // 2 / 4 / 16 free: 13.32-13.35 / 13.29-13.32 / 13.28-13.31)
            static const int rest_free = [] {
                const char* v = std::getenv("PARNN_NG_REST_FREE");
                return v ? std::atoi(v) : 8;
            }();
            if (rest_free > 0) gemm_set_grid_cap(r.ctx->num_sms - rest_free);
            gemm_launch(f.rest[blk], ts);
            if (rest_free > 0) gemm_set_grid_cap(0);
            r.mark("ng_potrf_trail", l, 1.0 * f.rest[blk].M * f.rest[blk].N * f.rest[blk].K, ts);
            if (conc) CUDA_THROW(cudaEventRecord(f.ev_trail[blk], ts));
        }
    }
    if (conc) {  // rejoin ts (graph capture requires every forked stream to join back)
        cudaEvent_t last = f.ev_trail.back();  // the last block never has a rest update
        CUDA_THROW(cudaEventRecord(last, ts));
        CUDA_THROW(cudaStreamWaitEvent(fs, last, 0));
    }
}

// Forward solve block by block, each block as soon as its column of L is final.
// In block pairs as well (ng_super() > 1): fdiag(i), the pair's small update of
// block i+1, fdiag(i+1), one K = 256 update of every row below the pair.
void solve_forward(NgFactor& f, NgSolve& sv, cudaStream_t s, bool conc) {
    const bool pairs = ng_super() > 1;
    const size_t nb = sv.fdiag.size();
    for (size_t i = 0; i < nb; ++i) {
        if (conc) CUDA_THROW(cudaStreamWaitEvent(s, f.ev_panel[i], 0));
        gemm_launch(sv.fdiag[i], s);
        if (pairs && i + 1 < nb) {
            gemm_launch(sv.fnext[i], s);
            if (conc) CUDA_THROW(cudaStreamWaitEvent(s, f.ev_panel[i + 1], 0));
            gemm_launch(sv.fdiag[i + 1], s);
            if (sv.fpair[i].M > 0) gemm_launch(sv.fpair[i], s);
            ++i;
            continue;
        }
        if (sv.fupd[i].M > 0) gemm_launch(sv.fupd[i], s);
    }
}

// Backward sweep in block pairs (ng_super() > 1): bdiag(i), the pair's small
// update of block i-1, bdiag(i-1), then ONE update of every row above the pair with
// K = 256 -- half as many of the large read-modify-writes of X.
void solve_backward(NgSolve& sv, cudaStream_t s) {
    const bool pairs = ng_super() > 1;
    for (long i = static_cast<long>(sv.bdiag.size()) - 1; i >= 0; --i) {
        gemm_launch(sv.bdiag[i], s);
        if (pairs && i >= 1) {
            gemm_launch(sv.bnext[i], s);
            gemm_launch(sv.bdiag[i - 1], s);
            if (sv.bpair[i].M > 0) gemm_launch(sv.bpair[i], s);
            --i;
            continue;
        }
        if (sv.bupd[i].M > 0) gemm_launch(sv.bupd[i], s);
    }
}

void sumsq(const float* x, long ld, long rows, long cols, double* part, double* out, cudaStream_t s) {
    const int g = 296;
    sumsq_partial_kernel<<<g, 256, 0, s>>>(x, ld, rows, cols, part);
    sum_final_kernel<<<1, 256, 0, s>>>(part, g, out);
}

}  // namespace

void ng_alloc(Replica& r) {
    r.ngl.assign(r.L, NgLayer());
    for (int l = 0; l < r.L; ++l) {
        NgLayer& g = r.ngl[l];
        const long din = r.dims[l], dout = r.dims[l + 1];
        for (auto [f, n] : {std::pair<NgFactor*, long>{&g.out, dout}, {&g.in, din}}) {
            f->n = n;
            f->ld = pad32(n);
            f->a = dalloc_f(n * f->ld);
            f->linv = dalloc_f(((n + NB - 1) / NB) * NB * NB);
        }
        g.ldt = pad32(din + 1);
        g.ld2 = pad32(dout);
        g.t1 = dalloc_f(dout * g.ldt);
        g.t2 = dalloc_f(din * g.ld2);
        CUDA_THROW(cudaMalloc(&g.part, 512 * sizeof(double)));
        // Stream priorities: each factor's diag -> panel -> look-ahead chain high, the
        // layer's chain (moments, solves, update) and the bulk trailing updates low.
        // Measured on the config-2 kron step: 14.5 ms all equal, 13.35 ms this way,
        // 15.3 ms with the layer chains high as well (the 14 layer chains then
        // crowd the output factor's critical chain). PARNN_NG_PRIO=0: all low.
        static const int lprio = [] {
            const char* v = std::getenv("PARNN_NG_PRIO");
            return v ? std::atoi(v) : 2;
        }();
        g.stream = lprio == 1 ? make_stream(0) : make_stream(2);
        CUDA_THROW(cudaEventCreateWithFlags(&g.done, cudaEventDisableTiming));
        CUDA_THROW(cudaEventCreateWithFlags(&g.ev_ready, cudaEventDisableTiming));
        CUDA_THROW(cudaEventCreateWithFlags(&g.ev_in_done, cudaEventDisableTiming));
        for (NgFactor* f : {&g.out, &g.in}) {
            const bool prio = lprio != 0;
            f->fs = prio ? make_stream(0) : make_stream(2);
            f->ts = make_stream(2);
            const long nb = (f->n + NB - 1) / NB;
            f->ev_panel.resize(nb);
            f->ev_trail.resize(nb);
            for (long i = 0; i < nb; ++i) {
                CUDA_THROW(cudaEventCreateWithFlags(&f->ev_panel[i], cudaEventDisableTiming));
                CUDA_THROW(cudaEventCreateWithFlags(&f->ev_trail[i], cudaEventDisableTiming));
            }
        }
    }
    CUDA_THROW(cudaEventCreateWithFlags(&r.ng_fork, cudaEventDisableTiming));
}

void ng_free(Replica& r) {
    for (NgLayer& g : r.ngl) {
        for (float* p : {g.out.a, g.out.linv, g.in.a, g.in.linv, g.t1, g.t2})
            if (p) cudaFree(p);
        if (g.part) cudaFree(g.part);
        if (g.stream) cudaStreamDestroy(g.stream);
        for (cudaEvent_t e : {g.done, g.ev_ready, g.ev_in_done})
            if (e) cudaEventDestroy(e);
        for (NgFactor* f : {&g.out, &g.in}) {
            for (cudaEvent_t e : f->ev_panel) cudaEventDestroy(e);
            for (cudaEvent_t e : f->ev_trail) cudaEventDestroy(e);
            if (f->fs) cudaStreamDestroy(f->fs);
            if (f->ts) cudaStreamDestroy(f->ts);
        }
    }
    if (r.ng_fork) cudaEventDestroy(r.ng_fork);
    r.ng_fork = nullptr;
    r.ngl.clear();
}

void ng_build_plans(Replica& r) {
    const int sms = r.ctx->num_sms;
    ensure_diag_attr();  // function attributes may not be set while a graph is being captured
    for (int l = 0; l < r.L; ++l) {
        NgLayer& g = r.ngl[l];
        build_factor(g.out, sms);
        build_factor(g.in, sms);
        build_solve(g.out, g.solve_out, g.t1, g.ldt, r.dims[l] + 1, sms);
        build_solve(g.in, g.solve_in, g.t2, g.ld2, r.dims[l + 1], sms);
    }
}

// ng_precondition (optimizer.cpp:123-157) for layer l: G is in r.grads (W part
// [dout x ldw], bias at b_off); leaves Ghat^T in t2, bhat in t1[:, din] and
// the four norms in r.scal. Runs on stream s; unless a profile is being taken
// the two factorizations fork onto their own streams and the forward S_out
// solve trails the S_out factorization block by block.
void ng_precondition_layer(Replica& r, int l, cudaStream_t s) {
    NgLayer& g = r.ngl[l];
    const bool conc = r.prof == nullptr;
    const long din = r.dims[l], dout = r.dims[l + 1];
    double* sc = r.scal + 16 * l;  // [0..3] norms, [4] lambda_in, [5] lambda_out
    double* part = g.part;
    float* gw = r.grads + r.w_off[l];
    float* gb = r.grads + r.b_off[l];
    const double fo = static_cast<double>(dout), fi = static_cast<double>(din);

    trace_lambda_kernel<<<1, 256, 0, s>>>(r.r_in[l], din, g.in.ld, r.ng_smoothing, sc + 4);
    trace_lambda_kernel<<<1, 256, 0, s>>>(r.r_out[l], dout, g.out.ld, r.ng_smoothing, sc + 5);
    shift_copy_kernel<<<grid_for(dout * g.out.ld), 256, 0, s>>>(r.r_out[l], dout, g.out.ld, sc + 5, g.out.a);
    shift_copy_kernel<<<grid_for(din * g.in.ld), 256, 0, s>>>(r.r_in[l], din, g.in.ld, sc + 4, g.in.a);
    r.mark("ng_smooth", l, 0, s);
    if (conc) {
        CUDA_THROW(cudaEventRecord(g.ev_ready, s));
        for (NgFactor* f : {&g.out, &g.in}) {
            CUDA_THROW(cudaStreamWaitEvent(f->fs, g.ev_ready, 0));
            CUDA_THROW(cudaStreamWaitEvent(f->ts, g.ev_ready, 0));
        }
        r.tmark("ready" + std::to_string(l), s);
        cholesky(r, l, g.out, r.d_err, g.out.fs, g.out.ts, true);
        r.tmark("fact_out" + std::to_string(l), g.out.fs);
        cholesky(r, l, g.in, r.d_err, g.in.fs, g.in.ts, true);
        r.tmark("fact_in" + std::to_string(l), g.in.fs);
        CUDA_THROW(cudaEventRecord(g.ev_in_done, g.in.fs));
    } else {
        cholesky(r, l, g.out, r.d_err, s, s, false);
        cholesky(r, l, g.in, r.d_err, s, s, false);
    }

    sumsq(gw, r.ldw[l], dout, din, part, sc + 0, s);
    sumsq(gb, 1, dout, 1, part, sc + 1, s);
    pack_rhs_kernel<<<grid_for(dout * g.ldt), 256, 0, s>>>(gw, r.ldw[l], gb, dout, din, g.t1, g.ldt);
    r.mark("ng_norms", l, 0, s);
    solve_forward(g.out, g.solve_out, s, conc);  // S_out^-1 [G | g_b], pipelined behind the factor
    if (conc) r.tmark("fsolve" + std::to_string(l), s);
    solve_backward(g.solve_out, s);
    if (conc) r.tmark("bsolve" + std::to_string(l), s);
    r.mark("ng_trsm", l, 2.0 * fo * fo * (fi + 1.0), s);
    {
        dim3 grid((din + 31) / 32, (dout + 31) / 32), block(32, 8);
        transpose_kernel<<<grid, block, 0, s>>>(g.t1, g.ldt, dout, din, g.t2, g.ld2);
    }
    r.mark("ng_transpose", l, 0, s);
    if (conc) CUDA_THROW(cudaStreamWaitEvent(s, g.ev_in_done, 0));
    solve_forward(g.in, g.solve_in, s, false);  // S_in^-1 (S_out^-1 G)^T
    solve_backward(g.solve_in, s);
    if (conc) r.tmark("insolve" + std::to_string(l), s);
    r.mark("ng_trsm", l, 2.0 * fi * fi * fo, s);
    sumsq(g.t2, g.ld2, din, dout, part, sc + 2, s);
    sumsq(g.t1 + din, g.ldt, dout, 1, part, sc + 3, s);
    r.mark("ng_norms", l, 0, s);
}

void ng_apply_update(Replica& r, int l, cudaStream_t s) {
    NgLayer& g = r.ngl[l];
    const long din = r.dims[l], dout = r.dims[l + 1];
    {
        dim3 grid((dout + 31) / 32, (din + 31) / 32), block(32, 8);
        transpose_kernel<<<grid, block, 0, s>>>(g.t2, g.ld2, din, dout, g.t1, g.ldt);
    }
    ng_update_kernel<<<grid_for(dout * din), 256, 0, s>>>(
        r.params + r.w_off[l], r.ldw[l], r.params + r.b_off[l], r.wshadow ? r.wshadow + r.w_off[l] : nullptr, g.t1,
        g.ldt, g.t1 + din, g.ldt, dout, din, r.scal + 16 * l, r.d_lr, r.d_step, r.d_flags, 2 * l);
    r.mark("ng_update", l, 0, s);
}

}  // namespace pnb
