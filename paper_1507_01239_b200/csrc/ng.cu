// NG-SGD, full Kronecker-factored variant (optimizer.cpp:108-157), on device
// in fp32 (SIMT FMA, fp32-accurate: SURVEY §7 "NG-SGD kron-full cost" rules
// out TF32-operand solves at kappa(S) ~ 1e2).
//
// Per layer: S = R + lambda I with lambda = max(alpha tr(R)/n, 1e-8)
// (smoothed_factor), blocked right-looking Cholesky of S_out and S_in
// (S_out factored ONCE; the reference re-factors it for the bias solve),
// Ghat = S_out^-1 [G | g_b] by blocked forward/back substitution, transpose,
// S_in^-1 on the weight part, transpose back, Frobenius rescale gamma and the
// fused SGD update (sgd_step_in_place) with the non-finite check.
#include <cfloat>

#include "runtime.h"

namespace pnb {

namespace {

constexpr int NB = 64;  // Cholesky / TRSM block

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

// S = R + lambda I (lower triangle incl. diagonal is all Cholesky reads).
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

// Unblocked Cholesky of the b x b diagonal block at (j, j), in shared memory.
__global__ void potrf_diag_kernel(float* __restrict__ a, long ld, long j, int b, DevErr* err) {
    __shared__ float t[NB][NB + 1];
    for (int idx = threadIdx.x; idx < b * b; idx += blockDim.x) {
        const int r = idx / b, c = idx % b;
        t[r][c] = a[(j + r) * ld + j + c];
    }
    __syncthreads();
    for (int k = 0; k < b; ++k) {
        if (threadIdx.x == 0) {
            const float piv = t[k][k];
            if (!(piv > 0.f) || !isfinite(piv)) {
                if (atomicCAS(&err->chol_failed, 0, 1) == 0) {
                    err->chol_index = static_cast<int>(j + k);
                    err->chol_value = piv;
                }
            }
            t[k][k] = sqrtf(piv);
        }
        __syncthreads();
        const float inv = 1.f / t[k][k];
        for (int r = k + 1 + threadIdx.x; r < b; r += blockDim.x) t[r][k] *= inv;
        __syncthreads();
        for (int idx = threadIdx.x; idx < (b - k - 1) * (b - k - 1); idx += blockDim.x) {
            const int r = k + 1 + idx / (b - k - 1), c = k + 1 + idx % (b - k - 1);
            if (c <= r) t[r][c] -= t[r][k] * t[c][k];
        }
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < b * b; idx += blockDim.x) {
        const int r = idx / b, c = idx % b;
        a[(j + r) * ld + j + c] = c <= r ? t[r][c] : 0.f;
    }
}

// Panel: rows [j+b, n) of columns [j, j+b): x L11^T = a  (forward substitution per row).
__global__ void trsm_panel_kernel(float* __restrict__ a, long ld, long j, int b, long n) {
    __shared__ float l11[NB][NB + 1];
    for (int idx = threadIdx.x; idx < b * b; idx += blockDim.x) {
        const int r = idx / b, c = idx % b;
        l11[r][c] = a[(j + r) * ld + j + c];
    }
    __syncthreads();
    const long row = j + b + blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (row >= n) return;
    float x[NB];
    float* ar = a + row * ld + j;
#pragma unroll
    for (int c = 0; c < NB; ++c) x[c] = c < b ? ar[c] : 0.f;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
        if (c < b) {
            float acc = x[c];
#pragma unroll
            for (int k = 0; k < NB; ++k)
                if (k < c) acc -= x[k] * l11[c][k];
            x[c] = acc / l11[c][c];
        }
    }
#pragma unroll
    for (int c = 0; c < NB; ++c)
        if (c < b) ar[c] = x[c];
}

// C[m, n] -= sum_k opA(m, k) * opB(k, n); opA = A[m*lda+k] (TA=0) or A[k*lda+m] (TA=1);
// opB = B[k*ldb+n] (TB=0) or B[n*ldb+k] (TB=1). LOWER: only tiles touching n <= m.
template <int TA, int TB, int LOWER>
__global__ void __launch_bounds__(256) gemm_sub_kernel(float* __restrict__ c, long ldc, const float* __restrict__ a,
                                                       long lda, const float* __restrict__ b, long ldb, long M, long N,
                                                       long K) {
    const long m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
    if (LOWER && n0 > m0 + 63) return;
    __shared__ float As[16][64 + 4];
    __shared__ float Bs[16][64 + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    float acc[4][4] = {};
    for (long k0 = 0; k0 < K; k0 += 16) {
        for (int idx = threadIdx.x; idx < 16 * 64; idx += 256) {
            int kk, mm;
            if (TA == 0) { kk = idx % 16; mm = idx / 16; } else { mm = idx % 64; kk = idx / 64; }
            const long gm = m0 + mm, gk = k0 + kk;
            float v = 0.f;
            if (gm < M && gk < K) v = TA == 0 ? a[gm * lda + gk] : a[gk * lda + gm];
            As[kk][mm] = v;
        }
        for (int idx = threadIdx.x; idx < 16 * 64; idx += 256) {
            int kk, nn;
            if (TB == 0) { nn = idx % 64; kk = idx / 64; } else { kk = idx % 16; nn = idx / 16; }
            const long gn = n0 + nn, gk = k0 + kk;
            float v = 0.f;
            if (gn < N && gk < K) v = TB == 0 ? b[gk * ldb + gn] : b[gn * ldb + gk];
            Bs[kk][nn] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            float av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int i = 0; i < 4; ++i) bv[i] = Bs[kk][tx * 4 + i];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[i][q] = fmaf(av[i], bv[q], acc[i][q]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const long gm = m0 + ty * 4 + i;
        if (gm >= M) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long gn = n0 + tx * 4 + q;
            if (gn < N && (!LOWER || gn <= gm)) c[gm * ldc + gn] -= acc[i][q];
        }
    }
}

// X_i = L_ii^-1 X_i (FWD) or L_ii^-T X_i (!FWD) for rows [i0, i0+b) of X, one thread per column.
template <int FWD>
__global__ void trsv_block_kernel(const float* __restrict__ l, long ld, long i0, int b, float* __restrict__ x,
                                  long ldx, long ncols) {
    __shared__ float t[NB][NB + 1];
    for (int idx = threadIdx.x; idx < b * b; idx += blockDim.x) {
        const int r = idx / b, c = idx % b;
        t[r][c] = l[(i0 + r) * ld + i0 + c];
    }
    __syncthreads();
    const long col = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (col >= ncols) return;
    float v[NB];
#pragma unroll
    for (int r = 0; r < NB; ++r) v[r] = r < b ? x[(i0 + r) * ldx + col] : 0.f;
    if (FWD) {
#pragma unroll
        for (int r = 0; r < NB; ++r) {
            if (r < b) {
                float acc = v[r];
#pragma unroll
                for (int k = 0; k < NB; ++k)
                    if (k < r) acc -= t[r][k] * v[k];
                v[r] = acc / t[r][r];
            }
        }
    } else {
#pragma unroll
        for (int r = NB - 1; r >= 0; --r) {
            if (r < b) {
                float acc = v[r];
#pragma unroll
                for (int k = 0; k < NB; ++k)
                    if (k > r && k < b) acc -= t[k][r] * v[k];
                v[r] = acc / t[r][r];
            }
        }
    }
#pragma unroll
    for (int r = 0; r < NB; ++r)
        if (r < b) x[(i0 + r) * ldx + col] = v[r];
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

// W -= lr * gamma * Ghat (transposed back from th [d_in x ldth]); b -= lr * gamma_b * bhat.
// scal: [0] |G|^2, [1] |g_b|^2, [2] |Ghat|^2, [3] |bhat|^2 (optimizer.cpp:142-154).
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

void cholesky(float* a, long n, long ld, DevErr* err, cudaStream_t s) {
    for (long j = 0; j < n; j += NB) {
        const int b = (int)std::min<long>(NB, n - j);
        potrf_diag_kernel<<<1, 256, 0, s>>>(a, ld, j, b, err);
        const long rest = n - j - b;
        if (rest <= 0) break;
        trsm_panel_kernel<<<(rest + 127) / 128, 128, 0, s>>>(a, ld, j, b, n);
        dim3 grid((rest + 63) / 64, (rest + 63) / 64);
        gemm_sub_kernel<0, 1, 1><<<grid, 256, 0, s>>>(a + (j + b) * ld + (j + b), ld, a + (j + b) * ld + j, ld,
                                                        a + (j + b) * ld + j, ld, rest, rest, b);
    }
}

// X <- L^-1 X then X <- L^-T X  (X is n x ncols, ld ldx): S^-1 X via the factor.
void chol_solve(const float* l, long n, long ld, float* x, long ldx, long ncols, cudaStream_t s) {
    const int tb = 128;
    const int gcols = (int)((ncols + tb - 1) / tb);
    for (long i0 = 0; i0 < n; i0 += NB) {
        const int b = (int)std::min<long>(NB, n - i0);
        trsv_block_kernel<1><<<gcols, tb, 0, s>>>(l, ld, i0, b, x, ldx, ncols);
        const long rest = n - i0 - b;
        if (rest > 0) {
            dim3 grid((ncols + 63) / 64, (rest + 63) / 64);
            gemm_sub_kernel<0, 0, 0><<<grid, 256, 0, s>>>(x + (i0 + b) * ldx, ldx, l + (i0 + b) * ld + i0, ld,
                                                            x + i0 * ldx, ldx, rest, ncols, b);
        }
    }
    const long last = ((n - 1) / NB) * NB;
    for (long i0 = last; i0 >= 0; i0 -= NB) {
        const int b = (int)std::min<long>(NB, n - i0);
        trsv_block_kernel<0><<<gcols, tb, 0, s>>>(l, ld, i0, b, x, ldx, ncols);
        if (i0 > 0) {
            dim3 grid((ncols + 63) / 64, (i0 + 63) / 64);
            // X[0:i0] -= L[i0:i0+b, 0:i0]^T X[i0:i0+b]
            gemm_sub_kernel<1, 0, 0><<<grid, 256, 0, s>>>(x, ldx, l + i0 * ld, ld, x + i0 * ldx, ldx, i0, ncols, b);
        }
    }
}

void sumsq(const float* x, long ld, long rows, long cols, double* part, double* out, cudaStream_t s) {
    const int g = 296;
    sumsq_partial_kernel<<<g, 256, 0, s>>>(x, ld, rows, cols, part);
    sum_final_kernel<<<1, 256, 0, s>>>(part, g, out);
}

}  // namespace

// ng_precondition (optimizer.cpp:123-157) for layer l of replica r; the
// gradient is in r.grads (W part [dout x ldw], bias part at b_off); writes the
// preconditioned direction into r.tbuf (transposed back) and scalars in r.scal.
void ng_precondition_layer(Replica& r, int l, cudaStream_t s) {
    const long din = r.dims[l], dout = r.dims[l + 1];
    const long ldi = pad32(din), ldo = pad32(dout);
    double* sc = r.scal + 16 * l;  // [0..3] norms, [4] lambda_in, [5] lambda_out
    double* part = r.scal + 16 * r.L;
    float* g = r.grads + r.w_off[l];
    float* gb = r.grads + r.b_off[l];
    const long ldt = pad32(din + 1);
    float* t1 = r.tbuf;                      // [dout x ldt] = [G | g_b]
    float* t2 = r.tbuf + dout * ldt;         // [din x ldo]  = transposed weight part

    // smoothed_factor: lambda = max(alpha tr(R)/n, 1e-8)
    trace_lambda_kernel<<<1, 256, 0, s>>>(r.r_in[l], din, ldi, r.ng_smoothing, sc + 4);
    trace_lambda_kernel<<<1, 256, 0, s>>>(r.r_out[l], dout, ldo, r.ng_smoothing, sc + 5);
    shift_copy_kernel<<<grid_for(dout * ldo), 256, 0, s>>>(r.r_out[l], dout, ldo, sc + 5, r.chol_a);
    shift_copy_kernel<<<grid_for(din * ldi), 256, 0, s>>>(r.r_in[l], din, ldi, sc + 4, r.chol_b);
    r.mark("ng_smooth", l, 0, s);
    const double fo = static_cast<double>(dout), fi = static_cast<double>(din);
    cholesky(r.chol_a, dout, ldo, r.d_err, s);
    r.mark("ng_potrf", l, fo * fo * fo / 3.0, s);
    cholesky(r.chol_b, din, ldi, r.d_err, s);
    r.mark("ng_potrf", l, fi * fi * fi / 3.0, s);

    sumsq(g, r.ldw[l], dout, din, part, sc + 0, s);
    sumsq(gb, 1, dout, 1, part, sc + 1, s);
    pack_rhs_kernel<<<grid_for(dout * ldt), 256, 0, s>>>(g, r.ldw[l], gb, dout, din, t1, ldt);
    r.mark("ng_norms", l, 0, s);
    chol_solve(r.chol_a, dout, ldo, t1, ldt, din + 1, s);  // S_out^-1 [G | g_b]
    r.mark("ng_trsm", l, 2.0 * fo * fo * (fi + 1.0), s);
    {
        dim3 grid((din + 31) / 32, (dout + 31) / 32), block(32, 8);
        transpose_kernel<<<grid, block, 0, s>>>(t1, ldt, dout, din, t2, ldo);
    }
    r.mark("ng_transpose", l, 0, s);
    chol_solve(r.chol_b, din, ldi, t2, ldo, dout, s);  // S_in^-1 (S_out^-1 G)^T
    r.mark("ng_trsm", l, 2.0 * fi * fi * fo, s);
    sumsq(t2, ldo, din, dout, part, sc + 2, s);
    sumsq(t1 + din, ldt, dout, 1, part, sc + 3, s);
    r.mark("ng_norms", l, 0, s);
}

void ng_apply_update(Replica& r, int l, cudaStream_t s) {
    const long din = r.dims[l], dout = r.dims[l + 1];
    const long ldt = pad32(din + 1);
    float* t1 = r.tbuf;
    float* t2 = r.tbuf + dout * ldt;
    // Ghat^T is t2 [din x ldo]; transpose back into t1's weight columns.
    {
        dim3 grid((dout + 31) / 32, (din + 31) / 32), block(32, 8);
        transpose_kernel<<<grid, block, 0, s>>>(t2, pad32(dout), din, dout, t1, ldt);
    }
    ng_update_kernel<<<grid_for(dout * din), 256, 0, s>>>(
        r.params + r.w_off[l], r.ldw[l], r.params + r.b_off[l], r.wshadow ? r.wshadow + r.w_off[l] : nullptr, t1,
        ldt, t1 + din, ldt, dout, din, r.scal + 16 * l, r.d_lr, r.d_step, r.d_flags, 2 * l);
    r.mark("ng_update", l, 0, s);
}

}  // namespace pnb
