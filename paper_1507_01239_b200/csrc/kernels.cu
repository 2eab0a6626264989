// HBM-bound helper kernels of the trainer step: minibatch gather, fused
// softmax + cross-entropy + (p - onehot), CE reduction, bias gradient with the
// fused SGD update, dtype conversion and the CV argmax.
#include <cfloat>

#include "runtime.h"

namespace pnb {

namespace {

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) {
    return v;
}
template <>
__device__ __forceinline__ float to_f<bf16>(bf16 v) {
    return __bfloat162float(v);
}

// Dataset::select / minibatches row gather (data.cpp:12-25, 185-203): one
// CTA per batch row, 16-byte vector copies (rows are 128-B aligned, zero padded).
// Row b of the batch <- dataset row rows[step * B + b] (Dataset::select,
// data.cpp:12-25). ones_col >= 0: that column of the output row is set to 1
// (the constant input whose dW column is the bias gradient, runtime.cu).
__global__ void gather_kernel(const uint4* __restrict__ x, long ldx_v, const int32_t* __restrict__ y,
                              const uint32_t* __restrict__ rows, const int* __restrict__ step, long B,
                              long nvec, uint4* __restrict__ out, long ldo_v, int32_t* __restrict__ yout,
                              long ones_col, int esz) {
    const long b = blockIdx.x;
    const long st = step ? *step : 0;
    const uint32_t src = rows[st * B + b];
    const uint4* xs = x + src * ldx_v;
    uint4* o = out + b * ldo_v;
    for (long j = threadIdx.x; j < nvec; j += blockDim.x) o[j] = xs[j];
    if (threadIdx.x == 0) yout[b] = y[src];
    if (ones_col >= 0) {
        __syncthreads();  // the vector holding column ones_col is written
        if (threadIdx.x == 0) {
            char* row = reinterpret_cast<char*>(o);
            if (esz == 4) reinterpret_cast<float*>(row)[ones_col] = 1.f;
            else reinterpret_cast<__nv_bfloat16*>(row)[ones_col] = __float2bfloat16_rn(1.f);
        }
    }
}

// column `col` of a [rows x ld] buffer (fp32 / bf16) <- 1
__global__ void fill_ones_column_kernel(void* buf, long ld, long rows, long col, int esz) {
    for (long r = blockIdx.x * (long)blockDim.x + threadIdx.x; r < rows; r += (long)gridDim.x * blockDim.x) {
        if (esz == 4) static_cast<float*>(buf)[r * ld + col] = 1.f;
        else static_cast<__nv_bfloat16*>(buf)[r * ld + col] = __float2bfloat16_rn(1.f);
    }
}

__device__ __forceinline__ float block_reduce_max(float v, float* sh) {
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffff, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        v = l < (blockDim.x >> 5) ? sh[l] : -FLT_MAX;
        for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffff, v, o));
        if (l == 0) sh[32] = v;
    }
    __syncthreads();
    v = sh[32];
    __syncthreads();
    return v;
}

__device__ __forceinline__ float block_reduce_sum(float v, float* sh) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        v = l < (blockDim.x >> 5) ? sh[l] : 0.f;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
        if (l == 0) sh[32] = v;
    }
    __syncthreads();
    v = sh[32];
    __syncthreads();
    return v;
}

// softmax_rows + cross_entropy + dz init (network.cpp:76-92, 145-160, 194-197):
// per row, max-subtracted softmax, CE_i = lse_i - z_{i,y}, dz = p - onehot.
// Register-resident variant (C <= 4 * 256 * kVec): one read of the row, float4
// loads, exp computed once.
constexpr int kVec = 12;
template <typename T>
__global__ void __launch_bounds__(256) softmax_ce_reg_kernel(const float* __restrict__ z, long ldz, long C,
                                                             const int32_t* __restrict__ y, T* __restrict__ dz,
                                                             long lddz, float* __restrict__ ce_rows) {
    __shared__ float sh[33];
    const long i = blockIdx.x;
    const float4* zr = reinterpret_cast<const float4*>(z + i * ldz);
    float4 v[kVec];
    float m = -FLT_MAX;
#pragma unroll
    for (int k = 0; k < kVec; ++k) {
        const long q = threadIdx.x + 256L * k, j = 4 * q;
        if (j + 3 < C) {
            v[k] = zr[q];
        } else {
            const float* s = z + i * ldz + j;
            v[k].x = j < C ? s[0] : -FLT_MAX;
            v[k].y = j + 1 < C ? s[1] : -FLT_MAX;
            v[k].z = j + 2 < C ? s[2] : -FLT_MAX;
            v[k].w = -FLT_MAX;
        }
        m = fmaxf(m, fmaxf(fmaxf(v[k].x, v[k].y), fmaxf(v[k].z, v[k].w)));
    }
    m = block_reduce_max(m, sh);
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < kVec; ++k) {
        v[k].x = expf(v[k].x - m);
        v[k].y = expf(v[k].y - m);
        v[k].z = expf(v[k].z - m);
        v[k].w = expf(v[k].w - m);
        s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
    }
    s = block_reduce_sum(s, sh);
    const float inv = 1.f / s;
    const int lab = y[i];
    T* dr = dz + i * lddz;
#pragma unroll
    for (int k = 0; k < kVec; ++k) {
        const long j = 4 * (threadIdx.x + 256L * k);
        float p[4] = {v[k].x * inv, v[k].y * inv, v[k].z * inv, v[k].w * inv};
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (j + e == lab) p[e] -= 1.f;
        if (j + 3 < C) {
            // one vector store per 4 outputs (rows are 64-byte aligned, j is a multiple of 4)
            if constexpr (sizeof(T) == 2) {
                const __nv_bfloat162 a = __floats2bfloat162_rn(p[0], p[1]), b = __floats2bfloat162_rn(p[2], p[3]);
                uint2 w;
                w.x = *reinterpret_cast<const unsigned*>(&a);
                w.y = *reinterpret_cast<const unsigned*>(&b);
                *reinterpret_cast<uint2*>(dr + j) = w;
            } else {
                *reinterpret_cast<float4*>(dr + j) = make_float4(p[0], p[1], p[2], p[3]);
            }
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (j + e < C) dr[j + e] = static_cast<T>(p[e]);
        }
    }
    if (threadIdx.x == 0) ce_rows[i] = logf(s) + m - z[i * ldz + lab];
}

template <typename T>
__global__ void softmax_ce_kernel(const float* __restrict__ z, long ldz, long C, const int32_t* __restrict__ y,
                                  T* __restrict__ dz, long lddz, float* __restrict__ ce_rows) {
    __shared__ float sh[33];
    const long i = blockIdx.x;
    const float* zr = z + i * ldz;
    float m = -FLT_MAX;
    for (long j = threadIdx.x; j < C; j += blockDim.x) m = fmaxf(m, zr[j]);
    m = block_reduce_max(m, sh);
    float s = 0.f;
    for (long j = threadIdx.x; j < C; j += blockDim.x) s += expf(zr[j] - m);
    s = block_reduce_sum(s, sh);
    const float inv = 1.f / s;
    const int lab = y[i];
    T* dr = dz + i * lddz;
    for (long j = threadIdx.x; j < C; j += blockDim.x) {
        float p = expf(zr[j] - m) * inv;
        if (j == lab) p -= 1.f;
        dr[j] = static_cast<T>(p);
    }
    if (threadIdx.x == 0) ce_rows[i] = logf(s) + m - zr[lab];
}

// Deterministic batch-mean CE into d_ce[*step]; optionally advances the step.
__global__ void ce_reduce_kernel(const float* __restrict__ ce_rows, long B, double* __restrict__ d_ce,
                                 int* __restrict__ step, int advance) {
    __shared__ double sh[256];
    double acc = 0.0;
    for (long i = threadIdx.x; i < B; i += blockDim.x) acc += ce_rows[i];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int st = *step;
        d_ce[st] = sh[0] / static_cast<double>(B);
        if (advance) *step = st + 1;
    }
}

// db = colsum(dz)/B (network.cpp:203-208); finite check (optimizer.cpp:26-28);
// SGD b -= lr*db (optimizer.cpp:32-34) when bias != null; db stored when gb != null.
// Column sums of dz (B x C): one block per 2 x 16-byte column vectors, 128 row lanes
// each keeping several 16-byte loads in flight, a fixed shuffle + shared-memory tree
// (deterministic). g = sum / B; SGD: bias -= lr g; NG: gb = g.
template <typename T>
__global__ void __launch_bounds__(256) bias_grad_kernel(const T* __restrict__ dz, long lddz, long B, long C,
                                                        float* __restrict__ bias, float* __restrict__ gb,
                                                        const float* __restrict__ lr, const int* __restrict__ step,
                                                        unsigned* __restrict__ flags, unsigned bit) {
    constexpr int VE = 16 / sizeof(T);
    __shared__ float red[8][2 * VE];
    const int t = threadIdx.x, cv = t & 1, rl = t >> 1;
    const long c0 = (blockIdx.x * 2L + cv) * VE;
    float acc[VE];
#pragma unroll
    for (int e = 0; e < VE; ++e) acc[e] = 0.f;
    if (c0 < C) {
        const T* p = dz + c0;
#pragma unroll 4
        for (long b = rl; b < B; b += 128) {
            const uint4 u = *reinterpret_cast<const uint4*>(p + b * lddz);
            const T* v = reinterpret_cast<const T*>(&u);
#pragma unroll
            for (int e = 0; e < VE; ++e) acc[e] += to_f<T>(v[e]);
        }
    }
#pragma unroll
    for (int o = 2; o < 32; o <<= 1)
#pragma unroll
        for (int e = 0; e < VE; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
    if ((t & 31) < 2)
#pragma unroll
        for (int e = 0; e < VE; ++e) red[t >> 5][cv * VE + e] = acc[e];
    __syncthreads();
    if (t < 2 * VE) {
        const long j = blockIdx.x * 2L * VE + t;
        if (j < C) {
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < 8; ++w) s += red[w][t];
            const float g = s * (1.f / static_cast<float>(B));
            if (!isfinite(g) && flags) atomicOr(flags, 1u << bit);
            if (gb) gb[j] = g;
            if (bias) bias[j] -= lr[step ? *step : 0] * g;
        }
    }
}

__global__ void f32_to_bf16_rows_kernel(const float* __restrict__ src, long ld, long rows, long cols,
                                        bf16* __restrict__ dst) {
    const long total = rows * ld;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const long c = i % ld;
        dst[i] = __float2bfloat16_rn(c < cols ? src[i] : 0.f);
    }
}

__global__ void argmax_correct_kernel(const float* __restrict__ z, long ldz, long C, const int32_t* __restrict__ y,
                                      unsigned long long* correct) {
    // accuracy (network.cpp:274-289): first maximum wins (strict >).
    __shared__ float sv[256];
    __shared__ int si[256];
    const long i = blockIdx.x;
    const float* zr = z + i * ldz;
    float best = -FLT_MAX;
    int bi = 0x7fffffff;
    for (long j = threadIdx.x; j < C; j += blockDim.x) {
        const float v = zr[j];
        if (v > best) { best = v; bi = (int)j; }
    }
    sv[threadIdx.x] = best;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if (threadIdx.x < o) {
            const float v2 = sv[threadIdx.x + o];
            const int i2 = si[threadIdx.x + o];
            if (v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 < si[threadIdx.x])) {
                sv[threadIdx.x] = v2;
                si[threadIdx.x] = i2;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && si[0] == y[i]) atomicAdd(correct, 1ull);
}

}  // namespace

void launch_gather(const void* x, long ldx, const int32_t* y, const uint32_t* rows, const int* step, long B, long d,
                   void* out, long ldo, int32_t* yout, bool f32, cudaStream_t s, long ones_col) {
    const long per = f32 ? 4 : 8;  // elements per uint4
    const long nvec = (pad32(d) + per - 1) / per;
    gather_kernel<<<B, 128, 0, s>>>(static_cast<const uint4*>(x), ldx / per, y, rows, step, B, nvec,
                                    static_cast<uint4*>(out), ldo / per, yout, ones_col, f32 ? 4 : 2);
}

void launch_fill_ones_column(void* buf, long ld, long rows, long col, bool f32, cudaStream_t s) {
    fill_ones_column_kernel<<<static_cast<int>(std::min<long>((rows + 255) / 256, 1024)), 256, 0, s>>>(
        buf, ld, rows, col, f32 ? 4 : 2);
}

void launch_softmax_ce(const float* z, long ldz, long B, long C, const int32_t* y, void* dz, long lddz,
                       float* ce_rows, bool f32, cudaStream_t s) {
    if (f32)
        if (C <= 4 * 256 * kVec)
            softmax_ce_reg_kernel<float><<<B, 256, 0, s>>>(z, ldz, C, y, static_cast<float*>(dz), lddz, ce_rows);
        else
            softmax_ce_kernel<float><<<B, 256, 0, s>>>(z, ldz, C, y, static_cast<float*>(dz), lddz, ce_rows);
    else
        if (C <= 4 * 256 * kVec)
            softmax_ce_reg_kernel<bf16><<<B, 256, 0, s>>>(z, ldz, C, y, static_cast<bf16*>(dz), lddz, ce_rows);
        else
            softmax_ce_kernel<bf16><<<B, 256, 0, s>>>(z, ldz, C, y, static_cast<bf16*>(dz), lddz, ce_rows);
}

void launch_ce_reduce(const float* ce_rows, long B, double* d_ce, int* step, int advance, cudaStream_t s) {
    ce_reduce_kernel<<<1, 256, 0, s>>>(ce_rows, B, d_ce, step, advance);
}

void launch_bias_grad(const void* dz, long lddz, long B, long C, bool f32, float* bias, float* gb, const float* lr,
                      const int* step, unsigned* flags, unsigned bit, cudaStream_t s) {
    const long cpb = 2 * (f32 ? 4 : 8);  // columns per block
    dim3 grid(static_cast<unsigned>((C + cpb - 1) / cpb)), block(256);
    if (f32)
        bias_grad_kernel<float><<<grid, block, 0, s>>>(static_cast<const float*>(dz), lddz, B, C, bias, gb, lr, step,
                                                       flags, bit);
    else
        bias_grad_kernel<bf16><<<grid, block, 0, s>>>(static_cast<const bf16*>(dz), lddz, B, C, bias, gb, lr, step,
                                                      flags, bit);
}

void launch_f32_to_bf16_rows(const float* src, long ld, long rows, long cols, bf16* dst, cudaStream_t s) {
    const long total = rows * ld;
    const int blocks = (int)std::min<long>((total + 255) / 256, 148L * 16);
    if (total > 0) f32_to_bf16_rows_kernel<<<blocks, 256, 0, s>>>(src, ld, rows, cols, dst);
}

void launch_convert_dataset(const float* x32, long n, long ld, bf16* x16, cudaStream_t s) {
    launch_f32_to_bf16_rows(x32, ld, n, ld, x16, s);
}

void launch_argmax_correct(const float* z, long ldz, long B, long C, const int32_t* y, unsigned long long* correct,
                           cudaStream_t s) {
    argmax_correct_kernel<<<B, 256, 0, s>>>(z, ldz, C, y, correct);
}

}  // namespace pnb
