// tcgen05 / TMEM / TMA GEMM for sm_100a with the trainer's fused epilogues.
//
//   D[m, n] = sum_k A(m, k) * B(n, k)          (fp32 accumulate in TMEM)
//
// A and B are row-major device buffers read by TMA in either of two
// orientations (template flags):
//   K-major : the buffer is [rows x K] with K contiguous   (box {128 B, rows})
//   MN-major: the buffer is [K x rows] with rows contiguous (box {128 B, BK})
// which covers every product of the path without transposed copies
// (SURVEY §7 "Operand majors"):
//   forward  Z  = A_prev . W^T      A K-major,  B K-major   (network.cpp:94-101)
//   dW       G  = dz^T . A_prev     A MN-major, B MN-major  (network.cpp:201-202)
//   dA       dA = dz . W            A K-major,  B MN-major  (network.cpp:214)
//   moments  C  = X^T . X           A MN-major, B MN-major  (optimizer.cpp:97-100)
//
// Operands are BF16 (kind::f16) or FP32 read as TF32 (kind::tf32). One CTA
// computes one 128 x BN tile: warp 0 lane 0 issues TMA into a STAGES-deep
// smem ring, warp 1 lane 0 issues tcgen05.mma (128 x BN x 16|8) into TMEM,
// then all four warps drain TMEM (tcgen05.ld 32x32b) through the epilogue.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <type_traits>

#include "ptx.cuh"

namespace pnb {

#ifdef PNB_GEMM_TRACE
// per-CTA %globaltimer stamps: entry, setup done, first operands in smem,
// last MMA issued, accumulator ready, epilogue done, exit
__device__ unsigned long long g_gemm_trace[1024][12];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define PNB_TRACE(i) g_gemm_trace[blockIdx.x][i] = gtime()
#else
#define PNB_TRACE(i) \
    do {             \
    } while (0)
#endif

enum EpiMode : int {
    EPI_FWD_ACT = 0,     // out(T)   = act(acc + bias[n])
    EPI_FWD_LINEAR = 1,  // out32    = acc + bias[n]
    EPI_GRAD = 2,        // out32    = alpha * acc            (+ finite flag)
    EPI_GRAD_SGD = 3,    // g = alpha*acc; W32 -= lr*g; shadow = bf16(W32)  (+ flag)
    EPI_ACTGRAD = 4,     // out(T)   = acc * act'(aux[m, n])
    EPI_EMA = 5,         // out32    = beta * out32 + alpha * acc
    EPI_AXPY = 6,        // out32   += alpha * acc; shadow = bf16(out32)   (CD-1 update)
    EPI_SUB = 7,         // out32   -= acc      (blocked Cholesky / TRSM updates)
    EPI_PARTIAL = 8,     // out32[ks * split_stride + ...] = acc   (split-K partial products)
    EPI_RESID = 9,       // out(T)   = aux(T) - acc; per-CTA sums of aux^2, out^2 -> part
};

struct GemmEpi {
    int mode = 0;
    int act = 0;  // 0 sigmoid, 1 tanh (network.cpp:64-73), 2 identity
    float out_scale = 1.f;  // FWD_ACT: multiplies the activated value (CD-1 stores -neg)
    void* out = nullptr;  // T-typed output (FWD_ACT, ACTGRAD)
    long ld_out = 0;
    float* out32 = nullptr;  // fp32 output / master params (FWD_LINEAR, GRAD, GRAD_SGD, EMA)
    long ld_out32 = 0;
    __nv_bfloat16* shadow = nullptr;  // bf16 operand shadow of out32 (GRAD_SGD, bf16 mode)
    long ld_shadow = 0;
    const float* bias = nullptr;
    const void* aux = nullptr;  // T-typed activations for ACTGRAD
    long ld_aux = 0;
    float alpha = 1.f;
    float beta = 0.f;
    const float* coef = nullptr;  // EMA: device {beta, alpha} overriding the scalars
    const float* lr = nullptr;  // device scalar array indexed by *step
    const int* step = nullptr;
    unsigned* flag = nullptr;  // bit `flag_bit` set on a non-finite gradient
    unsigned flag_bit = 0;
    int lower = 0;  // skip tiles strictly above the diagonal (SYRK-style updates)
    // GRAD_SGD extras (NG low-rank): alpha *= (*gscale_a) * (*gscale_b) (the two
    // sides' gamma), and output column bias_col is the bias gradient -> bias32[row]
    const double* gscale_a = nullptr;
    const double* gscale_b = nullptr;
    int bias_col = -1;
    float* bias32 = nullptr;
    int ksplit = 1;         // split-K factor (set by gemm_plan; every split non-empty)
    long split_stride = 0;  // PARTIAL: floats between the per-split outputs
    double* part = nullptr; // RESID: [gridDim.x][2] per-CTA {sum aux^2, sum out^2}
};

// Kernel parameters: NP problems (1, or up to kGroupMax for a grouped launch).
// Problem p owns the global tiles [tile0[p], tile0[p+1]).
constexpr int kGroupMax = 8;
template <int NP>
struct GemmParams {
    CUtensorMap ta[NP];
    CUtensorMap tb[NP];
    GemmEpi ep[NP];
    int M[NP], N[NP], K[NP];
    int tile0[NP + 1];
    int np;
};

template <typename T>
struct OpTraits;
template <>
struct OpTraits<__nv_bfloat16> {
    static constexpr bool kTf32 = false;
    static constexpr uint32_t kFmt = 1;
};
template <>
struct OpTraits<float> {
    static constexpr bool kTf32 = true;
    static constexpr uint32_t kFmt = 2;
};

// sigmoid on the MUFU path: 1 / (1 + 2^(-z log2 e)) with ex2.approx and
// rcp.approx (~2 ulp). The .ftz forms skip the denormal range fix-up that
// __expf adds (an e^-z below 2^-126 leaves 1 + e^-z == 1 either way).
__device__ __forceinline__ float sigmoid_fast(float z) {
    float t, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(-1.4426950408889634f * z));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.f + t));
    return r;
}
// ACT: 0 sigmoid, 1 tanh (the accurate tanhf: its 1 - 2/(1+e^2z) form cancels
// near 0), 2 identity. Compile-time, so the epilogue loops over a chunk's 32
// values carry no per-element branch and the MUFU chains interleave.
template <int ACT>
__device__ __forceinline__ float act_fwd_t(float z) {
    if constexpr (ACT == 0) return sigmoid_fast(z);
    else if constexpr (ACT == 1) return tanhf(z);
    else return z;
}
template <int ACT>
__device__ __forceinline__ float act_grad_t(float a) {
    if constexpr (ACT == 0) return a * (1.f - a);
    else return 1.f - a * a;
}
__device__ __forceinline__ float act_fwd(int act, float z) {
    return act == 0 ? act_fwd_t<0>(z) : (act == 1 ? act_fwd_t<1>(z) : z);
}
__device__ __forceinline__ float act_grad(int act, float a) {
    return act == 0 ? act_grad_t<0>(a) : act_grad_t<1>(a);
}
// apply f<ACT>(i) for the runtime activation with the switch outside the loop
template <typename F>
__device__ __forceinline__ void with_act(int act, F&& f) {
    if (act == 0) f(std::integral_constant<int, 0>{});
    else if (act == 1) f(std::integral_constant<int, 1>{});
    else f(std::integral_constant<int, 2>{});
}

template <typename T>
__device__ __forceinline__ float ld_as_float(const T* p);
template <>
__device__ __forceinline__ float ld_as_float<float>(const float* p) {
    return *p;
}
template <>
__device__ __forceinline__ float ld_as_float<__nv_bfloat16>(const __nv_bfloat16* p) {
    return __bfloat162float(*p);
}
template <typename T>
__device__ __forceinline__ void st_from_float(T* p, float v);
template <>
__device__ __forceinline__ void st_from_float<float>(float* p, float v) {
    *p = v;
}
template <>
__device__ __forceinline__ void st_from_float<__nv_bfloat16>(__nv_bfloat16* p, float v) {
    *p = __float2bfloat16_rn(v);
}

// PP "pieces" of a lane in the transposed epilogue layout: four consecutive
// values (columns c .. c+3, nvc of them valid) of rows rb, rb+4, ... (valid
// while < M), at base + row * ld. Whole aligned pieces move as one 16-byte
// (fp32) / 8-byte (bf16) access; all loads of a call are issued before any of
// their values is used. Partial pieces (matrix edges) go element-wise.
template <typename T>
__device__ __forceinline__ bool pieces_vec(const T* base, long ld, int nvc) {
    return nvc == 4 && ((reinterpret_cast<uintptr_t>(base) | static_cast<uintptr_t>(ld * sizeof(T))) &
                        (4 * sizeof(T) - 1)) == 0;
}

template <typename T, int PP>
__device__ __forceinline__ void load_pieces(const T* base, long ld, int rb, int M, int nvc, float (&x)[PP][4]) {
    if (pieces_vec(base, ld, nvc)) {
        if constexpr (sizeof(T) == 4) {
            float4 u[PP];
#pragma unroll
            for (int i = 0; i < PP; ++i)
                u[i] = rb + 4 * i < M ? *reinterpret_cast<const float4*>(base + static_cast<long>(rb + 4 * i) * ld)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int i = 0; i < PP; ++i) {
                x[i][0] = u[i].x; x[i][1] = u[i].y; x[i][2] = u[i].z; x[i][3] = u[i].w;
            }
        } else {
            uint2 u[PP];
#pragma unroll
            for (int i = 0; i < PP; ++i)
                u[i] = rb + 4 * i < M ? *reinterpret_cast<const uint2*>(base + static_cast<long>(rb + 4 * i) * ld)
                                      : make_uint2(0u, 0u);
#pragma unroll
            for (int i = 0; i < PP; ++i) {
                const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u[i].x));
                const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u[i].y));
                x[i][0] = lo.x; x[i][1] = lo.y; x[i][2] = hi.x; x[i][3] = hi.y;
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < PP; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e)
                x[i][e] = (rb + 4 * i < M && e < nvc) ? ld_as_float<T>(base + static_cast<long>(rb + 4 * i) * ld + e)
                                                      : 0.f;
    }
}

template <typename T, int PP>
__device__ __forceinline__ void store_pieces(T* base, long ld, int rb, int M, int nvc, const float (&x)[PP][4]) {
    if (pieces_vec(base, ld, nvc)) {
#pragma unroll
        for (int i = 0; i < PP; ++i) {
            if (rb + 4 * i >= M) continue;
            T* p = base + static_cast<long>(rb + 4 * i) * ld;
            if constexpr (sizeof(T) == 4) {
                *reinterpret_cast<float4*>(p) = make_float4(x[i][0], x[i][1], x[i][2], x[i][3]);
            } else {
                __nv_bfloat162 lo = __floats2bfloat162_rn(x[i][0], x[i][1]);
                __nv_bfloat162 hi = __floats2bfloat162_rn(x[i][2], x[i][3]);
                *reinterpret_cast<uint2*>(p) =
                    make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < PP; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (rb + 4 * i < M && e < nvc) st_from_float<T>(base + static_cast<long>(rb + 4 * i) * ld + e, x[i][e]);
    }
}

template <int BN, int STAGES, typename T, bool SPLIT = false, bool TE = true>
struct GemmSmem {
    static constexpr int kElem = sizeof(T);
    static constexpr int kBK = 128 / kElem;    // K per stage (one 128-B swizzle row)
    static constexpr int kUK = 32 / kElem;     // K per tcgen05.mma
    static constexpr int kAtom = 128 / kElem;  // MN elements per 128-B atom
    static constexpr int kABytes = 128 * 128;
    static constexpr int kBBytes = BN * 128;
    static constexpr int kLoad = kABytes + kBBytes;          // bytes TMA brings per stage
    static constexpr int kStage = kLoad * (SPLIT ? 2 : 1);   // + low-part copies for 3xTF32
    static constexpr int kEpiBuf = TE ? 8 * 32 * 32 * 4 : 0; // per epilogue warp: one 32 x 32 fp32 chunk
    static constexpr int kBytes = STAGES * kStage + 1024 /*align*/ + 512 /*barriers*/ + kEpiBuf;
    static constexpr int kThreads = SPLIT ? 448 : 320;       // TMA, MMA, 8 epilogue (+ 4 splitter) warps
    static constexpr uint32_t kTmemCols = 2 * BN;            // double-buffered accumulator
};

// Epilogue of one 32 x 32 accumulator chunk: rows r0 .. r0+31 (one TMEM lane
// quadrant), columns n .. n+31. tcgen05.ld gives one row per lane; the chunk
// is transposed through the warp's 4 KB buffer (16-byte slots XOR-swizzled by
// row: conflict-free both ways) so that lane l then owns columns
// c = n + 4 (l & 7) .. c+3 of rows r0 + 4 i + (l >> 3), i = 0..7. Every global
// access instruction of the warp then covers 4 rows x 128 B (fp32) / 64 B
// (bf16) instead of touching 32 rows, and each lane keeps 8 independent
// accesses in flight (all loads are issued before the first store).
template <typename T, int PP>
__device__ __forceinline__ bool epilogue_chunk(const GemmEpi& ep, const uint32_t (&r)[32], uint4* buf, int lane,
                                               int r0, int M, int n, int N, float lr, float alpha_eff, int ks,
                                               float& s_aux, float& s_out) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
        sts128(buf + lane * 8 + (k ^ (lane & 7)), make_uint4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]));
    __syncwarp();
    const int kk = lane & 7, rs = lane >> 3;
    const int c = n + 4 * kk;
    const int nvc = min(max(N - c, 0), 4);
    bool bad = false;
#pragma unroll
    for (int p0 = 0; p0 < 8; p0 += PP) {  // PP pieces per pass (register budget)
    float a[PP][4];
#pragma unroll
    for (int i = 0; i < PP; ++i) {
        const int rr = 4 * (p0 + i) + rs;
        const uint4 u = lds128(buf + rr * 8 + (kk ^ (rr & 7)));
        a[i][0] = __uint_as_float(u.x); a[i][1] = __uint_as_float(u.y);
        a[i][2] = __uint_as_float(u.z); a[i][3] = __uint_as_float(u.w);
    }
    // row of piece i and its valid column count (computed, not kept in registers)
    const int rb = r0 + rs + 4 * p0;

    switch (ep.mode) {
        case EPI_PARTIAL: {
            store_pieces<float, PP>(ep.out32 + ks * ep.split_stride + c, ep.ld_out32, rb, M, nvc, a);
            break;
        }
        case EPI_RESID: {
            float x[PP][4];
            load_pieces<T, PP>(static_cast<const T*>(ep.aux) + c, ep.ld_aux, rb, M, nvc, x);
#pragma unroll
            for (int i = 0; i < PP; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    float v = x[i][e] - a[i][e];
                    if constexpr (sizeof(T) == 2) v = __bfloat162float(__float2bfloat16_rn(v));  // as stored
                    a[i][e] = v;
                    s_aux = fmaf(x[i][e], x[i][e], s_aux);  // invalid elements: x = acc = 0
                    s_out = fmaf(v, v, s_out);
                }
            store_pieces<T, PP>(static_cast<T*>(ep.out) + c, ep.ld_out, rb, M, nvc, a);
            break;
        }
        case EPI_FWD_ACT: {
            float b[1][4];
            load_pieces<float, 1>(ep.bias + c, 0, 0, 1, nvc, b);
            with_act(ep.act, [&](auto A) {
#pragma unroll
                for (int i = 0; i < PP; ++i)
#pragma unroll
                    for (int e = 0; e < 4; ++e) a[i][e] = ep.out_scale * act_fwd_t<A.value>(a[i][e] + b[0][e]);
            });
            store_pieces<T, PP>(static_cast<T*>(ep.out) + c, ep.ld_out, rb, M, nvc, a);
            break;
        }
        case EPI_FWD_LINEAR: {
            float b[1][4];
            load_pieces<float, 1>(ep.bias + c, 0, 0, 1, nvc, b);
#pragma unroll
            for (int i = 0; i < PP; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) a[i][e] += b[0][e];
            store_pieces<float, PP>(ep.out32 + c, ep.ld_out32, rb, M, nvc, a);
            break;
        }
        case EPI_GRAD: {
#pragma unroll
            for (int i = 0; i < PP; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    a[i][e] *= ep.alpha;
                    bad |= (e < nvc && rb + 4 * i < M) && !isfinite(a[i][e]);
                }
            store_pieces<float, PP>(ep.out32 + c, ep.ld_out32, rb, M, nvc, a);
            break;
        }
        case EPI_GRAD_SGD: {
            const int bj = ep.bias_col - c;  // bias column among this lane's four?
            const bool has_b = bj >= 0 && bj < nvc;
            const int nw = has_b ? bj : nvc;
            float w[PP][4];
            load_pieces<float, PP>(ep.out32 + c, ep.ld_out32, rb, M, nw, w);
#pragma unroll
            for (int i = 0; i < PP; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float g = a[i][e] * alpha_eff;
                    bad |= (e < nw && rb + 4 * i < M) && !isfinite(g);
                    w[i][e] -= lr * g;
                }
            store_pieces<float, PP>(ep.out32 + c, ep.ld_out32, rb, M, nw, w);
            if (ep.shadow) store_pieces<__nv_bfloat16, PP>(ep.shadow + c, ep.ld_shadow, rb, M, nw, w);
            if (has_b) {
#pragma unroll
                for (int i = 0; i < PP; ++i) {
                    if (rb + 4 * i >= M) continue;
                    float vb = 0.f;
#pragma unroll
                    for (int e = 0; e < 4; ++e) vb = e == bj ? a[i][e] : vb;  // static register indexing
                    const float gb = vb * alpha_eff;
                    if (!isfinite(gb) && ep.flag) atomicOr(ep.flag, 1u << (ep.flag_bit + 1));
                    ep.bias32[rb + 4 * i] -= lr * gb;
                }
            }
            break;
        }
        case EPI_ACTGRAD: {
            float x[PP][4];
            load_pieces<T, PP>(static_cast<const T*>(ep.aux) + c, ep.ld_aux, rb, M, nvc, x);
            with_act(ep.act, [&](auto A) {
#pragma unroll
                for (int i = 0; i < PP; ++i)
#pragma unroll
                    for (int e = 0; e < 4; ++e) a[i][e] *= act_grad_t<A.value == 0 ? 0 : 1>(x[i][e]);
            });
            store_pieces<T, PP>(static_cast<T*>(ep.out) + c, ep.ld_out, rb, M, nvc, a);
            break;
        }
        case EPI_EMA: {
            float o[PP][4];
            const float beta = ep.coef ? ep.coef[0] : ep.beta;
            const float alpha = ep.coef ? ep.coef[1] : ep.alpha;
            if (beta != 0.f) load_pieces<float, PP>(ep.out32 + c, ep.ld_out32, rb, M, nvc, o);
#pragma unroll
            for (int i = 0; i < PP; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) o[i][e] = (beta != 0.f ? beta * o[i][e] : 0.f) + alpha * a[i][e];
            store_pieces<float, PP>(ep.out32 + c, ep.ld_out32, rb, M, nvc, o);
            break;
        }
        case EPI_SUB: {
            float o[PP][4];
            load_pieces<float, PP>(ep.out32 + c, ep.ld_out32, rb, M, nvc, o);
#pragma unroll
            for (int i = 0; i < PP; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) o[i][e] -= a[i][e];
            store_pieces<float, PP>(ep.out32 + c, ep.ld_out32, rb, M, nvc, o);
            break;
        }
        case EPI_AXPY: {
            float w[PP][4];
            load_pieces<float, PP>(ep.out32 + c, ep.ld_out32, rb, M, nvc, w);
#pragma unroll
            for (int i = 0; i < PP; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) w[i][e] += ep.alpha * a[i][e];
            store_pieces<float, PP>(ep.out32 + c, ep.ld_out32, rb, M, nvc, w);
            if (ep.shadow) store_pieces<__nv_bfloat16, PP>(ep.shadow + c, ep.ld_shadow, rb, M, nvc, w);
            break;
        }
        default:
            break;
    }
    }  // passes
    __syncwarp();  // the buffer is free for the next chunk
    return bad;
}

// 32 consecutive values of one row -> memory, vectorised when aligned. The
// ragged path is fully unrolled with predication so v[] stays in registers.
template <typename T>
__device__ __forceinline__ void store_row32(T* dst, const float (&v)[32], int valid) {
    if (valid == 32 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        if constexpr (sizeof(T) == 4) {
            float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
            for (int i = 0; i < 8; ++i) d4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        } else {
            uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                uint32_t w[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * i + 2 * j], v[8 * i + 2 * j + 1]);
                    w[j] = *reinterpret_cast<uint32_t*>(&h);
                }
                d4[i] = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < valid) st_from_float<T>(dst + j, v[j]);
    }
}

template <typename T>
__device__ __forceinline__ void load_row32(const T* src, float (&v)[32], int valid) {
    if (valid == 32 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        if constexpr (sizeof(T) == 4) {
            const float4* s4 = reinterpret_cast<const float4*>(src);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                float4 f = s4[i];
                v[4 * i] = f.x; v[4 * i + 1] = f.y; v[4 * i + 2] = f.z; v[4 * i + 3] = f.w;
            }
        } else {
            const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                uint4 u = s4[i];
                uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&w[j]);
                    float2 f = __bfloat1622float2(h);
                    v[8 * i + 2 * j] = f.x;
                    v[8 * i + 2 * j + 1] = f.y;
                }
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = j < valid ? ld_as_float<T>(src + j) : 0.f;
    }
}

// Row-wise epilogue (lane = row) for the bf16-output modes FWD_ACT, ACTGRAD
// and RESID, see gemm_epi_transposed(). Their second operand x (the bias of
// FWD_ACT, the activations of ACTGRAD, X of RESID) does not depend on the
// accumulator, so its 32 values per chunk are loaded into raw registers before
// the accumulator is ready (for a tile's first chunk: before the mainloop ends)
// and converted only when used.
template <typename T>
__device__ __forceinline__ bool rows_x_fetch(const GemmEpi& ep, int row, int n, int valid, uint4 (&raw)[8]) {
    const bool fp = ep.mode == EPI_FWD_ACT;  // fp32 bias; else T-typed aux row
    const char* src = fp ? reinterpret_cast<const char*>(ep.bias + n)
                         : static_cast<const char*>(ep.aux) + (row * ep.ld_aux + n) * static_cast<long>(sizeof(T));
    const bool ok = valid == 32 && (reinterpret_cast<uintptr_t>(src) & 15) == 0;
    if (ok) {
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
        if (fp || sizeof(T) == 4) {
#pragma unroll
            for (int i = 0; i < 8; ++i) raw[i] = s4[i];
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) raw[i] = s4[i];
        }
    }
    return ok;
}

template <typename S>
__device__ __forceinline__ void rows_x_convert(const uint4 (&raw)[8], float (&x)[32]) {
    if constexpr (sizeof(S) == 4) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            x[4 * i] = __uint_as_float(raw[i].x); x[4 * i + 1] = __uint_as_float(raw[i].y);
            x[4 * i + 2] = __uint_as_float(raw[i].z); x[4 * i + 3] = __uint_as_float(raw[i].w);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t w[4] = {raw[i].x, raw[i].y, raw[i].z, raw[i].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[j]));
                x[8 * i + 2 * j] = f.x;
                x[8 * i + 2 * j + 1] = f.y;
            }
        }
    }
}

template <typename T>
__device__ __forceinline__ void epilogue_chunk_rows(const GemmEpi& ep, float (&v)[32], int row, int n, int valid,
                                                    const uint4 (&raw)[8], bool have, float& s_aux, float& s_out) {
    float x[32];
    if (ep.mode == EPI_FWD_ACT) {
        if (have) rows_x_convert<float>(raw, x);
        else load_row32<float>(ep.bias + n, x, valid);
        with_act(ep.act, [&](auto A) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = ep.out_scale * act_fwd_t<A.value>(v[j] + x[j]);
        });
    } else {
        if (have) rows_x_convert<T>(raw, x);
        else load_row32<T>(static_cast<const T*>(ep.aux) + row * ep.ld_aux + n, x, valid);
        if (ep.mode == EPI_ACTGRAD) {
            with_act(ep.act, [&](auto A) {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] *= act_grad_t<A.value == 0 ? 0 : 1>(x[j]);
            });
        } else {  // EPI_RESID
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                v[j] = x[j] - v[j];
                if constexpr (sizeof(T) == 2) v[j] = __bfloat162float(__float2bfloat16_rn(v[j]));  // as stored
                s_aux = fmaf(x[j], x[j], s_aux);
                s_out = fmaf(v[j], v[j], s_out);  // padding columns: x = acc = 0
            }
        }
    }
    store_row32<T>(static_cast<T*>(ep.out) + row * ep.ld_out + n, v, valid);
}

// Epilogue style per mode. fp32 outputs (the read-modify-write weight updates
// above all) use the transposed layout: it cuts the L1 wavefronts of a 32 x 32
// chunk 8x and took the hidden dW GEMM (GRAD_SGD) from 22.9 to 18.6 us. For the
// bf16-output modes the row-wise form measured faster (and kernels built with
// the transposed code run their mainloop ~6% slower), so they keep it.
inline bool gemm_epi_transposed(int mode) {
    return !(mode == EPI_FWD_ACT || mode == EPI_ACTGRAD || mode == EPI_RESID);
}

// Persistent, warp-specialised tcgen05 GEMM. grid <= #tiles; CTA c handles
// tiles c, c + grid, ... (m fastest). Roles:
//   warp 0      TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1      MMA issuer (one elected lane); owns the TMEM allocation
//   warps 2-9   epilogue: TMEM lane quadrant (warp % 4) -> registers -> global,
//               two sets of four splitting the tile's column chunks
//   warps 10-13 (SPLIT only) 3xTF32 splitters
// The accumulator is double buffered in TMEM (2 x BN columns), so the
// epilogue of tile i overlaps the mainloop of tile i+1.
//
// SPLIT (fp32 mode, T = float): 3xTF32. The splitters rewrite every staged
// operand x as hi = x with the low 13 mantissa bits cleared (exact TF32, in
// place) and lo = x - hi (exact in fp32) next to it; the MMA warp then
// accumulates hi*hi + hi*lo + lo*hi: relative error ~2^-21 instead of 2^-11.
//
// NP > 1 (grouped launch, MC == 1 only): NP independent problems of the same
// operand type / tile shape / majors / epilogue style -- e.g. every layer's
// dW -- in one persistent grid. The global tile index runs over the problems'
// tiles back to back (problem p owns tiles [tile0[p], tile0[p+1])); each CTA
// takes tiles b, b + grid, ... whatever problem they belong to, so the
// epilogue of one problem's tile overlaps the mainloop of the next tile, of
// the same or another problem. Every role re-selects the tile's problem.
template <typename T, int BN, int STAGES, bool A_MN, bool B_MN, bool SPLIT, bool TE, int MC, int NP>
__global__ void __launch_bounds__(GemmSmem<BN, STAGES, T, SPLIT, TE>::kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ GemmParams<NP> P) {
    using S = GemmSmem<BN, STAGES, T, SPLIT, TE>;
    constexpr bool kTf32 = OpTraits<T>::kTf32;
    static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");
    static_assert(!SPLIT || kTf32, "3xTF32 split needs fp32 operands");
    static_assert(MC == 1 || ((MC == 2 || MC == 3) && !SPLIT && !kTf32 && BN >= 128), "CTA pairs: bf16, BN >= 128");
    static_assert(MC != 3 || STAGES * S::kStage >= 2 * 128 * (BN / 2) * 4, "split-K pair: receive + send buffers in the ring");
    static_assert(NP == 1 || MC == 1, "grouped launches: single-CTA tiles");
    // problem 0; a grouped launch re-selects per tile (select() below)
    const CUtensorMap& tmA = P.ta[0];
    const CUtensorMap& tmB = P.tb[0];
    const int M = P.M[0], N = P.N[0], K = P.K[0];
    const GemmEpi& ep = P.ep[0];

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStage);
    uint64_t* empty = full + STAGES;
    uint64_t* split_done = empty + STAGES;
    uint64_t* tfull = split_done + STAGES;  // [2] accumulator ready for the epilogue
    uint64_t* tempty = tfull + 2;           // [2] accumulator drained by the epilogue
    uint64_t* xbar = tempty + 2;  // MC == 3: [0] both CTAs' MMAs done, [1 + w] epilogue warp w's partial received
    uint32_t* tslot = reinterpret_cast<uint32_t*>(xbar + 9);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int tiles_m = (M + 127) / 128;
    const int tiles_mn = tiles_m * ((N + BN - 1) / BN);
    // MC == 1: work item = tile (split-K: tile = mn + tiles_mn * ks), CTA b takes
    // b, b + grid, ... MC == 2 (CTA pairs, 2-SM MMA): work item = a 256 x BN
    // pair tile, pair p takes p, p + grid/2, ...; CTA rank r of the pair holds
    // rows 128 r .. 128 r + 127 of it (A rows and accumulator) and half of the
    // B tile (columns r BN/2 .. ); the leader (rank 0) issues the M = 256 MMAs.
    // MC == 3 (split-K pairs): one 128 x BN tile per cluster (grid = 2 x tiles),
    // CTA rank r runs the k-blocks of half r; the partial tiles are exchanged
    // through distributed shared memory and rank r finalises columns r BN/2 ...
    const int tmp = (tiles_m + 1) / 2;
    const int tiles = NP > 1 ? P.tile0[P.np]
                             : (MC == 1 ? tiles_mn * ep.ksplit : (MC == 3 ? tiles_mn : tmp * ((N + BN - 1) / BN)));
    const int w0 = MC == 1 ? static_cast<int>(blockIdx.x) : static_cast<int>(blockIdx.x) / 2;
    const int wstep = MC == 1 ? static_cast<int>(gridDim.x) : static_cast<int>(gridDim.x) / 2;
    const int rank = MC == 1 ? 0 : static_cast<int>(cluster_ctarank());
    const int nk_all = (K + S::kBK - 1) / S::kBK;
    const int nk_per = (nk_all + ep.ksplit - 1) / ep.ksplit;
    // Work item -> problem, tile origin, split, k-block range [kb0, kb1) (gemm_plan
    // guarantees it is non-empty), and whether a SYRK-style update skips it.
    struct TileInfo {
        int p, m0, n0, ks, kb0, kb1, M, N;
        bool skip;
    };
    auto select = [&](int w) {
        TileInfo t;
        if constexpr (NP > 1) {
            int p = 0;
            while (p + 1 < P.np && w >= P.tile0[p + 1]) ++p;
            const int lw = w - P.tile0[p];
            const int tm = (P.M[p] + 127) / 128;
            t.p = p;
            t.M = P.M[p];
            t.N = P.N[p];
            t.m0 = (lw % tm) * 128;
            t.n0 = (lw / tm) * BN;
            t.ks = 0;
            t.kb0 = 0;
            t.kb1 = (P.K[p] + S::kBK - 1) / S::kBK;
            t.skip = false;
            return t;
        }
        t.p = 0;
        t.M = M;
        t.N = N;
        if (MC != 2) {
            t.m0 = (w % tiles_m) * 128;
            t.n0 = ((w % tiles_mn) / tiles_m) * BN;
        } else {
            t.m0 = (2 * (w % tmp) + rank) * 128;
            t.n0 = (w / tmp) * BN;
        }
        t.skip = ep.lower && t.n0 > t.m0 + 127;
        if (MC == 3) {
            const int half = (nk_all + 1) / 2;
            t.ks = 0;
            t.kb0 = rank * half;
            t.kb1 = min(nk_all, t.kb0 + half);
        } else {
            t.ks = w / tiles_mn;
            t.kb0 = t.ks * nk_per;
            t.kb1 = min(nk_all, t.kb0 + nk_per);
        }
        return t;
    };

    if (threadIdx.x == 0) {
        PNB_TRACE(0);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
            mbar_init(&split_done[s], 128);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], MC == 2 ? 16 : 256);  // pairs: one arrive per epilogue warp of both CTAs
        }
        mbar_init(&xbar[0], 2);  // MC == 3: each CTA's MMA completion, multicast to both
        for (int w = 1; w <= 8; ++w) mbar_init(&xbar[w], 1);  // MC == 3: own expect_tx + the peer warp's copy
        fence_barrier_init();
        for (int p = 0; p < (NP > 1 ? P.np : 1); ++p) {
            tma_prefetch_desc(&P.ta[p]);
            tma_prefetch_desc(&P.tb[p]);
        }
    }
    if (warp == 1) {
        if constexpr (MC == 2)
            tmem_alloc2<S::kTmemCols>(tslot);
        else
            tmem_alloc<S::kTmemCols>(tslot);
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (MC == 2) cluster_sync_all();  // the peer's barriers exist before any remote arrive
    // MC == 3: arrive now, wait right before each role's first remote operation
    if constexpr (MC == 3) cluster_arrive_relaxed();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    // Programmatic dependent launch (gemm_launch): everything above -- barrier
    // init, TMEM allocation, descriptor prefetch -- overlapped the previous
    // kernel of the stream; every operand, bias, aux or weight read comes after this.
    grid_dep_wait();
    if (threadIdx.x == 0) PNB_TRACE(1);

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            int it = 0;  // global k-block counter (ring position)
            for (int tile = w0; tile < tiles; tile += wstep) {
                const TileInfo ti = select(tile);
                if (ti.skip) continue;
                const int m0 = ti.m0, n0 = ti.n0, kb0 = ti.kb0, kb1 = ti.kb1;
                const CUtensorMap& tA = P.ta[ti.p];
                const CUtensorMap& tB = P.tb[ti.p];
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % STAGES;
                    if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
                    uint8_t* sa = smem + s * S::kStage;
                    uint8_t* sb = sa + S::kABytes;
                    const int k0 = kb * S::kBK;
                    if constexpr (MC == 2) {
                        // own A rows + own half of B, bytes counted on the leader's full barrier
                        if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * (S::kABytes + S::kBBytes / 2));
                        const uint32_t fb = mapa_cluster(&full[s], 0);
                        if constexpr (!A_MN) {
                            tma_load_2d_cg2(sa, &tmA, fb, k0, m0);
                        } else {
#pragma unroll
                            for (int a = 0; a < 128 / S::kAtom; ++a)
                                tma_load_2d_cg2(sa + a * (S::kBK * 128), &tmA, fb, m0 + a * S::kAtom, k0);
                        }
                        if constexpr (!B_MN) {
                            tma_load_2d_cg2(sb, &tmB, fb, k0, n0 + rank * (BN / 2));
                        } else {
                            constexpr int nb = BN / 2 / S::kAtom;
#pragma unroll
                            for (int a = 0; a < nb; ++a)
                                tma_load_2d_cg2(sb + a * (S::kBK * 128), &tmB, fb, n0 + (rank * nb + a) * S::kAtom, k0);
                        }
                        continue;
                    }
                    mbar_arrive_expect_tx(&full[s], S::kLoad);
                    if constexpr (!A_MN) {
                        tma_load_2d(sa, &tA, &full[s], k0, m0);
                    } else {
#pragma unroll
                        for (int a = 0; a < 128 / S::kAtom; ++a)
                            tma_load_2d(sa + a * (S::kBK * 128), &tA, &full[s], m0 + a * S::kAtom, k0);
                    }
                    if constexpr (!B_MN) {
                        tma_load_2d(sb, &tB, &full[s], k0, n0);
                    } else {
#pragma unroll
                        for (int a = 0; a < BN / S::kAtom; ++a)
                            tma_load_2d(sb + a * (S::kBK * 128), &tB, &full[s], n0 + a * S::kAtom, k0);
                    }
                }
            }
            if constexpr (MC == 2) {
                // drain: every stage's last phase released by the leader's MMAs, so
                // no remote arrive targets this CTA once it passes the exit barrier
                for (int j = (it > STAGES ? it - STAGES : 0); j < it; ++j)
                    mbar_wait(&empty[j % STAGES], (j / STAGES) & 1);
            }
        }
        if constexpr (MC == 3) cluster_wait();
    } else if (warp == 1) {
        // ---------------- MMA issuer (pairs: the leader only) ----------------
        if (lane == 0 && (MC != 2 || rank == 0)) {
            constexpr uint32_t idesc = make_idesc(OpTraits<T>::kFmt, A_MN ? 1 : 0, B_MN ? 1 : 0, MC == 2 ? 256 : 128, BN);
            constexpr uint32_t kMnLayout = kTf32 ? 1 : 2;  // BASE32B for TF32 MN-major
            constexpr uint32_t kMnSbo = kTf32 ? 512 : 1024;
            auto desc_a = [&](uint32_t base, int k) {
                return A_MN ? smem_desc_sw128(base + k * S::kUK * 128, S::kBK * 128, kMnSbo, kMnLayout)
                            : smem_desc_sw128(base + k * 32, 16, 1024);
            };
            auto desc_b = [&](uint32_t base, int k) {
                return B_MN ? smem_desc_sw128(base + k * S::kUK * 128, S::kBK * 128, kMnSbo, kMnLayout)
                            : smem_desc_sw128(base + k * 32, 16, 1024);
            };
            int it = 0, local = 0;
            for (int tile = w0; tile < tiles; tile += wstep) {
                const TileInfo ti = select(tile);
                if (ti.skip) continue;
                const int acc = local & 1;
                if (local >= 2) mbar_wait(&tempty[acc], ((local >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                const int kb0 = ti.kb0, kb1 = ti.kb1;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(SPLIT ? &split_done[s] : &full[s], (it / STAGES) & 1);
                    if (it == 0) PNB_TRACE(2);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + s * S::kStage);
                    const uint32_t sb = sa + S::kABytes;
#pragma unroll
                    for (int k = 0; k < S::kBK / S::kUK; ++k) {
                        if constexpr (MC == 2) {
                            umma2_bf16(d, desc_a(sa, k), desc_b(sb, k), idesc, (kb != kb0 || k != 0) ? 1u : 0u);
                            continue;
                        }
                        umma<kTf32>(d, desc_a(sa, k), desc_b(sb, k), idesc, (kb != kb0 || k != 0) ? 1u : 0u);
                        if constexpr (SPLIT) {
                            const uint32_t sal = sa + S::kLoad, sbl = sb + S::kLoad;
                            umma<kTf32>(d, desc_a(sa, k), desc_b(sbl, k), idesc, 1u);
                            umma<kTf32>(d, desc_a(sal, k), desc_b(sb, k), idesc, 1u);
                        }
                    }
                    if constexpr (MC == 2)
                        umma_commit2_mc(&empty[s], 3);  // both CTAs' stage s is free again
                    else
                        umma_commit(&empty[s]);
                }
                if constexpr (MC == 2)
                    umma_commit2_mc(&tfull[acc], 3);  // both CTAs' accumulator rows are ready
                else
                    umma_commit(&tfull[acc]);

                PNB_TRACE(3);
                ++local;
            }
        }
        if constexpr (MC == 3) {
            cluster_wait();  // the peer's barriers are initialised
            if (lane == 0) umma_commit_mc(&xbar[0], 3);  // after my MMAs: my ring is free for the peer's partial
        }
    } else if (warp < 10) {
        // ---------------- epilogue (8 warps: 2 sets x 128 TMEM lanes) ----------------
        // a warp may only touch its TMEM lane quadrant (warp % 4); the two sets
        // split the tile's 32-column chunks (even / odd), which halves the serial
        // per-row work of each thread
        const int quad = warp & 3;
        const int eset = (warp - 2) >> 2;
        uint4* ebuf = reinterpret_cast<uint4*>(smem + STAGES * S::kStage + 512) + (warp - 2) * 256;
        auto sgd_scalars = [](const GemmEpi& e, float& lr_, float& alpha_) {
            lr_ = 0.f;
            alpha_ = e.alpha;
            if (e.mode == EPI_GRAD_SGD) {
                lr_ = e.lr[e.step ? *e.step : 0];
                if (e.coef) alpha_ = e.alpha * e.coef[0];
                if (e.gscale_a) alpha_ = static_cast<float>(e.alpha * *e.gscale_a * *e.gscale_b);
            }
        };
        float lr, alpha_eff;
        sgd_scalars(ep, lr, alpha_eff);
        bool bad = false;
        float s_aux = 0.f, s_out = 0.f;  // RESID sums (per thread, this CTA's tiles)
        int local = 0;
        for (int tile = w0; tile < tiles; tile += wstep) {
            const TileInfo ti = select(tile);
            if (ti.skip) continue;
            const int m0 = ti.m0, n0 = ti.n0, ks = ti.ks;
            // this tile's problem (grouped launches); the names shadow problem 0's
            const GemmEpi& ep = P.ep[ti.p];
            const int M = ti.M, N = ti.N;
            if constexpr (NP > 1) sgd_scalars(ep, lr, alpha_eff);
            const int acc = local & 1;
            const int row = m0 + quad * 32 + lane;
            const bool row_ok = row < M;
            // Pull this tile's epilogue source rows (weights / activations /
            // factors being read-modify-written) into L2 while the MMAs run:
            // otherwise each 32-column chunk pays a full DRAM round trip.
            if (row_ok && eset == 0) {
                const char* src = nullptr;
                long bytes = 0;
                if (ep.mode == EPI_GRAD_SGD || ep.mode == EPI_EMA || ep.mode == EPI_SUB || ep.mode == EPI_AXPY) {
                    src = reinterpret_cast<const char*>(ep.out32 + row * ep.ld_out32 + n0);
                    bytes = static_cast<long>(min(BN, N - n0)) * 4;
                } else if (ep.mode == EPI_ACTGRAD || ep.mode == EPI_RESID) {
                    src = static_cast<const char*>(ep.aux) + (row * ep.ld_aux + n0) * static_cast<long>(sizeof(T));
                    bytes = static_cast<long>(min(BN, N - n0)) * static_cast<long>(sizeof(T));
                }
                for (long o = 0; o < bytes; o += 128) prefetch_l2(src + o);
            }
            // MC == 3: this CTA finalises the chunks of its half of the columns
            constexpr int kHalfChunks = BN / 64;
            const int c_begin = (MC == 3 ? rank * kHalfChunks : 0) + eset;
            const int c_end = MC == 3 ? (rank + 1) * kHalfChunks : BN / 32;
            // row-wise modes: the first chunk's x operand is fetched before the accumulator is ready
            uint4 xraw[8];
            bool xhave = false;
            if constexpr (!TE) {
                const int n = n0 + c_begin * 32;
                if (row_ok && n < N) xhave = rows_x_fetch<T>(ep, row, n, min(32, N - n), xraw);
            }
            mbar_wait_sleep(&tfull[acc], (local >> 1) & 1);
            // the mainloop of this CTA's first tile is done: the next kernel may
            // start its prologue on the SMs that free up
            if (local == 0) grid_dep_launch();
            if (warp == 2 && lane == 0) PNB_TRACE(4);
            tc_fence_after();
            // Exchange buffers in the idle ring, one contiguous region per epilogue warp
            // (quad, set): its 32 rows x the kJ chunks it finalises, 16-byte slots
            // XOR-swizzled by row (conflict-free both ways). Warp (quad, set) of one CTA
            // sends exactly what warp (quad, set) of the peer finalises.
            constexpr int kJ = BN / 128;  // chunks per warp per half
            uint4* xrecv = reinterpret_cast<uint4*>(smem) + ((warp - 2) * 32 + lane) * (kJ * 8);
            if constexpr (MC == 3) {
                cluster_wait();  // the peer's barriers are initialised
                constexpr uint32_t kWarpBytes = 32u * kJ * 32u * 4u;
                constexpr uint32_t kHalfBytes = 128u * (BN / 2) * 4u;
                uint4* xsend = xrecv + kHalfBytes / 16;
#pragma unroll
                for (int j = 0; j < kJ; ++j) {
                    const int c = (rank ^ 1) * kHalfChunks + eset + 2 * j;
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(quad * 32) << 16) + acc * BN + c * 32, r);
                    tmem_ld_wait();
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        sts128(xsend + j * 8 + (k ^ (lane & 7)), make_uint4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]));
                }
                fence_proxy_async_smem();  // generic writes -> visible to the bulk copy
                __syncwarp();
                uint64_t* wbar = &xbar[1 + (warp - 2)];
                if (lane == 0) {
                    mbar_arrive_expect_tx(wbar, kWarpBytes);  // the peer warp's copy into my ring
                    mbar_wait(&xbar[0], 0);                   // both MMAs done: the peer's ring is free
                    bulk_copy_to_peer(mapa_cluster(xrecv, rank ^ 1), xsend, kWarpBytes, mapa_cluster(wbar, rank ^ 1));
                    if (warp == 2) PNB_TRACE(7);
                }
                mbar_wait(wbar, 0);  // the peer's partial of my chunks has landed (bulk copy, like TMA)
                if (warp == 2 && lane == 0) PNB_TRACE(8);
            }
#pragma unroll 1
            for (int c = c_begin; c < c_end; c += 2) {
                const int n = n0 + c * 32;
                if (n >= N) break;  // warp-uniform
                if (m0 + quad * 32 >= M) break;  // warp-uniform: no rows of this quadrant
                uint32_t r[32];
                tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(quad * 32) << 16) + acc * BN + c * 32, r);
                tmem_ld_wait();
                if constexpr (MC == 3) {
                    const int j = (c - rank * kHalfChunks - eset) / 2;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint4 u = lds128(xrecv + j * 8 + (k ^ (lane & 7)));
                        // own + peer partial (fp32 addition commutes: both CTAs' halves round alike)
                        r[4 * k] = __float_as_uint(__uint_as_float(r[4 * k]) + __uint_as_float(u.x));
                        r[4 * k + 1] = __float_as_uint(__uint_as_float(r[4 * k + 1]) + __uint_as_float(u.y));
                        r[4 * k + 2] = __float_as_uint(__uint_as_float(r[4 * k + 2]) + __uint_as_float(u.z));
                        r[4 * k + 3] = __float_as_uint(__uint_as_float(r[4 * k + 3]) + __uint_as_float(u.w));
                    }
                }
                if constexpr (TE) {
                    bad |= epilogue_chunk<T, SPLIT ? 4 : 8>(ep, r, ebuf, lane, m0 + quad * 32, M, n, N, lr, alpha_eff,
                                                            ks, s_aux, s_out);
                } else if (row_ok) {
                    // next chunk of this warp: its x loads are issued before this chunk's
                    // math and stores, so their latency overlaps them
                    const int nn = n + 64;
                    uint4 xnext[8];
                    const bool nhave =
                        nn < N && c + 2 < c_end && rows_x_fetch<T>(ep, row, nn, min(32, N - nn), xnext);
                    float v[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                    epilogue_chunk_rows<T>(ep, v, row, n, min(32, N - n), xraw, xhave, s_aux, s_out);
#pragma unroll
                    for (int i = 0; i < 8; ++i) xraw[i] = xnext[i];
                    xhave = nhave;
                }
            }
            if (warp == 2 && lane == 0) PNB_TRACE(9);
            tc_fence_before();
            if constexpr (MC == 2) {
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(mapa_cluster(&tempty[acc], 0));  // the leader's MMA reuses it
            } else {
                mbar_arrive(&tempty[acc]);
            }
            if (warp == 2 && lane == 0) PNB_TRACE(5);
            ++local;
            if constexpr (NP > 1) {  // each problem has its own non-finite flag bit
                if (bad && ep.flag) atomicOr(ep.flag, 1u << ep.flag_bit);
                bad = false;
            }
        }
        if (bad && ep.flag) atomicOr(ep.flag, 1u << ep.flag_bit);
        if (ep.mode == EPI_RESID) {
            // deterministic per-CTA sums: fixed tile order, fixed reduction tree
            __shared__ float red[2][8];
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                s_aux += __shfl_xor_sync(0xffffffffu, s_aux, o);
                s_out += __shfl_xor_sync(0xffffffffu, s_out, o);
            }
            if (lane == 0) {
                red[0][warp - 2] = s_aux;
                red[1][warp - 2] = s_out;
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");  // the 8 epilogue warps
            if (warp == 2 && lane == 0) {
                double a = 0.0, b = 0.0;
                for (int i = 0; i < 8; ++i) {
                    a += red[0][i];
                    b += red[1][i];
                }
                ep.part[2 * blockIdx.x] = a;
                ep.part[2 * blockIdx.x + 1] = b;
            }
        }
    } else if (SPLIT) {
        // ---------------- 3xTF32 splitters (warps 10-13) ----------------
        const int t = threadIdx.x - 320;
        int it = 0;
        for (int tile = w0; tile < tiles; tile += wstep) {
            const TileInfo ti = select(tile);
            if (ti.skip) continue;
            for (int kb = ti.kb0; kb < ti.kb1; ++kb, ++it) {
                const int s = it % STAGES;
                mbar_wait(&full[s], (it / STAGES) & 1);
                float4* hi = reinterpret_cast<float4*>(smem + s * S::kStage);
                float4* lo = reinterpret_cast<float4*>(smem + s * S::kStage + S::kLoad);
#pragma unroll 4
                for (int i = t; i < S::kLoad / 16; i += 128) {
                    float4 x = hi[i], h, l;
                    h.x = __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
                    h.y = __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
                    h.z = __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
                    h.w = __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
                    l.x = x.x - h.x; l.y = x.y - h.y; l.z = x.z - h.z; l.w = x.w - h.w;
                    hi[i] = h;
                    lo[i] = l;
                }
                fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
                mbar_arrive(&split_done[s]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (MC == 2) {
        cluster_sync_all();
        if (warp == 1) tmem_dealloc2<S::kTmemCols>(tmem);
    } else if constexpr (MC == 3) {
        // no CTA leaves while its outgoing copy may still read its smem (the peer
        // arrives only after receiving it)
        cluster_arrive_relaxed();
        cluster_wait();
        if (warp == 1) tmem_dealloc<S::kTmemCols>(tmem);
    } else {
        if (warp == 1) tmem_dealloc<S::kTmemCols>(tmem);
    }
    if (threadIdx.x == 0) PNB_TRACE(6);
}

}  // namespace pnb
