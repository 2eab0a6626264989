// Model averaging (parallel.cpp:26-59, protocol :195-214) on device.
//
//  * local replicas of one GPU (virtual workers, config 5) are summed in the
//    reference's rank-ordered midpoint tree (tree_sum), in one HBM pass;
//  * across GPUs (one process per GPU) the partial sums go through one NCCL
//    all-reduce over NVLink on the averaging stream; with one replica per GPU
//    it is a single in-place ncclAllReduce(..., ncclAvg) -- the 1/m scale is
//    fused into the collective;
//  * the scaled result is written back into every local replica together with
//    its bf16 operand copy.
#include <nccl.h>

#include <utility>

#include "parallel.h"

namespace pnb {

namespace {

#define NCCL_THROW(x)                                                                             \
    do {                                                                                          \
        ncclResult_t r_ = (x);                                                                    \
        if (r_ != ncclSuccess)                                                                    \
            throw std::runtime_error(std::string("NCCL error: ") + ncclGetErrorString(r_) + " (" + \
                                     __FILE__ + ":" + std::to_string(__LINE__) + ")");            \
    } while (0)

__device__ float tree_sum_at(const float* const* src, int lo, int hi, long i) {
    // Same shape as tree_sum (parallel.cpp:28-36): [lo, mid) + [mid, hi).
    if (hi - lo == 1) return src[lo][i];
    const int mid = lo + (hi - lo) / 2;
    return tree_sum_at(src, lo, mid, i) + tree_sum_at(src, mid, hi, i);
}

// out_k[i] = scale * tree_sum(src)[i] for every destination k (+ bf16 copy).
__global__ void tree_avg_kernel(const float* const* src, int m, long n, float scale, int apply_scale,
                                float* const* dst, bf16* const* shadow, int ndst) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        float v = tree_sum_at(src, 0, m, i);
        if (apply_scale) v *= scale;
        for (int k = 0; k < ndst; ++k) {
            dst[k][i] = v;
            if (shadow[k]) shadow[k][i] = __float2bfloat16_rn(v);
        }
    }
}

// Vectorised form for m <= 32 local replicas: each thread loads the m float4s
// of its 4 elements into registers, then adds them in the same midpoint tree,
// unrolled at compile time (bitwise equal to tree_sum_at), so all m loads are
// in flight at once. Elements past the last whole float4 go through the scalar
// tree in block 0.
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float add4(float a, float b) { return a + b; }

template <int LO, int HI, typename V>
__device__ __forceinline__ V tree_reg(const V* x) {
    if constexpr (HI - LO == 1) {
        return x[LO];
    } else {
        constexpr int MID = LO + (HI - LO) / 2;
        return add4(tree_reg<LO, MID>(x), tree_reg<MID, HI>(x));
    }
}

template <int M>
__global__ void __launch_bounds__(256) tree_avg4_kernel(const float* const* src, long n, float scale, int apply_scale,
                                                        float* const* dst, bf16* const* shadow, int ndst) {
    const long n4 = n / 4;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
        float4 x[M];
#pragma unroll
        for (int k = 0; k < M; ++k) x[k] = reinterpret_cast<const float4*>(src[k])[i];  // warp-uniform pointer loads
        float4 v = tree_reg<0, M>(x);
        if (apply_scale) v = make_float4(v.x * scale, v.y * scale, v.z * scale, v.w * scale);
        for (int k = 0; k < ndst; ++k) {
            reinterpret_cast<float4*>(dst[k])[i] = v;
            if (shadow[k]) {
                const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
                reinterpret_cast<uint2*>(shadow[k])[i] =
                    make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
            }
        }
    }
    const long t = 4 * n4 + threadIdx.x;
    if (blockIdx.x == 0 && t < n) {
        float x[M];
#pragma unroll
        for (int k = 0; k < M; ++k) x[k] = src[k][t];
        float v = tree_reg<0, M>(x);
        if (apply_scale) v *= scale;
        for (int k = 0; k < ndst; ++k) {
            dst[k][t] = v;
            if (shadow[k]) shadow[k][t] = __float2bfloat16_rn(v);
        }
    }
}

using AvgFn = void (*)(const float* const*, long, float, int, float* const*, bf16* const*, int);

template <int... Ms>
AvgFn avg4_pick(int m, std::integer_sequence<int, Ms...>) {
    AvgFn fn = nullptr;
    ((m == Ms + 1 ? (fn = &tree_avg4_kernel<Ms + 1>, 0) : 0), ...);
    return fn;
}

__global__ void bf16_copy_kernel(const float* __restrict__ src, long n, bf16* __restrict__ dst) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        dst[i] = __float2bfloat16_rn(src[i]);
}

}  // namespace

Comm::Comm(Context* c, const unsigned char id[128], int nranks_, int rank_) : ctx(c), nranks(nranks_), rank(rank_) {
    CUDA_THROW(cudaSetDevice(c->device));
    ncclUniqueId uid;
    static_assert(sizeof(uid.internal) == 128, "ncclUniqueId size");
    std::memcpy(uid.internal, id, 128);
    ncclComm_t cm;
    NCCL_THROW(ncclCommInitRank(&cm, nranks, uid, rank));
    comm = cm;
    CUDA_THROW(cudaMalloc(&dscratch, 64));
}

Comm::~Comm() {
    if (comm) ncclCommDestroy(static_cast<ncclComm_t>(comm));
    if (dscratch) cudaFree(dscratch);
}

void nccl_unique_id(unsigned char out[128]) {
    ncclUniqueId uid;
    NCCL_THROW(ncclGetUniqueId(&uid));
    std::memcpy(out, uid.internal, 128);
}

double Comm::allreduce_sum(double v) {
    cudaStream_t s = ctx->stream;
    CUDA_THROW(cudaMemcpyAsync(dscratch, &v, 8, cudaMemcpyHostToDevice, s));
    NCCL_THROW(ncclAllReduce(dscratch, dscratch, 1, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm), s));
    CUDA_THROW(cudaMemcpyAsync(&v, dscratch, 8, cudaMemcpyDeviceToHost, s));
    CUDA_THROW(cudaStreamSynchronize(s));
    return v;
}

Averager::Averager(Context* c, const std::vector<Replica*>& r, Comm* cm, long m) : ctx(c), reps(r), comm(cm), m_total(m) {
    if (reps.empty()) throw std::runtime_error("allreduce_average: m must be >= 1");
    n = reps[0]->n_pad;
    for (Replica* p : reps)
        if (p->n_pad != n)
            throw std::runtime_error("allreduce_average: replica vector lengths differ");
    const int k = static_cast<int>(reps.size());
    std::vector<float*> src(k);
    std::vector<bf16*> sh(k);
    for (int i = 0; i < k; ++i) {
        src[i] = reps[i]->params;
        sh[i] = reps[i]->wshadow;
    }
    CUDA_THROW(cudaMalloc(&d_src, k * sizeof(float*)));
    CUDA_THROW(cudaMalloc(&d_shadow, k * sizeof(bf16*)));
    CUDA_THROW(cudaMemcpy(d_src, src.data(), k * sizeof(float*), cudaMemcpyHostToDevice));
    CUDA_THROW(cudaMemcpy(d_shadow, sh.data(), k * sizeof(bf16*), cudaMemcpyHostToDevice));
    if (comm && k > 1) {
        CUDA_THROW(cudaMalloc(&scratch, n * sizeof(float)));
        CUDA_THROW(cudaMalloc(&d_scratch_ptr, sizeof(float*)));
        CUDA_THROW(cudaMemcpy(d_scratch_ptr, &scratch, sizeof(float*), cudaMemcpyHostToDevice));
    }
    CUDA_THROW(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming));
    for (int i = 0; i < k; ++i) {
        cudaEvent_t e;
        CUDA_THROW(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ev_rep.push_back(e);
    }
}

Averager::~Averager() {
    if (d_src) cudaFree(d_src);
    if (d_shadow) cudaFree(d_shadow);
    if (scratch) cudaFree(scratch);
    if (d_scratch_ptr) cudaFree(d_scratch_ptr);
    if (ev_done) cudaEventDestroy(ev_done);
    for (auto e : ev_rep) cudaEventDestroy(e);
}

void Averager::run() {
    cudaStream_t s = ctx->stream;
    const int k = static_cast<int>(reps.size());
    for (int i = 0; i < k; ++i) {
        CUDA_THROW(cudaEventRecord(ev_rep[i], reps[i]->stream));
        CUDA_THROW(cudaStreamWaitEvent(s, ev_rep[i], 0));
    }
    const float inv = static_cast<float>(1.0 / static_cast<double>(m_total));
    const int grid = ctx->num_sms * 8;
    // float4 params / 8-byte bf16 shadows (cudaMalloc'd replica buffers always are)
    bool vec_ok = true;
    for (Replica* r : reps)
        vec_ok = vec_ok && (reinterpret_cast<uintptr_t>(r->params) & 15) == 0 &&
                 (reinterpret_cast<uintptr_t>(r->wshadow) & 7) == 0;
    if (scratch) vec_ok = vec_ok && (reinterpret_cast<uintptr_t>(scratch) & 15) == 0;
    if (!comm) {
        if (k > 1) {
            if (AvgFn f = vec_ok ? avg4_pick(k, std::make_integer_sequence<int, 32>{}) : nullptr)
                f<<<grid, 256, 0, s>>>(d_src, n, inv, 1, d_src, d_shadow, k);
            else
                tree_avg_kernel<<<grid, 256, 0, s>>>(d_src, k, n, inv, 1, d_src, d_shadow, k);
        }
        else if (m_total != 1)
            throw std::runtime_error("allreduce_average: got 1 contributions for m = " + std::to_string(m_total));
        // m == 1: x * 1.0 is the identity (parallel.cpp:56-57), nothing to do.
    } else if (k == 1) {
        ncclComm_t cm = static_cast<ncclComm_t>(comm->comm);
        if (comm->nranks == m_total) {
            NCCL_THROW(ncclAllReduce(reps[0]->params, reps[0]->params, n, ncclFloat, ncclAvg, cm, s));
        } else {
            throw std::runtime_error("allreduce_average: rank layout does not cover m workers");
        }
        if (reps[0]->wshadow) bf16_copy_kernel<<<grid, 256, 0, s>>>(reps[0]->params, n, reps[0]->wshadow);
    } else {
        // local subtree sum -> NCCL sum over GPUs -> x 1/m into every local replica
        if (AvgFn f = vec_ok ? avg4_pick(k, std::make_integer_sequence<int, 32>{}) : nullptr)
            f<<<grid, 256, 0, s>>>(d_src, n, 1.f, 0, d_scratch_ptr, d_shadow, 0);
        else
            tree_avg_kernel<<<grid, 256, 0, s>>>(d_src, k, n, 1.f, 0, d_scratch_ptr, d_shadow, 0);
        NCCL_THROW(ncclAllReduce(scratch, scratch, n, ncclFloat, ncclSum, static_cast<ncclComm_t>(comm->comm), s));
        tree_avg_kernel<<<grid, 256, 0, s>>>(d_scratch_ptr, 1, n, inv, 1, d_src, d_shadow, k);
    }
    CUDA_THROW(cudaGetLastError());
    CUDA_THROW(cudaEventRecord(ev_done, s));
    for (int i = 0; i < k; ++i) CUDA_THROW(cudaStreamWaitEvent(reps[i]->stream, ev_done, 0));
}

}  // namespace pnb
