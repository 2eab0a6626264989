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

#include <algorithm>
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

// out_k[i] = scale * tree_sum(src)[i] for every destination k (+ bf16 copy),
// i in [off, off + n).
__global__ void tree_avg_kernel(const float* const* src, int m, long off, long n, float scale, int apply_scale,
                                float* const* dst, bf16* const* shadow, int ndst) {
    for (long i = off + blockIdx.x * (long)blockDim.x + threadIdx.x; i < off + n; i += (long)gridDim.x * blockDim.x) {
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
// in flight at once. The range [off, off + n) starts on a float4 boundary
// (buckets are 128-byte aligned); elements past its last whole float4 go
// through the scalar tree in block 0. With M = 1 it is the fused scale pass:
// scratch * (1/m) -> every local replica and its bf16 operand copy.
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
__global__ void __launch_bounds__(256) tree_avg4_kernel(const float* const* src, long off, long n, float scale,
                                                        int apply_scale, float* const* dst, bf16* const* shadow,
                                                        int ndst) {
    const long n4 = n / 4, b4 = off / 4;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
        float4 x[M];
#pragma unroll
        for (int k = 0; k < M; ++k) x[k] = reinterpret_cast<const float4*>(src[k])[b4 + i];  // warp-uniform pointer loads
        float4 v = tree_reg<0, M>(x);
        if (apply_scale) v = make_float4(v.x * scale, v.y * scale, v.z * scale, v.w * scale);
        for (int k = 0; k < ndst; ++k) {
            reinterpret_cast<float4*>(dst[k])[b4 + i] = v;
            if (shadow[k]) {
                const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
                reinterpret_cast<uint2*>(shadow[k])[b4 + i] =
                    make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
            }
        }
    }
    const long t = off + 4 * n4 + threadIdx.x;
    if (blockIdx.x == 0 && t < off + n) {
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

using AvgFn = void (*)(const float* const*, long, long, float, int, float* const*, bf16* const*, int);

template <int... Ms>
AvgFn avg4_pick(int m, std::integer_sequence<int, Ms...>) {
    AvgFn fn = nullptr;
    ((m == Ms + 1 ? (fn = &tree_avg4_kernel<Ms + 1>, 0) : 0), ...);
    return fn;
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
    const long k = static_cast<long>(reps.size());
    // every worker contributes exactly once (allreduce_average, parallel.cpp:44-47)
    const long contributions = comm ? static_cast<long>(comm->nranks) * k : k;
    if (contributions != m_total)
        throw std::runtime_error("allreduce_average: got " + std::to_string(contributions) +
                                 " contributions for m = " + std::to_string(m_total));
    n = reps[0]->n_pad;
    for (Replica* p : reps)
        if (p->n_pad != n || p->L != reps[0]->L || p->w_off != reps[0]->w_off)
            throw std::runtime_error("allreduce_average: replica vector lengths differ");
    std::vector<float*> src(k);
    std::vector<bf16*> sh(k);
    for (long i = 0; i < k; ++i) {
        src[i] = reps[i]->params;
        sh[i] = reps[i]->wshadow;
    }
    CUDA_THROW(cudaMalloc(&d_src, k * sizeof(float*)));
    CUDA_THROW(cudaMalloc(&d_shadow, k * sizeof(bf16*)));
    CUDA_THROW(cudaMalloc(&d_null_shadow, sizeof(bf16*)));
    upload(d_src, src.data(), k * sizeof(float*));
    upload(d_shadow, sh.data(), k * sizeof(bf16*));
    zero(d_null_shadow, sizeof(bf16*));
    work = comm != nullptr || k > 1;
    if (work)
        for (Replica* p : reps) p->precapture_gates();
    if (comm && k > 1) {
        CUDA_THROW(cudaMalloc(&scratch, n * sizeof(float)));
        CUDA_THROW(cudaMalloc(&d_scratch_ptr, sizeof(float*)));
        upload(d_scratch_ptr, &scratch, sizeof(float*));
    }
}

Averager::~Averager() {
    if (d_src) cudaFree(d_src);
    if (d_shadow) cudaFree(d_shadow);
    if (d_null_shadow) cudaFree(d_null_shadow);
    if (scratch) cudaFree(scratch);
    if (d_scratch_ptr) cudaFree(d_scratch_ptr);
}

void Averager::run() {
    cudaStream_t s = ctx->avg;
    const int k = static_cast<int>(reps.size());
    const int L = reps[0]->L;
    const float inv = static_cast<float>(1.0 / static_cast<double>(m_total));
    // float4 params / 8-byte bf16 shadows (cudaMalloc'd replica buffers always are)
    bool vec_ok = true;
    for (Replica* r : reps)
        vec_ok = vec_ok && (reinterpret_cast<uintptr_t>(r->params) & 15) == 0 &&
                 (reinterpret_cast<uintptr_t>(r->wshadow) & 7) == 0;
    if (scratch) vec_ok = vec_ok && (reinterpret_cast<uintptr_t>(scratch) & 15) == 0;
    const AvgFn fk = vec_ok ? avg4_pick(k, std::make_integer_sequence<int, 32>{}) : nullptr;
    const AvgFn f1 = vec_ok ? avg4_pick(1, std::make_integer_sequence<int, 32>{}) : nullptr;
    ncclComm_t cm = comm ? static_cast<ncclComm_t>(comm->comm) : nullptr;
    // m == 1 without a communicator: x * 1.0 is the identity (parallel.cpp:56-57)
    if (!work) {
        for (Replica* r : reps) r->last_recorded = false;
        return;
    }
    // a replica whose last step was not launched as a window end (GATE_REC) has no
    // per-layer update events: wait for the whole step instead
    for (Replica* r : reps)
        if (!r->last_recorded) {
            CUDA_THROW(cudaEventRecord(r->ev_tail, r->stream));
            CUDA_THROW(cudaStreamWaitEvent(s, r->ev_tail, 0));
        }
    for (int l = L - 1; l >= 0; --l) {
        for (Replica* r : reps)
            if (r->last_recorded) CUDA_THROW(cudaStreamWaitEvent(s, r->ev_upd[l], 0));
        const long off = reps[0]->bucket_begin(l), len = reps[0]->bucket_end(l) - off;
        const int grid = static_cast<int>(std::min<long>(ctx->num_sms * 8L, std::max<long>(1, (len / 4 + 255) / 256)));
        if (!comm) {
            // local midpoint tree over the replicas x 1/m -> every replica (+ bf16 copy)
            if (fk) fk<<<grid, 256, 0, s>>>(d_src, off, len, inv, 1, d_src, d_shadow, k);
            else tree_avg_kernel<<<grid, 256, 0, s>>>(d_src, k, off, len, inv, 1, d_src, d_shadow, k);
        } else if (k == 1) {
            // one replica per GPU: in-place ncclAvg fuses the 1/m scale into the collective
            NCCL_THROW(ncclAllReduce(reps[0]->params + off, reps[0]->params + off, len, ncclFloat, ncclAvg, cm, s));
            if (reps[0]->wshadow) {
                if (f1) f1<<<grid, 256, 0, s>>>(d_src, off, len, 1.f, 0, d_src, d_shadow, 1);
                else tree_avg_kernel<<<grid, 256, 0, s>>>(d_src, 1, off, len, 1.f, 0, d_src, d_shadow, 1);
            }
        } else {
            // local subtree sum -> scratch (no shadow), NCCL sum over GPUs, then the
            // fused scale pass: scratch x 1/m -> every local replica and its bf16 copy
            if (fk) fk<<<grid, 256, 0, s>>>(d_src, off, len, 1.f, 0, d_scratch_ptr, d_null_shadow, 1);
            else tree_avg_kernel<<<grid, 256, 0, s>>>(d_src, k, off, len, 1.f, 0, d_scratch_ptr, d_null_shadow, 1);
            NCCL_THROW(ncclAllReduce(scratch + off, scratch + off, len, ncclFloat, ncclSum, cm, s));
            if (f1) f1<<<grid, 256, 0, s>>>(d_scratch_ptr, off, len, inv, 1, d_src, d_shadow, k);
            else tree_avg_kernel<<<grid, 256, 0, s>>>(d_scratch_ptr, 1, off, len, inv, 1, d_src, d_shadow, k);
        }
        for (Replica* r : reps) CUDA_THROW(cudaEventRecord(r->ev_gate[l], s));
    }
    for (Replica* r : reps) {
        r->gate_pending = true;  // the next step waits on the gates
        r->last_recorded = false;
    }
    CUDA_THROW(cudaGetLastError());
}

}  // namespace pnb
