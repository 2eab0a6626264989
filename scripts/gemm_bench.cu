// GEMM microbenchmark over the trainer's shapes on RANDOM operands (uniform in
// [-1, 1) from a hash, values of the operand type; zero operands under-load the
// tensor cores' power and are not comparable with the measured peaks):
// back-to-back launches (warm L2, CUDA events, 20 reps) and single launches
// after a 400 MB L2 flush (cold).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1507_01239_b200/csrc -I include \
//   scripts/gemm_bench.cu -o scripts/gemm_bench.bin
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1507_01239_b200/csrc/gemm.cu"
#include "../paper_1507_01239_b200/csrc/gemm_k_bf16_r.cu"
#include "../paper_1507_01239_b200/csrc/gemm_k_bf16_t.cu"
#include "../paper_1507_01239_b200/csrc/gemm_k_f32_r.cu"
#include "../paper_1507_01239_b200/csrc/gemm_k_f32_t.cu"
#include "../paper_1507_01239_b200/csrc/gemm_k_split_r.cu"
#include "../paper_1507_01239_b200/csrc/gemm_k_split_t.cu"
#include "../paper_1507_01239_b200/csrc/gemm_k_bf16_r_mc.cu"
#include "../paper_1507_01239_b200/csrc/gemm_k_bf16_t_mc.cu"
#include "../paper_1507_01239_b200/csrc/gemm_k_bf16_r_sk.cu"
#include "../paper_1507_01239_b200/csrc/gemm_k_bf16_t_sk.cu"
#include "../paper_1507_01239_b200/csrc/gemm_k_group.cu"
using namespace pnb;

__device__ __forceinline__ float hash_uniform(unsigned long long i, unsigned seed) {
    unsigned long long x = i * 0x9E3779B97F4A7C15ull + seed;
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    return (float)((x >> 40) & 0xFFFFFF) / 8388608.0f - 1.0f;
}
template <typename T>
__global__ void fill_random(T* p, long n, unsigned seed, float scale) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        p[i] = (T)(scale * hash_uniform(i, seed));
}

int main(int argc, char** argv) {
    int bnf = argc > 1 ? atoi(argv[1]) : 0;
    struct Case { const char* name; int prec; bool amn, bmn; int M, N, K; int mode; };
    std::vector<Case> cases = {
        {"fwd hidden 1024x2048x2048 ACT ", 0, false, false, 1024, 2048, 2048, EPI_FWD_ACT},
        {"fwd out    1024x8806x2048 LIN ", 0, false, false, 1024, 8806, 2048, EPI_FWD_LINEAR},
        {"dW hidden  2048x2048x1024 SGD ", 0, true, true, 2048, 2048, 1024, EPI_GRAD_SGD},
        {"dW out     8806x2048x1024 SGD ", 0, true, true, 8806, 2048, 1024, EPI_GRAD_SGD},
        {"dA hidden  1024x2048x2048 AGR ", 0, false, true, 1024, 2048, 2048, EPI_ACTGRAD},
        {"dA out     1024x2048x8806 AGR ", 0, false, true, 1024, 2048, 8806, EPI_ACTGRAD},
        {"dW hidden  2048x2048x1024 GRAD", 0, true, true, 2048, 2048, 1024, EPI_GRAD},
        {"big        8192x8192x8192 GRAD", 0, false, false, 8192, 8192, 8192, EPI_GRAD},
        {"f32 trsm   8678x2049x128  SUB ", 2, false, true, 8678, 2049, 128, EPI_SUB},
        {"f32 trail  8678x8678x128  SUB ", 2, false, false, 8678, 8678, 128, EPI_SUB},
    };
    void *A, *B;
    float* C;
    size_t maxe = 8192L * 8192;
    cudaMalloc(&A, maxe * 4);
    cudaMalloc(&B, maxe * 4);
    cudaMalloc(&C, maxe * 4);
    void *C2, *C3;
    float* bias;
    cudaMalloc(&C2, maxe * 4);
    cudaMalloc(&C3, maxe * 4);
    cudaMalloc(&bias, 65536 * 4);
    cudaMemset(C, 0, maxe * 4);
    cudaMemset(C2, 0, maxe * 4);
    cudaMemset(C3, 0, maxe * 4);
    cudaMemset(bias, 0, 65536 * 4);
    int sms = 148;
    void* flush;
    const size_t fl = 400L << 20;
    cudaMalloc(&flush, fl);
    fill_random<float><<<1184, 256>>>(bias, 65536, 7, 0.1f);
    fill_random<float><<<1184, 256>>>(C, maxe, 9, 1.0f);  // fp32 master weights / factors
    fill_random<__nv_bfloat16><<<1184, 256>>>(static_cast<__nv_bfloat16*>(C3), maxe, 11, 0.5f);  // activations
    const int only = argc > 2 ? atoi(argv[2]) : -1;  // run one case (profiling)
    for (size_t ci = 0; ci < cases.size(); ++ci) {
        auto& c = cases[ci];
        if (only >= 0 && static_cast<int>(ci) != only) continue;
        if (c.prec == 0) {
            fill_random<__nv_bfloat16><<<1184, 256>>>(static_cast<__nv_bfloat16*>(A), maxe, 1, 1.0f);
            fill_random<__nv_bfloat16><<<1184, 256>>>(static_cast<__nv_bfloat16*>(B), maxe, 2, 1.0f);
        } else {
            fill_random<float><<<1184, 256>>>(static_cast<float*>(A), maxe, 1, 1.0f);
            fill_random<float><<<1184, 256>>>(static_cast<float*>(B), maxe, 2, 1.0f);
        }
        cudaMemset(bias, 0, 64);  // lr[0] = 0: the SGD epilogue leaves the random weights in place
        GemmPlan p;
        GemmEpi e;
        e.mode = c.mode;
        e.out32 = C;
        e.ld_out32 = (c.N + 31) / 32 * 32;
        e.out = C2;
        e.ld_out = e.ld_out32;
        e.aux = C3;
        e.ld_aux = e.ld_out32;
        e.bias = bias;
        e.shadow = static_cast<__nv_bfloat16*>(C2);
        e.ld_shadow = e.ld_out32;
        e.lr = bias;
        e.step = nullptr;
        long lda = c.amn ? (c.M + 31) / 32 * 32 : (c.K + 31) / 32 * 32;
        long ldb = c.bmn ? (c.N + 31) / 32 * 32 : (c.K + 31) / 32 * 32;
        gemm_plan(p, c.prec, c.amn, A, lda, c.bmn, B, ldb, c.M, c.N, c.K, e, sms, bnf);
        cudaStream_t s;
        cudaStreamCreate(&s);
        for (int i = 0; i < 3; ++i) gemm_launch(p, s);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        const int reps = 20;
        for (int i = 0; i < reps; ++i) gemm_launch(p, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double us = ms * 1e3 / reps;
        // cold: one launch after flushing L2
        double cold = 0.0;
        for (int i = 0; i < 3; ++i) {
            cudaMemsetAsync(flush, i, fl, s);
            cudaEventRecord(e0, s);
            gemm_launch(p, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float m1;
            cudaEventElapsedTime(&m1, e0, e1);
            cold += m1 * 1e3 / 3;
        }
        double flop = 2.0 * c.M * c.N * c.K;
        printf("%-28s bn=%3d mc=%d grid=%3d  warm %8.2f us %7.1f TFLOP/s   cold %8.2f us %7.1f TFLOP/s%s  %s\n",
               c.name, p.bn, p.mc, gemm_launch_grid(p).x, us, flop / us / 1e6, cold, flop / cold / 1e6,
               c.prec == 2 ? " (fp32-accurate: 3 TF32 MMAs per product)" : "", cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
