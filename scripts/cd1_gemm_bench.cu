// CD-1 GEMM shapes (batch 128 against a 2048 x 2048 RBM): warm back-to-back
// time per launch (CUDA events, 50 reps; PDL overlaps consecutive launches
// unless PARNN_NO_PDL=1) for split-K factors and tile widths, and the K = 256
// weight update. Empty-kernel launch rate for the floor.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1507_01239_b200/csrc -I include \
//   scripts/cd1_gemm_bench.cu -o scripts/cd1_gemm_bench.bin -lcuda
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

__global__ void fill(float* p, long n, float s) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        p[i] = s * (float)((i * 2654435761u) % 1000) / 1000.f;
}
__global__ void fillh(__nv_bfloat16* p, long n, float s) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        p[i] = __float2bfloat16(s * (float)((i * 2654435761u) % 1000) / 1000.f);
}
__global__ void empty_kernel() {}

bool g_graph = false;

double time_plan(GemmPlan& p, cudaStream_t s) {
    if (g_graph) {  // 50 launches captured into one graph, replayed
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < 50; ++i) gemm_launch(p, s);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        for (int i = 0; i < 2; ++i) cudaGraphLaunch(ge, s);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        for (int i = 0; i < 4; ++i) cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
        return ms * 1e3 / 200;
    }
    for (int i = 0; i < 5; ++i) gemm_launch(p, s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    const int reps = 50;
    for (int i = 0; i < reps; ++i) gemm_launch(p, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e3 / reps;
}

int main(int argc, char** argv) {
    g_graph = argc > 1 && argv[1][0] == 'g';
    const long n = 4096L * 4096;
    void *A, *B, *C;
    cudaMalloc(&A, n * 4);
    cudaMalloc(&B, n * 4);
    cudaMalloc(&C, 32 * n * 4);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    {
        for (int i = 0; i < 5; ++i) empty_kernel<<<1, 32, 0, s>>>();
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        for (int i = 0; i < 200; ++i) empty_kernel<<<148, 128, 0, s>>>();
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("empty kernel launch: %.2f us each (back to back)\n", ms * 1e3 / 200);
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < 200; ++i) empty_kernel<<<148, 128, 0, s>>>();
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(e0, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("empty kernel in a graph: %.2f us each\n", ms * 1e3 / 200);
    }
    for (int prec : {0, 1, 2}) {
        if (prec == 0) {
            fillh<<<1184, 256>>>((__nv_bfloat16*)A, n, 1.f);
            fillh<<<1184, 256>>>((__nv_bfloat16*)B, n, 0.01f);
        } else {
            fill<<<1184, 256>>>((float*)A, n, 1.f);
            fill<<<1184, 256>>>((float*)B, n, 0.01f);
        }
        const int M = 128, N = 2048, K = 2048;
        const double flop = 2.0 * M * N * K;
        for (int bn : {64, 128, 256}) {
            for (int ks : {1, 2, 4, 8, 16, 32}) {
                GemmEpi e;
                e.mode = ks == 1 ? EPI_FWD_LINEAR : EPI_PARTIAL;
                e.out32 = (float*)C;
                e.ld_out32 = N;
                e.split_stride = (long)M * N;
                e.ksplit = ks;
                e.bias = (float*)C + 31 * n;
                GemmPlan p;
                try {
                    gemm_plan(p, prec, false, A, K, false, B, K, M, N, K, e, 148, bn);
                } catch (std::exception& ex) {
                    continue;
                }
                const double us = time_plan(p, s);
                printf("prec %d  X W^T 128x2048x2048 bn %3d ksplit %2d grid %3d: %6.2f us  %6.1f TFLOP/s %s\n", prec, bn,
                       p.ep.ksplit, gemm_launch_grid(p).x, us, flop / us / 1e6, cudaGetErrorString(cudaGetLastError()));
            }
        }
        for (int bn : {64, 128, 256}) {
            GemmEpi u;
            u.mode = EPI_AXPY;
            u.out32 = (float*)C;
            u.ld_out32 = 2048;
            u.alpha = 0.f;
            u.shadow = prec == 0 ? (__nv_bfloat16*)((float*)C + 8 * n) : nullptr;
            u.ld_shadow = 2048;
            GemmPlan p;
            try {
                gemm_plan(p, prec, true, A, 2048, true, B, 2048, 2048, 2048, 256, u, 148, bn);
            } catch (std::exception& ex) {
                continue;
            }
            const double us = time_plan(p, s);
            printf("prec %d  update 2048x2048x256 AXPY bn %3d grid %3d: %6.2f us  %6.1f TFLOP/s %s\n", prec, bn,
                   gemm_launch_grid(p).x, us, 2.0 * 2048 * 2048 * 256 / us / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
