// Per-CTA phase timeline of the tcgen05 GEMM (globaltimer stamps, -DPNB_GEMM_TRACE)
// for the trainer's hidden-layer shapes with their real epilogues, warm and cold L2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DPNB_GEMM_TRACE \
//     -I paper_1507_01239_b200/csrc -I include scripts/gemm_trace.cu -o scripts/gemm_trace.bin -lcuda
#include <algorithm>
#include <cstdio>
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

__global__ void fill_random_bf16(__nv_bfloat16* p, long n, unsigned seed) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        unsigned long long x = i * 0x9E3779B97F4A7C15ull + seed;
        x ^= x >> 33;
        x *= 0xff51afd7ed558ccdull;
        x ^= x >> 33;
        p[i] = __float2bfloat16((float)((x >> 40) & 0xFFFFFF) / 8388608.0f - 1.0f);
    }
}

int main() {
    const int M = 1024, N = 2048, K = 2048;
    void *A, *Bm, *out, *flush;
    float *w32, *bias;
    cudaMalloc(&A, 8192L * 8192 * 2);
    cudaMalloc(&Bm, 8192L * 8192 * 2);
    cudaMalloc(&out, 8192L * 8192 * 4);
    cudaMalloc(&w32, 8192L * 8192 * 4);
    cudaMalloc(&bias, 65536 * 4);
    const size_t fl = 400L << 20;
    cudaMalloc(&flush, fl);
    // random operands (zeros under-load the tensor cores)
    fill_random_bf16<<<1184, 256>>>(static_cast<__nv_bfloat16*>(A), 8192L * 8192, 1);
    fill_random_bf16<<<1184, 256>>>(static_cast<__nv_bfloat16*>(Bm), 8192L * 8192, 2);
    cudaMemset(bias, 0, 65536 * 4);
    float* lr;
    int* step;
    cudaMalloc(&lr, 64);
    cudaMalloc(&step, 64);
    cudaMemset(lr, 0, 64);
    cudaMemset(step, 0, 64);
    struct Case {
        const char* name;
        bool amn, bmn;
        int M, N, K;
        int mode;
    };
    std::vector<Case> cases = {{"fwd  1024x2048x2048 FWD_ACT", false, false, 1024, 2048, 2048, EPI_FWD_ACT},
                               {"dA   1024x2048x2048 ACTGRAD", false, true, 1024, 2048, 2048, EPI_ACTGRAD},
                               {"dW   2048x2048x1024 GRAD_SGD", true, true, 2048, 2048, 1024, EPI_GRAD_SGD},
                               {"dW   2048x2048x1024 GRAD", true, true, 2048, 2048, 1024, EPI_GRAD},
                               {"dW128 2048x2048x1024 GRAD_SGD", true, true, 2048, 2048, 1024, 100 + EPI_GRAD_SGD},
                               {"dAout 1024x2048x8806 ACTGRAD", false, true, 1024, 2048, 8806, EPI_ACTGRAD}};
    for (auto& c : cases) {
        GemmEpi e;
        const int force_bn = c.mode >= 100 ? 128 : 0;
        e.mode = c.mode % 100;
        e.act = 0;
        e.out = out;
        e.ld_out = (c.N + 31) / 32 * 32;
        e.bias = bias;
        e.aux = A;
        e.ld_aux = (c.N + 31) / 32 * 32;
        e.out32 = w32;
        e.ld_out32 = (c.N + 31) / 32 * 32;
        e.shadow = static_cast<__nv_bfloat16*>(out);
        e.ld_shadow = (c.N + 31) / 32 * 32;
        e.lr = lr;
        e.step = step;
        e.alpha = 1e-3f;
        GemmPlan p;
        long lda = ((c.amn ? c.M : c.K) + 31) / 32 * 32, ldb = ((c.bmn ? c.N : c.K) + 31) / 32 * 32;
        gemm_plan(p, 0, c.amn, A, lda, c.bmn, Bm, ldb, c.M, c.N, c.K, e, 148, force_bn);
        for (int cold = 0; cold < 2; ++cold) {
            for (int rep = 0; rep < 3; ++rep) {
                if (cold) cudaMemset(flush, rep, fl);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                gemm_launch(p, 0);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep < 2) continue;
                unsigned long long tr[1024][12];
                cudaMemcpyFromSymbol(tr, g_gemm_trace, sizeof(tr));
                const int g = p.grid.x;
                unsigned long long t0 = ~0ull;
                for (int b = 0; b < g; ++b) t0 = std::min(t0, tr[b][0]);
                printf("%-30s %s grid=%d bn=%d  %.2f us (events)\n", c.name, cold ? "cold" : "warm", g, p.bn, ms * 1e3);
                const char* nm[10] = {"entry", "setup", "first-data", "last-mma", "acc-ready", "epi-done", "exit", "sent", "recv(w2)", "chunks(w2)"};
                for (int i = 0; i < 10; ++i) {
                    double mn = 1e30, mx = 0, av = 0;
                    for (int b = 0; b < g; ++b) {
                        const double v = (tr[b][i] - t0) * 1e-3;
                        mn = std::min(mn, v);
                        mx = std::max(mx, v);
                        av += v / g;
                    }
                    printf("   %-11s min %7.2f  avg %7.2f  max %7.2f us\n", nm[i], mn, av, mx);
                }
            }
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
