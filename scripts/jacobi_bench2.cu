// Cycles per Jacobi round for incremental variants (fp64, n=80, 640 threads).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void rounds(int n, int nround, double* out, long long* cyc) {
    extern __shared__ double Bc[];
    const int t = threadIdx.x, h = n / 2, ldb = n;
    for (int i = t; i < n * n; i += blockDim.x) Bc[i] = 1.0 / (1 + (i % 97));
    __syncthreads();
    const int hw = t >> 4, hl = t & 15;
    double acc = 0;
    long long c0 = clock64();
    for (int k = 0; k < nround; ++k) {
        const int p = hw % h, q = (hw + 1 + (k & 3)) % h + (hw < h ? 0 : 0);
        double al = 0, be = 0, ga = 0;
        if (MODE >= 1) {
            const double* cp = Bc + p * ldb;
            const double* cq = Bc + (h + q) * ldb % (n * ldb);
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                const int r = hl + 16 * i;
                const double x = r < n ? cp[r] : 0.0, y = r < n ? cq[r] : 0.0;
                al = fma(x, x, al); be = fma(y, y, be); ga = fma(x, y, ga);
            }
        }
        if (MODE >= 2) {
#pragma unroll
            for (int o = 8; o; o >>= 1) {
                al += __shfl_xor_sync(0xffffffffu, al, o, 16);
                be += __shfl_xor_sync(0xffffffffu, be, o, 16);
                ga += __shfl_xor_sync(0xffffffffu, ga, o, 16);
            }
        }
        if (MODE >= 3) {
            double* cp = Bc + p * ldb;
            double* cq = Bc + (h + q) * ldb % (n * ldb);
            const double c = 1.0 / sqrt(1.0 + ga * ga * 1e-30), s = 1e-3 * c;
            if (hw < h)
#pragma unroll
                for (int i = 0; i < 5; ++i) {
                    const int r = hl + 16 * i;
                    if (r < n) {
                        const double x = cp[r], y = cq[r];
                        cp[r] = c * x - s * y;
                        cq[r] = s * x + c * y;
                    }
                }
        }
        acc += al + be + ga;
        if (MODE != 4) __syncthreads();
    }
    long long c1 = clock64();
    if (t == 0) { *cyc = (c1 - c0) / nround; }
    out[t] = acc;
}
int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 8 * 1024); cudaMalloc(&cyc, 8);
    const int n = 80, threads = 640;
    const size_t sm = n * n * 8;
    auto run = [&](auto kern, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        kern<<<1, threads, sm>>>(n, 400, out, cyc);
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-36s %lld cycles/round (%s)\n", name, c, cudaGetErrorString(cudaGetLastError()));
    };
    run(rounds<0>, "sync only");
    run(rounds<1>, "+ dot loads");
    run(rounds<2>, "+ shuffles (full mask)");
    run(rounds<3>, "+ rotation");
    run(rounds<4>, "all, no sync");
    return 0;
}
