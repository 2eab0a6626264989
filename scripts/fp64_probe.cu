// FP64 vs FP32 FMA throughput/latency on this part (one SM).
#include <cstdio>
#include <cuda_runtime.h>
template <typename T, int ILP>
__global__ void k(T* out, long long* cyc, int iters) {
    T a[ILP];
    for (int i = 0; i < ILP; ++i) a[i] = (T)(threadIdx.x + i) * (T)1e-3;
    const T b = (T)0.999, c = (T)1e-4;
    __syncthreads();
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) a[i] = a[i] * b + c;
    __syncthreads();
    long long c1 = clock64();
    T s = 0;
    for (int i = 0; i < ILP; ++i) s += a[i];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = c1 - c0;
}
int main() {
    double* o; long long* cyc; cudaMalloc(&o, 8 * 1024); cudaMalloc(&cyc, 8);
    const int iters = 4096;
    for (int threads : {32, 128, 512, 1024}) {
        long long c;
        k<double, 8><<<1, threads>>>(o, cyc, iters); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        double d_per = (double)c / (iters * 8);  // cycles per dependent-ILP slot
        double d_rate = (double)threads * iters * 8 / c;  // DFMA per clock per SM
        k<float, 8><<<1, threads>>>((float*)o, cyc, iters); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        double f_rate = (double)threads * iters * 8 / c;
        printf("threads %4d: fp64 %.2f FMA/clk/SM (%.1f clk per 8-ILP step)   fp32 %.2f FMA/clk/SM\n", threads, d_rate,
               d_per * 8, f_rate);
    }
    return 0;
}
