// Microbenchmark of one-sided Jacobi rounds (fp64, half-warp per column pair):
// cycles per round for variants of the pair computation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/jacobi_bench.bin scripts/jacobi_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void rounds(int n, int nround, double* out, long long* cyc) {
    extern __shared__ double Bc[];
    const int t = threadIdx.x, h = n / 2, ldb = n;
    for (int i = t; i < n * n; i += blockDim.x) Bc[i] = 1.0 / (1 + (i % 97)) + (i % n == i / n ? 10.0 : 0.0);
    __syncthreads();
    const int hw = t >> 4, hl = t & 15, nhw = blockDim.x >> 4;
    const unsigned hmask = 0xFFFFu << (t & 16);
    long long c0 = clock64();
    for (int k = 0; k < nround; ++k) {
        for (int pr = hw; pr < h; pr += nhw) {
            int p, q;
            if (MODE >= 4) {  // pair table: no integer modulo
                p = pr;
                q = (pr + 1 + (k & 7)) % n == pr ? (pr + 1) % n : h + pr;
            } else {
                const int kk = k % (n - 1);
                if (pr == 0) { p = 0; q = kk + 1; }
                else { p = ((pr + kk) % (n - 1)) + 1; q = ((n - 1 - pr + kk) % (n - 1)) + 1; }
            }
            double* cp = Bc + p * ldb;
            double* cq = Bc + q * ldb;
            double al = 0, be = 0, ga = 0;
            for (int r = hl; r < n; r += 16) {
                const double x = cp[r], y = cq[r];
                al = fma(x, x, al); be = fma(y, y, be); ga = fma(x, y, ga);
            }
            if (MODE != 1) {
#pragma unroll
                for (int o = 8; o; o >>= 1) {
                    al += __shfl_xor_sync(hmask, al, o, 16);
                    be += __shfl_xor_sync(hmask, be, o, 16);
                    ga += __shfl_xor_sync(hmask, ga, o, 16);
                }
            }
            double c = 0.9, sn = 0.1;
            if (MODE == 0 || MODE == 1) {  // full fp64 angle
                if (fabs(ga) > 1e-13 * sqrt(al * be)) {
                    const double zeta = (be - al) / (2.0 * ga);
                    const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    c = 1.0 / sqrt(1.0 + tt * tt);
                    sn = c * tt;
                }
            } else if (MODE == 3) {  // fp32 angle + fp64 Newton
                if (ga * ga > 1e-26 * al * be) {
                    const float zeta = (float)((be - al) * __drcp_rn(2.0 * ga));
                    const float az = fabsf(zeta);
                    const float tf = 1.f / (az + sqrtf(fmaf(az, az, 1.f)));
                    const double tt = zeta >= 0.f ? (double)tf : -(double)tf;
                    const double w = fma(tt, tt, 1.0);
                    c = (double)rsqrtf((float)w);
                    c = c * (1.5 - 0.5 * w * c * c);
                    c = c * (1.5 - 0.5 * w * c * c);
                    sn = c * tt;
                }
            }
            // MODE 2: no angle math at all
            if (MODE != 5) for (int r = hl; r < n; r += 16) {
                const double x = cp[r], y = cq[r];
                cp[r] = c * x - sn * y;
                cq[r] = sn * x + c * y;
            }
        }
        if (MODE != 6) __syncthreads();
    }
    long long c1 = clock64();
    if (t == 0) { *cyc = (c1 - c0) / nround; *out = Bc[5]; }
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
    for (int n : {20, 80}) {
        const int threads = std::max(64, (n / 2 * 16 + 31) / 32 * 32);
        const size_t sm = n * n * 8;
        auto run = [&](auto kern, const char* name) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            kern<<<1, threads, sm>>>(n, 400, out, cyc);
            long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("n=%d threads=%d %-28s %lld cycles/round (%s)\n", n, threads, name, c, cudaGetErrorString(cudaGetLastError()));
        };
        run(rounds<0>, "fp64 full");
        run(rounds<1>, "no shuffle");
        run(rounds<2>, "no angle math");
        run(rounds<3>, "fp32 angle + newton");
        run(rounds<4>, "fixed pairs, no angle");
        run(rounds<5>, "fixed pairs, no rotate");
        run(rounds<6>, "fixed pairs no angle no sync");
    }
    return 0;
}
