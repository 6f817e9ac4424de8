// fp64 FMA throughput per SM (independent chains, many warps), plus the
// throughput of DMUL, SHFL and LDS, in instructions per cycle per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__global__ void dfma_t(double *out, long long *cyc, int n) {
    double x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (K == 0) x[k] = fma(x[k], 0.999999, 1e-9);
            if (K == 1) x[k] = __shfl_xor_sync(0xffffffff, x[k], 1);
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    double s = 0; for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 1.2345) out[0] = s;
}
int main() {
    double *out; long long *cyc, h;
    cudaMalloc(&out, 8); cudaMalloc(&cyc, 148 * 8 * 8);
    const int n = 2048;
    for (int warps = 4; warps <= 32; warps *= 2) {
        dfma_t<0><<<148, warps * 32>>>(out, cyc, n); cudaDeviceSynchronize();
        dfma_t<0><<<148, warps * 32>>>(out, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        double ops = (double)n * 8 * warps;  // warp-instructions per SM
        printf("DFMA  warps/SM %2d: %.3f warp-inst/clk/SM = %.1f FMA/clk/SM\n", warps, ops / h, 32 * ops / h);
        dfma_t<1><<<148, warps * 32>>>(out, cyc, n); cudaDeviceSynchronize();
        dfma_t<1><<<148, warps * 32>>>(out, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("SHFL64 warps/SM %2d: %.3f warp-inst/clk/SM\n", warps, ops / h);
    }
    return 0;
}
