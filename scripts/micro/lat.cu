// Dependent-chain latency microbenchmarks on B200 (one warp, clock64 deltas).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double *out, long long *cyc, int n, double a, double b) {
    __shared__ double sh[64];
    const int lane = threadIdx.x;
    sh[lane] = lane * 1.0; sh[lane + 32] = 1.0;
    __syncwarp();
    double x = lane * 1e-3 + 1.0;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, a, b);
    t1 = clock64(); if (lane == 0) cyc[0] = (t1 - t0);
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x * a;
    t1 = clock64(); if (lane == 0) cyc[1] = (t1 - t0);
    // SHFL 64-bit chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffff, x, (lane + 1) & 31);
    t1 = clock64(); if (lane == 0) cyc[2] = (t1 - t0);
    // SHFL 32-bit chain
    int y = lane;
    t0 = clock64();
    for (int i = 0; i < n; ++i) y = __shfl_sync(0xffffffff, y, (y + 1) & 31);
    t1 = clock64(); if (lane == 0) cyc[3] = (t1 - t0);
    // LDS chain (pointer chase through shared memory)
    int idx = lane;
    int *shi = (int *)sh;
    shi[lane] = (lane + 1) & 31;
    __syncwarp();
    t0 = clock64();
    for (int i = 0; i < n; ++i) idx = shi[idx];
    t1 = clock64(); if (lane == 0) cyc[4] = (t1 - t0);
    // sqrt + div chain (IEEE)
    double z = 2.0 + lane;
    t0 = clock64();
    for (int i = 0; i < n; ++i) z = 1.0 / sqrt(z + 1.0);
    t1 = clock64(); if (lane == 0) cyc[5] = (t1 - t0);
    // stage-like chain: DMUL -> SHFL -> DFMA
    double t = 1.0 + lane;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { double l = __shfl_sync(0xffffffff, t * a, i & 31); t = fma(-l, b, t); }
    t1 = clock64(); if (lane == 0) cyc[6] = (t1 - t0);
    out[lane] = x + y + idx + z + t;
}
int main() {
    double *out; long long *cyc, h[8];
    cudaMalloc(&out, 64 * 8); cudaMalloc(&cyc, 8 * 8);
    const int n = 4096;
    for (int r = 0; r < 2; ++r) lat<<<1, 32>>>(out, cyc, n, 0.9999999, 1e-9);
    cudaMemcpy(h, cyc, 8 * 8, cudaMemcpyDeviceToHost);
    const char *nm[] = {"DFMA", "DMUL", "SHFL64", "SHFL32", "LDS", "sqrt+div", "DMUL->SHFL->DFMA"};
    for (int k = 0; k < 7; ++k) printf("%-18s %.1f cycles/op\n", nm[k], (double)h[k] / n);
    return 0;
}
