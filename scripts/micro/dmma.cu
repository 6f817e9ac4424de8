// Does the fp64 tensor core (DMMA, mma.sync m8n8k4 f64) pay off for the set-up?
// BASELINE.json north_star: "tensor cores (DMMA) used only if measured to pay off at
// these tiny block sizes".  Measures, per SM, with independent accumulator chains:
//   (1) DFMA throughput (FMA/clk/SM),
//   (2) DMMA m8n8k4 throughput in fp64 FMA/clk/SM (256 FMAs per warp-level mma),
//   (3) DMMA dependent-chain latency (cycles per mma, one warp),
//   (4) DFMA dependent-chain latency.
// Also whether DMMA's k=4 dot product rounds like four sequential fma() (the
// arithmetic contract's fold, C5-C7) on adversarial inputs.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/dmma scripts/micro/dmma.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <int CH>
__global__ void dmma_tput(double *out, long long *cyc, int n) {
    double acc[CH][2];
    const double a = 1.0 + threadIdx.x * 1e-7, b = 0.999999;
    for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = c;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) dmma(acc[c], a, b);
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    double s = 0;
    for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
    if (s == 1.2345) out[0] = s;
}

__global__ void dfma_tput(double *out, long long *cyc, int n) {
    double x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], 0.999999, 1e-9);
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    double s = 0;
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 1.2345) out[0] = s;
}

// rounding: lane layout of m8n8k4 (row A 8x4, col B 4x8): A[g][t] held by lane 4g+t,
// B[t][g] by lane 4g+t; C/D[g][2t], [g][2t+1] by lane 4g+t.
__global__ void dmma_round(const double *A, const double *B, const double *C, double *D) {
    const int lane = threadIdx.x;
    const int g = lane >> 2, t = lane & 3;
    double d[2] = {C[g * 8 + 2 * t], C[g * 8 + 2 * t + 1]};
    dmma(d, A[g * 4 + t], B[t * 8 + g]);
    D[g * 8 + 2 * t] = d[0];
    D[g * 8 + 2 * t + 1] = d[1];
}

int main() {
    double *out;
    long long *cyc, h;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 148 * 8 * 8);
    const int n = 4096;
    printf("# per SM, 148 CTAs of W warps\n");
    for (int warps = 4; warps <= 32; warps *= 2) {
        dfma_tput<<<148, warps * 32>>>(out, cyc, n);
        dfma_tput<<<148, warps * 32>>>(out, cyc, n);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        const double fma_dfma = 32.0 * 8 * n * warps / h;
        dmma_tput<4><<<148, warps * 32>>>(out, cyc, n);
        dmma_tput<4><<<148, warps * 32>>>(out, cyc, n);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        const double fma_dmma = 256.0 * 4 * n * warps / h;
        printf("warps/SM %2d: DFMA %.1f FMA/clk/SM   DMMA m8n8k4 %.1f FMA/clk/SM (%.3f mma/clk/SM)\n", warps, fma_dfma,
               fma_dmma, fma_dmma / 256.0);
    }
    // latency: one warp, dependent chain
    dmma_tput<1><<<1, 32>>>(out, cyc, n);
    dmma_tput<1><<<1, 32>>>(out, cyc, n);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DMMA dependent-chain latency: %.1f cycles per mma (one warp)\n", (double)h / n);
    dfma_tput<<<1, 32>>>(out, cyc, n);
    dfma_tput<<<1, 32>>>(out, cyc, n);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent-chain: %.1f cycles per 8 independent fma (one warp; latency ~ this / 1)\n", (double)h / n);
    // rounding order: d = c + sum_t a_t b_t vs the sequential fma fold of the contract
    double hA[32], hB[32], hC[64], hD[64];
    unsigned long long st = 12345;
    auto rnd = [&]() {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        return ((double)(st >> 11) / 9007199254740992.0 - 0.5) * std::pow(2.0, (double)((st >> 3) % 60) - 30);
    };
    int diff_seq = 0, diff_rev = 0, total = 0;
    double *dA, *dB, *dC, *dD;
    cudaMalloc(&dA, 256);
    cudaMalloc(&dB, 256);
    cudaMalloc(&dC, 512);
    cudaMalloc(&dD, 512);
    for (int trial = 0; trial < 200; ++trial) {
        for (int k = 0; k < 32; ++k) hA[k] = rnd(), hB[k] = rnd();
        for (int k = 0; k < 64; ++k) hC[k] = rnd();
        cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
        cudaMemcpy(dC, hC, 512, cudaMemcpyHostToDevice);
        dmma_round<<<1, 32>>>(dA, dB, dC, dD);
        cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost);
        for (int g = 0; g < 8; ++g)
            for (int j = 0; j < 8; ++j) {
                double s = hC[g * 8 + j], r = hC[g * 8 + j];
                for (int t = 0; t < 4; ++t) s = std::fma(hA[g * 4 + t], hB[t * 8 + j], s);
                for (int t = 3; t >= 0; --t) r = std::fma(hA[g * 4 + t], hB[t * 8 + j], r);
                diff_seq += s != hD[g * 8 + j];
                diff_rev += r != hD[g * 8 + j];
                ++total;
            }
    }
    printf("DMMA vs sequential fma fold t=0..3: %d of %d results differ; vs t=3..0: %d differ\n", diff_seq, total,
           diff_rev);
    return 0;
}
