// Microbenchmarks of the fp64 / shuffle constants K1 depends on (B200):
// dependent-chain latency (1 warp) and throughput (many warps per SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench exp/ubench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void lat_dfma(double *out, long long *cyc, double a, double b) {
    double x = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_dadd(double *out, long long *cyc, double a) {
    double x = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = x + a;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_shfl(double *out, long long *cyc, double a) {
    double x = threadIdx.x;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N / 4; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_div(double *out, long long *cyc, double a) {
    double x = threadIdx.x + 1.5;
    long long t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < N / 16; ++i) x = a / x + 1.0;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput: 8 independent chains per thread
__global__ void tput_dfma(double *out, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void tput_dsetp_sel(double *out, double a, double b) {
    double x[8];
    unsigned m = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            x[k] = x[k] >= a ? b : x[k] + a;
        }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + m;
}

int main() {
    double *out;
    long long *cyc, h;
    cudaMalloc(&out, 1 << 26);
    cudaMalloc(&cyc, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        lat_dfma<<<1, 32>>>(out, cyc, 1.0000001, 1e-9);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("DFMA dependent latency: %.2f cyc\n", (double)h / N);
        lat_dadd<<<1, 32>>>(out, cyc, 1e-9);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("DADD dependent latency: %.2f cyc\n", (double)h / N);
        lat_shfl<<<1, 32>>>(out, cyc, 1e-9);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("SHFL.f64 + DADD dependent step: %.2f cyc\n", (double)h / (N / 4));
        lat_div<<<1, 32>>>(out, cyc, 3.0);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("fp64 a/x + 1 dependent: %.2f cyc\n", (double)h / (N / 16));
        for (int warps : {4, 8, 16, 32}) {
            const int blocks = 148;
            cudaEventRecord(e0);
            tput_dfma<<<blocks, 32 * warps>>>(out, 1.0000001, 1e-9);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double flops = 2.0 * 8 * N * blocks * 32 * warps;
            printf("DFMA tput %2d warps/SM: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
            cudaEventRecord(e0);
            tput_dsetp_sel<<<blocks, 32 * warps>>>(out, 0.5, 1e-9);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            double ops = 8.0 * N * blocks * 32 * warps;
            printf("DSETP+DADD+sel tput %2d warps/SM: %.2f Gop/s (%.3f ns per warp-op-triple per SM)\n", warps,
                   ops / ms / 1e6, ms * 1e6 / (8.0 * N * warps));
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
