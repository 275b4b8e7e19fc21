// FP64 pipe microbenchmark: measures DFMA / DADD / DSQRT throughput on the
// device so the FFT roofline has a measured FP64 denominator (the driver's
// MEASURED_PEAKS.json carries no FP64 figure).
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dadd_kernel(double* out, int iters, double a) {
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) x[c] = x[c] + a;
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dsqrt_kernel(float* out, int iters) {
    double x[CHAINS];
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c + 1.5;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            acc += __double2float_rn(__dsqrt_rn(x[c]));
            x[c] += 1.0;
        }
    }
    if (acc == 12345.678f) out[0] = acc;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* d;
    cudaMalloc(&d, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int threads = 256, blocks = sms * 8, iters = 4096;
    const int chains = 8;
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
        dfma_kernel<chains><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
        cudaEventRecord(e0);
        dfma_kernel<chains><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)blocks * threads * iters * chains;
        printf("DFMA: %.3f ms  %.2f Gop/s  %.2f TFLOP/s  (%.1f ops/clk/SM @ %d MHz max)\n", ms,
               ops / ms * 1e-6, 2 * ops / ms * 1e-9, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
        dadd_kernel<chains><<<blocks, threads>>>(d, iters, 1e-7);
        cudaEventRecord(e0);
        dadd_kernel<chains><<<blocks, threads>>>(d, iters, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("DADD: %.3f ms  %.2f Gop/s\n", ms, ops / ms * 1e-6);
        dsqrt_kernel<chains><<<blocks, threads>>>((float*)d, iters / 8);
        cudaEventRecord(e0);
        dsqrt_kernel<chains><<<blocks, threads>>>((float*)d, iters / 8);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("DSQRT_RN+cvt: %.3f ms  %.2f Gop/s\n", ms, ops / 8 / ms * 1e-6);
    }
    cudaError_t err = cudaGetLastError();
    printf("err=%s\n", cudaGetErrorString(err));
    return 0;
}
