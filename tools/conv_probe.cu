// Probe: F2F throughput vs integer bit-construction, and rsqrt.approx.ftz.f64 accuracy.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsq64(double x) { double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }
__global__ void f2f_kernel(const float* in, double* out, int iters) {
  float x = in[threadIdx.x]; double acc = 0;
  for (int i = 0; i < iters; ++i) { acc += (double)x; x = x * 1.0000001f; acc += (double)x; x = x * 0.9999999f; }
  if (acc == 1.2345) out[0] = acc;
}
__device__ __forceinline__ double f2d_int(float f) {
  unsigned u = __float_as_uint(f);
  unsigned hi = (u & 0x80000000u) | (((u & 0x7fffffffu) >> 3) + 0x38000000u);
  unsigned lo = u << 29;
  return __hiloint2double((int)hi, (int)lo);
}
__global__ void f2i_kernel(const float* in, double* out, int iters) {
  float x = in[threadIdx.x]; double acc = 0;
  for (int i = 0; i < iters; ++i) { acc += f2d_int(x); x = x * 1.0000001f; acc += f2d_int(x); x = x * 0.9999999f; }
  if (acc == 1.2345) out[0] = acc;
}
__global__ void rsq_err(double* maxerr, unsigned long long n) {
  double m = 0;
  for (unsigned long long i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double x = 1.0 + (double)i / n * 3.0;  // [1,4)
    double y = rsq64(x);
    double e = fabs(y * sqrt(x) - 1.0);
    m = fmax(m, e);
  }
  // crude reduce
  unsigned long long* p = (unsigned long long*)maxerr;
  atomicMax(p, __double_as_longlong(m));
}
int main() {
  float* in; double* out; cudaMalloc(&in, 4096); cudaMalloc(&out, 64); cudaMemset(in, 0, 4096);
  float h[1024]; for (int i = 0; i < 1024; ++i) h[i] = 1.0f + i * 1e-3f; cudaMemcpy(in, h, 4096, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); f2f_kernel<<<148*8, 256>>>(in, out, 4096); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    double ops = 148.0*8*256*4096*2; printf("F2F.F64.F32: %.3f ms -> %.1f Gconv/s (%.1f /clk/SM @1.965GHz)\n", ms, ops/ms*1e-6, ops/(ms*1e-3)/148/1.965e9);
    cudaEventRecord(a); f2i_kernel<<<148*8, 256>>>(in, out, 4096); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("int f->d   : %.3f ms -> %.1f Gconv/s\n", ms, ops/ms*1e-6);
  }
  cudaMemset(out, 0, 8); rsq_err<<<1024,256>>>(out, 1ull<<28); double e; cudaMemcpy(&e, out, 8, cudaMemcpyDeviceToHost);
  printf("rsqrt.approx.ftz.f64 max rel err on [1,4): %.3e (2^%.1f)\n", e, log2(e));
  return 0;
}
