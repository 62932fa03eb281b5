// Throughput of FP64 tensor-core MMA (mma.sync m8n8k4 f64) vs scalar DFMA on
// this GPU: decides whether the network layers use DMMA.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(int iters, double* out) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[2 * i], c[2 * i + 1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 1234.5) out[0] = s;
}

__global__ void dfma_kernel(int iters, double* out) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 0.999999, 1e-7);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1234.5) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps = 4; warps <= 32; warps *= 2) {
    const int iters = 4096, blocks = sms * 2, thr = warps * 16;
    dmma_kernel<<<blocks, thr>>>(16, out);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, thr>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 2.0 * 256 * 8 * (double)iters * blocks * (thr / 32);
    printf("dmma  warps/SM %2d : %.1f TFLOP/s\n", warps, flop / (ms * 1e-3) / 1e12);
    dfma_kernel<<<blocks, thr>>>(16, out);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, thr>>>(iters / 4, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double f2 = 2.0 * 64 * (double)(iters / 4) * blocks * thr;
    printf("dfma  warps/SM %2d : %.1f TFLOP/s\n", warps, f2 / (ms * 1e-3) / 1e12);
  }
  return 0;
}
