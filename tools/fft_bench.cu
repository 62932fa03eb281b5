// Warp-FFT microbenchmark (design input, not part of the product): cycles per
// forward + inverse length-128 / 512 transform of pdf_common.cuh's warp FFT
// for 1..8 warps per SM sub-partition group.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2602_13805_b200/csrc -o /tmp/fftb tools/fft_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "pdf_common.cuh"
using namespace pdf;

template <int E, int NC>
__global__ void fft_kernel(int iters, const double2* tw, double2* out, long long* cyc) {
  __shared__ double2 stw[32 * E];
  for (int i = threadIdx.x; i < 32 * E; i += blockDim.x) stw[i] = tw[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  LaneTw<double, E> lt;
  lt.load(stw, lane);
  double2 x[NC][E];
  for (int c = 0; c < NC; ++c)
    for (int k = 0; k < E; ++k) x[c][k] = make_double2(1e-3 * (lane + k + c), 1e-3 * (lane - k));
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < NC; ++c) warp_fft_fwd<double, E>(x[c], lt, lane);
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int k = 0; k < E; ++k) x[c][k] = cscale<double>(x[c][k], 1.0 / (32 * E));
#pragma unroll
    for (int c = 0; c < NC; ++c) warp_fft_inv<double, E>(x[c], lt, lane);
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  double2 s = make_double2(0, 0);
  for (int c = 0; c < NC; ++c)
    for (int k = 0; k < E; ++k) s = cadd<double>(s, x[c][k]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int E, int NC>
void run(int warps, const double2* tw, double2* out, long long* cyc) {
  const int iters = 200;
  fft_kernel<E, NC><<<148, 32 * warps>>>(iters, tw, out, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("P=%4d  warps/CTA=%2d  transforms in flight per warp=%d : %8.1f cycles per (fwd+inv) per transform, %8.1f per warp-iteration\n",
         32 * E, warps, NC, (double)mx / iters / NC, (double)mx / iters);
}

int main() {
  double2 *tw, *out;
  long long* cyc;
  cudaMalloc(&tw, 512 * sizeof(double2));
  cudaMalloc(&out, 148 * 1024 * sizeof(double2));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  double2 h[512];
  for (int P : {128, 512}) {
    for (int i = 0; i < P; ++i) h[i] = make_double2(cos(-2 * M_PI * i / P), sin(-2 * M_PI * i / P));
    cudaMemcpy(tw, h, P * sizeof(double2), cudaMemcpyHostToDevice);
    for (int w : {1, 4, 8, 16}) {
      if (P == 128) { run<4, 1>(w, tw, out, cyc); run<4, 2>(w, tw, out, cyc); }
      else { run<16, 1>(w, tw, out, cyc); }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
