// Fixed-cost microbenchmarks on B200 (design input, not part of the product):
//  1. graph-replayed empty kernels (launch + drain per node)
//  2. hot-L2 streaming: 128 CTAs read 8 MiB of doubles already in L2
//  3. 8-CTA cluster barrier round trip
//  4. dependent FP64 FMA chain latency
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void empty_kernel(int* p) { if (p && threadIdx.x == 9999) p[0] = 1; }

__global__ void stream_kernel(const double* __restrict__ a, double* out, size_t n) {
  double s = 0;
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) s += a[i];
  if (s == 1234.5) out[0] = s;
}

__global__ void __cluster_dims__(8, 1, 1) cluster_kernel(int iters, int* out) {
  cg::cluster_group cl = cg::this_cluster();
  for (int i = 0; i < iters; ++i) cl.sync();
  if (threadIdx.x == 9999) out[0] = iters;
}

__global__ void chain_kernel(int iters, double* out) {
  double a = threadIdx.x * 1e-9, x = 0.999999, y = 1e-7;
  for (int i = 0; i < iters; ++i) a = fma(a, x, y);
  if (a == 1234.5) out[0] = a;
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // 1. graph of 100 empty kernels, 128 x 256
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 100; ++i) empty_kernel<<<128, 256, 0, st>>>(nullptr);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEventRecord(e0, st);
  for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, st);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("empty kernel in graph: %.2f us/node\n", ms * 1e3 / 1000);
  // 2. hot-L2 stream
  size_t n = (8u << 20) / 8;
  double *a, *o;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&o, 8);
  cudaMemset(a, 0, n * 8);
  for (int grid : {128, 148, 296, 592}) {
    for (int w = 0; w < 3; ++w) stream_kernel<<<grid, 256, 0, st>>>(a, o, n);
    cudaEventRecord(e0, st);
    for (int r = 0; r < 20; ++r) stream_kernel<<<grid, 256, 0, st>>>(a, o, n);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("hot-L2 8 MiB read, grid %d x 256: %.2f us  (%.0f GB/s)\n", grid, ms * 1e3 / 20, 8.0 * (1 << 20) / (ms / 20 * 1e-3) / 1e9);
  }
  // 3. cluster barrier
  int* io;
  cudaMalloc(&io, 4);
  cluster_kernel<<<128, 256, 0, st>>>(10, io);
  cudaEventRecord(e0, st);
  cluster_kernel<<<128, 256, 0, st>>>(1000, io);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("cluster(8) barrier: %.3f us each\n", ms * 1e3 / 1000);
  // 4. DFMA dependent chain
  chain_kernel<<<1, 32, 0, st>>>(100, o);
  cudaEventRecord(e0, st);
  chain_kernel<<<1, 32, 0, st>>>(100000, o);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("dependent DFMA: %.2f ns each (%.1f cycles at 1.965 GHz)\n", ms * 1e6 / 100000, ms * 1e6 / 100000 * 1.965);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
