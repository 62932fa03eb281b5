// Design microbenchmark (not product): per-phase fixed cost of
//  (a) a CUDA graph of empty kernels chained with programmatic dependent launch
//  (b) a grid barrier inside one persistent cluster kernel (all CTAs resident)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbb tools/mb_barrier.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void pdl_kernel(int* p) {
  extern __shared__ int sm[];
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (p) {   // dependent read of the previous node's write, then a write
    int v = p[(blockIdx.x * 7) & 1023];
    if (threadIdx.x == 0) p[blockIdx.x & 1023] = v + 1;
    if (threadIdx.x == 9999) sm[0] = v;
  }
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

static float chain(cudaStream_t st, int grid, int cl, int smem_a, int smem_b, int* p, bool pdl) {
  const int N = 90;
  cudaFuncSetAttribute((const void*)pdl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaGraph_t g;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < N; ++i) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = (i & 1) ? smem_b : smem_a;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = cl; at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, pdl_kernel, p);
  }
  cudaStreamEndCapture(st, &g);
  cudaGraphExec_t ge;
  cudaGraphInstantiate(&ge, g, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
  cudaEventRecord(e0, st);
  for (int r = 0; r < 20; ++r) cudaGraphLaunch(ge, st);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 1e3f * ms / (20 * N);
}

// sense-free barrier: monotonically increasing counter, target = k * nblocks
__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

__global__ void __cluster_dims__(8, 1, 1) persist_kernel(unsigned* ctr, int phases, double* sink) {
  const unsigned nb = gridDim.x;
  double s = 0;
  for (int i = 0; i < phases; ++i) {
    s += sink[(blockIdx.x * 37 + i) & 1023];
    grid_barrier(ctr, (unsigned)(i + 1) * nb);
  }
  if (s == 1234.5) sink[0] = s;
}

int main() {
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // (a) graph of N PDL-chained empty kernels, 128 CTAs each
  for (int grid : {128, 256}) {
    const int N = 90;
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < N; ++i) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(256);
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, pdl_kernel, (int*)nullptr);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphExec_t ge;
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
    cudaEventRecord(e0, st);
    for (int r = 0; r < 20; ++r) cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("pdl graph, grid %d: %.3f us per kernel node\n", grid, 1e3 * ms / (20 * N));
  }
  int* pbuf;
  cudaMalloc(&pbuf, 4096);
  cudaMemset(pbuf, 0, 4096);
  struct { int grid, cl, sa, sb; bool mem, pdl; } cases[] = {
      {128, 1, 0, 0, false, true},      {128, 1, 0, 0, true, true},       {128, 1, 0, 0, true, false},
      {128, 8, 0, 0, true, true},       {128, 8, 100000, 100000, true, true},
      {128, 1, 0, 150000, true, true},  {128, 8, 30000, 150000, true, true},
      {512, 1, 32000, 32000, true, true}, {144, 8, 200000, 200000, true, true}};
  for (auto& c : cases)
    printf("chain grid %d cluster %d smem %d/%d mem %d pdl %d: %.3f us per node\n", c.grid, c.cl, c.sa, c.sb,
           (int)c.mem, (int)c.pdl, chain(st, c.grid, c.cl, c.sa, c.sb, c.mem ? pbuf : nullptr, c.pdl));
  // (b) persistent kernel with grid barriers
  unsigned* ctr;
  double* sink;
  cudaMalloc(&ctr, 4);
  cudaMalloc(&sink, 1024 * 8);
  cudaMemset(sink, 0, 1024 * 8);
  for (int grid : {16, 64, 128, 144}) {
    const int phases = 1000;
    for (int w = 0; w < 2; ++w) {
      cudaMemsetAsync(ctr, 0, 4, st);
      persist_kernel<<<grid, 256, 0, st>>>(ctr, phases, sink);
    }
    cudaMemsetAsync(ctr, 0, 4, st);
    cudaEventRecord(e0, st);
    persist_kernel<<<grid, 256, 0, st>>>(ctr, phases, sink);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    printf("grid barrier, %d CTAs: %.3f us per barrier (%s)\n", grid, 1e3 * ms / phases, cudaGetErrorString(e));
  }
  return 0;
}
