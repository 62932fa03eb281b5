// How many 8-CTA clusters of a 256-thread, ~100 KB shared-memory kernel are co-resident on a
// B200, at 128 and at 144 registers per thread (design input for the view kernels: 16 views =
// 16 clusters must run in one wave).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_capacity tools/cluster_capacity.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int R>
__global__ void __maxnreg__(R) k(double* o) {
  extern __shared__ double s[];
  double a[48];
  for (int i = 0; i < 48; ++i) a[i] = o[i * 7 + threadIdx.x];
  double t = 0;
  for (int j = 0; j < 48; ++j) for (int i = 0; i < 48; ++i) t += a[i] * a[(i + j) % 48];
  s[threadIdx.x] = t;
  o[threadIdx.x] = s[(threadIdx.x + 1) % 256];
}
template <int R> void probe(int cs) {
  cudaFuncSetAttribute(k<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 104000);
  cudaFuncSetAttribute(k<R>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs, 16); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 104000;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  int n = 0;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k<R>, &cfg);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k<R>);
  printf("cluster size %d, maxnreg %d (uses %d): max active clusters %d (%s)\n", cs, R, fa.numRegs, n, cudaGetErrorString(e));
}
int main() {
  for (int cs : {4, 8, 16}) { probe<128>(cs); probe<144>(cs); }
  return 0;
}
