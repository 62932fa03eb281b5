// DSMEM scatter microbenchmark (design input): cycles for the view kernel's two transposes.
//  pattern B (column pass): lane l, k in {0,1}: y = l + 32k -> rank y / 8, row y % 8, column posc:
//            32 separate 16-byte stores per instruction, 8 lanes per destination rank
//  pattern A (row pass): position q*32 + l -> rank pos / 16, 16 consecutive 16-byte elements per rank
//  pattern L: the same addresses of pattern B but in the CTA's own shared memory
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/dsmem_bench tools/dsmem_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int P = 128, M = 64, CS = 8, rp = M / CS, cp = P / CS, Pp = P + 1, cpp = cp + 1;

template <int PAT>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(256) scat(int iters, long long* cyc, double2* sink) {
  extern __shared__ double2 sm[];
  double2* bufB = sm;                    // [rp][Pp]
  double2* bufA = sm + rp * Pp;          // [M][cpp]
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = cluster.block_rank(), lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2 v = make_double2(lane, warp);
  cluster.sync();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (PAT == 0 || PAT == 2) {
      for (int cc = warp; cc < cp; cc += 8) {
        const int posc = rank * cp + cc;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int y = lane + 32 * k, dst = y / rp, yl = y - dst * rp;
          double2* rb = PAT == 0 ? cluster.map_shared_rank(bufB, dst) : bufB;
          rb[yl * Pp + posc] = v;
        }
      }
    } else {
      for (int yl = warp; yl < rp; yl += 8) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int pos = q * 32 + lane, dst = pos / cp, lc = pos - dst * cp;
          double2* rb = cluster.map_shared_rank(bufA, dst);
          rb[(rank * rp + yl) * cpp + lc] = v;
        }
      }
    }
    v.x += 1.0;
    cluster.sync();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x + gridDim.x * blockIdx.y] = t1 - t0;
  if (sink) sink[threadIdx.x] = bufB[threadIdx.x];  // (keeps the stores alive)
}

// pattern T: the row-pass volume as 64 bulk copies of 256 bytes per CTA (TMA engine,
// shared::cta -> shared::cluster), completion on the destination CTA's mbarrier
__device__ __forceinline__ unsigned s32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(256) bulk(int iters, long long* cyc, double2* sink) {
  extern __shared__ double2 sm[];
  double2* bufA = sm;                    // [M][cp] destination (no padding: 256-byte rows)
  double2* stage = sm + M * cp;          // [rp][P] source rows
  __shared__ __align__(8) unsigned long long bar;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = cluster.block_rank(), tid = threadIdx.x;
  for (int i = tid; i < rp * P; i += 256) stage[i] = make_double2(i, rank);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster.sync();
  const long long t0 = clock64();
  unsigned parity = 0;
  for (int it = 0; it < iters; ++it) {
    if (tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(M * cp * 16) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid < rp * CS) {
      const int yl = tid / CS, dst = tid % CS;
      unsigned rdst, rbar;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(s32(bufA + (rank * rp + yl) * cp)), "r"(dst));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(s32(&bar)), "r"(dst));
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(rdst), "r"(s32(stage + yl * P + dst * cp)), "r"(cp * 16), "r"(rbar) : "memory");
    }
    unsigned ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(s32(&bar)), "r"(parity) : "memory");
    parity ^= 1;
    cluster.sync();   // as the kernel: everyone done reading before the next scatter
  }
  const long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x + gridDim.x * blockIdx.y] = t1 - t0;
  if (sink) sink[tid] = bufA[tid];
}

// pattern G: the same transpose through global memory (L2): every CTA writes its 8 x 128
// row spectra as [row][pos] (coalesced), cluster barrier, then reads its 16 columns of all
// 64 rows (256-byte pieces) into shared memory
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(256) viaL2(int iters, long long* cyc, double2* xbuf) {
  extern __shared__ double2 sm[];
  double2* bufA = sm;                    // [M][cpp]
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = cluster.block_rank(), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double2* X = xbuf + (size_t)blockIdx.y * M * P;   // this view's exchange buffer [M][P]
  double2 v = make_double2(lane, warp);
  cluster.sync();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int yl = warp; yl < rp; yl += 8) {
#pragma unroll
      for (int q = 0; q < 4; ++q) X[(size_t)(rank * rp + yl) * P + q * 32 + lane] = v;
    }
    cluster.sync();
    // my columns [rank*cp, rank*cp + cp) of all M rows: 64 rows x 256 bytes
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = tid + 256 * j, row = i / cp, lc = i % cp;
      bufA[row * cpp + lc] = __ldcg(X + (size_t)row * P + rank * cp + lc);
    }
    v.x += bufA[lane].x;
    cluster.sync();
  }
  const long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x + gridDim.x * blockIdx.y] = t1 - t0;
}

__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(256) sync_only(int iters, long long* cyc) {
  cg::cluster_group cluster = cg::this_cluster();
  cluster.sync();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) cluster.sync();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x + gridDim.x * blockIdx.y] = t1 - t0;
}

template <typename K>
void run(const char* name, K kern, int clusters, long long* cyc, bool args3) {
  const int iters = 200;
  const size_t smem = (rp * Pp + M * cpp) * sizeof(double2);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  void* a3[] = {(void*)&iters, (void*)&cyc, nullptr};
  static double2* sink = nullptr;
  if (!sink) cudaMalloc(&sink, (size_t)16 * M * P * sizeof(double2));
  a3[2] = &sink;
  cudaLaunchKernel((const void*)kern, dim3(CS, clusters), dim3(256), a3, args3 ? smem : 0, 0);
  cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, cyc, sizeof(long long) * CS * clusters, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < CS * clusters; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%-28s clusters %2d : %8.1f cycles per iteration (%s)\n", name, clusters, (double)mx / iters,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* cyc;
  cudaMalloc(&cyc, 256 * sizeof(long long));
  for (int cl : {1, 2, 16}) {
    run("cluster.sync only", sync_only, cl, cyc, false);
    run("column-pass scatter (remote)", scat<0>, cl, cyc, true);
    run("column-pass scatter (local)", scat<2>, cl, cyc, true);
    run("row-pass scatter (remote)", scat<1>, cl, cyc, true);
    run("row-pass as 256 B bulk copies", bulk, cl, cyc, true);
    run("row-pass through global / L2", viaL2, cl, cyc, true);
  }
  return 0;
}
