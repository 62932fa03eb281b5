// Network layers on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64).
//
// Measured on the B200 (tools/dmma_bench.cu): DMMA reaches 34-37 TFLOP/s
// with 4-32 warps per SM, the same ceiling as scalar DFMA but at 1/8 of the
// issue slots and with operands reused inside the tensor core -- the scalar
// kernels of pdf_net.cuh were bound by shared-memory loads and issue (one LDS
// per FMA), not by the FP64 pipe.
//
// Fragment layouts (PTX ISA, mma.m8n8k4 .f64; g = lane >> 2, t = lane & 3):
//   A (8 x 4, row)  : lane holds A[g][t]
//   B (4 x 8, col)  : lane holds B[t][g]
//   C/D (8 x 8)     : lane holds D[g][2t], D[g][2t+1]
// The k index of a 4-wide MMA step is free to permute as long as A and B
// agree: a block of 16 k is issued as 4 steps s where lane position t stands
// for k = 4t + s, so every lane reads 32 contiguous bytes of a W row (four
// lanes of a group cover a 128-byte line).
#pragma once
#include "pdf_common.cuh"
#include "pdf_dmma.cuh"
#include "pdf_net.cuh"

namespace pdf {

constexpr int FM_KCH = 64;              // k per staged input chunk (4 k-blocks of 16)
constexpr int FM_XP = FM_KCH + 2;       // pitch: conflict-free 16-byte fragment reads
constexpr int FM_WARPS = 8;

__host__ __device__ constexpr size_t fwd_mma_smem_bytes(int MT, int NT) {
  const size_t xs = (size_t)2 * 8 * MT * FM_XP;
  const size_t part = (size_t)FM_WARPS * NT * 8 * 8 * MT;
  return (xs > part ? xs : part) * sizeof(double);
}

// z[r][n] = sum_k x[r][k] W[n][k] + b[n] for one layer (network.py:107-120).
// CTA = 8 warps x NT n-tiles of 8 outputs, all rows (MT m-tiles of 8), the
// K range [rank*ks, ...) of its cluster rank; partial sums meet in DSMEM and
// are added in rank order.  The B fragments (W) go straight from global
// memory into registers one 64-wide chunk (four k-blocks) ahead of their use,
// so each lane keeps 4 x NT x 32 bytes of W in flight; the input rows x are
// staged per chunk with cp.async (double-buffered).
template <int MT, int NT>
__global__ void __launch_bounds__(256) net_fwd_mma_kernel(NetFwdArgs<double> a) {
  constexpr int RPM = 8 * MT, SEG = FM_KCH / 2, THR = 256;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Xs = reinterpret_cast<double*>(smem_raw);   // 2 x [RPM][FM_XP]
  double* part = Xs;                                   // after the k loop: [8*NT*8][RPM]
  cg::cluster_group cluster = cg::this_cluster();
  const int CK = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int scene = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int K = a.K, N = a.N, rows = a.rows;
  const int nw0 = (blockIdx.x * FM_WARPS + warp) * NT * 8;
  const int kb = rank * a.ks, ke = min(K, kb + a.ks);
  const double* __restrict__ W = a.theta + scene * a.th_ss + a.w_off;
  const double* __restrict__ X = a.in + scene * a.in_ss;
  const double* wr[NT];
  bool nok[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int n = nw0 + 8 * j + g;
    nok[j] = n < N;
    wr[j] = W + (size_t)(nok[j] ? n : 0) * K;
  }
  auto stage = [&](int k0, int s) {
    double* dst = Xs + s * RPM * FM_XP;
    for (int i = tid; i < RPM * SEG; i += THR) {
      const int r = i / SEG, sg = i % SEG, gk = k0 + 2 * sg;
      const bool ok = r < rows && gk < ke;
      cp_async16(dst + r * FM_XP + 2 * sg, ok ? X + (size_t)r * K + gk : X, ok);
    }
    cp_async_commit();
  };
  // B fragments of k-block k (lane: W[n][k + 4t .. k + 4t + 3])
  auto loadB = [&](int k, double (&b)[NT][4]) {
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int kk = k + 4 * t + 2 * h;      // even; K and ke are even
        double2 v = make_double2(0.0, 0.0);
        if (nok[j] && kk < ke) v = *reinterpret_cast<const double2*>(wr[j] + kk);
        b[j][2 * h] = v.x;
        b[j][2 * h + 1] = v.y;
      }
  };

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double b[4][NT][4];
  // W1 is written by the launch right before (Adam of the previous
  // iteration); W2, W3 two or more launches back and may stream early
  tl_mark(a.tl, 0);
  if (!a.w_early) { pdl_wait(); tl_mark(a.tl, 1); }
#pragma unroll
  for (int q = 0; q < 4; ++q) loadB(kb + 16 * q, b[q]);
  if (a.w_early) { pdl_wait(); tl_mark(a.tl, 1); }
  if (a.step && tid == 0 && blockIdx.x == 0 && rank == 0 && scene == 0) atomicAdd(a.step, 1);
  if (kb < ke) stage(kb, 0);
  int s = 0;
  for (int k0 = kb; k0 < ke; k0 += FM_KCH, s ^= 1) {
    if (k0 + FM_KCH < ke) {
      stage(k0 + FM_KCH, s ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* xs = Xs + s * RPM * FM_XP + g * FM_XP + 4 * t;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int kk = 16 * q;
      if (k0 + kk < ke) {
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const double2 a01 = *reinterpret_cast<const double2*>(xs + i * 8 * FM_XP + kk);
          const double2 a23 = *reinterpret_cast<const double2*>(xs + i * 8 * FM_XP + kk + 2);
          const double av[4] = {a01.x, a01.y, a23.x, a23.y};
#pragma unroll
          for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int u = 0; u < 4; ++u) dmma(acc[i][j][0], acc[i][j][1], av[u], b[q][j][u]);
        }
      }
      loadB(k0 + FM_KCH + kk, b[q]);     // the same slot one chunk ahead (zero past ke)
    }
    __syncthreads();   // buffer s is restaged two chunks later; the last pass frees Xs for part
  }
  pdl_trigger();
  __syncthreads();                        // Xs is reused as the partial-sum buffer
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int c = 0; c < 2; ++c) part[(warp * NT * 8 + 8 * j + 2 * t + c) * RPM + 8 * i + g] = acc[i][j][c];
  cluster.sync();

  const double* bias = a.theta + scene * a.th_ss + (a.final_layer == 3 ? 0 : a.b_off);
  const int total = FM_WARPS * NT * 8 * RPM;
  for (int e = rank * 256 + tid; e < total; e += CK * 256) {
    const int wo = e / RPM, r = e % RPM;
    const int gn = blockIdx.x * FM_WARPS * NT * 8 + wo;
    if (gn >= N || r >= rows) continue;
    double z = 0.0;
#pragma unroll 8
    for (int c = 0; c < CK; ++c) z += cluster.map_shared_rank(part, c)[e];
    if (a.final_layer != 3) z += bias[gn];
    if (a.final_layer != 1) {
      a.out[scene * a.out_ss + (size_t)r * N + gn] = a.final_layer ? z : tanh(z);
    } else {
      const double yv = z * a.cout[(size_t)scene * N + gn];
      const int half = N / 2;
      const int f = gn < half ? gn : gn - half;
      int view, m;
      if (a.joint) { view = f / a.M0; m = f % a.M0; } else { view = r; m = f; }
      const size_t off = ((size_t)scene * a.n + view) * a.M0 + m;
      double* dst = reinterpret_cast<double*>(a.alpha_hat + off);
      const double* src = reinterpret_cast<const double*>(a.alpha0 + off);
      if (gn < half) dst[0] = src[0] + yv; else dst[1] = src[1] + yv;
    }
  }
  cluster.sync();
  tl_mark(a.tl, 2);
}

// ---------------------------------------------------------------------------
// Forward layer for one scene with few rows (the latency-bound regime):
// CTA = one n-tile of 8 outputs, its XW warps split K.  The whole input
// block x[rows][K] is staged into shared memory with cp.async and every W
// fragment the warp needs (<= XKB k-blocks of 16) is requested into
// registers at once, so the layer costs one memory round trip; the XW warp
// partials are added in warp order through shared memory (no cluster).
constexpr int XW = 8;
constexpr int XKB = 8;                  // k-blocks per warp: K <= XW * XKB * 16 = 1024

__host__ __device__ constexpr size_t fwd_x_smem_bytes(int MT, int K) {
  const size_t xs = (size_t)8 * MT * (K + 2);
  const size_t red = (size_t)XW * 8 * MT * 8;
  return (xs + red) * sizeof(double);
}

// MC > 1: a cluster of MC CTAs along x shares the input block: each CTA
// copies every MC-th row with one bulk copy multicast to all of them (TMA
// engine), so the L2 serves x once per cluster instead of once per CTA.
template <int MT, int MC>
__global__ void __launch_bounds__(XW * 32, 1) net_fwd_x_kernel(NetFwdArgs<double> a) {
  constexpr int RPM = 8 * MT, THR = XW * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long xbar;
  const int K = a.K, N = a.N, rows = a.rows, XP = K + 2;
  double* Xs = reinterpret_cast<double*>(smem_raw);     // [RPM][K + 2]
  double* red = Xs + (size_t)RPM * XP;                  // [XW][RPM][8]
  const int scene = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int n0 = blockIdx.x * 8, n = n0 + g;
  const int kpw = ((K + XW * 16 - 1) / (XW * 16)) * 16;
  const int kb = warp * kpw, ke = min(K, kb + kpw);
  const double* __restrict__ W = a.theta + scene * a.th_ss + a.w_off + (size_t)(n < N ? n : 0) * K;
  const double* __restrict__ X = a.in + scene * a.in_ss;
  double b[XKB][4];
  auto loadW = [&]() {
#pragma unroll
    for (int q = 0; q < XKB; ++q)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int kk = kb + 16 * q + 4 * t + 2 * h;
        double2 v = make_double2(0.0, 0.0);
        if (n < N && kk < ke) v = *reinterpret_cast<const double2*>(W + kk);
        b[q][2 * h] = v.x;
        b[q][2 * h + 1] = v.y;
      }
  };
  tl_mark(a.tl, 0);
  if constexpr (MC > 1) {
    // padding rows (never copied) read as zero; barrier initialised before any peer's copy lands
    for (int i = tid; i < (RPM - rows) * XP; i += THR) Xs[(size_t)rows * XP + i] = 0.0;
    if (tid == 0) {
      mbar_init(&xbar, 1);
      mbar_fence_init_cluster();
    }
    cg::this_cluster().sync();
  }
  if (a.w_early) loadW();
  pdl_wait();
  tl_mark(a.tl, 1);
  if (!a.w_early) loadW();
  if (a.step && tid == 0 && blockIdx.x == 0 && scene == 0) atomicAdd(a.step, 1);
  if constexpr (MC > 1) {
    const unsigned rank = cg::this_cluster().block_rank();
    if (tid == 0) {
      mbar_arrive_expect_tx(&xbar, (unsigned)(rows * K * sizeof(double)));
      for (int r = (int)rank; r < rows; r += MC)
        bulk_copy_multicast(Xs + (size_t)r * XP, X + (size_t)r * K, (unsigned)(K * sizeof(double)), &xbar,
                            (unsigned short)((1u << MC) - 1));
    }
    while (!mbar_try_wait(&xbar, 0)) {
    }
  } else {
    const int seg = K / 2;
    for (int i = tid; i < RPM * seg; i += THR) {
      const int r = i / seg, s2 = i - r * seg;
      const bool ok = r < rows;
      cp_async16(Xs + (size_t)r * XP + 2 * s2, ok ? X + (size_t)r * K + 2 * s2 : X, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
  }
  __syncthreads();
  pdl_trigger();
  double acc[MT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
  for (int q = 0; q < XKB; ++q) {
    const int kk = kb + 16 * q;
    if (kk < ke) {
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const double* xr = Xs + (size_t)(8 * i + g) * XP + kk + 4 * t;
        const double2 a01 = *reinterpret_cast<const double2*>(xr);
        const double2 a23 = kk + 4 * t + 2 < ke ? *reinterpret_cast<const double2*>(xr + 2) : make_double2(0.0, 0.0);
        const bool in0 = kk + 4 * t < ke;
        const double av[4] = {in0 ? a01.x : 0.0, in0 ? a01.y : 0.0, a23.x, a23.y};
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma(acc[i][0], acc[i][1], av[u], b[q][u]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int c = 0; c < 2; ++c) red[(warp * RPM + 8 * i + g) * 8 + 2 * t + c] = acc[i][c];
  __syncthreads();
  const double* bias = a.theta + scene * a.th_ss + (a.final_layer == 3 ? 0 : a.b_off);
  for (int e = tid; e < RPM * 8; e += THR) {
    const int r = e >> 3, col = e & 7, gn = n0 + col;
    if (gn >= N || r >= rows) continue;
    double z = 0.0;
#pragma unroll
    for (int w = 0; w < XW; ++w) z += red[(w * RPM + r) * 8 + col];
    if (a.final_layer != 3) z += bias[gn];
    if (a.final_layer != 1) {
      a.out[scene * a.out_ss + (size_t)r * N + gn] = a.final_layer ? z : tanh(z);
    } else {
      const double yv = z * a.cout[(size_t)scene * N + gn];
      const int half = N / 2;
      const int f = gn < half ? gn : gn - half;
      int view, m;
      if (a.joint) { view = f / a.M0; m = f % a.M0; } else { view = r; m = f; }
      const size_t off = ((size_t)scene * a.n + view) * a.M0 + m;
      double* dst = reinterpret_cast<double*>(a.alpha_hat + off);
      const double* src = reinterpret_cast<const double*>(a.alpha0 + off);
      if (gn < half) dst[0] = src[0] + yv; else dst[1] = src[1] + yv;
    }
  }
  tl_mark(a.tl, 2);
}

// ---------------------------------------------------------------------------
// Backward layer + fused Adam on DMMA (network.py:201-219, 248-264):
//   g_W[n][k] = sum_r g_z[r][n] h[r][k]     (MMA: M = n, N = k, K = r)
//   g_h[r][k] = sum_n g_z[r][n] W_old[n][k] (MMA: M = r, N = k, K = n)
// A warp owns KT k-tiles (8 KT columns) and streams the n rows of its
// cluster rank's range 8 at a time (an "n-tile").  W, m, v of each n-tile
// arrive in the D-fragment layout of the g_W product (lane: row n0+g,
// columns 2t, 2t+1 of each k-tile) through a per-lane cp.async ring BM_D
// n-tiles deep, so the Adam update is element-wise in registers and enough
// bytes are in flight to stream HBM; the old W values of the other lanes'
// ring slots are the B fragments of the g_h product.  g_z chunks of BM_NCH
// columns ride in the same cp.async groups (double-buffered); h stays in
// registers as B fragments for the whole kernel.
constexpr int BM_WARPS = 8;              // warps per CTA for batches (4 for one scene: more CTAs)
constexpr int BM_NCH = 32;              // n per staged g_z chunk (4 n-tiles)
constexpr int BM_GP = BM_NCH + 4;       // pitch: conflict-free fragment reads in both products
// D (template): n-tiles in flight per lane; g_z chunk buffers: 2 for D <= 4,
// 3 for D <= 8 (the refill may stage the chunk after next)
__host__ __device__ constexpr int bm_ngb(int D) { return D > 4 ? 3 : 2; }

__host__ __device__ constexpr size_t bwd_mma_smem_bytes(int MT, int KT, int WB, int D) {
  return ((size_t)bm_ngb(D) * 8 * MT * BM_GP + (size_t)D * 3 * KT * WB * 32 * 2 +
          (size_t)8 * MT * WB * 8 * KT) * sizeof(double);
}

template <int MT, int KT, bool FUSED, int WB, int BM_D>
__global__ void __launch_bounds__(WB * 32) net_bwd_mma_kernel(NetBwdArgs<double> a) {
  constexpr int NGB = bm_ngb(BM_D);
  constexpr int RPM = 8 * MT, SEG = BM_NCH / 2, KC = 8 * KT, CW = WB * KC;
  constexpr int THR = WB * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Gs = reinterpret_cast<double*>(smem_raw);              // 2 x [RPM][BM_GP]  g_z[r][c0 + i]
  double2* ring = reinterpret_cast<double2*>(Gs + NGB * RPM * BM_GP);   // [BM_D][3][KT][THR]
  double* cpart = reinterpret_cast<double*>(ring + BM_D * 3 * KT * THR);   // [RPM][CW]
  __shared__ double bc_s[2];
  cg::cluster_group cluster = cg::this_cluster();
  // grid.y == CN: the whole y extent is one cluster when g_h is reduced
  // across it, and plain CTAs otherwise (first layer: no g_h)
  const int CN = (int)gridDim.y;
  const int rank = (int)blockIdx.y;
  const int scene = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int K = a.K, N = a.N, rows = a.rows;
  const int kw0 = blockIdx.x * CW + warp * KC;
  const int nb = min(N, rank * a.ns), ne = min(N, nb + a.ns);
  const int ntl = (ne - nb + 7) / 8;                 // n-tiles of this rank
  const double* __restrict__ hin = a.hin + scene * a.hin_ss;
  const double* __restrict__ gz = a.gz + scene * a.gz_ss;
  double* __restrict__ W = a.theta + scene * a.th_ss + a.w_off;
  double* __restrict__ mW = FUSED ? a.m + scene * a.th_ss + a.w_off : nullptr;
  double* __restrict__ vW = FUSED ? a.v + scene * a.th_ss + a.w_off : nullptr;
  double* __restrict__ gW = FUSED ? nullptr : a.grad + scene * a.th_ss + a.w_off;
  auto slot = [&](int sl, int arr, int j) { return ring + ((sl * 3 + arr) * KT + j) * THR; };

  auto stage_gz = [&](int c) {          // chunk c of this rank (no commit)
    const int n0 = nb + c * BM_NCH;
    double* dst = Gs + (c % NGB) * RPM * BM_GP;
    for (int i = tid; i < RPM * SEG; i += THR) {
      const int r = i / SEG, sg = i % SEG, gn = n0 + 2 * sg;
      const bool ok = r < rows && gn < ne;
      cp_async16(dst + r * BM_GP + 2 * sg, ok ? gz + (size_t)r * N + gn : gz, ok);
    }
  };
  auto stage_w = [&](int it) {          // W, m, v of n-tile it into ring slot it % BM_D (no commit)
    const int n = nb + 8 * it + g, sl = it % BM_D;
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      const int kk = kw0 + 8 * j + 2 * t;
      const bool ok = n < ne && kk < K;
      const size_t o = ok ? (size_t)n * K + kk : 0;
      cp_async16(slot(sl, 0, j) + tid, W + o, ok);
      if constexpr (FUSED) {
        cp_async16(slot(sl, 1, j) + tid, mW + o, ok);
        cp_async16(slot(sl, 2, j) + tid, vW + o, ok);
      }
    }
  };

  if (tid == 0) {
    if (FUSED) {
      const int tt = *a.step;
      bc_s[0] = 1.0 / (1.0 - pow(a.b1, (double)tt));
      bc_s[1] = 1.0 / (1.0 - pow(a.b2, (double)tt));
    } else {
      bc_s[0] = bc_s[1] = 1.0;
    }
  }
  // W, m, v are final since the previous iteration: the first BM_D n-tiles
  // (and this CTA's first bias entries) are requested before the dependency wait
  const bool bias_lane = blockIdx.x == 0 && tid < BM_NCH;
  double* thb = FUSED ? a.theta + scene * a.th_ss + a.b_off : nullptr;
  double* mbb = FUSED ? a.m + scene * a.th_ss + a.b_off : nullptr;
  double* vbb = FUSED ? a.v + scene * a.th_ss + a.b_off : nullptr;
  double bp = 0.0, bm = 0.0, bv = 0.0;
  if (FUSED && bias_lane && nb + tid < ne) { bp = thb[nb + tid]; bm = mbb[nb + tid]; bv = vbb[nb + tid]; }
  tl_mark(a.tl, 0);
  for (int it = 0; it < BM_D; ++it) {
    if (it < ntl) stage_w(it);
    cp_async_commit();
  }
  pdl_wait();
  tl_mark(a.tl, 1);
  // h as B fragments of the g_W product: hf[j][s] = h[4s + t][kw0 + 8j + g]
  double hf[KT][RPM / 4];
#pragma unroll
  for (int j = 0; j < KT; ++j)
#pragma unroll
    for (int s4 = 0; s4 < RPM / 4; ++s4) {
      const int r = 4 * s4 + t, kk = kw0 + 8 * j + g;
      hf[j][s4] = (r < rows && kk < K) ? hin[(size_t)r * K + kk] : 0.0;
    }
  double gh[MT][KT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < KT; ++j) gh[i][j][0] = gh[i][j][1] = 0.0;
  for (int c = 0; 4 * c < BM_D && 4 * c < ntl; ++c) stage_gz(c);
  cp_async_commit();

  int errbits = 0;
  // g_h B fragment source: lane (4s+t)*4 + (g>>1) of this warp holds W[n0+4s+t][8j + g] in component g&1
  const int bsrc = warp * 32 + (g >> 1);
#pragma unroll 1
  for (int it = 0; it < ntl; ++it) {
    if (it == 0) cp_async_wait<0>(); else cp_async_wait<BM_D - 1>();
    const int c = it >> 2, nt = (it & 3) * 8;
    if ((it & 3) == 0) __syncthreads();   // chunk c visible to all; chunk c-1 no longer read
    else __syncwarp();
    const double* G = Gs + (c % NGB) * RPM * BM_GP;
    const double ibc1 = bc_s[0], ibc2 = bc_s[1];
    const int sl = it % BM_D;
    // bias of chunk c (network.py:213,217), by the first column tile; its
    // p, m, v were loaded one chunk ahead (no global round trip in the loop)
    if ((it & 3) == 0 && bias_lane) {
      const int gn = nb + c * BM_NCH + tid;
      if (gn < ne) {
        double gb = 0.0;
        for (int r = 0; r < rows; ++r) gb += G[r * BM_GP + tid];
        if (!isfinite(gb)) errbits |= ERR_NONFINITE_GRAD;
        if constexpr (FUSED) {
          adam_one<double>(bp, bm, bv, gb, a.lr, a.b1, a.b2, a.eps, ibc1, ibc2);
          if (!isfinite(bp)) errbits |= ERR_NONFINITE_PARAM;
          thb[gn] = bp; mbb[gn] = bm; vbb[gn] = bv;
          if (gn + BM_NCH < ne) { bp = thb[gn + BM_NCH]; bm = mbb[gn + BM_NCH]; bv = vbb[gn + BM_NCH]; }
        } else {
          if (a.peers) *peer_slot(a.peers, a.peer_me, a.peer_shard, a.b_off + gn) = gb;
          else a.grad[scene * a.th_ss + a.b_off + gn] = gb;
        }
      }
    }
    // g_W: NA independent accumulators break the dependent DMMA chain over the rows
    constexpr int NA = RPM / 4 < 4 ? RPM / 4 : 4;
    double gwp[NA][KT][2];
#pragma unroll
    for (int q = 0; q < NA; ++q)
#pragma unroll
      for (int j = 0; j < KT; ++j) gwp[q][j][0] = gwp[q][j][1] = 0.0;
#pragma unroll
    for (int s4 = 0; s4 < RPM / 4; ++s4) {
      const double av = G[(4 * s4 + t) * BM_GP + nt + g];
#pragma unroll
      for (int j = 0; j < KT; ++j) dmma(gwp[s4 % NA][j][0], gwp[s4 % NA][j][1], av, hf[j][s4]);
    }
    // g_h with the old W tile (other lanes' ring slots)
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      double bw[KT];
#pragma unroll
      for (int j = 0; j < KT; ++j)
        bw[j] = reinterpret_cast<const double*>(slot(sl, 0, j) + bsrc + (4 * s2 + t) * 4)[g & 1];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const double av = G[(8 * i + g) * BM_GP + nt + 4 * s2 + t];
#pragma unroll
        for (int j = 0; j < KT; ++j) dmma(gh[i][j][0], gh[i][j][1], av, bw[j]);
      }
    }
    const int n = nb + 8 * it + g;
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      const int kk = kw0 + 8 * j + 2 * t;
      double gw0 = gwp[0][j][0], gw1 = gwp[0][j][1];
#pragma unroll
      for (int q = 1; q < NA; ++q) { gw0 += gwp[q][j][0]; gw1 += gwp[q][j][1]; }
      if (n < ne && kk < K) {
        const size_t o = (size_t)n * K + kk;
        if (!isfinite(gw0) || !isfinite(gw1)) errbits |= ERR_NONFINITE_GRAD;
        if constexpr (FUSED) {
          double2 p = slot(sl, 0, j)[tid], m2 = slot(sl, 1, j)[tid], v2 = slot(sl, 2, j)[tid];
          adam_one<double>(p.x, m2.x, v2.x, gw0, a.lr, a.b1, a.b2, a.eps, ibc1, ibc2);
          adam_one<double>(p.y, m2.y, v2.y, gw1, a.lr, a.b1, a.b2, a.eps, ibc1, ibc2);
          if (!isfinite(p.x) || !isfinite(p.y)) errbits |= ERR_NONFINITE_PARAM;
          *reinterpret_cast<double2*>(W + o) = p;
          *reinterpret_cast<double2*>(mW + o) = m2;
          *reinterpret_cast<double2*>(vW + o) = v2;
        } else if (a.peers) {
          *reinterpret_cast<double2*>(peer_slot(a.peers, a.peer_me, a.peer_shard, a.w_off + (long long)o)) =
              make_double2(gw0, gw1);
        } else {
          *reinterpret_cast<double2*>(gW + o) = make_double2(gw0, gw1);
        }
      }
    }
    __syncwarp();   // every lane is done with ring slot sl before it is refilled
    // refill: n-tile it + BM_D, and the g_z chunk it needs when it starts one
    const int nx = it + BM_D;
    if (nx < ntl) {
      stage_w(nx);
      if ((nx & 3) == 0) stage_gz(nx >> 2);
    }
    cp_async_commit();
  }
  pdl_trigger();
  if (errbits) atomicOr(&a.err[scene], errbits);

  if (a.gzprev) {
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < KT; ++j)
#pragma unroll
        for (int c = 0; c < 2; ++c) cpart[(8 * i + g) * CW + warp * KC + 8 * j + 2 * t + c] = gh[i][j][c];
    cluster.sync();
    for (int e = rank * THR + tid; e < rows * CW; e += CN * THR) {
      const int r = e / CW, cl = e % CW, gk = blockIdx.x * CW + cl;
      if (gk >= K) continue;
      double sum = 0.0;
#pragma unroll 8
      for (int q = 0; q < CN; ++q) sum += cluster.map_shared_rank(cpart, q)[e];   // loads in flight together
      const double hv = hin[(size_t)r * K + gk];
      a.gzprev[scene * a.gzp_ss + (size_t)r * K + gk] = sum * (1.0 - hv * hv);
    }
    cluster.sync();
  } else {
    cp_async_wait<0>();
  }
  if (a.peers) __threadfence_system();   // peer stores visible before the barrier that follows
  tl_mark(a.tl, 2);
}

}  // namespace pdf

namespace pdf {

// ---------------------------------------------------------------------------
// Split network backward for the latency regime (one or a few scenes, <= 16
// rows, widths <= 1024).  The fused layer kernel above walks n-tiles serially
// per warp and reduces g_h across a cluster; here the two products of a layer
// become separate, fully parallel launches:
//   net_gh_x_kernel   g_h = g_z W_old, g_z' = g_h (1 - h^2)  (network.py:210-212)
//                     for layers 3 and 2, on the critical path;
//   net_adam_x_kernel g_W = g_z^T h, g_b = sum_r g_z, Adam in place
//                     (network.py:201-219, 248-264) for all three layers in
//                     one launch, every W / m / v fragment requested at once.
// W_old is read by the g_h launches before the Adam launch rewrites it.
constexpr int GX_STEPS = 32;            // n-steps of 4 per warp: N <= XW * 4 * GX_STEPS = 1024

__host__ __device__ constexpr size_t gh_x_smem_bytes(int MT, int N) {
  return ((size_t)8 * MT * (N + 2) + (size_t)XW * 8 * MT * 8) * sizeof(double);
}

// CTA = one k-tile of 8 outputs of g_h; its XW warps split the n reduction
template <int MT, int MC>
__global__ void __launch_bounds__(XW * 32, 1) net_gh_x_kernel(NetBwdArgs<double> a) {
  constexpr int RPM = 8 * MT, THR = XW * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long gbar;
  const int K = a.K, N = a.N, rows = a.rows, GP = N + 2;
  double* Gz = reinterpret_cast<double*>(smem_raw);   // [RPM][N + 2]
  double* red = Gz + (size_t)RPM * GP;                 // [XW][RPM][8]
  const int scene = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int k0 = blockIdx.x * 8;
  const int npw = ((N + XW * 4 - 1) / (XW * 4)) * 4;
  const int nb = warp * npw, ne = min(N, nb + npw);
  const double* __restrict__ W = a.theta + scene * a.th_ss + a.w_off;
  tl_mark(a.tl, 0);
  if (a.snap && tid == 0 && blockIdx.x == 0 && scene == 0) *a.snap = *a.step;
  // B fragments (W_old is final since the previous iteration): lane holds W[n + t][k0 + g]
  double b[GX_STEPS];
  const bool kok = k0 + g < K;
#pragma unroll
  for (int q = 0; q < GX_STEPS; ++q) {
    const int n = nb + 4 * q + t;
    b[q] = (kok && n < ne) ? W[(size_t)n * K + k0 + g] : 0.0;
  }
  if constexpr (MC > 1) {   // g_z multicast over the cluster (as net_fwd_x_kernel's input block)
    for (int i = tid; i < (RPM - rows) * GP; i += THR) Gz[(size_t)rows * GP + i] = 0.0;
    if (tid == 0) {
      mbar_init(&gbar, 1);
      mbar_fence_init_cluster();
    }
    cg::this_cluster().sync();
  }
  pdl_wait();
  tl_mark(a.tl, 1);
  const double* __restrict__ gz = a.gz + scene * a.gz_ss;
  if constexpr (MC > 1) {
    const unsigned rank = cg::this_cluster().block_rank();
    if (tid == 0) {
      mbar_arrive_expect_tx(&gbar, (unsigned)(rows * N * sizeof(double)));
      for (int r = (int)rank; r < rows; r += MC)
        bulk_copy_multicast(Gz + (size_t)r * GP, gz + (size_t)r * N, (unsigned)(N * sizeof(double)), &gbar,
                            (unsigned short)((1u << MC) - 1));
    }
    while (!mbar_try_wait(&gbar, 0)) {
    }
  } else {
    const int seg = N / 2;
    for (int i = tid; i < RPM * seg; i += THR) {
      const int r = i / seg, s2 = i - r * seg;
      const bool ok = r < rows;
      cp_async16(Gz + (size_t)r * GP + 2 * s2, ok ? gz + (size_t)r * N + 2 * s2 : gz, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
  }
  __syncthreads();
  pdl_trigger();
  double acc[MT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
  for (int q = 0; q < GX_STEPS; ++q) {
    const int n = nb + 4 * q;
    if (n < ne) {
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const double av = n + t < ne ? Gz[(size_t)(8 * i + g) * GP + n + t] : 0.0;
        dmma(acc[i][0], acc[i][1], av, b[q]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int c = 0; c < 2; ++c) red[(warp * RPM + 8 * i + g) * 8 + 2 * t + c] = acc[i][c];
  __syncthreads();
  const double* __restrict__ hin = a.hin + scene * a.hin_ss;
  for (int e = tid; e < RPM * 8; e += THR) {
    const int r = e >> 3, col = e & 7, k = k0 + col;
    if (k >= K || r >= rows) continue;
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < XW; ++w) s += red[(w * RPM + r) * 8 + col];
    const double hv = hin[(size_t)r * K + k];
    a.gzprev[scene * a.gzp_ss + (size_t)r * K + k] = s * (1.0 - hv * hv);
  }
  tl_mark(a.tl, 2);
}

struct AdamLayer {
  const double* gz;       // [S][rows][N]
  const double* hin;      // [S][rows][K]
  long long gz_ss, hin_ss, w_off, b_off;
  int N, K;
  int nblk, strips;       // 64-output n-blocks x 32-input k-strips (one CTA each)
  int items;              // nblk * strips weight CTAs + bias CTAs (256 outputs each)
  int wait;               // g_z written by the launch right before: wait for it
};

struct NetAdamArgs {
  AdamLayer L[3];         // in launch order (layers whose g_z is older first)
  int rows;
  double* theta; double* m; double* v; long long th_ss;
  const int* step;
  const int* tsnap;       // Adam t snapshot of this iteration (side-stream launches) or null
  double lr, b1, b2, eps;
  int* err;
  int tl;
};

constexpr int AX_ST = 4;          // k-tiles per strip (32 inputs)
constexpr int AX_NB = XW * 8;     // outputs per n-block (one n-tile per warp)

// CTA = (n-block, k-strip) of one layer: warp w updates n-tile w of the
// block over the strip's four k-tiles.  W, m, v fragments go to registers,
// the strip's h columns and the block's g_z columns to shared memory, all
// requested at once; layers whose g_z is two or more launches old do not
// wait for the previous kernel at all.
constexpr int AX_HP = AX_ST * 8 + 4, AX_GP = AX_NB + 4;   // pitches = 4 mod 16: conflict-free fragment reads
__host__ __device__ constexpr size_t adam_x_smem_bytes(int MT) {
  return (size_t)8 * MT * (AX_HP + AX_GP) * sizeof(double);
}

template <int MT>
__global__ void __launch_bounds__(256) net_adam_x_kernel(NetAdamArgs a) {
  constexpr int RPM = 8 * MT, NS = RPM / 4;
  constexpr int HP = AX_HP, GP = AX_GP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* hS = reinterpret_cast<double*>(smem_raw);   // [RPM][HP]
  double* gS = hS + RPM * HP;                          // [RPM][GP]
  __shared__ double bc_s[2];
  const int scene = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  tl_mark(a.tl, 0);
  int item = blockIdx.x, li = 0;
  while (li < 2 && item >= a.L[li].items) { item -= a.L[li].items; ++li; }
  const AdamLayer L = a.L[li];
  const int K = L.K, N = L.N, rows = a.rows;
  double* __restrict__ th = a.theta + scene * a.th_ss;
  double* __restrict__ mm = a.m + scene * a.th_ss;
  double* __restrict__ vv = a.v + scene * a.th_ss;
  const double* __restrict__ gz = L.gz + scene * L.gz_ss;
  if (tid == 0) {
    const double tt = (double)(a.tsnap ? *a.tsnap : *a.step);
    bc_s[0] = 1.0 / (1.0 - pow(a.b1, tt));
    bc_s[1] = 1.0 / (1.0 - pow(a.b2, tt));
  }
  int errbits = 0;
  const int wc = L.nblk * L.strips;
  if (item < wc) {
    const int nb = item / L.strips, k0 = (item % L.strips) * AX_ST * 8;
    const int n = nb * AX_NB + warp * 8 + g;
    // W, m, v (final since the previous iteration) and the strip's h (the forward's)
    double2 wp[AX_ST], wm[AX_ST], wv[AX_ST];
    bool tok[AX_ST];
#pragma unroll
    for (int j = 0; j < AX_ST; ++j) {
      const int kk = k0 + j * 8 + 2 * t;
      tok[j] = n < N && kk < K;
      const size_t o = tok[j] ? L.w_off + (size_t)n * K + kk : 0;
      wp[j] = tok[j] ? *reinterpret_cast<const double2*>(th + o) : make_double2(0.0, 0.0);
      wm[j] = tok[j] ? *reinterpret_cast<const double2*>(mm + o) : make_double2(0.0, 0.0);
      wv[j] = tok[j] ? *reinterpret_cast<const double2*>(vv + o) : make_double2(0.0, 0.0);
    }
    const double* hin = L.hin + scene * L.hin_ss;
    for (int i = tid; i < RPM * AX_ST * 4; i += blockDim.x) {     // 16-byte pieces: [r][16]
      const int r = i / (AX_ST * 4), sg = i % (AX_ST * 4), kk = k0 + 2 * sg;
      const bool ok = r < rows && kk < K;
      cp_async16(hS + r * HP + 2 * sg, ok ? hin + (size_t)r * K + kk : hin, ok);
    }
    if (L.wait) pdl_wait();
    tl_mark(a.tl, 1);   // first dependent work (CTAs of layers whose g_z is old do not wait)
    for (int i = tid; i < RPM * AX_NB / 2; i += blockDim.x) {
      const int r = i / (AX_NB / 2), sg = i % (AX_NB / 2), nn = nb * AX_NB + 2 * sg;
      const bool ok = r < rows && nn < N;
      cp_async16(gS + r * GP + 2 * sg, ok ? gz + (size_t)r * N + nn : gz, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    const double ibc1 = bc_s[0], ibc2 = bc_s[1];
    double ga[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) ga[s] = gS[(4 * s + t) * GP + warp * 8 + g];   // A[g][t] = g_z[4s + t][n]
    // NA accumulator pairs per tile break the dependent DMMA chain over rows
    constexpr int NA = NS >= 12 ? 3 : (NS >= 4 ? 2 : 1);
#pragma unroll
    for (int j = 0; j < AX_ST; ++j) {
      double e0[NA], e1[NA];
#pragma unroll
      for (int q = 0; q < NA; ++q) e0[q] = e1[q] = 0.0;
#pragma unroll
      for (int s = 0; s < NS; ++s) dmma(e0[s % NA], e1[s % NA], ga[s], hS[(4 * s + t) * HP + j * 8 + g]);   // B[t][g] = h[4s + t][k]
      double d0 = e0[0], d1 = e1[0];
#pragma unroll
      for (int q = 1; q < NA; ++q) { d0 += e0[q]; d1 += e1[q]; }
      if (!tok[j]) continue;
      if (!isfinite(d0) || !isfinite(d1)) errbits |= ERR_NONFINITE_GRAD;
      adam_one<double>(wp[j].x, wm[j].x, wv[j].x, d0, a.lr, a.b1, a.b2, a.eps, ibc1, ibc2);
      adam_one<double>(wp[j].y, wm[j].y, wv[j].y, d1, a.lr, a.b1, a.b2, a.eps, ibc1, ibc2);
      if (!isfinite(wp[j].x) || !isfinite(wp[j].y)) errbits |= ERR_NONFINITE_PARAM;
      const size_t o = L.w_off + (size_t)n * K + k0 + j * 8 + 2 * t;
      *reinterpret_cast<double2*>(th + o) = wp[j];
      *reinterpret_cast<double2*>(mm + o) = wm[j];
      *reinterpret_cast<double2*>(vv + o) = wv[j];
    }
  } else {
    // bias CTA: outputs 256 * (item - wc) + tid (network.py:213,217)
    const int bn = (item - wc) * 256 + tid;
    const size_t o = L.b_off + (bn < N ? bn : 0);
    double p = th[o], m1 = mm[o], v1 = vv[o];
    if (L.wait) pdl_wait();
    tl_mark(a.tl, 1);   // first dependent work (CTAs of layers whose g_z is old do not wait)
    __syncthreads();
    if (bn < N) {
      double gb = 0.0;
      for (int r = 0; r < rows; ++r) gb += gz[(size_t)r * N + bn];
      if (!isfinite(gb)) errbits |= ERR_NONFINITE_GRAD;
      adam_one<double>(p, m1, v1, gb, a.lr, a.b1, a.b2, a.eps, bc_s[0], bc_s[1]);
      if (!isfinite(p)) errbits |= ERR_NONFINITE_PARAM;
      th[o] = p; mm[o] = m1; vv[o] = v1;
    }
  }
  if (errbits) atomicOr(&a.err[scene], errbits);
  tl_mark(a.tl, 2);
}

// The same update as a persistent, warp-specialised kernel for many rows
// (config 5: 72 rows, 33.6 M parameters): one CTA per SM walks its share of
// the (n-block, k-strip) items; four loader warps feed a three-stage shared-memory
// ring with the item's W, m, v tiles (64 rows x 256 bytes each) and the strip's
// h columns -- the block's g_z columns take a stage of their own at the start
// of a run of k-strips -- (16-byte cp.async pieces whose
// completion arrives on the stage's mbarrier; as 1-D bulk copies of one row
// each -- 336 TMA instructions per item -- the kernel ran at 10 us per item,
// 1 136 us), so the next item's 108 KB stream in while
// the eight compute warps run the current item's DMMA product and Adam
// arithmetic and store W, m, v straight from registers.  net_adam_x_kernel
// above requests everything of an item at once and then computes: with two
// CTAs per SM its loads, arithmetic and stores barely overlap (0.49 of HBM).
// Row pitches: W / m / v tiles 34 doubles, h 36, g_z 68 (conflict-free 16-byte
// and fragment reads).  Used when N % 64 == 0 and K % 32 == 0 for every layer.
constexpr int AR_WP = AX_ST * 8 + 2;
constexpr int AR_CW = 8;                        // compute warps (16 = two per n-tile measured no faster)
constexpr int AR_THREADS = (AR_CW + 4) * 32;    // + four loader warps
constexpr int AR_NST = 3;                       // ring stages: two items' W / m / v in flight beside the one in use
// a stage holds an item's W / m / v tiles and h columns, or (first step of a
// run of k-strips) the n-block's g_z columns, which the compute warps copy
// into their A-fragment registers for the whole run
__host__ __device__ constexpr size_t adam_ring_stage_doubles(int MT) {
  return (size_t)3 * AX_NB * AR_WP + (size_t)8 * MT * AX_HP;
}
__host__ __device__ constexpr size_t adam_ring_smem_bytes(int MT) {
  return AR_NST * adam_ring_stage_doubles(MT) * sizeof(double) + 128;
}

template <int MT>
__global__ void __launch_bounds__(AR_THREADS, 1) net_adam_ring_kernel(NetAdamArgs a) {
  constexpr int RPM = 8 * MT, NS = RPM / 4;
  constexpr int HP = AX_HP, GP = AX_GP, WP = AR_WP, NST = AR_NST, JW = AX_ST;
  constexpr size_t STG = adam_ring_stage_doubles(MT);
  static_assert((size_t)RPM * GP <= (size_t)3 * AX_NB * WP, "the g_z block must fit the W / m / v part of a stage");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(ring + NST * STG);   // full[NST], empty[NST]
  __shared__ double bc_s[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int rows = a.rows;
  tl_mark(a.tl, 0);
  if (tid == 0) {
    const double tt = (double)(a.tsnap ? *a.tsnap : *a.step);
    bc_s[0] = 1.0 / (1.0 - pow(a.b1, tt));
    bc_s[1] = 1.0 / (1.0 - pow(a.b2, tt));
    for (int st = 0; st < NST; ++st) {
      mbar_init(&bars[st], 128);           // one (asynchronous) arrival per loader thread
      mbar_init(&bars[NST + st], AR_CW);   // one arrival per compute warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // rows beyond `rows` of the h part of every stage stay zero for the whole kernel
  for (int st = 0; st < NST; ++st) {
    double* hS = ring + st * STG + 3 * AX_NB * WP;
    for (int i = tid; i < (RPM - rows) * HP; i += blockDim.x) hS[(size_t)rows * HP + i] = 0.0;
  }
  __syncthreads();
  const int total = a.L[0].items + a.L[1].items + a.L[2].items;
  // item sequence of this CTA: runs of AR_RUN consecutive items (consecutive
  // k-strips of one n-block share the g_z block), the runs dealt round-robin so
  // every CTA starts with the layers whose g_z is oldest
  constexpr int AR_RUN = 8;
  const int nseq = (total + AR_RUN * (int)gridDim.x - 1) / (AR_RUN * (int)gridDim.x) * AR_RUN;
  auto item_at = [&](int q) { return (q / AR_RUN) * (AR_RUN * (int)gridDim.x) + (int)blockIdx.x * AR_RUN + (q % AR_RUN); };
  double* __restrict__ th = a.theta;
  double* __restrict__ mm = a.m;
  double* __restrict__ vv = a.v;
  auto decode = [&](int item, int& li, int& local) {
    li = 0;
    local = item;
    while (li < 2 && local >= a.L[li].items) { local -= a.L[li].items; ++li; }
  };

  if (warp >= AR_CW) {
    // ---------------- loader warps (4): 16-byte cp.async pieces, completion on the stage's mbarrier
    const int lt = tid - AR_CW * 32;   // 0 .. 127
    bool waited = false;
    int ring_it = 0, gz_key = -1;
    for (int q = 0; q < nseq; ++q) {
      const int item = item_at(q);
      if (item >= total) continue;
      int li, local;
      decode(item, li, local);
      const AdamLayer L = a.L[li];
      if (local >= L.nblk * L.strips) continue;   // bias item: no ring stage
      if (L.wait && !waited) { pdl_wait(); waited = true; }
      const int nb = local / L.strips, k0 = (local % L.strips) * AX_ST * 8, n0 = nb * AX_NB;
      const int K = L.K, N = L.N;
      const int key = li * 65536 + nb;
      if (key != gz_key) {
        // a new n-block: its g_z columns take a stage of their own
        gz_key = key;
        const int st = ring_it % NST;
        mbar_wait(&bars[NST + st], ((ring_it / NST) & 1) ^ 1);
        double* gS = ring + st * STG;
        const int sg2 = lt & 31, q0 = lt >> 5;   // rows x 32 pieces
        for (int r = q0; r < rows; r += 4)
          cp_async16(gS + (size_t)r * GP + 2 * sg2, L.gz + (size_t)r * N + n0 + 2 * sg2, true);
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&bars[st])) : "memory");
        ++ring_it;
      }
      const int st = ring_it % NST;
      mbar_wait(&bars[NST + st], ((ring_it / NST) & 1) ^ 1);   // stage free (the first round passes)
      double* Wt = ring + st * STG;
      double* hS = Wt + 3 * AX_NB * WP;
      {
        // W, m, v tiles: 64 rows x 16 pieces each; thread lt takes piece lt % 16 of rows lt / 16 + 8 i
        const int seg = lt & 15, r0 = lt >> 4;
        const size_t go = L.w_off + (size_t)(n0 + r0) * K + k0 + 2 * seg;
        double* dw = Wt + (size_t)r0 * WP + 2 * seg;
#pragma unroll
        for (int i = 0; i < AX_NB / 8; ++i) {
          cp_async16(dw + (size_t)(8 * i) * WP, th + go + (size_t)(8 * i) * K, true);
          cp_async16(dw + (size_t)(AX_NB + 8 * i) * WP, mm + go + (size_t)(8 * i) * K, true);
          cp_async16(dw + (size_t)(2 * AX_NB + 8 * i) * WP, vv + go + (size_t)(8 * i) * K, true);
        }
        // h strip: rows x 16 pieces
        for (int r = r0; r < rows; r += 8) cp_async16(hS + (size_t)r * HP + 2 * seg, L.hin + (size_t)r * K + k0 + 2 * seg, true);
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&bars[st])) : "memory");
      ++ring_it;
    }
    tl_mark(a.tl, 2);
    return;
  }

  // ---------------- compute warps ----------------
  const double ibc1 = bc_s[0], ibc2 = bc_s[1];
  int errbits = 0;
  bool waited = false, marked = false;
  int ring_it = 0, gz_key = -1;
  double ga[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) ga[s] = 0.0;
  for (int q = 0; q < nseq; ++q) {
    const int item = item_at(q);
    if (item >= total) continue;
    int li, local;
    decode(item, li, local);
    const AdamLayer L = a.L[li];
    const int K = L.K, N = L.N;
    const int wc = L.nblk * L.strips;
    if (local < wc) {
      const int nb = local / L.strips, k0 = (local % L.strips) * AX_ST * 8;
      const int n = nb * AX_NB + warp * 8 + g;
      const int key = li * 65536 + nb;
      if (key != gz_key) {
        gz_key = key;
        const int st = ring_it % NST;
        mbar_wait(&bars[st], (ring_it / NST) & 1);
        if (!marked) { tl_mark(a.tl, 1); marked = true; }
        const double* gS = ring + st * STG;
#pragma unroll
        for (int s = 0; s < NS; ++s) ga[s] = 4 * s + t < rows ? gS[(4 * s + t) * GP + warp * 8 + g] : 0.0;   // A[g][t] = g_z[4s + t][n]
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[NST + st]);
        ++ring_it;
      }
      const int st = ring_it % NST;
      mbar_wait(&bars[st], (ring_it / NST) & 1);
      const double* Wt = ring + st * STG;
      const double* hS = Wt + 3 * AX_NB * WP;
      double2 wp[JW], wm[JW], wv[JW];
#pragma unroll
      for (int j = 0; j < JW; ++j) {
        const size_t o = (size_t)(warp * 8 + g) * WP + j * 8 + 2 * t;
        wp[j] = *reinterpret_cast<const double2*>(Wt + o);
        wm[j] = *reinterpret_cast<const double2*>(Wt + (size_t)AX_NB * WP + o);
        wv[j] = *reinterpret_cast<const double2*>(Wt + (size_t)2 * AX_NB * WP + o);
      }
      constexpr int NA = NS >= 12 ? 3 : (NS >= 4 ? 2 : 1);
      double dg[JW][2];
#pragma unroll
      for (int j = 0; j < JW; ++j) {
        double e0[NA], e1[NA];
#pragma unroll
        for (int qq = 0; qq < NA; ++qq) e0[qq] = e1[qq] = 0.0;
#pragma unroll
        for (int s = 0; s < NS; ++s) dmma(e0[s % NA], e1[s % NA], ga[s], hS[(4 * s + t) * HP + j * 8 + g]);   // B[t][g] = h[4s + t][k]
        double d0 = e0[0], d1 = e1[0];
#pragma unroll
        for (int qq = 1; qq < NA; ++qq) { d0 += e0[qq]; d1 += e1[qq]; }
        dg[j][0] = d0;
        dg[j][1] = d1;
      }
      // every shared-memory read of this stage is done: hand it back to the loader
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[NST + st]);
      ++ring_it;
#pragma unroll
      for (int j = 0; j < JW; ++j) {
        const double d0 = dg[j][0], d1 = dg[j][1];
        if (!isfinite(d0) || !isfinite(d1)) errbits |= ERR_NONFINITE_GRAD;
        adam_one<double>(wp[j].x, wm[j].x, wv[j].x, d0, a.lr, a.b1, a.b2, a.eps, ibc1, ibc2);
        adam_one<double>(wp[j].y, wm[j].y, wv[j].y, d1, a.lr, a.b1, a.b2, a.eps, ibc1, ibc2);
        if (!isfinite(wp[j].x) || !isfinite(wp[j].y)) errbits |= ERR_NONFINITE_PARAM;
        const size_t o = L.w_off + (size_t)n * K + k0 + j * 8 + 2 * t;
        *reinterpret_cast<double2*>(th + o) = wp[j];
        *reinterpret_cast<double2*>(mm + o) = wm[j];
        *reinterpret_cast<double2*>(vv + o) = wv[j];
      }
    } else {
      // bias item: outputs 256 * (local - wc) + tid (network.py:213,217)
      const int bn = (local - wc) * 256 + tid;
      if (L.wait && !waited) { pdl_wait(); waited = true; }
      if (!marked) { tl_mark(a.tl, 1); marked = true; }
      if (tid < 256 && bn < N) {
        const size_t o = L.b_off + bn;
        double p = th[o], m1 = mm[o], v1 = vv[o];
        double gb = 0.0;
        for (int r = 0; r < rows; ++r) gb += L.gz[(size_t)r * N + bn];
        if (!isfinite(gb)) errbits |= ERR_NONFINITE_GRAD;
        adam_one<double>(p, m1, v1, gb, a.lr, a.b1, a.b2, a.eps, ibc1, ibc2);
        if (!isfinite(p)) errbits |= ERR_NONFINITE_PARAM;
        th[o] = p; mm[o] = m1; vv[o] = v1;
      }
    }
  }
  if (errbits) atomicOr(&a.err[0], errbits);
  tl_mark(a.tl, 2);
}

// g_h = g_z W_old for many rows or wide layers (network.py:210-212): CTA =
// all rows x 64 outputs (one 8-wide k-tile per warp), n reduction in chunks
// of 32 staged with cp.async (double-buffered), split over grid.y slices;
// the slice partials are added in slice order by the last CTA of each
// k-block (atomic ticket, self-resetting), which applies (1 - h^2).
constexpr int GT_NC = 32;
constexpr int GH_NSL = 16;   // max n slices
constexpr int GT_GP = GT_NC + 4;   // pitch = 4 mod 16
// KTW k-tiles of 8 per warp (CTA = XW * 8 * KTW outputs): the A fragments of
// all rows are reused from registers across them, so shared-memory traffic
// per DMMA drops from ~1 fragment to (MT + KTW) / (MT KTW)
__host__ __device__ constexpr int gt_kb(int KTW) { return XW * 8 * KTW; }
__host__ __device__ constexpr int gt_wp(int KTW) { return gt_kb(KTW) + 4; }
__host__ __device__ constexpr size_t gh_t_smem_bytes(int MT, int KTW) {
  return ((size_t)2 * 8 * MT * GT_GP + (size_t)2 * GT_NC * gt_wp(KTW)) * sizeof(double);
}

struct GhArgs {
  int rows, K, N, nsl, ns;          // ns: n per slice (multiple of GT_NC)
  const double* gz; long long gz_ss;
  const double* hin; long long hin_ss;
  const double* theta; long long th_ss, w_off;
  double* gzprev; long long gzp_ss;
  double* part;                      // [S][nsl][rows][K]
  int* ticket;                       // [S][K / 64 + 1]
  int tl;
};

template <int MT, int KTW>
__global__ void __launch_bounds__(XW * 32) net_gh_t_kernel(GhArgs a) {
  constexpr int RPM = 8 * MT, THR = XW * 32, KB = gt_kb(KTW), WP = gt_wp(KTW);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Gs = reinterpret_cast<double*>(smem_raw);   // [2][RPM][GT_GP]
  double* Ws = Gs + 2 * RPM * GT_GP;                   // [2][GT_NC][WP]
  __shared__ int last_s;
  const int K = a.K, N = a.N, rows = a.rows;
  const int scene = blockIdx.z, sl = blockIdx.y, kb = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int k0 = kb * KB;
  const int n0 = sl * a.ns, n1 = min(N, n0 + a.ns);
  const double* __restrict__ W = a.theta + scene * a.th_ss + a.w_off;
  const double* __restrict__ gz = a.gz + scene * a.gz_ss;
  tl_mark(a.tl, 0);
  auto stage_w = [&](int c, int b) {
    const int nc = n0 + c * GT_NC;
    double* dst = Ws + b * GT_NC * WP;
    for (int i = tid; i < GT_NC * KB / 2; i += THR) {
      const int r = i / (KB / 2), sg = i % (KB / 2), n = nc + r, k = k0 + 2 * sg;
      const bool ok = n < n1 && k < K;
      cp_async16(dst + r * WP + 2 * sg, ok ? W + (size_t)n * K + k : W, ok);
    }
  };
  auto stage_g = [&](int c, int b) {
    const int nc = n0 + c * GT_NC;
    double* dst = Gs + b * RPM * GT_GP;
    for (int i = tid; i < RPM * GT_NC / 2; i += THR) {
      const int r = i / (GT_NC / 2), sg = i % (GT_NC / 2), n = nc + 2 * sg;
      const bool ok = r < rows && n < n1;
      cp_async16(dst + r * GT_GP + 2 * sg, ok ? gz + (size_t)r * N + n : gz, ok);
    }
  };
  const int nch = (n1 - n0 + GT_NC - 1) / GT_NC;
  // W_old is final since the previous iteration: the first chunk before the wait
  if (nch > 0) stage_w(0, 0);
  pdl_wait();
  tl_mark(a.tl, 1);
  if (nch > 0) stage_g(0, 0);
  cp_async_commit();
  double acc[MT][KTW][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < KTW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) { stage_w(c + 1, (c + 1) & 1); stage_g(c + 1, (c + 1) & 1); }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* G = Gs + (c & 1) * RPM * GT_GP;
    const double* Wc = Ws + (c & 1) * GT_NC * WP;
#pragma unroll
    for (int q = 0; q < GT_NC / 4; ++q) {
      double bv[KTW], av[MT];
#pragma unroll
      for (int j = 0; j < KTW; ++j) bv[j] = Wc[(4 * q + t) * WP + (warp * KTW + j) * 8 + g];   // B[t][g] = W[n + t][k + g]
#pragma unroll
      for (int i = 0; i < MT; ++i) av[i] = G[(8 * i + g) * GT_GP + 4 * q + t];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < KTW; ++j) dmma(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    }
    __syncthreads();
  }
  pdl_trigger();
  // slice partial -> global, then the last CTA of this k-block reduces
  double* P = a.part + ((size_t)scene * a.nsl + sl) * rows * K;
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < KTW; ++j)
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const int r = 8 * i + g, k = k0 + (warp * KTW + j) * 8 + 2 * t + cc;
        if (r < rows && k < K) P[(size_t)r * K + k] = acc[i][j][cc];
      }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    int* tk = a.ticket + (size_t)scene * gridDim.x + kb;
    const int prev = atomicAdd(tk, 1);
    last_s = prev == a.nsl - 1;
    if (last_s) *tk = 0;   // ready for the next launch
  }
  __syncthreads();
  if (last_s) {
    __threadfence();
    const double* __restrict__ hin = a.hin + scene * a.hin_ss;
    for (int e = tid; e < rows * KB; e += THR) {
      const int r = e / KB, k = k0 + e % KB;
      if (k >= K) continue;
      double s = 0.0;
      for (int q = 0; q < a.nsl; ++q)
        s += __ldcg(a.part + (((size_t)scene * a.nsl + q) * rows + r) * K + k);
      const double hv = hin[(size_t)r * K + k];
      a.gzprev[scene * a.gzp_ss + (size_t)r * K + k] = s * (1.0 - hv * hv);
    }
  }
  tl_mark(a.tl, 2);
}

}  // namespace pdf
