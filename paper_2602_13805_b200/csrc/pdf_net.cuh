// The per-scene corrective network (network.py:53-223) and its Adam update
// (network.py:230-264), batched over scenes.
//
// Parameters live in one flat buffer per scene in the reference order
// w1, b1, w2, b2, w3, b3 with weights row-major (fan_out, fan_in), so
// grad_loss / adam_step see the same flat vector the reference does.
//
// Forward layer  z = h W^T + b: CTA = 128 outputs x all rows for one K-slice;
//   the CK CTAs of a cluster split K and reduce their partials through
//   distributed shared memory in a fixed order (no float atomics).
// Backward layer: CTA = 128 input columns x one slice of the outputs;
//   it computes the partial g_h = g_z W from the OLD weights, the weight
//   gradient g_W = g_z^T h tile by tile, and applies Adam in the same pass
//   (the gradient never round-trips through HBM).  The CN CTAs of a
//   cluster split the outputs and reduce g_h through DSMEM, then apply the
//   tanh' of the layer input to produce the next g_z.
#pragma once
#include "pdf_common.cuh"

namespace pdf {

constexpr int NET_TILE = 128;   // outputs (fwd) / input columns (bwd) per CTA
constexpr int NET_THREADS = 128;
constexpr int NET_KC = 16;      // K (fwd) / N (bwd) chunk staged per step
constexpr double OUTPUT_GAIN = 8.0;   // network.py:85

template <typename T>
struct NetFwdArgs {
  int rows, K, N;
  const T* in; long long in_ss;       // [S][rows][K]
  const T* theta; long long th_ss;    // [S][Np]
  long long w_off, b_off;
  T* out; long long out_ss;           // [S][rows][N]   (tanh layers)
  int final_layer;
  // final layer: alpha_hat = alpha0 + merge(y * cout)
  const T* cout;                      // [S][N]
  const C<T>* alpha0;                 // [S][n][M0]
  C<T>* alpha_hat;                    // [S][n][M0]
  int n, M0, joint;
  int* step;                          // incremented once (train mode) or null
};

// rows padded to 16*RB; thread (rg, ng) of warp w owns rows rb*16+rg*4+{0..3}
// and outputs w*32+ng*4+{0..3}
template <typename T, int RB>
__global__ void __launch_bounds__(NET_THREADS) net_fwd_kernel(NetFwdArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  const int CK = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int scene = blockIdx.z;
  const int n0 = blockIdx.x * NET_TILE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rg = lane >> 3, ng = lane & 7;
  const int RP = 16 * RB;
  const int K = a.K, N = a.N, rows = a.rows;

  if (a.step && tid == 0 && blockIdx.x == 0 && blockIdx.y == 0 && scene == 0) atomicAdd(a.step, 1);

  T* Ws = reinterpret_cast<T*>(smem_raw);            // [TILE][KC+1]
  T* Xs = Ws + NET_TILE * (NET_KC + 1);              // [RP][KC+1]
  T* red = Xs + RP * (NET_KC + 1);                   // [RP][TILE] partial output

  const int ks = (K + CK - 1) / CK;
  const int kb = rank * ks, ke = min(K, kb + ks);
  const T* W = a.theta + scene * a.th_ss + a.w_off;
  const T* X = a.in + scene * a.in_ss;

  T acc[RB][4][4];
#pragma unroll
  for (int b = 0; b < RB; ++b)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[b][i][j] = T(0);

  for (int k0 = kb; k0 < ke; k0 += NET_KC) {
    __syncthreads();
    for (int idx = tid; idx < NET_TILE * NET_KC; idx += NET_THREADS) {
      const int nn = idx / NET_KC, kk = idx % NET_KC;
      const int gn = n0 + nn, gk = k0 + kk;
      Ws[nn * (NET_KC + 1) + kk] = (gn < N && gk < ke) ? W[(size_t)gn * K + gk] : T(0);
    }
    for (int idx = tid; idx < RP * NET_KC; idx += NET_THREADS) {
      const int r = idx / NET_KC, kk = idx % NET_KC;
      const int gk = k0 + kk;
      Xs[r * (NET_KC + 1) + kk] = (r < rows && gk < ke) ? X[(size_t)r * K + gk] : T(0);
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < NET_KC; ++kk) {
      T wv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) wv[j] = Ws[(warp * 32 + ng * 4 + j) * (NET_KC + 1) + kk];
#pragma unroll
      for (int b = 0; b < RB; ++b) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const T xv = Xs[(b * 16 + rg * 4 + i) * (NET_KC + 1) + kk];
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[b][i][j] += xv * wv[j];
        }
      }
    }
  }
#pragma unroll
  for (int b = 0; b < RB; ++b)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) red[(b * 16 + rg * 4 + i) * NET_TILE + warp * 32 + ng * 4 + j] = acc[b][i][j];
  cluster.sync();

  // reduce-scatter over the cluster, fixed rank order, then the epilogue
  const T* bias = a.theta + scene * a.th_ss + a.b_off;
  const int total = rows * NET_TILE;
  for (int e = rank + CK * tid; e < total; e += CK * NET_THREADS) {
    const int r = e / NET_TILE, nn = e % NET_TILE, gn = n0 + nn;
    if (gn >= N) continue;
    T s = T(0);
    for (int c = 0; c < CK; ++c) s += cluster.map_shared_rank(red, c)[r * NET_TILE + nn];
    const T z = s + bias[gn];
    if (!a.final_layer) {
      a.out[scene * a.out_ss + (size_t)r * N + gn] = tanh(z);
    } else {
      const T yv = z * a.cout[(size_t)scene * N + gn];
      // [Re | Im] feature layout (network.py:123-136)
      const int half = N / 2;
      const int f = gn < half ? gn : gn - half;
      int view, m;
      if (a.joint) { view = f / a.M0; m = f % a.M0; } else { view = r; m = f; }
      const size_t o = ((size_t)scene * a.n + view) * a.M0 + m;
      T* dst = reinterpret_cast<T*>(a.alpha_hat + o);
      const T* src = reinterpret_cast<const T*>(a.alpha0 + o);
      if (gn < half) dst[0] = src[0] + yv; else dst[1] = src[1] + yv;
    }
  }
  cluster.sync();
}

template <typename T>
struct NetBwdArgs {
  int rows, K, N;
  const T* gz; long long gz_ss;       // [S][rows][N]   gradient at this layer's pre-activation
  const T* hin; long long hin_ss;     // [S][rows][K]   this layer's input
  T* theta; long long th_ss;          // [S][Np] (updated in place when fused)
  long long w_off, b_off;
  T* m; T* v;                         // Adam moments, same layout as theta
  T* grad;                            // [S][Np] gradient out (unfused mode) or null
  int fused;                          // 1: apply Adam, 0: write grad
  const int* step;                    // Adam t (device)
  T lr, b1, b2, eps;
  T* gzprev; long long gzp_ss;        // [S][rows][K] or null (first layer)
  int* err;                           // [S]
};

template <typename T>
__device__ __forceinline__ void adam_one(T& p, T& m, T& v, T g, T lr, T b1, T b2, T eps, T bc1, T bc2) {
  m = b1 * m + (T(1) - b1) * g;
  v = b2 * v + (T(1) - b2) * g * g;
  const T mh = m / bc1;
  const T vh = v / bc2;
  p = p - lr * mh / (sqrt_<T>(vh) + eps);
}

// thread (warp w, lane): gh micro-tile rows rb*16 + (lane>>3)*4 + i, columns (lane&7)*4 + j + 32*w
template <typename T, int RB>
__global__ void __launch_bounds__(NET_THREADS) net_bwd_kernel(NetBwdArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  const int CN = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int scene = blockIdx.z;
  const int k0 = blockIdx.x * NET_TILE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rg = lane >> 3, cg_ = lane & 7;
  const int RP = 16 * RB;
  const int K = a.K, N = a.N, rows = a.rows;

  T* Hs = reinterpret_cast<T*>(smem_raw);       // [RP][TILE]
  T* Ws = Hs + RP * NET_TILE;                   // [KC][TILE]
  T* Gs = Ws + NET_KC * NET_TILE;               // [RP][KC+1]
  T* red = Gs + RP * (NET_KC + 1);              // [RP][TILE]

  const T* hin = a.hin + scene * a.hin_ss;
  const T* gz = a.gz + scene * a.gz_ss;
  T* th = a.theta + scene * a.th_ss;
  T* W = th + a.w_off;
  T* bia = th + a.b_off;
  T* mW = a.m + scene * a.th_ss + a.w_off;
  T* vW = a.v + scene * a.th_ss + a.w_off;
  T* mb = a.m + scene * a.th_ss + a.b_off;
  T* vb = a.v + scene * a.th_ss + a.b_off;
  T* gW = a.grad ? a.grad + scene * a.th_ss + a.w_off : nullptr;
  T* gB = a.grad ? a.grad + scene * a.th_ss + a.b_off : nullptr;

  T bc1 = T(1), bc2 = T(1);
  if (a.fused) {
    const int t = *a.step;
    bc1 = T(1.0 - pow((double)a.b1, (double)t));
    bc2 = T(1.0 - pow((double)a.b2, (double)t));
  }

  for (int idx = tid; idx < RP * NET_TILE; idx += NET_THREADS) {
    const int r = idx / NET_TILE, kk = idx % NET_TILE, gk = k0 + kk;
    Hs[idx] = (r < rows && gk < K) ? hin[(size_t)r * K + gk] : T(0);
  }

  const int ns = (N + CN - 1) / CN;
  const int nb = rank * ns, ne = min(N, nb + ns);

  T acc[RB][4][4];
#pragma unroll
  for (int b = 0; b < RB; ++b)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[b][i][j] = T(0);

  int errbits = 0;
  for (int c0 = nb; c0 < ne; c0 += NET_KC) {
    __syncthreads();
    for (int idx = tid; idx < NET_KC * NET_TILE; idx += NET_THREADS) {
      const int nn = idx / NET_TILE, kk = idx % NET_TILE;
      const int gn = c0 + nn, gk = k0 + kk;
      Ws[idx] = (gn < ne && gk < K) ? W[(size_t)gn * K + gk] : T(0);
    }
    for (int idx = tid; idx < RP * NET_KC; idx += NET_THREADS) {
      const int r = idx / NET_KC, nn = idx % NET_KC, gn = c0 + nn;
      Gs[r * (NET_KC + 1) + nn] = (r < rows && gn < ne) ? gz[(size_t)r * N + gn] : T(0);
    }
    __syncthreads();
    // g_h partial with the old weights
#pragma unroll 4
    for (int nn = 0; nn < NET_KC; ++nn) {
      T wv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) wv[j] = Ws[nn * NET_TILE + warp * 32 + cg_ * 4 + j];
#pragma unroll
      for (int b = 0; b < RB; ++b)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const T gv = Gs[(b * 16 + rg * 4 + i) * (NET_KC + 1) + nn];
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[b][i][j] += gv * wv[j];
        }
    }
    // weight gradient + Adam for the chunk: thread owns n = c0 + warp*4 + i (i<4),
    // k = k0 + lane + 32*j (j<4) so each warp touches contiguous rows of m, v, W
    {
      T g[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) g[i][j] = T(0);
      for (int r = 0; r < rows; ++r) {
        T hv[4], gv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) hv[j] = Hs[r * NET_TILE + lane + 32 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i) gv[i] = Gs[r * (NET_KC + 1) + warp * 4 + i];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) g[i][j] += gv[i] * hv[j];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int gn = c0 + warp * 4 + i;
        if (gn >= ne) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int gk = k0 + lane + 32 * j;
          if (gk >= K) continue;
          const size_t o = (size_t)gn * K + gk;
          const T gg = g[i][j];
          if (!isfinite(gg)) errbits |= ERR_NONFINITE_GRAD;
          if (a.fused) {
            T p = Ws[(warp * 4 + i) * NET_TILE + lane + 32 * j];
            T mm = mW[o], vv = vW[o];
            adam_one<T>(p, mm, vv, gg, a.lr, a.b1, a.b2, a.eps, bc1, bc2);
            if (!isfinite(p)) errbits |= ERR_NONFINITE_PARAM;
            W[o] = p; mW[o] = mm; vW[o] = vv;
          } else {
            gW[o] = gg;
          }
        }
      }
      // bias: owned by the first column tile
      if (blockIdx.x == 0 && tid < NET_KC) {
        const int gn = c0 + tid;
        if (gn < ne) {
          T gb = T(0);
          for (int r = 0; r < rows; ++r) gb += Gs[r * (NET_KC + 1) + tid];
          if (!isfinite(gb)) errbits |= ERR_NONFINITE_GRAD;
          if (a.fused) {
            T p = bia[gn], mm = mb[gn], vv = vb[gn];
            adam_one<T>(p, mm, vv, gb, a.lr, a.b1, a.b2, a.eps, bc1, bc2);
            if (!isfinite(p)) errbits |= ERR_NONFINITE_PARAM;
            bia[gn] = p; mb[gn] = mm; vb[gn] = vv;
          } else {
            gB[gn] = gb;
          }
        }
      }
    }
  }
  if (errbits) atomicOr(&a.err[scene], errbits);

  if (a.gzprev) {
#pragma unroll
    for (int b = 0; b < RB; ++b)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          red[(b * 16 + rg * 4 + i) * NET_TILE + warp * 32 + cg_ * 4 + j] = acc[b][i][j];
    cluster.sync();
    const int total = rows * NET_TILE;
    for (int e = rank + CN * tid; e < total; e += CN * NET_THREADS) {
      const int r = e / NET_TILE, kk = e % NET_TILE, gk = k0 + kk;
      if (gk >= K) continue;
      T s = T(0);
      for (int c = 0; c < CN; ++c) s += cluster.map_shared_rank(red, c)[r * NET_TILE + kk];
      const T h = Hs[r * NET_TILE + kk];
      a.gzprev[scene * a.gzp_ss + (size_t)r * K + gk] = s * (T(1) - h * h);
    }
    cluster.sync();
  }
}

// Per-scene whitening (network.py:88-104), network input rows x0 = [Re|Im]/s
// and output gains 8 s / sqrt(4 M0) (network.py:107-120).
template <typename T>
struct NetSetupArgs {
  int n, M0, joint, H;
  const C<T>* alpha0;   // [S][n][M0]
  T* x0;                // [S][rows][D0]
  T* cout;              // [S][D0]
};

template <typename T>
__global__ void net_setup_kernel(NetSetupArgs<T> a) {
  const int scene = blockIdx.x, tid = threadIdx.x;
  const int n = a.n, M0 = a.M0;
  const C<T>* al = a.alpha0 + (size_t)scene * n * M0;
  __shared__ double red[32];
  __shared__ double gl_s;
  // global mean |alpha|^2 (fixed order)
  double loc = 0.0;
  for (int i = tid; i < n * M0; i += blockDim.x) loc += (double)cabs2<T>(al[i]);
  loc = warp_sum<double>(loc);
  if ((tid & 31) == 0) red[tid >> 5] = loc;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    gl_s = sqrt(s / (double)(n * M0));
  }
  __syncthreads();
  const double glob = gl_s;
  const int D0 = 2 * M0 * (a.joint ? n : 1);
  const int rows = a.joint ? 1 : n;
  T* x0 = a.x0 + (size_t)scene * rows * D0;
  T* co = a.cout + (size_t)scene * D0;
  const double gain = OUTPUT_GAIN / sqrt((double)a.H);
  for (int m = tid; m < M0; m += blockDim.x) {
    double sc = 1.0;
    if (glob != 0.0) {
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc += (double)cabs2<T>(al[(size_t)i * M0 + m]);
      const double mode = sqrt(acc / n);
      sc = pow(mode, 0.7) * pow(glob, 1.0 - 0.7);
      const double fl = 0.1 * glob;
      sc = sc > fl ? sc : fl;
    }
    for (int i = 0; i < n; ++i) {
      const C<T> z = al[(size_t)i * M0 + m];
      const int row = a.joint ? 0 : i;
      const int fre = a.joint ? i * M0 + m : m;
      x0[(size_t)row * D0 + fre] = (T)(z.x / sc);
      x0[(size_t)row * D0 + fre + D0 / 2] = (T)(z.y / sc);
      if (!a.joint && i > 0) continue;
      co[fre] = (T)(gain * sc);
      co[fre + D0 / 2] = (T)(gain * sc);
    }
  }
}

// Standalone Adam over flat vectors (network.py:248-264), for the
// reference-shaped adam_step API; the training loop uses the fused path.
template <typename T>
__global__ void adam_flat_kernel(T* p, T* m, T* v, const T* g, long long count, T lr, T b1, T b2, T eps,
                                 T bc1, T bc2, int* err) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int bits = 0;
  for (; i < count; i += (long long)gridDim.x * blockDim.x) {
    T pp = p[i], mm = m[i], vv = v[i];
    const T gg = g[i];
    adam_one<T>(pp, mm, vv, gg, lr, b1, b2, eps, bc1, bc2);
    if (!isfinite(pp)) bits |= ERR_NONFINITE_PARAM;
    p[i] = pp; m[i] = mm; v[i] = vv;
  }
  if (bits) atomicOr(err, bits);
}

}  // namespace pdf
