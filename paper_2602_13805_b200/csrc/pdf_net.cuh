// The per-scene corrective network (network.py:53-223) and its Adam update
// (network.py:230-264), batched over scenes.
//
// Parameters live in one flat buffer per scene in the reference order
// w1, b1, w2, b2, w3, b3 with weights row-major (fan_out, fan_in), so
// grad_loss / adam_step see the same flat vector the reference does.
//
// The layers are skinny (rows = incidences, 1..80) and wide (hundreds to
// thousands of columns).  Both kernels stream every weight exactly once,
// need no inter-CTA communication, and reduce in a fixed order:
//
// Forward  z = h W^T + b: a warp owns OPW output rows and its lanes split K
//   (lane-contiguous 16-byte weight loads); the input rows arrive in
//   double-buffered shared tiles (cp.async) and are reused by all OPW rows;
//   the 32 lane partials are folded with a fixed shuffle tree.
// Backward: a CTA owns 8 input columns k; its 256 threads are 8 columns x
//   32 row subsets.  Each thread keeps h[:, k] and a partial g_h[:, k] and
//   walks its rows n four at a time: W, m, v come straight from memory
//   (64-byte row segments per warp), g_W[n,k] = sum_r g_z[r,n] h[r,k] and
//   g_h[:,k] += g_z[:,n] W_old[n,k] use the same broadcast g_z values, Adam
//   writes W, m, v back -- the weight gradient never round-trips through
//   memory.  The 32 row-subset partials of g_h are summed in shared memory
//   in a fixed order and multiplied by tanh'(h) to give the next g_z.
#pragma once
#include "pdf_common.cuh"

namespace pdf {

constexpr double OUTPUT_GAIN = 8.0;   // network.py:85
constexpr int NET_THREADS = 256;
template <typename T> struct Epc { static constexpr int v = 16 / sizeof(T); };   // elements per 16 B

template <typename T>
struct NetFwdArgs {
  int rows, K, N, ks;                 // ks: K range per cluster rank (multiple of the chunk)
  const T* in; long long in_ss;       // [S][rows][K]
  const T* theta; long long th_ss;    // [S][Np]
  long long w_off, b_off;
  T* out; long long out_ss;           // [S][rows][N]   (tanh layers)
  int final_layer;                    // 0 tanh(z + b); 1 final: alpha_hat = alpha0 + merge((z + b) * cout);
                                      // 2 z + b; 3 z (float64 DMMA kernels; tensor-parallel slices)
  // final layer: alpha_hat = alpha0 + merge(y * cout)
  const T* cout;                      // [S][N]
  const C<T>* alpha0;                 // [S][n][M0]
  C<T>* alpha_hat;                    // [S][n][M0]
  int n, M0, joint;
  int* step;                          // incremented once (train mode) or null
  int w_early;                        // weights final two launches back: prefetch before pdl_wait
  int tl;                             // timeline slot + 1 (0: off)
};

template <typename T, int RB> struct FwdShape {
  static constexpr int KCH = RB <= 2 ? 256 : 128;    // K per staged input chunk
  static constexpr int P = KCH + Epc<T>::v;           // padded pitch
  static constexpr int VL = KCH / 32;                 // elements per lane per chunk
};

template <typename T, int RB>
__host__ __device__ constexpr size_t fwd_smem_elems(int opw) {
  return (size_t)2 * 16 * RB * FwdShape<T, RB>::P + (size_t)(NET_THREADS / 32) * opw * 16 * RB;
}

// The K range is split across the CK CTAs of a cluster (CK = 1 when the
// batch alone fills the GPU): a single scene then keeps ~4 CTAs per SM in
// flight, which is what hot-L2 streaming needs (bytes in flight, not
// launches, bound these skinny layers).  Partial row sums meet in DSMEM and
// are added in rank order (deterministic).
template <typename T, int RB, int OPW>
__global__ void __launch_bounds__(NET_THREADS, RB <= 2 ? 2 : 1) net_fwd_kernel(NetFwdArgs<T> a) {
  using Sh = FwdShape<T, RB>;
  constexpr int RP = 16 * RB, KCH = Sh::KCH, P = Sh::P, VL = Sh::VL, EPC = Epc<T>::v;
  constexpr int SEG = KCH / EPC;
  constexpr int NWP = NET_THREADS / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Xs = reinterpret_cast<T*>(smem_raw);            // 2 x [RP][P]
  T* part = Xs + 2 * RP * P;                         // [NWP*OPW][RP] partial sums for the cluster
  cg::cluster_group cluster = cg::this_cluster();
  const int CK = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int scene = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = a.K, N = a.N, rows = a.rows;
  const int nbase = (blockIdx.x * NWP + warp) * OPW;
  const int kb = rank * a.ks, ke = min(K, kb + a.ks);
  // (step counter is bumped after pdl_wait: the previous backward kernels read it)
  const T* __restrict__ W = a.theta + scene * a.th_ss + a.w_off;
  const T* __restrict__ X = a.in + scene * a.in_ss;

  auto stage = [&](int k0, int s) {
    T* dst = Xs + s * RP * P;
    for (int i = tid; i < RP * SEG; i += NET_THREADS) {
      const int r = i / SEG, sg = i % SEG, gk = k0 + sg * EPC;
      const bool ok = r < rows && gk < ke;
      cp_async16(dst + r * P + sg * EPC, ok ? X + (size_t)r * K + gk : X, ok);
    }
    cp_async_commit();
  };
  // this warp's weights for a chunk: lane covers k0 + lane + 32 j (coalesced
  // global rows, conflict-free shared reads)
  auto load_w = [&](int k0, T (&w)[OPW][VL]) {
#pragma unroll
    for (int o = 0; o < OPW; ++o) {
      const int n = nbase + o;
#pragma unroll
      for (int j = 0; j < VL; ++j) {
        const int kk = k0 + lane + 32 * j;
        w[o][j] = (n < N && kk < ke) ? W[(size_t)n * K + kk] : T(0);
      }
    }
  };

  T acc[OPW][RP];
#pragma unroll
  for (int o = 0; o < OPW; ++o)
#pragma unroll
    for (int r = 0; r < RP; ++r) acc[o][r] = T(0);

  constexpr bool PF = OPW == 1;      // register prefetch of the next chunk (keeps 2 CTAs/SM otherwise)
  T w[OPW][VL], wn[PF ? OPW : 1][PF ? VL : 1];
  if (a.w_early && kb < ke) load_w(kb, w);
  pdl_wait();
  if (!a.w_early && kb < ke) load_w(kb, w);
  if (a.step && tid == 0 && blockIdx.x == 0 && rank == 0 && scene == 0) atomicAdd(a.step, 1);
  if (kb < ke) stage(kb, 0);
  int s = 0;
  for (int k0 = kb; k0 < ke; k0 += KCH, s ^= 1) {
    if constexpr (PF) { if (k0 + KCH < ke) load_w(k0 + KCH, wn); }
    if (k0 + KCH < ke) {
      stage(k0 + KCH, s ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const T* xs = Xs + s * RP * P + lane;
#pragma unroll
    for (int r = 0; r < RP; ++r) {
      T xv[VL];
#pragma unroll
      for (int j = 0; j < VL; ++j) xv[j] = xs[r * P + 32 * j];
#pragma unroll
      for (int o = 0; o < OPW; ++o) {
        T t = T(0);
#pragma unroll
        for (int j = 0; j < VL; ++j) t += xv[j] * w[o][j];
        acc[o][r] += t;
      }
    }
    if constexpr (PF) {
#pragma unroll
      for (int o = 0; o < OPW; ++o)
#pragma unroll
        for (int j = 0; j < VL; ++j) w[o][j] = wn[o][j];
    } else {
      if (k0 + KCH < ke) load_w(k0 + KCH, w);
    }
    __syncthreads();   // buffer s is restaged two chunks later
  }
  pdl_trigger();
  // fixed-order lane reduction; every lane ends with all row sums
#pragma unroll
  for (int o = 0; o < OPW; ++o)
#pragma unroll
    for (int r = 0; r < RP; ++r) acc[o][r] = warp_sum<T>(acc[o][r]);
  // lane r publishes row r (and r+32, r+64) of this warp's outputs
#pragma unroll
  for (int o = 0; o < OPW; ++o)
#pragma unroll
    for (int r = 0; r < RP; ++r)
      if ((r & 31) == lane) part[(warp * OPW + o) * RP + r] = acc[o][r];
  cluster.sync();

  // reduce over the cluster ranks (fixed order) and apply the epilogue
  const T* bias = a.theta + scene * a.th_ss + a.b_off;
  const int total = NWP * OPW * RP;
  for (int e = rank * NET_THREADS + tid; e < total; e += CK * NET_THREADS) {
    const int wo = e / RP, r = e % RP;
    const int gn = blockIdx.x * NWP * OPW + wo;
    if (gn >= N || r >= rows) continue;
    T z = T(0);
    for (int c = 0; c < CK; ++c) z += cluster.map_shared_rank(part, c)[e];
    z += bias[gn];
    if (!a.final_layer) {
      a.out[scene * a.out_ss + (size_t)r * N + gn] = tanh(z);
    } else {
      const T yv = z * a.cout[(size_t)scene * N + gn];
      // [Re | Im] feature layout (network.py:123-136)
      const int half = N / 2;
      const int f = gn < half ? gn : gn - half;
      int view, m;
      if (a.joint) { view = f / a.M0; m = f % a.M0; } else { view = r; m = f; }
      const size_t off = ((size_t)scene * a.n + view) * a.M0 + m;
      T* dst = reinterpret_cast<T*>(a.alpha_hat + off);
      const T* src = reinterpret_cast<const T*>(a.alpha0 + off);
      if (gn < half) dst[0] = src[0] + yv; else dst[1] = src[1] + yv;
    }
  }
  cluster.sync();
}

template <typename T>
struct NetBwdArgs {
  int rows, K, N, ns;                 // ns: rows of W per cluster rank (multiple of 128)
  const T* gz; long long gz_ss;       // [S][rows][N]   gradient at this layer's pre-activation
  const T* hin; long long hin_ss;     // [S][rows][K]   this layer's input
  T* theta; long long th_ss;          // [S][Np] (updated in place when fused)
  long long w_off, b_off;
  T* m; T* v;                         // Adam moments, same layout as theta
  T* grad;                            // [S][Np] gradient out (unfused mode) or null
  const int* step;                    // Adam t (device)
  T lr, b1, b2, eps;
  T* gzprev; long long gzp_ss;        // [S][rows][K] or null (first layer)
  int* err;                           // [S]
  int tl;                             // timeline slot + 1 (0: off)
  int* snap;                          // split backward: *snap = *step (Adam t of this iteration) or null
  // peer scatter (incidence sharding, unfused mode): g_W / g_b entry at flat index f goes to
  // rank o = f / peer_shard, slot [peer_me][f - o peer_shard] of that rank's receive buffer
  // peers[o] (a peer-mapped address on the multi-GPU box): the reduce-scatter of the gradient
  // happens in the epilogue of the kernel that computes it
  double* const* peers;
  int peer_me;
  long long peer_shard;
};

// destination of flat parameter index f in the peer-scatter layout
__device__ __forceinline__ double* peer_slot(double* const* peers, int me, long long shard, long long f) {
  const long long o = f / shard;
  return peers[o] + (size_t)me * shard + (f - o * shard);
}

// Adam in the reference's operation order (network.py:252-257).  The bias
// corrections are applied as products with 1/(1-b^t) and the remaining
// division and square root use hardware approximations refined by Newton
// steps: agreement with the IEEE sequence to ~1 ulp, at a fraction of the
// instruction count of the library routines (whose slow paths dominated).
__device__ __forceinline__ double rcp_nr(double y) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
  double e = fma(-y, r, 1.0);   // the approximation is good to ~2^-23: two steps reach 2^-92
  r = fma(r, e, r);
  e = fma(-y, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double div_nr(double x, double y) {
  const double r = rcp_nr(y);
  const double q = x * r;
  return fma(r, fma(-y, q, x), q);
}
__device__ __forceinline__ double sqrt_nr(double v) {
  if (!(v > 0.0)) return v == 0.0 ? 0.0 : sqrt(v);   // 0, negative, NaN: exact IEEE semantics
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v));
  const double hv = 0.5 * v;
  r = r * fma(-hv * r, r, 1.5);
  r = r * fma(-hv * r, r, 1.5);
  const double s = v * r;
  return fma(0.5 * r, fma(-s, s, v), s);
}
__device__ __forceinline__ float div_nr(float x, float y) { return x / y; }
__device__ __forceinline__ float sqrt_nr(float v) { return sqrtf(v); }

template <typename T>
__device__ __forceinline__ void adam_one(T& p, T& m, T& v, T g, T lr, T b1, T b2, T eps, T ibc1, T ibc2) {
  m = b1 * m + (T(1) - b1) * g;
  v = b2 * v + (T(1) - b2) * g * g;
  const T mh = m * ibc1;
  const T vh = v * ibc2;
  p = p - div_nr(lr * mh, sqrt_nr(vh) + eps);
}

// Thread layout of the backward kernel by row count (RP = 16*RB rows):
//   RB <= 2 : 8 columns x 32 row subsets, h and the g_h partial in registers
//   RB == 3 : same, h[:, k] shared per column in shared memory
//   RB >= 4 : 128 threads = 16 columns x 8 subsets, g_h partial in shared memory
template <typename T, int RB> struct BwdShape {
  static constexpr int THR = RB >= 4 ? 128 : 256;
  static constexpr int COLS = RB >= 4 ? 16 : 8;        // input columns per CTA
  static constexpr int SUB = THR / COLS;                // row subsets per CTA
  static constexpr int UR = RB >= 4 ? 2 : 4;            // rows per thread per step (ILP)
  static constexpr int NCH = SUB * UR;                  // rows of g_z staged per step
  static constexpr bool HR = RB <= 2;                   // h in registers
  static constexpr bool GR = RB <= 3;                   // g_h partial in registers
  static constexpr int GP = NCH + Epc<T>::v;            // padded pitch of the staged g_z rows
};
constexpr int BWD_NCH_MAX = 128;

template <typename T, int RB>
__host__ __device__ constexpr size_t bwd_smem_elems() {
  using Sh = BwdShape<T, RB>;
  constexpr int RP = 16 * RB;
  return (size_t)2 * RP * Sh::GP + (size_t)Sh::SUB * 16 * Sh::COLS + (size_t)RP * Sh::COLS +
         (Sh::HR ? 0 : (size_t)RP * Sh::COLS) + (Sh::GR ? 0 : (size_t)RP * Sh::THR);
}

template <typename T, int RB, bool FUSED>
__global__ void __launch_bounds__(BwdShape<T, RB>::THR, RB == 1 ? 2 : 1) net_bwd_kernel(NetBwdArgs<T> a) {
  using Sh = BwdShape<T, RB>;
  constexpr int RP = 16 * RB, EPC = Epc<T>::v, GP = Sh::GP;
  constexpr int THR = Sh::THR, COLS = Sh::COLS, SUB = Sh::SUB, UR = Sh::UR, NCH = Sh::NCH;
  constexpr bool HR = Sh::HR, GR = Sh::GR;
  constexpr int SEG = NCH / EPC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Gs = reinterpret_cast<T*>(smem_raw);            // 2 x [RP][GP]   g_z[r][n0 + i]
  T* red = Gs + 2 * RP * GP;                         // [SUB][16][COLS] reduction scratch
  T* cpart = red + SUB * 16 * COLS;                  // [RP][COLS] CTA partial of g_h
  T* Hs = cpart + RP * COLS;                         // [RP][COLS] h when !HR
  T* GHs = Hs + (HR ? 0 : RP * COLS);                // [RP][THR]  g_h partial when !GR
  __shared__ T bc_s[2];
  cg::cluster_group cluster = cg::this_cluster();
  const int CN = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int scene = blockIdx.z;
  const int tid = threadIdx.x;
  const int col = tid % COLS, sub = tid / COLS;
  const int k = blockIdx.x * COLS + col;
  const int K = a.K, N = a.N, rows = a.rows;
  const bool kok = k < K;
  // this cluster rank's rows of W (CN = 1 when the batch alone fills the GPU)
  const int nb = min(N, rank * a.ns), ne = min(N, nb + a.ns);

  const T* __restrict__ hin = a.hin + scene * a.hin_ss;
  const T* __restrict__ gz = a.gz + scene * a.gz_ss;
  T* __restrict__ W = a.theta + scene * a.th_ss + a.w_off;
  T* __restrict__ mW = FUSED ? a.m + scene * a.th_ss + a.w_off : nullptr;
  T* __restrict__ vW = FUSED ? a.v + scene * a.th_ss + a.w_off : nullptr;
  T* __restrict__ gW = FUSED ? nullptr : a.grad + scene * a.th_ss + a.w_off;

  auto stage = [&](int n0, int s) {
    T* dst = Gs + s * RP * GP;
    for (int i = tid; i < RP * SEG; i += THR) {
      const int r = i / SEG, sg = i % SEG, gn = n0 + sg * EPC;
      const bool ok = r < rows && gn < ne;
      cp_async16(dst + r * GP + sg * EPC, ok ? gz + (size_t)r * N + gn : gz, ok);
    }
    cp_async_commit();
  };

  if (tid == 0) {
    if (FUSED) {
      const int t = *a.step;
      bc_s[0] = T(1.0 / (1.0 - pow((double)a.b1, (double)t)));
      bc_s[1] = T(1.0 / (1.0 - pow((double)a.b2, (double)t)));
    } else {
      bc_s[0] = bc_s[1] = T(1);
    }
  }
  T h[HR ? RP : 1], gh[GR ? RP : 1];
#pragma unroll(GR ? RP : 4)
  for (int r = 0; r < RP; ++r) {
    const T hv = (kok && r < rows) ? hin[(size_t)r * K + k] : T(0);
    if constexpr (HR) h[r] = hv; else if (sub == 0) Hs[r * COLS + col] = hv;
    if constexpr (GR) gh[r] = T(0); else GHs[r * THR + tid] = T(0);
  }
  if constexpr (!HR) __syncthreads();
  // this thread's rows of a step: n0 + sub + SUB*u.  W, m, v of the first
  // step are final since the previous iteration, so they are loaded before
  // pdl_wait; later steps are prefetched one step ahead (register double
  // buffer where the register budget allows it).
  constexpr bool DB = !GR;
  auto load_step = [&](int n0, T (&w_)[UR], T (&m_)[UR], T (&v_)[UR]) {
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const int n = n0 + sub + SUB * u;
      const bool ok = kok && n < ne;
      const size_t o = (size_t)n * K + k;
      w_[u] = ok ? W[o] : T(0);
      if constexpr (FUSED) {
        m_[u] = ok ? mW[o] : T(0);
        v_[u] = ok ? vW[o] : T(0);
      }
    }
  };
  int errbits = 0;
  int s = 0;
  T wv[UR], mv[UR], vv[UR];
  if (nb < ne) load_step(nb, wv, mv, vv);
  pdl_wait();
  if (nb < ne) stage(nb, 0);
  for (int n0 = nb; n0 < ne; n0 += NCH, s ^= 1) {
    T wn[DB ? UR : 1], mn[DB ? UR : 1], vn[DB ? UR : 1];
    if constexpr (DB) {
      if (n0 + NCH < ne) load_step(n0 + NCH, wn, mn, vn);
    }
    if (n0 + NCH < ne) {
      stage(n0 + NCH, s ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const T* G = Gs + s * RP * GP;
    const T ibc1 = bc_s[0], ibc2 = bc_s[1];
    T gw[UR];
#pragma unroll
    for (int u = 0; u < UR; ++u) gw[u] = T(0);
#pragma unroll(GR ? RP : 4)
    for (int r = 0; r < RP; ++r) {
      T hr;
      if constexpr (HR) hr = h[r]; else hr = Hs[r * COLS + col];
      T ghs = T(0);
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const T g = G[r * GP + sub + SUB * u];
        gw[u] += g * hr;
        ghs += g * wv[u];
      }
      if constexpr (GR) gh[r] += ghs; else GHs[r * THR + tid] += ghs;
    }
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const int n = n0 + sub + SUB * u;
      if (!kok || n >= ne) continue;
      const size_t o = (size_t)n * K + k;
      if (!isfinite(gw[u])) errbits |= ERR_NONFINITE_GRAD;
      if constexpr (FUSED) {
        T p = wv[u], mm = mv[u], vq = vv[u];
        adam_one<T>(p, mm, vq, gw[u], a.lr, a.b1, a.b2, a.eps, ibc1, ibc2);
        if (!isfinite(p)) errbits |= ERR_NONFINITE_PARAM;
        W[o] = p; mW[o] = mm; vW[o] = vq;
      } else {
        gW[o] = gw[u];
      }
    }
    // bias (network.py:213,217): gb[n] = sum_r g_z[r, n], owned by the first column tile
    if (blockIdx.x == 0 && tid < NCH && n0 + tid < ne) {
      T gb = T(0);
      for (int r = 0; r < rows; ++r) gb += G[r * GP + tid];
      const int gn = n0 + tid;
      if (!isfinite(gb)) errbits |= ERR_NONFINITE_GRAD;
      if constexpr (FUSED) {
        T* th = a.theta + scene * a.th_ss + a.b_off;
        T* mb = a.m + scene * a.th_ss + a.b_off;
        T* vb = a.v + scene * a.th_ss + a.b_off;
        T p = th[gn], mm = mb[gn], vq = vb[gn];
        adam_one<T>(p, mm, vq, gb, a.lr, a.b1, a.b2, a.eps, ibc1, ibc2);
        if (!isfinite(p)) errbits |= ERR_NONFINITE_PARAM;
        th[gn] = p; mb[gn] = mm; vb[gn] = vq;
      } else {
        a.grad[scene * a.th_ss + a.b_off + gn] = gb;
      }
    }
    if constexpr (DB) {
#pragma unroll
      for (int u = 0; u < UR; ++u) { wv[u] = wn[u]; mv[u] = mn[u]; vv[u] = vn[u]; }
    } else {
      if (n0 + NCH < ne) load_step(n0 + NCH, wv, mv, vv);
    }
    __syncthreads();   // buffer s is restaged two steps later
  }
  pdl_trigger();
  if (errbits) atomicOr(&a.err[scene], errbits);

  if (a.gzprev) {
    // g_h[r][k]: sum over the 32 row subsets (fixed order) into cpart, then over
    // the cluster ranks (fixed order) through DSMEM
#pragma unroll
    for (int rb = 0; rb < RP; rb += 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int r = rb + j;
        T v_;
        if constexpr (GR) {
          v_ = T(0);
#pragma unroll
          for (int q = 0; q < RP; ++q) if (q == r) v_ = gh[q];
        } else {
          v_ = GHs[r * THR + tid];
        }
        red[(sub * 16 + j) * COLS + col] = v_;
      }
      __syncthreads();
      for (int e = tid; e < 16 * COLS; e += THR) {   // 16 * COLS exceeds THR when RB >= 4
        const int j = e / COLS, c = e % COLS;
        T sum = T(0);
        for (int q = 0; q < SUB; ++q) sum += red[(q * 16 + j) * COLS + c];
        cpart[(rb + j) * COLS + c] = sum;
      }
      __syncthreads();
    }
    cluster.sync();
    for (int e = rank * THR + tid; e < rows * COLS; e += CN * THR) {
      const int r = e / COLS, c = e % COLS, gk = blockIdx.x * COLS + c;
      if (gk >= K) continue;
      T sum = T(0);
      for (int q = 0; q < CN; ++q) sum += cluster.map_shared_rank(cpart, q)[e];
      const T hv = hin[(size_t)r * K + gk];
      a.gzprev[scene * a.gzp_ss + (size_t)r * K + gk] = sum * (T(1) - hv * hv);
    }
    cluster.sync();
  }
}

// Per-scene whitening (network.py:88-104), network input rows x0 = [Re|Im]/s
// and output gains 8 s / sqrt(4 M0) (network.py:107-120).
template <typename T>
struct NetSetupArgs {
  int n, M0, joint, H;
  int n_all, off;       // alpha0 holds n_all views; this context's rows are views [off, off+n)
  const C<T>* alpha0;   // [S][n_all][M0]
  T* x0;                // [S][rows][D0]
  T* cout;              // [S][D0]
};

template <typename T>
__global__ void net_setup_kernel(NetSetupArgs<T> a) {
  const int scene = blockIdx.x, tid = threadIdx.x;
  const int n = a.n, M0 = a.M0, na = a.n_all;
  const C<T>* al = a.alpha0 + (size_t)scene * na * M0;
  __shared__ double red[32];
  __shared__ double gl_s;
  // global mean |alpha|^2 (fixed order)
  double loc = 0.0;
  for (int i = tid; i < na * M0; i += blockDim.x) loc += (double)cabs2<T>(al[i]);
  loc = warp_sum<double>(loc);
  if ((tid & 31) == 0) red[tid >> 5] = loc;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    gl_s = sqrt(s / (double)(na * M0));
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
      for (int i = 0; i < na; ++i) acc += (double)cabs2<T>(al[(size_t)i * M0 + m]);
      const double mode = sqrt(acc / na);
      sc = pow(mode, 0.7) * pow(glob, 1.0 - 0.7);
      const double fl = 0.1 * glob;
      sc = sc > fl ? sc : fl;
    }
    for (int i = 0; i < n; ++i) {
      const C<T> z = al[(size_t)(a.off + i) * M0 + m];
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

// same update with the step t read from device memory (capturable in a CUDA graph);
// bias corrections as in the fused kernels (pow in float64)
template <typename T>
__global__ void adam_flat_dev_kernel(T* p, T* m, T* v, const T* g, long long count, T lr, T b1, T b2, T eps,
                                     const int* t_dev, int* err) {
  const double t = (double)*t_dev;
  const T bc1 = T(1.0 / (1.0 - pow((double)b1, t))), bc2 = T(1.0 / (1.0 - pow((double)b2, t)));
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int bits = 0;
  for (; i < count; i += (long long)gridDim.x * blockDim.x) {
    T pp = p[i], mm = m[i], vv = v[i];
    const T gg = g[i];
    if (!isfinite(gg)) bits |= ERR_NONFINITE_GRAD;
    adam_one<T>(pp, mm, vv, gg, lr, b1, b2, eps, bc1, bc2);
    if (!isfinite(pp)) bits |= ERR_NONFINITE_PARAM;
    p[i] = pp; m[i] = mm; v[i] = vv;
  }
  if (bits) atomicOr(err, bits);
}

// owner side of the peer-scattered gradient (incidence sharding): for this rank's
// shard [me shard, (me + 1) shard) of the flat parameters, g = sum over source
// ranks r of recv[r][i] (rank order), one Adam step (step t from device
// memory), and the updated parameter written to every rank's theta (peer
// stores: the all-gather of the parameters)
__global__ void adam_gather_kernel(const double* __restrict__ recv, double* const* thetas, double* __restrict__ m,
                                   double* __restrict__ v, int world, int me, long long shard, long long np,
                                   double lr, double b1, double b2, double eps, const int* t_dev, int* err) {
  const double t = (double)*t_dev;
  const double bc1 = 1.0 / (1.0 - pow(b1, t)), bc2 = 1.0 / (1.0 - pow(b2, t));
  const long long base = (long long)me * shard;
  const double* own = thetas[me];
  int bits = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < shard; i += (long long)gridDim.x * blockDim.x) {
    const long long f = base + i;
    if (f >= np) break;
    double g = 0.0;
    for (int r = 0; r < world; ++r) g += recv[(size_t)r * shard + i];
    if (!isfinite(g)) bits |= ERR_NONFINITE_GRAD;
    double p = own[f], mm = m[i], vv = v[i];
    adam_one<double>(p, mm, vv, g, lr, b1, b2, eps, bc1, bc2);
    if (!isfinite(p)) bits |= ERR_NONFINITE_PARAM;
    m[i] = mm;
    v[i] = vv;
    for (int r = 0; r < world; ++r) thetas[r][f] = p;
  }
  __threadfence_system();
  if (bits) atomicOr(err, bits);
}

}  // namespace pdf
