// Per-incidence ("view") kernels: the zero-padded P x P FFT convolution that
// applies the domain Green's operator G_D, fused with what sits either side
// of it on the PDF hot path.
//
//   VIEW_FWD  : alpha -> J = expand(alpha) (spectral.py:68-79)
//               E = E_inc + G_D J          (forward.py:140-146, losses.py:220)
//               D = J G_S^T - d = alpha H^T - d (masked), ||D||^2, g_rows
//               (losses.py:229-232,285-287; H = G_S o expand, pdf_aux.cuh)
//               ||E_i||^2 partials for eps_reg (cie.py:42-50)
//   VIEW_BWD  : g_J = g_J_local + G_D^H g_E   (forward.py:149-151, losses.py:303)
//               g_alpha = truncate(g_J)/(m1 m2) (spectral.py:56-65, losses.py:306)
//                         + g_rows conj(H)      (the G_S^H g_rows part of g_J)
//               optionally scattered straight into the network's output
//               gradient rows (network.py:575-582)
//   VIEW_APPLY: y = G_D x or G_D^H x on dense images (init path, tests)
//
// One thread-block CLUSTER per view.  Rank c of CS owns spatial rows
// [c*M/CS, (c+1)*M/CS) and spectral columns [c*P/CS, (c+1)*P/CS).  The
// two 2-D transposes of the row-column FFT go through distributed shared
// memory, so the padded P x P spectrum never touches HBM:
//   A: row FFTs of my (nonzero) rows      -> DSMEM scatter by column owner
//   B: per column  FFT, x K^, inverse FFT -> DSMEM scatter by row owner
//   C: inverse row FFTs of my rows, crop to M columns
#pragma once
#include "pdf_aux.cuh"
#include "pdf_common.cuh"
#include "pdf_dmma.cuh"
#include "pdf_pixel.cuh"

namespace pdf {

enum { VIEW_FWD = 0, VIEW_BWD = 1, VIEW_APPLY = 2 };

template <typename T>
struct ViewArgs {
  int M, mf, R, n, CS;
  const C<T>* khat;   // permuted / 1/P^2-scaled kernel spectrum, [P(col pos)][P(row pos)]
  const C<T>* twP;    // exp(-2 pi i k / P), k < P
  const C<T>* twM;    // exp(-2 pi i k / M), k < M
  // FWD
  const C<T>* alpha;  // [S*n][M0]
  const C<T>* einc;   // [S or 1][n][M][M]
  long long einc_scene_stride;   // elements; 0 = shared across scenes
  const C<T>* hs;     // [R][M0] spectral receiver operator (pdf_aux.cuh)
  const C<T>* data;   // [S][n][R]
  const T* mask;      // [S][n][R] or null
  const double* c_sca;  // [S]
  C<T>* J;            // [S*n][M][M]
  C<T>* E;            // [S*n][M][M]
  double* norms;      // [S*n][CS]
  C<T>* grows;        // [S*n][R]
  double* dloss;      // [S*n]
  int do_data;        // 0: the data term runs as a separate GEMM over the scene's views (data_mma_kernel)
  // BWD
  const C<T>* gE;     // [S*n][M][M]
  const C<T>* gJloc;  // [S*n][M][M]
  C<T>* galpha;       // [S*n][M0] or null
  const C<T>* gad;    // [S*n][M0] data part of g_alpha (slot order, gad_kernel) or null: computed here
  T* gy;              // [S][rows][D0] or null
  const T* cout;      // [S][D0] output gain per feature
  int joint;
  // BWD: the scene's loss breakdown is finalised by (view 0, rank 0)
  FinalizeArgs fin;
  int do_fin;
  // APPLY
  const C<T>* x;
  C<T>* y;
  int conj_in, conj_out;
  int tl;             // timeline slot + 1 (0: off)
};

constexpr int VIEW_MAX_THREADS = 256;
constexpr int VIEW_SOLO_THREADS = 512;   // CS = 1: one 16-warp CTA per view

template <typename T>
struct ViewSmem {
  C<T>* tw;     // P
  C<T>* twm;    // M
  C<T>* bufA;   // M * (P/CS + 1)   (rows padded by one element: conflict-free column reads)
  C<T>* bufB;   // (M/CS) * (P + 1)
  C<T>* rows;   // (M/CS) * M
  C<T>* small;  // M0 + (M/CS)*K : A (spectral grid) then V / U
  C<T>* khs;    // (P/CS) * P : my K^ columns (constant: prefetched before the dependency wait)
  C<T>* pre;    // (M/CS) * M : FWD: my E_inc rows (constant, prefetched); BWD: my g_J local rows
  C<T>* dsum;   // 32 * nw + M0/CS + 1 : BWD data-adjoint scratch and per-output sums
  // followed by xch: max(CS*R, M0) partial-sum exchange (read remotely)
};

template <typename T>
__host__ __device__ inline size_t view_smem_bytes(int M, int mf, int R, int CS) {
  const int P = 2 * M, K = 2 * mf, M0 = K * K;
  const int rp = M / CS;
  size_t a = (size_t)M0 + (size_t)rp * K;
  // exchange: data-term partials (CS R) or the pushed truncation partials (CS ceil(M0 / CS))
  const size_t xr = (size_t)CS * R, xt = (size_t)CS * ((M0 + CS - 1) / CS);
  size_t xch = xr > xt ? xr : xt;
  // 8-CTA clusters (latency regime, one CTA per SM) also stage the constant
  // K^ columns and the E_inc / g_J-local rows; 4-CTA clusters (batches) keep
  // two CTAs per SM and read them from L2 in place
  const size_t stage = CS == 8 ? (size_t)(P / CS) * P + (size_t)rp * M : 0;
  size_t pre = stage + (size_t)32 * (VIEW_SOLO_THREADS / 32) + (size_t)M0 / CS + 1;
  // CS = 1 (one CTA per view, batches): both transpose buffers and the row buffer
  // are the same M x (P + 1) array (every stage works in place, row or column wise)
  const size_t bufs = CS == 1 ? (size_t)M * (P + 1) : (size_t)M * (P / CS + 1) + (size_t)rp * (P + 1) + (size_t)rp * M;
  size_t n = (size_t)P + M + bufs + a + pre + xch;
  return n * sizeof(C<T>) + 64 * sizeof(double);
}

template <typename T>
__device__ inline int corner_freq(int u, int mf, int M) { return u < mf ? u : M - 2 * mf + u; }
// index in the reference coefficient vector of spectral grid entry (u, v)
__device__ inline int corner_slot(int u, int v, int mf) {
  return (((u / mf) * 2 + (v / mf)) * mf + (u % mf)) * mf + (v % mf);
}

template <typename T>
__device__ inline double block_sum_d(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum<double>(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += red[i];   // fixed order
  return s;
}

template <typename T, int E, int MODE, int CSZ>
__global__ void __launch_bounds__(CSZ == 1 ? VIEW_SOLO_THREADS : VIEW_MAX_THREADS) view_kernel(ViewArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int P = 32 * E;
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int CS = CSZ;   // cluster size: compile-time so the row / column owner maps are shifts
  const int rank = (int)cluster.block_rank();
  constexpr int M = P / 2;
  const int mf = a.mf, K = 2 * mf, M0 = K * K;
  constexpr int rp = M / CS, cp = P / CS;
  const int y0 = rank * rp;
  const int v = blockIdx.y;                 // global view index (scene*n + view)
  const int scene = v / a.n, view = v % a.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  // element n = lane + 32k of a length-P line is inside the unpadded M = P/2
  // window iff k < E/2 (E >= 2) or, for P = 32, lane < 16
  constexpr int KH = E >= 2 ? E / 2 : 1;
  const bool lane_ok = (E >= 2) || (lane < 16);

  ViewSmem<T> s;
  C<T>* p = reinterpret_cast<C<T>*>(smem_raw);
  s.tw = p; p += P;
  s.twm = p; p += M;
  const int cpp = cp + 1, Pp = P + 1;       // padded pitches of the transpose buffers
  // CS = 1: bufA = bufB = rows, one M x (P + 1) array (cpp == Pp): a warp reads a
  // whole row / column into registers before it writes the transformed one back
  constexpr bool SOLO = CS == 1;
  constexpr int RP = SOLO ? P + 1 : M;      // pitch of the row buffer
  s.bufA = p; p += (size_t)M * cpp;
  s.bufB = SOLO ? s.bufA : p; p += SOLO ? 0 : (size_t)rp * Pp;
  s.rows = SOLO ? s.bufA : p; p += SOLO ? 0 : (size_t)rp * M;
  s.small = p; p += (size_t)M0 + (size_t)rp * K;
  constexpr bool PRE = CS == 8;   // staged constants (view_smem_bytes)
  s.khs = p; p += PRE ? (size_t)cp * P : 0;
  s.pre = p; p += PRE ? (size_t)rp * M : 0;
  s.dsum = p; p += (size_t)32 * (VIEW_SOLO_THREADS / 32) + M0 / CS + 1;
  const int opr = (M0 + CS - 1) / CS;   // truncation outputs owned per rank
  C<T>* xch = p; p += ((size_t)CS * a.R > (size_t)CS * opr ? (size_t)CS * a.R : (size_t)CS * opr);
  double* red = reinterpret_cast<double*>(p);

  for (int i = tid; i < P; i += blockDim.x) s.tw[i] = a.twP[i];
  for (int i = tid; i < M; i += blockDim.x) s.twm[i] = a.twM[i];
  __syncthreads();
  LaneTw<T, E> ltw;
  ltw.load(s.tw, lane);
  // constants: my K^ columns (and E_inc rows) stream in while the previous
  // kernel drains
  tl_mark(a.tl, 0);
  const size_t img = (size_t)M * M;
  constexpr int EPC = 16 / sizeof(C<T>) > 0 ? 16 / sizeof(C<T>) : 1;
  if constexpr (PRE && MODE != VIEW_APPLY) {
    const C<T>* src = a.khat + (size_t)rank * cp * P;
    for (int i = tid; i < cp * P / EPC; i += blockDim.x) cp_async16(s.khs + i * EPC, src + i * EPC, true);
  }
  if constexpr (PRE && MODE == VIEW_FWD) {
    const C<T>* src = a.einc + (size_t)scene * a.einc_scene_stride + (size_t)view * img + (size_t)y0 * M;
    for (int i = tid; i < rp * M / EPC; i += blockDim.x) cp_async16(s.pre + i * EPC, src + i * EPC, true);
  }
  cp_async_commit();
  pdl_wait();   // everything below reads the previous kernel's outputs
  tl_mark(a.tl, 1);

  // ---------------- stage 0: my input rows -> s.rows ----------------------
  if constexpr (MODE == VIEW_FWD) {
    const C<T>* al = a.alpha + (size_t)v * M0;
    for (int i = tid; i < M0; i += blockDim.x) {
      const int u = i / K, w = i % K;
      s.small[i] = al[corner_slot(u, w, mf)];      // A[u][w]
    }
    __syncthreads();
    // V[yl][w] = sum_u A[u][w] exp(+2 pi i kr_u y / M)  -> stored after A
    // J[yl][x] = sum_w V[yl][w] exp(+2 pi i kc_w x / M) / (m1 m2)
    C<T>* V = s.small + M0;
    const T inv = T(1) / (T(M) * T(M));
    C<T>* Jg = a.J + (size_t)v * img + (size_t)y0 * M;
    if constexpr (sizeof(T) == 8) {
      // the two contractions as complex GEMMs on the FP64 tensor cores
      const C<T>* A_ = s.small;
      const C<T>* tw_ = s.twm;
      cgemm_dmma(rp, K, K,
                 [&](int yl, int u) { return conj_<T>(tw_[(corner_freq<T>(u, mf, M) * (y0 + yl)) & (M - 1)]); },
                 [&](int u, int w) { return A_[u * K + w]; },
                 [&](int yl, int w, C<T> val) { V[yl * K + w] = val; });
      __syncthreads();
      cgemm_dmma(rp, M, K, [&](int yl, int w) { return V[yl * K + w]; },
                 [&](int w, int x) { return conj_<T>(tw_[(corner_freq<T>(w, mf, M) * x) & (M - 1)]); },
                 [&](int yl, int x, C<T> val) {
                   val = cscale<T>(val, inv);
                   s.rows[yl * RP + x] = val;
                   Jg[yl * M + x] = val;
                 });
    } else {
      for (int i = tid; i < rp * K; i += blockDim.x) {
        const int yl = i / K, w = i % K, y = y0 + yl;
        C<T> acc = czero<T>();
        for (int u = 0; u < K; ++u) {
          const int f = corner_freq<T>(u, mf, M);
          acc = cadd<T>(acc, cmulc<T>(s.small[u * K + w], s.twm[(f * y) & (M - 1)]));
        }
        V[i] = acc;
      }
      __syncthreads();
      for (int i = tid; i < rp * M; i += blockDim.x) {
        const int yl = i / M, x = i % M;
        C<T> acc = czero<T>();
        for (int w = 0; w < K; ++w) {
          const int f = corner_freq<T>(w, mf, M);
          acc = cadd<T>(acc, cmulc<T>(V[yl * K + w], s.twm[(f * x) & (M - 1)]));
        }
        acc = cscale<T>(acc, inv);
        s.rows[yl * RP + x] = acc;
        Jg[i] = acc;
      }
    }
    __syncthreads();
  } else if constexpr (MODE == VIEW_BWD) {
    // my g_E rows (conjugated) now; my g_J local rows stream in for stage C
    if constexpr (PRE) {
      const C<T>* gl = a.gJloc + (size_t)v * img + (size_t)y0 * M;
      for (int i = tid; i < rp * M / EPC; i += blockDim.x) cp_async16(s.pre + i * EPC, gl + i * EPC, true);
      cp_async_commit();
    }
    const C<T>* g = a.gE + (size_t)v * img + (size_t)y0 * M;
    for (int i = tid; i < rp * M; i += blockDim.x) s.rows[(i / M) * RP + (i % M)] = conj_<T>(g[i]);
    __syncthreads();
  } else {
    const C<T>* g = a.x + (size_t)v * img + (size_t)y0 * M;
    for (int i = tid; i < rp * M; i += blockDim.x) {
      C<T> t = g[i];
      s.rows[(i / M) * RP + (i % M)] = a.conj_in ? conj_<T>(t) : t;
    }
    __syncthreads();
  }

  tl_stage(a.tl, 0);
  // ---------------- stage A: row FFTs, scatter to column owners ------------
  for (int yl = warp; yl < rp; yl += nw) {
    C<T> x[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int col = lane + 32 * k;
      x[k] = (k < KH && lane_ok) ? s.rows[yl * RP + col] : czero<T>();
    }
    warp_fft_fwd<T, E>(x, ltw, lane);
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const int pos = q * 32 + lane;
      const int dst = pos / cp, lc = pos - dst * cp;
      C<T>* rb = cluster.map_shared_rank(s.bufA, dst);
      rb[(size_t)(y0 + yl) * cpp + lc] = x[q];
    }
  }

  // Split cluster barrier: the arrive releases my stage-A scatter; the data
  // term (receivers rank, rank + CS, ...; H rows from L2) then runs while the
  // other CTAs finish theirs, and the wait acquires everyone's scatter.
  tl_stage(a.tl, 1);
  if constexpr (!SOLO) asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  if (MODE == VIEW_BWD && !a.gad) {
    // G_S^H g_rows through H (pdf_aux.cuh) for my outputs i = rank + CS*o,
    // while the other CTAs finish their stage-A scatter; warp w sums
    // receivers w, w + nw, ...
    const C<T>* grow = a.grows + (size_t)v * a.R;
    const int nout = (M0 - rank + CS - 1) / CS;
    C<T>* scr = s.dsum + M0 / CS + 1;   // [nw][32]
    for (int ob = 0; ob < nout; ob += 32) {
      const int o = ob + lane, i = rank + CS * o;
      if (o < nout) scr[warp * 32 + lane] = data_adjoint_at<T>(grow, a.hs, a.R, M0, corner_slot(i / K, i % K, mf), warp, nw);
      __syncthreads();
      if (warp == 0 && o < nout) {
        C<T> d = czero<T>();
        for (int w = 0; w < nw; ++w) d = cadd<T>(d, scr[w * 32 + lane]);
        s.dsum[o] = d;
      }
      __syncthreads();
    }
  }
  if (MODE == VIEW_FWD && a.do_data) {
    // D[r] = sum_m alpha[m] H[r][m] - d[r] (masked), g_rows = 2 D mask / c_sca
    const C<T>* al = a.alpha + (size_t)v * M0;
    const double csca = a.c_sca[scene];
    double dl = 0.0;
    for (int r = rank + CS * warp; r < a.R; r += CS * nw) {
      const C<T>* h = a.hs + (size_t)r * M0;
      C<T> acc = czero<T>(), acc1 = czero<T>();
      int i = lane;
      for (; i + 32 < M0; i += 64) {
        acc = cadd<T>(acc, cmul<T>(al[i], h[i]));
        acc1 = cadd<T>(acc1, cmul<T>(al[i + 32], h[i + 32]));
      }
      if (i < M0) acc = cadd<T>(acc, cmul<T>(al[i], h[i]));
      acc = cadd<T>(acc, acc1);
      acc.x = warp_sum<T>(acc.x);
      acc.y = warp_sum<T>(acc.y);
      if (lane == 0) {
        const size_t di = (size_t)v * a.R + r;
        C<T> d = csub<T>(acc, a.data[di]);
        const T mk_ = a.mask ? a.mask[di] : T(1);
        d = cscale<T>(d, mk_);
        dl += (double)cabs2<T>(d);
        a.grows[di] = cscale<T>(d, T(2.0 / csca) * mk_);
      }
    }
    if (lane == 0) red[16 + warp] = dl;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < nw; ++w) t += red[16 + w];
      cluster.map_shared_rank(red, 0)[40 + rank] = t;   // published by the cluster.sync after stage B
    }
  }
  cp_async_wait<0>();   // K^ columns, E_inc / g_J local rows (own copies: a CTA barrier follows)
  __syncthreads();
  if constexpr (!SOLO) asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");

  tl_stage(a.tl, 2);
  // ---------------- stage B: columns: FFT, x K^, inverse FFT ---------------
  for (int cc = warp; cc < cp; cc += nw) {
    const int posc = rank * cp + cc;
    C<T> x[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int row = lane + 32 * k;
      x[k] = (k < KH && lane_ok) ? s.bufA[(size_t)row * cpp + cc] : czero<T>();
    }
    warp_fft_fwd<T, E>(x, ltw, lane);
    if constexpr (PRE && MODE != VIEW_APPLY) {
      const C<T>* kh = s.khs + (size_t)cc * P;
#pragma unroll
      for (int q = 0; q < E; ++q) x[q] = cmul<T>(x[q], kh[q * 32 + lane]);
    } else {
      const C<T>* kh = a.khat + (size_t)posc * P;
#pragma unroll
      for (int q = 0; q < E; ++q) x[q] = cmul<T>(x[q], kh[q * 32 + lane]);
    }
    warp_fft_inv<T, E>(x, ltw, lane);
#pragma unroll
    for (int k = 0; k < KH; ++k) {
      if (!lane_ok) break;
      const int y = lane + 32 * k;
      const int dst = y / rp, yl = y - dst * rp;
      C<T>* rb = cluster.map_shared_rank(s.bufB, dst);
      rb[(size_t)yl * Pp + posc] = x[k];
    }
  }
  tl_stage(a.tl, 3);
  if constexpr (SOLO) __syncthreads(); else cluster.sync();   // also publishes the data partials (written before this arrive) to rank 0

  if (MODE == VIEW_FWD && a.do_data && rank == 0 && tid == 0) {
    double t = 0.0;
    for (int c = 0; c < CS; ++c) t += red[40 + c];
    a.dloss[v] = t;
  }

  tl_stage(a.tl, 4);
  // ---------------- stage C: inverse row FFTs, crop ------------------------
  double nrm = 0.0;
  for (int yl = warp; yl < rp; yl += nw) {
    C<T> x[E];
#pragma unroll
    for (int q = 0; q < E; ++q) x[q] = s.bufB[(size_t)yl * Pp + q * 32 + lane];
    warp_fft_inv<T, E>(x, ltw, lane);
    const size_t rowoff = (size_t)v * img + (size_t)(y0 + yl) * M;
#pragma unroll
    for (int k = 0; k < KH; ++k) {
      if (!lane_ok) break;
      const int col = lane + 32 * k;
      if constexpr (MODE == VIEW_FWD) {
        const C<T> ei = PRE ? s.pre[yl * M + col]
                            : a.einc[(size_t)scene * a.einc_scene_stride + (size_t)view * img + (size_t)(y0 + yl) * M + col];
        C<T> e = cadd<T>(ei, x[k]);
        a.E[rowoff + col] = e;
        nrm += (double)cabs2<T>(e);
      } else if constexpr (MODE == VIEW_BWD) {
        const C<T> gl = PRE ? s.pre[yl * M + col] : a.gJloc[rowoff + col];
        s.rows[yl * RP + col] = cadd<T>(gl, conj_<T>(x[k]));
      } else {
        a.y[rowoff + col] = a.conj_out ? conj_<T>(x[k]) : x[k];
      }
    }
  }

  tl_stage(a.tl, 5);
  pdl_trigger();
  if constexpr (MODE == VIEW_FWD) {
    double tot = block_sum_d<T>(nrm, red);
    if (tid == 0) a.norms[(size_t)v * CS + rank] = tot;
  }

  if constexpr (MODE == VIEW_BWD) {
    __syncthreads();
    if (a.do_fin && view == 0 && rank == 0) {
      finalize_block(a.fin, scene, reinterpret_cast<double(*)[4]>(red));
      __syncthreads();
    }
    // U[yl][w] = sum_x gJ[yl][x] exp(-2 pi i kc_w x / M)
    // my partial G[u][w] = sum_yl exp(-2 pi i kr_u y / M) U[yl][w], pushed
    // straight into the owner's exchange slot [my rank][i / CS] (owner i % CS):
    // one cluster barrier, and every CTA then reads only its own shared memory
    C<T>* U = s.small + M0;
    auto push = [&](int i, C<T> val) {
      cluster.map_shared_rank(xch, i % CS)[rank * opr + i / CS] = val;
    };
    if constexpr (sizeof(T) == 8) {
      const C<T>* tw_ = s.twm;
      const C<T>* rw = s.rows;
      cgemm_dmma(rp, K, M, [&](int yl, int x) { return rw[yl * RP + x]; },
                 [&](int x, int w) { return tw_[(corner_freq<T>(w, mf, M) * x) & (M - 1)]; },
                 [&](int yl, int w, C<T> val) { U[yl * K + w] = val; });
      __syncthreads();
      cgemm_dmma(K, K, rp, [&](int u, int yl) { return tw_[(corner_freq<T>(u, mf, M) * (y0 + yl)) & (M - 1)]; },
                 [&](int yl, int w) { return U[yl * K + w]; },
                 [&](int u, int w, C<T> val) { push(u * K + w, val); });
    } else {
      for (int i = tid; i < rp * K; i += blockDim.x) {
        const int yl = i / K, w = i % K;
        const int f = corner_freq<T>(w, mf, M);
        C<T> acc = czero<T>();
        C<T> acc1 = czero<T>(), acc2 = czero<T>(), acc3 = czero<T>();
        for (int x = 0; x < M; x += 4) {   // M is a multiple of 4: four independent chains
          acc = cadd<T>(acc, cmul<T>(s.rows[yl * RP + x], s.twm[(f * x) & (M - 1)]));
          acc1 = cadd<T>(acc1, cmul<T>(s.rows[yl * RP + x + 1], s.twm[(f * (x + 1)) & (M - 1)]));
          acc2 = cadd<T>(acc2, cmul<T>(s.rows[yl * RP + x + 2], s.twm[(f * (x + 2)) & (M - 1)]));
          acc3 = cadd<T>(acc3, cmul<T>(s.rows[yl * RP + x + 3], s.twm[(f * (x + 3)) & (M - 1)]));
        }
        acc = cadd<T>(cadd<T>(acc, acc1), cadd<T>(acc2, acc3));
        U[i] = acc;
      }
      __syncthreads();
      for (int i = tid; i < M0; i += blockDim.x) {
        const int u = i / K, w = i % K;
        const int f = corner_freq<T>(u, mf, M);
        C<T> acc = czero<T>();
        for (int yl = 0; yl < rp; ++yl) acc = cadd<T>(acc, cmul<T>(U[yl * K + w], s.twm[(f * (y0 + yl)) & (M - 1)]));
        push(i, acc);
      }
    }
    tl_stage(a.tl, 6);
    if constexpr (SOLO) __syncthreads(); else cluster.sync();
    tl_stage(a.tl, 7);
    const T inv = T(1) / (T(M) * T(M));
    for (int i = rank + CS * tid; i < M0; i += CS * blockDim.x) {
      C<T> acc = czero<T>();
      for (int c = 0; c < CS; ++c) acc = cadd<T>(acc, xch[c * opr + i / CS]);   // rank order
      acc = cscale<T>(acc, inv);
      const int u = i / K, w = i % K;
      const int slot = corner_slot(u, w, mf);
      acc = cadd<T>(acc, a.gad ? a.gad[(size_t)v * M0 + slot] : s.dsum[(i - rank) / CS]);
      if (a.galpha) a.galpha[(size_t)v * M0 + slot] = acc;
      if (a.gy) {
        const int D0 = 2 * M0 * (a.joint ? a.n : 1);
        const int rows = a.joint ? 1 : a.n;
        const int re = a.joint ? view * M0 + slot : slot;
        const int row = a.joint ? 0 : view;
        T* gyrow = a.gy + ((size_t)scene * rows + row) * D0;
        const T* co = a.cout + (size_t)scene * D0;
        gyrow[re] = acc.x * co[re];
        gyrow[re + D0 / 2] = acc.y * co[re + D0 / 2];
      }
    }
  }
  tl_mark(a.tl, 2);
}

}  // namespace pdf
