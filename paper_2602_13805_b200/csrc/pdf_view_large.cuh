// Large-grid view path (BASELINE config 5: M = 256, P = 512).
//
// A float64 P x P spectrum (4 MiB at P = 512) does not fit one cluster's
// shared memory, so the zero-padded convolution of forward.py:140-146 runs
// as three passes over a column-major spectrum buffer spec[view][P][M] that
// stays L2-resident for a chunk of views:
//
//   rows pass : the M nonzero rows of the padded input (expand(alpha) in the
//               forward, conj(g_E) in the adjoint), warp FFT each, write the
//               permuted spectrum positions as columns (transposed through
//               shared memory in 128-byte row segments)
//   cols pass : per spectrum column: FFT of the M nonzero entries, x K^,
//               inverse FFT, keep the first M entries -- in place
//   out pass  : gather 8 rows, inverse row FFTs, crop to M columns, and the
//               epilogue (E = E_inc + G_D J and ||E||^2 partials; or
//               g_J = g_J_local + G_D^H g_E and the truncation partials)
//
// The data term D = J G_S^T - d (losses.py:229-232) is a tall complex GEMM
// (views x pixels) x (pixels x receivers) here: data_mma_kernel (float64,
// DMMA) or data_gemm_kernel (float32, register-tiled 4x4 outputs) split the
// pixels over CTAs, and a fixed-order reduce finishes D.
// The warp FFT, the K^ permutation and every reduction order are the ones the
// cluster path uses (pdf_view.cuh), so both paths are interchangeable; the
// cluster path is kept for M <= 128 where its DSMEM transposes win.
#pragma once
#include "pdf_common.cuh"
#include "pdf_dmma.cuh"
#include "pdf_pixel.cuh"
#include "pdf_view.cuh"

namespace pdf {

constexpr int VL_ROWS = 8;   // rows per CTA in the rows / out passes (one per warp)

template <typename T>
struct VLArgs {
  int M, mf, R, n, NPV;       // NPV = M / VL_ROWS partials per view
  int v0;                      // first global view (scene * n + view) of this chunk
  int nview;                   // views in this chunk (cols pass: two views per CTA)
  const C<T>* khat;            // permuted, 1/P^2-scaled kernel spectrum [P col pos][P row pos]
  const C<T>* twP;
  const C<T>* twM;
  C<T>* spec;                  // [chunk views][P][M]
  // rows pass
  const C<T>* alpha;           // FWD  [S*n][M0]
  C<T>* J;                     // FWD  [S*n][M][M]
  const C<T>* gE;              // BWD
  const C<T>* x;               // APPLY
  int conj_in, conj_out;
  // out pass
  const C<T>* einc;
  long long einc_scene_stride;
  C<T>* E;
  double* norms;               // [S*n][NPV]
  const C<T>* gJloc;
  C<T>* gpart;                 // [S*n][NPV][M0] truncation partials
  C<T>* y;                     // APPLY
  // truncation reduce
  C<T>* galpha;
  T* gy;
  const T* cout;
  int joint;
  const C<T>* grows;           // [S*n][R] data-residual gradient rows
  const C<T>* hs;              // [R][M0] spectral receiver operator (pdf_aux.cuh)
  const C<T>* gad;             // [S*n][M0] data part of g_alpha (slot order, gad_kernel) or null: computed here
  FinalizeArgs fin;
  int do_fin;
  int tl;                      // timeline slot + 1 (0: off)
};

template <typename T>
__device__ __forceinline__ int vl_corner_freq(int u, int mf, int M) { return u < mf ? u : M - 2 * mf + u; }
__device__ __forceinline__ int vl_corner_slot(int u, int v, int mf) {
  return (((u / mf) * 2 + (v / mf)) * mf + (u % mf)) * mf + (v % mf);
}

template <typename T>
__host__ __device__ inline size_t vl_rows_smem(int E, int mf) {
  const int P = 32 * E, M = P / 2, K = 2 * mf;
  return ((size_t)P + P / 2 + M + (size_t)P * (VL_ROWS + 1) + (size_t)K * K + (size_t)VL_ROWS * K) * sizeof(C<T>);
}

// cols pass: the warps' kernel-spectrum columns (float64 split path)
template <typename T>
__host__ __device__ inline size_t vl_cols_smem(int E) {
  return sizeof(T) == 8 && E >= 4 ? (size_t)8 * (32 * E + 16 * E) * sizeof(C<T>) : 0;   // K^ columns + the second view's inputs
}

template <typename T>
__host__ __device__ inline size_t vl_out_smem(int E, int mf) {
  const int P = 32 * E, M = P / 2, K = 2 * mf;
  (void)M;
  return ((size_t)P + P / 2 + M + (size_t)VL_ROWS * (P + 1) + (size_t)VL_ROWS * K) * sizeof(C<T>) + 16 * sizeof(double);
}

// ---------------------------------------------------------------------------
template <typename T, int E, int MODE>
__global__ void __launch_bounds__(256) vl_rows_kernel(VLArgs<T> a) {
  tl_mark(a.tl, 0);
  TlExit tl_exit_{a.tl};
  constexpr int P = 32 * E, M = P / 2, KH = E / 2, TP = VL_ROWS + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int mf = a.mf, K = 2 * mf, M0 = K * K;
  constexpr bool SPLIT = E >= 4;
  constexpr int EH = E / 2;
  C<T>* tw = reinterpret_cast<C<T>*>(smem_raw);
  C<T>* twh = tw + P;                   // exp(-2 pi i k / (P/2)), the half-length FFT table
  C<T>* twm = twh + P / 2;
  C<T>* tile = twm + M;                 // [P][TP]
  C<T>* A = tile + P * TP;              // [K][K]
  C<T>* V = A + M0;                     // [VL_ROWS][K]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int vr = blockIdx.y, v = a.v0 + vr, y0 = blockIdx.x * VL_ROWS, y = y0 + warp;
  const size_t img = (size_t)M * M;
  for (int i = tid; i < P; i += blockDim.x) tw[i] = a.twP[i];
  for (int i = tid; i < P / 2; i += blockDim.x) twh[i] = a.twP[2 * i];
  for (int i = tid; i < M; i += blockDim.x) twm[i] = a.twM[i];
  __syncthreads();
  LaneTw<T, E> ltw;
  LaneTw<T, (SPLIT ? E / 2 : 1)> ltwh;
  if constexpr (SPLIT) ltwh.load(twh, lane); else ltw.load(tw, lane);
  pdl_wait();
  tl_mark(a.tl, 1);

  C<T> x[E];
#pragma unroll
  for (int k = 0; k < E; ++k) x[k] = czero<T>();
  bool even_done = false;   // FWD split path: the even half of the padded spectrum is written with the expansion
  if constexpr (MODE == VIEW_FWD && sizeof(T) == 8 && SPLIT) {
    // J = expand(alpha) rows y0..y0+7 (spectral.py:68-79).  V = Tr A (the
    // contraction over the row frequencies) is a small complex GEMM on the
    // FP64 tensor cores; the contraction over the column frequencies is an
    // inverse length-M FFT of the K nonzero coefficients, placed at the
    // slots the warp FFT's permuted order assigns to their frequencies.
    // Those same coefficients, times M, ARE the even half of the padded
    // row's spectrum (F_M of the row), so only the odd half needs a forward
    // transform below.
    const C<T>* al = a.alpha + (size_t)v * M0;
    for (int i = tid; i < M0; i += blockDim.x) A[i] = al[vl_corner_slot(i / K, i % K, mf)];
    __syncthreads();
    cgemm_dmma(VL_ROWS, K, K,
               [&](int yl, int u) { return conj_<T>(twm[(vl_corner_freq<T>(u, mf, M) * (y0 + yl)) & (M - 1)]); },
               [&](int u, int w) { return A[u * K + w]; }, [&](int yl, int w, C<T> val) { V[yl * K + w] = val; });
    __syncthreads();
    const T inv = T(1) / (T(M) * T(M));
    C<T> t[EH];
#pragma unroll
    for (int q = 0; q < EH; ++q) {
      const int f = spectrum_slot_freq(lane, q, EH);
      const int w = f < mf ? f : (f >= M - mf ? f - (M - 2 * mf) : -1);
      t[q] = w >= 0 ? cscale<T>(V[warp * K + w], inv) : czero<T>();
      tile[(q * 32 + lane) * TP + warp] = cscale<T>(t[q], T(M));
    }
    warp_fft_inv<T, EH>(t, ltwh, lane);
    C<T>* jrow = a.J + (size_t)v * img + (size_t)y * M;
#pragma unroll
    for (int k = 0; k < EH; ++k) {
      x[k] = t[k];
      jrow[lane + 32 * k] = t[k];
    }
    even_done = true;
  } else if constexpr (MODE == VIEW_FWD && sizeof(T) == 8) {
    // J = expand(alpha) rows y0..y0+7 (spectral.py:68-79): V = Tr A, J = V T as
    // complex GEMMs on the FP64 tensor cores, J staged through `tile`
    const C<T>* al = a.alpha + (size_t)v * M0;
    for (int i = tid; i < M0; i += blockDim.x) A[i] = al[vl_corner_slot(i / K, i % K, mf)];
    __syncthreads();
    cgemm_dmma(VL_ROWS, K, K,
               [&](int yl, int u) { return conj_<T>(twm[(vl_corner_freq<T>(u, mf, M) * (y0 + yl)) & (M - 1)]); },
               [&](int u, int w) { return A[u * K + w]; }, [&](int yl, int w, C<T> val) { V[yl * K + w] = val; });
    __syncthreads();
    const T inv = T(1) / (T(M) * T(M));
    C<T>* jrows = tile;   // [VL_ROWS][M] (tile is free until after the FFT)
    cgemm_dmma(VL_ROWS, M, K, [&](int yl, int w) { return V[yl * K + w]; },
               [&](int w, int x) { return conj_<T>(twm[(vl_corner_freq<T>(w, mf, M) * x) & (M - 1)]); },
               [&](int yl, int x, C<T> val) { jrows[yl * M + x] = cscale<T>(val, inv); });
    __syncthreads();
    C<T>* jrow = a.J + (size_t)v * img + (size_t)y * M;
#pragma unroll
    for (int k = 0; k < KH; ++k) {
      const int col = lane + 32 * k;
      x[k] = jrows[warp * M + col];
      jrow[col] = x[k];
    }
    __syncthreads();   // tile is rewritten by the transposed spectrum below
  } else if constexpr (MODE == VIEW_FWD) {
    // J = expand(alpha) rows y0..y0+7 (spectral.py:68-79), separable direct sums
    const C<T>* al = a.alpha + (size_t)v * M0;
    for (int i = tid; i < M0; i += blockDim.x) A[i] = al[vl_corner_slot(i / K, i % K, mf)];
    __syncthreads();
    for (int i = tid; i < VL_ROWS * K; i += blockDim.x) {
      const int yl = i / K, w = i % K, yy = y0 + yl;
      C<T> acc = czero<T>();
      for (int u = 0; u < K; ++u)
        acc = cadd<T>(acc, cmulc<T>(A[u * K + w], twm[(vl_corner_freq<T>(u, mf, M) * yy) & (M - 1)]));
      V[i] = acc;
    }
    __syncthreads();
    const T inv = T(1) / (T(M) * T(M));
    C<T>* jrow = a.J + (size_t)v * img + (size_t)y * M;
#pragma unroll
    for (int k = 0; k < KH; ++k) {
      const int col = lane + 32 * k;
      C<T> acc = czero<T>(), acc1 = czero<T>();
      for (int w = 0; w < K; w += 2) {
        acc = cadd<T>(acc, cmulc<T>(V[warp * K + w], twm[(vl_corner_freq<T>(w, mf, M) * col) & (M - 1)]));
        acc1 = cadd<T>(acc1, cmulc<T>(V[warp * K + w + 1], twm[(vl_corner_freq<T>(w + 1, mf, M) * col) & (M - 1)]));
      }
      acc = cscale<T>(cadd<T>(acc, acc1), inv);
      x[k] = acc;
      jrow[col] = acc;
    }
  } else if constexpr (MODE == VIEW_BWD) {
    const C<T>* g = a.gE + (size_t)v * img + (size_t)y * M;
#pragma unroll
    for (int k = 0; k < KH; ++k) x[k] = conj_<T>(g[lane + 32 * k]);
  } else {
    const C<T>* g = a.x + (size_t)v * img + (size_t)y * M;
#pragma unroll
    for (int k = 0; k < KH; ++k) {
      const C<T> t = g[lane + 32 * k];
      x[k] = a.conj_in ? conj_<T>(t) : t;
    }
  }
  if constexpr (SPLIT) {
    // zero padding: X[2m] = F_{P/2}(x)[m], X[2m+1] = F_{P/2}(x w^n)[m], w = exp(-2 pi i / P)
    C<T> t[EH];
    if (!even_done) {
#pragma unroll
      for (int k = 0; k < EH; ++k) t[k] = x[k];
      warp_fft_fwd<T, EH>(t, ltwh, lane);
#pragma unroll
      for (int q = 0; q < EH; ++q) tile[(q * 32 + lane) * TP + warp] = t[q];
    }
#pragma unroll
    for (int k = 0; k < EH; ++k) t[k] = cmul<T>(x[k], tw[lane + 32 * k]);
    warp_fft_fwd<T, EH>(t, ltwh, lane);
#pragma unroll
    for (int q = 0; q < EH; ++q) tile[(P / 2 + q * 32 + lane) * TP + warp] = t[q];
  } else {
    warp_fft_fwd<T, E>(x, ltw, lane);
#pragma unroll
    for (int q = 0; q < E; ++q) tile[(q * 32 + lane) * TP + warp] = x[q];
  }
  __syncthreads();
  pdl_trigger();
  C<T>* out = a.spec + (size_t)vr * P * M + y0;
  for (int i = tid; i < P * VL_ROWS; i += blockDim.x) {
    const int pos = i / VL_ROWS, yl = i % VL_ROWS;
    out[(size_t)pos * M + yl] = tile[pos * TP + yl];
  }
}

// ---------------------------------------------------------------------------
template <typename T, int E>
__global__ void __launch_bounds__(256, (E >= 4 ? 2 : 1)) vl_cols_kernel(VLArgs<T> a) {
  tl_mark(a.tl, 0);
  TlExit tl_exit_{a.tl};
  constexpr int P = 32 * E, M = P / 2, KH = E / 2;
  constexpr bool SPLIT = E >= 4;
  constexpr int EH = E / 2;
  __shared__ C<T> tw[P];
  __shared__ C<T> twh[P / 2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < P; i += blockDim.x) tw[i] = a.twP[i];
  for (int i = tid; i < P / 2; i += blockDim.x) twh[i] = a.twP[2 * i];
  __syncthreads();
  const int pos = blockIdx.x * (blockDim.x >> 5) + warp;
  const C<T>* kh = a.khat + (size_t)pos * P;
  if constexpr (SPLIT) {
    // y[n] = F^-1(K_e F(x))[n] + w^-n F^-1(K_o F(x w^n))[n] for the first P/2 outputs
    LaneTw<T, E / 2> lt;
    lt.load(twh, lane);
    if constexpr (sizeof(T) == 8) {
      // the column's kernel spectrum (constant) streams into shared memory while
      // the previous pass drains; lane l copies exactly the entries it reads
      extern __shared__ __align__(16) unsigned char smem_raw[];
      C<T>* khs = reinterpret_cast<C<T>*>(smem_raw) + (size_t)warp * P;
#pragma unroll
      for (int q = 0; q < E; ++q) cp_async16(khs + q * 32 + lane, kh + q * 32 + lane, true);
      cp_async_commit();
      kh = khs;
    }
    pdl_wait();
  tl_mark(a.tl, 1);
    // float64: two views per CTA (the same kernel-spectrum columns serve both);
    // the second view's column streams into shared memory while the first is
    // transformed, and the first's stores drain behind the second's transforms
    constexpr int NV = sizeof(T) == 8 ? 2 : 1;
    const int v0 = blockIdx.y * NV;
    C<T>* xs = nullptr;
    if constexpr (NV == 2) {
      extern __shared__ __align__(16) unsigned char smem_raw2[];
      xs = reinterpret_cast<C<T>*>(smem_raw2) + (size_t)8 * P + (size_t)warp * M;
      if (v0 + 1 < a.nview) {
        const C<T>* c1 = a.spec + ((size_t)(v0 + 1) * P + pos) * M;
#pragma unroll
        for (int k = 0; k < EH; ++k) cp_async16(xs + lane + 32 * k, c1 + lane + 32 * k, true);
      }
      cp_async_commit();
    }
#pragma unroll 1
    for (int vi = 0; vi < NV; ++vi) {
      if (v0 + vi >= a.nview) break;
      C<T>* col = a.spec + ((size_t)(v0 + vi) * P + pos) * M;
      C<T> xin[EH], r[EH], t[EH];
      if (vi == 0) {
#pragma unroll
        for (int k = 0; k < EH; ++k) xin[k] = col[lane + 32 * k];
      } else {
        cp_async_wait<0>();   // (lane l reads the entries it copied)
#pragma unroll
        for (int k = 0; k < EH; ++k) xin[k] = xs[lane + 32 * k];
      }
#pragma unroll
      for (int k = 0; k < EH; ++k) t[k] = xin[k];
      warp_fft_fwd<T, EH>(t, lt, lane);
      if constexpr (sizeof(T) == 8) {
        if (vi == 0) cp_async_wait<1>();   // the kernel-spectrum column (older group)
      }
#pragma unroll
      for (int q = 0; q < EH; ++q) t[q] = cmul<T>(t[q], kh[q * 32 + lane]);
      warp_fft_inv<T, EH>(t, lt, lane);
#pragma unroll
      for (int k = 0; k < EH; ++k) r[k] = t[k];
#pragma unroll
      for (int k = 0; k < EH; ++k) t[k] = cmul<T>(xin[k], tw[lane + 32 * k]);
      warp_fft_fwd<T, EH>(t, lt, lane);
#pragma unroll
      for (int q = 0; q < EH; ++q) t[q] = cmul<T>(t[q], kh[P / 2 + q * 32 + lane]);
      warp_fft_inv<T, EH>(t, lt, lane);
      if (vi == NV - 1 || v0 + vi + 1 >= a.nview) pdl_trigger();
#pragma unroll
      for (int k = 0; k < EH; ++k) col[lane + 32 * k] = cadd<T>(r[k], cmulc<T>(t[k], tw[lane + 32 * k]));
    }
    return;
  }
  LaneTw<T, E> ltw;
  ltw.load(tw, lane);
  pdl_wait();
  tl_mark(a.tl, 1);
  C<T>* col = a.spec + ((size_t)blockIdx.y * P + pos) * M;
  C<T> x[E];
#pragma unroll
  for (int k = 0; k < E; ++k) x[k] = k < KH ? col[lane + 32 * k] : czero<T>();
  warp_fft_fwd<T, E>(x, ltw, lane);
#pragma unroll
  for (int q = 0; q < E; ++q) x[q] = cmul<T>(x[q], kh[q * 32 + lane]);
  warp_fft_inv<T, E>(x, ltw, lane);
  pdl_trigger();
#pragma unroll
  for (int k = 0; k < KH; ++k) col[lane + 32 * k] = x[k];
}

// ---------------------------------------------------------------------------
template <typename T, int E, int MODE>
__global__ void __launch_bounds__(256, 2) vl_out_kernel(VLArgs<T> a) {
  tl_mark(a.tl, 0);
  TlExit tl_exit_{a.tl};
  constexpr int P = 32 * E, M = P / 2, KH = E / 2, SP = P + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int mf = a.mf, K = 2 * mf, M0 = K * K;
  constexpr bool SPLIT = E >= 4;
  constexpr int EH = E / 2;
  C<T>* tw = reinterpret_cast<C<T>*>(smem_raw);
  C<T>* twh = tw + P;
  C<T>* twm = twh + P / 2;
  C<T>* S = twm + M;                     // [VL_ROWS][SP]; reused as rows [VL_ROWS][M] (BWD)
  C<T>* U = S + VL_ROWS * SP;            // [VL_ROWS][K]
  double* red = reinterpret_cast<double*>(U + VL_ROWS * K);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int vr = blockIdx.y, v = a.v0 + vr, y0 = blockIdx.x * VL_ROWS, y = y0 + warp;
  const int scene = v / a.n, view = v % a.n;
  const size_t img = (size_t)M * M;
  for (int i = tid; i < P; i += blockDim.x) tw[i] = a.twP[i];
  for (int i = tid; i < P / 2; i += blockDim.x) twh[i] = a.twP[2 * i];
  for (int i = tid; i < M; i += blockDim.x) twm[i] = a.twM[i];
  // forward: the epilogue's second operand (E_inc, constant) is requested before the
  // dependency wait (the adjoint's g_J local rows are read at their use: registers)
  const size_t rowoff = (size_t)v * img + (size_t)y * M;
  C<T> epi[KH];
  if constexpr (MODE == VIEW_FWD) {
    const C<T>* ei = a.einc + (size_t)scene * a.einc_scene_stride + (size_t)view * img + (size_t)y * M;
#pragma unroll
    for (int k = 0; k < KH; ++k) epi[k] = ei[lane + 32 * k];
  }
  pdl_wait();
  tl_mark(a.tl, 1);
  const C<T>* in = a.spec + (size_t)vr * P * M + y0;
  if constexpr (sizeof(C<T>) == 16) {
    // 8 consecutive rows of one spectrum position = 128 bytes: all pieces in flight at once
    for (int i = tid; i < P * VL_ROWS; i += blockDim.x) {
      const int pos = i / VL_ROWS, yl = i % VL_ROWS;
      cp_async16(S + yl * SP + pos, in + (size_t)pos * M + yl, true);
    }
    cp_async_commit();
    cp_async_wait<0>();
  } else {
    for (int i = tid; i < P * VL_ROWS; i += blockDim.x) {
      const int pos = i / VL_ROWS, yl = i % VL_ROWS;
      S[yl * SP + pos] = in[(size_t)pos * M + yl];
    }
  }
  __syncthreads();
  C<T> x[E];
  LaneTw<T, (SPLIT ? E / 2 : 1)> lt;
  if constexpr (SPLIT) {
    lt.load(twh, lane);
    C<T> t[EH];
#pragma unroll
    for (int q = 0; q < EH; ++q) t[q] = S[warp * SP + q * 32 + lane];
    warp_fft_inv<T, EH>(t, lt, lane);
#pragma unroll
    for (int k = 0; k < EH; ++k) x[k] = t[k];
#pragma unroll
    for (int q = 0; q < EH; ++q) t[q] = S[warp * SP + P / 2 + q * 32 + lane];
    warp_fft_inv<T, EH>(t, lt, lane);
#pragma unroll
    for (int k = 0; k < EH; ++k) x[k] = cadd<T>(x[k], cmulc<T>(t[k], tw[lane + 32 * k]));
  } else {
    LaneTw<T, E> ltw;
    ltw.load(tw, lane);
#pragma unroll
    for (int q = 0; q < E; ++q) x[q] = S[warp * SP + q * 32 + lane];
    warp_fft_inv<T, E>(x, ltw, lane);
  }
  pdl_trigger();
  if constexpr (MODE == VIEW_FWD) {
    double nrm = 0.0;
#pragma unroll
    for (int k = 0; k < KH; ++k) {
      const int col = lane + 32 * k;
      const C<T> e = cadd<T>(epi[k], x[k]);
      a.E[rowoff + col] = e;
      nrm += (double)cabs2<T>(e);
    }
    const double tot = block_sum_d<T>(nrm, red);
    if (tid == 0) a.norms[(size_t)v * a.NPV + blockIdx.x] = tot;
  } else if constexpr (MODE == VIEW_BWD && sizeof(T) == 8 && SPLIT) {
    // g_J row = g_J_local + G_D^H g_E; the truncation's contraction over x
    // (spectral.py:56-65), U[yl][w] = F_M(g_J row)[f_w], is one forward
    // length-M FFT of the row (in registers) whose K corner frequencies are
    // picked from the slots holding them; the contraction over the rows stays
    // a small complex GEMM
    C<T> t[EH];
#pragma unroll
    for (int k = 0; k < KH; ++k) t[k] = cadd<T>(a.gJloc[rowoff + lane + 32 * k], conj_<T>(x[k]));
    warp_fft_fwd<T, EH>(t, lt, lane);
#pragma unroll
    for (int q = 0; q < EH; ++q) {
      const int f = spectrum_slot_freq(lane, q, EH);
      const int w = f < mf ? f : (f >= M - mf ? f - (M - 2 * mf) : -1);
      if (w >= 0) U[warp * K + w] = t[q];
    }
    __syncthreads();
    C<T>* gp = a.gpart + ((size_t)v * a.NPV + blockIdx.x) * M0;
    cgemm_dmma(K, K, VL_ROWS,
               [&](int u, int yl) { return twm[(vl_corner_freq<T>(u, mf, M) * (y0 + yl)) & (M - 1)]; },
               [&](int yl, int w) { return U[yl * K + w]; }, [&](int u, int w, C<T> val) { gp[u * K + w] = val; });
  } else if constexpr (MODE == VIEW_BWD) {
    __syncthreads();                     // S is reused as the g_J rows
    C<T>* rows = S;
#pragma unroll
    for (int k = 0; k < KH; ++k) {
      const int col = lane + 32 * k;
      rows[warp * M + col] = cadd<T>(a.gJloc[rowoff + col], conj_<T>(x[k]));
    }
    __syncthreads();
    // U[yl][w] = sum_x gJ[yl][x] exp(-2 pi i kc_w x / M)   (spectral.py:56-65)
    C<T>* gp = a.gpart + ((size_t)v * a.NPV + blockIdx.x) * M0;
    if constexpr (sizeof(T) == 8) {
      cgemm_dmma(VL_ROWS, K, M, [&](int yl, int xx) { return rows[yl * M + xx]; },
                 [&](int xx, int w) { return twm[(vl_corner_freq<T>(w, mf, M) * xx) & (M - 1)]; },
                 [&](int yl, int w, C<T> val) { U[yl * K + w] = val; });
      __syncthreads();
      cgemm_dmma(K, K, VL_ROWS,
                 [&](int u, int yl) { return twm[(vl_corner_freq<T>(u, mf, M) * (y0 + yl)) & (M - 1)]; },
                 [&](int yl, int w) { return U[yl * K + w]; }, [&](int u, int w, C<T> val) { gp[u * K + w] = val; });
    } else {
    for (int i = tid; i < VL_ROWS * K; i += blockDim.x) {
      const int yl = i / K, w = i % K;
      const int f = vl_corner_freq<T>(w, mf, M);
      C<T> acc = czero<T>(), acc1 = czero<T>(), acc2 = czero<T>(), acc3 = czero<T>();
      for (int xx = 0; xx < M; xx += 4) {
        acc = cadd<T>(acc, cmul<T>(rows[yl * M + xx], twm[(f * xx) & (M - 1)]));
        acc1 = cadd<T>(acc1, cmul<T>(rows[yl * M + xx + 1], twm[(f * (xx + 1)) & (M - 1)]));
        acc2 = cadd<T>(acc2, cmul<T>(rows[yl * M + xx + 2], twm[(f * (xx + 2)) & (M - 1)]));
        acc3 = cadd<T>(acc3, cmul<T>(rows[yl * M + xx + 3], twm[(f * (xx + 3)) & (M - 1)]));
      }
      U[i] = cadd<T>(cadd<T>(acc, acc1), cadd<T>(acc2, acc3));
    }
    __syncthreads();
    for (int i = tid; i < M0; i += blockDim.x) {
      const int u = i / K, w = i % K;
      const int f = vl_corner_freq<T>(u, mf, M);
      C<T> acc = czero<T>();
      for (int yl = 0; yl < VL_ROWS; ++yl) acc = cadd<T>(acc, cmul<T>(U[yl * K + w], twm[(f * (y0 + yl)) & (M - 1)]));
      gp[i] = acc;
    }
    }
  } else {
#pragma unroll
    for (int k = 0; k < KH; ++k) {
      const int col = lane + 32 * k;
      a.y[rowoff + col] = a.conj_out ? conj_<T>(x[k]) : x[k];
    }
  }
}

// g_alpha = sum of the truncation partials / (m1 m2) + g_rows conj(H) (the
// G_S^H g_rows part of g_J, pdf_aux.cuh), scattered into the network's
// output-gradient rows; (view 0, block 0) of each scene finalises
// the loss breakdown (losses.py:36-49)
template <typename T>
__global__ void __launch_bounds__(256) vl_trunc_reduce_kernel(VLArgs<T> a) {
  tl_mark(a.tl, 0);
  TlExit tl_exit_{a.tl};
  __shared__ double red[4][4];
  const int M = a.M, mf = a.mf, K = 2 * mf, M0 = K * K;
  const int v = blockIdx.y, scene = v / a.n, view = v % a.n;
  pdl_wait();
  tl_mark(a.tl, 1);
  if (a.do_fin && view == 0 && blockIdx.x == 0) finalize_block(a.fin, scene, red);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M0) return;
  C<T> acc = czero<T>();
  const C<T>* gp = a.gpart + (size_t)v * a.NPV * M0 + i;
  for (int c = 0; c < a.NPV; ++c) acc = cadd<T>(acc, gp[(size_t)c * M0]);
  acc = cscale<T>(acc, T(1) / (T(M) * T(M)));
  const int u = i / K, w = i % K;
  const int slot = vl_corner_slot(u, w, mf);
  acc = cadd<T>(acc, a.gad ? a.gad[(size_t)v * M0 + slot]
                           : data_adjoint_at<T>(a.grows + (size_t)v * a.R, a.hs, a.R, M0, slot, 0, 1));
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

// ---------------------------------------------------------------------------
// Data term D = J G_S^T - d as a split-K complex GEMM.
template <typename T>
struct DataArgs {
  int n, R, npix, chunk, nchunks;
  int nq;               // pixel sub-ranges per chunk (data_mma_kernel)
  const C<T>* J;        // [S*n][npix]
  const C<T>* gs;       // [R][npix]
  C<T>* dpart;          // [S][nchunks][n][R]
  const C<T>* data;     // [S][n][R]
  const T* mask;
  const double* c_sca;
  C<T>* grows;
  double* dloss;
  int tl;               // timeline slot + 1 (0: off)
};

constexpr int DG_KC = 32;          // pixels per staged sub-tile

template <typename T>
__host__ __device__ inline int dg_threads(int n, int R) {
  const int t = ((n + 3) / 4) * ((R + 3) / 4);
  return (t + 31) / 32 * 32;
}
template <typename T>
__host__ __device__ inline size_t dg_smem(int n, int R) {
  return (size_t)2 * (4 * ((n + 3) / 4) + 4 * ((R + 3) / 4)) * (DG_KC + 16 / sizeof(C<T>)) * sizeof(C<T>);
}

// CTA = (pixel chunk, scene).  Thread (ti, tr) owns views ti + NI*a and
// receivers tr + NR*b (a, b < 4): strided ownership keeps the shared reads of
// one warp on distinct banks.  Sub-tiles of DG_KC pixels are double-buffered
// with cp.async.
template <typename T>
__global__ void __launch_bounds__(512) data_gemm_kernel(DataArgs<T> a) {
  tl_mark(a.tl, 0);
  TlExit tl_exit_{a.tl};
  constexpr int EPC = 16 / sizeof(C<T>) > 0 ? 16 / sizeof(C<T>) : 1;   // complex per 16 B
  constexpr int PT = DG_KC + EPC;                                         // padded pitch
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = a.n, R = a.R, NI = (n + 3) / 4, NR = (R + 3) / 4;
  const int nr = 4 * NI, rr = 4 * NR;
  C<T>* Js = reinterpret_cast<C<T>*>(smem_raw);   // 2 x [nr][PT]
  C<T>* Gs = Js + 2 * nr * PT;                     // 2 x [rr][PT]
  const int tid = threadIdx.x, scene = blockIdx.y, chunk = blockIdx.x;
  const int ti = tid / NR, tr = tid % NR;
  const bool active = ti < NI;
  const int p0 = chunk * a.chunk, p1 = min(a.npix, p0 + a.chunk);
  const C<T>* Jb = a.J + (size_t)scene * n * a.npix;
  constexpr int SEG = DG_KC / EPC;
  auto stage = [&](int k0, int s) {
    C<T>* js = Js + s * nr * PT;
    C<T>* gsm = Gs + s * rr * PT;
    for (int i = tid; i < (nr + rr) * SEG; i += blockDim.x) {
      const int row = i / SEG, sg = i % SEG, p = k0 + sg * EPC;
      if (row < nr) {
        const bool ok = row < n && p < p1;
        cp_async16(js + row * PT + sg * EPC, ok ? Jb + (size_t)row * a.npix + p : Jb, ok);
      } else {
        const int r = row - nr;
        const bool ok = r < R && p < p1;
        cp_async16(gsm + r * PT + sg * EPC, ok ? a.gs + (size_t)r * a.npix + p : a.gs, ok);
      }
    }
    cp_async_commit();
  };
  C<T> acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = czero<T>();
  pdl_wait();
  tl_mark(a.tl, 1);
  stage(p0, 0);
  int s = 0;
  for (int k0 = p0; k0 < p1; k0 += DG_KC, s ^= 1) {
    if (k0 + DG_KC < p1) {
      stage(k0 + DG_KC, s ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (active) {
      const C<T>* js = Js + s * nr * PT;
      const C<T>* gsm = Gs + s * rr * PT;
#pragma unroll 4
      for (int kk = 0; kk < DG_KC; ++kk) {
        C<T> jv[4], gv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) jv[i] = js[(ti + NI * i) * PT + kk];
#pragma unroll
        for (int j = 0; j < 4; ++j) gv[j] = gsm[(tr + NR * j) * PT + kk];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc[i][j].x = fma(jv[i].x, gv[j].x, acc[i][j].x);
            acc[i][j].x = fma(-jv[i].y, gv[j].y, acc[i][j].x);
            acc[i][j].y = fma(jv[i].x, gv[j].y, acc[i][j].y);
            acc[i][j].y = fma(jv[i].y, gv[j].x, acc[i][j].y);
          }
      }
    }
    __syncthreads();
  }
  pdl_trigger();
  if (!active) return;
  C<T>* dp = a.dpart + ((size_t)scene * a.nchunks + chunk) * n * R;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int vi = ti + NI * i, r = tr + NR * j;
      if (vi < n && r < R) dp[vi * R + r] = acc[i][j];
    }
}

// The same split-K data GEMM on the FP64 tensor cores (mma.m8n8k4, see
// pdf_net_mma.cuh for the fragment layouts).  A work item is (8 views, 16
// receivers, a pixel sub-range); a complex product is four real MMAs
// (Dr += Jr Gr - Ji Gi, Di += Jr Gi + Ji Gr).  Lane (g, t) streams pixels
// p + 4t .. p + 4t + 3 of one J row and of two G_S rows as 64-byte pieces
// (k permuted identically in A and B), so a 4-lane group reads 256
// contiguous bytes.  Sub-range partials meet in shared memory in a fixed
// order; chunk partials are summed by data_reduce_kernel.
constexpr int DM_NTL = 2;   // receiver n-tiles (of 8) per work item

__host__ __device__ inline size_t dm_smem(int n, int R, int nq) {
  return (size_t)nq * 8 * ((n + 7) / 8) * (8 * DM_NTL) * ((R + 8 * DM_NTL - 1) / (8 * DM_NTL)) * 16;
}


__global__ void __launch_bounds__(256) data_mma_kernel(DataArgs<double> a) {
  tl_mark(a.tl, 0);
  TlExit tl_exit_{a.tl};
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = a.n, R = a.R, npix = a.npix, NQ = a.nq;
  const int MTs = (n + 7) / 8, RGs = (R + 8 * DM_NTL - 1) / (8 * DM_NTL), NTP = MTs * RGs;
  const int NP = 8 * MTs, RP = 8 * DM_NTL * RGs;
  double2* part = reinterpret_cast<double2*>(smem_raw);   // [NQ][NP][RP]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int chunk = blockIdx.x, scene = blockIdx.y;
  const int p0 = chunk * a.chunk, p1 = min(npix, p0 + a.chunk);
  const int sub = ((a.chunk + NQ - 1) / NQ + 15) / 16 * 16;
  const double2* J = reinterpret_cast<const double2*>(a.J) + (size_t)scene * n * npix;
  const double2* G = reinterpret_cast<const double2*>(a.gs);
  pdl_wait();
  tl_mark(a.tl, 1);
  for (int item = warp; item < NTP * NQ; item += 8) {
    const int tp = item % NTP, q = item / NTP, mt = tp / RGs, rg = tp % RGs;
    const int v = 8 * mt + g;
    const double2* jr = J + (size_t)(v < n ? v : 0) * npix;
    const double2* gr[DM_NTL];
    bool rok[DM_NTL];
#pragma unroll
    for (int j = 0; j < DM_NTL; ++j) {
      const int r = rg * 8 * DM_NTL + 8 * j + g;
      rok[j] = r < R;
      gr[j] = G + (size_t)(rok[j] ? r : 0) * npix;
    }
    double dr[DM_NTL][2], di[DM_NTL][2];
#pragma unroll
    for (int j = 0; j < DM_NTL; ++j) dr[j][0] = dr[j][1] = di[j][0] = di[j][1] = 0.0;
    const int ps = p0 + q * sub, pe = min(p1, ps + sub);
    for (int p = ps; p < pe; p += 16) {
      double2 jv[4], gv[DM_NTL][4];
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
        const int pp = p + 4 * t + s4;
        const bool ok = pp < pe;
        jv[s4] = (ok && v < n) ? jr[pp] : make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < DM_NTL; ++j) gv[j][s4] = (ok && rok[j]) ? gr[j][pp] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
        for (int j = 0; j < DM_NTL; ++j) {
          dmma(dr[j][0], dr[j][1], jv[s4].x, gv[j][s4].x);
          dmma(dr[j][0], dr[j][1], -jv[s4].y, gv[j][s4].y);
          dmma(di[j][0], di[j][1], jv[s4].x, gv[j][s4].y);
          dmma(di[j][0], di[j][1], jv[s4].y, gv[j][s4].x);
        }
    }
#pragma unroll
    for (int j = 0; j < DM_NTL; ++j)
#pragma unroll
      for (int c = 0; c < 2; ++c)
        part[((size_t)q * NP + v) * RP + rg * 8 * DM_NTL + 8 * j + 2 * t + c] = make_double2(dr[j][c], di[j][c]);
  }
  __syncthreads();
  pdl_trigger();
  double2* dp = reinterpret_cast<double2*>(a.dpart) + ((size_t)scene * a.nchunks + chunk) * n * R;
  for (int e = tid; e < n * R; e += blockDim.x) {
    const int v = e / R, r = e % R;
    double2 acc = part[(size_t)v * RP + r];
    for (int q = 1; q < NQ; ++q) {
      const double2 x = part[((size_t)q * NP + v) * RP + r];
      acc.x += x.x;
      acc.y += x.y;
    }
    dp[e] = acc;
  }
}

// D = sum of chunk partials - d (masked), g_rows = 2 D mask / c_sca, ||D||^2 per view
template <typename T>
__global__ void __launch_bounds__(128) data_reduce_kernel(DataArgs<T> a) {
  tl_mark(a.tl, 0);
  TlExit tl_exit_{a.tl};
  __shared__ double red[4];
  const int v = blockIdx.x, scene = v / a.n, i = v % a.n, R = a.R;
  pdl_wait();
  tl_mark(a.tl, 1);
  double part = 0.0;
  const double csca = a.c_sca[scene];
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    C<T> acc = czero<T>();
    const C<T>* dp = a.dpart + ((size_t)scene * a.nchunks * a.n + i) * R + r;
    for (int c = 0; c < a.nchunks; ++c) acc = cadd<T>(acc, dp[(size_t)c * a.n * R]);
    const size_t di = (size_t)v * R + r;
    C<T> d = csub<T>(acc, a.data[di]);
    const T mk_ = a.mask ? a.mask[di] : T(1);
    d = cscale<T>(d, mk_);
    part += (double)cabs2<T>(d);
    a.grows[di] = cscale<T>(d, T(2.0 / csca) * mk_);
  }
  pdl_trigger();
  part = warp_sum<double>(part);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    a.dloss[v] = s;
  }
}

}  // namespace pdf
