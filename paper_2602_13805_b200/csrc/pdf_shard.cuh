// Incidence-sharded pixel stage.
//
// With the views of one scene split across ranks, the per-pixel algebra of
// pixel_kernel couples all views twice:
//   (1) chi = sum_i J_i conj(E_i) / (sum_i |E_i|^2 + eps), eps from the max view power
//   (2) g_chi needs g_R = sum_i conj(P_i) g_S_i
// so the fused kernel splits into three, with a host all-reduce after the
// first two (the library exposes the buffers; the caller owns the collective):
//   shard_numden  : own-view partial num / den per pixel, max own view power
//   shard_pixel_a : chi, R, regulariser values and chi-gradients (redundant on
//                   every rank), own-view state residual, partial g_R per pixel
//   shard_pixel_b : g_chi from the reduced g_R, LS-quotient adjoint, own-view
//                   g_J (incl. G_S^H g_rows) and g_E
// Reduction buffers per scene: red1 = [num (M^2 complex) | den (M^2 real) | pmax]
//                              red2 = [g_R (M^2 complex) | state_sum, data_sum]
// All sums inside a kernel are fixed-order; the cross-rank sums are the
// caller's all-reduce (NCCL ring/tree order is deterministic for a fixed
// topology).
#pragma once
#include "pdf_common.cuh"
#include "pdf_pixel.cuh"

namespace pdf {

template <typename T>
struct ShardArgs {
  int M, n, R, CS;
  T beta, l1, l2, l3, tau;
  const C<T>* J;        // [S*n][M*M] own views
  const C<T>* E;
  const double* norms;  // [S*n][CS]
  const C<T>* grows;    // [S*n][R]
  const C<T>* rfixed;   // [S][M*M] or null
  const double* c_inc;
  double* red1;         // [S][3*M*M + 1] doubles: num (re,im interleaved), den, pmax
  double* red2;         // [S][2*M*M + 2]: g_R (re,im), state_sum, data_sum
  const double* dloss;  // [S*n] own-view data loss
  double* pix;          // [S][M*M][12] per-pixel scalars: chi, R, chain, greg (complex) | den, pad
  double* part;         // [S][ntiles][4]
  C<T>* gJ;
  C<T>* gE;
  C<T>* chi_out;        // [S][M*M] or null
  int* err;
};

template <typename T>
__global__ void shard_numden_kernel(ShardArgs<T> a) {
  const int M = a.M, n = a.n, scene = blockIdx.y;
  const size_t img = (size_t)M * M;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  double* r1 = a.red1 + (size_t)scene * (3 * img + 1);
  pdl_wait();
  if (p < (int)img) {
    C<T> num = czero<T>();
    T den = T(0);
    for (int i = 0; i < n; ++i) {
      const C<T> j = a.J[((size_t)scene * n + i) * img + p];
      const C<T> e = a.E[((size_t)scene * n + i) * img + p];
      num = cadd<T>(num, cmulc<T>(j, e));
      den += cabs2<T>(e);
    }
    r1[2 * p] = num.x;
    r1[2 * p + 1] = num.y;
    r1[2 * img + p] = den;
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    const double mx = warp_max_view_power(a.norms + (size_t)scene * n * a.CS, n, a.CS);
    if (threadIdx.x == 0) r1[3 * img] = mx;
  }
}

// stage A: CTA = scene, row y, TX columns (same tiling as pixel_kernel)
template <typename T>
__global__ void __launch_bounds__(PIX_NW * 32) shard_pixel_a_kernel(ShardArgs<T> a) {
  constexpr int W = PIX_TX + 2;
  __shared__ C<T> chis[3 * W];
  __shared__ C<T> twx[2][W], twy[2][W];
  __shared__ T ts[2][W], bsig[2][W], bdamp[2][W], bcx[2][W], bcy[2][W];
  __shared__ C<T> Rs[PIX_TX];
  __shared__ C<T> pgr[PIX_NW][PIX_TX];
  __shared__ double red[PIX_NW][4];
  const int M = a.M, n = a.n;
  const int TX = M < PIX_TX ? M : PIX_TX, WW = TX + 2, NH = 3 * WW;
  const int tilesx = M / TX;
  const int x0 = blockIdx.x * TX, y = blockIdx.y, scene = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const size_t img = (size_t)M * M;
  const double* r1 = a.red1 + (size_t)scene * (3 * img + 1);
  pdl_wait();
  const double eps = 1e-10 * r1[3 * img] / (double)img;   // cie.py:49-50 with the global max
  for (int h = tid; h < NH; h += blockDim.x) {
    const int hy = y - 1 + h / WW, hx = x0 - 1 + h % WW;
    C<T> chi = czero<T>();
    if (hy >= 0 && hy < M && hx >= 0 && hx < M) {
      const size_t p = (size_t)hy * M + hx;
      const T den = (T)(r1[2 * img + p] + eps);
      chi = mk<T>((T)r1[2 * p] / den, (T)r1[2 * p + 1] / den);
    }
    chis[h] = chi;
  }
  __syncthreads();
  const T tau = a.tau;
  for (int q = tid; q < 2 * WW; q += blockDim.x) {
    const int row = q / WW, cix = q % WW;
    const int yy = y - 1 + row, xx = x0 - 1 + cix;
    C<T> wx = czero<T>(), wy = czero<T>();
    T s = T(0), sig = T(0), damp = T(0), cx = T(0), cy = T(0);
    if (yy >= 0 && yy < M && xx >= 0 && xx < M) {
      const C<T> c = chis[row * WW + cix];
      const C<T> dx = (xx + 1 < M) ? csub<T>(chis[row * WW + cix + 1], c) : czero<T>();
      const C<T> dy = (yy + 1 < M) ? csub<T>(chis[(row + 1) * WW + cix], c) : czero<T>();
      s = sqrt_<T>(cabs2<T>(dx) + cabs2<T>(dy) + T(EPS_TV));
      wx = mk<T>(dx.x / s, dx.y / s);
      wy = mk<T>(dy.x / s, dy.y / s);
      const T am = amag<T>(c);
      const T gx = (xx + 1 < M) ? amag<T>(chis[row * WW + cix + 1]) - am : T(0);
      const T gy = (yy + 1 < M) ? amag<T>(chis[(row + 1) * WW + cix]) - am : T(0);
      sig = sigmoid_<T>((am - tau) / tau);
      damp = exp_<T>(-(gx * gx + gy * gy));
      cx = T(-2) * sig * damp * gx;
      cy = T(-2) * sig * damp * gy;
    }
    twx[row][cix] = wx; twy[row][cix] = wy; ts[row][cix] = s;
    bsig[row][cix] = sig; bdamp[row][cix] = damp; bcx[row][cix] = cx; bcy[row][cix] = cy;
  }
  __syncthreads();
  double vb = 0.0, vt = 0.0, vr = 0.0;
  if (tid < TX) {
    const int x = x0 + tid, c1 = tid + 1;
    const size_t p = (size_t)y * M + x;
    const C<T> chi = chis[WW + c1];
    const T neg = chi.x < T(0) ? chi.x : T(0);
    vb = (double)(neg * neg);
    vt = (double)ts[1][c1];
    vr = (double)(bsig[1][c1] * bdamp[1][c1]);
    if (a.chi_out) a.chi_out[(size_t)scene * img + p] = chi;
    C<T> g = czero<T>();
    if (a.l1 != T(0)) g = cadd<T>(g, mk<T>(a.l1 * (T(2) * neg), T(0)));
    if (a.l2 != T(0)) {
      C<T> gt = mk<T>(-twx[1][c1].x - twy[1][c1].x, -twx[1][c1].y - twy[1][c1].y);
      if (x >= 1) gt = cadd<T>(gt, twx[1][c1 - 1]);
      if (y >= 1) gt = cadd<T>(gt, twy[0][c1]);
      g = cadd<T>(g, cscale<T>(gt, a.l2));
    }
    if (a.l3 != T(0)) {
      const T sg = bsig[1][c1];
      T ga = sg * (T(1) - sg) / tau * bdamp[1][c1];
      ga -= bcx[1][c1];
      ga -= bcy[1][c1];
      if (x >= 1) ga += bcx[1][c1 - 1];
      if (y >= 1) ga += bcy[0][c1];
      const T am = amag<T>(chi);
      const C<T> ph = am > T(0) ? mk<T>(chi.x / am, chi.y / am) : czero<T>();
      g = cadd<T>(g, cscale<T>(ph, a.l3 * ga));
    }
    C<T> R_, chn;
    if (a.rfixed) {
      R_ = a.rfixed[(size_t)scene * img + p];
      chn = czero<T>();
    } else {
      const C<T> q = mk<T>(a.beta * chi.x + T(1), a.beta * chi.y);
      if (sqrt_<T>(cabs2<T>(q)) < T(1e-14)) atomicOr(&a.err[scene], ERR_POLE);
      R_ = cdiv<T>(mk<T>(a.beta * chi.x, a.beta * chi.y), q);
      chn = conj_<T>(cdiv<T>(mk<T>(a.beta, T(0)), cmul<T>(q, q)));
    }
    Rs[tid] = R_;
    double* px = a.pix + ((size_t)scene * img + p) * 12;
    px[0] = chi.x; px[1] = chi.y; px[2] = R_.x; px[3] = R_.y; px[4] = chn.x; px[5] = chn.y;
    px[6] = g.x; px[7] = g.y;
    px[8] = r1[2 * img + p] + eps;
  }
  __syncthreads();
  const T beta = a.beta;
  const T gsc = T(2.0 / a.c_inc[scene]);
  double vs = 0.0;
  if (lane < TX) {
    const size_t pix = (size_t)y * M + x0 + lane;
    const C<T> R_ = Rs[lane];
    C<T> gr = czero<T>();
    for (int i = warp; i < n; i += nw) {
      const C<T> j = a.J[((size_t)scene * n + i) * img + pix];
      const C<T> e = a.E[((size_t)scene * n + i) * img + pix];
      const C<T> P = mk<T>(e.x + beta * j.x, e.y + beta * j.y);
      const C<T> Sr = csub<T>(cmul<T>(R_, P), mk<T>(beta * j.x, beta * j.y));
      vs += (double)cabs2<T>(Sr);
      gr = cadd<T>(gr, cmulc<T>(cscale<T>(Sr, gsc), P));
    }
    pgr[warp][lane] = gr;
  }
  __syncthreads();
  if (tid < TX) {
    C<T> gr = czero<T>();
    for (int w = 0; w < nw; ++w) gr = cadd<T>(gr, pgr[w][tid]);
    double* r2 = a.red2 + (size_t)scene * (2 * img + 2);
    const size_t p = (size_t)y * M + x0 + tid;
    r2[2 * p] = gr.x;
    r2[2 * p + 1] = gr.y;
  }
  pdl_trigger();
  vs = warp_sum<double>(vs);
  vb = warp_sum<double>(vb);
  vt = warp_sum<double>(vt);
  vr = warp_sum<double>(vr);
  if (lane == 0) { red[warp][0] = vs; red[warp][1] = vb; red[warp][2] = vt; red[warp][3] = vr; }
  __syncthreads();
  if (tid < 4) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[w][tid];
    const int tile = y * tilesx + blockIdx.x;
    a.part[((size_t)scene * (tilesx * M) + tile) * 4 + tid] = s;
  }
}

// the rank's state / data loss sums into red2's tail (before the all-reduce)
__global__ void shard_loss_sums_kernel(const double* part, const double* dloss, double* red2, int ntiles, int n,
                                       size_t img) {
  const int scene = blockIdx.x;
  __shared__ double red[4][4];
  const int tid = threadIdx.x;
  double s = 0.0;
  if (tid < 128)
    for (int t = tid; t < ntiles; t += 128) s += part[((size_t)scene * ntiles + t) * 4];
  s = warp_sum<double>(s);
  if ((tid & 31) == 0 && tid < 128) red[tid >> 5][0] = s;
  __syncthreads();
  if (tid == 0) {
    double st = 0.0, da = 0.0;
    for (int w = 0; w < 4; ++w) st += red[w][0];
    for (int i = 0; i < n; ++i) da += dloss[(size_t)scene * n + i];
    double* r2 = red2 + (size_t)scene * (2 * img + 2);
    r2[2 * img] = st;
    r2[2 * img + 1] = da;
  }
}

// stage B: g_chi from the reduced g_R, outputs for the own views (thread per pixel x view slot)
template <typename T>
__global__ void __launch_bounds__(PIX_NW * 32) shard_pixel_b_kernel(ShardArgs<T> a) {
  const int M = a.M, n = a.n, R = a.R;
  const int TX = M < PIX_TX ? M : PIX_TX;
  const int x0 = blockIdx.x * TX, y = blockIdx.y, scene = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const size_t img = (size_t)M * M;
  pdl_wait();
  if (lane >= TX) return;
  const size_t pix = (size_t)y * M + x0 + lane;
  const double* px = a.pix + ((size_t)scene * img + pix) * 12;
  const double* r2 = a.red2 + (size_t)scene * (2 * img + 2);
  const C<T> chi = mk<T>((T)px[0], (T)px[1]);
  const C<T> R_ = mk<T>((T)px[2], (T)px[3]);
  const C<T> chn = mk<T>((T)px[4], (T)px[5]);
  C<T> gchi = mk<T>((T)px[6], (T)px[7]);
  const T den = (T)px[8];
  if (!a.rfixed) gchi = cadd<T>(gchi, cmul<T>(chn, mk<T>((T)r2[2 * pix], (T)r2[2 * pix + 1])));
  const C<T> gn = mk<T>(gchi.x / den, gchi.y / den);
  const T gd = -(gchi.x * chi.x + gchi.y * chi.y) / den;
  const T beta = a.beta;
  const T gsc = T(2.0 / a.c_inc[scene]);
  for (int i = warp; i < n; i += nw) {
    const size_t o = ((size_t)scene * n + i) * img + pix;
    const C<T> j = a.J[o];
    const C<T> e = a.E[o];
    const C<T> P = mk<T>(e.x + beta * j.x, e.y + beta * j.y);
    const C<T> Sr = csub<T>(cmul<T>(R_, P), mk<T>(beta * j.x, beta * j.y));
    const C<T> gS = cscale<T>(Sr, gsc);
    const C<T> gP = cmul<T>(conj_<T>(R_), gS);
    C<T> gj = cscale<T>(csub<T>(gP, gS), beta);
    // (G_S^H g_rows enters g_alpha through H in the view backward, pdf_aux.cuh)
    gj = cadd<T>(gj, cmul<T>(e, gn));
    C<T> ge = cadd<T>(gP, cmul<T>(conj_<T>(gn), j));
    ge = cadd<T>(ge, cscale<T>(e, T(2) * gd));
    a.gJ[o] = gj;
    a.gE[o] = ge;
  }
}

// breakdown from the reduced sums (state, data) and the local regulariser partials
__global__ void shard_finalize_kernel(FinalizeArgs f, const double* red2, size_t img) {
  const int scene = blockIdx.x;
  __shared__ double red[4][4];
  const int tid = threadIdx.x;
  double s[3] = {0, 0, 0};
  if (tid < 128)
    for (int t = tid; t < f.ntiles; t += 128)
      for (int k = 0; k < 3; ++k) s[k] += f.part[((size_t)scene * f.ntiles + t) * 4 + 1 + k];
  for (int k = 0; k < 3; ++k) s[k] = warp_sum<double>(s[k]);
  if ((tid & 31) == 0 && tid < 128) for (int k = 0; k < 3; ++k) red[tid >> 5][k] = s[k];
  __syncthreads();
  if (tid == 0) {
    double bo = 0, tv = 0, br = 0;
    for (int w = 0; w < 4; ++w) { bo += red[w][0]; tv += red[w][1]; br += red[w][2]; }
    const double* r2 = red2 + (size_t)scene * (2 * img + 2);
    const double st = r2[2 * img] / f.c_inc[scene];
    const double da = r2[2 * img + 1] / f.c_sca[scene];
    const double tot = st + da + f.l1 * bo + f.l2 * tv + f.l3 * br;
    double* o = f.bd + (size_t)scene * 6;
    o[0] = st; o[1] = da; o[2] = bo; o[3] = tv; o[4] = br; o[5] = tot;
    if (f.trace) {
      double* tr = f.trace + ((size_t)(*f.step - 1) * f.S + scene) * 6;
      for (int k = 0; k < 6; ++k) tr[k] = o[k];
    }
    if (!isfinite(tot)) {
      int bits = 0;
      if (!isfinite(st)) bits |= ERR_NONFINITE_STATE;
      if (!isfinite(da)) bits |= ERR_NONFINITE_DATA;
      if (!isfinite(bo)) bits |= ERR_NONFINITE_BOUND;
      if (!isfinite(tv)) bits |= ERR_NONFINITE_TV;
      if (!isfinite(br)) bits |= ERR_NONFINITE_BRIDGE;
      if (!bits) bits = ERR_NONFINITE_STATE;
      atomicOr(&f.err[scene], bits);
    }
  }
}

}  // namespace pdf
