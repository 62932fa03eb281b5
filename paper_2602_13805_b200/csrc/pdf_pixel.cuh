// Per-pixel kernel of the PDF hot path: everything between the forward and
// the adjoint G_D convolutions that couples the incidences at one pixel.
//
//   chi = sum_i J_i conj(E_i) / (sum_i |E_i|^2 + eps_reg)   cie.py:66-80
//   R   = beta chi / (beta chi + 1), pole check             cie.py:24-30
//   P = E + beta J, S = R P - beta J, ||S||^2               losses.py:225-227
//   bound / tv / bridge values and chi-gradients            losses.py:115-195
//   reverse pass (losses.py:279-300):
//     g_S = 2S/c_inc, g_P = conj(R) g_S, g_J = beta (g_P - g_S)
//     (the G_S^H g_rows part of g_J enters g_alpha through the spectral
//     receiver operator in the view backward, pdf_aux.cuh)
//     g_chi = g_reg + conj(beta/(beta chi+1)^2) sum_i conj(P_i) g_S_i
//     g_num = g_chi/den, g_den = -Re(conj(g_chi) chi)/den
//     g_J += E g_num, g_E = g_P + conj(g_num) J + 2 g_den E
//
// CTA = one scene, one image row y, TX consecutive columns.  Warp w handles
// incidences i = w, w+NW, ...; lane = column inside the tile, so every global
// access is a coalesced row segment.  The regulariser stencils need chi on a
// one-pixel halo, which the CTA recomputes (rows y-1..y+1) instead of a
// separate launch; the stencil terms of rows y-1 and y are computed once per
// halo pixel by parallel threads.  All cross-view sums are fixed-order
// (deterministic).
#pragma once
#include "pdf_common.cuh"
#include "pdf_dmma.cuh"

namespace pdf {

template <typename T>
struct PixelArgs {
  int M, n, R, CS, S;
  T beta, l1, l2, l3, tau;
  const C<T>* J;        // [S*n][M][M]
  const C<T>* E;        // [S*n][M][M]
  const double* norms;  // [S*n][CS]
  const C<T>* rfixed;   // [S][M][M] or null
  const double* c_inc;  // [S]
  C<T>* gJ;             // [S*n][M][M]  (g_J local part)
  C<T>* gE;             // [S*n][M][M]
  double* part;         // [S][ntiles][4]  state, bound, tv, bridge
  C<T>* chi_out;        // [S][M][M] or null
  int* err;             // [S]
  int tl;               // timeline slot + 1 (0: off)
};

constexpr double EPS_TV = 1e-12;   // losses.py:29
constexpr int PIX_TX = 32;         // max tile width
constexpr int PIX_NW = 8;          // warps per CTA

template <typename T>
__device__ __forceinline__ T amag(C<T> z) { return sqrt_<T>(cabs2<T>(z)); }

// ILP2: the halo pass loads two views per pass (latency regime: few CTAs;
// doubles the registers, so batches keep one view per pass)
template <typename T, bool GRAD, bool ILP2 = false>
__global__ void __launch_bounds__(PIX_NW * 32) pixel_kernel(PixelArgs<T> a) {
  constexpr int W = PIX_TX + 2;
  __shared__ C<T> pnum[PIX_NW][3 * W];
  __shared__ T pden[PIX_NW][3 * W];
  __shared__ C<T> chis[3 * W];
  // stencil terms for rows y-1 (index 0) and y (index 1) over columns x0-1 .. x0+TX
  __shared__ C<T> twx[2][W], twy[2][W];       // tv weights dx/s, dy/s
  __shared__ T ts[2][W];                      // tv value s
  __shared__ T bsig[2][W], bdamp[2][W], bcx[2][W], bcy[2][W];
  __shared__ T dens[PIX_TX];
  __shared__ C<T> Rs[PIX_TX], chain[PIX_TX], greg[PIX_TX], gnum[PIX_TX];
  __shared__ T gden[PIX_TX];
  __shared__ C<T> pgr[PIX_NW][PIX_TX];
  __shared__ double red[PIX_NW][4];
  __shared__ double eps_s;

  const int M = a.M, n = a.n;
  const int TX = M < PIX_TX ? M : PIX_TX;
  const int NH = 3 * (TX + 2);
  const int WW = TX + 2;
  const int tilesx = M / TX;
  const int x0 = blockIdx.x * TX, y = blockIdx.y, scene = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const size_t img = (size_t)M * M;
  const size_t vbase = (size_t)scene * n;

  tl_mark(a.tl, 0);
  pdl_wait();   // J, E, norms come from the previous kernel
  tl_mark(a.tl, 1);

  if (warp == 0) {
    const double mx = warp_max_view_power(a.norms + vbase * a.CS, n, a.CS);
    if (lane == 0) eps_s = 1e-10 * mx / (double)img;   // cie.py:49-50
  }

  // ---- per-warp partial num/den on the halo --------------------------------
  // halo entries h = lane + 32 q (NH <= 3 (32 + 2) < 128): the four entries'
  // loads of one view are in flight together; per entry the views are summed
  // in increasing order
  {
    constexpr int QH = 4;
    C<T> num[QH];
    T den[QH];
    size_t pix[QH];
    bool ok[QH];
#pragma unroll
    for (int q = 0; q < QH; ++q) {
      const int h = lane + 32 * q;
      const int hy = y - 1 + h / WW, hx = x0 - 1 + h % WW;
      ok[q] = h < NH && hy >= 0 && hy < M && hx >= 0 && hx < M;
      pix[q] = ok[q] ? (size_t)hy * M + hx : 0;
      num[q] = czero<T>();
      den[q] = T(0);
    }
    // two views per pass: 16 loads in flight per thread, added in view order
    int i = warp;
    for (; ILP2 && i + nw < n; i += 2 * nw) {
      C<T> j[2][QH], e[2][QH];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int q = 0; q < QH; ++q) {
          const size_t o = (vbase + i + u * nw) * img + pix[q];
          j[u][q] = ok[q] ? a.J[o] : czero<T>();
          e[u][q] = ok[q] ? a.E[o] : czero<T>();
        }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int q = 0; q < QH; ++q) {
          num[q] = cadd<T>(num[q], cmulc<T>(j[u][q], e[u][q]));
          den[q] += cabs2<T>(e[u][q]);
        }
    }
    for (; i < n; i += nw) {
      C<T> j[QH], e[QH];
#pragma unroll
      for (int q = 0; q < QH; ++q) {
        j[q] = ok[q] ? a.J[(vbase + i) * img + pix[q]] : czero<T>();
        e[q] = ok[q] ? a.E[(vbase + i) * img + pix[q]] : czero<T>();
      }
#pragma unroll
      for (int q = 0; q < QH; ++q) {
        num[q] = cadd<T>(num[q], cmulc<T>(j[q], e[q]));
        den[q] += cabs2<T>(e[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < QH; ++q) {
      const int h = lane + 32 * q;
      if (h < NH) { pnum[warp][h] = num[q]; pden[warp][h] = den[q]; }
    }
  }
  __syncthreads();
  tl_stage(a.tl, 0);
  const T eps = (T)eps_s;
  for (int h = tid; h < NH; h += blockDim.x) {
    C<T> num = czero<T>();
    T den = T(0);
    for (int w = 0; w < nw; ++w) { num = cadd<T>(num, pnum[w][h]); den += pden[w][h]; }
    den += eps;
    chis[h] = mk<T>(num.x / den, num.y / den);   // numpy complex/real division
    if (h / WW == 1 && (h % WW) >= 1 && (h % WW) <= TX) dens[h % WW - 1] = den;
  }
  __syncthreads();
  tl_stage(a.tl, 1);

  // ---- stencil terms at rows y-1, y (forward differences, losses.py:139-144)
  const T tau = a.tau;
  for (int q = tid; q < 2 * WW; q += blockDim.x) {
    const int row = q / WW, cix = q % WW;           // row 0: y-1, row 1: y
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
  tl_stage(a.tl, 2);

  // ---- per-pixel scalar work ------------------------------------------------
  double vb = 0.0, vt = 0.0, vr = 0.0;
  if (tid < TX) {
    const int x = x0 + tid, c1 = tid + 1;            // column index of x in the halo arrays
    const C<T> chi = chis[WW + c1];
    const T neg = chi.x < T(0) ? chi.x : T(0);
    vb = (double)(neg * neg);
    vt = (double)ts[1][c1];
    vr = (double)(bsig[1][c1] * bdamp[1][c1]);
    if (a.chi_out) a.chi_out[(size_t)scene * img + (size_t)y * M + x] = chi;
    if (GRAD) {
      C<T> g = czero<T>();
      if (a.l1 != T(0)) g = cadd<T>(g, mk<T>(a.l1 * (T(2) * neg), T(0)));
      if (a.l2 != T(0)) {
        // g += wx(y, x-1) - wx(y, x) + wy(y-1, x) - wy(y, x)   (losses.py:156-165)
        C<T> gt = mk<T>(-twx[1][c1].x - twy[1][c1].x, -twx[1][c1].y - twy[1][c1].y);
        if (x >= 1) gt = cadd<T>(gt, twx[1][c1 - 1]);
        if (y >= 1) gt = cadd<T>(gt, twy[0][c1]);
        g = cadd<T>(g, cscale<T>(gt, a.l2));
      }
      if (a.l3 != T(0)) {
        // (losses.py:168-182)
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
      greg[tid] = g;
    }
    C<T> R_;
    if (a.rfixed) {
      R_ = a.rfixed[(size_t)scene * img + (size_t)y * M + x];
      chain[tid] = czero<T>();
    } else {
      const C<T> q = mk<T>(a.beta * chi.x + T(1), a.beta * chi.y);
      if (sqrt_<T>(cabs2<T>(q)) < T(1e-14)) atomicOr(&a.err[scene], ERR_POLE);
      R_ = cdiv<T>(mk<T>(a.beta * chi.x, a.beta * chi.y), q);
      chain[tid] = conj_<T>(cdiv<T>(mk<T>(a.beta, T(0)), cmul<T>(q, q)));   // conj(beta / q^2)
    }
    Rs[tid] = R_;
  }
  __syncthreads();
  tl_stage(a.tl, 3);

  // ---- state residual, R-chain partial ------------------------------------
  const T beta = a.beta;
  const T gsc = T(2.0 / a.c_inc[scene]);
  double vs = 0.0;
  if (lane < TX) {
    const size_t pix = (size_t)y * M + x0 + lane;
    const C<T> R_ = Rs[lane];
    C<T> gr = czero<T>();
    for (int i = warp; i < n; i += nw) {
      const C<T> j = a.J[(vbase + i) * img + pix];
      const C<T> e = a.E[(vbase + i) * img + pix];
      const C<T> P = mk<T>(e.x + beta * j.x, e.y + beta * j.y);
      const C<T> Sr = csub<T>(cmul<T>(R_, P), mk<T>(beta * j.x, beta * j.y));
      vs += (double)cabs2<T>(Sr);
      if (GRAD) gr = cadd<T>(gr, cmulc<T>(cscale<T>(Sr, gsc), P));   // conj(P) g_S
    }
    if (GRAD) pgr[warp][lane] = gr;
  }
  pdl_trigger();
  if (GRAD) {
    __syncthreads();
    tl_stage(a.tl, 4);
    if (tid < TX) {
      C<T> gr = czero<T>();
      for (int w = 0; w < nw; ++w) gr = cadd<T>(gr, pgr[w][tid]);
      const C<T> chi = chis[WW + 1 + tid];
      C<T> gchi = greg[tid];
      if (!a.rfixed) gchi = cadd<T>(gchi, cmul<T>(chain[tid], gr));
      const T den = dens[tid];
      gnum[tid] = mk<T>(gchi.x / den, gchi.y / den);
      gden[tid] = -(gchi.x * chi.x + gchi.y * chi.y) / den;   // -Re(conj(g_chi) chi)/den
    }
    __syncthreads();
    tl_stage(a.tl, 5);
    if (lane < TX) {
      const size_t pix = (size_t)y * M + x0 + lane;
      const C<T> R_ = Rs[lane];
      const C<T> gn = gnum[lane];
      const T gd = gden[lane];
      for (int i = warp; i < n; i += nw) {
        const size_t o = (vbase + i) * img + pix;
        const C<T> j = a.J[o];
        const C<T> e = a.E[o];
        const C<T> P = mk<T>(e.x + beta * j.x, e.y + beta * j.y);
        const C<T> Sr = csub<T>(cmul<T>(R_, P), mk<T>(beta * j.x, beta * j.y));
        const C<T> gS = cscale<T>(Sr, gsc);
        const C<T> gP = cmul<T>(conj_<T>(R_), gS);
        C<T> gj = cscale<T>(csub<T>(gP, gS), beta);
        gj = cadd<T>(gj, cmul<T>(e, gn));
        C<T> ge = cadd<T>(gP, cmul<T>(conj_<T>(gn), j));
        ge = cadd<T>(ge, cscale<T>(e, T(2) * gd));
        a.gJ[o] = gj;
        a.gE[o] = ge;
      }
    }
  }

  tl_stage(a.tl, 6);
  // ---- loss partials (fixed order) ----------------------------------------
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
  tl_mark(a.tl, 2);
}

// breakdown per scene: [state, data, bound, tv, bridge, total] (losses.py:36-49)
struct FinalizeArgs {
  int n, ntiles, S;
  double l1, l2, l3;
  const double* c_inc;
  const double* c_sca;
  const double* dloss;   // [S*n]
  const double* part;    // [S][ntiles][4]
  double* bd;            // [S][6]
  double* trace;         // [k][S][6] or null
  const int* step;       // device step counter (trace row = step-1)
  int* err;              // [S]
};

// One CTA (>= 128 threads) reduces a scene's partials; the first 128 threads
// take part in a fixed pattern, so the result does not depend on blockDim and
// is bitwise identical wherever it runs (standalone or inside view_bwd).
__device__ inline void finalize_block(const FinalizeArgs& a, int scene, double (*red)[4]) {
  const int tid = threadIdx.x;
  double s[4] = {0, 0, 0, 0};
  if (tid < 128)
    for (int t = tid; t < a.ntiles; t += 128)
      for (int k = 0; k < 4; ++k) s[k] += a.part[((size_t)scene * a.ntiles + t) * 4 + k];
  for (int k = 0; k < 4; ++k) s[k] = warp_sum<double>(s[k]);
  if ((tid & 31) == 0 && tid < 128) for (int k = 0; k < 4; ++k) red[tid >> 5][k] = s[k];
  __syncthreads();
  if (tid == 0) {
    double st = 0, bo = 0, tv = 0, br = 0, da = 0;
    for (int w = 0; w < 4; ++w) { st += red[w][0]; bo += red[w][1]; tv += red[w][2]; br += red[w][3]; }
    for (int i = 0; i < a.n; ++i) da += a.dloss[(size_t)scene * a.n + i];
    st /= a.c_inc[scene];
    da /= a.c_sca[scene];
    const double tot = st + da + a.l1 * bo + a.l2 * tv + a.l3 * br;
    double* o = a.bd + (size_t)scene * 6;
    o[0] = st; o[1] = da; o[2] = bo; o[3] = tv; o[4] = br; o[5] = tot;
    if (a.trace) {
      double* tr = a.trace + ((size_t)(*a.step - 1) * a.S + scene) * 6;
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
      atomicOr(&a.err[scene], bits);
    }
  }
}

__global__ void finalize_kernel(FinalizeArgs a) {
  __shared__ double red[4][4];
  finalize_block(a, blockIdx.x, red);
}

}  // namespace pdf
