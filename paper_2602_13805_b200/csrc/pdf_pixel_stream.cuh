// Throughput form of the per-pixel stage (batches, many views): the fused
// pixel_kernel (pdf_pixel.cuh) serialises load -> chi -> stencil -> scalar ->
// state -> gradient inside one CTA, with block barriers between phases that
// only a few warps execute; with two CTAs per SM the SM idles most of the
// time (0.27 of HBM in the cfg4 batch).  Here the stage is three streaming
// kernels without a view loop inside any barrier phase:
//
//   pix_sums_kernel   per pixel  num = sum_i J_i conj(E_i), den0 = sum_i |E_i|^2,
//                                cj = sum_i |J_i|^2                (one pass over J, E)
//   pix_point_kernel  per pixel  chi, R, regulariser values / gradients (1-pixel
//                                halo of chi recomputed from the sums, no field
//                                traffic), state term and the R-chain sum in
//                                closed form, LS-quotient adjoint coefficients
//   pix_grad_kernel   per pixel and view  g_J, g_E                 (one pass over J, E)
//
// Closed forms (P_i = E_i + beta J_i, S_i = R P_i - beta J_i, losses.py:225-227,
// 279-300): with A = sum_i |P_i|^2 = den0 + 2 beta Re(num) + beta^2 cj and
// B = sum_i J_i conj(P_i) = num + beta cj,
//     sum_i |S_i|^2            = |R|^2 A - 2 beta Re(conj(R) B) + beta^2 cj
//     sum_i conj(P_i) g_S_i    = (2 / c_inc) (R A - beta B)
// so neither needs a pass over the views once the three sums exist.  The
// price is cancellation: both are differences of terms of size beta^2 cj, so
// they carry an absolute error of ~1e-16 beta^2 sum_i |J_i|^2 where the
// per-view form of pixel_kernel resolves the residual itself.  On the
// BASELINE scenes the state term is 1e-4 .. 1e-2 of that size (relative error
// 1e-12 .. 1e-14, inside the 1e-10 parity gates: tests compare this path with
// the fused kernel and the goldens); a state residual that cancels to
// rounding (the reference's near-pole test, tests/test_gpu_edges.py) is only
// resolved by the fused kernel, which keeps the per-view pass and serves every
// problem below the batch threshold.  Every
// sum runs in a fixed order (views per warp in increasing order, then warps
// in order; loss partials per image row as in pixel_kernel).
#pragma once
#include "pdf_common.cuh"
#include "pdf_pixel.cuh"

namespace pdf {

template <typename T>
struct PixStreamArgs {
  PixelArgs<T> p;
  double* sums;   // [S][M*M][4]  num.x num.y den0 cj
  double* coef;   // [S][M*M][6]  R.x R.y gn.x gn.y gd pad
};

// CTA = 32 consecutive pixels of a scene (lane = pixel), warp w sums views
// w, w + 8, ...; partial sums meet in shared memory in warp order
template <typename T>
__global__ void __launch_bounds__(256) pix_sums_kernel(PixStreamArgs<T> a) {
  __shared__ double part[8][32][4];
  const int n = a.p.n, scene = blockIdx.y;
  const size_t img = (size_t)a.p.M * a.p.M;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t pix = (size_t)blockIdx.x * 32 + lane;
  tl_mark(a.p.tl, 0);
  pdl_wait();
  tl_mark(a.p.tl, 1);
  const C<T>* J = a.p.J + (size_t)scene * n * img + pix;
  const C<T>* E = a.p.E + (size_t)scene * n * img + pix;
  C<T> num = czero<T>();
  T den = T(0), cj = T(0);
  int i = warp;
  for (; i + 8 < n; i += 16) {   // two views in flight per warp
    const C<T> j0 = J[(size_t)i * img], e0 = E[(size_t)i * img];
    const C<T> j1 = J[(size_t)(i + 8) * img], e1 = E[(size_t)(i + 8) * img];
    num = cadd<T>(num, cmulc<T>(j0, e0));
    den += cabs2<T>(e0);
    cj += cabs2<T>(j0);
    num = cadd<T>(num, cmulc<T>(j1, e1));
    den += cabs2<T>(e1);
    cj += cabs2<T>(j1);
  }
  if (i < n) {
    const C<T> j0 = J[(size_t)i * img], e0 = E[(size_t)i * img];
    num = cadd<T>(num, cmulc<T>(j0, e0));
    den += cabs2<T>(e0);
    cj += cabs2<T>(j0);
  }
  part[warp][lane][0] = (double)num.x;
  part[warp][lane][1] = (double)num.y;
  part[warp][lane][2] = (double)den;
  part[warp][lane][3] = (double)cj;
  __syncthreads();
  pdl_trigger();
  if (threadIdx.x < 128) {
    const int px = threadIdx.x >> 2, k = threadIdx.x & 3;
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += part[w][px][k];
    a.sums[((size_t)scene * img + (size_t)blockIdx.x * 32 + px) * 4 + k] = s;
  }
}

// CTA = TY image rows x TX columns of a scene; everything per pixel.  The
// stencil terms are the ones of pixel_kernel (same expressions, same order).
// FUSE (with GRAD): the gradient pass over the views runs in this kernel, thread
// = pixel (a warp = 32 consecutive pixels of a row): the coefficients stay in
// registers and the per-pixel arithmetic of one CTA hides behind the field
// streaming of the others on its SM (pix_point + pix_grad as two launches:
// 79 + 168 us at cfg4, the second with 16 % of its issue slots used).
template <typename T, bool GRAD, int TY, bool FUSE>
__global__ void __launch_bounds__(128) pix_point_kernel(PixStreamArgs<T> a) {
  constexpr int W = PIX_TX + 2, HR = TY + 2;
  __shared__ C<T> chis[HR][W];
  __shared__ C<T> twx[TY + 1][W], twy[TY + 1][W];
  __shared__ T ts[TY + 1][W], bsig[TY + 1][W], bdamp[TY + 1][W], bcx[TY + 1][W], bcy[TY + 1][W];
  __shared__ double eps_s;
  const int M = a.p.M, n = a.p.n;
  const int TX = M < PIX_TX ? M : PIX_TX, WW = TX + 2;
  const int tilesx = M / TX;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY, scene = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t img = (size_t)M * M;
  const double* sm = a.sums + (size_t)scene * img * 4;
  pdl_wait();
  if (warp == 0) {
    const double mx = warp_max_view_power(a.p.norms + (size_t)scene * n * a.p.CS, n, a.p.CS);
    if (lane == 0) eps_s = 1e-10 * mx / (double)img;   // cie.py:49-50
  }
  __syncthreads();
  const T eps = (T)eps_s;
  for (int h = tid; h < HR * WW; h += blockDim.x) {
    const int r = h / WW, cix = h % WW;
    const int yy = y0 - 1 + r, xx = x0 - 1 + cix;
    C<T> chi = czero<T>();
    if (yy >= 0 && yy < M && xx >= 0 && xx < M) {
      const double* s4 = sm + ((size_t)yy * M + xx) * 4;
      const T den = (T)s4[2] + eps;
      chi = mk<T>((T)s4[0] / den, (T)s4[1] / den);   // numpy complex / real division
    }
    chis[r][cix] = chi;
  }
  __syncthreads();
  const T tau = a.p.tau;
  for (int q = tid; q < (TY + 1) * WW; q += blockDim.x) {
    const int row = q / WW, cix = q % WW;
    const int yy = y0 - 1 + row, xx = x0 - 1 + cix;
    C<T> wx = czero<T>(), wy = czero<T>();
    T s_ = T(0), sig = T(0), damp = T(0), cx = T(0), cy = T(0);
    if (yy >= 0 && yy < M && xx >= 0 && xx < M) {
      const C<T> c = chis[row][cix];
      const C<T> dx = (xx + 1 < M) ? csub<T>(chis[row][cix + 1], c) : czero<T>();
      const C<T> dy = (yy + 1 < M) ? csub<T>(chis[row + 1][cix], c) : czero<T>();
      s_ = sqrt_<T>(cabs2<T>(dx) + cabs2<T>(dy) + T(EPS_TV));
      wx = mk<T>(dx.x / s_, dx.y / s_);
      wy = mk<T>(dy.x / s_, dy.y / s_);
      const T am = amag<T>(c);
      const T gx = (xx + 1 < M) ? amag<T>(chis[row][cix + 1]) - am : T(0);
      const T gy = (yy + 1 < M) ? amag<T>(chis[row + 1][cix]) - am : T(0);
      sig = sigmoid_<T>((am - tau) / tau);
      damp = exp_<T>(-(gx * gx + gy * gy));
      cx = T(-2) * sig * damp * gx;
      cy = T(-2) * sig * damp * gy;
    }
    twx[row][cix] = wx; twy[row][cix] = wy; ts[row][cix] = s_;
    bsig[row][cix] = sig; bdamp[row][cix] = damp; bcx[row][cix] = cx; bcy[row][cix] = cy;
  }
  __syncthreads();
  // pixel (row pr, column pc): one warp per image row of the tile (TY <= 4 warps)
  double vs = 0.0, vb_ = 0.0, vt = 0.0, vr = 0.0;
  C<T> fR = czero<T>(), fgn = czero<T>();   // the pixel's R and LS-quotient adjoint coefficients
  T fgd = T(0);
  const int pr = warp, pc = lane;
  if (pr < TY && pc < TX) {
    const int x = x0 + pc, y = y0 + pr, c1 = pc + 1, hr = pr + 1;
    const size_t p = (size_t)y * M + x;
    const C<T> chi = chis[hr][c1];
    const T neg = chi.x < T(0) ? chi.x : T(0);
    vb_ = (double)(neg * neg);
    vt = (double)ts[hr][c1];
    vr = (double)(bsig[hr][c1] * bdamp[hr][c1]);
    if (a.p.chi_out) a.p.chi_out[(size_t)scene * img + p] = chi;
    C<T> g = czero<T>();
    if (GRAD) {
      if (a.p.l1 != T(0)) g = cadd<T>(g, mk<T>(a.p.l1 * (T(2) * neg), T(0)));
      if (a.p.l2 != T(0)) {
        C<T> gt = mk<T>(-twx[hr][c1].x - twy[hr][c1].x, -twx[hr][c1].y - twy[hr][c1].y);
        if (x >= 1) gt = cadd<T>(gt, twx[hr][c1 - 1]);
        if (y >= 1) gt = cadd<T>(gt, twy[hr - 1][c1]);
        g = cadd<T>(g, cscale<T>(gt, a.p.l2));
      }
      if (a.p.l3 != T(0)) {
        const T sg = bsig[hr][c1];
        T ga = sg * (T(1) - sg) / tau * bdamp[hr][c1];
        ga -= bcx[hr][c1];
        ga -= bcy[hr][c1];
        if (x >= 1) ga += bcx[hr][c1 - 1];
        if (y >= 1) ga += bcy[hr - 1][c1];
        const T am = amag<T>(chi);
        const C<T> ph = am > T(0) ? mk<T>(chi.x / am, chi.y / am) : czero<T>();
        g = cadd<T>(g, cscale<T>(ph, a.p.l3 * ga));
      }
    }
    const T beta = a.p.beta;
    C<T> R_, chn;
    if (a.p.rfixed) {
      R_ = a.p.rfixed[(size_t)scene * img + p];
      chn = czero<T>();
    } else {
      const C<T> q = mk<T>(beta * chi.x + T(1), beta * chi.y);
      if (sqrt_<T>(cabs2<T>(q)) < T(1e-14)) atomicOr(&a.p.err[scene], ERR_POLE);
      R_ = cdiv<T>(mk<T>(beta * chi.x, beta * chi.y), q);
      chn = conj_<T>(cdiv<T>(mk<T>(beta, T(0)), cmul<T>(q, q)));   // conj(beta / q^2)
    }
    // closed forms over the views (header)
    const double* s4 = sm + p * 4;
    const C<T> num = mk<T>((T)s4[0], (T)s4[1]);
    const T den0 = (T)s4[2], cj = (T)s4[3];
    const T A = den0 + T(2) * beta * num.x + beta * beta * cj;
    const C<T> B = mk<T>(num.x + beta * cj, num.y);
    const T r2 = cabs2<T>(R_);
    vs = (double)(r2 * A - T(2) * beta * (R_.x * B.x + R_.y * B.y) + beta * beta * cj);
    if (GRAD) {
      const T gsc = T(2.0 / a.p.c_inc[scene]);
      const C<T> gr = cscale<T>(mk<T>(R_.x * A - beta * B.x, R_.y * A - beta * B.y), gsc);
      C<T> gchi = g;
      if (!a.p.rfixed) gchi = cadd<T>(gchi, cmul<T>(chn, gr));
      const T den = den0 + eps;
      fR = R_;
      fgn = mk<T>(gchi.x / den, gchi.y / den);
      fgd = -(gchi.x * chi.x + gchi.y * chi.y) / den;   // -Re(conj(g_chi) chi) / den
      if constexpr (!FUSE) {
        double* co = a.coef + ((size_t)scene * img + p) * 6;
        co[0] = (double)fR.x;
        co[1] = (double)fR.y;
        co[2] = (double)fgn.x;
        co[3] = (double)fgn.y;
        co[4] = (double)fgd;
      }
    }
  }
  pdl_trigger();
  if constexpr (GRAD && FUSE) {
    if (pr < TY && pc < TX) {
      const size_t pix = (size_t)(y0 + pr) * M + x0 + pc;
      const T beta = a.p.beta;
      const T gsc = T(2.0 / a.p.c_inc[scene]);
      auto one = [&](size_t o, C<T> j, C<T> e) {
        const C<T> P = mk<T>(e.x + beta * j.x, e.y + beta * j.y);
        const C<T> Sr = csub<T>(cmul<T>(fR, P), mk<T>(beta * j.x, beta * j.y));
        const C<T> gS = cscale<T>(Sr, gsc);
        const C<T> gP = cmul<T>(conj_<T>(fR), gS);
        C<T> gj = cscale<T>(csub<T>(gP, gS), beta);
        gj = cadd<T>(gj, cmul<T>(e, fgn));
        C<T> ge = cadd<T>(gP, cmul<T>(conj_<T>(fgn), j));
        ge = cadd<T>(ge, cscale<T>(e, T(2) * fgd));
        a.p.gJ[o] = gj;
        a.p.gE[o] = ge;
      };
      const size_t o0 = (size_t)scene * n * img + pix;
      int i = 0;
      for (; i + 3 < n; i += 4) {   // four views in flight per thread
        const size_t oa = o0 + (size_t)i * img, ob = oa + img, oc = ob + img, od = oc + img;
        const C<T> ja = a.p.J[oa], ea = a.p.E[oa], jb = a.p.J[ob], eb = a.p.E[ob];
        const C<T> jc = a.p.J[oc], ec = a.p.E[oc], jd = a.p.J[od], ed = a.p.E[od];
        one(oa, ja, ea);
        one(ob, jb, eb);
        one(oc, jc, ec);
        one(od, jd, ed);
      }
      for (; i < n; ++i) {
        const size_t oa = o0 + (size_t)i * img;
        one(oa, a.p.J[oa], a.p.E[oa]);
      }
    }
  }
  // loss partials per image row: a TX-lane tree over the row's pixels
  if (pr < TY) {
    for (int o = TX / 2; o >= 1; o >>= 1) {
      vs += __shfl_xor_sync(0xffffffffu, vs, o);
      vb_ += __shfl_xor_sync(0xffffffffu, vb_, o);
      vt += __shfl_xor_sync(0xffffffffu, vt, o);
      vr += __shfl_xor_sync(0xffffffffu, vr, o);
    }
    if (lane == 0) {
      const int tile = (y0 + pr) * tilesx + blockIdx.x;
      double* o4 = a.p.part + ((size_t)scene * (tilesx * M) + tile) * 4;
      o4[0] = vs; o4[1] = vb_; o4[2] = vt; o4[3] = vr;
    }
  }
  if constexpr (FUSE) tl_mark(a.p.tl, 2);
}

// thread = pixel, grid.y = group of up to PG_VIEWS views, grid.z = scene
constexpr int PG_VIEWS = 16;
template <typename T>
__global__ void __launch_bounds__(256) pix_grad_kernel(PixStreamArgs<T> a) {
  const int n = a.p.n, scene = blockIdx.z;
  const size_t img = (size_t)a.p.M * a.p.M;
  const size_t pix = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  pdl_wait();
  if (pix >= img) return;
  const double* co = a.coef + ((size_t)scene * img + pix) * 6;
  const C<T> R_ = mk<T>((T)co[0], (T)co[1]);
  const C<T> gn = mk<T>((T)co[2], (T)co[3]);
  const T gd = (T)co[4];
  const T beta = a.p.beta;
  const T gsc = T(2.0 / a.p.c_inc[scene]);
  const int i0 = blockIdx.y * PG_VIEWS, i1 = min(n, i0 + PG_VIEWS);
  auto one = [&](size_t o, C<T> j, C<T> e) {
    const C<T> P = mk<T>(e.x + beta * j.x, e.y + beta * j.y);
    const C<T> Sr = csub<T>(cmul<T>(R_, P), mk<T>(beta * j.x, beta * j.y));
    const C<T> gS = cscale<T>(Sr, gsc);
    const C<T> gP = cmul<T>(conj_<T>(R_), gS);
    C<T> gj = cscale<T>(csub<T>(gP, gS), beta);
    gj = cadd<T>(gj, cmul<T>(e, gn));
    C<T> ge = cadd<T>(gP, cmul<T>(conj_<T>(gn), j));
    ge = cadd<T>(ge, cscale<T>(e, T(2) * gd));
    a.p.gJ[o] = gj;
    a.p.gE[o] = ge;
  };
  int i = i0;
  for (; i + 1 < i1; i += 2) {   // two views in flight
    const size_t o0 = ((size_t)scene * n + i) * img + pix, o1 = o0 + img;
    const C<T> j0 = a.p.J[o0], e0 = a.p.E[o0], j1 = a.p.J[o1], e1 = a.p.E[o1];
    one(o0, j0, e0);
    one(o1, j1, e1);
  }
  if (i < i1) {
    const size_t o0 = ((size_t)scene * n + i) * img + pix;
    one(o0, a.p.J[o0], a.p.E[o0]);
  }
  tl_mark(a.p.tl, 2);
}

}  // namespace pdf
