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

// CTA = one scene, TY image rows y0 .. y0+TY-1, TX consecutive columns; lane
// = column inside the tile (coalesced row segments), warp w handles views
// w, w + nw, ...  One load pass per view brings the TY + 2 halo rows (plus
// the two edge columns) into registers: the halo rows feed the per-pixel
// num / den sums, the TY inner rows of the first VC views of each warp stay
// in registers for the state and gradient passes (views beyond VC * nw are
// re-read from L2).  TY > 1 shares the halo rows between output rows (batch
// regime: halo read amplification (TY + 2) / TY instead of 3).  Every sum
// over views runs in increasing view order per warp, then in warp order, and
// every loss partial is per image row, so results do not depend on TY / VC.
template <typename T, bool GRAD, int TY, int VC>
__global__ void __launch_bounds__(PIX_NW * 32) pixel_kernel(PixelArgs<T> a) {
  constexpr int W = PIX_TX + 2;
  constexpr int HR = TY + 2;                 // halo rows
  // per-warp halo partials, dead once chi is formed: the R-chain partials reuse the space
  constexpr size_t PART_B = sizeof(C<T>) * PIX_NW * HR * W + sizeof(T) * PIX_NW * HR * W;
  constexpr size_t PGR_B = sizeof(C<T>) * PIX_NW * TY * PIX_TX;
  __shared__ __align__(16) unsigned char scratch[PART_B > PGR_B ? PART_B : PGR_B];
  auto pnum = reinterpret_cast<C<T>(*)[HR][W]>(scratch);
  auto pden = reinterpret_cast<T(*)[HR][W]>(scratch + sizeof(C<T>) * PIX_NW * HR * W);
  auto pgr = reinterpret_cast<C<T>(*)[TY][PIX_TX]>(scratch);
  __shared__ C<T> chis[HR][W];
  // stencil terms for halo rows 0 .. TY (image rows y0-1 .. y0+TY-1) over columns x0-1 .. x0+TX
  __shared__ C<T> twx[TY + 1][W], twy[TY + 1][W];   // tv weights dx/s, dy/s
  __shared__ T ts[TY + 1][W];                       // tv value s
  __shared__ T bsig[TY + 1][W], bdamp[TY + 1][W], bcx[TY + 1][W], bcy[TY + 1][W];
  __shared__ T dens[TY][PIX_TX];
  __shared__ C<T> Rs[TY][PIX_TX], chain[TY][PIX_TX], greg[TY][PIX_TX], gnum[TY][PIX_TX];
  __shared__ T gden[TY][PIX_TX];
  __shared__ double red[PIX_NW][TY][4];
  __shared__ double rgp[TY][3];
  __shared__ double eps_s;

  const int M = a.M, n = a.n;
  const int TX = M < PIX_TX ? M : PIX_TX;
  const int WW = TX + 2;
  const int tilesx = M / TX;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY, scene = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const size_t img = (size_t)M * M;
  const size_t vbase = (size_t)scene * n;
  const bool col_ok = lane < TX;
  // edge entries: lane e < 2 HR loads halo row e / 2, column x0 - 1 (e even) or x0 + TX (e odd)
  const int erow = lane >> 1, eside = lane & 1;
  const int ex = eside ? x0 + TX : x0 - 1, ey = y0 - 1 + erow;
  const bool e_ok = lane < 2 * HR && ex >= 0 && ex < M && ey >= 0 && ey < M;
  const size_t epix = e_ok ? (size_t)ey * M + ex : 0;
  bool r_ok[HR];
  size_t rpix[HR];
#pragma unroll
  for (int r = 0; r < HR; ++r) {
    const int yy = y0 - 1 + r;
    r_ok[r] = col_ok && yy >= 0 && yy < M;
    rpix[r] = r_ok[r] ? (size_t)yy * M + x0 + lane : 0;
  }

  tl_mark(a.tl, 0);
  pdl_wait();   // J, E, norms come from the previous kernel
  tl_mark(a.tl, 1);

  if (warp == 0) {
    const double mx = warp_max_view_power(a.norms + vbase * a.CS, n, a.CS);
    if (lane == 0) eps_s = 1e-10 * mx / (double)img;   // cie.py:49-50
  }

  // ---- halo pass: per-warp partial num / den, inner rows cached ------------
  C<T> jc[VC][TY], ec[VC][TY];
  {
    C<T> num[HR], nume = czero<T>();
    T den[HR], dene = T(0);
#pragma unroll
    for (int r = 0; r < HR; ++r) { num[r] = czero<T>(); den[r] = T(0); }
    auto view_pass = [&](int i, C<T>* jin, C<T>* ein) {
      C<T> j[HR], e[HR], je, ee;
      const size_t vo = (vbase + i) * img;
#pragma unroll
      for (int r = 0; r < HR; ++r) {
        j[r] = r_ok[r] ? a.J[vo + rpix[r]] : czero<T>();
        e[r] = r_ok[r] ? a.E[vo + rpix[r]] : czero<T>();
      }
      je = e_ok ? a.J[vo + epix] : czero<T>();
      ee = e_ok ? a.E[vo + epix] : czero<T>();
#pragma unroll
      for (int r = 0; r < HR; ++r) {
        num[r] = cadd<T>(num[r], cmulc<T>(j[r], e[r]));
        den[r] += cabs2<T>(e[r]);
      }
      nume = cadd<T>(nume, cmulc<T>(je, ee));
      dene += cabs2<T>(ee);
      if (jin) {
#pragma unroll
        for (int r = 0; r < TY; ++r) { jin[r] = j[r + 1]; ein[r] = e[r + 1]; }
      }
    };
#pragma unroll
    for (int vb = 0; vb < VC; ++vb) {
      const int i = warp + vb * nw;
      if (i < n) view_pass(i, jc[vb], ec[vb]);
    }
#pragma unroll 2
    for (int i = warp + VC * nw; i < n; i += nw) view_pass(i, nullptr, nullptr);
#pragma unroll
    for (int r = 0; r < HR; ++r)
      if (col_ok) { pnum[warp][r][lane + 1] = num[r]; pden[warp][r][lane + 1] = den[r]; }
    if (lane < 2 * HR) {
      const int c = eside ? TX + 1 : 0;
      pnum[warp][erow][c] = nume;
      pden[warp][erow][c] = dene;
    }
  }
  __syncthreads();
  tl_stage(a.tl, 0);
  const T eps = (T)eps_s;
  for (int h = tid; h < HR * WW; h += blockDim.x) {
    const int r = h / WW, cix = h % WW;
    C<T> num = czero<T>();
    T den = T(0);
    for (int w = 0; w < nw; ++w) { num = cadd<T>(num, pnum[w][r][cix]); den += pden[w][r][cix]; }
    den += eps;
    chis[r][cix] = mk<T>(num.x / den, num.y / den);   // numpy complex/real division
    if (r >= 1 && r <= TY && cix >= 1 && cix <= TX) dens[r - 1][cix - 1] = den;
  }
  __syncthreads();
  tl_stage(a.tl, 1);

  // ---- stencil terms at halo rows 0 .. TY (forward differences, losses.py:139-144)
  const T tau = a.tau;
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
  tl_stage(a.tl, 2);

  // ---- per-pixel scalar work ------------------------------------------------
  double vb_ = 0.0, vt = 0.0, vr = 0.0;
  const int pr = tid / TX, pc = tid % TX;          // pixel (row pr, column pc) of thread tid < TY TX
  if (tid < TY * TX) {
    const int x = x0 + pc, y = y0 + pr, c1 = pc + 1, hr = pr + 1;
    const C<T> chi = chis[hr][c1];
    const T neg = chi.x < T(0) ? chi.x : T(0);
    vb_ = (double)(neg * neg);
    vt = (double)ts[hr][c1];
    vr = (double)(bsig[hr][c1] * bdamp[hr][c1]);
    if (a.chi_out) a.chi_out[(size_t)scene * img + (size_t)y * M + x] = chi;
    if (GRAD) {
      C<T> g = czero<T>();
      if (a.l1 != T(0)) g = cadd<T>(g, mk<T>(a.l1 * (T(2) * neg), T(0)));
      if (a.l2 != T(0)) {
        // g += wx(y, x-1) - wx(y, x) + wy(y-1, x) - wy(y, x)   (losses.py:156-165)
        C<T> gt = mk<T>(-twx[hr][c1].x - twy[hr][c1].x, -twx[hr][c1].y - twy[hr][c1].y);
        if (x >= 1) gt = cadd<T>(gt, twx[hr][c1 - 1]);
        if (y >= 1) gt = cadd<T>(gt, twy[hr - 1][c1]);
        g = cadd<T>(g, cscale<T>(gt, a.l2));
      }
      if (a.l3 != T(0)) {
        // (losses.py:168-182)
        const T sg = bsig[hr][c1];
        T ga = sg * (T(1) - sg) / tau * bdamp[hr][c1];
        ga -= bcx[hr][c1];
        ga -= bcy[hr][c1];
        if (x >= 1) ga += bcx[hr][c1 - 1];
        if (y >= 1) ga += bcy[hr - 1][c1];
        const T am = amag<T>(chi);
        const C<T> ph = am > T(0) ? mk<T>(chi.x / am, chi.y / am) : czero<T>();
        g = cadd<T>(g, cscale<T>(ph, a.l3 * ga));
      }
      greg[pr][pc] = g;
    }
    C<T> R_;
    if (a.rfixed) {
      R_ = a.rfixed[(size_t)scene * img + (size_t)y * M + x];
      chain[pr][pc] = czero<T>();
    } else {
      const C<T> q = mk<T>(a.beta * chi.x + T(1), a.beta * chi.y);
      if (sqrt_<T>(cabs2<T>(q)) < T(1e-14)) atomicOr(&a.err[scene], ERR_POLE);
      R_ = cdiv<T>(mk<T>(a.beta * chi.x, a.beta * chi.y), q);
      chain[pr][pc] = conj_<T>(cdiv<T>(mk<T>(a.beta, T(0)), cmul<T>(q, q)));   // conj(beta / q^2)
    }
    Rs[pr][pc] = R_;
  }
  __syncthreads();
  tl_stage(a.tl, 3);

  // ---- state residual, R-chain partial ------------------------------------
  const T beta = a.beta;
  const T gsc = T(2.0 / a.c_inc[scene]);
  double vs[TY];
#pragma unroll
  for (int r = 0; r < TY; ++r) vs[r] = 0.0;
  if (col_ok) {
    C<T> R_[TY], gr[TY];
#pragma unroll
    for (int r = 0; r < TY; ++r) { R_[r] = Rs[r][lane]; gr[r] = czero<T>(); }
    auto state_view = [&](const C<T>* jv, const C<T>* ev) {
#pragma unroll
      for (int r = 0; r < TY; ++r) {
        const C<T> P = mk<T>(ev[r].x + beta * jv[r].x, ev[r].y + beta * jv[r].y);
        const C<T> Sr = csub<T>(cmul<T>(R_[r], P), mk<T>(beta * jv[r].x, beta * jv[r].y));
        vs[r] += (double)cabs2<T>(Sr);
        if (GRAD) gr[r] = cadd<T>(gr[r], cmulc<T>(cscale<T>(Sr, gsc), P));   // conj(P) g_S
      }
    };
#pragma unroll
    for (int vb = 0; vb < VC; ++vb)
      if (warp + vb * nw < n) state_view(jc[vb], ec[vb]);
    for (int i = warp + VC * nw; i < n; i += nw) {
      C<T> j[TY], e[TY];
#pragma unroll
      for (int r = 0; r < TY; ++r) {
        const size_t o = (vbase + i) * img + rpix[r + 1];
        j[r] = a.J[o];
        e[r] = a.E[o];
      }
      state_view(j, e);
    }
    if (GRAD) {
#pragma unroll
      for (int r = 0; r < TY; ++r) pgr[warp][r][lane] = gr[r];
    }
  }
  pdl_trigger();
  if (GRAD) {
    __syncthreads();
    tl_stage(a.tl, 4);
    if (tid < TY * TX) {
      C<T> gr = czero<T>();
      for (int w = 0; w < nw; ++w) gr = cadd<T>(gr, pgr[w][pr][pc]);
      const C<T> chi = chis[pr + 1][pc + 1];
      C<T> gchi = greg[pr][pc];
      if (!a.rfixed) gchi = cadd<T>(gchi, cmul<T>(chain[pr][pc], gr));
      const T den = dens[pr][pc];
      gnum[pr][pc] = mk<T>(gchi.x / den, gchi.y / den);
      gden[pr][pc] = -(gchi.x * chi.x + gchi.y * chi.y) / den;   // -Re(conj(g_chi) chi)/den
    }
    __syncthreads();
    tl_stage(a.tl, 5);
    if (col_ok) {
      C<T> R_[TY], gn[TY];
      T gd[TY];
#pragma unroll
      for (int r = 0; r < TY; ++r) { R_[r] = Rs[r][lane]; gn[r] = gnum[r][lane]; gd[r] = gden[r][lane]; }
      auto grad_view = [&](int i, const C<T>* jv, const C<T>* ev) {
#pragma unroll
        for (int r = 0; r < TY; ++r) {
          const size_t o = (vbase + i) * img + rpix[r + 1];
          const C<T> j = jv[r], e = ev[r];
          const C<T> P = mk<T>(e.x + beta * j.x, e.y + beta * j.y);
          const C<T> Sr = csub<T>(cmul<T>(R_[r], P), mk<T>(beta * j.x, beta * j.y));
          const C<T> gS = cscale<T>(Sr, gsc);
          const C<T> gP = cmul<T>(conj_<T>(R_[r]), gS);
          C<T> gj = cscale<T>(csub<T>(gP, gS), beta);
          gj = cadd<T>(gj, cmul<T>(e, gn[r]));
          C<T> ge = cadd<T>(gP, cmul<T>(conj_<T>(gn[r]), j));
          ge = cadd<T>(ge, cscale<T>(e, T(2) * gd[r]));
          a.gJ[o] = gj;
          a.gE[o] = ge;
        }
      };
#pragma unroll
      for (int vb = 0; vb < VC; ++vb) {
        const int i = warp + vb * nw;
        if (i < n) grad_view(i, jc[vb], ec[vb]);
      }
      for (int i = warp + VC * nw; i < n; i += nw) {
        C<T> j[TY], e[TY];
#pragma unroll
        for (int r = 0; r < TY; ++r) {
          const size_t o = (vbase + i) * img + rpix[r + 1];
          j[r] = a.J[o];
          e[r] = a.E[o];
        }
        grad_view(i, j, e);
      }
    }
  }

  tl_stage(a.tl, 6);
  // ---- loss partials per image row (fixed order) --------------------------
  // state: per lane over its warp's views, warp_sum, then warps in order;
  // bound / tv / bridge: a TX-lane tree over the row's pixels (threads
  // r TX .. r TX + TX - 1 hold row r), so a row's partial is the same for any TY
#pragma unroll
  for (int r = 0; r < TY; ++r) {
    const double v0 = warp_sum<double>(vs[r]);
    if (lane == 0) red[warp][r][0] = v0;
  }
  {
    double b1 = vb_, t1 = vt, r1 = vr;
    for (int o = TX / 2; o >= 1; o >>= 1) {
      b1 += __shfl_xor_sync(0xffffffffu, b1, o);
      t1 += __shfl_xor_sync(0xffffffffu, t1, o);
      r1 += __shfl_xor_sync(0xffffffffu, r1, o);
    }
    if (tid < TY * TX && pc == 0) { rgp[pr][0] = b1; rgp[pr][1] = t1; rgp[pr][2] = r1; }
  }
  __syncthreads();
  if (tid < TY * 4) {
    const int r = tid >> 2, k = tid & 3;
    double s_ = 0.0;
    if (k == 0) {
      for (int w = 0; w < nw; ++w) s_ += red[w][r][0];
    } else {
      s_ = rgp[r][k - 1];
    }
    const int tile = (y0 + r) * tilesx + blockIdx.x;
    a.part[((size_t)scene * (tilesx * M) + tile) * 4 + k] = s_;
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
