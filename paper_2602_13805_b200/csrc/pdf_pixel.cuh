// Per-pixel kernel of the PDF hot path: everything between the forward and
// the adjoint G_D convolutions that couples the incidences at one pixel.
//
//   chi = sum_i J_i conj(E_i) / (sum_i |E_i|^2 + eps_reg)   cie.py:66-80
//   R   = beta chi / (beta chi + 1), pole check             cie.py:24-30
//   P = E + beta J, S = R P - beta J, ||S||^2               losses.py:225-227
//   bound / tv / bridge values and chi-gradients            losses.py:115-195
//   reverse pass (losses.py:279-300):
//     g_S = 2S/c_inc, g_P = conj(R) g_S, g_J = beta (g_P - g_S) + G_S^H g_rows
//     g_chi = g_reg + conj(beta/(beta chi+1)^2) sum_i conj(P_i) g_S_i
//     g_num = g_chi/den, g_den = -Re(conj(g_chi) chi)/den
//     g_J += E g_num, g_E = g_P + conj(g_num) J + 2 g_den E
//
// CTA = one scene, one image row y, TX consecutive columns.  Warp w handles
// incidences i = w, w+NW, ...; lane = column inside the tile, so every global
// access is a coalesced row segment.  The regulariser stencils need chi on a
// one-pixel halo, which the CTA recomputes (rows y-1..y+1) instead of a
// separate launch.  All cross-view sums are fixed-order (deterministic).
#pragma once
#include "pdf_common.cuh"

namespace pdf {

template <typename T>
struct PixelArgs {
  int M, n, R, CS, S;
  T beta, l1, l2, l3, tau;
  const C<T>* J;        // [S*n][M][M]
  const C<T>* E;        // [S*n][M][M]
  const double* norms;  // [S*n][CS]
  const C<T>* grows;    // [S*n][R]
  const C<T>* gs;       // [R][M*M]
  const C<T>* rfixed;   // [S][M][M] or null
  const double* c_inc;  // [S]
  C<T>* gJ;             // [S*n][M][M]  (g_J local part)
  C<T>* gE;             // [S*n][M][M]
  double* part;         // [S][ntiles][4]  state, bound, tv, bridge
  C<T>* chi_out;        // [S][M][M] or null
  int* err;             // [S]
};

constexpr double EPS_TV = 1e-12;   // losses.py:29

template <typename T>
struct Nb {  // chi at a 3-row halo of the tile; NaN-free "outside" handled by flags
  const C<T>* chi;
  int W, x0, y, M;
  __device__ C<T> at(int yy, int xx) const {
    return chi[(yy - y + 1) * W + (xx - x0 + 1)];
  }
};

template <typename T>
__device__ inline void tv_terms(const Nb<T>& nb, int yy, int xx, C<T>& dx, C<T>& dy, T& s) {
  const int M = nb.M;
  const C<T> c = nb.at(yy, xx);
  dx = (xx + 1 < M) ? csub<T>(nb.at(yy, xx + 1), c) : czero<T>();
  dy = (yy + 1 < M) ? csub<T>(nb.at(yy + 1, xx), c) : czero<T>();
  s = sqrt_<T>(cabs2<T>(dx) + cabs2<T>(dy) + T(EPS_TV));
}

template <typename T>
__device__ inline T amag(C<T> z) { return sqrt_<T>(cabs2<T>(z)); }

template <typename T>
__device__ inline void bridge_terms(const Nb<T>& nb, int yy, int xx, T tau, T& sig, T& damp, T& gx, T& gy) {
  const int M = nb.M;
  const T a = amag<T>(nb.at(yy, xx));
  gx = (xx + 1 < M) ? amag<T>(nb.at(yy, xx + 1)) - a : T(0);
  gy = (yy + 1 < M) ? amag<T>(nb.at(yy + 1, xx)) - a : T(0);
  sig = sigmoid_<T>((a - tau) / tau);
  damp = exp_<T>(-(gx * gx + gy * gy));
}

template <typename T, bool GRAD>
__global__ void __launch_bounds__(256) pixel_kernel(PixelArgs<T> a) {
  constexpr int MAXTX = 32;
  constexpr int MAXW = 8;
  __shared__ C<T> pnum[MAXW][3 * (MAXTX + 2)];
  __shared__ T pden[MAXW][3 * (MAXTX + 2)];
  __shared__ C<T> chis[3 * (MAXTX + 2)];
  __shared__ T dens[MAXTX];
  __shared__ C<T> Rs[MAXTX], chain[MAXTX], greg[MAXTX], gnum[MAXTX];
  __shared__ T gden[MAXTX];
  __shared__ C<T> pgr[MAXW][MAXTX];
  __shared__ double red[MAXW][4];
  __shared__ double eps_s;

  const int M = a.M, n = a.n;
  const int TX = M < MAXTX ? M : MAXTX;
  const int W = TX + 2;
  const int NH = 3 * W;
  const int tilesx = M / TX;
  const int x0 = blockIdx.x * TX, y = blockIdx.y, scene = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const size_t img = (size_t)M * M;
  const size_t vbase = (size_t)scene * n;

  if (tid == 0) {
    double mx = 0.0;
    for (int i = 0; i < n; ++i) {
      double pw = 0.0;
      for (int c = 0; c < a.CS; ++c) pw += a.norms[(vbase + i) * a.CS + c];
      mx = i == 0 ? pw : (pw > mx ? pw : mx);
    }
    eps_s = 1e-10 * mx / (double)img;               // cie.py:49-50
  }

  // ---- per-warp partial num/den on the halo --------------------------------
  for (int h = lane; h < NH; h += 32) {
    const int hy = y - 1 + h / W, hx = x0 - 1 + h % W;
    C<T> num = czero<T>();
    T den = T(0);
    if (hy >= 0 && hy < M && hx >= 0 && hx < M) {
      const size_t pix = (size_t)hy * M + hx;
      for (int i = warp; i < n; i += nw) {
        const C<T> j = a.J[(vbase + i) * img + pix];
        const C<T> e = a.E[(vbase + i) * img + pix];
        num = cadd<T>(num, cmulc<T>(j, e));
        den += cabs2<T>(e);
      }
    }
    pnum[warp][h] = num;
    pden[warp][h] = den;
  }
  __syncthreads();
  const T eps = (T)eps_s;
  for (int h = tid; h < NH; h += blockDim.x) {
    C<T> num = czero<T>();
    T den = T(0);
    for (int w = 0; w < nw; ++w) { num = cadd<T>(num, pnum[w][h]); den += pden[w][h]; }
    den += eps;
    chis[h] = mk<T>(num.x / den, num.y / den);   // numpy complex/real division
    if (h / W == 1 && (h % W) >= 1 && (h % W) <= TX) dens[h % W - 1] = den;
  }
  __syncthreads();

  // ---- per-pixel scalar work (warp 0) -------------------------------------
  double vb = 0.0, vt = 0.0, vr = 0.0;
  if (warp == 0 && lane < TX) {
    const int x = x0 + lane;
    Nb<T> nb{chis, W, x0, y, M};
    const C<T> chi = nb.at(y, x);
    const T tau = a.tau;
    // values (losses.py:115-136)
    const T neg = chi.x < T(0) ? chi.x : T(0);
    vb = (double)(neg * neg);
    C<T> dx, dy; T s;
    tv_terms<T>(nb, y, x, dx, dy, s);
    vt = (double)s;
    T sig, damp, gx, gy;
    bridge_terms<T>(nb, y, x, tau, sig, damp, gx, gy);
    vr = (double)(sig * damp);
    if (a.chi_out) a.chi_out[(size_t)scene * img + (size_t)y * M + x] = chi;
    if (GRAD) {
      C<T> g = czero<T>();
      if (a.l1 != T(0)) g = cadd<T>(g, mk<T>(a.l1 * (T(2) * neg), T(0)));
      if (a.l2 != T(0)) {
        C<T> gt = mk<T>(-dx.x / s - dy.x / s, -dx.y / s - dy.y / s);
        if (x >= 1) {
          C<T> dx2, dy2; T s2;
          tv_terms<T>(nb, y, x - 1, dx2, dy2, s2);
          gt = cadd<T>(gt, mk<T>(dx2.x / s2, dx2.y / s2));
        }
        if (y >= 1) {
          C<T> dx2, dy2; T s2;
          tv_terms<T>(nb, y - 1, x, dx2, dy2, s2);
          gt = cadd<T>(gt, mk<T>(dy2.x / s2, dy2.y / s2));
        }
        g = cadd<T>(g, cscale<T>(gt, a.l2));
      }
      if (a.l3 != T(0)) {
        T ga = sig * (T(1) - sig) / tau * damp;
        ga -= T(-2) * sig * damp * gx;
        ga -= T(-2) * sig * damp * gy;
        if (x >= 1) {
          T s2, d2, gx2, gy2;
          bridge_terms<T>(nb, y, x - 1, tau, s2, d2, gx2, gy2);
          ga += T(-2) * s2 * d2 * gx2;
        }
        if (y >= 1) {
          T s2, d2, gx2, gy2;
          bridge_terms<T>(nb, y - 1, x, tau, s2, d2, gx2, gy2);
          ga += T(-2) * s2 * d2 * gy2;
        }
        const T am = amag<T>(chi);
        C<T> ph = am > T(0) ? mk<T>(chi.x / am, chi.y / am) : czero<T>();
        g = cadd<T>(g, cscale<T>(ph, a.l3 * ga));
      }
      greg[lane] = g;
    }
    C<T> R;
    if (a.rfixed) {
      R = a.rfixed[(size_t)scene * img + (size_t)y * M + x];
      chain[lane] = czero<T>();
    } else {
      const C<T> q = mk<T>(a.beta * chi.x + T(1), a.beta * chi.y);
      if (sqrt_<T>(cabs2<T>(q)) < T(1e-14)) atomicOr(&a.err[scene], ERR_POLE);
      R = cdiv<T>(mk<T>(a.beta * chi.x, a.beta * chi.y), q);
      // conj(beta / q^2)
      const C<T> q2 = cmul<T>(q, q);
      chain[lane] = conj_<T>(cdiv<T>(mk<T>(a.beta, T(0)), q2));
    }
    Rs[lane] = R;
  }
  __syncthreads();

  // ---- state residual, R-chain partial ------------------------------------
  const T beta = a.beta;
  const T gsc = T(2.0 / a.c_inc[scene]);
  double vs = 0.0;
  if (lane < TX) {
    const int x = x0 + lane;
    const size_t pix = (size_t)y * M + x;
    const C<T> R = Rs[lane];
    C<T> gr = czero<T>();
    for (int i = warp; i < n; i += nw) {
      const C<T> j = a.J[(vbase + i) * img + pix];
      const C<T> e = a.E[(vbase + i) * img + pix];
      const C<T> P = mk<T>(e.x + beta * j.x, e.y + beta * j.y);
      const C<T> Sr = csub<T>(cmul<T>(R, P), mk<T>(beta * j.x, beta * j.y));
      vs += (double)cabs2<T>(Sr);
      if (GRAD) gr = cadd<T>(gr, cmulc<T>(cscale<T>(Sr, gsc), P));   // conj(P) g_S
    }
    if (GRAD) pgr[warp][lane] = gr;
  }
  if (GRAD) {
    __syncthreads();
    if (warp == 0 && lane < TX) {
      C<T> gr = czero<T>();
      for (int w = 0; w < nw; ++w) gr = cadd<T>(gr, pgr[w][lane]);
      const C<T> chi = chis[W + 1 + lane];
      C<T> gchi = greg[lane];
      if (!a.rfixed) gchi = cadd<T>(gchi, cmul<T>(chain[lane], gr));
      const T den = dens[lane];
      gnum[lane] = mk<T>(gchi.x / den, gchi.y / den);
      gden[lane] = -(gchi.x * chi.x + gchi.y * chi.y) / den;   // -Re(conj(g_chi) chi)/den
    }
    __syncthreads();
    if (lane < TX) {
      const int x = x0 + lane;
      const size_t pix = (size_t)y * M + x;
      const C<T> R = Rs[lane];
      const C<T> gn = gnum[lane];
      const T gd = gden[lane];
      for (int i = warp; i < n; i += nw) {
        const size_t o = (vbase + i) * img + pix;
        const C<T> j = a.J[o];
        const C<T> e = a.E[o];
        const C<T> P = mk<T>(e.x + beta * j.x, e.y + beta * j.y);
        const C<T> Sr = csub<T>(cmul<T>(R, P), mk<T>(beta * j.x, beta * j.y));
        const C<T> gS = cscale<T>(Sr, gsc);
        const C<T> gP = cmul<T>(conj_<T>(R), gS);
        C<T> gj = cscale<T>(csub<T>(gP, gS), beta);
        // G_S^H g_rows at this pixel (forward.py:303-306)
        const C<T>* gr = a.grows + (vbase + i) * a.R;
        C<T> acc = czero<T>();
        for (int r = 0; r < a.R; ++r) acc = cadd<T>(acc, cmulc<T>(gr[r], a.gs[(size_t)r * img + pix]));
        gj = cadd<T>(gj, acc);
        gj = cadd<T>(gj, cmul<T>(e, gn));
        C<T> ge = cadd<T>(gP, cmul<T>(conj_<T>(gn), j));
        ge = cadd<T>(ge, cscale<T>(e, T(2) * gd));
        a.gJ[o] = gj;
        a.gE[o] = ge;
      }
    }
  }

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

__global__ void finalize_kernel(FinalizeArgs a) {
  const int scene = blockIdx.x;
  __shared__ double red[32][4];
  const int tid = threadIdx.x;
  double s[4] = {0, 0, 0, 0};
  for (int t = tid; t < a.ntiles; t += blockDim.x)
    for (int k = 0; k < 4; ++k) s[k] += a.part[((size_t)scene * a.ntiles + t) * 4 + k];
  // deterministic: fixed blockDim, fixed strides, fixed tree
  for (int k = 0; k < 4; ++k) s[k] = warp_sum<double>(s[k]);
  if ((tid & 31) == 0) for (int k = 0; k < 4; ++k) red[tid >> 5][k] = s[k];
  __syncthreads();
  if (tid == 0) {
    double st = 0, bo = 0, tv = 0, br = 0, da = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { st += red[w][0]; bo += red[w][1]; tv += red[w][2]; br += red[w][3]; }
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

}  // namespace pdf
