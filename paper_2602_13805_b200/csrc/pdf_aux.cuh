// Operator primitives and one-time kernels around the hot loop:
// expand / truncate (spectral.py:56-79), G_S products (forward.py:303-306,
// losses.py:229), the contrast-compensation epilogue (filters.py:16-67) and
// the kernel-spectrum permutation used by the view FFT.
#pragma once
#include "pdf_common.cuh"

namespace pdf {

__device__ inline int bitrev5(int l) { return __brev((unsigned)l) >> 27; }

// khat_p[pos_c * P + pos_r] = khat[f(pos_r)][f(pos_c)] / P^2, f(q*32+l) = spectrum_slot_freq(l, q, E);
// split (large-grid path): pos = h * P/2 + q*32 + l holds frequency 2 f_{E/2}(q*32+l) + h
__device__ inline int khat_pos_freq(int pos, int P, int split) {
  const int E = P / 32;
  if (!split) return spectrum_slot_freq(pos % 32, pos / 32, E);
  const int h = pos / (P / 2), r = pos % (P / 2);
  return 2 * spectrum_slot_freq(r % 32, r / 32, E / 2) + h;
}

// ---------------------------------------------------------------------------
// Spectral receiver operator H = G_S o expand (built once per geometry).
// expand (spectral.py:68-79) is linear, J = sum_m alpha[m] phi_m with
// phi_m(y, x) = exp(+2 pi i (f_u y + f_w x) / M) / M^2, so the data residual
// of the loss (losses.py:229-232) is
//     D[v][r] = sum_p J[v][p] G_S[r][p] = sum_m alpha[v][m] H[r][m],
//     H[r][m] = sum_p G_S[r][p] phi_m(p)                (R x M0, slot order)
// and its adjoint contribution to g_alpha (forward.py:303-306 followed by
// truncate / (m1 m2), spectral.py:56-65, losses.py:288,306) is
//     g_alpha[v][m] += sum_r g_rows[v][r] conj(H[r][m]).
// The hot loop then never touches the R x M^2 receiver matrix.  Built in
// float64 with fixed-order sums: stage 1 contracts x, stage 2 contracts y.
__device__ __forceinline__ int spec_corner_freq(int u, int mf, int M) { return u < mf ? u : M - 2 * mf + u; }

template <typename T>
__global__ void hs_rows_kernel(const C<T>* gs, double2* t1, int M, int mf, int R) {
  // t1[r][y][w] = sum_x G_S[r][y M + x] exp(+2 pi i f_w x / M)
  const int K = 2 * mf;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)R * M * K) return;
  const int w = (int)(idx % K), y = (int)((idx / K) % M), r = (int)(idx / ((long long)K * M));
  const int f = spec_corner_freq(w, mf, M);
  const C<T>* g = gs + (size_t)r * M * M + (size_t)y * M;
  double sr = 0.0, si = 0.0;
  for (int x = 0; x < M; ++x) {
    double s, c;
    sincospi(2.0 * (double)((f * x) % M) / (double)M, &s, &c);
    const double gr = (double)g[x].x, gi = (double)g[x].y;
    sr += gr * c - gi * s;
    si += gr * s + gi * c;
  }
  t1[idx] = make_double2(sr, si);
}

template <typename T>
__global__ void hs_cols_kernel(const double2* t1, C<T>* hs, int M, int mf, int R) {
  // H[r][slot(u, w)] = sum_y t1[r][y][w] exp(+2 pi i f_u y / M) / M^2
  const int K = 2 * mf, M0 = K * K;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= R * M0) return;
  const int r = idx / M0, i = idx % M0, u = i / K, w = i % K;
  const int f = spec_corner_freq(u, mf, M);
  double sr = 0.0, si = 0.0;
  for (int y = 0; y < M; ++y) {
    double s, c;
    sincospi(2.0 * (double)((f * y) % M) / (double)M, &s, &c);
    const double2 v = t1[((size_t)r * M + y) * K + w];
    sr += v.x * c - v.y * s;
    si += v.x * s + v.y * c;
  }
  const double inv = 1.0 / ((double)M * (double)M);
  const int slot = (((u / mf) * 2 + (w / mf)) * mf + (u % mf)) * mf + (w % mf);   // spectral.py:29-44
  hs[(size_t)r * M0 + slot] = mk<T>((T)(sr * inv), (T)(si * inv));
}

// sum_r g_rows[r] conj(H[r][slot]) over receivers r0, r0 + rstep, ... (fixed order)
template <typename T>
__device__ __forceinline__ C<T> data_adjoint_at(const C<T>* grow, const C<T>* hs, int R, int M0, int slot, int r0,
                                                int rstep) {
  C<T> a0 = czero<T>(), a1 = czero<T>();
  int r = r0;
  for (; r + rstep < R; r += 2 * rstep) {
    a0 = cadd<T>(a0, cmulc<T>(grow[r], hs[(size_t)r * M0 + slot]));
    a1 = cadd<T>(a1, cmulc<T>(grow[r + rstep], hs[(size_t)(r + rstep) * M0 + slot]));
  }
  if (r < R) a0 = cadd<T>(a0, cmulc<T>(grow[r], hs[(size_t)r * M0 + slot]));
  return cadd<T>(a0, a1);
}

// gad[v][slot] = sum_r g_rows[v][r] conj(H[r][slot]) for every view (the data
// part of g_alpha, see above): CTA = 256 coefficients of one view
template <typename T>
__global__ void __launch_bounds__(256) gad_kernel(const C<T>* grows, const C<T>* hs, C<T>* gad, int R, int M0) {
  const int v = blockIdx.y, m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M0) return;
  gad[(size_t)v * M0 + m] = data_adjoint_at<T>(grows + (size_t)v * R, hs, R, M0, m, 0, 1);
}

template <typename T>
__global__ void permute_khat_kernel(const C<T>* khat, C<T>* out, int P, int split) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= P * P) return;
  const int posc = idx / P, posr = idx % P;
  const int fr = khat_pos_freq(posr, P, split);
  const int fc = khat_pos_freq(posc, P, split);
  const T s = T(1) / (T(P) * T(P));
  out[idx] = cscale<T>(khat[(size_t)fr * P + fc], s);
}

__global__ void set_ints_kernel(int* p, int a, int b) { p[0] = a; p[1] = b; }

// J = expand(alpha): one thread per pixel, direct corner-sparse inverse DFT
template <typename T>
__global__ void expand_kernel(const C<T>* alpha, C<T>* img, const C<T>* twM, int M, int mf) {
  const int K = 2 * mf, M0 = K * K;
  const int v = blockIdx.y;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= M * M) return;
  const int y = p / M, x = p % M;
  const C<T>* al = alpha + (size_t)v * M0;
  C<T> acc = czero<T>();
  for (int u = 0; u < K; ++u) {
    const int fr = u < mf ? u : M - K + u;
    C<T> row = czero<T>();
    for (int w = 0; w < K; ++w) {
      const int fc = w < mf ? w : M - K + w;
      const int slot = (((u / mf) * 2 + (w / mf)) * mf + (u % mf)) * mf + (w % mf);
      row = cadd<T>(row, cmulc<T>(al[slot], twM[(fc * x) & (M - 1)]));
    }
    acc = cadd<T>(acc, cmulc<T>(row, twM[(fr * y) & (M - 1)]));
  }
  img[(size_t)v * M * M + p] = cscale<T>(acc, T(1) / (T(M) * T(M)));
}

// alpha = truncate(img): one block per (coefficient chunk, image); fixed-order sums
template <typename T>
__global__ void truncate_kernel(const C<T>* img, C<T>* alpha, const C<T>* twM, int M, int mf) {
  const int K = 2 * mf, M0 = K * K;
  const int v = blockIdx.y;
  const int c = blockIdx.x;     // coefficient slot
  if (c >= M0) return;
  const int blk = c / (mf * mf), rem = c % (mf * mf);
  const int u = (blk / 2) * mf + rem / mf, w = (blk % 2) * mf + rem % mf;
  const int fr = u < mf ? u : M - K + u, fc = w < mf ? w : M - K + w;
  const C<T>* im = img + (size_t)v * M * M;
  C<T> acc = czero<T>();
  for (int p = threadIdx.x; p < M * M; p += blockDim.x) {
    const int y = p / M, x = p % M;
    acc = cadd<T>(acc, cmul<T>(im[p], twM[(fr * y + fc * x) & (M - 1)]));
  }
  __shared__ C<T> red[32];
  acc.x = warp_sum<T>(acc.x);
  acc.y = warp_sum<T>(acc.y);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    C<T> s = czero<T>();
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s = cadd<T>(s, red[i]);
    alpha[(size_t)v * M0 + c] = s;
  }
}

// rows[v][r] = sum_p img[v][p] gs[r][p]
template <typename T>
__global__ void gs_forward_kernel(const C<T>* img, C<T>* rows, const C<T>* gs, int npix, int R) {
  const int r = blockIdx.x, v = blockIdx.y;
  const C<T>* im = img + (size_t)v * npix;
  const C<T>* g = gs + (size_t)r * npix;
  C<T> acc = czero<T>();
  for (int p = threadIdx.x; p < npix; p += blockDim.x) acc = cadd<T>(acc, cmul<T>(im[p], g[p]));
  __shared__ C<T> red[32];
  acc.x = warp_sum<T>(acc.x);
  acc.y = warp_sum<T>(acc.y);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    C<T> s = czero<T>();
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s = cadd<T>(s, red[i]);
    rows[(size_t)v * R + r] = s;
  }
}

// img[v][p] = sum_r rows[v][r] conj(gs[r][p])
template <typename T>
__global__ void gs_adjoint_kernel(const C<T>* rows, C<T>* img, const C<T>* gs, int npix, int R) {
  const int v = blockIdx.y;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npix) return;
  const C<T>* rw = rows + (size_t)v * R;
  C<T> acc = czero<T>();
  for (int r = 0; r < R; ++r) acc = cadd<T>(acc, cmulc<T>(rw[r], gs[(size_t)r * npix + p]));
  img[(size_t)v * npix + p] = acc;
}

// ---- contrast compensation (filters.py:16-67) ----------------------------
// box mean over (2r+1)^2 windows with edge replication
template <typename T>
__device__ inline T box_at(const T* img, int M, int y, int x, int r) {
  T s = T(0);
  for (int dy = -r; dy <= r; ++dy) {
    const int yy = min(max(y + dy, 0), M - 1);
    for (int dx = -r; dx <= r; ++dx) {
      const int xx = min(max(x + dx, 0), M - 1);
      s += img[yy * M + xx];
    }
  }
  const int w = 2 * r + 1;
  return s / T(w * w);
}

// pass 1: per channel (re, im) the self-guided filter coefficients a, b
template <typename T>
__global__ void cco_pass1_kernel(const C<T>* chi, T* ab, int M, int r, T eps_gf) {
  const int v = blockIdx.y, ch = blockIdx.z;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= M * M) return;
  const int y = p / M, x = p % M;
  const T* base = reinterpret_cast<const T*>(chi + (size_t)v * M * M) + ch;
  // strided channel view: element q at base[2q]
  T mi = 0, mii = 0;
  const int w = 2 * r + 1;
  for (int dy = -r; dy <= r; ++dy) {
    const int yy = min(max(y + dy, 0), M - 1);
    for (int dx = -r; dx <= r; ++dx) {
      const int xx = min(max(x + dx, 0), M - 1);
      const T g = base[2 * (yy * M + xx)];
      mi += g;
      mii += g * g;
    }
  }
  mi /= T(w * w);
  mii /= T(w * w);
  // self-guided: p == I, so cov = var
  const T var = mii - mi * mi;
  const T a = var / (var + eps_gf);
  const T b = mi - a * mi;
  T* o = ab + (((size_t)v * 2 + ch) * 2) * M * M;
  o[p] = a;
  o[M * M + p] = b;
}

template <typename T>
__global__ void cco_pass2_kernel(const C<T>* chi, const T* ab, C<T>* out, int M, int r, T tau, T eta_max,
                                 T delta) {
  const int v = blockIdx.y;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= M * M) return;
  const int y = p / M, x = p % M;
  const C<T> c = chi[(size_t)v * M * M + p];
  T sm[2];
  for (int ch = 0; ch < 2; ++ch) {
    const T* a = ab + (((size_t)v * 2 + ch) * 2) * M * M;
    const T* b = a + M * M;
    const T g = ch == 0 ? c.x : c.y;
    sm[ch] = box_at<T>(a, M, y, x, r) * g + box_at<T>(b, M, y, x, r);
  }
  const T am = sqrt_<T>(cabs2<T>(c));
  const T eta = eta_max * sigmoid_<T>((am - tau) / delta);
  out[(size_t)v * M * M + p] = mk<T>((T(1) + eta) * sm[0] + eta * c.x, (T(1) + eta) * sm[1] + eta * c.y);
}

}  // namespace pdf
