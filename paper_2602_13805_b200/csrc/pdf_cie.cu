// Contrast-integral-equation algebra, the regularisers and the guided filter as standalone,
// context-free entry points (SURVEY §2 ★ rows cie.py / filters.py; §8 a8, a9,
// a22).  Inside the training step these operations are fused into the view
// and pixel kernels; these entry points serve the reference's module-level
// functions (chi_to_r, r_to_chi, default_eps_reg, pixel_least_squares,
// cie_state_residual, box_mean, guided_filter) and the pipeline_forward /
// recover_contrast(full=True) intermediates.
//
// Element arithmetic is written with explicit round-to-nearest intrinsics in the
// operation order numpy evaluates (Smith's division with a reciprocal, the FMA form
// of its complex multiply), so the elementwise maps (chi_to_r, r_to_chi, the state
// residual) can reproduce the reference's float64 results bit for bit
// (tests/test_gpu_algebra.py measures it); reductions (the per-pixel sums over
// views, the power of a view, the box sums) and the transcendental functions
// (hypot, exp) differ by rounding only.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pdf_abi.h"
#include "pdf_internal.h"

namespace {

constexpr int THREADS = 256;

// a * b as numpy's complex128 multiply loop evaluates it on an FMA host (measured on the
// golden-generating build: re = fma(ar, br, -(ai bi)), im = fma(ar, bi, ai br))
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)), __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}

__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}

// Smith's division, the form numpy's complex128 true_divide uses
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double ar = fabs(b.x), ai = fabs(b.y);
  if (ar >= ai) {
    if (ar == 0.0 && ai == 0.0) return make_double2(__ddiv_rn(a.x, ar), __ddiv_rn(a.y, ai));
    const double rat = __ddiv_rn(b.y, b.x);
    const double scl = __ddiv_rn(1.0, __dadd_rn(b.x, __dmul_rn(b.y, rat)));
    return make_double2(__dmul_rn(__dadd_rn(a.x, __dmul_rn(a.y, rat)), scl),
                        __dmul_rn(__dsub_rn(a.y, __dmul_rn(a.x, rat)), scl));
  }
  const double rat = __ddiv_rn(b.x, b.y);
  const double scl = __ddiv_rn(1.0, __dadd_rn(b.y, __dmul_rn(b.x, rat)));
  return make_double2(__dmul_rn(__dadd_rn(__dmul_rn(a.x, rat), a.y), scl),
                      __dmul_rn(__dsub_rn(__dmul_rn(a.y, rat), a.x), scl));
}

// |z| as numpy's np.abs (hypot)
__device__ __forceinline__ double cabs_(double2 z) { return hypot(z.x, z.y); }

// cie.py:24-39: forward R = beta chi / (beta chi + 1), inverse chi = R / (beta (1 - R));
// pixels whose denominator is below 1e-14 in modulus are counted into *poles
__global__ void chi_to_r_kernel(const double2* __restrict__ x, double2* __restrict__ y, long long n, double2 beta,
                                int inverse, int* __restrict__ poles) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 v = x[i];
  double2 out;
  bool pole;
  if (!inverse) {
    const double2 bc = cmul(beta, v);
    const double2 den = make_double2(__dadd_rn(bc.x, 1.0), __dadd_rn(bc.y, 0.0));
    pole = cabs_(den) < 1e-14;
    out = cdiv(bc, den);
  } else {
    const double2 den = make_double2(__dsub_rn(1.0, v.x), __dsub_rn(0.0, v.y));
    pole = cabs_(den) < 1e-14;
    out = cdiv(v, cmul(beta, den));
  }
  if (pole) atomicAdd(poles, 1);
  y[i] = out;
}

// cie.py:42-50: eps = 1e-10 max_v ||E_v||^2 / n_pix.  One CTA per view; the scaled
// powers are non-negative doubles, whose bit patterns order like the values, so an
// integer atomicMax selects the largest (scaling is monotone, so max(c p) = c max(p)).
__global__ void __launch_bounds__(THREADS) default_eps_kernel(const double2* __restrict__ e, long long npix,
                                                              double* __restrict__ eps) {
  __shared__ double sp[THREADS];
  const double2* ev = e + (long long)blockIdx.x * npix;
  double p = 0.0;
  for (long long q = threadIdx.x; q < npix; q += THREADS) {
    const double2 z = ev[q];
    p += z.x * z.x + z.y * z.y;
  }
  sp[threadIdx.x] = p;
  __syncthreads();
  for (int h = THREADS / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) sp[threadIdx.x] += sp[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double v = __ddiv_rn(__dmul_rn(1e-10, sp[0]), (double)npix);
    atomicMax(reinterpret_cast<unsigned long long*>(eps), (unsigned long long)__double_as_longlong(v));
  }
}

// cie.py:66-80: num = sum_v J_v conj(E_v), den = sum_v |E_v|^2 + eps, chi = num / den
// (complex / real promotes den to complex: Smith with a zero imaginary part is
// num * (1 / den)), degenerate = den <= 10 eps.  One thread per pixel, views in order.
__global__ void pixel_ls_kernel(const double2* __restrict__ j, const double2* __restrict__ e, int nv, long long npix,
                                const double* __restrict__ eps_p, double2* __restrict__ num_out,
                                double* __restrict__ den_out, double2* __restrict__ chi_out,
                                uint8_t* __restrict__ degen) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npix) return;
  double2 num = make_double2(0.0, 0.0);
  double den = 0.0;
  for (int v = 0; v < nv; ++v) {
    const double2 jv = j[(long long)v * npix + p], ev = e[(long long)v * npix + p];
    num = cadd(num, cmul(jv, make_double2(ev.x, -ev.y)));
    den = __dadd_rn(den, __dsub_rn(__dmul_rn(ev.x, ev.x), __dmul_rn(ev.y, -ev.y)));
  }
  const double eps = *eps_p;
  den = __dadd_rn(den, eps);
  if (num_out) num_out[p] = num;
  if (den_out) den_out[p] = den;
  if (chi_out) {
    const double scl = __ddiv_rn(1.0, den);
    chi_out[p] = make_double2(__dmul_rn(num.x, scl), __dmul_rn(num.y, scl));
  }
  if (degen) degen[p] = den <= __dmul_rn(10.0, eps);
}

// cie.py:92-114 / losses.py:215-237 per view v, pixel p:
//   E = E_inc + G_D J          (e_out; gdj may be null: E = E_inc)
//   P = E + beta J             (p_out)
//   res = R P - beta J         (res_out; R shared by the views)
__global__ void cie_fields_kernel(const double2* __restrict__ j, const double2* __restrict__ gdj,
                                  const double2* __restrict__ e_in, long long e_stride, const double2* __restrict__ r,
                                  double2 beta, int nv, long long npix, double2* __restrict__ e_out,
                                  double2* __restrict__ p_out, double2* __restrict__ res_out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)nv * npix) return;
  const long long v = i / npix, p = i % npix;
  double2 e = e_in[v * e_stride + p];
  if (gdj) e = cadd(e, gdj[i]);
  if (e_out) e_out[i] = e;
  if (!p_out && !res_out) return;
  const double2 bj = cmul(beta, j[i]);
  const double2 pv = cadd(e, bj);
  if (p_out) p_out[i] = pv;
  if (res_out) res_out[i] = csub(cmul(r[p], pv), bj);
}

// losses.py:225-231: (G_S J - data) * mask, mask optional (real, same shape)
__global__ void masked_residual_kernel(const double2* __restrict__ a, const double2* __restrict__ b,
                                       const double* __restrict__ mask, double2* __restrict__ out, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 d = csub(a[i], b[i]);
  if (mask) d = make_double2(__dmul_rn(d.x, mask[i]), __dmul_rn(d.y, mask[i]));
  out[i] = d;
}

// filters.py:16-33: mean over (2r+1)^2 windows, edge-replicated borders
__device__ __forceinline__ double box_at(const double* img, int m1, int m2, int y, int x, int r) {
  double s = 0.0;
  for (int dy = -r; dy <= r; ++dy) {
    const double* row = img + (long long)min(max(y + dy, 0), m1 - 1) * m2;
    for (int dx = -r; dx <= r; ++dx) s += row[min(max(x + dx, 0), m2 - 1)];
  }
  const int w = 2 * r + 1;
  return s / (double)(w * w);
}

__global__ void box_mean_kernel(const double* __restrict__ img, double* __restrict__ out, int m1, int m2, int r) {
  const long long np = (long long)m1 * m2;
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const long long off = (long long)blockIdx.y * np;
  out[off + p] = box_at(img + off, m1, m2, (int)(p / m2), (int)(p % m2), r);
}

// filters.py:36-53 pass 1: the per-window linear model a, b of inp ~ a guide + b.
// Images are read with an element stride (1: float64 images; 2: the re / im channel
// of complex128 images, channel = blockIdx.z); a, b of (image, channel) land at
// ab + 2 (image * channels + channel) n_pix.
__global__ void guided_ab_kernel(const double* __restrict__ inp, const double* __restrict__ guide, int stride,
                                 double* __restrict__ ab, int m1, int m2, int r, double eps_gf) {
  const long long np = (long long)m1 * m2;
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const long long base = (long long)blockIdx.y * np * stride + blockIdx.z;
  const double* I = guide + base;
  const double* P = inp + base;
  const int y = (int)(p / m2), x = (int)(p % m2);
  double mi = 0.0, mp = 0.0, mip = 0.0, mii = 0.0;
  for (int dy = -r; dy <= r; ++dy) {
    const long long row = (long long)min(max(y + dy, 0), m1 - 1) * m2;
    for (int dx = -r; dx <= r; ++dx) {
      const long long q = (row + min(max(x + dx, 0), m2 - 1)) * stride;
      const double g = I[q], v = P[q];
      mi += g;
      mp += v;
      mip += g * v;
      mii += g * g;
    }
  }
  const double w2 = (double)((2 * r + 1) * (2 * r + 1));
  mi /= w2;
  mp /= w2;
  mip /= w2;
  mii /= w2;
  const double a = (mip - mi * mp) / (mii - mi * mi + eps_gf);
  double* o = ab + 2 * ((long long)blockIdx.y * gridDim.z + blockIdx.z) * np;
  o[p] = a;
  o[np + p] = mp - a * mi;
}

// pass 2: out = box(a) guide + box(b)
__global__ void guided_out_kernel(const double* __restrict__ guide, const double* __restrict__ ab,
                                  double* __restrict__ out, int m1, int m2, int r) {
  const long long np = (long long)m1 * m2;
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const long long off = (long long)blockIdx.y * np;
  const double* a = ab + 2 * off;
  const int y = (int)(p / m2), x = (int)(p % m2);
  out[off + p] = box_at(a, m1, m2, y, x, r) * guide[off + p] + box_at(a + np, m1, m2, y, x, r);
}

// filters.py:56-67: eta = eta_max sig((|chi| - tau) / delta);
// out = (1 + eta) (G(Re|Re) + i G(Im|Im)) + eta chi, for any m1 x m2
__global__ void cco_out_kernel(const double2* __restrict__ chi, const double* __restrict__ ab,
                               double2* __restrict__ out, int m1, int m2, int r, double tau, double eta_max,
                               double delta) {
  const long long np = (long long)m1 * m2;
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const long long off = (long long)blockIdx.y * np;
  const double2 c = chi[off + p];
  const int y = (int)(p / m2), x = (int)(p % m2);
  double sm[2];
  for (int ch = 0; ch < 2; ++ch) {
    const double* a = ab + 2 * (2 * (long long)blockIdx.y + ch) * np;
    sm[ch] = box_at(a, m1, m2, y, x, r) * (ch == 0 ? c.x : c.y) + box_at(a + np, m1, m2, y, x, r);
  }
  const double eta = eta_max * (1.0 / (1.0 + exp(-((hypot(c.x, c.y) - tau) / delta))));
  const double g = 1.0 + eta;
  out[off + p] = make_double2(__dadd_rn(__dmul_rn(g, sm[0]), __dmul_rn(eta, c.x)),
                              __dadd_rn(__dmul_rn(g, sm[1]), __dmul_rn(eta, c.y)));
}

// ---- regularisers and their contrast gradients (losses.py:121-196) ----------
// per pixel (y, x) of an m1 x m2 image, forward differences zero on the last
// row / column:
//   bound   min(Re chi, 0)^2                       grad 2 min(Re chi, 0)
//   tv      s = sqrt(|dx|^2 + |dy|^2 + eps_tv)       grad = div-form of (dx, dy) / s
//   bridge  sig((|chi| - tau)/tau) exp(-|grad|chi||^2), grad through |chi| times chi/|chi|
struct RegPix {
  double2 wx, wy;   // tv: dx / s, dy / s
  double s;         // tv summand
  double sd, cx, cy, base;   // bridge: sig damp, sig damp (-2 gx), sig damp (-2 gy), sig (1-sig)/tau damp
};

__device__ __forceinline__ double sigm(double z) { return 1.0 / (1.0 + exp(-z)); }

__device__ RegPix reg_at(const double2* c, int m1, int m2, int y, int x, double tau, double eps_tv, bool need_tv,
                         bool need_br) {
  RegPix o;
  const long long q = (long long)y * m2 + x;
  const double2 v = c[q];
  const bool rx = x < m2 - 1, ry = y < m1 - 1;
  if (need_tv) {
    const double2 dx = rx ? csub(c[q + 1], v) : make_double2(0.0, 0.0);
    const double2 dy = ry ? csub(c[q + m2], v) : make_double2(0.0, 0.0);
    const double hx = hypot(dx.x, dx.y), hy = hypot(dy.x, dy.y);
    o.s = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(hx, hx), __dmul_rn(hy, hy)), eps_tv));
    const double r = __ddiv_rn(1.0, o.s);
    o.wx = make_double2(__dmul_rn(dx.x, r), __dmul_rn(dx.y, r));
    o.wy = make_double2(__dmul_rn(dy.x, r), __dmul_rn(dy.y, r));
  }
  if (need_br) {
    const double a = hypot(v.x, v.y);
    const double gx = rx ? __dsub_rn(hypot(c[q + 1].x, c[q + 1].y), a) : 0.0;
    const double gy = ry ? __dsub_rn(hypot(c[q + m2].x, c[q + m2].y), a) : 0.0;
    const double sig = sigm(__ddiv_rn(__dsub_rn(a, tau), tau));
    const double damp = exp(-__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)));
    o.sd = __dmul_rn(sig, damp);
    o.cx = __dmul_rn(o.sd, __dmul_rn(-2.0, gx));
    o.cy = __dmul_rn(o.sd, __dmul_rn(-2.0, gy));
    o.base = __dmul_rn(__ddiv_rn(__dmul_rn(sig, __dsub_rn(1.0, sig)), tau), damp);
  }
  return o;
}

__global__ void __launch_bounds__(THREADS) reg_values_kernel(const double2* __restrict__ chi, int m1, int m2,
                                                             double tau, double eps_tv, double* __restrict__ vals) {
  __shared__ double sb[THREADS], st[THREADS], sr[THREADS];
  const long long np = (long long)m1 * m2;
  const double2* c = chi + (long long)blockIdx.x * np;
  double b = 0.0, t = 0.0, r = 0.0;
  for (long long p = threadIdx.x; p < np; p += THREADS) {
    const int y = (int)(p / m2), x = (int)(p % m2);
    const RegPix o = reg_at(c, m1, m2, y, x, tau, eps_tv, true, true);
    const double ng = fmin(c[p].x, 0.0);
    b += ng * ng;
    t += o.s;
    r += o.sd;
  }
  sb[threadIdx.x] = b;
  st[threadIdx.x] = t;
  sr[threadIdx.x] = r;
  __syncthreads();
  for (int h = THREADS / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
      sb[threadIdx.x] += sb[threadIdx.x + h];
      st[threadIdx.x] += st[threadIdx.x + h];
      sr[threadIdx.x] += sr[threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    vals[3 * blockIdx.x + 0] = sb[0];
    vals[3 * blockIdx.x + 1] = st[0];
    vals[3 * blockIdx.x + 2] = sr[0];
  }
}

__global__ void reg_grad_kernel(const double2* __restrict__ chi, int m1, int m2, double tau, double eps_tv, double l1,
                                double l2, double l3, double2* __restrict__ gb_out, double2* __restrict__ gt_out,
                                double2* __restrict__ gr_out, double2* __restrict__ g_out) {
  const long long np = (long long)m1 * m2;
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const long long off = (long long)blockIdx.y * np;
  const double2* c = chi + off;
  const int y = (int)(p / m2), x = (int)(p % m2);
  const bool need_tv = gt_out || (g_out && l2 != 0.0), need_br = gr_out || (g_out && l3 != 0.0);
  const double2 v = c[p];
  const double2 gb = make_double2(__dmul_rn(2.0, fmin(v.x, 0.0)), 0.0);
  double2 gt = make_double2(0.0, 0.0), gr = make_double2(0.0, 0.0);
  const RegPix me = reg_at(c, m1, m2, y, x, tau, eps_tv, need_tv, need_br);
  const RegPix left = x > 0 ? reg_at(c, m1, m2, y, x - 1, tau, eps_tv, need_tv, need_br) : RegPix{};
  const RegPix up = y > 0 ? reg_at(c, m1, m2, y - 1, x, tau, eps_tv, need_tv, need_br) : RegPix{};
  if (need_tv) {
    // g[:, 1:] += wx[:, :-1]; g[:, :-1] -= wx[:, :-1]; g[1:, :] += wy[:-1, :]; g[:-1, :] -= wy[:-1, :]
    if (x > 0) gt = cadd(gt, left.wx);
    if (x < m2 - 1) gt = csub(gt, me.wx);
    if (y > 0) gt = cadd(gt, up.wy);
    if (y < m1 - 1) gt = csub(gt, me.wy);
  }
  if (need_br) {
    double ga = me.base;
    if (x > 0) ga = __dadd_rn(ga, left.cx);
    if (x < m2 - 1) ga = __dsub_rn(ga, me.cx);
    if (y > 0) ga = __dadd_rn(ga, up.cy);
    if (y < m1 - 1) ga = __dsub_rn(ga, me.cy);
    const double a = hypot(v.x, v.y);
    if (a > 0.0) {
      const double r = __ddiv_rn(1.0, a);
      gr = make_double2(__dmul_rn(ga, __dmul_rn(v.x, r)), __dmul_rn(ga, __dmul_rn(v.y, r)));
    }
  }
  if (gb_out) gb_out[off + p] = gb;
  if (gt_out) gt_out[off + p] = gt;
  if (gr_out) gr_out[off + p] = gr;
  if (g_out) {
    double2 g = make_double2(0.0, 0.0);
    if (l1 != 0.0) g = cadd(g, make_double2(__dmul_rn(l1, gb.x), __dmul_rn(l1, gb.y)));
    if (l2 != 0.0) g = cadd(g, make_double2(__dmul_rn(l2, gt.x), __dmul_rn(l2, gt.y)));
    if (l3 != 0.0) g = cadd(g, make_double2(__dmul_rn(l3, gr.x), __dmul_rn(l3, gr.y)));
    g_out[off + p] = g;
  }
}

unsigned blocks(long long n) { return (unsigned)((n + THREADS - 1) / THREADS); }

int launched(const char* what) {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PDF_OK : pdf_fail(PDF_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

extern "C" int pdf_chi_to_r(const void* x, void* y, int64_t n, double beta_re, double beta_im, int32_t inverse,
                            int32_t* poles, void* stream) {
  if (n < 0 || !poles || (n > 0 && (!x || !y))) return pdf_fail(PDF_EINVAL, "pdf_chi_to_r: bad arguments");
  const cudaStream_t st = (cudaStream_t)stream;
  PDF_CK(cudaMemsetAsync(poles, 0, sizeof(int32_t), st));
  if (n == 0) return PDF_OK;
  chi_to_r_kernel<<<blocks(n), THREADS, 0, st>>>((const double2*)x, (double2*)y, n, make_double2(beta_re, beta_im),
                                                 inverse, poles);
  return launched("chi_to_r_kernel");
}

extern "C" int pdf_default_eps_reg(const void* e, int32_t n_views, int64_t n_pix, double* eps, void* stream) {
  if (n_views < 1 || n_pix < 1 || !e || !eps) return pdf_fail(PDF_EINVAL, "pdf_default_eps_reg: bad arguments");
  const cudaStream_t st = (cudaStream_t)stream;
  PDF_CK(cudaMemsetAsync(eps, 0, sizeof(double), st));
  default_eps_kernel<<<n_views, THREADS, 0, st>>>((const double2*)e, n_pix, eps);
  return launched("default_eps_kernel");
}

extern "C" int pdf_pixel_ls(const void* j, const void* e, int32_t n_views, int64_t n_pix, const double* eps,
                            void* num, double* den, void* chi, uint8_t* degenerate, void* stream) {
  if (n_views < 1 || n_pix < 1 || !j || !e || !eps) return pdf_fail(PDF_EINVAL, "pdf_pixel_ls: bad arguments");
  pixel_ls_kernel<<<blocks(n_pix), THREADS, 0, (cudaStream_t)stream>>>(
      (const double2*)j, (const double2*)e, n_views, n_pix, eps, (double2*)num, den, (double2*)chi, degenerate);
  return launched("pixel_ls_kernel");
}

extern "C" int pdf_cie_fields(const void* j, const void* gdj, const void* e_in, int64_t e_view_stride,
                              const void* r_hat, double beta_re, double beta_im, int32_t n_views, int64_t n_pix,
                              void* e_out, void* p_out, void* res_out, void* stream) {
  if (n_views < 1 || n_pix < 1 || !e_in || ((p_out || res_out) && !j) || (res_out && !r_hat))
    return pdf_fail(PDF_EINVAL, "pdf_cie_fields: bad arguments");
  cie_fields_kernel<<<blocks((long long)n_views * n_pix), THREADS, 0, (cudaStream_t)stream>>>(
      (const double2*)j, (const double2*)gdj, (const double2*)e_in, e_view_stride, (const double2*)r_hat,
      make_double2(beta_re, beta_im), n_views, n_pix, (double2*)e_out, (double2*)p_out, (double2*)res_out);
  return launched("cie_fields_kernel");
}

extern "C" int pdf_masked_residual(const void* a, const void* b, const double* mask, void* out, int64_t n,
                                   void* stream) {
  if (n < 1 || !a || !b || !out) return pdf_fail(PDF_EINVAL, "pdf_masked_residual: bad arguments");
  masked_residual_kernel<<<blocks(n), THREADS, 0, (cudaStream_t)stream>>>((const double2*)a, (const double2*)b, mask,
                                                                          (double2*)out, n);
  return launched("masked_residual_kernel");
}

extern "C" int pdf_box_mean(const double* img, double* out, int32_t m1, int32_t m2, int32_t radius, int32_t count,
                            void* stream) {
  if (radius < 1) return pdf_fail(PDF_EINVAL, "radius must be >= 1");
  if (m1 < 1 || m2 < 1 || count < 1 || count > 65535 || !img || !out)
    return pdf_fail(PDF_EINVAL, "pdf_box_mean: bad arguments");
  box_mean_kernel<<<dim3(blocks((long long)m1 * m2), count), THREADS, 0, (cudaStream_t)stream>>>(img, out, m1, m2,
                                                                                                 radius);
  return launched("box_mean_kernel");
}

extern "C" int pdf_guided_filter(const double* inp, const double* guide, double* out, int32_t m1, int32_t m2,
                                 int32_t radius, double eps_gf, int32_t count, double* scratch, void* stream) {
  if (radius < 1) return pdf_fail(PDF_EINVAL, "radius must be >= 1");
  if (m1 < 1 || m2 < 1 || count < 1 || count > 65535 || !inp || !guide || !out || !scratch)
    return pdf_fail(PDF_EINVAL, "pdf_guided_filter: bad arguments");
  const dim3 g(blocks((long long)m1 * m2), count);
  const cudaStream_t st = (cudaStream_t)stream;
  guided_ab_kernel<<<g, THREADS, 0, st>>>(inp, guide, 1, scratch, m1, m2, radius, eps_gf);
  guided_out_kernel<<<g, THREADS, 0, st>>>(guide, scratch, out, m1, m2, radius);
  return launched("guided_filter");
}

extern "C" int pdf_regularizers(const void* chi, int32_t m1, int32_t m2, int32_t count, double tau_b, double eps_tv,
                                double l1, double l2, double l3, double* values, void* g_bound, void* g_tv,
                                void* g_bridge, void* g_total, void* stream) {
  if (m1 < 1 || m2 < 1 || count < 1 || count > 65535 || !chi || !(tau_b > 0.0))
    return pdf_fail(PDF_EINVAL, "pdf_regularizers: bad arguments");
  const cudaStream_t st = (cudaStream_t)stream;
  if (values) reg_values_kernel<<<count, THREADS, 0, st>>>((const double2*)chi, m1, m2, tau_b, eps_tv, values);
  if (g_bound || g_tv || g_bridge || g_total)
    reg_grad_kernel<<<dim3(blocks((long long)m1 * m2), count), THREADS, 0, st>>>(
        (const double2*)chi, m1, m2, tau_b, eps_tv, l1, l2, l3, (double2*)g_bound, (double2*)g_tv,
        (double2*)g_bridge, (double2*)g_total);
  return launched("regularizers");
}

extern "C" int pdf_cco_image(const void* chi, void* out, int32_t m1, int32_t m2, int32_t count, double tau,
                             double eta_max, double delta, int32_t radius, double eps_gf, double* scratch,
                             void* stream) {
  if (radius < 1) return pdf_fail(PDF_EINVAL, "radius must be >= 1");
  if (m1 < 1 || m2 < 1 || count < 1 || count > 65535 || !chi || !out || !scratch)
    return pdf_fail(PDF_EINVAL, "pdf_cco_image: bad arguments");
  const unsigned gx = blocks((long long)m1 * m2);
  const cudaStream_t st = (cudaStream_t)stream;
  guided_ab_kernel<<<dim3(gx, count, 2), THREADS, 0, st>>>((const double*)chi, (const double*)chi, 2, scratch, m1,
                                                           m2, radius, eps_gf);
  cco_out_kernel<<<dim3(gx, count), THREADS, 0, st>>>((const double2*)chi, scratch, (double2*)out, m1, m2, radius,
                                                      tau, eta_max, delta);
  return launched("cco_image");
}
