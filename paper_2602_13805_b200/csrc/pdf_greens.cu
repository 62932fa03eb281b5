// One-time operator construction on the device:
//   cylinder functions J0, J1, Y0, Y1 and H^(1) = J + iY     special.py:20-106
//   G_D displacement kernel on the doubled grid + its fft2   forward.py:101-130, 136
//   receiver matrix G_S                                      forward.py:130-134
//   incident fields: unit line sources / plane waves          forward.py:174-181, SURVEY 8(d)
// Time convention exp(-i w t): first-kind Hankel functions (forward.py:10-11).
// The Bessel functions are Chebyshev series in t = 2 (x/8)^2 - 1 below x = 8
// (log / pole parts of Y peeled off) and Hankel's modulus/phase form above,
// tables generated at 60 digits by tools/gen_bessel_tables.py (worst error
// 1.3e-15 absolute against mpmath on [0, 400]).  The 2-D FFT of the kernel is
// a shared-memory radix-2 pass per row, then per column (sizes up to 512).
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/pdf_abi.h"
#include "pdf_bessel_tables.h"
#include "pdf_internal.h"

namespace pdf {
namespace {

template <int N>
__device__ __forceinline__ double clenshaw(const double (&c)[N], double t) {
  double b1 = 0.0, b2 = 0.0;
  const double t2 = 2.0 * t;
#pragma unroll
  for (int k = N - 1; k >= 1; --k) {
    const double b0 = fma(t2, b1, c[k] - b2);
    b2 = b1;
    b1 = b0;
  }
  return fma(t, b1, c[0] - b2);
}

// (J_n(x), Y_n(x)) for x > 0, n = 0 or 1
__device__ void bessel_jy(int n, double x, double* j, double* y) {
  constexpr double two_over_pi = 0.63661977236758134308;
  if (x <= BESSEL_SPLIT) {
    const double q = x / BESSEL_SPLIT;
    const double t = 2.0 * q * q - 1.0;
    const double ln = two_over_pi * log(0.5 * x);
    if (n == 0) {
      const double j0 = clenshaw(J0_IN, t);
      *j = j0;
      *y = fma(ln, j0, clenshaw(Y0_IN, t));
    } else {
      const double j1 = x * clenshaw(J1_IN, t);
      *j = j1;
      *y = ln * j1 - two_over_pi / x + x * clenshaw(Y1_IN, t);
    }
    return;
  }
  const double z = BESSEL_SPLIT / x;
  const double t = 2.0 * z * z - 1.0;
  const double amp = sqrt(two_over_pi / x);
  const double ph = x - (n == 0 ? 0.78539816339744830962 : 2.35619449019234492885);
  double s, c;
  sincos(ph, &s, &c);
  const double p = n == 0 ? clenshaw(P0_OUT, t) : clenshaw(P1_OUT, t);
  const double qz = z * (n == 0 ? clenshaw(Q0_OUT, t) : clenshaw(Q1_OUT, t));
  *j = amp * (p * c - qz * s);
  *y = amp * (p * s + qz * c);
}

__global__ void bessel_kernel(int n, const double* __restrict__ x, double* __restrict__ j, double* __restrict__ y,
                              long long count) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const double xi = x[i];
  double jv, yv;
  if (xi == 0.0) {
    jv = n == 0 ? 1.0 : 0.0;
    yv = -INFINITY;
  } else {
    bessel_jy(n, fabs(xi), &jv, &yv);
    if (xi < 0.0) {            // J0 even, J1 odd; Y is defined for x >= 0 only
      if (n == 1) jv = -jv;
      yv = NAN;
    }
  }
  if (j) j[i] = jv;
  if (y) y[i] = yv;
}

struct Cell {
  double2 coef;      // i pi k0 a / 2
  double2 off_w;     // coef J1(k0 a)
};

__device__ __forceinline__ double2 cm(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ Cell cell_weights(double k0, double a) {
  Cell w;
  w.coef = make_double2(0.0, 3.14159265358979323846 * k0 * a / 2.0);
  double j1, y1;
  bessel_jy(1, k0 * a, &j1, &y1);
  w.off_w = make_double2(w.coef.x * j1, w.coef.y * j1);
  return w;
}

// wrap-indexed kernel on the (2 m1) x (2 m2) grid; row m1 / column m2 zero;
// [0][0] = coef H1(k0 a) - 1 (forward.py:113-128)
__global__ void gd_kernel_kernel(double k0, double cs, int m1, int m2, double2* __restrict__ ker,
                                 double2* __restrict__ diag_out) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int P1 = 2 * m1, P2 = 2 * m2;
  if (idx >= (long long)P1 * P2) return;
  const int i = (int)(idx / P2), jj = (int)(idx % P2);
  const double a = cs / sqrt(3.14159265358979323846);
  const Cell w = cell_weights(k0, a);
  double2 v = make_double2(0.0, 0.0);
  if (i == 0 && jj == 0) {
    double j1, y1;
    bessel_jy(1, k0 * a, &j1, &y1);
    v = cm(w.coef, make_double2(j1, y1));
    v.x -= 1.0;
    if (diag_out) *diag_out = v;
  } else if (i != m1 && jj != m2) {
    const double di = i < m1 ? i : i - P1, dj = jj < m2 ? jj : jj - P2;
    const double rho = cs * hypot(di, dj);
    double j0, y0;
    bessel_jy(0, k0 * rho, &j0, &y0);
    v = cm(w.off_w, make_double2(j0, y0));
  }
  ker[idx] = v;
}

// G_S[r][p] = coef J1(k0 a) H0(k0 |rx_r - c_p|); flags a receiver inside the grid
__global__ void gs_kernel(double k0, double cs, int m1, int m2, const double* __restrict__ xs,
                          const double* __restrict__ ys, const double* __restrict__ rx, int R,
                          double2* __restrict__ gs, int* __restrict__ flag) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long np = (long long)m1 * m2;
  if (idx >= np * R) return;
  const int r = (int)(idx / np), p = (int)(idx % np);
  const double dx = __dsub_rn(rx[2 * r], xs[p % m2]), dy = __dsub_rn(rx[2 * r + 1], ys[p / m2]);
  const double d = sqrt(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
  if (d < cs / 2.0) atomicOr(flag, 1);
  const double a = cs / sqrt(3.14159265358979323846);
  const Cell w = cell_weights(k0, a);
  double j0, y0;
  bessel_jy(0, k0 * d, &j0, &y0);
  gs[idx] = cm(w.off_w, make_double2(j0, y0));
}

// kind 0: (i/4) H0(k0 |tx_v - c_p|) (forward.py:174-181); kind 1: exp(i k0 (x cos phi_v + y sin phi_v))
__global__ void incident_kernel(int kind, double k0, int m1, int m2, const double* __restrict__ xs,
                                const double* __restrict__ ys, const double* __restrict__ src, int n,
                                double2* __restrict__ out, int* __restrict__ flag) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long np = (long long)m1 * m2;
  if (idx >= np * n) return;
  const int v = (int)(idx / np), p = (int)(idx % np);
  const double x = xs[p % m2], y = ys[p / m2];
  if (kind == 0) {
    const double dx = __dsub_rn(src[2 * v], x), dy = __dsub_rn(src[2 * v + 1], y);
    const double d = sqrt(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
    if (d <= 0.0) atomicOr(flag, 1);
    double j0, y0;
    bessel_jy(0, k0 * d, &j0, &y0);
    out[idx] = make_double2(-0.25 * y0, 0.25 * j0);
  } else {
    double c, s;
    sincos(src[v], &s, &c);
    const double ph = k0 * __dadd_rn(__dmul_rn(c, x), __dmul_rn(s, y));
    double sp, cp;
    sincos(ph, &sp, &cp);
    out[idx] = make_double2(cp, sp);
  }
}

// in-place unnormalised forward DFT (exp(-2 pi i k n / N)) of `count` vectors of
// length N (power of two <= 1024): element e of vector v at data[v * vstride + e * estride]
__global__ void fft_pass_kernel(double2* data, int N, int logN, long long vstride, long long estride) {
  extern __shared__ double2 sh[];
  double2* base = data + (long long)blockIdx.x * vstride;
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    const int rev = (int)(__brev((unsigned)e) >> (32 - logN));
    sh[rev] = base[(long long)e * estride];
  }
  __syncthreads();
  for (int len = 2; len <= N; len <<= 1) {
    const int half = len >> 1;
    for (int b = threadIdx.x; b < N / 2; b += blockDim.x) {
      const int grp = b / half, k = b % half;
      const int i0 = grp * len + k, i1 = i0 + half;
      double s, c;
      sincospi(-2.0 * (double)k / (double)len, &s, &c);
      const double2 u = sh[i0], t = sh[i1];
      const double2 w = make_double2(c * t.x - s * t.y, c * t.y + s * t.x);
      sh[i0] = make_double2(u.x + w.x, u.y + w.y);
      sh[i1] = make_double2(u.x - w.x, u.y - w.y);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < N; e += blockDim.x) base[(long long)e * estride] = sh[e];
}

int ilog2(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  return (1 << l) == v ? l : -1;
}

}  // namespace
}  // namespace pdf

using namespace pdf;

extern "C" int pdf_bessel(int32_t order, const double* x, double* j, double* y, int64_t count, void* stream) {
  if ((order != 0 && order != 1) || !x || (!j && !y) || count < 0) return pdf_fail(PDF_EINVAL, "pdf_bessel: bad argument");
  if (count == 0) return PDF_OK;
  bessel_kernel<<<(unsigned)((count + 255) / 256), 256, 0, (cudaStream_t)stream>>>(order, x, j, y, count);
  PDF_CK(cudaGetLastError());
  return PDF_OK;
}

extern "C" int pdf_build_greens(double k0, double cell_size, int32_t m1, int32_t m2, const double* xs, const double* ys,
                                const double* rx, int32_t R, void* gd_kernel, void* gd_kernel_hat, void* gs_matrix,
                                double* gd_diag_host, void* stream) {
  if (!(k0 > 0.0) || !(cell_size > 0.0) || m1 < 1 || m2 < 1 || !gd_kernel || !gd_kernel_hat)
    return pdf_fail(PDF_EINVAL, "pdf_build_greens: bad argument");
  const int l1 = ilog2(2 * m1), l2 = ilog2(2 * m2);
  if (l1 < 0 || l2 < 0 || 2 * m1 > 1024 || 2 * m2 > 1024)
    return pdf_fail(PDF_EINVAL, "pdf_build_greens: m1, m2 must be powers of two <= 512");
  if (gs_matrix && (!xs || !ys || !rx || R < 1)) return pdf_fail(PDF_EINVAL, "pdf_build_greens: receivers");
  cudaStream_t st = (cudaStream_t)stream;
  const long long P = 4LL * m1 * m2;
  double2* ker = (double2*)gd_kernel;
  double2* hat = (double2*)gd_kernel_hat;
  int* dflag = nullptr;
  double2* ddiag = nullptr;
  PDF_CK(cudaMallocAsync((void**)&ddiag, sizeof(double2) + sizeof(int), st));
  dflag = (int*)(ddiag + 1);
  PDF_CK(cudaMemsetAsync(dflag, 0, sizeof(int), st));
  gd_kernel_kernel<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(k0, cell_size, m1, m2, ker, ddiag);
  PDF_CK(cudaMemcpyAsync(hat, ker, sizeof(double2) * P, cudaMemcpyDeviceToDevice, st));
  // fft2: rows (length 2 m2), then columns (length 2 m1)
  fft_pass_kernel<<<2 * m1, 256, sizeof(double2) * 2 * m2, st>>>(hat, 2 * m2, l2, 2 * m2, 1);
  fft_pass_kernel<<<2 * m2, 256, sizeof(double2) * 2 * m1, st>>>(hat, 2 * m1, l1, 1, 2 * m2);
  if (gs_matrix) {
    const long long n = (long long)m1 * m2 * R;
    gs_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(k0, cell_size, m1, m2, xs, ys, rx, R, (double2*)gs_matrix,
                                                          dflag);
  }
  PDF_CK(cudaGetLastError());
  double2 diag_h;
  int flag_h = 0;
  PDF_CK(cudaMemcpyAsync(&diag_h, ddiag, sizeof(double2), cudaMemcpyDeviceToHost, st));
  PDF_CK(cudaMemcpyAsync(&flag_h, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
  PDF_CK(cudaFreeAsync(ddiag, st));
  PDF_CK(cudaStreamSynchronize(st));
  if (gd_diag_host) {
    gd_diag_host[0] = diag_h.x;
    gd_diag_host[1] = diag_h.y;
  }
  if (flag_h) return pdf_fail(PDF_EGEOMETRY, "a receiver lies inside the pixel grid");
  return PDF_OK;
}

extern "C" int pdf_incident_fields(int32_t kind, double k0, int32_t m1, int32_t m2, const double* xs, const double* ys,
                                   const double* src, int32_t n, void* out, void* stream) {
  if ((kind != 0 && kind != 1) || !(k0 > 0.0) || m1 < 1 || m2 < 1 || !xs || !ys || !src || n < 1 || !out)
    return pdf_fail(PDF_EINVAL, "pdf_incident_fields: bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  int* dflag = nullptr;
  PDF_CK(cudaMallocAsync((void**)&dflag, sizeof(int), st));
  PDF_CK(cudaMemsetAsync(dflag, 0, sizeof(int), st));
  const long long tot = (long long)m1 * m2 * n;
  incident_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(kind, k0, m1, m2, xs, ys, src, n, (double2*)out,
                                                                dflag);
  PDF_CK(cudaGetLastError());
  int flag_h = 0;
  PDF_CK(cudaMemcpyAsync(&flag_h, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
  PDF_CK(cudaFreeAsync(dflag, st));
  PDF_CK(cudaStreamSynchronize(st));
  if (flag_h) return pdf_fail(PDF_EGEOMETRY, "a transmitter coincides with a cell center");
  return PDF_OK;
}
