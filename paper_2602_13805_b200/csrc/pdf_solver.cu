// Batched BiCGStab forward solve on the device:
// (I - G_D chi) x = b for every view of S scenes at once, the method of
// moments' state equation E = E_inc + G_D (chi E) (reference
// forward.py:193-248 _solve_bicgstab and forward.py:251-275 solve_total_field).
//
// Same algorithm and per-view semantics as the reference:
//   x0 = b, r0 = b - A x0, shadow residual rhat = r0, rho = alpha = omega = 1;
//   a view iterates while its residual ||r|| / ||b|| exceeds tol and keeps its
//   x / r frozen afterwards;
//   when |<rhat, r>| < 1e-300 |<r, r>| the shadow residual lost orthogonality
//   and the view restarts (rhat = r, p = v = 0, rho = alpha = omega = 1);
//   the run succeeds iff every view has converged at one of the checks made
//   before iterations 0 .. maxiter-1 (so maxiter = 0 never succeeds), else it
//   returns PDF_ENOCONV (NoConvergenceError) naming the views above tol.
// A = I - G_D chi applies the context's G_D (pdf_apply_gd: the cluster /
// large-grid FFT convolution of the hot loop).  Every dot product is a fixed
// two-level reduction (4096-element chunks, then chunk order), so the solve
// is bitwise deterministic.  The host looks at the active-view count every
// CHECK_EVERY iterations only; converged views are frozen on the device, so
// the extra iterations leave x unchanged (same result as the reference).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/pdf_abi.h"
#include "pdf_internal.h"

namespace {

using cd = double2;
__device__ __forceinline__ cd mkc(double a, double b) { return make_double2(a, b); }
__device__ __forceinline__ cd cadd(cd a, cd b) { return mkc(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ cd csub(cd a, cd b) { return mkc(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ cd cmul(cd a, cd b) { return mkc(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ cd conjmul(cd a, cd b) { return mkc(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x); }
__device__ __forceinline__ cd cdiv(cd a, cd b) {
  const double d = b.x * b.x + b.y * b.y;
  return mkc((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
__device__ __forceinline__ bool czero(cd a) { return a.x == 0.0 && a.y == 0.0; }
__device__ __forceinline__ double cabs_(cd a) { return hypot(a.x, a.y); }

constexpr int TH = 256;
constexpr int PER = 16;
constexpr int CHUNK = TH * PER;   // elements per reduction chunk
constexpr int CHECK_EVERY = 8;

struct ViewScalars {
  cd rho, alpha, omega, beta, acc0, acc1;
  double nb, res;
  int active, restart;
};

struct Vecs {
  cd *r, *rhat, *p, *v, *s, *t, *tmp, *g;
  double4* part;   // [V][nchunk] partial sums (two complex accumulators)
  ViewScalars* sc;
  int* nactive;
};

// block reduction of two complex accumulators in a fixed tree, written to part[view][chunk]
__device__ __forceinline__ void block_reduce_store(double4 acc, double4* part, int nchunk) {
  __shared__ double4 sh[TH];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int h = TH / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
      double4 a = sh[threadIdx.x], b = sh[threadIdx.x + h];
      sh[threadIdx.x] = make_double4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(size_t)blockIdx.y * nchunk + blockIdx.x] = sh[0];
}

__device__ __forceinline__ double4 chunk_sum(const double4* part, int view, int nchunk) {
  double4 s = make_double4(0, 0, 0, 0);
  for (int k = 0; k < nchunk; ++k) {
    const double4 a = part[(size_t)view * nchunk + k];
    s.x += a.x; s.y += a.y; s.z += a.z; s.w += a.w;
  }
  return s;
}

#define ELEM_LOOP(...)                                                                   \
  for (int k = 0; k < PER; ++k) {                                                        \
    const long long e = (long long)blockIdx.x * CHUNK + k * TH + threadIdx.x;            \
    if (e >= npix) break;                                                                \
    const size_t i = (size_t)view * npix + e;                                            \
    __VA_ARGS__                                                                          \
  }

struct Geo {
  long long npix;
  int n;                 // views per scene
  int nchunk;
  long long b_scene_stride;   // elements between scenes of b (0 = shared)
};

__device__ __forceinline__ const cd* b_of(const cd* b, const Geo& G, int view) {
  return b + (size_t)(view / G.n) * G.b_scene_stride + (size_t)(view % G.n) * G.npix;
}
__device__ __forceinline__ const cd* chi_of(const cd* chi, const Geo& G, int view) {
  return chi + (size_t)(view / G.n) * G.npix;
}

// x = b, tmp = chi x
__global__ void __launch_bounds__(TH) init_kernel(Geo G, const cd* __restrict__ chi, const cd* __restrict__ b,
                                                  cd* __restrict__ x, cd* __restrict__ tmp) {
  const int view = blockIdx.y;
  const long long npix = G.npix;
  const cd* bv = b_of(b, G, view);
  const cd* cv = chi_of(chi, G, view);
  ELEM_LOOP({
    const cd bb = bv[e];
    x[i] = bb;
    tmp[i] = cmul(cv[e], bb);
  })
}

// r = b - (x - g), rhat = r, p = v = 0; partials ||b||^2, ||r||^2
__global__ void __launch_bounds__(TH) init2_kernel(Geo G, const cd* __restrict__ b, const cd* __restrict__ x, Vecs V) {
  const int view = blockIdx.y;
  const long long npix = G.npix;
  const cd* bv = b_of(b, G, view);
  double4 acc = make_double4(0, 0, 0, 0);
  ELEM_LOOP({
    const cd bb = bv[e];
    const cd r = csub(bb, csub(x[i], V.g[i]));
    V.r[i] = r;
    V.rhat[i] = r;
    V.p[i] = mkc(0, 0);
    V.v[i] = mkc(0, 0);
    acc.x += bb.x * bb.x + bb.y * bb.y;
    acc.z += r.x * r.x + r.y * r.y;
  })
  block_reduce_store(acc, V.part, G.nchunk);
}

__global__ void sc_init_kernel(Geo G, int nviews, double tol, Vecs V) {
  const int view = blockIdx.x * blockDim.x + threadIdx.x;
  if (view >= nviews) return;
  const double4 s = chunk_sum(V.part, view, G.nchunk);
  ViewScalars& q = V.sc[view];
  const double nb = sqrt(s.x);
  q.nb = nb > 0.0 ? nb : 1.0;
  q.res = sqrt(s.z) / q.nb;
  q.rho = q.alpha = q.omega = mkc(1, 0);
  q.active = q.res > tol;
  q.restart = 0;
  if (q.active) atomicAdd(V.nactive, 1);
}

// partials <rhat, r>, <r, r>
__global__ void __launch_bounds__(TH) dots1_kernel(Geo G, Vecs V) {
  const int view = blockIdx.y;
  const long long npix = G.npix;
  double4 acc = make_double4(0, 0, 0, 0);
  ELEM_LOOP({
    const cd r = V.r[i];
    const cd d = conjmul(V.rhat[i], r);
    acc.x += d.x;
    acc.y += d.y;
    acc.z += r.x * r.x + r.y * r.y;
  })
  block_reduce_store(acc, V.part, G.nchunk);
}

// restart test, beta, rho (forward.py:217-234)
__global__ void sc1_kernel(Geo G, int nviews, double tol, Vecs V) {
  const int view = blockIdx.x * blockDim.x + threadIdx.x;
  if (view >= nviews) return;
  const double4 s = chunk_sum(V.part, view, G.nchunk);
  ViewScalars& q = V.sc[view];
  q.active = q.res > tol;
  cd rho_new = mkc(s.x, s.y);
  const double rr = s.z;
  q.restart = cabs_(rho_new) < 1e-300 * rr;
  if (q.restart) {
    rho_new = mkc(rr, 0.0);      // <r, r> after rhat = r
    q.omega = q.alpha = q.rho = mkc(1, 0);
  }
  const cd rho_d = czero(q.rho) ? mkc(1, 0) : q.rho;
  const cd om_d = czero(q.omega) ? mkc(1, 0) : q.omega;
  q.beta = cmul(cdiv(rho_new, rho_d), cdiv(q.alpha, om_d));
  q.rho = rho_new;
}

// restart resets; p = r + beta (p - omega v) on active views; tmp = chi p
__global__ void __launch_bounds__(TH) p_kernel(Geo G, const cd* __restrict__ chi, Vecs V) {
  const int view = blockIdx.y;
  const long long npix = G.npix;
  const ViewScalars q = V.sc[view];
  const cd* cv = chi_of(chi, G, view);
  ELEM_LOOP({
    cd p = V.p[i], v = V.v[i];
    if (q.restart) {
      V.rhat[i] = V.r[i];
      p = v = mkc(0, 0);
      V.v[i] = v;
    }
    if (q.active) p = cadd(V.r[i], cmul(q.beta, csub(p, cmul(q.omega, v))));
    V.p[i] = p;
    V.tmp[i] = cmul(cv[e], p);
  })
}

// v = p - G_D(chi p) on active views; partial <rhat, v>
__global__ void __launch_bounds__(TH) v_kernel(Geo G, Vecs V) {
  const int view = blockIdx.y;
  const long long npix = G.npix;
  const int active = V.sc[view].active;
  double4 acc = make_double4(0, 0, 0, 0);
  ELEM_LOOP({
    cd v = V.v[i];
    if (active) {
      v = csub(V.p[i], V.g[i]);
      V.v[i] = v;
    }
    const cd d = conjmul(V.rhat[i], v);
    acc.x += d.x;
    acc.y += d.y;
  })
  block_reduce_store(acc, V.part, G.nchunk);
}

__global__ void sc2_kernel(Geo G, int nviews, Vecs V) {
  const int view = blockIdx.x * blockDim.x + threadIdx.x;
  if (view >= nviews) return;
  const double4 s = chunk_sum(V.part, view, G.nchunk);
  ViewScalars& q = V.sc[view];
  const cd den = mkc(s.x, s.y);
  q.alpha = cdiv(q.rho, czero(den) ? mkc(1, 0) : den);
}

// s = r - alpha v; tmp = chi s
__global__ void __launch_bounds__(TH) s_kernel(Geo G, const cd* __restrict__ chi, Vecs V) {
  const int view = blockIdx.y;
  const long long npix = G.npix;
  const cd alpha = V.sc[view].alpha;
  const cd* cv = chi_of(chi, G, view);
  ELEM_LOOP({
    const cd s = csub(V.r[i], cmul(alpha, V.v[i]));
    V.s[i] = s;
    V.tmp[i] = cmul(cv[e], s);
  })
}

// t = s - G_D(chi s); partials <t, t>, <t, s>
__global__ void __launch_bounds__(TH) t_kernel(Geo G, Vecs V) {
  const int view = blockIdx.y;
  const long long npix = G.npix;
  double4 acc = make_double4(0, 0, 0, 0);
  ELEM_LOOP({
    const cd s = V.s[i];
    const cd t = csub(s, V.g[i]);
    V.t[i] = t;
    acc.x += t.x * t.x + t.y * t.y;
    const cd d = conjmul(t, s);
    acc.z += d.x;
    acc.w += d.y;
  })
  block_reduce_store(acc, V.part, G.nchunk);
}

__global__ void sc3_kernel(Geo G, int nviews, Vecs V) {
  const int view = blockIdx.x * blockDim.x + threadIdx.x;
  if (view >= nviews) return;
  const double4 s = chunk_sum(V.part, view, G.nchunk);
  ViewScalars& q = V.sc[view];
  const double tt = s.x == 0.0 ? 1.0 : s.x;
  q.omega = mkc(s.z / tt, s.w / tt);
}

// x += alpha p + omega s, r = s - omega t on active views; partial <r, r>
__global__ void __launch_bounds__(TH) x_kernel(Geo G, cd* __restrict__ x, Vecs V) {
  const int view = blockIdx.y;
  const long long npix = G.npix;
  const ViewScalars q = V.sc[view];
  double4 acc = make_double4(0, 0, 0, 0);
  ELEM_LOOP({
    cd r = V.r[i];
    if (q.active) {
      const cd s = V.s[i];
      x[i] = cadd(cadd(x[i], cmul(q.alpha, V.p[i])), cmul(q.omega, s));
      r = csub(s, cmul(q.omega, V.t[i]));
      V.r[i] = r;
    }
    acc.x += r.x * r.x + r.y * r.y;
  })
  block_reduce_store(acc, V.part, G.nchunk);
}

__global__ void sc4_kernel(Geo G, int nviews, double tol, Vecs V) {
  const int view = blockIdx.x * blockDim.x + threadIdx.x;
  if (view >= nviews) return;
  ViewScalars& q = V.sc[view];
  if (q.active) q.res = sqrt(chunk_sum(V.part, view, G.nchunk).x) / q.nb;
  if (q.res > tol) atomicAdd(V.nactive, 1);
}

// true relative residuals ||x - b - G_D(chi x)|| / ||b|| (forward.py:278-284): partials
__global__ void __launch_bounds__(TH) resid_kernel(Geo G, const cd* __restrict__ b, const cd* __restrict__ x, Vecs V) {
  const int view = blockIdx.y;
  const long long npix = G.npix;
  const cd* bv = b_of(b, G, view);
  double4 acc = make_double4(0, 0, 0, 0);
  ELEM_LOOP({
    const cd bb = bv[e];
    const cd num = csub(csub(x[i], bb), V.g[i]);
    acc.x += num.x * num.x + num.y * num.y;
    acc.z += bb.x * bb.x + bb.y * bb.y;
  })
  block_reduce_store(acc, V.part, G.nchunk);
}

size_t vec_bytes(long long nviews, long long npix) { return (size_t)nviews * npix * sizeof(cd); }
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t plan(long long nviews, long long npix, char* base, Vecs* V) {
  size_t off = 0;
  cd** vecs[8] = {&V->r, &V->rhat, &V->p, &V->v, &V->s, &V->t, &V->tmp, &V->g};
  for (cd** pv : vecs) {
    if (base) *pv = (cd*)(base + off);
    off = align256(off + vec_bytes(nviews, npix));
  }
  const int nchunk = (int)((npix + CHUNK - 1) / CHUNK);
  if (base) V->part = (double4*)(base + off);
  off = align256(off + (size_t)nviews * nchunk * sizeof(double4));
  if (base) V->sc = (ViewScalars*)(base + off);
  off = align256(off + (size_t)nviews * sizeof(ViewScalars));
  if (base) V->nactive = (int*)(base + off);
  off = align256(off + sizeof(int));
  return off;
}

__global__ void resid_out_kernel(Geo G, int nviews, const double4* part, double* out) {
  const int view = blockIdx.x * blockDim.x + threadIdx.x;
  if (view >= nviews) return;
  const double4 s = chunk_sum(part, view, G.nchunk);
  const double dd = sqrt(s.z);
  out[view] = sqrt(s.x) / (dd > 0.0 ? dd : 1.0);
}

}  // namespace

extern "C" size_t pdf_solver_workspace_bytes(const pdf_ctx* c, int32_t count_views) {
  int M = 0, dt = 0;
  if (!c || count_views < 1 || pdf_ctx_info(c, &M, &dt) != PDF_OK) return 0;
  Vecs V{};
  return plan(count_views, (long long)M * M, nullptr, &V) + 256;
}

extern "C" int pdf_solve_total_field(pdf_ctx* c, const void* chi, const void* b, int64_t b_scene_stride, void* x,
                                     int32_t S, int32_t n, double tol, int32_t maxiter, void* workspace,
                                     size_t workspace_bytes, double* residuals, int32_t* iters_out, void* stream) {
  int M = 0, dt = 0;
  if (!c || !chi || !b || !x || !workspace || S < 1 || n < 1 || maxiter < 0 || !(tol >= 0.0))
    return pdf_fail(PDF_EINVAL, "pdf_solve_total_field: bad argument");
  if (pdf_ctx_info(c, &M, &dt) != PDF_OK) return PDF_EINVAL;
  if (dt != PDF_F64) return pdf_fail(PDF_EINVAL, "pdf_solve_total_field: the forward solve runs in float64");
  cudaStream_t st = (cudaStream_t)stream;
  const long long npix = (long long)M * M;
  const int nviews = S * n;
  Vecs V{};
  char* base = (char*)(((uintptr_t)workspace + 255) & ~uintptr_t(255));
  if (plan(nviews, npix, nullptr, &V) + (base - (char*)workspace) > workspace_bytes)
    return pdf_fail(PDF_ENOMEM, "pdf_solve_total_field: workspace too small (pdf_solver_workspace_bytes)");
  plan(nviews, npix, base, &V);
  Geo G{npix, n, (int)((npix + CHUNK - 1) / CHUNK), b_scene_stride};
  const dim3 eg(G.nchunk, nviews), sg((nviews + 127) / 128);
  const cd* chid = (const cd*)chi;
  const cd* bd = (const cd*)b;
  cd* xd = (cd*)x;
  int rc;
  auto gd = [&](void) { return pdf_apply_gd(c, V.tmp, V.g, nviews, 0, stream); };
  int nact = 0;
  auto read_active = [&](bool reset) -> int {
    PDF_CK(cudaMemcpyAsync(&nact, V.nactive, sizeof(int), cudaMemcpyDeviceToHost, st));
    PDF_CK(cudaStreamSynchronize(st));
    if (reset) PDF_CK(cudaMemsetAsync(V.nactive, 0, sizeof(int), st));
    return PDF_OK;
  };

  PDF_CK(cudaMemsetAsync(V.nactive, 0, sizeof(int), st));
  init_kernel<<<eg, TH, 0, st>>>(G, chid, bd, xd, V.tmp);
  if ((rc = gd()) != PDF_OK) return rc;
  init2_kernel<<<eg, TH, 0, st>>>(G, bd, xd, V);
  sc_init_kernel<<<sg, 128, 0, st>>>(G, nviews, tol, V);
  PDF_CK(cudaGetLastError());
  if ((rc = read_active(true)) != PDF_OK) return rc;
  auto step = [&](bool count_active) -> int {
    dots1_kernel<<<eg, TH, 0, st>>>(G, V);
    sc1_kernel<<<sg, 128, 0, st>>>(G, nviews, tol, V);
    p_kernel<<<eg, TH, 0, st>>>(G, chid, V);
    int r_;
    if ((r_ = gd()) != PDF_OK) return r_;
    v_kernel<<<eg, TH, 0, st>>>(G, V);
    sc2_kernel<<<sg, 128, 0, st>>>(G, nviews, V);
    s_kernel<<<eg, TH, 0, st>>>(G, chid, V);
    if ((r_ = gd()) != PDF_OK) return r_;
    t_kernel<<<eg, TH, 0, st>>>(G, V);
    sc3_kernel<<<sg, 128, 0, st>>>(G, nviews, V);
    x_kernel<<<eg, TH, 0, st>>>(G, xd, V);
    if (count_active) PDF_CK(cudaMemsetAsync(V.nactive, 0, sizeof(int), st));
    sc4_kernel<<<sg, 128, 0, st>>>(G, nviews, tol, V);
    return PDF_OK;
  };
  int it = 0;
  bool converged = nact == 0 && maxiter > 0;
  while (!converged && it < maxiter - 1) {
    // iterations it .. it + k - 1 are each preceded by a check the reference makes;
    // the last check that can succeed is the one before iteration maxiter - 1
    const int k = std::min(CHECK_EVERY, maxiter - 1 - it);
    for (int j = 0; j < k; ++j)
      if ((rc = step(j == k - 1)) != PDF_OK) return rc;
    PDF_CK(cudaGetLastError());
    it += k;
    if ((rc = read_active(false)) != PDF_OK) return rc;
    converged = nact == 0;
  }
  if (!converged && maxiter > 0) {   // the reference runs iteration maxiter - 1 before it raises
    if ((rc = step(false)) != PDF_OK) return rc;
    ++it;
  }
  if (iters_out) *iters_out = it;
  if (!converged) {
    std::vector<ViewScalars> h(nviews);
    PDF_CK(cudaMemcpyAsync(h.data(), V.sc, sizeof(ViewScalars) * nviews, cudaMemcpyDeviceToHost, st));
    PDF_CK(cudaStreamSynchronize(st));
    int above = 0;
    double worst = 0.0;
    for (const auto& q : h) {
      above += q.res > tol;
      worst = std::max(worst, q.res);
    }
    char msg[200];
    snprintf(msg, sizeof msg, "forward solve: %d view(s) above tol after %d iterations (max residual %.3e)", above,
             maxiter, worst);
    return pdf_fail(PDF_ENOCONV, msg);
  }
  if (residuals) {
    // true residuals of the returned fields (forward.py:267-269 via _relative_residuals)
    Geo Gx = G;
    Gx.b_scene_stride = (long long)n * npix;                       // x as the "b" operand: [S][n] layout
    init_kernel<<<eg, TH, 0, st>>>(Gx, chid, xd, V.s, V.tmp);       // s = x (scratch), tmp = chi x
    if ((rc = gd()) != PDF_OK) return rc;
    resid_kernel<<<eg, TH, 0, st>>>(G, bd, xd, V);
    resid_out_kernel<<<sg, 128, 0, st>>>(G, nviews, V.part, residuals);
    PDF_CK(cudaGetLastError());
  }
  return PDF_OK;
}
