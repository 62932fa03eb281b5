// Reconstruction metrics on the device (reference
// reconstruct.py:243-254):
//   relative_error   ||Re eps_hat - Re eps_true||_F / ||Re eps_true||_F
//   count_components number of 4-connected components of {Re eps > threshold}
//                    (scipy.ndimage.label with the 4-neighbour structure)
// Inputs are the real parts of float64 images read with an element stride
// (1 = float64 image, 2 = interleaved complex128), plus an offset added to
// every real part (eps = chi + 1 when the caller passes contrast images).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pdf_abi.h"
#include "pdf_internal.h"

namespace {

constexpr int RE_THREADS = 256;

// one CTA per image: per-thread strided partial sums, then a fixed shared-memory
// tree (deterministic, no atomics)
__global__ void __launch_bounds__(RE_THREADS) relerr_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                           int stride, long long npix, double offset,
                                                           double* __restrict__ out) {
  __shared__ double sn[RE_THREADS], sd[RE_THREADS];
  const long long base = (long long)blockIdx.x * npix * stride;
  double num = 0.0, den = 0.0;
  for (long long p = threadIdx.x; p < npix; p += RE_THREADS) {
    const double eb = b[base + p * stride] + offset;
    const double d = (a[base + p * stride] + offset) - eb;
    num = fma(d, d, num);
    den = fma(eb, eb, den);
  }
  sn[threadIdx.x] = num;
  sd[threadIdx.x] = den;
  __syncthreads();
  for (int h = RE_THREADS / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
      sn[threadIdx.x] += sn[threadIdx.x + h];
      sd[threadIdx.x] += sd[threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = sqrt(sn[0]) / sqrt(sd[0]);
}

// ---- connected components: union-find over a forest whose parent links always
// point to a smaller pixel index (atomicMin keeps that invariant), so every
// component ends with exactly one root L[p] == p.
__device__ __forceinline__ bool fg(const double* x, long long i, int stride, double offset, double thr) {
  return x[i * stride] + offset > thr;
}

// labels are image-local pixel indices (image k's labels live at L + k * npix)
__global__ void ccl_init_kernel(const double* __restrict__ x, int stride, long long npix, long long total,
                                double offset, double thr, int* __restrict__ L) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) L[i] = fg(x, i, stride, offset, thr) ? (int)(i % npix) : -1;
}

__device__ __forceinline__ int find_root(volatile int* L, int x) {
  int y;
  while ((y = L[x]) != x) x = y;
  return x;
}

__device__ void unite(int* L, int a, int b) {
  for (;;) {
    a = find_root(L, a);
    b = find_root(L, b);
    if (a == b) return;
    if (a < b) { const int t = a; a = b; b = t; }
    const int old = atomicMin(&L[a], b);
    if (old == a) return;   // a was a root and now hangs under b
    a = old;                // a had been re-linked meanwhile: retry from its new parent
  }
}

__global__ void ccl_merge_kernel(int m1, int m2, long long total, int* __restrict__ Lall) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const long long npix = (long long)m1 * m2;
  int* L = Lall + (i / npix) * npix;
  const int p = (int)(i % npix);
  if (L[p] < 0) return;
  const int r = p / m2, c = p % m2;
  if (c > 0 && L[p - 1] >= 0) unite(L, p, p - 1);
  if (r > 0 && L[p - m2] >= 0) unite(L, p, p - m2);
}

__global__ void ccl_count_kernel(long long npix, long long total, const int* __restrict__ Lall, int* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int p = (int)(i % npix);
  if (Lall[i] == p) atomicAdd(&out[i / npix], 1);   // integer count: order-independent
}

}  // namespace

extern "C" int pdf_relative_error(const double* eps_hat, const double* eps_true, int32_t stride, int64_t n_pix,
                                  int32_t count, double offset, double* out, void* stream) {
  if (!eps_hat || !eps_true || !out || stride < 1 || n_pix < 1 || count < 1)
    return pdf_fail(PDF_EINVAL, "pdf_relative_error: bad argument");
  relerr_kernel<<<count, RE_THREADS, 0, (cudaStream_t)stream>>>(eps_hat, eps_true, stride, n_pix, offset, out);
  PDF_CK(cudaGetLastError());
  return PDF_OK;
}

extern "C" int pdf_count_components(const double* eps, int32_t stride, int32_t m1, int32_t m2, int32_t count,
                                    double offset, double threshold, int32_t* labels, int32_t* out, void* stream) {
  if (!eps || !labels || !out || stride < 1 || m1 < 1 || m2 < 1 || count < 1)
    return pdf_fail(PDF_EINVAL, "pdf_count_components: bad argument");
  if ((long long)m1 * m2 >= 0x7fffffffLL) return pdf_fail(PDF_EINVAL, "pdf_count_components: image too large");
  cudaStream_t st = (cudaStream_t)stream;
  const long long npix = (long long)m1 * m2, total = npix * count;
  const int th = 256;
  const unsigned blocks = (unsigned)((total + th - 1) / th);
  PDF_CK(cudaMemsetAsync(out, 0, sizeof(int32_t) * count, st));
  ccl_init_kernel<<<blocks, th, 0, st>>>(eps, stride, npix, total, offset, threshold, labels);
  ccl_merge_kernel<<<blocks, th, 0, st>>>(m1, m2, total, labels);
  ccl_count_kernel<<<blocks, th, 0, st>>>(npix, total, labels, out);
  PDF_CK(cudaGetLastError());
  return PDF_OK;
}
