// FP64 tensor-core helpers (mma.sync.aligned.m8n8k4 .f64, "DMMA").
//
// Fragment layouts (PTX ISA; g = lane >> 2, t = lane & 3):
//   A (8 x 4, row) : lane holds A[g][t]
//   B (4 x 8, col) : lane holds B[t][g]
//   C/D (8 x 8)    : lane holds D[g][2t], D[g][2t + 1]
#pragma once
#include <cuda_runtime.h>

namespace pdf {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// C (Mr x Nc) = A (Mr x Kd) B (Kd x Nc) for small complex float64 matrices
// whose entries come from functors (shared-memory arrays or twiddle-table
// lookups): 8x8 output tiles spread over the CTA's warps, 4-wide k steps, one
// complex product = four real MMAs.  Used for the corner-sparse DFT
// contractions of expand / truncate (spectral.py:56-79).  Every warp of the
// CTA must call it (mma.sync is warp-collective).
template <typename FA, typename FB, typename FO>
__device__ __forceinline__ void cgemm_dmma(int Mr, int Nc, int Kd, FA a_at, FB b_at, FO out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int mt = (Mr + 7) >> 3, nt = (Nc + 7) >> 3;
  for (int tile = warp; tile < mt * nt; tile += nw) {
    const int m0 = (tile / nt) * 8, n0 = (tile % nt) * 8;
    double cr0 = 0.0, cr1 = 0.0, ci0 = 0.0, ci1 = 0.0;
    for (int k0 = 0; k0 < Kd; k0 += 4) {
      const int k = k0 + t;
      const double2 av = (m0 + g < Mr && k < Kd) ? a_at(m0 + g, k) : make_double2(0.0, 0.0);
      const double2 bv = (k < Kd && n0 + g < Nc) ? b_at(k, n0 + g) : make_double2(0.0, 0.0);
      dmma(cr0, cr1, av.x, bv.x);
      dmma(ci0, ci1, av.x, bv.y);
      dmma(cr0, cr1, -av.y, bv.y);
      dmma(ci0, ci1, av.y, bv.x);
    }
    const int row = m0 + g, c0 = n0 + 2 * t;
    if (row < Mr) {
      if (c0 < Nc) out(row, c0, make_double2(cr0, ci0));
      if (c0 + 1 < Nc) out(row, c0 + 1, make_double2(cr1, ci1));
    }
  }
}

}  // namespace pdf
