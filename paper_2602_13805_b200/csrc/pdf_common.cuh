// Common device helpers for the PDF solver hot path (sm_100a).
//
// Complex numbers are stored interleaved (re, im) as float2 / double2 so an
// n x m1 x m2 field stack is one contiguous c64 / c128 array with the same
// memory image as numpy's complex64 / complex128.
#pragma once
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <stdint.h>

namespace cg = cooperative_groups;

namespace pdf {

template <typename T> struct cx;
template <> struct cx<float> { using t = float2; };
template <> struct cx<double> { using t = double2; };
template <typename T> using C = typename cx<T>::t;

template <typename T> __host__ __device__ __forceinline__ C<T> mk(T a, T b) { C<T> r; r.x = a; r.y = b; return r; }
template <typename T> __host__ inline C<T> mk_host(double a, double b) { C<T> r; r.x = (T)a; r.y = (T)b; return r; }
template <typename T> __device__ __forceinline__ C<T> cadd(C<T> a, C<T> b) { return mk<T>(a.x + b.x, a.y + b.y); }
template <typename T> __device__ __forceinline__ C<T> csub(C<T> a, C<T> b) { return mk<T>(a.x - b.x, a.y - b.y); }
template <typename T> __device__ __forceinline__ C<T> cmul(C<T> a, C<T> b) {
  return mk<T>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
template <typename T> __device__ __forceinline__ C<T> cmulc(C<T> a, C<T> b) {
  return mk<T>(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
template <typename T> __device__ __forceinline__ C<T> conj_(C<T> a) { return mk<T>(a.x, -a.y); }
template <typename T> __device__ __forceinline__ C<T> cscale(C<T> a, T s) { return mk<T>(a.x * s, a.y * s); }
template <typename T> __device__ __forceinline__ T cabs2(C<T> a) { return a.x * a.x + a.y * a.y; }
template <typename T> __device__ __forceinline__ C<T> cdiv(C<T> a, C<T> b) {
  // plain formula, as numpy's complex division (no Smith scaling needed at
  // these magnitudes)
  T d = b.x * b.x + b.y * b.y;
  return mk<T>((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
template <typename T> __device__ __forceinline__ C<T> czero() { return mk<T>(T(0), T(0)); }

template <typename T> __device__ __forceinline__ C<T> shfl_xor(C<T> v, int m) {
  return mk<T>(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}

template <typename T> __device__ __forceinline__ T sqrt_(T x);
template <> __device__ __forceinline__ float sqrt_<float>(float x) { return sqrtf(x); }
template <> __device__ __forceinline__ double sqrt_<double>(double x) { return sqrt(x); }
template <typename T> __device__ __forceinline__ T exp_(T x);
template <> __device__ __forceinline__ float exp_<float>(float x) { return expf(x); }
template <> __device__ __forceinline__ double exp_<double>(double x) { return exp(x); }

// mbarrier + bulk copy (TMA engine, non-tensor) helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(void* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init_cluster() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(void* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(void* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// global -> the same shared offset in every CTA of `mask` (cluster), completion
// counted in bytes on each destination CTA's mbarrier at `bar`'s offset
__device__ __forceinline__ void bulk_copy_multicast(void* dst, const void* src, unsigned bytes, void* bar,
                                                    unsigned short mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
      "%4;\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

// global -> this CTA's shared memory (TMA engine, 1-D bulk copy), completion in bytes on `bar`
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, void* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(void* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(void* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// 16-byte asynchronous global -> shared copy (LDGSTS); zero-fills when !pred
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Programmatic dependent launch.  Kernels of the hot loop are launched with
// programmatic stream serialization: code before pdl_wait() may overlap the
// previous kernel, so it only touches data finalised two or more launches
// earlier (weights, Adam moments, operators, constants); pdl_trigger() lets
// the next kernel start its own prologue.  Both are no-ops without PDL.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// Measurement timeline (pdf_timeline; off unless a launch carries a slot):
// per slot the first CTA entry, the first CTA past the dependency wait and
// the last CTA exit, in globaltimer nanoseconds.
constexpr int TL_SLOTS = 128;   // = PDF_TL_SLOTS (pdf_abi.h)
__device__ unsigned long long g_tl[TL_SLOTS][3];
__device__ __forceinline__ void tl_mark(int slot1, int k) {
  if (slot1 <= 0 || threadIdx.x != 0) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (k < 2) atomicMin(&g_tl[slot1 - 1][k], t); else atomicMax(&g_tl[slot1 - 1][2], t);
}
// exit stamp on every return path of a kernel (measurement timeline)
struct TlExit {
  int slot1;
  __device__ __forceinline__ ~TlExit() { tl_mark(slot1, 2); }
};
// stage stamps inside a kernel: the last CTA to reach stage k (measurement)
constexpr int TL_STAGES = 8;
__device__ unsigned long long g_tls[TL_SLOTS][TL_STAGES];
__device__ __forceinline__ void tl_stage(int slot1, int k) {
  if (slot1 <= 0 || threadIdx.x != 0) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  atomicMax(&g_tls[slot1 - 1][k], t);
}
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// numerically stable logistic, scipy.special.expit semantics
template <typename T> __device__ __forceinline__ T sigmoid_(T z) {
  if (z >= T(0)) { T e = exp_<T>(-z); return T(1) / (T(1) + e); }
  T e = exp_<T>(z);
  return e / (T(1) + e);
}

// ---------------------------------------------------------------------------
// Warp FFT of length P = 32*E, one transform per warp.
//
// Element n = l + 32*k lives in lane l, register k.  The forward transform is
// decimation-in-frequency: an E-point DFT over the registers (stride 32),
// a twiddle exp(-2 pi i l q / P), then a 32-point DFT across the lanes with
// five shuffle butterflies.  Lane l, register q then holds the spectrum at
// frequency q + E * bitrev5(l).  The inverse consumes exactly that order
// (decimation in time) and returns natural order, so a convolution never
// permutes data: the pointwise kernel is stored in the same permuted order.
// Both directions are unnormalised.
//
// tw[k] = exp(-2 pi i k / P), k < P, lives in shared memory.
// ---------------------------------------------------------------------------

// exp(-2 pi i j / N) for compile-time N <= 16 (N a power of two)
template <typename T, int N, int J>
struct RootTab {
  __device__ __forceinline__ static C<T> get() {
    constexpr double c16[16] = {1.0, 0.92387953251128674, 0.70710678118654757, 0.38268343236508984,
                                0.0, -0.38268343236508984, -0.70710678118654757, -0.92387953251128674,
                                -1.0, -0.92387953251128674, -0.70710678118654757, -0.38268343236508984,
                                0.0, 0.38268343236508984, 0.70710678118654757, 0.92387953251128674};
    constexpr int idx = (J * (16 / N)) & 15;
    constexpr int sidx = (idx + 12) & 15;  // sin(theta) = cos(theta - pi/2)
    return mk<T>(T(c16[idx]), T(-c16[sidx]));
  }
};

// multiply by exp(SIGN * 2 pi i J / N) with exact handling of the trivial roots
template <typename T, int N, int J, int SIGN>
__device__ __forceinline__ C<T> twiddle_ct(C<T> v) {
  constexpr int j = ((J % N) + N) % N;
  if constexpr (j == 0) {
    return v;
  } else if constexpr (4 * j == N) {       // exp(-i pi/2) = -i  (SIGN=-1)
    return SIGN < 0 ? mk<T>(v.y, -v.x) : mk<T>(-v.y, v.x);
  } else if constexpr (2 * j == N) {
    return mk<T>(-v.x, -v.y);
  } else if constexpr (4 * j == 3 * N) {
    return SIGN < 0 ? mk<T>(-v.y, v.x) : mk<T>(v.y, -v.x);
  } else {
    C<T> w = RootTab<T, N, j>::get();     // exp(-2 pi i j/N)
    if (SIGN > 0) w.y = -w.y;
    return cmul<T>(v, w);
  }
}

template <int B, int V> struct BitRev {
  static constexpr int value = (B <= 1) ? 0 : (((V & 1) << (B - 1)) | BitRev<B - 1, (V >> 1)>::value);
};
template <int V> struct BitRev<0, V> { static constexpr int value = 0; };
template <int V> struct BitRev<1, V> { static constexpr int value = V & 1; };

template <int E> struct Log2 { static constexpr int value = 1 + Log2<E / 2>::value; };
template <> struct Log2<1> { static constexpr int value = 0; };

// in-register DIF butterflies for one stage (span = LEN/2) over all blocks
template <typename T, int E, int LEN, int SIGN, int START, int J>
struct RegStage {
  __device__ __forceinline__ static void run(C<T> (&a)[E]) {
    if constexpr (START < E) {
      if constexpr (J < LEN / 2) {
        C<T> u = a[START + J], v = a[START + J + LEN / 2];
        a[START + J] = cadd<T>(u, v);
        a[START + J + LEN / 2] = twiddle_ct<T, LEN, J, SIGN>(csub<T>(u, v));
        RegStage<T, E, LEN, SIGN, START, J + 1>::run(a);
      } else {
        RegStage<T, E, LEN, SIGN, START + LEN, 0>::run(a);
      }
    }
  }
};

template <typename T, int E, int LEN, int SIGN>
struct RegDif {
  __device__ __forceinline__ static void run(C<T> (&a)[E]) {
    if constexpr (LEN >= 2) {
      RegStage<T, E, LEN, SIGN, 0, 0>::run(a);
      RegDif<T, E, LEN / 2, SIGN>::run(a);
    }
  }
};

template <typename T, int E, int I>
struct RegPermute {
  __device__ __forceinline__ static void run(const C<T> (&a)[E], C<T> (&o)[E]) {
    if constexpr (I < E) {
      o[BitRev<Log2<E>::value, I>::value] = a[I];
      RegPermute<T, E, I + 1>::run(a, o);
    }
  }
};

// natural-order E-point DFT over registers: x[q] <- sum_k x[k] exp(SIGN 2 pi i k q / E)
template <typename T, int E, int SIGN>
__device__ __forceinline__ void reg_dft(C<T> (&x)[E]) {
  if constexpr (E > 1) {
    RegDif<T, E, E, SIGN>::run(x);
    C<T> o[E];
    RegPermute<T, E, 0>::run(x, o);
#pragma unroll
    for (int i = 0; i < E; ++i) x[i] = o[i];
  }
}

template <typename T> __device__ __forceinline__ C<T> tw_get(const C<T>* tw, int k, bool inv) {
  C<T> w = tw[k];
  if (inv) w.y = -w.y;
  return w;
}

// Lane stages.  For E >= 2 each stage pairs lanes l, l^h and splits the
// butterflies between them instead of having both lanes compute both halves:
// the lower lane keeps register slots [0, E/2), the upper lane [E/2, E); each
// lane ships the other half to its partner (one shuffle per pair), computes
// its butterflies completely and stores sum -> slot j, (difference x twiddle)
// -> slot j + E/2.  Every stage therefore swaps lane bit h with the top
// register bit: after the five stages lane p, slot s holds the spectrum at
//   f = R + E * bitrev5(L),  L = ((p & 15) << 1) | (s >> (e-1)),
//                            R = ((p >> 4) << (e-1)) | (s & (E/2 - 1)),  E = 2^e
// (host side: spectrum_slot_freq).  The inverse mirrors the stages exactly.
// Per-lane twiddles are the same for every transform a lane runs, so they are
// read from the shared table once per thread and kept in registers:
//   st[i]  = tw[(lane & (h-1)) * P/(2h)] for the lane stage h = 16 >> i
//   rq[q]  = tw[(lane * q) mod P]         for the register-to-lane twiddle
template <typename T, int E>
struct LaneTw {
  // E >= 8 keeps the register-to-lane twiddles in the shared table (register
  // pressure of the large-grid passes; M = 128 is not a BASELINE config)
  static constexpr bool RQREG = E <= 4;
  C<T> st[5];
  C<T> rq[RQREG ? E : 1];
  const C<T>* tw;
  int ln;
  __device__ __forceinline__ void load(const C<T>* __restrict__ tw_, int lane) {
    constexpr int P = 32 * E;
    tw = tw_;
    ln = lane;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const int h = 16 >> i;
      st[i] = tw_[(lane & (h - 1)) * (P / (2 * h))];
    }
    if constexpr (RQREG) {
#pragma unroll
      for (int q = 0; q < E; ++q) rq[q] = tw_[(lane * q) & (P - 1)];
    }
  }
  __device__ __forceinline__ C<T> r(int q) const {
    if constexpr (RQREG) return rq[q];
    else return tw[(ln * q) & (32 * E - 1)];
  }
};

template <typename T, int E>
__device__ __forceinline__ void warp_fft_fwd(C<T> (&x)[E], const LaneTw<T, E>& lt, int lane) {
  reg_dft<T, E, -1>(x);
#pragma unroll
  for (int q = 1; q < E; ++q) x[q] = cmul<T>(x[q], lt.r(q));
  if constexpr (E == 1) {
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const int h = 16 >> i;
      const bool upper = (lane & h) != 0;
      C<T> o = shfl_xor<T>(x[0], h);
      x[0] = upper ? cmul<T>(csub<T>(o, x[0]), lt.st[i]) : cadd<T>(x[0], o);
    }
  } else {
    constexpr int H2 = E / 2;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const int h = 16 >> i;
      const bool upper = (lane & h) != 0;
      C<T> w = lt.st[i];
      if (upper) w = mk<T>(-w.x, -w.y);
#pragma unroll
      for (int j = 0; j < H2; ++j) {
        const C<T> own = upper ? x[j + H2] : x[j];
        const C<T> snd = upper ? x[j] : x[j + H2];
        const C<T> rcv = shfl_xor<T>(snd, h);
        x[j] = cadd<T>(own, rcv);
        x[j + H2] = cmul<T>(csub<T>(own, rcv), w);
      }
    }
  }
}

template <typename T, int E>
__device__ __forceinline__ void warp_fft_inv(C<T> (&x)[E], const LaneTw<T, E>& lt, int lane) {
  if constexpr (E == 1) {
#pragma unroll
    for (int i = 4; i >= 0; --i) {
      const int h = 16 >> i;
      const bool upper = (lane & h) != 0;
      const C<T> w = conj_<T>(lt.st[i]);
      C<T> o = shfl_xor<T>(x[0], h);
      x[0] = upper ? csub<T>(o, cmul<T>(x[0], w)) : cadd<T>(x[0], cmul<T>(o, w));
    }
  } else {
    constexpr int H2 = E / 2;
#pragma unroll
    for (int i = 4; i >= 0; --i) {
      const int h = 16 >> i;
      const bool upper = (lane & h) != 0;
      C<T> w = conj_<T>(lt.st[i]);
      if (upper) w = mk<T>(-w.x, -w.y);
#pragma unroll
      for (int j = 0; j < H2; ++j) {
        const C<T> t = cmul<T>(x[j + H2], w);
        const C<T> own = cadd<T>(x[j], t);
        const C<T> oth = csub<T>(x[j], t);
        const C<T> rcv = shfl_xor<T>(oth, h);
        x[j] = upper ? rcv : own;
        x[j + H2] = upper ? own : rcv;
      }
    }
  }
#pragma unroll
  for (int q = 1; q < E; ++q) x[q] = cmulc<T>(x[q], lt.r(q));
  reg_dft<T, E, +1>(x);
}

// frequency held by lane p, register slot s after warp_fft_fwd (see above)
__host__ __device__ inline int spectrum_slot_freq(int p, int s, int E) {
  auto br5 = [](int l) { int r = 0; for (int i = 0; i < 5; ++i) r |= ((l >> i) & 1) << (4 - i); return r; };
  if (E == 1) return br5(p);
  int e = 0;
  while ((1 << e) < E) ++e;
  const int L = ((p & 15) << 1) | (s >> (e - 1));
  const int R = ((p >> 4) << (e - 1)) | (s & ((1 << (e - 1)) - 1));
  return R + E * br5(L);
}

// max over views of sum_c norms[v][c] (fixed-order partial sums, exact max):
// eps_reg's view power (cie.py:49-50).  Called by one full warp.
__device__ __forceinline__ double warp_max_view_power(const double* norms, int n, int np) {
  const int lane = threadIdx.x & 31;
  double mx = -1.0;
  for (int i = lane; i < n; i += 32) {
    double pw = 0.0;
    for (int c = 0; c < np; ++c) pw += norms[(size_t)i * np + c];
    mx = pw > mx ? pw : mx;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = t > mx ? t : mx;
  }
  return mx;
}

// deterministic fixed-order warp sum
template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// error word bits (sticky, per scene) -- mirrored in include/pdf_abi.h
enum : int {
  ERR_POLE = 1,
  ERR_NONFINITE_STATE = 2,
  ERR_NONFINITE_DATA = 4,
  ERR_NONFINITE_BOUND = 8,
  ERR_NONFINITE_TV = 16,
  ERR_NONFINITE_BRIDGE = 32,
  ERR_NONFINITE_GRAD = 64,
  ERR_NONFINITE_PARAM = 128,
};

}  // namespace pdf
