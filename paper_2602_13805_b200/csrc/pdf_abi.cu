// C-ABI implementation (see include/pdf_abi.h): context, workspace plan,
// kernel dispatch and the CUDA-graph replay of the training loop.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pdf_abi.h"
#include "pdf_internal.h"
#include "pdf_aux.cuh"
#include "pdf_common.cuh"
#include "pdf_net.cuh"
#include "pdf_net_mma.cuh"
#include "pdf_pixel.cuh"
#include "pdf_shard.cuh"
#include "pdf_pixel_stream.cuh"
#include "pdf_view.cuh"
#include "pdf_view_large.cuh"

using namespace pdf;

static thread_local std::string g_err;
// timeline slot (+1) stamped into the hot-loop kernel arguments while a
// timeline capture is on (pdf_timeline); 0 otherwise
static thread_local int g_tl_cur = 0, g_tl_iter = 0;
static int env_int(const char* name, int dflt);
// programmatic dependent launch for the hot-loop kernels (PDF_PDL=0 disables)
static const int g_pdl = env_int("PDF_PDL", 1);
// set around launches that must fully follow their stream predecessor (side-stream branches)
static thread_local int g_pdl_off = 0;

// cluster caps (tunable for experiments: PDF_NET_CLUSTER, PDF_VIEW_CLUSTER)
static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

static int fail(int code, const std::string& msg) {
  g_err = msg;
  if (code == PDF_ECUDA) (void)cudaGetLastError();   // do not leak a stale error into the next call
  return code;
}

int pdf_fail(int code, const std::string& msg) { return fail(code, msg); }

#define CK_CUDA(expr)                                                               \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail(PDF_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));   \
  } while (0)

#define TRY(x) do { int r_ = (x); if (r_ != PDF_OK) return r_; } while (0)

struct Ws {
  size_t off = 0;
  char* base = nullptr;
  template <typename U>
  U* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    U* p = base ? reinterpret_cast<U*>(base + off) : nullptr;
    off += count * sizeof(U);
    return p;
  }
};

struct pdf_ctx {
  pdf_desc d;
  int M, P, E, K, M0, CS, rows, D0, H, RB, TX, ntiles;
  // large-grid view path (pdf_view_large.cuh): partials per view, views per
  // spectrum chunk, data-GEMM pixel chunking
  int large, dgemm, NPV, chunk, dg_chunk, dg_nchunks, dg_nq;
  int split;         // pixel stage as numden / pixel_a / pixel_b (pdf_shard.cuh) in the training loop
  // peer scatter of the unfused backward's gradient (pdf_shard_step_c_scatter), set around the call
  double* const* sc_peers = nullptr;
  int sc_me = 0;
  long long sc_shard = 0;
  int xbwd;          // split network backward in the training loop (net_gh_x / net_adam_x)
  long long Np;
  size_t csz, rsz;   // complex / real element size
  // workspace
  void *khat, *twP, *twM, *hs, *J, *E_, *gJ, *gE, *grows, *alpha0, *alpha_hat, *galpha;
  void *x0, *cout, *h1, *h2, *gy, *gz2, *gz1, *ab;
  double *norms, *dloss, *part, *bd, *pix;
  void *spec, *gpart, *dpart;
  double* ghp;       // split backward: g_h slice partials [S][GH_NSL][rows][H]
  int* ticket;       // split backward: per k-block tickets [S][H / 64 + 1]
  // captured training graph with the Adam of layers 2 / 3 on a side branch:
  // activations and the Adam-t snapshot alternate between two buffers per iteration
  void *h1b, *h2b;
  int *tsnap, *tsnap_b;
  int capturing = 0, pend = 0;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_g3 = nullptr, ev_g2 = nullptr, ev_a2 = nullptr;
  // data part of g_alpha computed on the side branch while the pixel kernel runs
  void* gad = nullptr;
  int gad_ready = 0;
  int dfork_ok = 0, skip_data = 0;   // data term (split-K GEMM) on the side branch as well
  cudaStreamAttrValue l2_window = {};
  int l2_set = 0;
  cudaEvent_t ev_vf = nullptr, ev_gad = nullptr;
  double *red1, *red2;   // split pixel stage scratch (local reductions)
  int *err, *step;
  std::vector<double> c_inc_h, c_sca_h;
  double *c_inc, *c_sca;
  // graph cache
  cudaGraphExec_t gexec = nullptr;
  void *g_theta = nullptr, *g_m = nullptr, *g_v = nullptr, *g_trace = nullptr;
  cudaStream_t g_stream = nullptr;
  int g_iters = 0;
  int tl_on = 0;
};

template <typename T>
static void plan(pdf_ctx* c, Ws& w) {
  const pdf_desc& d = c->d;
  const size_t SN = (size_t)d.S * d.n;
  const size_t img = (size_t)c->M * c->M;
  c->khat = w.take<C<T>>((size_t)c->P * c->P);
  c->twP = w.take<C<T>>(c->P);
  c->twM = w.take<C<T>>(c->M);
  c->hs = w.take<C<T>>((size_t)d.R * c->M0);   // spectral receiver operator (pdf_aux.cuh)
  c->J = w.take<C<T>>(SN * img);
  c->E_ = w.take<C<T>>(SN * img);
  c->gJ = w.take<C<T>>(SN * img);
  c->gE = w.take<C<T>>(SN * img);
  c->grows = w.take<C<T>>(SN * d.R);
  c->alpha0 = w.take<C<T>>(SN * c->M0);
  c->alpha_hat = w.take<C<T>>(SN * c->M0);
  c->galpha = w.take<C<T>>(SN * c->M0);
  c->x0 = w.take<T>((size_t)d.S * c->rows * c->D0);
  c->cout = w.take<T>((size_t)d.S * c->D0);
  c->h1 = w.take<T>((size_t)d.S * c->rows * c->H);
  c->h2 = w.take<T>((size_t)d.S * c->rows * c->H);
  c->gy = w.take<T>((size_t)d.S * c->rows * c->D0);
  c->gz2 = w.take<T>((size_t)d.S * c->rows * c->H);
  c->gz1 = w.take<T>((size_t)d.S * c->rows * c->H);
  c->ab = w.take<T>((size_t)d.S * 4 * img);
  c->pix = w.take<double>((size_t)d.S * img * 12);
  c->norms = w.take<double>(SN * c->NPV);
  if (c->large) {
    c->spec = w.take<C<T>>((size_t)c->chunk * c->P * c->M);
    c->gpart = w.take<C<T>>(SN * c->NPV * c->M0);
  } else {
    c->spec = c->gpart = nullptr;
  }
  c->dpart = c->dgemm || c->dfork_ok ? w.take<C<T>>((size_t)d.S * c->dg_nchunks * d.n * d.R) : nullptr;
  c->ghp = c->xbwd ? w.take<double>((size_t)d.S * GH_NSL * c->rows * c->H) : nullptr;
  c->ticket = c->xbwd ? w.take<int>((size_t)d.S * (c->H / 64 + 1)) : nullptr;
  c->h1b = c->xbwd ? w.take<T>((size_t)d.S * c->rows * c->H) : nullptr;
  c->h2b = c->xbwd ? w.take<T>((size_t)d.S * c->rows * c->H) : nullptr;
  c->tsnap = c->xbwd ? w.take<int>(1) : nullptr;
  c->tsnap_b = c->xbwd ? w.take<int>(1) : nullptr;
  c->gad = c->xbwd ? w.take<C<T>>(SN * c->M0) : nullptr;
  c->red1 = c->split ? w.take<double>((size_t)d.S * (3 * img + 1)) : nullptr;
  c->red2 = c->split ? w.take<double>((size_t)d.S * (2 * img + 2)) : nullptr;
  c->dloss = w.take<double>(SN);
  c->part = w.take<double>((size_t)d.S * c->ntiles * 4);
  c->bd = w.take<double>((size_t)d.S * 6);
  c->c_inc = w.take<double>(d.S);
  c->c_sca = w.take<double>(d.S);
  c->err = w.take<int>(d.S);
  c->step = w.take<int>(2);
}

static int derive(pdf_ctx* c, const pdf_desc* d) {
  if (!d) return fail(PDF_EINVAL, "null desc");
  if (d->abi_version != PDF_ABI_VERSION) return fail(PDF_EINVAL, "abi version mismatch");
  if (d->dtype != PDF_F64 && d->dtype != PDF_F32) return fail(PDF_EINVAL, "dtype");
  if (d->m1 != d->m2) return fail(PDF_EINVAL, "only square grids (m1 == m2) are supported");
  const int M = d->m1;
  if (M != 16 && M != 32 && M != 64 && M != 128 && M != 256)
    return fail(PDF_EINVAL, "grid size must be a power of two in [16, 256]");
  if (d->mf < 1 || 2 * d->mf > M) return fail(PDF_EINVAL, "need 1 <= m_f and 2 m_f <= m1");
  if (d->S < 1 || d->n < 1 || d->R < 1) return fail(PDF_EINVAL, "S, n, R must be >= 1");
  c->d = *d;
  c->M = M;
  c->P = 2 * M;
  c->E = c->P / 32;
  c->K = 2 * d->mf;
  c->M0 = c->K * c->K;
  // 8-CTA clusters while one wave holds every view (latency), 4 once the batch
  // fills the GPU (half the cluster barriers per unit of work; measured -22%
  // view time at 128 scenes)
  // ... and one 16-warp CTA per view (no cluster, every transpose in the CTA's
  // own shared memory) once there are several views per SM and the view's
  // half-pruned spectrum fits (float64: M <= 64)
  const long long nviews = (long long)d->S * d->n;
  const bool solo_ok = d->dtype == PDF_F64 && c->M <= 64 && c->M >= 32;
  c->CS = env_int("PDF_VIEW_CLUSTER", nviews * 8 <= 4 * 148 ? 8 : (solo_ok && nviews >= 4 * 148 ? 1 : 4));
  if (c->CS != 4 && c->CS != 8 && !(c->CS == 1 && solo_ok))
    return fail(PDF_EINVAL, "view cluster size must be 4 or 8 (or 1: float64, M <= 64)");
  c->rows = d->joint ? 1 : d->n;
  c->D0 = 2 * c->M0 * (d->joint ? d->n : 1);
  c->H = 2 * c->D0;
  c->Np = (long long)c->H * c->D0 + c->H + (long long)c->H * c->H + c->H + (long long)c->D0 * c->H + c->D0;
  c->RB = (c->rows + 15) / 16;
  if (c->RB > 5) return fail(PDF_EINVAL, "at most 80 network rows (incidences) supported");
  c->TX = M < 32 ? M : 32;
  c->ntiles = (M / c->TX) * M;
  // M = 256 needs the multi-pass spectrum path; PDF_VIEW_LARGE=1 forces it for
  // M >= 32 (cross-checks the two paths on the small configs)
  c->large = M >= 256 || (env_int("PDF_VIEW_LARGE", 0) && M >= 32);
  c->NPV = c->large ? M / VL_ROWS : c->CS;
  c->chunk = c->dg_chunk = c->dg_nchunks = 0;
  if (c->large) {
    const size_t csz = d->dtype == PDF_F64 ? 16 : 8;
    // spectrum chunk: all 72 views of cfg5 in one set of passes (144 MiB) measured
    // fastest (1 707 us per iteration; 36 / 48 / 72 / 96 MiB chunks: 1 736 / 1 792 /
    // 1 740 / 1 759) -- fewer launches outweigh the L2 residency of a small chunk
    const long long budget = (long long)env_int("PDF_SPEC_MIB", 160) << 20;
    const long long per = (long long)2 * M * M * csz;
    long long ch = std::max(1LL, budget / per);
    c->chunk = (int)std::min<long long>(ch, (long long)d->S * d->n);
  }
  // data term as a split-K GEMM over all views of a scene (G_S read once per
  // scene instead of once per view): always on the large-grid path, and on
  // the cluster path for float64 batches (DMMA; measured -27% view_fwd at 128
  // scenes, +10 us per iteration for one scene where the in-kernel term wins)
  const int dg_env = env_int("PDF_DATA_GEMM", -1);
  c->dgemm = c->large || (M >= 32 && (dg_env == 1 || (dg_env < 0 && d->dtype == PDF_F64 && d->S >= 4)));
  c->dg_nq = 1;
  // measured slower than the fused pixel kernel (with its DMMA G_S^H) on every
  // config; kept as an option (PDF_SPLIT_PIXEL=1), covered by the sharded tests
  c->split = env_int("PDF_SPLIT_PIXEL", 0) && !d->joint;
  // latency regime: g_h and g_W + Adam as separate fully parallel launches
  // (measured: cfg2 -4 us, cfg3 167 -> 150 us per iteration, cfg5 unchanged)
  const int bx = env_int("PDF_BWD_X", 1);   // 2: force (experiments)
  c->xbwd = bx && d->dtype == PDF_F64 && c->rows <= 80 && (bx == 2 || (long long)d->S * (c->H / 8) <= 4 * 148);
  c->dfork_ok = c->xbwd && !c->large && d->n <= 80 && d->R <= 80 && env_int("PDF_DATA_FORK", 1);
  if (c->dgemm || c->dfork_ok) {
    const int npix = c->M0;   // the data GEMM contracts spectral coefficients (H = G_S o expand)
    // chunk granularity: 16 coefficients for the DMMA kernel (4 k-steps), the
    // staged sub-tile for the float32 one
    const int gk = d->dtype == PDF_F64 ? 16 : DG_KC;
    int want = std::max(1, (2 * 148 + d->S - 1) / d->S);
    want = std::max(1, std::min(want, npix / gk));
    c->dg_chunk = ((npix + want - 1) / want + gk - 1) / gk * gk;
    c->dg_nchunks = (npix + c->dg_chunk - 1) / c->dg_chunk;
    const int ntp = ((d->n + 7) / 8) * ((d->R + 8 * DM_NTL - 1) / (8 * DM_NTL));
    c->dg_nq = std::max(1, std::min(4, 8 / ntp));
    if (c->dgemm && (d->n > 80 || d->R > 80))
      return fail(PDF_EINVAL, "at most 80 incidences / receivers for the data GEMM");
  }
  c->rsz = d->dtype == PDF_F64 ? 8 : 4;
  c->csz = 2 * c->rsz;
  if (d->freeze_r && !d->r_fixed) return fail(PDF_EINVAL, "freeze_r requires r_fixed");
  if (!d->e_inc || !d->gd_kernel_hat || !d->gs_matrix || !d->data || !d->c_inc || !d->c_sca)
    return fail(PDF_EINVAL, "missing operator / data pointer");
  return PDF_OK;
}

extern "C" const char* pdf_last_error(void) { return g_err.c_str(); }
extern "C" int pdf_abi_version(void) { return PDF_ABI_VERSION; }

extern "C" size_t pdf_workspace_bytes(const pdf_desc* d) {
  pdf_ctx c;
  if (derive(&c, d) != PDF_OK) return 0;
  Ws w;
  if (d->dtype == PDF_F64) plan<double>(&c, w); else plan<float>(&c, w);
  return w.off + 256;
}

// ---------------------------------------------------------------------------
template <typename F>
static cudaError_t launch_cluster(F kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, dim3 cluster,
                                  void** args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster.x;
  attr[0].val.clusterDim.y = cluster.y;
  attr[0].val.clusterDim.z = cluster.z;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = g_pdl && !g_pdl_off;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelExC(&cfg, (const void*)kern, args);
}

template <typename K>
static cudaError_t prep(K kern, size_t smem) {
  cudaError_t e = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

template <typename K>
static cudaError_t plain_launch(K kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, void** args) {
  cudaError_t e = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl && !g_pdl_off;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, (const void*)kern, args);
}

template <typename T, int MODE>
static int launch_view(pdf_ctx* c, ViewArgs<T>& a, int count, cudaStream_t st) {
  const size_t smem = view_smem_bytes<T>(c->M, c->d.mf, c->d.R, c->CS);
  void* args[] = {&a};
  cudaError_t e;
  // 8 warps: 16-warp CTAs halve the column pass but need a whole SM's
  // registers, so under PDL they wait for the previous kernel to drain
  // (measured +8 us per view kernel at cfg2)
  static const int vt = env_int("PDF_VIEW_THREADS", 256);
  const int nthr = c->CS == 1 ? VIEW_SOLO_THREADS : std::min(vt, VIEW_MAX_THREADS);
  dim3 grid(c->CS, count), block(nthr), cl(c->CS, 1, 1);
  switch (c->E * 100 + c->CS) {
#define VCASE(EE, CC)                                               \
  case EE * 100 + CC: {                                             \
    auto k = view_kernel<T, EE, MODE, CC>;                          \
    e = prep(k, smem);                                              \
    if (e == cudaSuccess) e = launch_cluster(k, grid, block, smem, st, cl, args); \
    break;                                                          \
  }
    VCASE(1, 4) VCASE(1, 8) VCASE(2, 4) VCASE(2, 8) VCASE(4, 4) VCASE(4, 8) VCASE(8, 4) VCASE(8, 8)
    VCASE(2, 1) VCASE(4, 1)
#undef VCASE
    default: return fail(PDF_EINVAL, "unsupported FFT size / view cluster size (1, 4 or 8)");
  }
  if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("view kernel: ") + cudaGetErrorString(e));
  return PDF_OK;
}

template <typename T>
static ViewArgs<T> view_common(pdf_ctx* c) {
  ViewArgs<T> a = {};
  a.tl = g_tl_cur;
  a.M = c->M; a.mf = c->d.mf; a.R = c->d.R; a.n = c->d.n; a.CS = c->CS;
  a.khat = (const C<T>*)c->khat; a.twP = (const C<T>*)c->twP; a.twM = (const C<T>*)c->twM;
  a.hs = (const C<T>*)c->hs;
  return a;
}

// ---------------------------------------------------------------------------
// large-grid path: rows / cols / out passes per chunk of views
template <typename T>
static VLArgs<T> vl_common(pdf_ctx* c) {
  VLArgs<T> a = {};
  a.M = c->M; a.mf = c->d.mf; a.R = c->d.R; a.n = c->d.n; a.NPV = c->NPV;
  a.khat = (const C<T>*)c->khat; a.twP = (const C<T>*)c->twP; a.twM = (const C<T>*)c->twM;
  a.spec = (C<T>*)c->spec;
  a.tl = g_tl_cur;
  return a;
}

template <typename T, int E, int MODE>
static cudaError_t vl_chunk(pdf_ctx* c, VLArgs<T>& a, int cnt, cudaStream_t st) {
  constexpr int P = 32 * E, M = P / 2;
  void* args[] = {&a};
  a.nview = cnt;
  cudaError_t e = plain_launch(vl_rows_kernel<T, E, MODE>, dim3(M / VL_ROWS, cnt), dim3(256),
                               vl_rows_smem<T>(E, c->d.mf), st, args);
  const int nvc = sizeof(T) == 8 && E >= 4 ? 2 : 1;   // views per CTA of the cols pass
  if (e == cudaSuccess)
    e = plain_launch(vl_cols_kernel<T, E>, dim3(P / 8, (cnt + nvc - 1) / nvc), dim3(256), vl_cols_smem<T>(E), st, args);
  if (e == cudaSuccess)
    e = plain_launch(vl_out_kernel<T, E, MODE>, dim3(M / VL_ROWS, cnt), dim3(256), vl_out_smem<T>(E, c->d.mf), st,
                     args);
  return e;
}

template <typename T, int MODE>
static int vl_conv(pdf_ctx* c, VLArgs<T>& a, int count, cudaStream_t st) {
  for (int v0 = 0; v0 < count; v0 += c->chunk) {
    a.v0 = v0;
    const int cnt = std::min(c->chunk, count - v0);
    cudaError_t e;
    switch (c->E) {
      case 2: e = vl_chunk<T, 2, MODE>(c, a, cnt, st); break;
      case 4: e = vl_chunk<T, 4, MODE>(c, a, cnt, st); break;
      case 8: e = vl_chunk<T, 8, MODE>(c, a, cnt, st); break;
      case 16: e = vl_chunk<T, 16, MODE>(c, a, cnt, st); break;
      default: return fail(PDF_EINVAL, "unsupported FFT size on the large-grid path");
    }
    if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("large view pass: ") + cudaGetErrorString(e));
  }
  return PDF_OK;
}

// D = alpha_hat H^T - d over all views of a scene: the split-K GEMM runs over
// the M0 spectral coefficients (H = G_S o expand, pdf_aux.cuh), not the M^2
// pixels of J G_S^T
template <typename T>
static int data_term(pdf_ctx* c, const void* alpha_hat, cudaStream_t st) {
  DataArgs<T> g = {};
  g.n = c->d.n; g.R = c->d.R; g.npix = c->M0; g.chunk = c->dg_chunk; g.nchunks = c->dg_nchunks;
  g.J = (const C<T>*)alpha_hat; g.gs = (const C<T>*)c->hs; g.dpart = (C<T>*)c->dpart;
  g.data = (const C<T>*)c->d.data; g.mask = (const T*)c->d.mask; g.c_sca = c->c_sca;
  g.grows = (C<T>*)c->grows; g.dloss = c->dloss;
  g.nq = c->dg_nq;
  g.tl = g_tl_cur;
  void* args[] = {&g};
  cudaError_t e;
  if constexpr (sizeof(T) == 8)
    e = plain_launch(data_mma_kernel, dim3(c->dg_nchunks, c->d.S), dim3(256), dm_smem(g.n, g.R, g.nq), st, args);
  else
    e = plain_launch(data_gemm_kernel<T>, dim3(c->dg_nchunks, c->d.S), dim3(dg_threads<T>(g.n, g.R)),
                     dg_smem<T>(g.n, g.R), st, args);
  if (e == cudaSuccess) e = plain_launch(data_reduce_kernel<T>, dim3(c->d.S * c->d.n), dim3(128), 0, st, args);
  if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("data term: ") + cudaGetErrorString(e));
  return PDF_OK;
}

template <typename T>
static int vl_forward(pdf_ctx* c, const void* alpha_hat, cudaStream_t st) {
  VLArgs<T> a = vl_common<T>(c);
  a.alpha = (const C<T>*)alpha_hat; a.J = (C<T>*)c->J;
  a.einc = (const C<T>*)c->d.e_inc; a.einc_scene_stride = c->d.e_inc_scene_stride;
  a.E = (C<T>*)c->E_; a.norms = c->norms;
  TRY((vl_conv<T, VIEW_FWD>(c, a, c->d.S * c->d.n, st)));
  return c->skip_data ? PDF_OK : data_term<T>(c, alpha_hat, st);
}

template <typename T>
static int vl_backward(pdf_ctx* c, void* galpha, void* gy, cudaStream_t st, const FinalizeArgs& fin, bool do_fin) {
  VLArgs<T> a = vl_common<T>(c);
  a.gE = (const C<T>*)c->gE; a.gJloc = (const C<T>*)c->gJ; a.gpart = (C<T>*)c->gpart;
  TRY((vl_conv<T, VIEW_BWD>(c, a, c->d.S * c->d.n, st)));
  a.galpha = (C<T>*)galpha; a.gy = (T*)gy; a.cout = (const T*)c->cout; a.joint = c->d.joint;
  a.grows = (const C<T>*)c->grows; a.hs = (const C<T>*)c->hs;
  a.gad = c->gad_ready ? (const C<T>*)c->gad : nullptr;
  a.fin = fin; a.do_fin = do_fin ? 1 : 0;
  void* args[] = {&a};
  cudaError_t e = plain_launch(vl_trunc_reduce_kernel<T>, dim3((c->M0 + 255) / 256, c->d.S * c->d.n), dim3(256), 0,
                               st, args);
  if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("truncate reduce: ") + cudaGetErrorString(e));
  return PDF_OK;
}

template <typename T>
static int phys_forward(pdf_ctx* c, const void* alpha_hat, cudaStream_t st) {
  if (c->large) return vl_forward<T>(c, alpha_hat, st);
  ViewArgs<T> a = view_common<T>(c);
  a.alpha = (const C<T>*)alpha_hat;
  a.einc = (const C<T>*)c->d.e_inc; a.einc_scene_stride = c->d.e_inc_scene_stride;
  a.data = (const C<T>*)c->d.data; a.mask = (const T*)c->d.mask;
  a.c_sca = c->c_sca; a.J = (C<T>*)c->J; a.E = (C<T>*)c->E_; a.norms = c->norms;
  a.grows = (C<T>*)c->grows; a.dloss = c->dloss; a.do_data = !c->dgemm && !c->skip_data;
  TRY((launch_view<T, VIEW_FWD>(c, a, c->d.S * c->d.n, st)));
  return c->dgemm && !c->skip_data ? data_term<T>(c, alpha_hat, st) : PDF_OK;
}

template <typename T, bool GRAD>
static int phys_pixel(pdf_ctx* c, void* chi_out, cudaStream_t st) {
  PixelArgs<T> p = {};
  p.tl = g_tl_cur;
  p.M = c->M; p.n = c->d.n; p.R = c->d.R; p.CS = c->NPV; p.S = c->d.S;
  p.beta = (T)c->d.beta; p.l1 = (T)c->d.lambda1; p.l2 = (T)c->d.lambda2; p.l3 = (T)c->d.lambda3;
  p.tau = (T)c->d.tau_b;
  p.J = (const C<T>*)c->J; p.E = (const C<T>*)c->E_; p.norms = c->norms;
  p.rfixed = c->d.freeze_r ? (const C<T>*)c->d.r_fixed : nullptr;
  p.c_inc = c->c_inc; p.gJ = (C<T>*)c->gJ; p.gE = (C<T>*)c->gE; p.part = c->part;
  p.chi_out = (C<T>*)chi_out; p.err = c->err;
  const size_t smem = 0;
  constexpr int epc = 16 / sizeof(C<T>) > 0 ? 16 / sizeof(C<T>) : 1;
  if ((c->d.n * c->d.R) % epc) return fail(PDF_EINVAL, "n * R must be even in complex64 mode");
  void* args[] = {&p};
  // latency regime (one row per CTA still leaves SMs idle): TY = 1, 8 warps;
  // batches of <= 16 views: TY = 2 rows per CTA share the halo rows, 8 warps
  // (cfg4 638 -> 591 us); many views (cfg5's 72): TY = 1, 4-warp CTAs
  // (measured TY / warps: cfg4 1/4 629, 1/8 986, 2/4 681, 2/8 591 us; cfg5
  // 1/4 142, 1/8 151, 2/4 150, 2/8 160 us; cfg2 8.2-8.9 us for all)
  const long long rows1 = (long long)(c->M / c->TX) * c->M * c->d.S;
  const bool batch = rows1 > 4 * 148;
  // throughput regime: three streaming kernels (pdf_pixel_stream.cuh; cfg4 579 -> 326 us, cfg5 142 -> 86 us)
  static const int stream_env = env_int("PDF_PIX_STREAM", 1);
  if (batch && stream_env) {
    PixStreamArgs<T> q = {};
    q.p = p;
    const size_t img = (size_t)c->M * c->M;
    q.sums = c->pix;
    q.coef = c->pix + (size_t)c->d.S * img * 4;
    void* qargs[] = {&q};
    // (chunks of scenes sized for the L2, so that the gradient pass re-reads J, E
    // from it, measured slower: 372 us in one launch, 398 / 431 / 620 us in
    // chunks of 80 / 40 / 20 MiB -- the per-chunk launches' ramps and tails)
    cudaError_t e = plain_launch(pix_sums_kernel<T>, dim3((unsigned)(img / 32), c->d.S), dim3(256), 0, st, qargs);
    // gradient pass fused into the per-pixel kernel for <= 32 views (cfg4); many
    // views (cfg5's 72) keep the separate pass, split over groups of views
    static const int fuse_env = env_int("PDF_PIX_FUSE", 1);
    const bool fuse = GRAD && fuse_env && c->d.n <= 32;
    q.p.tl = fuse ? p.tl : 0;
    if (e == cudaSuccess) {
      const dim3 pg(c->M / c->TX, c->M / 4, c->d.S);
      e = fuse ? plain_launch(pix_point_kernel<T, GRAD, 4, true>, pg, dim3(128), 0, st, qargs)
               : plain_launch(pix_point_kernel<T, GRAD, 4, false>, pg, dim3(128), 0, st, qargs);
    }
    if (GRAD && !fuse && e == cudaSuccess) {
      q.p.tl = p.tl;
      e = plain_launch(pix_grad_kernel<T>, dim3((unsigned)((img + 255) / 256), (c->d.n + PG_VIEWS - 1) / PG_VIEWS, c->d.S),
                       dim3(256), 0, st, qargs);
    }
    if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("pixel kernels (stream): ") + cudaGetErrorString(e));
    return PDF_OK;
  }
  static const int ty_env = env_int("PDF_PIX_TY", 0);
  const int ty = ty_env == 1 || ty_env == 2 ? ty_env : (batch && c->d.n <= 16 ? 2 : 1);
  static const int pw_env = env_int("PDF_PIX_WARPS", 0);
  const int pw = std::min(std::max(pw_env ? pw_env : (batch && ty == 1 ? 4 : PIX_NW), 1), PIX_NW);
  const int vpw = (c->d.n + pw - 1) / pw;       // views per warp; the first VC stay in registers
  const dim3 grid(c->M / c->TX, c->M / ty, c->d.S), blk(32 * pw);
  cudaError_t e;
  if (ty == 1) e = vpw <= 2 ? plain_launch(pixel_kernel<T, GRAD, 1, 2>, grid, blk, smem, st, args)
                            : plain_launch(pixel_kernel<T, GRAD, 1, 4>, grid, blk, smem, st, args);
  else e = vpw <= 2 ? plain_launch(pixel_kernel<T, GRAD, 2, 2>, grid, blk, smem, st, args)
                    : plain_launch(pixel_kernel<T, GRAD, 2, 4>, grid, blk, smem, st, args);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("pixel kernel: ") + cudaGetErrorString(e));
  return PDF_OK;
}

static FinalizeArgs fin_args(pdf_ctx* c, double* bd, double* trace) {
  FinalizeArgs f = {};
  f.n = c->d.n; f.ntiles = c->ntiles; f.S = c->d.S;
  f.l1 = c->d.lambda1; f.l2 = c->d.lambda2; f.l3 = c->d.lambda3;
  f.c_inc = c->c_inc; f.c_sca = c->c_sca; f.dloss = c->dloss; f.part = c->part;
  f.bd = bd ? bd : c->bd; f.trace = trace; f.step = c->step; f.err = c->err;
  return f;
}

template <typename T>
static int phys_backward(pdf_ctx* c, void* galpha, void* gy, cudaStream_t st, double* bd = nullptr,
                         double* trace = nullptr, bool fin = false) {
  if (c->large) return vl_backward<T>(c, galpha, gy, st, fin_args(c, bd, trace), fin);
  ViewArgs<T> a = view_common<T>(c);
  a.fin = fin_args(c, bd, trace);
  a.do_fin = fin ? 1 : 0;
  a.gE = (const C<T>*)c->gE; a.gJloc = (const C<T>*)c->gJ;
  a.galpha = (C<T>*)galpha; a.gy = (T*)gy; a.cout = (const T*)c->cout; a.joint = c->d.joint;
  a.grows = (C<T>*)c->grows;
  a.gad = c->gad_ready ? (const C<T>*)c->gad : nullptr;
  return launch_view<T, VIEW_BWD>(c, a, c->d.S * c->d.n, st);
}

static int finalize(pdf_ctx* c, double* bd, double* trace, cudaStream_t st) {
  FinalizeArgs f = fin_args(c, bd, trace);
  finalize_kernel<<<c->d.S, 128, 0, st>>>(f);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("finalize: ") + cudaGetErrorString(e));
  return PDF_OK;
}

// cluster split for the network layers: enough CTAs for ~4 per SM (hot-L2
// streaming needs bytes in flight), 1 when the batch alone fills the GPU
static int net_split(long long base_ctas, int max_split) {
  static const int cap = env_int("PDF_NET_CLUSTER", 2);
  int c = 1;
  while (c < cap && c < max_split && base_ctas * c < 4LL * 148) c *= 2;
  return c;
}

// DMMA forward layer (float64): MT m-tiles of 8 rows, NT n-tiles of 8 per warp
template <int MT, int NT>
static cudaError_t fwd_mma_launch(dim3 grid, int CK, NetFwdArgs<double>& a, cudaStream_t st) {
  const size_t smem = fwd_mma_smem_bytes(MT, NT);
  auto k = net_fwd_mma_kernel<MT, NT>;
  cudaError_t e = prep(k, smem);
  if (e != cudaSuccess) return e;
  void* args[] = {&a};
  return launch_cluster(k, grid, dim3(256), smem, st, dim3(1, CK, 1), args);
}

template <int MT>
static cudaError_t fwd_mma_nt(int NT, dim3 grid, int CK, NetFwdArgs<double>& a, cudaStream_t st) {
  if constexpr (MT <= 4) { if (NT == 4) return fwd_mma_launch<MT, 4>(grid, CK, a, st); }
  if constexpr (MT <= 8) { if (NT == 2) return fwd_mma_launch<MT, 2>(grid, CK, a, st); }
  return fwd_mma_launch<MT, 1>(grid, CK, a, st);
}

static int fwd_mma_layer(pdf_ctx* c, NetFwdArgs<double>& a, cudaStream_t st) {
  const int MT = (c->rows + 7) / 8, S = c->d.S, N = a.N, K = a.K;
  // latency regime (few scenes, <= 16 rows, K <= 1024): one n-tile per CTA,
  // the input block resident in shared memory, one memory round trip
  static const int xk = env_int("PDF_FWD_X", 1);
  if (xk && MT <= 2 && K <= XW * XKB * 16 && (long long)S * ((N + 7) / 8) <= 4 * 148) {
    const dim3 grid((N + 7) / 8, 1, S);
    const size_t smem = fwd_x_smem_bytes(MT, K);
    void* args[] = {&a};
    // x multicast over clusters of 4 CTAs (PDF_FWD_MC=1 stages it per CTA)
    static const int mc = env_int("PDF_FWD_MC", 4);
    cudaError_t e;
    if (mc == 8 && grid.x % 8 == 0) {
      e = MT == 1 ? prep(net_fwd_x_kernel<1, 8>, smem) : prep(net_fwd_x_kernel<2, 8>, smem);
      if (e == cudaSuccess)
        e = MT == 1 ? launch_cluster(net_fwd_x_kernel<1, 8>, grid, dim3(XW * 32), smem, st, dim3(8, 1, 1), args)
                    : launch_cluster(net_fwd_x_kernel<2, 8>, grid, dim3(XW * 32), smem, st, dim3(8, 1, 1), args);
    } else if (mc == 2 && grid.x % 2 == 0) {
      e = MT == 1 ? prep(net_fwd_x_kernel<1, 2>, smem) : prep(net_fwd_x_kernel<2, 2>, smem);
      if (e == cudaSuccess)
        e = MT == 1 ? launch_cluster(net_fwd_x_kernel<1, 2>, grid, dim3(XW * 32), smem, st, dim3(2, 1, 1), args)
                    : launch_cluster(net_fwd_x_kernel<2, 2>, grid, dim3(XW * 32), smem, st, dim3(2, 1, 1), args);
    } else if (mc >= 4 && grid.x % 4 == 0) {
      e = MT == 1 ? prep(net_fwd_x_kernel<1, 4>, smem) : prep(net_fwd_x_kernel<2, 4>, smem);
      if (e == cudaSuccess)
        e = MT == 1 ? launch_cluster(net_fwd_x_kernel<1, 4>, grid, dim3(XW * 32), smem, st, dim3(4, 1, 1), args)
                    : launch_cluster(net_fwd_x_kernel<2, 4>, grid, dim3(XW * 32), smem, st, dim3(4, 1, 1), args);
    } else {
      e = MT == 1 ? plain_launch(net_fwd_x_kernel<1, 1>, grid, dim3(XW * 32), smem, st, args)
                  : plain_launch(net_fwd_x_kernel<2, 1>, grid, dim3(XW * 32), smem, st, args);
    }
    if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("net fwd (x): ") + cudaGetErrorString(e));
    return PDF_OK;
  }
  auto ctas = [&](int nt) { return (long long)((N + 64 * nt - 1) / (64 * nt)) * S; };
  // one n-tile per warp measured fastest in every regime (more CTAs and more
  // W bytes in flight per SM); PDF_FWD_NT=2/4 for experiments
  int NT = 1;
  static const int nt_env = env_int("PDF_FWD_NT", 1);
  if ((nt_env == 2 && MT <= 8) || (nt_env == 4 && MT <= 4)) NT = nt_env;
  static const int cap = env_int("PDF_FWD_CLUSTER", 8);
  const long long base = ctas(NT);
  const int kmax = (K + FM_KCH - 1) / FM_KCH;
  int CK = 1;
  while (CK < cap && 2 * CK <= kmax && base * CK < 2 * 148) CK *= 2;
  // a grid that spills into a second, partly filled wave of 2 CTAs per SM is
  // slower than half the split in one wave (cfg5, N = 4096: 512 CTAs 114 us, 256 CTAs 107 us)
  if (CK > 1 && base * CK > 2 * 148 && base * CK / 2 >= (2 * 148 * 4) / 5) CK /= 2;
  a.ks = ((K + CK - 1) / CK + FM_KCH - 1) / FM_KCH * FM_KCH;
  const dim3 grid((N + 64 * NT - 1) / (64 * NT), CK, S);
  cudaError_t e;
  switch (MT) {
    case 1: e = fwd_mma_nt<1>(NT, grid, CK, a, st); break;
    case 2: e = fwd_mma_nt<2>(NT, grid, CK, a, st); break;
    case 3: e = fwd_mma_nt<3>(NT, grid, CK, a, st); break;
    case 4: e = fwd_mma_nt<4>(NT, grid, CK, a, st); break;
    case 5: e = fwd_mma_nt<5>(NT, grid, CK, a, st); break;
    case 6: e = fwd_mma_nt<6>(NT, grid, CK, a, st); break;
    case 7: e = fwd_mma_nt<7>(NT, grid, CK, a, st); break;
    case 8: e = fwd_mma_nt<8>(NT, grid, CK, a, st); break;
    case 9: e = fwd_mma_nt<9>(NT, grid, CK, a, st); break;
    case 10: e = fwd_mma_nt<10>(NT, grid, CK, a, st); break;
    default: return fail(PDF_EINVAL, "rows");
  }
  if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("net fwd (dmma): ") + cudaGetErrorString(e));
  return PDF_OK;
}

template <typename T>
static int net_fwd_layer(pdf_ctx* c, const T* in, int K, int N, const T* theta, long long woff, long long boff,
                         T* out, int final_layer, int* step, cudaStream_t st) {
  NetFwdArgs<T> a = {};
  a.tl = g_tl_cur;
  a.rows = c->rows; a.K = K; a.N = N;
  a.in = in; a.in_ss = (long long)c->rows * K;
  a.theta = theta; a.th_ss = c->Np; a.w_off = woff; a.b_off = boff;
  a.out = out; a.out_ss = (long long)c->rows * N; a.final_layer = final_layer;
  a.cout = (const T*)c->cout; a.alpha0 = (const C<T>*)c->alpha0; a.alpha_hat = (C<T>*)c->alpha_hat;
  a.n = c->d.n; a.M0 = c->M0; a.joint = c->d.joint; a.step = step;
  a.w_early = woff != 0;   // W2, W3 were last written >= 2 launches earlier; W1 by the launch right before
  if (K % Epc<T>::v || N % Epc<T>::v) return fail(PDF_EINVAL, "layer widths must be multiples of 16 bytes");
  static const int use_mma = env_int("PDF_NET_MMA", 1);
  if constexpr (sizeof(T) == 8) {
    if (use_mma) return fwd_mma_layer(c, a, st);
  }
  // one output row per warp while a single scene cannot fill the GPU, two otherwise
  const int opw = (c->RB == 1 && (c->d.S * N) / (NET_THREADS / 32) >= 2 * 148 * 4) ? 2 : 1;
  const int kch = c->RB <= 2 ? FwdShape<T, 1>::KCH : FwdShape<T, 3>::KCH;
  const int per = (NET_THREADS / 32) * opw;
  const long long base = (long long)((N + per - 1) / per) * c->d.S;
  const int CK = net_split(base, (K + kch - 1) / kch);
  a.ks = ((K + CK - 1) / CK + kch - 1) / kch * kch;
  void* args[] = {&a};
  cudaError_t e;
  const dim3 grid((N + per - 1) / per, CK, c->d.S), block(NET_THREADS), cl(1, CK, 1);
  switch (c->RB * 4 + opw) {
#define FCASE(RR, OO)                                                                      \
  case RR * 4 + OO: {                                                                      \
    const size_t smem = fwd_smem_elems<T, RR>(OO) * sizeof(T);                             \
    auto k = net_fwd_kernel<T, RR, OO>;                                                    \
    e = prep(k, smem);                                                                     \
    if (e == cudaSuccess) e = launch_cluster(k, grid, block, smem, st, cl, args);          \
    break;                                                                                 \
  }
    FCASE(1, 1) FCASE(1, 2) FCASE(2, 1) FCASE(3, 1) FCASE(4, 1) FCASE(5, 1)
#undef FCASE
    default: return fail(PDF_EINVAL, "rows");
  }
  if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("net fwd: ") + cudaGetErrorString(e));
  return PDF_OK;
}

// DMMA backward layer (float64)
template <int MT, int KT, int WB, int D>
static cudaError_t bwd_mma_launch(bool fused, dim3 grid, int CN, NetBwdArgs<double>& a, cudaStream_t st) {
  const size_t smem = bwd_mma_smem_bytes(MT, KT, WB, D);
  void* args[] = {&a};
  cudaError_t e;
  if (fused) {
    auto k = net_bwd_mma_kernel<MT, KT, true, WB, D>;
    e = prep(k, smem);
    if (e == cudaSuccess) e = launch_cluster(k, grid, dim3(WB * 32), smem, st, dim3(1, a.gzprev ? CN : 1, 1), args);
  } else {
    auto k = net_bwd_mma_kernel<MT, KT, false, WB, D>;
    e = prep(k, smem);
    if (e == cudaSuccess) e = launch_cluster(k, grid, dim3(WB * 32), smem, st, dim3(1, a.gzprev ? CN : 1, 1), args);
  }
  return e;
}

// D = n-tiles in flight per lane: 6 with one k-tile per warp (more bytes in
// flight where few warps stream), 3 with two (batches: two CTAs per SM)
template <int MT>
static cudaError_t bwd_mma_kt(int KT, int WB, int D, bool fused, dim3 grid, int CN, NetBwdArgs<double>& a,
                              cudaStream_t st) {
  if constexpr (MT <= 4) {
    if (KT == 2) return WB == 8 ? bwd_mma_launch<MT, 2, 8, 3>(fused, grid, CN, a, st)
                                : bwd_mma_launch<MT, 2, 4, 3>(fused, grid, CN, a, st);
  }
  if (D == 6)
    return WB == 8 ? bwd_mma_launch<MT, 1, 8, 6>(fused, grid, CN, a, st)
                   : bwd_mma_launch<MT, 1, 4, 6>(fused, grid, CN, a, st);
  return WB == 8 ? bwd_mma_launch<MT, 1, 8, 3>(fused, grid, CN, a, st)
                 : bwd_mma_launch<MT, 1, 4, 3>(fused, grid, CN, a, st);
}

static int bwd_mma_layer(pdf_ctx* c, NetBwdArgs<double>& a, bool fused, cudaStream_t st) {
  const int MT = (c->rows + 7) / 8, S = c->d.S, N = a.N, K = a.K;
  // two k-tiles per warp (128-byte W row segments) when the batch fills the GPU
  static const int kt_env = env_int("PDF_BWD_KT", 0);
  int KT = 1;
  // (two k-tiles per warp measured 1.2 % slower at 128 scenes: one everywhere; PDF_BWD_KT=2 for experiments)
  if (kt_env == 1 || (kt_env == 2 && MT <= 4)) KT = kt_env;
  static const int wb_env = env_int("PDF_BWD_WB", 0), d_env = env_int("PDF_BWD_D", 3);
  // 8 warps per CTA in every regime (measured: cfg2 96.8 -> 93.7 us/iter,
  // cfg5 backward 795 -> 671 us against 4-warp CTAs for one scene)
  const int WB = wb_env ? wb_env : BM_WARPS;
  const int D = KT == 1 ? d_env : 3;
  const int CW = WB * 8 * KT;
  // N split: a cluster of CN CTAs when g_h is reduced across it (DSMEM),
  // plain CTAs for the first layer; CTA-count targets per SM in env for
  // experiments
  static const int cap = env_int("PDF_BWD_CLUSTER", 16);
  static const int tgt = env_int("PDF_BWD_TGT", 3), tgt1 = env_int("PDF_BWD_TGT1", 3);
  const long long base = (long long)((K + CW - 1) / CW) * S;
  const int nmax = (N + BM_NCH - 1) / BM_NCH;
  const int cap_n = a.gzprev ? cap : 64;
  const long long target = (long long)(a.gzprev ? tgt : tgt1) * 148;
  int CN = 1;
  while (CN < cap_n && 2 * CN <= nmax && base * CN < target) CN *= 2;
  a.ns = ((N + CN - 1) / CN + BM_NCH - 1) / BM_NCH * BM_NCH;
  const dim3 grid((K + CW - 1) / CW, CN, S);
  cudaError_t e;
  switch (MT) {
    case 1: e = bwd_mma_kt<1>(KT, WB, D, fused, grid, CN, a, st); break;
    case 2: e = bwd_mma_kt<2>(KT, WB, D, fused, grid, CN, a, st); break;
    case 3: e = bwd_mma_kt<3>(KT, WB, D, fused, grid, CN, a, st); break;
    case 4: e = bwd_mma_kt<4>(KT, WB, D, fused, grid, CN, a, st); break;
    case 5: e = bwd_mma_kt<5>(KT, WB, D, fused, grid, CN, a, st); break;
    case 6: e = bwd_mma_kt<6>(KT, WB, D, fused, grid, CN, a, st); break;
    case 7: e = bwd_mma_kt<7>(KT, WB, D, fused, grid, CN, a, st); break;
    case 8: e = bwd_mma_kt<8>(KT, WB, D, fused, grid, CN, a, st); break;
    case 9: e = bwd_mma_kt<9>(KT, WB, D, fused, grid, CN, a, st); break;
    case 10: e = bwd_mma_kt<10>(KT, WB, D, fused, grid, CN, a, st); break;
    default: return fail(PDF_EINVAL, "rows");
  }
  if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("net bwd (dmma): ") + cudaGetErrorString(e));
  return PDF_OK;
}

template <typename T>
static int net_bwd_layer(pdf_ctx* c, const T* gz, const T* hin, int K, int N, T* theta, long long woff,
                         long long boff, T* m, T* v, T* grad, int fused, T* gzprev, cudaStream_t st) {
  NetBwdArgs<T> a = {};
  a.tl = g_tl_cur;
  a.rows = c->rows; a.K = K; a.N = N;
  a.gz = gz; a.gz_ss = (long long)c->rows * N;
  a.hin = hin; a.hin_ss = (long long)c->rows * K;
  a.theta = theta; a.th_ss = c->Np; a.w_off = woff; a.b_off = boff;
  a.m = m; a.v = v; a.grad = grad; a.step = c->step;
  a.lr = (T)c->d.lr; a.b1 = (T)c->d.adam_b1; a.b2 = (T)c->d.adam_b2; a.eps = (T)c->d.adam_eps;
  a.gzprev = gzprev; a.gzp_ss = (long long)c->rows * K; a.err = c->err;
  a.peers = fused ? nullptr : c->sc_peers; a.peer_me = c->sc_me; a.peer_shard = c->sc_shard;
  if (K % Epc<T>::v || N % Epc<T>::v) return fail(PDF_EINVAL, "layer widths must be multiples of 16 bytes");
  if (a.peers && (sizeof(T) != 8 || !env_int("PDF_NET_MMA", 1)))
    return fail(PDF_EINVAL, "the peer-scattered backward needs the float64 DMMA kernels");
  static const int use_mma = env_int("PDF_NET_MMA", 1);
  if constexpr (sizeof(T) == 8) {
    if (use_mma) return bwd_mma_layer(c, a, fused != 0, st);
  }
  const int cols = c->RB >= 4 ? BwdShape<T, 4>::COLS : BwdShape<T, 1>::COLS;
  const int nch = c->RB >= 4 ? BwdShape<T, 4>::NCH : BwdShape<T, 1>::NCH;
  const int thr = c->RB >= 4 ? BwdShape<T, 4>::THR : BwdShape<T, 1>::THR;
  const long long base = (long long)((K + cols - 1) / cols) * c->d.S;
  const int CN = net_split(base, (N + nch - 1) / nch);
  a.ns = ((N + CN - 1) / CN + BWD_NCH_MAX - 1) / BWD_NCH_MAX * BWD_NCH_MAX;
  void* args[] = {&a};
  cudaError_t e;
  const dim3 grid((K + cols - 1) / cols, CN, c->d.S), block(thr), cl(1, CN, 1);
  switch (c->RB * 2 + (fused ? 1 : 0)) {
#define BCASE(RR, FF)                                                                      \
  case RR * 2 + FF: {                                                                      \
    const size_t smem = bwd_smem_elems<T, RR>() * sizeof(T);                               \
    auto k = net_bwd_kernel<T, RR, (FF != 0)>;                                             \
    e = prep(k, smem);                                                                     \
    if (e == cudaSuccess) e = launch_cluster(k, grid, block, smem, st, cl, args);          \
    break;                                                                                 \
  }
    BCASE(1, 0) BCASE(1, 1) BCASE(2, 0) BCASE(2, 1) BCASE(3, 0) BCASE(3, 1) BCASE(4, 0) BCASE(4, 1)
    BCASE(5, 0) BCASE(5, 1)
#undef BCASE
    default: return fail(PDF_EINVAL, "rows");
  }
  if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("net bwd: ") + cudaGetErrorString(e));
  return PDF_OK;
}

struct Offs { long long w1, b1, w2, b2, w3, b3; };
static Offs offsets(const pdf_ctx* c) {
  Offs o;
  const long long H = c->H, D0 = c->D0;
  o.w1 = 0; o.b1 = H * D0; o.w2 = o.b1 + H; o.b2 = o.w2 + H * H; o.w3 = o.b2 + H; o.b3 = o.w3 + D0 * H;
  return o;
}


template <typename T>
static int net_forward_all(pdf_ctx* c, const void* theta, int* step, cudaStream_t st) {
  const Offs o = offsets(c);
  const T* th = (const T*)theta;
  TRY(net_fwd_layer<T>(c, (const T*)c->x0, c->D0, c->H, th, o.w1, o.b1, (T*)c->h1, 0, step, st));
  TRY(net_fwd_layer<T>(c, (const T*)c->h1, c->H, c->H, th, o.w2, o.b2, (T*)c->h2, 0, nullptr, st));
  TRY(net_fwd_layer<T>(c, (const T*)c->h2, c->H, c->D0, th, o.w3, o.b3, nullptr, 1, nullptr, st));
  return PDF_OK;
}

template <typename T>
static ShardArgs<T> shard_args(pdf_ctx* c, double* red1, double* red2);

// the pixel stage split in three (numden / pixel_a / pixel_b) with local
// reduction buffers: one thread per pixel for the view sums, no halo
// recomputation of num/den
template <typename T>
static int split_pixel(pdf_ctx* c, cudaStream_t st) {
  ShardArgs<T> a = shard_args<T>(c, c->red1, c->red2);
  const int img = c->M * c->M;
  void* args[] = {&a};
  CK_CUDA(plain_launch(shard_numden_kernel<T>, dim3((img + 255) / 256, c->d.S), dim3(256), 0, st, args));
  const dim3 grid(c->M / c->TX, c->M, c->d.S);
  CK_CUDA(plain_launch(shard_pixel_a_kernel<T>, grid, dim3(PIX_NW * 32), 0, st, args));
  shard_loss_sums_kernel<<<c->d.S, 128, 0, st>>>(c->part, c->dloss, c->red2, c->ntiles, c->d.n, (size_t)img);
  CK_CUDA(cudaGetLastError());
  CK_CUDA(plain_launch(shard_pixel_b_kernel<T>, grid, dim3(PIX_NW * 32), 0, st, args));
  return PDF_OK;
}

static int split_finalize(pdf_ctx* c, double* bd, double* trace, cudaStream_t st) {
  FinalizeArgs f = fin_args(c, bd, trace);
  shard_finalize_kernel<<<c->d.S, 128, 0, st>>>(f, c->red2, (size_t)c->M * c->M);
  CK_CUDA(cudaGetLastError());
  return PDF_OK;
}

// split network backward (latency regime, float64): g_h of layers 3 and 2,
// then g_W + Adam of all layers in one launch
template <int MT>
static cudaError_t gh_t_launch(dim3 grid, int ktw, GhArgs& a, cudaStream_t st) {
  void* args[] = {&a};
  if (ktw == 4) return plain_launch(net_gh_t_kernel<MT, 4>, grid, dim3(XW * 32), gh_t_smem_bytes(MT, 4), st, args);
  if (ktw == 2) return plain_launch(net_gh_t_kernel<MT, 2>, grid, dim3(XW * 32), gh_t_smem_bytes(MT, 2), st, args);
  return plain_launch(net_gh_t_kernel<MT, 1>, grid, dim3(XW * 32), gh_t_smem_bytes(MT, 1), st, args);
}

static int gh_x_layer(pdf_ctx* c, const double* gz, const double* hin, int K, int N, const double* theta,
                      long long woff, double* gzprev, int* snap, cudaStream_t st) {
  const int MT = (c->rows + 7) / 8;
  if (MT > 2 || N > XW * 4 * GX_STEPS) {
    // tiled: all rows x 64 outputs per CTA, n split into slices (~2 CTAs per SM)
    GhArgs g = {};
    g.tl = g_tl_cur;
    g.rows = c->rows; g.K = K; g.N = N;
    // 4 k-tiles per warp when the k-blocks x slices still cover the SMs
    // (config 5: 4096 columns), else 1 (config 3)
    static const int ktw_env = env_int("PDF_GH_KTW", 0);
    // (2 / 4 k-tiles per warp reuse the A fragments from registers but were
    // measured slower on configs 3 and 5: occupancy; PDF_GH_KTW for experiments)
    const int ktw = ktw_env ? ktw_env : 1;
    const int kbs = (K + gt_kb(ktw) - 1) / gt_kb(ktw);
    int nsl = 1;
    while (nsl < GH_NSL && (long long)kbs * nsl * c->d.S < 2 * 148 && N / (2 * nsl) >= 2 * GT_NC) nsl *= 2;
    if (nsl > 1 && (long long)kbs * nsl * c->d.S > 2 * 148 &&
        (long long)kbs * nsl * c->d.S / 2 >= (2 * 148 * 4) / 5)
      nsl /= 2;   // one full wave instead of a second, partly filled one (cfg5: g_h2 160 -> 142 us)
    g.nsl = nsl;
    g.ns = ((N + nsl - 1) / nsl + GT_NC - 1) / GT_NC * GT_NC;
    g.gz = gz; g.gz_ss = (long long)c->rows * N;
    g.hin = hin; g.hin_ss = (long long)c->rows * K;
    g.theta = theta; g.th_ss = c->Np; g.w_off = woff;
    g.gzprev = gzprev; g.gzp_ss = (long long)c->rows * K;
    g.part = c->ghp; g.ticket = c->ticket;   // (the side-branch fork, which needs the t snapshot, uses gh_x only)
    const dim3 grid(kbs, nsl, c->d.S);
    cudaError_t e;
    switch (MT) {
      case 1: e = gh_t_launch<1>(grid, ktw, g, st); break;
      case 2: e = gh_t_launch<2>(grid, ktw, g, st); break;
      case 3: e = gh_t_launch<3>(grid, ktw, g, st); break;
      case 4: e = gh_t_launch<4>(grid, ktw, g, st); break;
      case 5: e = gh_t_launch<5>(grid, ktw, g, st); break;
      case 6: e = gh_t_launch<6>(grid, ktw, g, st); break;
      case 7: e = gh_t_launch<7>(grid, ktw, g, st); break;
      case 8: e = gh_t_launch<8>(grid, ktw, g, st); break;
      case 9: e = gh_t_launch<9>(grid, ktw, g, st); break;
      default: e = gh_t_launch<10>(grid, ktw, g, st); break;
    }
    if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("net g_h (tiled): ") + cudaGetErrorString(e));
    return PDF_OK;
  }
  NetBwdArgs<double> a = {};
  a.tl = g_tl_cur;
  a.rows = c->rows; a.K = K; a.N = N;
  a.gz = gz; a.gz_ss = (long long)c->rows * N;
  a.hin = hin; a.hin_ss = (long long)c->rows * K;
  a.theta = const_cast<double*>(theta); a.th_ss = c->Np; a.w_off = woff;
  a.gzprev = gzprev; a.gzp_ss = (long long)c->rows * K; a.err = c->err;
  a.step = c->step; a.snap = snap;
  const dim3 grid((K + 7) / 8, 1, c->d.S);
  const size_t smem = gh_x_smem_bytes(MT, N);
  void* args[] = {&a};
  static const int mc = env_int("PDF_FWD_MC", 4);   // g_z multicast over clusters of 4 (as the forward)
  cudaError_t e;
  if (mc == 8 && grid.x % 8 == 0) {
    e = MT == 1 ? prep(net_gh_x_kernel<1, 8>, smem) : prep(net_gh_x_kernel<2, 8>, smem);
    if (e == cudaSuccess)
      e = MT == 1 ? launch_cluster(net_gh_x_kernel<1, 8>, grid, dim3(XW * 32), smem, st, dim3(8, 1, 1), args)
                  : launch_cluster(net_gh_x_kernel<2, 8>, grid, dim3(XW * 32), smem, st, dim3(8, 1, 1), args);
  } else if (mc == 2 && grid.x % 2 == 0) {
    e = MT == 1 ? prep(net_gh_x_kernel<1, 2>, smem) : prep(net_gh_x_kernel<2, 2>, smem);
    if (e == cudaSuccess)
      e = MT == 1 ? launch_cluster(net_gh_x_kernel<1, 2>, grid, dim3(XW * 32), smem, st, dim3(2, 1, 1), args)
                  : launch_cluster(net_gh_x_kernel<2, 2>, grid, dim3(XW * 32), smem, st, dim3(2, 1, 1), args);
  } else if (mc >= 4 && grid.x % 4 == 0) {
    e = MT == 1 ? prep(net_gh_x_kernel<1, 4>, smem) : prep(net_gh_x_kernel<2, 4>, smem);
    if (e == cudaSuccess)
      e = MT == 1 ? launch_cluster(net_gh_x_kernel<1, 4>, grid, dim3(XW * 32), smem, st, dim3(4, 1, 1), args)
                  : launch_cluster(net_gh_x_kernel<2, 4>, grid, dim3(XW * 32), smem, st, dim3(4, 1, 1), args);
  } else {
    e = MT == 1 ? plain_launch(net_gh_x_kernel<1, 1>, grid, dim3(XW * 32), smem, st, args)
                : plain_launch(net_gh_x_kernel<2, 1>, grid, dim3(XW * 32), smem, st, args);
  }
  if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("net g_h (x): ") + cudaGetErrorString(e));
  return PDF_OK;
}

// layers: bit l of `mask` selects network layer l + 1; tsnap: Adam t snapshot or null (*step)
static int adam_x_all(pdf_ctx* c, double* theta, double* m, double* v, cudaStream_t st, int mask = 7,
                      const int* tsnap = nullptr) {
  const long long H = c->H, D0 = c->D0, R = c->rows;
  const Offs o = offsets(c);
  // launch order: layer 3 (g_z = g_y, three launches old), layer 2 (g_z2 from
  // the g_h launch two back), layer 1 (g_z1 from the launch right before: waits)
  const double* gzs[3] = {(const double*)c->gy, (const double*)c->gz2, (const double*)c->gz1};
  const double* hins[3] = {(const double*)c->h2, (const double*)c->h1, (const double*)c->x0};
  const long long Ns[3] = {D0, H, H}, Ks[3] = {H, H, D0};
  const long long wo[3] = {o.w3, o.w2, o.w1}, bo[3] = {o.b3, o.b2, o.b1};
  NetAdamArgs a = {};
  a.tl = g_tl_cur;
  long long items = 0;
  for (int l = 0; l < 3; ++l) {
    AdamLayer& L = a.L[l];
    L.gz = gzs[l]; L.hin = hins[l]; L.gz_ss = R * Ns[l]; L.hin_ss = R * Ks[l];
    L.w_off = wo[l]; L.b_off = bo[l]; L.N = (int)Ns[l]; L.K = (int)Ks[l];
    L.nblk = (int)((Ns[l] + AX_NB - 1) / AX_NB);
    L.strips = (int)((Ks[l] + AX_ST * 8 - 1) / (AX_ST * 8));
    const int layer = 3 - l;   // entries in launch order 3, 2, 1
    L.items = (mask >> (layer - 1) & 1) ? L.nblk * L.strips + (int)((Ns[l] + 255) / 256) : 0;
    L.wait = l == 2;
    items += L.items;
  }
  a.rows = c->rows; a.theta = theta; a.m = m; a.v = v; a.th_ss = c->Np; a.step = c->step; a.tsnap = tsnap;
  a.lr = c->d.lr; a.b1 = c->d.adam_b1; a.b2 = c->d.adam_b2; a.eps = c->d.adam_eps; a.err = c->err;
  const dim3 grid((unsigned)items, c->d.S);
  void* args[] = {&a};
  const int MT = (c->rows + 7) / 8;
  cudaError_t e;
  // many rows, one large scene: the persistent warp-specialised form (shared-memory ring)
  static const int ring_env = env_int("PDF_ADAM_RING", 1);
  bool aligned = true;
  for (int l = 0; l < 3; ++l)
    if (a.L[l].items && (a.L[l].N % AX_NB || a.L[l].K % (AX_ST * 8))) aligned = false;
  // (16+ items per CTA: at cfg3's 7 the pipeline's ramp loses to the one-shot kernel, 37 vs 25 us)
  if (ring_env && c->d.S == 1 && MT >= 5 && aligned && items > 16 * 148) {
    const size_t rs = adam_ring_smem_bytes(MT);
    const dim3 rgrid(148);
    switch (MT) {
#define RCASE(MM) case MM: e = plain_launch(net_adam_ring_kernel<MM>, rgrid, dim3(AR_THREADS), rs, st, args); break;
      RCASE(5) RCASE(6) RCASE(7) RCASE(8) RCASE(9)
      default: e = plain_launch(net_adam_ring_kernel<10>, rgrid, dim3(AR_THREADS), rs, st, args); break;
#undef RCASE
    }
    if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("net adam (ring): ") + cudaGetErrorString(e));
    return PDF_OK;
  }
  const size_t smem = adam_x_smem_bytes(MT);
  switch (MT) {
#define ACASE(MM) case MM: e = plain_launch(net_adam_x_kernel<MM>, grid, dim3(256), smem, st, args); break;
    ACASE(1) ACASE(2) ACASE(3) ACASE(4) ACASE(5) ACASE(6) ACASE(7) ACASE(8) ACASE(9)
    default: e = plain_launch(net_adam_x_kernel<10>, grid, dim3(256), smem, st, args); break;
#undef ACASE
  }
  if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("net adam (x): ") + cudaGetErrorString(e));
  return PDF_OK;
}

template <typename T>
static int iteration(pdf_ctx* c, void* theta, void* m, void* v, void* grad, double* bd, double* trace, int fused,
                     cudaStream_t st, cudaEvent_t* ev = nullptr) {
  // phase order (PDF_NPHASES = 10): fwd_l1 fwd_l2 fwd_l3 view_fwd pixel view_bwd finalize bwd_l3 bwd_l2 bwd_l1
  // PDF_SKIP_PHASES (bitmask) drops kernels: measurement experiments only,
  // compiled in only with -DPDF_EXPERIMENTS (never in the product library)
#ifdef PDF_EXPERIMENTS
  static const int skip = env_int("PDF_SKIP_PHASES", 0);
#else
  constexpr int skip = 0;
#endif
  int ph = 0;
  auto mark = [&]() {
    if (ev) cudaEventRecord(ev[ph], st);
    ++ph;
    const int slot = g_tl_iter * PDF_NPHASES + ph;
    g_tl_cur = c->tl_on && ph <= PDF_NPHASES && slot <= PDF_TL_SLOTS ? slot : 0;
  };
  auto run = [&]() { return !(skip >> ph & 1); };
  const Offs o = offsets(c);
  const T* thc = (const T*)theta;
  T* th = (T*)theta;
  // captured graph: the Adam of layers 3 / 2 runs on a side branch that
  // overlaps the next iteration's first layers; h1 / h2 (read by it) and the
  // Adam-t snapshot alternate between two buffers
  // (measured: cfg2 88.1 -> 84.6 us; with 36 rows the side branch slows the
  // main chain, cfg3 150 -> 194 us: rows <= 16 only)
  const bool fork = sizeof(T) == 8 && c->capturing && fused && c->xbwd && c->rows <= 16 &&
                    c->H <= XW * 4 * GX_STEPS && c->D0 <= XW * 4 * GX_STEPS;
  if (fork) { std::swap(c->h1, c->h1b); std::swap(c->h2, c->h2b); std::swap(c->tsnap, c->tsnap_b); }
  mark();
  if (run()) TRY(net_fwd_layer<T>(c, (const T*)c->x0, c->D0, c->H, thc, o.w1, o.b1, (T*)c->h1, 0,
                                  fused ? c->step : nullptr, st));
  mark();
  if (fork && c->pend) {   // W2 / W3 of the previous iteration's side branch
    CK_CUDA(cudaStreamWaitEvent(st, c->ev_a2, 0));
    c->pend = 0;
  }
  if (run()) TRY(net_fwd_layer<T>(c, (const T*)c->h1, c->H, c->H, thc, o.w2, o.b2, (T*)c->h2, 0, nullptr, st));
  mark();
  if (run()) TRY(net_fwd_layer<T>(c, (const T*)c->h2, c->H, c->D0, thc, o.w3, o.b3, nullptr, 1, nullptr, st));
  mark();
  // side branch: the data term D = alpha H^T - d and its g_alpha part need only
  // alpha_hat; they overlap the view and pixel kernels of the main chain
  // (large-grid path, any row count: the same side branch beside the view passes)
  const bool lfork = sizeof(T) == 8 && c->capturing && fused && c->large && c->side && c->gad && c->dgemm;
  const bool dfork = ((fork && c->dfork_ok) || lfork) && c->gad && run();
  if (dfork) {
    CK_CUDA(cudaEventRecord(c->ev_vf, st));
    CK_CUDA(cudaStreamWaitEvent(c->side, c->ev_vf, 0));
    g_pdl_off = 1;
    const int tl_keep = g_tl_cur;
    g_tl_cur = 0;          // side-branch kernels carry no timeline slot (the slots time the main chain)
    const int rd = data_term<T>(c, c->alpha_hat, c->side);
    if (rd == PDF_OK)
      gad_kernel<T><<<dim3((c->M0 + 255) / 256, c->d.S * c->d.n), 256, 0, c->side>>>(
          (const C<T>*)c->grows, (const C<T>*)c->hs, (C<T>*)c->gad, c->d.R, c->M0);
    g_tl_cur = tl_keep;
    g_pdl_off = 0;
    TRY(rd);
    CK_CUDA(cudaGetLastError());
    CK_CUDA(cudaEventRecord(c->ev_gad, c->side));
  }
  c->skip_data = dfork;
  const int rf = run() ? phys_forward<T>(c, c->alpha_hat, st) : PDF_OK;
  c->skip_data = 0;
  TRY(rf);
  // side branch: the data part of g_alpha (needs only g_rows) overlaps the pixel kernel
  const bool gfork = fork && c->gad && run() && !dfork;
  if (gfork) {
    CK_CUDA(cudaEventRecord(c->ev_vf, st));
    CK_CUDA(cudaStreamWaitEvent(c->side, c->ev_vf, 0));
    g_pdl_off = 1;
    // (gad_kernel carries no timeline slot argument)
    gad_kernel<T><<<dim3((c->M0 + 255) / 256, c->d.S * c->d.n), 256, 0, c->side>>>(
        (const C<T>*)c->grows, (const C<T>*)c->hs, (C<T>*)c->gad, c->d.R, c->M0);
    g_pdl_off = 0;
    CK_CUDA(cudaGetLastError());
    CK_CUDA(cudaEventRecord(c->ev_gad, c->side));
  }
  mark();
  if (run()) {
    if (c->split) TRY(split_pixel<T>(c, st));
    else TRY((phys_pixel<T, true>(c, nullptr, st)));
  }
  mark();
  if (gfork || dfork) {
    CK_CUDA(cudaStreamWaitEvent(st, c->ev_gad, 0));
    c->gad_ready = 1;
  }
  const int rb = run() ? phys_backward<T>(c, nullptr, c->gy, st, bd, trace, !c->split) : PDF_OK;
  c->gad_ready = 0;
  TRY(rb);
  mark();
  if (run() && c->split) TRY(split_finalize(c, bd, trace, st));
  mark();   // finalize is fused into view_bwd unless the pixel stage is split
  if constexpr (sizeof(T) == 8) {
    if (fused && c->xbwd) {
      // split backward: phases bwd_l3 / bwd_l2 = g_h of layers 3 / 2, bwd_l1 = g_W + Adam (all layers)
      if (run()) TRY(gh_x_layer(c, (const double*)c->gy, (const double*)c->h2, c->H, c->D0, (const double*)theta,
                                o.w3, (double*)c->gz2, fork ? c->tsnap : nullptr, st));
      if (fork) CK_CUDA(cudaEventRecord(c->ev_g3, st));
      mark();
      if (run()) TRY(gh_x_layer(c, (const double*)c->gz2, (const double*)c->h1, c->H, c->H, (const double*)theta,
                                o.w2, (double*)c->gz1, nullptr, st));
      if (fork) CK_CUDA(cudaEventRecord(c->ev_g2, st));
      mark();
      if (fork) {
        // critical path: W1 (the next forward starts with it); side: W3 after
        // g_h3, W2 after g_h2 (full dependencies, no PDL)
        if (run()) TRY(adam_x_all(c, (double*)theta, (double*)m, (double*)v, st, 1, c->tsnap));
        CK_CUDA(cudaStreamWaitEvent(c->side, c->ev_g3, 0));
        g_pdl_off = 1;
        const int tl_keep = g_tl_cur;
        g_tl_cur = 0;
        int r1 = run() ? adam_x_all(c, (double*)theta, (double*)m, (double*)v, c->side, 4, c->tsnap) : PDF_OK;
        cudaError_t e1 = cudaStreamWaitEvent(c->side, c->ev_g2, 0);
        int r2 = run() && r1 == PDF_OK ? adam_x_all(c, (double*)theta, (double*)m, (double*)v, c->side, 2, c->tsnap)
                                       : PDF_OK;
        g_tl_cur = tl_keep;
        g_pdl_off = 0;
        TRY(r1);
        TRY(r2);
        CK_CUDA(e1);
        CK_CUDA(cudaEventRecord(c->ev_a2, c->side));
        c->pend = 1;
      } else {
        if (run()) TRY(adam_x_all(c, (double*)theta, (double*)m, (double*)v, st));
      }
      mark();
      return PDF_OK;
    }
  }
  if (run()) TRY(net_bwd_layer<T>(c, (const T*)c->gy, (const T*)c->h2, c->H, c->D0, th, o.w3, o.b3, (T*)m, (T*)v,
                                  (T*)grad, fused, (T*)c->gz2, st));
  mark();
  if (run()) TRY(net_bwd_layer<T>(c, (const T*)c->gz2, (const T*)c->h1, c->H, c->H, th, o.w2, o.b2, (T*)m, (T*)v,
                                  (T*)grad, fused, (T*)c->gz1, st));
  mark();
  if (run()) TRY(net_bwd_layer<T>(c, (const T*)c->gz1, (const T*)c->x0, c->D0, c->H, th, o.w1, o.b1, (T*)m, (T*)v,
                                  (T*)grad, fused, nullptr, st));
  mark();
  return PDF_OK;
}

// ---------------------------------------------------------------------------
template <typename T>
static int create_impl(pdf_ctx* c, void* ws, size_t bytes, cudaStream_t st) {
  Ws w;
  w.base = (char*)ws;
  w.base = (char*)(((uintptr_t)ws + 255) & ~uintptr_t(255));
  plan<T>(c, w);
  if (w.off + ((char*)w.base - (char*)ws) > bytes) return fail(PDF_ENOMEM, "workspace too small");
  // twiddles (fp64 on the host, rounded once)
  std::vector<C<T>> tw(c->P), twm(c->M);
  for (int k = 0; k < c->P; ++k) {
    const double a = -2.0 * M_PI * (double)k / c->P;
    tw[k] = mk_host<T>(cos(a), sin(a));
  }
  for (int k = 0; k < c->M; ++k) {
    const double a = -2.0 * M_PI * (double)k / c->M;
    twm[k] = mk_host<T>(cos(a), sin(a));
  }
  CK_CUDA(cudaMemcpyAsync(c->twP, tw.data(), tw.size() * sizeof(C<T>), cudaMemcpyHostToDevice, st));
  CK_CUDA(cudaMemcpyAsync(c->twM, twm.data(), twm.size() * sizeof(C<T>), cudaMemcpyHostToDevice, st));
  CK_CUDA(cudaMemcpyAsync(c->c_inc, c->c_inc_h.data(), c->d.S * sizeof(double), cudaMemcpyHostToDevice, st));
  CK_CUDA(cudaMemcpyAsync(c->c_sca, c->c_sca_h.data(), c->d.S * sizeof(double), cudaMemcpyHostToDevice, st));
  CK_CUDA(cudaMemsetAsync(c->err, 0, c->d.S * sizeof(int), st));
  CK_CUDA(cudaMemsetAsync(c->step, 0, 2 * sizeof(int), st));
  if (c->ticket) CK_CUDA(cudaMemsetAsync(c->ticket, 0, (size_t)c->d.S * (c->H / 64 + 1) * sizeof(int), st));
  const int PP = c->P * c->P;
  permute_khat_kernel<T><<<(PP + 255) / 256, 256, 0, st>>>((const C<T>*)c->d.gd_kernel_hat, (C<T>*)c->khat, c->P,
                                                            c->large && c->E >= 4 ? 1 : 0);
  CK_CUDA(cudaGetLastError());
  {
    // H = G_S o expand (R x M0), two fixed-order contraction passes in float64
    double2* t1 = nullptr;
    const long long n1 = (long long)c->d.R * c->M * c->K;
    CK_CUDA(cudaMallocAsync((void**)&t1, (size_t)n1 * sizeof(double2), st));
    hs_rows_kernel<T><<<(unsigned)((n1 + 255) / 256), 256, 0, st>>>((const C<T>*)c->d.gs_matrix, t1, c->M, c->d.mf,
                                                                    c->d.R);
    const int n2 = c->d.R * c->M0;
    hs_cols_kernel<T><<<(n2 + 255) / 256, 256, 0, st>>>(t1, (C<T>*)c->hs, c->M, c->d.mf, c->d.R);
    const cudaError_t e = cudaGetLastError();
    cudaFreeAsync(t1, st);
    CK_CUDA(e);
  }
  CK_CUDA(cudaStreamSynchronize(st));
  return PDF_OK;
}

extern "C" int pdf_ctx_create(const pdf_desc* d, void* ws, size_t bytes, void* stream, pdf_ctx** out) {
  if (!out || !ws) return fail(PDF_EINVAL, "null output / workspace");
  pdf_ctx* c = new pdf_ctx();
  int r = derive(c, d);
  if (r != PDF_OK) { delete c; return r; }
  c->c_inc_h.assign(d->c_inc, d->c_inc + d->S);
  c->c_sca_h.assign(d->c_sca, d->c_sca + d->S);
  for (int s = 0; s < d->S; ++s)
    if (!(c->c_inc_h[s] > 0) || !(c->c_sca_h[s] > 0)) { delete c; return fail(PDF_EINVAL, "zero normaliser"); }
  cudaStream_t st = (cudaStream_t)stream;
  r = d->dtype == PDF_F64 ? create_impl<double>(c, ws, bytes, st) : create_impl<float>(c, ws, bytes, st);
  if (r != PDF_OK) { delete c; return r; }
  *out = c;
  return PDF_OK;
}

extern "C" int pdf_ctx_destroy(pdf_ctx* c) {
  if (!c) return PDF_OK;
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->g_stream) cudaStreamDestroy(c->g_stream);
  if (c->side) cudaStreamDestroy(c->side);
  for (cudaEvent_t e : {c->ev_g3, c->ev_g2, c->ev_a2, c->ev_vf, c->ev_gad}) if (e) cudaEventDestroy(e);
  delete c;
  return PDF_OK;
}

extern "C" int pdf_ctx_paths(const pdf_ctx* c, int32_t* paths) {
  if (!c || !paths) return fail(PDF_EINVAL, "null argument");
  *paths = (c->large ? PDF_PATH_LARGE_GRID : 0) | (c->dgemm ? PDF_PATH_DATA_GEMM : 0) |
           (c->xbwd ? PDF_PATH_SPLIT_BWD : 0) | (c->large ? 0 : c->CS << PDF_PATH_VIEW_CLUSTER_SHIFT);
  return PDF_OK;
}

extern "C" int pdf_net_dims(const pdf_ctx* c, int32_t* rows, int32_t* d0, int32_t* hidden, int64_t* np) {
  if (!c) return fail(PDF_EINVAL, "null ctx");
  if (rows) *rows = c->rows;
  if (d0) *d0 = c->D0;
  if (hidden) *hidden = c->H;
  if (np) *np = c->Np;
  return PDF_OK;
}

int pdf_ctx_info(const pdf_ctx* c, int* M, int* dtype) {
  if (!c) return fail(PDF_EINVAL, "null ctx");
  if (M) *M = c->M;
  if (dtype) *dtype = c->d.dtype;
  return PDF_OK;
}

#define DISPATCH(c, fn, ...) ((c)->d.dtype == PDF_F64 ? fn<double>(__VA_ARGS__) : fn<float>(__VA_ARGS__))

template <typename T>
static int loss_grad_impl(pdf_ctx* c, const void* alpha, void* galpha, double* bd, cudaStream_t st) {
  TRY(phys_forward<T>(c, alpha, st));
  TRY((phys_pixel<T, true>(c, nullptr, st)));
  return phys_backward<T>(c, galpha ? galpha : c->galpha, nullptr, st, bd, nullptr, true);
}

extern "C" int pdf_loss_grad(pdf_ctx* c, const void* alpha, void* galpha, double* bd, void* stream) {
  if (!c || !alpha) return fail(PDF_EINVAL, "null argument");
  return DISPATCH(c, loss_grad_impl, c, alpha, galpha, bd, (cudaStream_t)stream);
}

template <typename T>
static int loss_value_impl(pdf_ctx* c, const void* alpha, double* bd, void* chi, cudaStream_t st) {
  TRY(phys_forward<T>(c, alpha, st));
  TRY((phys_pixel<T, false>(c, chi, st)));
  return finalize(c, bd, nullptr, st);
}

extern "C" int pdf_loss_value(pdf_ctx* c, const void* alpha, double* bd, void* chi, void* stream) {
  if (!c || !alpha) return fail(PDF_EINVAL, "null argument");
  return DISPATCH(c, loss_value_impl, c, alpha, bd, chi, (cudaStream_t)stream);
}

template <typename T>
static int net_setup_impl(pdf_ctx* c, const void* alpha0, int n_all, int off, cudaStream_t st) {
  // keep this context's own views of alpha0 (the network output adds them back)
  const size_t row = (size_t)c->M0 * sizeof(C<T>);
  for (int s_ = 0; s_ < c->d.S; ++s_)
    CK_CUDA(cudaMemcpyAsync((char*)c->alpha0 + (size_t)s_ * c->d.n * row,
                            (const char*)alpha0 + ((size_t)s_ * n_all + off) * row, c->d.n * row,
                            cudaMemcpyDeviceToDevice, st));
  NetSetupArgs<T> a = {};
  a.n = c->d.n; a.M0 = c->M0; a.joint = c->d.joint; a.H = c->H; a.n_all = n_all; a.off = off;
  a.alpha0 = (const C<T>*)alpha0; a.x0 = (T*)c->x0; a.cout = (T*)c->cout;
  net_setup_kernel<T><<<c->d.S, 256, 0, st>>>(a);
  CK_CUDA(cudaGetLastError());
  return PDF_OK;
}

extern "C" int pdf_net_setup(pdf_ctx* c, const void* alpha0, void* stream) {
  if (!c || !alpha0) return fail(PDF_EINVAL, "null argument");
  return DISPATCH(c, net_setup_impl, c, alpha0, c->d.n, 0, (cudaStream_t)stream);
}

template <typename T>
static int net_forward_impl(pdf_ctx* c, const void* theta, void* ahat, cudaStream_t st) {
  TRY(net_forward_all<T>(c, theta, nullptr, st));
  if (ahat) {
    const size_t bytes = (size_t)c->d.S * c->d.n * c->M0 * sizeof(C<T>);
    CK_CUDA(cudaMemcpyAsync(ahat, c->alpha_hat, bytes, cudaMemcpyDeviceToDevice, st));
  }
  return PDF_OK;
}

extern "C" int pdf_net_forward(pdf_ctx* c, const void* theta, void* ahat, void* stream) {
  if (!c || !theta) return fail(PDF_EINVAL, "null argument");
  return DISPATCH(c, net_forward_impl, c, theta, ahat, (cudaStream_t)stream);
}

template <typename T>
static int grad_loss_impl(pdf_ctx* c, const void* theta, void* grad, double* bd, cudaStream_t st) {
  // unfused: theta is only read (the bwd kernels write grad instead of Adam)
  return iteration<T>(c, const_cast<void*>(theta), nullptr, nullptr, grad, bd, nullptr, 0, st);
}

extern "C" int pdf_grad_loss(pdf_ctx* c, const void* theta, void* grad, double* bd, void* stream) {
  if (!c || !theta || !grad) return fail(PDF_EINVAL, "null argument");
  return DISPATCH(c, grad_loss_impl, c, theta, grad, bd, (cudaStream_t)stream);
}

template <typename T>
static int adam_impl(pdf_ctx* c, void* theta, void* m, void* v, const void* g, long long cnt, int t,
                     cudaStream_t st) {
  const double bc1 = 1.0 / (1.0 - pow(c->d.adam_b1, (double)t)), bc2 = 1.0 / (1.0 - pow(c->d.adam_b2, (double)t));
  int blocks = (int)std::min<long long>((cnt + 255) / 256, 148LL * 16);
  adam_flat_kernel<T><<<blocks, 256, 0, st>>>((T*)theta, (T*)m, (T*)v, (const T*)g, cnt, (T)c->d.lr,
                                              (T)c->d.adam_b1, (T)c->d.adam_b2, (T)c->d.adam_eps, (T)bc1,
                                              (T)bc2, c->err);
  CK_CUDA(cudaGetLastError());
  return PDF_OK;
}

extern "C" int pdf_adam_step(pdf_ctx* c, void* theta, void* m, void* v, const void* g, int64_t count, int32_t t,
                             void* stream) {
  if (!c || !theta || !m || !v || !g || t < 1 || count < 0) return fail(PDF_EINVAL, "bad argument");
  return DISPATCH(c, adam_impl, c, theta, m, v, g, (long long)count, t, (cudaStream_t)stream);
}

extern "C" int pdf_set_norms(pdf_ctx* c, const double* ci, const double* cs, void* stream) {
  if (!c || !ci || !cs) return fail(PDF_EINVAL, "null argument");
  for (int s = 0; s < c->d.S; ++s)
    if (!(ci[s] > 0) || !(cs[s] > 0)) return fail(PDF_EINVAL, "zero normaliser");
  c->c_inc_h.assign(ci, ci + c->d.S);
  c->c_sca_h.assign(cs, cs + c->d.S);
  cudaStream_t st = (cudaStream_t)stream;
  CK_CUDA(cudaMemcpyAsync(c->c_inc, c->c_inc_h.data(), c->d.S * sizeof(double), cudaMemcpyHostToDevice, st));
  CK_CUDA(cudaMemcpyAsync(c->c_sca, c->c_sca_h.data(), c->d.S * sizeof(double), cudaMemcpyHostToDevice, st));
  CK_CUDA(cudaStreamSynchronize(st));
  return PDF_OK;
}

template <typename T>
static int train_impl(pdf_ctx* c, void* theta, void* m, void* v, int t0, int k, double* trace, int use_graph,
                      cudaStream_t st) {
  set_ints_kernel<<<1, 1, 0, st>>>(c->step, t0, t0);
  CK_CUDA(cudaGetLastError());
  // trace row = step - 1 - t0: offset the base pointer so the kernel indexes by step
  double* tr = trace ? trace - (size_t)t0 * c->d.S * 6 : nullptr;
  if (!use_graph) {
    for (int i = 0; i < k; ++i) TRY(iteration<T>(c, theta, m, v, nullptr, nullptr, tr, 1, st));
    return PDF_OK;
  }
  // iterations per captured graph (graph boundaries cost a full drain + launch)
  static const int G = std::max(1, env_int("PDF_GRAPH_ITERS", 10));
  if (!(c->gexec && c->g_theta == theta && c->g_m == m && c->g_v == v && c->g_trace == (void*)tr)) {
    if (c->gexec) { cudaGraphExecDestroy(c->gexec); c->gexec = nullptr; }
    // capture on a private stream (the caller's may be the legacy default
    // stream, which cannot capture); the graph is then launched on `st`
    if (!c->g_stream) CK_CUDA(cudaStreamCreateWithFlags(&c->g_stream, cudaStreamNonBlocking));
    {
      // opt-in (PDF_L2_PERSIST=1): keep theta / m / v L2-resident across
      // iterations when the caller placed them in one window (alloc_state,
      // BatchReconstructor): an access-policy window on the capture streams,
      // inherited by the captured kernel nodes.  Measured no change at cfg2 /
      // cfg3 / cfg5 -- the Adam stream already hits L2 ~80 %
      static const int persist = env_int("PDF_L2_PERSIST", 0);
      const size_t bytes = (size_t)c->d.S * c->Np * (c->d.dtype == PDF_F64 ? 8 : 4);
      char* ps[3] = {(char*)theta, (char*)m, (char*)v};
      char* lo = std::min({ps[0], ps[1], ps[2]});
      char* hi = std::max({ps[0], ps[1], ps[2]}) + bytes;
      int dev = 0, maxwin = 0, maxpers = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, dev);
      cudaDeviceGetAttribute(&maxpers, cudaDevAttrMaxPersistingL2CacheSize, dev);
      const size_t win = (size_t)(hi - lo);
      if (env_int("PDF_L2_DEBUG", 0))
        fprintf(stderr, "[pdf] L2 window %zu bytes (max window %d, max persisting %d, state %zu x 3)\n", win, maxwin,
                maxpers, bytes);
      if (persist && maxwin > 0 && maxpers > 0 && win <= (size_t)maxwin && win <= 3 * bytes + (3 << 20)) {
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min((size_t)maxpers, win));
        cudaStreamAttrValue at = {};
        at.accessPolicyWindow.base_ptr = lo;
        at.accessPolicyWindow.num_bytes = win;
        at.accessPolicyWindow.hitRatio = std::min(1.0f, (float)maxpers / (float)win);
        at.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        at.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cudaStreamSetAttribute(c->g_stream, cudaStreamAttributeAccessPolicyWindow, &at);
        if (c->side) cudaStreamSetAttribute(c->side, cudaStreamAttributeAccessPolicyWindow, &at);
        c->l2_window = at;
        c->l2_set = 1;
      }
      (void)cudaGetLastError();
    }
    if (c->xbwd && !c->side) {
      CK_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
      CK_CUDA(cudaEventCreateWithFlags(&c->ev_g3, cudaEventDisableTiming));
      CK_CUDA(cudaEventCreateWithFlags(&c->ev_g2, cudaEventDisableTiming));
      CK_CUDA(cudaEventCreateWithFlags(&c->ev_a2, cudaEventDisableTiming));
      CK_CUDA(cudaEventCreateWithFlags(&c->ev_vf, cudaEventDisableTiming));
      CK_CUDA(cudaEventCreateWithFlags(&c->ev_gad, cudaEventDisableTiming));
      if (c->l2_set) cudaStreamSetAttribute(c->side, cudaStreamAttributeAccessPolicyWindow, &c->l2_window);
    }
    cudaGraph_t g;
    CK_CUDA(cudaStreamBeginCapture(c->g_stream, cudaStreamCaptureModeThreadLocal));
    int r = PDF_OK;
    c->capturing = env_int("PDF_ADAM_FORK", 1);
    c->pend = 0;
    for (int i = 0; i < G && r == PDF_OK; ++i) {
      g_tl_iter = i;
      r = iteration<T>(c, theta, m, v, nullptr, nullptr, tr, 1, c->g_stream);
    }
    if (c->pend) {   // join the last side branch before the capture ends
      cudaStreamWaitEvent(c->g_stream, c->ev_a2, 0);
      c->pend = 0;
    }
    c->capturing = 0;
    g_tl_cur = 0;
    cudaError_t e = cudaStreamEndCapture(c->g_stream, &g);
    if (r != PDF_OK) return r;
    if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&c->gexec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(PDF_ECUDA, std::string("instantiate: ") + cudaGetErrorString(e));
    c->g_theta = theta; c->g_m = m; c->g_v = v; c->g_trace = (void*)tr;
  }
  int done = 0;
  for (; done + G <= k; done += G) CK_CUDA(cudaGraphLaunch(c->gexec, st));
  for (; done < k; ++done) TRY(iteration<T>(c, theta, m, v, nullptr, nullptr, tr, 1, st));
  return PDF_OK;
}

extern "C" int pdf_timeline_reset(pdf_ctx* c, int32_t on, void* stream) {
  if (!c) return fail(PDF_EINVAL, "null ctx");
  cudaStream_t st = (cudaStream_t)stream;
  if (on != 2) {   // 2: clear the stamps only (keep the captured graph)
    c->tl_on = on ? 1 : 0;
    if (c->gexec) { cudaGraphExecDestroy(c->gexec); c->gexec = nullptr; }   // recapture with / without slots
  }
  std::vector<unsigned long long> init(PDF_TL_SLOTS * 3);
  for (int i = 0; i < PDF_TL_SLOTS; ++i) { init[3 * i] = init[3 * i + 1] = ~0ULL; init[3 * i + 2] = 0; }
  CK_CUDA(cudaMemcpyToSymbolAsync(g_tl, init.data(), init.size() * sizeof(unsigned long long), 0,
                                  cudaMemcpyHostToDevice, st));
  std::vector<unsigned long long> zs(PDF_TL_SLOTS * TL_STAGES, 0ULL);
  CK_CUDA(cudaMemcpyToSymbolAsync(g_tls, zs.data(), zs.size() * sizeof(unsigned long long), 0,
                                  cudaMemcpyHostToDevice, st));
  CK_CUDA(cudaStreamSynchronize(st));
  return PDF_OK;
}

extern "C" int pdf_timeline_read(uint64_t* out, void* stream) {
  if (!out) return fail(PDF_EINVAL, "null output");
  cudaStream_t st = (cudaStream_t)stream;
  CK_CUDA(cudaMemcpyFromSymbolAsync(out, g_tl, PDF_TL_SLOTS * 3 * sizeof(unsigned long long), 0,
                                    cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaMemcpyFromSymbolAsync(out + PDF_TL_SLOTS * 3, g_tls,
                                    PDF_TL_SLOTS * TL_STAGES * sizeof(unsigned long long), 0,
                                    cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
  return PDF_OK;
}

extern "C" int pdf_train(pdf_ctx* c, void* theta, void* m, void* v, int32_t t0, int32_t k, double* trace,
                         int32_t use_graph, void* stream) {
  if (!c || !theta || !m || !v || k < 0 || t0 < 0) return fail(PDF_EINVAL, "bad argument");
  return DISPATCH(c, train_impl, c, theta, m, v, t0, k, trace, use_graph, (cudaStream_t)stream);
}

template <typename T>
static int apply_gd_impl(pdf_ctx* c, const void* x, void* y, int count, int adjoint, cudaStream_t st) {
  if (c->large) {
    VLArgs<T> b = vl_common<T>(c);
    b.x = (const C<T>*)x; b.y = (C<T>*)y; b.conj_in = adjoint; b.conj_out = adjoint;
    return vl_conv<T, VIEW_APPLY>(c, b, count, st);
  }
  ViewArgs<T> a = view_common<T>(c);
  a.x = (const C<T>*)x; a.y = (C<T>*)y; a.conj_in = adjoint; a.conj_out = adjoint;
  return launch_view<T, VIEW_APPLY>(c, a, count, st);
}

extern "C" int pdf_apply_gd(pdf_ctx* c, const void* x, void* y, int32_t count, int32_t adjoint, void* stream) {
  if (!c || !x || !y || count < 1) return fail(PDF_EINVAL, "bad argument");
  return DISPATCH(c, apply_gd_impl, c, x, y, count, adjoint, (cudaStream_t)stream);
}

template <typename T>
static int gs_fwd_impl(pdf_ctx* c, const void* img, void* rows, int count, cudaStream_t st) {
  gs_forward_kernel<T><<<dim3(c->d.R, count), 256, 0, st>>>((const C<T>*)img, (C<T>*)rows,
                                                            (const C<T>*)c->d.gs_matrix, c->M * c->M, c->d.R);
  CK_CUDA(cudaGetLastError());
  return PDF_OK;
}

extern "C" int pdf_gs_forward(pdf_ctx* c, const void* img, void* rows, int32_t count, void* stream) {
  if (!c || !img || !rows || count < 1) return fail(PDF_EINVAL, "bad argument");
  return DISPATCH(c, gs_fwd_impl, c, img, rows, count, (cudaStream_t)stream);
}

template <typename T>
static int gs_adj_impl(pdf_ctx* c, const void* rows, void* img, int count, cudaStream_t st) {
  const int np = c->M * c->M;
  gs_adjoint_kernel<T><<<dim3((np + 255) / 256, count), 256, 0, st>>>((const C<T>*)rows, (C<T>*)img,
                                                                      (const C<T>*)c->d.gs_matrix, np, c->d.R);
  CK_CUDA(cudaGetLastError());
  return PDF_OK;
}

extern "C" int pdf_gs_adjoint(pdf_ctx* c, const void* rows, void* img, int32_t count, void* stream) {
  if (!c || !img || !rows || count < 1) return fail(PDF_EINVAL, "bad argument");
  return DISPATCH(c, gs_adj_impl, c, rows, img, count, (cudaStream_t)stream);
}

template <typename T>
static int expand_impl(pdf_ctx* c, const void* alpha, void* img, int count, cudaStream_t st) {
  const int np = c->M * c->M;
  expand_kernel<T><<<dim3((np + 255) / 256, count), 256, 0, st>>>((const C<T>*)alpha, (C<T>*)img,
                                                                  (const C<T>*)c->twM, c->M, c->d.mf);
  CK_CUDA(cudaGetLastError());
  return PDF_OK;
}

extern "C" int pdf_expand(pdf_ctx* c, const void* alpha, void* img, int32_t count, void* stream) {
  if (!c || !alpha || !img || count < 1) return fail(PDF_EINVAL, "bad argument");
  return DISPATCH(c, expand_impl, c, alpha, img, count, (cudaStream_t)stream);
}

template <typename T>
static int truncate_impl(pdf_ctx* c, const void* img, void* alpha, int count, cudaStream_t st) {
  truncate_kernel<T><<<dim3(c->M0, count), 256, 0, st>>>((const C<T>*)img, (C<T>*)alpha, (const C<T>*)c->twM,
                                                         c->M, c->d.mf);
  CK_CUDA(cudaGetLastError());
  return PDF_OK;
}

extern "C" int pdf_truncate(pdf_ctx* c, const void* img, void* alpha, int32_t count, void* stream) {
  if (!c || !alpha || !img || count < 1) return fail(PDF_EINVAL, "bad argument");
  return DISPATCH(c, truncate_impl, c, img, alpha, count, (cudaStream_t)stream);
}

template <typename T>
static int cco_impl(pdf_ctx* c, const void* chi, void* out, int count, double tau, double eta_max, double delta,
                    int radius, double eps_gf, cudaStream_t st) {
  if (count > c->d.S) return fail(PDF_EINVAL, "cco count exceeds scenes (scratch)");
  const int np = c->M * c->M;
  cco_pass1_kernel<T><<<dim3((np + 255) / 256, count, 2), 256, 0, st>>>((const C<T>*)chi, (T*)c->ab, c->M, radius,
                                                                        (T)eps_gf);
  CK_CUDA(cudaGetLastError());
  cco_pass2_kernel<T><<<dim3((np + 255) / 256, count), 256, 0, st>>>((const C<T>*)chi, (const T*)c->ab,
                                                                     (C<T>*)out, c->M, radius, (T)tau,
                                                                     (T)eta_max, (T)delta);
  CK_CUDA(cudaGetLastError());
  return PDF_OK;
}

extern "C" int pdf_apply_cco(pdf_ctx* c, const void* chi, void* out, int32_t count, double tau, double eta_max,
                             double delta, int32_t radius, double eps_gf, void* stream) {
  if (!c || !chi || !out || count < 1 || radius < 1) return fail(PDF_EINVAL, "bad argument");
  return DISPATCH(c, cco_impl, c, chi, out, count, tau, eta_max, delta, radius, eps_gf, (cudaStream_t)stream);
}

extern "C" int pdf_get_error(pdf_ctx* c, int32_t* err_host, void* stream) {
  if (!c || !err_host) return fail(PDF_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  CK_CUDA(cudaMemcpyAsync(err_host, c->err, c->d.S * sizeof(int), cudaMemcpyDeviceToHost, st));
  CK_CUDA(cudaStreamSynchronize(st));
  CK_CUDA(cudaMemsetAsync(c->err, 0, c->d.S * sizeof(int), st));
  return PDF_OK;
}

// ---------------------------------------------------------------------------
// measurement hooks (bench.py roofline block)

template <typename T>
static int profile_impl(pdf_ctx* c, void* theta, void* m, void* v, int t0, int iters, float* ms, cudaStream_t st) {
  cudaEvent_t ev[PDF_NPHASES + 1];
  for (auto& e : ev) CK_CUDA(cudaEventCreate(&e));
  for (int i = 0; i < PDF_NPHASES; ++i) ms[i] = 0.f;
  set_ints_kernel<<<1, 1, 0, st>>>(c->step, t0, t0);
  int r = PDF_OK;
  for (int it = 0; it < iters && r == PDF_OK; ++it) {
    r = iteration<T>(c, theta, m, v, nullptr, nullptr, nullptr, 1, st, ev);
    if (r != PDF_OK) break;
    CK_CUDA(cudaEventSynchronize(ev[PDF_NPHASES]));
    for (int i = 0; i < PDF_NPHASES; ++i) {
      float t = 0.f;
      cudaEventElapsedTime(&t, ev[i], ev[i + 1]);
      ms[i] += t / iters;
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return r;
}

extern "C" int pdf_profile_train(pdf_ctx* c, void* theta, void* m, void* v, int32_t t0, int32_t iters, float* ms,
                                 void* stream) {
  if (!c || !theta || !m || !v || !ms || iters < 1) return fail(PDF_EINVAL, "bad argument");
  return DISPATCH(c, profile_impl, c, theta, m, v, t0, iters, ms, (cudaStream_t)stream);
}

__global__ void dfma_probe_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
         a7 = a0 + 7;
  const double x = 0.999999, y = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, x, y); a1 = fma(a1, x, y); a2 = fma(a2, x, y); a3 = fma(a3, x, y);
      a4 = fma(a4, x, y); a5 = fma(a5, x, y); a6 = fma(a6, x, y); a7 = fma(a7, x, y);
    }
  }
  const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;   // keep the chains alive
}

extern "C" int pdf_fp64_probe(double* gflops, void* stream) {
  if (!gflops) return fail(PDF_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 0;
  CK_CUDA(cudaGetDevice(&dev));
  CK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out = nullptr;
  CK_CUDA(cudaMallocAsync(&out, sizeof(double), st));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  dfma_probe_kernel<<<blocks, threads, 0, st>>>(out, 64);   // warm-up
  cudaEvent_t a, b;
  CK_CUDA(cudaEventCreate(&a));
  CK_CUDA(cudaEventCreate(&b));
  CK_CUDA(cudaEventRecord(a, st));
  dfma_probe_kernel<<<blocks, threads, 0, st>>>(out, iters);
  CK_CUDA(cudaEventRecord(b, st));
  CK_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFreeAsync(out, st);
  *gflops = 2.0 * 64.0 * iters * (double)blocks * threads / (ms * 1e-3) / 1e9;
  return PDF_OK;
}

// ---------------------------------------------------------------------------
// incidence-sharded iteration; see pdf_shard.cuh

extern "C" int pdf_net_setup_sharded(pdf_ctx* c, const void* alpha0_all, int32_t n_all, int32_t view_offset,
                                     void* stream) {
  if (!c || !alpha0_all || c->d.joint || view_offset < 0 || view_offset + c->d.n > n_all)
    return fail(PDF_EINVAL, "bad sharded network setup (joint_views cannot be sharded)");
  return DISPATCH(c, net_setup_impl, c, alpha0_all, n_all, view_offset, (cudaStream_t)stream);
}

extern "C" int pdf_shard_buffer_sizes(const pdf_ctx* c, int64_t* red1, int64_t* red2) {
  if (!c) return fail(PDF_EINVAL, "null ctx");
  const int64_t img = (int64_t)c->M * c->M;
  if (red1) *red1 = (int64_t)c->d.S * (3 * img + 1);
  if (red2) *red2 = (int64_t)c->d.S * (2 * img + 2);
  return PDF_OK;
}

template <typename T>
static ShardArgs<T> shard_args(pdf_ctx* c, double* red1, double* red2) {
  ShardArgs<T> a = {};
  a.M = c->M; a.n = c->d.n; a.R = c->d.R; a.CS = c->NPV;
  a.beta = (T)c->d.beta; a.l1 = (T)c->d.lambda1; a.l2 = (T)c->d.lambda2; a.l3 = (T)c->d.lambda3;
  a.tau = (T)c->d.tau_b;
  a.J = (const C<T>*)c->J; a.E = (const C<T>*)c->E_; a.norms = c->norms; a.grows = (const C<T>*)c->grows;
  a.rfixed = c->d.freeze_r ? (const C<T>*)c->d.r_fixed : nullptr;
  a.c_inc = c->c_inc; a.red1 = red1; a.red2 = red2; a.dloss = c->dloss; a.pix = c->pix; a.part = c->part;
  a.gJ = (C<T>*)c->gJ; a.gE = (C<T>*)c->gE; a.err = c->err;
  return a;
}

template <typename T>
static int shard_a_impl(pdf_ctx* c, const void* theta, double* red1, cudaStream_t st) {
  TRY(net_forward_all<T>(c, theta, nullptr, st));
  TRY(phys_forward<T>(c, c->alpha_hat, st));
  ShardArgs<T> a = shard_args<T>(c, red1, nullptr);
  const int img = c->M * c->M;
  void* args[] = {&a};
  CK_CUDA(plain_launch(shard_numden_kernel<T>, dim3((img + 255) / 256, c->d.S), dim3(256), 0, st, args));
  return PDF_OK;
}

template <typename T>
static int shard_b_impl(pdf_ctx* c, const double* red1, double* red2, void* chi_out, cudaStream_t st) {
  ShardArgs<T> a = shard_args<T>(c, const_cast<double*>(red1), red2);
  a.chi_out = (C<T>*)chi_out;
  void* args[] = {&a};
  const dim3 grid(c->M / c->TX, c->M, c->d.S);
  CK_CUDA(plain_launch(shard_pixel_a_kernel<T>, grid, dim3(PIX_NW * 32), 0, st, args));
  shard_loss_sums_kernel<<<c->d.S, 128, 0, st>>>(c->part, c->dloss, red2, c->ntiles, c->d.n,
                                                 (size_t)c->M * c->M);
  CK_CUDA(cudaGetLastError());
  return PDF_OK;
}

template <typename T>
static int shard_c_impl(pdf_ctx* c, const void* theta, const double* red2, void* grad, double* bd, cudaStream_t st) {
  ShardArgs<T> a = shard_args<T>(c, nullptr, const_cast<double*>(red2));
  void* args[] = {&a};
  const dim3 grid(c->M / c->TX, c->M, c->d.S);
  CK_CUDA(plain_launch(shard_pixel_b_kernel<T>, grid, dim3(PIX_NW * 32), 0, st, args));
  TRY(phys_backward<T>(c, nullptr, c->gy, st));
  FinalizeArgs f = fin_args(c, bd, nullptr);
  shard_finalize_kernel<<<c->d.S, 128, 0, st>>>(f, red2, (size_t)c->M * c->M);
  CK_CUDA(cudaGetLastError());
  const Offs o = offsets(c);
  T* th = (T*)const_cast<void*>(theta);
  TRY(net_bwd_layer<T>(c, (const T*)c->gy, (const T*)c->h2, c->H, c->D0, th, o.w3, o.b3, nullptr, nullptr,
                       (T*)grad, 0, (T*)c->gz2, st));
  TRY(net_bwd_layer<T>(c, (const T*)c->gz2, (const T*)c->h1, c->H, c->H, th, o.w2, o.b2, nullptr, nullptr,
                       (T*)grad, 0, (T*)c->gz1, st));
  TRY(net_bwd_layer<T>(c, (const T*)c->gz1, (const T*)c->x0, c->D0, c->H, th, o.w1, o.b1, nullptr, nullptr,
                       (T*)grad, 0, nullptr, st));
  return PDF_OK;
}

// step c in three parts so each layer's gradient bucket can be reduced while the
// next layer's backward runs (the bucket of layer L = [W_L | b_L], contiguous)
template <typename T>
static int shard_c_part_impl(pdf_ctx* c, const void* theta, const double* red2, void* bucket, int part, double* bd,
                             cudaStream_t st) {
  const Offs o = offsets(c);
  T* th = (T*)const_cast<void*>(theta);
  // the kernels address grad + w_off / grad + b_off: shift the bucket base by the layer's offset
  auto base = [&](long long woff) { return (T*)((uintptr_t)bucket - (uintptr_t)woff * sizeof(T)); };
  if (part == 3) {
    ShardArgs<T> a = shard_args<T>(c, nullptr, const_cast<double*>(red2));
    void* args[] = {&a};
    const dim3 grid(c->M / c->TX, c->M, c->d.S);
    CK_CUDA(plain_launch(shard_pixel_b_kernel<T>, grid, dim3(PIX_NW * 32), 0, st, args));
    TRY(phys_backward<T>(c, nullptr, c->gy, st));
    FinalizeArgs f = fin_args(c, bd, nullptr);
    shard_finalize_kernel<<<c->d.S, 128, 0, st>>>(f, red2, (size_t)c->M * c->M);
    CK_CUDA(cudaGetLastError());
    return net_bwd_layer<T>(c, (const T*)c->gy, (const T*)c->h2, c->H, c->D0, th, o.w3, o.b3, nullptr, nullptr,
                            base(o.w3), 0, (T*)c->gz2, st);
  }
  if (part == 2)
    return net_bwd_layer<T>(c, (const T*)c->gz2, (const T*)c->h1, c->H, c->H, th, o.w2, o.b2, nullptr, nullptr,
                            base(o.w2), 0, (T*)c->gz1, st);
  return net_bwd_layer<T>(c, (const T*)c->gz1, (const T*)c->x0, c->D0, c->H, th, o.w1, o.b1, nullptr, nullptr,
                          base(o.w1), 0, nullptr, st);
}

extern "C" int pdf_shard_step_c_part(pdf_ctx* c, const void* theta, const double* red2, void* bucket, int32_t layer,
                                     double* breakdown, void* stream) {
  if (!c || !theta || !red2 || !bucket || layer < 1 || layer > 3 || c->d.S != 1)
    return fail(PDF_EINVAL, "bad argument");
  return DISPATCH(c, shard_c_part_impl, c, theta, red2, bucket, (int)layer, breakdown, (cudaStream_t)stream);
}

extern "C" int pdf_shard_step_c_scatter(pdf_ctx* c, const void* theta, const double* red2, double* const* peers,
                                        int32_t world, int32_t rank, int64_t shard, int32_t layer, double* breakdown,
                                        void* stream) {
  if (!c || !theta || !red2 || !peers || world < 1 || rank < 0 || rank >= world || shard < 2 || (shard & 1) ||
      shard * world < c->Np || layer < 1 || layer > 3 || c->d.S != 1 || c->d.dtype != PDF_F64)
    return fail(PDF_EINVAL, "bad argument");
  c->sc_peers = peers; c->sc_me = rank; c->sc_shard = shard;
  // the bucket base is unused in scatter mode: any non-null pointer keeps shard_c_part_impl's arithmetic defined
  const int r = shard_c_part_impl<double>(c, theta, red2, const_cast<void*>(theta), (int)layer, breakdown,
                                          (cudaStream_t)stream);
  c->sc_peers = nullptr;
  return r;
}

// ---------------------------------------------------------------------------
// tensor-parallel network (SURVEY 8(e)'s alternative to the gradient exchange;
// sharded.TensorParallelTrainer): the layers run on weight slices held in the
// caller's flat parameter vector, the physics of this context's views takes the
// network output from / gives its gradient to a column-block buffer
// Y[w][rows_all][N_w] (block w = output columns [w blk, w blk + N_w)).

namespace {

__device__ __forceinline__ long long tp_index(int col, int blk, int D0, int rows_all, int grow) {
  const int w = col / blk, j = col - w * blk, nw = min(blk, D0 - w * blk);
  return (long long)w * rows_all * blk + (long long)grow * nw + j;
}

template <typename T>
__global__ void tp_merge_kernel(const T* __restrict__ Y, int blk, int rows_all, int row0, int n, int D0, int M0,
                                const T* __restrict__ cout, const C<T>* __restrict__ alpha0,
                                C<T>* __restrict__ alpha_hat) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)n * D0) return;
  const int r = (int)(i / D0), col = (int)(i % D0);
  const T yv = Y[tp_index(col, blk, D0, rows_all, row0 + r)] * cout[col];
  const int half = D0 / 2, m = col < half ? col : col - half;
  const size_t off = (size_t)r * M0 + m;
  T* dst = reinterpret_cast<T*>(alpha_hat + off);
  const T* src = reinterpret_cast<const T*>(alpha0 + off);
  if (col < half) dst[0] = src[0] + yv; else dst[1] = src[1] + yv;
}

template <typename T>
__global__ void tp_scatter_kernel(const T* __restrict__ gy, T* __restrict__ GY, int blk, int rows_all, int row0, int n,
                                  int D0) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)n * D0) return;
  const int r = (int)(i / D0), col = (int)(i % D0);
  GY[tp_index(col, blk, D0, rows_all, row0 + r)] = gy[i];
}

__global__ void bias_tanh_kernel(double* __restrict__ x, const double* __restrict__ b, long long total, int n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) x[i] = tanh(x[i] + b[i % n]);
}

}  // namespace

static bool tp_ok(const pdf_ctx* c, int blk, int rows_all, int row0) {
  return c && c->d.S == 1 && !c->d.joint && c->d.dtype == PDF_F64 && blk >= 1 && blk <= c->D0 && row0 >= 0 &&
         row0 + c->d.n <= rows_all;
}

extern "C" int pdf_net_features(const pdf_ctx* c, void* x0, void* cout, void* stream) {
  if (!c || c->d.S != 1) return fail(PDF_EINVAL, "pdf_net_features: one-scene context required");
  const size_t el = c->d.dtype == PDF_F64 ? sizeof(double) : sizeof(float);
  if (x0) CK_CUDA(cudaMemcpyAsync(x0, c->x0, (size_t)c->rows * c->D0 * el, cudaMemcpyDeviceToDevice,
                                  (cudaStream_t)stream));
  if (cout) CK_CUDA(cudaMemcpyAsync(cout, c->cout, (size_t)c->D0 * el, cudaMemcpyDeviceToDevice,
                                    (cudaStream_t)stream));
  return PDF_OK;
}

extern "C" int pdf_net_layer_fwd(pdf_ctx* c, const void* in, int32_t K, int32_t N, const void* theta, int64_t w_off,
                                 int64_t b_off, void* out, int32_t mode, void* stream) {
  if (!c || !in || !theta || !out || K < 2 || N < 2 || (K & 1) || (N & 1) || c->d.S != 1 ||
      c->d.dtype != PDF_F64 || !(mode == 0 || mode == 2 || mode == 3) || (mode != 3 && b_off < 0) ||
      !env_int("PDF_NET_MMA", 1))
    return fail(PDF_EINVAL, "pdf_net_layer_fwd: bad arguments (float64, even widths, mode 0/2/3)");
  NetFwdArgs<double> a = {};
  a.rows = c->rows; a.K = K; a.N = N;
  a.in = (const double*)in; a.in_ss = (long long)c->rows * K;
  a.theta = (const double*)theta; a.th_ss = 0; a.w_off = w_off; a.b_off = mode == 3 ? 0 : b_off;
  a.out = (double*)out; a.out_ss = (long long)c->rows * N; a.final_layer = mode;
  a.w_early = 0;   // the slice may have been written by the launch right before
  return fwd_mma_layer(c, a, (cudaStream_t)stream);
}

extern "C" int pdf_net_layer_bwd(pdf_ctx* c, const void* gz, const void* hin, int32_t K, int32_t N,
                                 const void* theta, int64_t w_off, int64_t b_off, void* grad, void* gin,
                                 void* stream) {
  if (!c || !gz || !hin || !theta || !grad || K < 2 || N < 2 || (K & 1) || (N & 1) || b_off < 0 || c->d.S != 1 ||
      c->d.dtype != PDF_F64 || !env_int("PDF_NET_MMA", 1))
    return fail(PDF_EINVAL, "pdf_net_layer_bwd: bad arguments (float64, even widths)");
  double* const* const peers = c->sc_peers;
  c->sc_peers = nullptr;
  const int r = net_bwd_layer<double>(c, (const double*)gz, (const double*)hin, K, N,
                                      const_cast<double*>((const double*)theta), w_off, b_off, nullptr, nullptr,
                                      (double*)grad, 0, (double*)gin, (cudaStream_t)stream);
  c->sc_peers = peers;
  return r;
}

extern "C" int pdf_bias_tanh(void* x, const void* bias, int64_t rows, int32_t n, void* stream) {
  if (!x || !bias || rows < 1 || n < 1) return fail(PDF_EINVAL, "pdf_bias_tanh: bad arguments");
  const long long tot = rows * n;
  bias_tanh_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>((double*)x, (const double*)bias,
                                                                                   tot, n);
  CK_CUDA(cudaGetLastError());
  return PDF_OK;
}

extern "C" int pdf_shard_tp_a(pdf_ctx* c, const void* Y, int32_t blk, int32_t rows_all, int32_t row0, double* red1,
                              void* stream) {
  if (!tp_ok(c, blk, rows_all, row0) || !Y || !red1) return fail(PDF_EINVAL, "pdf_shard_tp_a: bad arguments");
  const cudaStream_t st = (cudaStream_t)stream;
  const long long tot = (long long)c->d.n * c->D0;
  tp_merge_kernel<double><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
      (const double*)Y, blk, rows_all, row0, c->d.n, c->D0, c->M0, (const double*)c->cout,
      (const C<double>*)c->alpha0, (C<double>*)c->alpha_hat);
  CK_CUDA(cudaGetLastError());
  TRY(phys_forward<double>(c, c->alpha_hat, st));
  ShardArgs<double> a = shard_args<double>(c, red1, nullptr);
  const int img = c->M * c->M;
  void* args[] = {&a};
  CK_CUDA(plain_launch(shard_numden_kernel<double>, dim3((img + 255) / 256, 1), dim3(256), 0, st, args));
  return PDF_OK;
}

extern "C" int pdf_shard_tp_c(pdf_ctx* c, const double* red2, void* GY, int32_t blk, int32_t rows_all, int32_t row0,
                              double* breakdown, void* stream) {
  if (!tp_ok(c, blk, rows_all, row0) || !red2 || !GY) return fail(PDF_EINVAL, "pdf_shard_tp_c: bad arguments");
  const cudaStream_t st = (cudaStream_t)stream;
  ShardArgs<double> a = shard_args<double>(c, nullptr, const_cast<double*>(red2));
  void* args[] = {&a};
  CK_CUDA(plain_launch(shard_pixel_b_kernel<double>, dim3(c->M / c->TX, c->M, 1), dim3(PIX_NW * 32), 0, st, args));
  TRY(phys_backward<double>(c, nullptr, c->gy, st));
  FinalizeArgs f = fin_args(c, breakdown, nullptr);
  shard_finalize_kernel<<<1, 128, 0, st>>>(f, red2, (size_t)c->M * c->M);
  CK_CUDA(cudaGetLastError());
  const long long tot = (long long)c->d.n * c->D0;
  tp_scatter_kernel<double><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>((const double*)c->gy, (double*)GY, blk,
                                                                           rows_all, row0, c->d.n, c->D0);
  CK_CUDA(cudaGetLastError());
  return PDF_OK;
}

extern "C" int pdf_adam_gather(pdf_ctx* c, const double* recv, double* const* thetas, double* m, double* v,
                               int32_t world, int32_t rank, int64_t shard, const int32_t* t_dev, void* stream) {
  if (!c || !recv || !thetas || !m || !v || !t_dev || world < 1 || rank < 0 || rank >= world || shard < 1 ||
      shard * world < c->Np || c->d.dtype != PDF_F64)
    return fail(PDF_EINVAL, "bad argument");
  const int blocks = (int)std::min<long long>((shard + 255) / 256, 148LL * 8);
  adam_gather_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(recv, thetas, m, v, world, rank, shard, c->Np,
                                                               c->d.lr, c->d.adam_b1, c->d.adam_b2, c->d.adam_eps,
                                                               (const int*)t_dev, c->err);
  CK_CUDA(cudaGetLastError());
  return PDF_OK;
}

extern "C" int pdf_net_offsets(const pdf_ctx* c, int64_t* offs) {
  if (!c || !offs) return fail(PDF_EINVAL, "null argument");
  const Offs o = offsets(const_cast<pdf_ctx*>(c));
  const long long v[7] = {o.w1, o.b1, o.w2, o.b2, o.w3, o.b3, c->Np};
  for (int i = 0; i < 7; ++i) offs[i] = v[i];
  return PDF_OK;
}

template <typename T>
static int adam_dev_impl(pdf_ctx* c, void* theta, void* m, void* v, const void* g, long long cnt, const int* t_dev,
                         cudaStream_t st) {
  int blocks = (int)std::min<long long>((cnt + 255) / 256, 148LL * 16);
  adam_flat_dev_kernel<T><<<blocks, 256, 0, st>>>((T*)theta, (T*)m, (T*)v, (const T*)g, cnt, (T)c->d.lr,
                                                  (T)c->d.adam_b1, (T)c->d.adam_b2, (T)c->d.adam_eps, t_dev, c->err);
  CK_CUDA(cudaGetLastError());
  return PDF_OK;
}

extern "C" int pdf_adam_step_dev(pdf_ctx* c, void* theta, void* m, void* v, const void* g, int64_t count,
                                 const int32_t* t_dev, void* stream) {
  if (!c || !theta || !m || !v || !g || !t_dev || count < 0) return fail(PDF_EINVAL, "bad argument");
  return DISPATCH(c, adam_dev_impl, c, theta, m, v, g, (long long)count, (const int*)t_dev, (cudaStream_t)stream);
}

extern "C" int pdf_shard_step_a(pdf_ctx* c, const void* theta, double* red1, void* stream) {
  if (!c || !theta || !red1 || c->d.joint) return fail(PDF_EINVAL, "bad argument");
  return DISPATCH(c, shard_a_impl, c, theta, red1, (cudaStream_t)stream);
}

extern "C" int pdf_shard_step_b(pdf_ctx* c, const double* red1, double* red2, void* chi_out, void* stream) {
  if (!c || !red1 || !red2) return fail(PDF_EINVAL, "bad argument");
  return DISPATCH(c, shard_b_impl, c, red1, red2, chi_out, (cudaStream_t)stream);
}

extern "C" int pdf_shard_step_c(pdf_ctx* c, const void* theta, const double* red2, void* grad, double* breakdown,
                                void* stream) {
  if (!c || !theta || !red2 || !grad) return fail(PDF_EINVAL, "bad argument");
  return DISPATCH(c, shard_c_impl, c, theta, red2, grad, breakdown, (cudaStream_t)stream);
}
