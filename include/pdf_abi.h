/*
 * pdf_abi.h -- C ABI of the B200 (sm_100a) PDF inverse-scattering hot path.
 *
 * The reference (`pdfisp`, pure Python) has no FFI; its drop-in boundary for
 * this path is a set of Python functions.  Each entry point below replaces
 * one of them (citations relative to /root/reference/pkg/src/pdfisp/):
 *
 *   pdf_ctx_create      LossContext.__post_init__      losses.py:52-80
 *                       (+ GreensOperators upload,      forward.py:69-94)
 *   pdf_loss_grad       grad_alpha / pipeline_forward   losses.py:309-312,
 *                       + pipeline_backward             losses.py:215-306
 *   pdf_loss_value      loss_total / recover_contrast   losses.py:250-252, cie.py:83-99
 *   pdf_net_setup       _feature_scales/_split_views    network.py:88-136
 *   pdf_net_forward     alpha0 + forward_net            network.py:143-150
 *   pdf_grad_loss       grad_loss                       network.py:183-223
 *   pdf_adam_step       adam_step                       network.py:248-264
 *   pdf_set_norms       LossContext c_inc / c_sca       losses.py:67-76
 *   pdf_train           reconstruct hot loop            reconstruct.py:217-221
 *   pdf_apply_gd        apply_gd / apply_gd_adjoint     forward.py:140-151
 *   pdf_gs_forward      J @ gs_matrix.T                 losses.py:229, reconstruct.py:62
 *   pdf_gs_adjoint      apply_gs_adjoint                forward.py:303-306
 *   pdf_expand          expand                          spectral.py:68-79
 *   pdf_truncate        truncate                        spectral.py:56-65
 *   pdf_apply_cco       apply_cco                       filters.py:56-67
 *   pdf_shard_step_a/b/c(_part)  one incidence-sharded iteration  losses.py:215-306, network.py:183-223
 *   pdf_net_layer_fwd/bwd, pdf_shard_tp_a/c  the same iteration with a    network.py:107-120, 183-223
 *                       tensor-parallel network (weight slices per rank)
 *                       (views split over ranks, caller all-reduces between the steps)
 *   pdf_bessel          bessel_j0/j1/y0/y1, hankel1_*   special.py:64-106
 *   pdf_build_greens    build_greens                    forward.py:101-137
 *   pdf_incident_fields incident_fields (line sources)  forward.py:174-181
 *                       (+ plane waves)
 *   pdf_solve_total_field _solve_bicgstab /            forward.py:193-248,
 *                       solve_total_field               forward.py:251-275
 *   pdf_relative_error  relative_error                  reconstruct.py:243-247
 *   pdf_count_components count_components               reconstruct.py:250-254
 *   pdf_chi_to_r        chi_to_r / r_to_chi             cie.py:24-39
 *   pdf_default_eps_reg default_eps_reg                 cie.py:42-50
 *   pdf_pixel_ls        pixel_least_squares             cie.py:66-80
 *   pdf_cie_fields      E = E_inc + G_D J, P, state     cie.py:92-114, losses.py:219-228
 *                       residual (cie_state_residual)
 *   pdf_masked_residual data residual                   losses.py:229-231
 *   pdf_regularizers    loss_bound/tv/bridge + grads,   losses.py:121-196
 *                       regularizer_chi_grad
 *   pdf_box_mean        box_mean                        filters.py:16-33
 *   pdf_guided_filter   guided_filter                   filters.py:36-53
 *   pdf_cco_image       apply_cco on any m1 x m2        filters.py:56-67
 *   pdf_get_error       PoleError / FloatingPointError  cie.py:27-29, losses.py:239-243,
 *                                                       network.py:221-222, 260-261
 *
 * Conventions: all array pointers are DEVICE pointers owned by the caller,
 * complex numbers are interleaved (re, im) in the context's real type
 * (complex128 for PDF_F64, complex64 for PDF_F32), arrays are C-contiguous
 * with the reference's shapes, `stream` is a cudaStream_t (NULL = legacy
 * default stream).  Every call is asynchronous on `stream` except
 * pdf_ctx_create (synchronous upload of constants) and pdf_get_error
 * (synchronises `stream`).  A context is not thread-safe; separate contexts
 * may run concurrently.  Return value 0 = success, < 0 = error, message via
 * pdf_last_error().
 */
#ifndef PDF_ABI_H
#define PDF_ABI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PDF_ABI_VERSION 1

enum pdf_dtype { PDF_F64 = 0, PDF_F32 = 1 };

/* sticky device error bits (per scene) */
enum pdf_error_bits {
  PDF_ERR_POLE = 1,             /* PoleError: |beta chi + 1| < 1e-14            */
  PDF_ERR_NONFINITE_STATE = 2,  /* FloatingPointError: nonfinite loss term(s)   */
  PDF_ERR_NONFINITE_DATA = 4,
  PDF_ERR_NONFINITE_BOUND = 8,
  PDF_ERR_NONFINITE_TV = 16,
  PDF_ERR_NONFINITE_BRIDGE = 32,
  PDF_ERR_NONFINITE_GRAD = 64,  /* FloatingPointError: nonfinite parameter grad */
  PDF_ERR_NONFINITE_PARAM = 128 /* FloatingPointError: nonfinite params after Adam */
};

enum pdf_status {
  PDF_OK = 0,
  PDF_EINVAL = -1,      /* bad argument / unsupported shape */
  PDF_ECUDA = -2,       /* CUDA runtime error */
  PDF_ENOMEM = -3,      /* workspace too small */
  PDF_ENOCONV = -4,     /* NoConvergenceError: an iterative solve stopped at maxiter */
  PDF_EGEOMETRY = -5    /* GeometryError: an antenna inside the grid / on a cell centre */
};

typedef struct pdf_ctx pdf_ctx;

typedef struct pdf_desc {
  int32_t abi_version;   /* PDF_ABI_VERSION */
  int32_t dtype;         /* enum pdf_dtype */
  int32_t S;             /* scenes sharing one geometry (batched reconstruction) */
  int32_t n;             /* incidences (views) */
  int32_t m1, m2;        /* grid; m1 == m2, power of two, 16..128 */
  int32_t R;             /* receivers */
  int32_t mf;            /* corner-block edge, m0 = 4 mf^2 */
  int32_t joint;         /* ImagingConfig.joint_views */
  int32_t freeze_r;      /* ImagingConfig.freeze_r (r_fixed must be given) */
  double beta, lambda1, lambda2, lambda3, tau_b;
  double lr, adam_b1, adam_b2, adam_eps;
  const void* e_inc;           /* [S or 1][n][m1][m2] complex */
  int64_t e_inc_scene_stride;  /* elements between scenes; 0 = shared */
  const void* gd_kernel_hat;   /* [2 m1][2 m2] complex, natural fft2 order */
  const void* gs_matrix;       /* [R][m1 m2] complex */
  const void* data;            /* [S][n][R] complex measured field */
  const void* mask;            /* [S][n][R] real, or NULL */
  const void* r_fixed;         /* [S][m1][m2] complex, or NULL */
  const double* c_inc;         /* HOST [S]: ||E_inc||^2   (losses.py:72) */
  const double* c_sca;         /* HOST [S]: ||mask d||^2  (losses.py:71) */
  int32_t k_iters_max;         /* reserved */
} pdf_desc;

const char* pdf_last_error(void);
int pdf_abi_version(void);

size_t pdf_workspace_bytes(const pdf_desc* desc);
int pdf_ctx_create(const pdf_desc* desc, void* workspace, size_t workspace_bytes, void* stream,
                   pdf_ctx** out);
int pdf_ctx_destroy(pdf_ctx* ctx);

/* network geometry: rows, d0 (= input/output width), hidden, n_params per scene */
int pdf_net_dims(const pdf_ctx* ctx, int32_t* rows, int32_t* d0, int32_t* hidden, int64_t* n_params);
/* kernel paths chosen at create (bits): PDF_PATH_LARGE_GRID, PDF_PATH_DATA_GEMM, PDF_PATH_SPLIT_BWD;
 * bits 8-11: CTAs per view of the cluster path (8 / 4: thread-block clusters, 1: one CTA per view) */
#define PDF_PATH_LARGE_GRID 1
#define PDF_PATH_DATA_GEMM 2
#define PDF_PATH_SPLIT_BWD 4
#define PDF_PATH_VIEW_CLUSTER_SHIFT 8
int pdf_ctx_paths(const pdf_ctx* ctx, int32_t* paths);

/* physics: alpha_hat [S][n][m0] -> g_alpha [S][n][m0] (NULL = skip), breakdown [S][6] f64
 * in LossBreakdown.as_row order (state, data, bound, tv, bridge, total) */
int pdf_loss_grad(pdf_ctx* ctx, const void* alpha_hat, void* g_alpha, double* breakdown, void* stream);
/* loss only; chi_out [S][m1][m2] (NULL = skip) is recover_contrast at alpha_hat */
int pdf_loss_value(pdf_ctx* ctx, const void* alpha_hat, double* breakdown, void* chi_out, void* stream);

/* network (parameters theta [S][n_params] in the reference flat order) */
int pdf_net_setup(pdf_ctx* ctx, const void* alpha0, void* stream);
int pdf_net_forward(pdf_ctx* ctx, const void* theta, void* alpha_hat, void* stream);
int pdf_grad_loss(pdf_ctx* ctx, const void* theta, void* grad, double* breakdown, void* stream);
int pdf_adam_step(pdf_ctx* ctx, void* theta, void* m, void* v, const void* grad, int64_t count, int32_t t,
                  void* stream);
/* replace the per-scene normalisers after the caller rewrote data / e_inc in place (new batch) */
int pdf_set_norms(pdf_ctx* ctx, const double* c_inc_host, const double* c_sca_host, void* stream);
/* k fused iterations {grad_loss -> trace row -> Adam} starting from Adam step t0;
 * trace [k][S][6] f64.  use_graph != 0 replays a captured CUDA graph. */
int pdf_train(pdf_ctx* ctx, void* theta, void* m, void* v, int32_t t0, int32_t k_iters, double* trace,
              int32_t use_graph, void* stream);

/* operator primitives over `count` images / row vectors */
int pdf_apply_gd(pdf_ctx* ctx, const void* x, void* y, int32_t count, int32_t adjoint, void* stream);
int pdf_gs_forward(pdf_ctx* ctx, const void* img, void* rows, int32_t count, void* stream);
int pdf_gs_adjoint(pdf_ctx* ctx, const void* rows, void* img, int32_t count, void* stream);
int pdf_expand(pdf_ctx* ctx, const void* alpha, void* img, int32_t count, void* stream);
int pdf_truncate(pdf_ctx* ctx, const void* img, void* alpha, int32_t count, void* stream);
int pdf_apply_cco(pdf_ctx* ctx, const void* chi, void* out, int32_t count, double tau, double eta_max,
                  double delta, int32_t radius, double eps_gf, void* stream);

/* measurement hooks: `iters` un-graphed fused iterations with an event between each of the
 * PDF_NPHASES kernels (fwd_l1 fwd_l2 fwd_l3 view_fwd pixel view_bwd finalize bwd_l3 bwd_l2 bwd_l1);
 * ms[PDF_NPHASES] = mean milliseconds per launch.  pdf_fp64_probe: DFMA-bound kernel, GFLOP/s. */
#define PDF_NPHASES 10
int pdf_profile_train(pdf_ctx* ctx, void* theta, void* m, void* v, int32_t t0, int32_t iters, float* ms,
                      void* stream);
int pdf_fp64_probe(double* gflops, void* stream);
/* timeline of the replayed training graph: pdf_timeline_reset(on = 1) makes the next captured
 * graph of pdf_train stamp slot = iteration * PDF_NPHASES + phase into its kernels and clears the
 * stamps (on = 0: off, recapture without; on = 2: clear the stamps only); after one replay pdf_timeline_read copies [PDF_TL_SLOTS][3] globaltimer ns (first CTA
 * entry, first CTA past the dependency wait, last CTA exit; unused: UINT64_MAX / 0) followed by
 * [PDF_TL_SLOTS][8] in-kernel stage stamps (last CTA reaching each stage; 0 = none). */
#define PDF_TL_SLOTS 128
int pdf_timeline_reset(pdf_ctx* ctx, int32_t on, void* stream);
int pdf_timeline_read(uint64_t* out_host, void* stream);

/* incidence sharding (one large scene, views split over ranks).
 * The context is created for this rank's views only (desc.n = own views, c_inc / c_sca
 * GLOBAL via pdf_set_norms).  One iteration =
 *   pdf_shard_step_a  -> all-reduce red1: SUM over [0, 3 m1 m2) per scene, MAX of the last entry
 *   pdf_shard_step_b  -> all-reduce red2: SUM
 *   pdf_shard_step_c  -> all-reduce grad: SUM, then pdf_adam_step on every rank
 * red1 / red2 are caller-owned float64 device buffers (sizes from pdf_shard_buffer_sizes);
 * the collective is the caller's (NCCL over NVLink via torch.distributed). */
int pdf_net_setup_sharded(pdf_ctx* ctx, const void* alpha0_all, int32_t n_all, int32_t view_offset, void* stream);
int pdf_shard_buffer_sizes(const pdf_ctx* ctx, int64_t* red1_doubles, int64_t* red2_doubles);
int pdf_shard_step_a(pdf_ctx* ctx, const void* theta, double* red1, void* stream);
int pdf_shard_step_b(pdf_ctx* ctx, const double* red1, double* red2, void* chi_out, void* stream);
int pdf_shard_step_c(pdf_ctx* ctx, const void* theta, const double* red2, void* grad, double* breakdown,
                     void* stream);
/* step c in per-layer parts (S = 1): layer 3 first (it also runs the pixel adjoint, G_D^H, truncation
 * and the loss breakdown), then 2, then 1; each writes its gradient bucket [W_L | b_L] (contiguous,
 * flat-order slice [offs[2L-2], offs[2L-1] + fan_out)) to `bucket`, so the caller can reduce a
 * layer's bucket while the next layer's backward runs.  pdf_net_offsets: offs[7] = w1, b1, w2, b2,
 * w3, b3 offsets in the flat parameter vector and n_params. */
int pdf_shard_step_c_part(pdf_ctx* ctx, const void* theta, const double* red2, void* bucket, int32_t layer,
                          double* breakdown, void* stream);
int pdf_net_offsets(const pdf_ctx* ctx, int64_t* offs);
/* Reduce-scatter fused into the backward (float64, S = 1): like pdf_shard_step_c_part, but every
 * g_W / g_b entry at flat parameter index f is stored, in the epilogue of the kernel that computes
 * it, to rank o = f / shard at slot [rank][f - o shard] of that rank's receive buffer peers[o]
 * (peers: DEVICE array of `world` pointers -- peer-mapped symmetric-memory addresses on a
 * multi-GPU node; shard even, world * shard >= n_params).  After a cross-rank barrier,
 * pdf_adam_gather on every rank sums its shard over the source ranks in rank order (recv =
 * this rank's receive buffer, [world][shard]), applies Adam (m, v: [shard], step t from device
 * memory) and writes the updated parameters into every rank's theta (thetas: DEVICE array of
 * `world` pointers): the all-gather as peer stores. */
int pdf_shard_step_c_scatter(pdf_ctx* ctx, const void* theta, const double* red2, double* const* peers,
                             int32_t world, int32_t rank, int64_t shard, int32_t layer, double* breakdown,
                             void* stream);
int pdf_adam_gather(pdf_ctx* ctx, const double* recv, double* const* thetas, double* m, double* v, int32_t world,
                    int32_t rank, int64_t shard, const int32_t* t_dev, void* stream);

/* tensor-parallel network for the incidence-sharded scene (SURVEY 8(e)'s alternative to the gradient
 * exchange; sharded.TensorParallelTrainer), float64, one scene per context.  Layer L on this rank
 * holds a slice of W_L ([N][K] row-major, out x in) in the caller's flat parameter vector `theta`:
 * W1 / W3 output rows (column-parallel), W2 input columns (row-parallel).  The context supplies the
 * row count (its views; a network context holds all views of the scene) and scratch.
 *   pdf_net_features   copies the context's network input x0 [rows][D0] and output gains cout [D0]
 *   pdf_net_layer_fwd  out[r][n] = f(sum_k in[r][k] W[n][k]), W = theta + w_off, b = theta + b_off:
 *                      mode 0 f = tanh(z + b), 2 f = z + b, 3 f = z (b unused)
 *   pdf_net_layer_bwd  grad[w_off + n K + k] = sum_r gz[r][n] hin[r][k]; grad[b_off + n] = sum_r gz[r][n];
 *                      gin[r][k] = (sum_n gz[r][n] W[n][k]) (1 - hin[r][k]^2) when gin is not NULL
 *   pdf_bias_tanh      x[r][n] = tanh(x[r][n] + bias[n]) in place (after the row-parallel all-reduce)
 *   pdf_shard_tp_a     step a of the sharded iteration with the network output read from the
 *                      column-block buffer Y[w][rows_all][N_w] (block w = output columns
 *                      [w blk, w blk + N_w), N_w = min(blk, D0 - w blk)); this context's views are rows
 *                      row0 .. row0 + n - 1 of the scene
 *   pdf_shard_tp_c     step c without the network: writes this context's rows of the gradient with
 *                      respect to the network output into the same block layout GY (other rows untouched) */
int pdf_net_features(const pdf_ctx* ctx, void* x0, void* cout, void* stream);
int pdf_net_layer_fwd(pdf_ctx* ctx, const void* in, int32_t K, int32_t N, const void* theta, int64_t w_off,
                      int64_t b_off, void* out, int32_t mode, void* stream);
int pdf_net_layer_bwd(pdf_ctx* ctx, const void* gz, const void* hin, int32_t K, int32_t N, const void* theta,
                      int64_t w_off, int64_t b_off, void* grad, void* gin, void* stream);
int pdf_bias_tanh(void* x, const void* bias, int64_t rows, int32_t n, void* stream);
int pdf_shard_tp_a(pdf_ctx* ctx, const void* Y, int32_t blk, int32_t rows_all, int32_t row0, double* red1,
                   void* stream);
int pdf_shard_tp_c(pdf_ctx* ctx, const double* red2, void* GY, int32_t blk, int32_t rows_all, int32_t row0,
                   double* breakdown, void* stream);
/* pdf_adam_step with the step t read from device memory (*t_dev, >= 1): capturable in a CUDA graph;
 * also flags a nonfinite gradient (network.py:221-222) */
int pdf_adam_step_dev(pdf_ctx* ctx, void* theta, void* m, void* v, const void* grad, int64_t count,
                      const int32_t* t_dev, void* stream);

/* one-time operator construction on the device (context-free, float64 / complex128, device arrays).
 *   pdf_bessel           j[k] = J_order(x[k]), y[k] = Y_order(x[k]) (order 0 or 1; either output may be
 *                        NULL); J even / odd in x, Y = NaN for x < 0, -inf at 0
 *   pdf_build_greens     gd_kernel [2 m1][2 m2] (wrap-indexed displacement kernel), gd_kernel_hat = its
 *                        unnormalised fft2, gs_matrix [R][m1 m2] (NULL = skip), *gd_diag_host (2 doubles,
 *                        may be NULL) = the self term; xs [m2] / ys [m1] cell-centre coordinates, rx [R][2]
 *                        receiver positions; m1, m2 powers of two <= 512; synchronises `stream`;
 *                        PDF_EGEOMETRY if a receiver lies inside the pixel grid
 *   pdf_incident_fields  out [n][m1][m2]: kind 0 = unit line sources (i/4) H0(k0 |r - src_v|) with
 *                        src [n][2] positions (PDF_EGEOMETRY if one coincides with a cell centre),
 *                        kind 1 = plane waves exp(i k0 (x cos src_v + y sin src_v)) with src [n] angles;
 *                        synchronises `stream` */
int pdf_bessel(int32_t order, const double* x, double* j, double* y, int64_t count, void* stream);
int pdf_build_greens(double k0, double cell_size, int32_t m1, int32_t m2, const double* xs, const double* ys,
                     const double* rx, int32_t R, void* gd_kernel, void* gd_kernel_hat, void* gs_matrix,
                     double* gd_diag_host, void* stream);
int pdf_incident_fields(int32_t kind, double k0, int32_t m1, int32_t m2, const double* xs, const double* ys,
                        const double* src, int32_t n, void* out, void* stream);

/* forward solve (method of moments): (I - G_D chi) x = b for the n views of
 * S scenes by batched BiCGStab with the reference's restart clause, on the context's G_D (the context
 * must be float64; its S / n / R are not used).  chi [S][m1][m2], b [S or 1][n][m1][m2] (b_scene_stride
 * elements between scenes, 0 = shared), x [S][n][m1][m2] output; workspace (device) of
 * pdf_solver_workspace_bytes(ctx, S * n) bytes.  residuals (device [S * n], may be NULL) receives
 * ||x - b - G_D(chi x)|| / ||b|| per view; *iters_out (host) the iterations run.  Synchronises
 * `stream` every few iterations.  Returns PDF_ENOCONV (message names the views above tol) when some
 * view has not converged at the check before iteration maxiter - 1, as the reference raises. */
size_t pdf_solver_workspace_bytes(const pdf_ctx* ctx, int32_t count_views);
int pdf_solve_total_field(pdf_ctx* ctx, const void* chi, const void* b, int64_t b_scene_stride, void* x, int32_t S,
                          int32_t n, double tol, int32_t maxiter, void* workspace, size_t workspace_bytes,
                          double* residuals, int32_t* iters_out, void* stream);

/* reconstruction metrics (reconstruct.py:243-254), context-free, float64 images.
 * Real parts are read with an element stride (1 = float64 image, 2 = interleaved complex128) and
 * `offset` is added to each (eps = chi + offset).  Results are DEVICE arrays of `count` entries.
 *   pdf_relative_error    out[k] = ||Re a_k - Re b_k||_F / ||Re b_k||_F   (relative_error)
 *   pdf_count_components  out[k] = 4-connected components of {Re a_k > threshold} (count_components,
 *                         scipy.ndimage.label with the 4-neighbour structure); labels = device
 *                         workspace of count * m1 * m2 int32 */
int pdf_relative_error(const double* eps_hat, const double* eps_true, int32_t stride, int64_t n_pix, int32_t count,
                       double offset, double* out, void* stream);
int pdf_count_components(const double* eps, int32_t stride, int32_t m1, int32_t m2, int32_t count, double offset,
                         double threshold, int32_t* labels, int32_t* out, void* stream);

/* contrast-integral-equation algebra, regularisers and filters (cie.py, losses.py:121-196,
 * filters.py:16-53), context-free, complex128 / float64 device arrays.  Elementwise maps use the
 * reference's float64 operation order (numpy's Smith division, no FMA contraction).
 *   pdf_chi_to_r        y = beta x / (beta x + 1) (inverse = 0) or x / (beta (1 - x)) (inverse = 1);
 *                       *poles (device int32) = pixels whose denominator is below 1e-14 in modulus
 *                       (the caller raises PoleError)
 *   pdf_default_eps_reg *eps (device) = 1e-10 max_v ||E_v||^2 / n_pix over e [n_views][n_pix]
 *   pdf_pixel_ls        per pixel: num = sum_v J_v conj(E_v), den = sum_v |E_v|^2 + *eps, chi = num / den,
 *                       degenerate = den <= 10 *eps (each output may be NULL)
 *   pdf_cie_fields      per view v: E = e_in[v * e_view_stride] (+ gdj[v] when not NULL), P = E + beta J,
 *                       res = r_hat P - beta J (r_hat [n_pix] shared); each output may be NULL
 *   pdf_masked_residual out = (a - b) * mask (mask float64, may be NULL)
 *   pdf_regularizers    values [count][3] = (bound, tv, bridge) sums; unweighted contrast gradients
 *                       g_bound / g_tv / g_bridge and g_total = l1 g_bound + l2 g_tv + l3 g_bridge
 *                       (terms with a zero weight skipped); every output may be NULL
 *   pdf_box_mean        (2r+1)^2 window means, edge-replicated, count images of m1 x m2 (radius >= 1)
 *   pdf_guided_filter   guided_filter(inp, guide, r, eps_gf) per image; scratch = 2 count m1 m2 doubles
 *   pdf_cco_image       apply_cco per complex image (self-guided filter of Re and Im, sigmoid gain);
 *                       scratch = 4 count m1 m2 doubles */
int pdf_chi_to_r(const void* x, void* y, int64_t n, double beta_re, double beta_im, int32_t inverse, int32_t* poles,
                 void* stream);
int pdf_default_eps_reg(const void* e, int32_t n_views, int64_t n_pix, double* eps, void* stream);
int pdf_pixel_ls(const void* j, const void* e, int32_t n_views, int64_t n_pix, const double* eps, void* num,
                 double* den, void* chi, uint8_t* degenerate, void* stream);
int pdf_cie_fields(const void* j, const void* gdj, const void* e_in, int64_t e_view_stride, const void* r_hat,
                   double beta_re, double beta_im, int32_t n_views, int64_t n_pix, void* e_out, void* p_out,
                   void* res_out, void* stream);
int pdf_masked_residual(const void* a, const void* b, const double* mask, void* out, int64_t n, void* stream);
int pdf_regularizers(const void* chi, int32_t m1, int32_t m2, int32_t count, double tau_b, double eps_tv, double l1,
                     double l2, double l3, double* values, void* g_bound, void* g_tv, void* g_bridge, void* g_total,
                     void* stream);
int pdf_box_mean(const double* img, double* out, int32_t m1, int32_t m2, int32_t radius, int32_t count, void* stream);
int pdf_guided_filter(const double* inp, const double* guide, double* out, int32_t m1, int32_t m2, int32_t radius,
                      double eps_gf, int32_t count, double* scratch, void* stream);
int pdf_cco_image(const void* chi, void* out, int32_t m1, int32_t m2, int32_t count, double tau, double eta_max,
                  double delta, int32_t radius, double eps_gf, double* scratch, void* stream);

/* copies the per-scene sticky error words to host (synchronises stream), then clears them */
int pdf_get_error(pdf_ctx* ctx, int32_t* err_host, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PDF_ABI_H */
