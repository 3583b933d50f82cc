/*
 * kernid_cuda.h -- C-ABI of libkernid_cuda.so, the B200 (sm_100a) implementation of the
 * far-field hot path of arXiv 1409.2802's reference (`kernid`, /root/reference/proj).
 *
 * The reference has no FFI layer: its hot path is the header-only C++ API in
 * proj/include/kernid/ headers. Each entry point below replaces the
 * device-side work of one reference function; the cited reference function is what a
 * maintainer would re-point at this ABI (bindings in INTEGRATION.md).
 *
 * Conventions (mirroring the reference):
 *   - matrices are column-major FP64 (Eigen default, kernel.hpp:14); indices int64
 *     (Eigen::Index, geometry.hpp:23-24);
 *   - no exceptions cross the boundary: every call returns a kid status code that maps
 *     1:1 onto the reference exception taxonomy (errors.hpp:11-77), message via
 *     kid_last_error();
 *   - buffers passed to the plain entry points are HOST memory (caller-allocated);
 *     the *_dev variants take device pointers, run asynchronously on the context stream
 *     and are what bench.py times and what the multi-GPU host layer all-reduces;
 *   - one context per device per host thread; a context is not re-entrant.
 *   - the Gaussian kernel K(y, x) = exp(-||x - y||^2 / (2 h^2)) (kernel.hpp:77-79) is the
 *     only family on this path (BASELINE.json north_star).
 */
#ifndef KERNID_CUDA_H
#define KERNID_CUDA_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> reference exceptions (errors.hpp) */
#define KID_OK 0
#define KID_E_RANGE 1        /* RangeError */
#define KID_E_DIM 2          /* DimensionError */
#define KID_E_NO_TARGETS 3   /* NoTargetsError (geometry.hpp:61-63) */
#define KID_E_NUMERICAL 4    /* NumericalError (lowrank.hpp:301-302) */
#define KID_E_ERROR 5        /* Error (base class) */
#define KID_E_CUDA 6         /* Error: CUDA runtime failure */
#define KID_E_OOM 7          /* Error: device allocation failed */
#define KID_E_ILLCOND 8      /* IllConditionedSkeletonError (lowrank.hpp:243-246) */
#define KID_E_CONFIG 9       /* ConfigError (kernel.hpp:29-36, h <= 0) */

/* kid_recon_error flags */
#define KID_RECON_DTD 1u     /* accumulate the residual Gram D^T D (spectral norm, compress.hpp:141-154) */
#define KID_RECON_KTK 2u     /* also form K^T K (matrix_norm, compress.hpp:156-159): a second Gram pass over the block */

typedef struct kid_ctx kid_ctx;

int kid_abi_version(void);
/* Page-locked host memory for the host-buffer entry points (optional; any host buffer works,
 * pinned ones avoid the driver's staging copy). */
void* kid_host_alloc(size_t bytes);
void kid_host_free(void* p);
/* Create a context on CUDA device `device` (one per process/GPU). */
int kid_create(kid_ctx** out, int32_t device);
void kid_destroy(kid_ctx* ctx);
const char* kid_last_error(const kid_ctx* ctx);
/* Run subsequent work on an external cudaStream_t (NULL: the context's own stream). */
int kid_set_stream(kid_ctx* ctx, void* cuda_stream);
int kid_synchronize(kid_ctx* ctx);
/* Kernel family of the Gram / leverage / projected passes. AUTO: the single-CTA fused kernels where the
   block fits one SM, the 2-CTA cluster kernel otherwise (m = 256 / 512). CLUSTER: always the cluster
   kernel (used by the tests to check both families on the same small blocks). Replaces no reference
   interface: the reference has one dense path (kernel.hpp:202-208). */
#define KID_PATH_AUTO 0
#define KID_PATH_CLUSTER 1
int kid_set_path(kid_ctx* ctx, int32_t path);
/* Name of the dominant kernel the last pass launched ("k_gram", "k_fused", "k_sumsq", ...): the
   bench labels its roofline line with the kernel that actually ran. */
const char* kid_last_kernel(const kid_ctx* ctx);
/* Tuning options of the cluster kernel (no effect on results): KID_OPT_EVAL_WARPS = 0 (auto), 8 or 12
   eval warps of 16 per CTA (the rest run the DMMA contractions). */
#define KID_OPT_EVAL_WARPS 1
#define KID_OPT_CHUNK_COLS 2 /* K_A chunk width: 0 (auto), 32, 48, 64, 96 */
#define KID_OPT_KERNEL 3     /* 0 auto, 1 the warp-specialised k_fused, 2 the warp-tile k_fused_w (n <= 32), 3 k_gram2 for K^T K at any m */
#define KID_OPT_TILE_WARPS 4 /* warps per CTA of k_fused_w: 0 auto (12 where shared memory allows), 8 */
#define KID_OPT_TILE_FORM 5  /* k_fused_w form: 0 auto (one CTA per SM where M and the sources fit it), 1 solo, 2 the CTA pair */
int kid_set_option(kid_ctx* ctx, int32_t key, int64_t value);
/* Plumbing for a multi-GPU host (kernid_b200::DeviceGroup): the context's device, its stream, device
   buffers on it and a synchronous read-back. */
int32_t kid_device_id(const kid_ctx* ctx);
void* kid_stream(kid_ctx* ctx);
void* kid_device_alloc(kid_ctx* ctx, size_t bytes);
void kid_device_free(kid_ctx* ctx, void* p);
int kid_memcpy_dtoh(kid_ctx* ctx, void* dst, const void* src, size_t bytes);

/* ---- point set (PointSet, kernel.hpp:14): N x d column-major ----
 * index_offset: global index of local row 0 when the point set is sharded across ranks. */
int kid_set_points(kid_ctx* ctx, const double* host_pts, int64_t N, int32_t d, int64_t index_offset);
/* Borrow an existing device buffer (no copy; must outlive its use). */
int kid_set_points_device(kid_ctx* ctx, const double* dev_pts, int64_t N, int32_t d, int64_t index_offset);

/* ---- pass 1: split_sources_targets (geometry.hpp:29-65) ----
 * Exact (dist, idx) selection of the n nearest points to `center`, rho, and the stable
 * compaction of targets {i not source : dist_i >= xi * rho} (ascending index). Distances are
 * computed bit-exactly as the reference (sequential sum of squared differences, no FMA,
 * correctly-rounded sqrt). Targets stay on the device; fetch them with kid_get_targets. */
int kid_split(kid_ctx* ctx, const double* center, int64_t n, double xi, int64_t* src_idx_out,
              double* rho_out, int64_t* n_targets_out);
/* Sharded split, step 1: the local n smallest (dist, global idx) keys, ascending. */
int kid_split_candidates(kid_ctx* ctx, const double* center, int64_t n, double* cand_dist,
                         int64_t* cand_idx);
/* Sharded split, step 2: given the global source set (ascending global indices) and rho,
 * compact the local targets. Also fixes the source coordinates used by the FP64 passes
 * (src_points: n x d column-major, host). */
int kid_split_finish(kid_ctx* ctx, const int64_t* src_idx, int64_t n, const double* src_points,
                     double rho, double xi, int64_t* n_targets_out);
int kid_get_targets(kid_ctx* ctx, int64_t* tgt_idx_out, int64_t count);
/* Explicit block K(T, S) (kernel_matrix(spec, targets, sources), kernel.hpp:202): targets
 * nt x d and sources m x d, both column-major host arrays. Replaces the split's block. */
int kid_set_block(kid_ctx* ctx, const double* targets, int64_t nt, const double* sources, int64_t m,
                  int32_t d);
int kid_block_shape(const kid_ctx* ctx, int64_t* nt, int64_t* m, int32_t* d);

/* ---- pass 2a: EuclideanNorm weights w_i = ||K_i||_2 (sampling.hpp:189-196) ---- */
int kid_row_norms(kid_ctx* ctx, double h, double* w_out);
int kid_row_norms_dev(kid_ctx* ctx, double h, double* d_w);

/* ---- pass 2b: Gram K^T K (m x m col-major) for the right factor / spectrum of K
 * (lowrank.hpp:56-90, replaced by the Gram route) and ||K||_F^2 ---- */
int kid_gram(kid_ctx* ctx, double h, double* G_out, double* sumsq_K_out);
int kid_gram_dev(kid_ctx* ctx, double h, double* d_G, double* d_sumsq);

/* ---- pass 2b': leverage scores l_i = ||K_i W||^2, W = V_r Sigma_r^-1 (m x r col-major),
 * lowrank.hpp:304-305 ---- */
int kid_leverage(kid_ctx* ctx, double h, const double* W, int64_t r, double* scores_out);
int kid_leverage_dev(kid_ctx* ctx, double h, const double* d_W, int64_t r, double* d_scores);

/* ---- pass 3: fused reconstruction-error pass (compress.hpp:141-159, 199-206) ----
 * D = K - K[:, skel] P (never materialised). Outputs ||D||_F^2, ||K||_F^2 and, per flags,
 * D^T D and K^T K (m x m col-major; rows/cols of skeleton columns of D^T D are exactly 0). */
int kid_recon_error(kid_ctx* ctx, double h, const int64_t* skel, int64_t r, const double* P,
                    uint32_t flags, double* sumsq_D, double* sumsq_K, double* DtD, double* KtK);
/* device variant (after kid_recon_prepare): d_out receives [sumsq_D, sumsq_K, D^T D restricted
 * to the m - r non-skeleton columns ((m-r) x (m-r) col-major, ascending original column)] */
int kid_recon_prepare(kid_ctx* ctx, const int64_t* skel, int64_t r, const double* P);
int kid_recon_error_dev(kid_ctx* ctx, double h, uint32_t flags, double* d_out);

/* ---- TSQR: the stable spectrum of the full K (lowrank.hpp:56-90 right_factor / singular_values
 * of K; harness.hpp:176-184 full_sv) ----
 * R (m x m col-major, upper triangular, m <= 128) with R^T R = K^T K by Householder TSQR over all
 * targets: the singular values / right singular vectors of R are those of K, including the ones
 * below sqrt(u) sigma_1 that the Gram route (kid_gram) cannot resolve. R is unique up to row
 * signs. kid_tsqr_combine folds `count` stacked factors (m x m each, host) into one (the
 * per-rank factors of a sharded block). */
int kid_tsqr_r(kid_ctx* ctx, double h, double* R);
int kid_tsqr_r_dev(kid_ctx* ctx, double h, double* d_R);
int kid_tsqr_combine(kid_ctx* ctx, const double* Rs, int64_t count, int64_t m, double* R);

/* ---- projected Gram: the compress_svd error pass (compress.hpp:243-262) ----
 * D = K C for an m x n coefficient matrix C (col-major, 1 <= n <= m), never materialised.
 * Outputs ||D||_F^2, ||K||_F^2 and D^T D (n x n col-major, nullable). With C = V_perp, an
 * orthonormal basis of the complement of V_r, ||K - K V_r V_r^T||_2 = sqrt(lambda_max(D^T D)).
 * The device variant takes d_C (device) and writes d_out = [||D||_F^2, ||K||_F^2, D^T D]. */
int kid_proj_gram(kid_ctx* ctx, double h, const double* C, int64_t n, double* sumsq_D, double* sumsq_K,
                  double* DtD);
int kid_proj_gram_dev(kid_ctx* ctx, double h, const double* d_C, int64_t n, double* d_out);

/* ---- gather_rows of K on the device (compress.hpp:130-137): Ks (count x m col-major) ---- */
int kid_eval_rows(kid_ctx* ctx, double h, const int64_t* rows, int64_t count, double* Ks_out);

/* ---- skeleton matvec (compress.hpp:309-325) ----
 * u_i = sum_j Ker(y_i, x_skel_j) (P q)_j over the block's targets y_i, x_skel_j = the block's
 * source skel[j]; P is r x m col-major (the ID projection), q the m charges; u_out n_targets.
 * The device variant takes q_skel = P q (r entries, host) and writes d_u (n_targets, device). */
int kid_apply_skeleton(kid_ctx* ctx, double h, const int64_t* skel, int64_t r, const double* P, const double* q,
                       double* u_out);
int kid_apply_skeleton_dev(kid_ctx* ctx, double h, const int64_t* skel, int64_t r, const double* q_skel,
                           double* d_u);

/* ---- row-subset view (mc_error, compress.hpp:279-305) ----
 * Restricts the block's targets to rows[0..n) of the full target list (row numbers as in K);
 * every pass above then runs on that subset. n < 0 (rows ignored) restores the full list;
 * kid_split / kid_set_block also reset it. */
int kid_select_rows(kid_ctx* ctx, const int64_t* rows, int64_t n);

/* ---- diagnostics: the FP64 passes' exp(x), x <= 0 (for accuracy checks against libm) ---- */
int kid_exp_check(kid_ctx* ctx, const double* x, int64_t n, double* y);

/* ---- diagnostics: canary check of a -DKID_GUARD build (64 KB guard zones around every device buffer of the
 * library): corrupted guard bytes, 0 = clean; -1 when the library was built without the guards ---- */
int64_t kid_guard_check(kid_ctx* ctx);

/* ---- instrumentation: number of kernels this context has launched ---- */
int64_t kid_launch_count(const kid_ctx* ctx);
/* Kernel timing: when enabled, each pass records a CUDA event pair on its stream around its
 * dominant kernel (k_dist_cand / k_compact, k_row_norms, k_gram, k_leverage); kid_profile_read
 * returns the per-launch durations in ms (oldest first) and resets the list. */
int kid_profile(kid_ctx* ctx, int32_t enable);
int kid_profile_read(kid_ctx* ctx, double* ms_each, int64_t cap, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif
