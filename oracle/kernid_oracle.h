/*
 * kernid_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference's far-field hot path
 * (/root/reference/proj/include/kernid/ headers). It is the CHECKER for the
 * CUDA product path, never part of it: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Pinning: the RNG streams (rng.hpp) are pinned bit-exactly against a binary
 * compiled from the reference's own rng.hpp (oracle/_ref, recipe in
 * oracle/Makefile; fixtures in tests/golden/). The rest is pinned against the
 * reference's known-answer tests (proj/tests/test_*.cpp), ported in
 * tests/test_oracle.py. The reference's Eigen-based QR/BDCSVD cannot be built
 * here (no Eigen), so singular values / V from this restatement
 * match real Eigen only to the relational tolerances of the reference tests.
 *
 * Arithmetic contract: compiled with -ffp-contract=off (proj/CMakeLists.txt:12-15),
 * sequential single-accumulator reductions as in kernel.hpp:60-68.
 * All matrices are column-major (Eigen default), indices int64.
 */
#ifndef KERNID_ORACLE_H
#define KERNID_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:19-78 ---- */
uint64_t or_splitmix64(uint64_t* state);
uint64_t or_derive_seed(uint64_t master, uint64_t key_a, uint64_t key_b);
typedef struct {
  uint64_t mt[312];
  int idx;
  int has_spare;
  double spare;
} or_rng;
void or_rng_init(or_rng* r, uint64_t seed);
uint64_t or_rng_next(or_rng* r);
double or_rng_uniform01(or_rng* r);
uint64_t or_rng_below(or_rng* r, uint64_t n);
double or_rng_normal(or_rng* r);
/* dump helpers for the RNG pin: n draws of each stream */
void or_rng_dump(uint64_t seed, int64_t n, uint64_t* u64, double* unif, double* normal,
                 uint64_t below_n, uint64_t* below);

/* ---- datagen.hpp:35-43 : N x d col-major, point-major draw order ---- */
int or_gen_normal(int32_t d, int64_t N, uint64_t seed, double* out);

/* ---- kernel.hpp:119-123 ---- */
double or_silverman_bandwidth(int32_t d, int64_t N);

/* ---- harness.hpp:95-100 (RandomPoint center): returns the row index ---- */
int64_t or_random_center_index(int64_t N, uint64_t data_seed);

/* ---- geometry.hpp:29-65 ----
 * returns 0 ok, 1 RangeError, 2 DimensionError (unused: d is shared), 3 NoTargetsError.
 * src_idx[n] ascending; tgt_idx must hold N entries; dist_out (nullable) N distances. */
int or_split(const double* pts, int64_t N, int32_t d, const double* center, int64_t n, double xi,
             int64_t* src_idx, int64_t* tgt_idx, int64_t* n_tgt, double* rho, double* dist_out);

/* gather rows of a col-major N x d point set: out (count x d col-major) */
void or_gather_points(const double* pts, int64_t N, int32_t d, const int64_t* idx, int64_t count,
                      double* out);

/* ---- kernel.hpp:60-79, 134-146, 164-172, 202-208 ----
 * K (nt x m, col-major) = exp(-sqdist / (2.0*h*h)), row-block threaded as parallel_for_rows. */
void or_kernel_matrix(const double* tgt, int64_t nt, const double* src, int64_t m, int32_t d,
                      double h, double* K, int32_t threads);
/* single entry (eval_kernel, kernel.hpp:94-115) */
double or_eval_gaussian(const double* x, const double* y, int32_t d, double h);

/* ---- sampling.hpp ---- */
int64_t or_sample_count(double s, int64_t m); /* -1 on RangeError */
/* rows norms of a col-major K: w_i = ||K_i||_2 sequential over j (sampling.hpp:189-196) */
void or_row_norms(const double* K, int64_t nt, int64_t m, double* w);
/* weighted_draw (sampling.hpp:108-149); returns 0 ok, 1 RangeError, 5 Error */
int or_weighted_draw(const double* w, int64_t n, int64_t count, int32_t replacement, or_rng* rng,
                     int64_t* out);
/* sample_rows for Uniform / EuclideanNorm / Leverage(with given scores) given weights;
 * kind 0 Uniform, 1 Bernoulli (random count, out holds m), 2 EuclideanNorm (weights = row norms),
 * 4 Leverage (weights = scores).
 * out must hold sample_count entries (or m for replacement). returns count or negative error. */
int64_t or_sample_rows(int32_t kind, int32_t replacement, int64_t m, const double* weights, double s,
                       uint64_t seed, int64_t* out);

/* ---- lowrank.hpp ---- */
/* Householder QR of a (rows x cols, rows >= cols) col-major matrix; R (cols x cols, col-major). */
void or_qr_r(const double* A, int64_t rows, int64_t cols, double* R);
/* One-sided Jacobi SVD of a square col-major n x n matrix: sv (desc), V (n x n col-major, nullable). */
void or_jacobi_svd(const double* A, int64_t n, double* sv, double* V);
/* singular_values (lowrank.hpp:70-77): sv has min(rows, cols) entries */
void or_singular_values(const double* A, int64_t rows, int64_t cols, double* sv);
/* right_factor (lowrank.hpp:81-90) for rows >= cols: sv (cols), V (cols x cols) */
void or_right_factor(const double* A, int64_t rows, int64_t cols, double* sv, double* V);
int64_t or_epsilon_rank(const double* sv, int64_t n, double eps, double ref_sigma1 /* <=0: sv[0] */);
/* row_leverage_scores (lowrank.hpp:296-308); returns 0, 1 RangeError, 4 NumericalError */
int or_row_leverage_scores(const double* A, int64_t rows, int64_t cols, int64_t r, double* scores,
                           int32_t* degenerate_gap);
/* interpolative_decomposition (lowrank.hpp:235-262): skel[r], P (r x n col-major).
 * returns 0, 1 RangeError, 8 IllConditionedSkeletonError */
int or_interpolative_decomposition(const double* A, int64_t m, int64_t n, int64_t r, int64_t* skel,
                                   double* P);
/* power_iteration_norm on an explicit matrix (lowrank.hpp:320-356) */
double or_power_iteration_norm(const double* A, int64_t rows, int64_t cols, double tol, int32_t cap);
/* spectral_norm_exact (lowrank.hpp:359) */
double or_spectral_norm_exact(const double* A, int64_t rows, int64_t cols);

/* ---- compress.hpp ---- */
/* reconstruction_error_norm (compress.hpp:141-154) with C = K[:, skel]; policy budget/tol/cap */
double or_reconstruction_error_norm(const double* K, int64_t nt, int64_t m, const int64_t* skel,
                                    int64_t r, const double* P, double budget, double tol, int32_t cap);
double or_matrix_norm(const double* K, int64_t nt, int64_t m, double budget, double tol, int32_t cap);
/* D = K - K[:,skel] P, Frobenius sums and the m x m Grams K^T K and D^T D (sequential over rows) */
void or_residual_stats(const double* K, int64_t nt, int64_t m, const int64_t* skel, int64_t r,
                       const double* P, double* sumsq_D, double* sumsq_K, double* DtD, double* KtK);
double or_bound_id_value(int64_t n, int64_t r, double sigma_r1);
double or_reconstruction_bound(int64_t m, int64_t s_count, double eps, double sigma_r1);

/* compress_id (compress.hpp:168-215). Inputs K (nt x m) and a row sample.
 * eps > 0: RankRule::from_eps(eps) (ref_sigma1 <= 0: none); else fixed_r.
 * k_norm <= 0: computed by matrix_norm. Outputs: rank, rel_error, skel (m), P (m*m),
 * sigma1_sample, sigma_r1_sample, bound_id. returns 0 or the error code. */
int or_compress_id(const double* K, int64_t nt, int64_t m, const int64_t* rows, int64_t nrows,
                   double eps, int64_t fixed_r, double ref_sigma1, double k_norm, double budget,
                   double tol, int32_t cap, int64_t* rank, double* rel_error, int64_t* skel,
                   double* P, double* sigma1_sample, double* sigma_r1_sample, double* bound_id);

/* apply_skeleton (compress.hpp:309-325): u (nt) */
void or_apply_skeleton(const double* tgt, int64_t nt, const double* skel_pts, int64_t r, int32_t d, double h,
                       const double* P, int64_t m, const double* q, double* u);
/* mc_error (compress.hpp:279-305) for khat_row(i) = K[i, skel] P; est (n_mc); 0, 1 RangeError, 5 Error */
int or_mc_error(const double* K, int64_t nt, int64_t m, const int64_t* skel, int64_t r, const double* P,
                double s_mc, int32_t n_mc, uint64_t seed, double budget, double tol, int32_t cap, double* est);
/* compress_svd numerator (compress.hpp:243-262): ||K V_r V_r^T - K|| */
double or_svd_error_norm(const double* K, int64_t nt, int64_t m, const double* Vr, int64_t r, double budget,
                         double tol, int32_t cap);

/* sym eigen (Jacobi, tests/oracles.hpp:19-66 style), evals desc, evecs col-major */
void or_jacobi_eigen(const double* A, int64_t n, double* evals, double* evecs);

#ifdef __cplusplus
}
#endif
#endif
