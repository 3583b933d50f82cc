// kid_internal.cuh -- shared device helpers and the context of libkernid_cuda.so.
//
// Layout in HBM:
//   points   N x d column-major FP64 (Eigen PointSet, kernel.hpp:14): coordinate k of
//            point i at pts[i + k*N]; every pass reads a coordinate column coalesced;
//   dist     N FP64, the bit-exact ||p_i - c|| of pass 1 (geometry.hpp:36-37);
//   tgt_idx  N_T int64 local indices of the targets, ascending (geometry.hpp:58-60);
//   sources  m x d column-major (gathered once per split); the FP64 passes stage them
//            in shared memory, permuted [skeleton | non-skeleton] for pass 3.
// K itself is never stored: every FP64 pass re-evaluates its target tile in registers
// / shared memory (SURVEY.md 8a A5 "never materialised on GPU").
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/kernid_cuda.h"

namespace kid {

// ---------------------------------------------------------------- device math

// Sequential squared distance with no FMA contraction (kernel.hpp:60-68): acc starts
// at 0.0, acc += (a_k - b_k)^2 in k order; __d*_rn keep nvcc from fusing.
__device__ __forceinline__ double sqdist_exact(const double* a, int64_t sa, const double* b,
                                               int64_t sb, int d) {
  double acc = 0.0;
  for (int k = 0; k < d; ++k) {
    const double diff = __dsub_rn(a[k * sa], b[k * sb]);
    acc = __dadd_rn(acc, __dmul_rn(diff, diff));
  }
  return acc;
}

// Gaussian entry exp(-sq / (2 h^2)) with the reference's argument rounding
// (kernel.hpp:77-79: -sq / (2.0*h*h), denom = (2.0*h)*h computed on the host).
__device__ __forceinline__ double gauss_exact(double sq, double denom) {
  return exp(__ddiv_rn(-sq, denom));
}

// exp(-q), q >= 0, for the Gaussian entries of the FP64 passes: table-driven and branch-free.
//   -q = (64k + j) ln2/64 + r,  |r| <= ln2/128,  e^r - 1 by a degree-5 Taylor polynomial
//   (truncation r^6/720 < 4e-17), exp(-q) = 2^k (T[j] + T[j] (e^r - 1)); the 2^k is applied as
//   2^(k+600) on the exponent field and one multiply by 2^-600 (exact for normal results,
//   correctly rounded into the subnormal range; k is clamped where the result rounds to 0).
// T[j] = 2^(j/64) (correctly rounded, c_exp2_tab) is staged in shared memory REPLICATED per lane,
// [j][lane] (kExpTab x 32 doubles = 16 KB): a lane reads tabl[j * 32] with tabl = tab + lane, so
// the 32 random lookups of a warp never share a bank pair (2 wavefronts, the minimum for a
// 64-bit load; an unreplicated table costs ~5 for random indices) -- shared-memory bandwidth,
// not the FP64 pipe, bounds the fused pass (profiles/).
// 12 FP64-pipe ops; max error 1 ulp against glibc (tests/test_gpu_parity.py::test_fast_exp_accuracy).
// q >= 0 of any size: q is clamped to <= 2^17 on its high word (one integer min; exp(-2^17) == 0
// in double anyway), which keeps the rounded multiple of ln2/64 inside int32.
constexpr int kExpTab = 64;
constexpr int kExpRep = 32;  // replicas (one per lane)
constexpr int kExpTabWords = kExpTab * kExpRep;
__device__ __forceinline__ double exp_neg_fast(double q, const double* __restrict__ tabl) {
  const double shifter = 6755399441055744.0;  // 1.5 * 2^52: round-to-nearest-integer
  q = __hiloint2double(min(__double2hiint(q), 0x41000000), __double2loint(q));  // q <= ~2^17
  double kd = fma(q, -92.33248261689366, shifter);  // round(-q * 64 / ln2)
  const int n = __double2loint(kd);
  const double t = tabl[(n & (kExpTab - 1)) * kExpRep];
  kd -= shifter;
  double r = fma(kd, -0.010830424667801708, -q);  // Cody-Waite: ln2/64 = hi (28 bits) + lo
  r = fma(kd, -2.8447437476627285e-11, r);
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p *= r;  // e^r - 1
  const double y = fma(t, p, t);
  const int k = max(n >> 6, -1100);  // floor(n / 64), clamped: 2^(k+600) stays normal
  return __hiloint2double(__double2hiint(y) + ((k + 600) << 20), __double2loint(y)) * 0x1p-600;
}

// exp_neg_fast on N independent arguments, written step-major (each step of the evaluation is
// applied to all N before the next) so the N dependency chains stay interleaved in the SASS --
// ptxas otherwise tends to serialise them under a tight register budget. Same arithmetic, same
// results as N calls of exp_neg_fast.
// REP: table replicas (row stride of the [j][replica] table): 32 (one per lane), or 16 -- a 64-bit
// shared load is served per half-warp, so lanes l and l + 16 may share a replica conflict-free.
template <int N, int REP = kExpRep>
__device__ __forceinline__ void exp_neg_fast_n(double (&q)[N], const double* __restrict__ tabl) {
  const double shifter = 6755399441055744.0;
  double kd[N], r[N], p[N], t[N];
  int n[N];
#pragma unroll
  for (int u = 0; u < N; ++u) q[u] = __hiloint2double(min(__double2hiint(q[u]), 0x41000000), __double2loint(q[u]));
#pragma unroll
  for (int u = 0; u < N; ++u) kd[u] = fma(q[u], -92.33248261689366, shifter);
#pragma unroll
  for (int u = 0; u < N; ++u) {
    n[u] = __double2loint(kd[u]);
    t[u] = tabl[(n[u] & (kExpTab - 1)) * REP];
  }
#pragma unroll
  for (int u = 0; u < N; ++u) kd[u] -= shifter;
#pragma unroll
  for (int u = 0; u < N; ++u) r[u] = fma(kd[u], -0.010830424667801708, -q[u]);
#pragma unroll
  for (int u = 0; u < N; ++u) r[u] = fma(kd[u], -2.8447437476627285e-11, r[u]);
#pragma unroll
  for (int u = 0; u < N; ++u) p[u] = fma(r[u], 1.0 / 120.0, 1.0 / 24.0);
#pragma unroll
  for (int u = 0; u < N; ++u) p[u] = fma(p[u], r[u], 1.0 / 6.0);
#pragma unroll
  for (int u = 0; u < N; ++u) p[u] = fma(p[u], r[u], 0.5);
#pragma unroll
  for (int u = 0; u < N; ++u) p[u] = fma(p[u], r[u], 1.0);
#pragma unroll
  for (int u = 0; u < N; ++u) p[u] *= r[u];
#pragma unroll
  for (int u = 0; u < N; ++u) {
    const double y = fma(t[u], p[u], t[u]);
    const int k = max(n[u] >> 6, -1100);
    q[u] = __hiloint2double(__double2hiint(y) + ((k + 600) << 20), __double2loint(y)) * 0x1p-600;
  }
}

// exp(x), x <= 0 (diagnostics and callers holding the argument)
__device__ __forceinline__ double exp_fast(double x, const double* __restrict__ tabl) {
  return exp_neg_fast(-x, tabl);
}

// FP64 tensor-core MMA (SASS DMMA.8x8x4): C[8x8] += A[8x4] * B[4x8].
// Fragments: A[row = lane>>2][k = lane&3], B[k = lane&3][col = lane>>2],
// C[row = lane>>2][col = 2*(lane&3) + {0,1}].
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace kid

// ---------------------------------------------------------------- context
struct kid_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;

  // point set
  const double* pts = nullptr;  // device, N x d col-major (owned or borrowed)
  double* pts_own = nullptr;
  size_t pts_own_cap = 0;
  int64_t N = 0;
  int32_t d = 0;
  int64_t offset = 0;

  // split state
  double* dist = nullptr;
  size_t dist_cap = 0;
  unsigned char* flag = nullptr;  // pass 1 fast path: 1 = surely a target, 0 = near (exact dist kept)
  size_t flag_cap = 0;
  int64_t* tgt_idx = nullptr;
  size_t tgt_cap = 0;
  int64_t n_split_targets = 0;

  // current block K(T, S)
  const double* tbase = nullptr;  // target coordinate base (points or explicit targets)
  int64_t tld = 0;                // leading dimension of tbase
  const int64_t* tidx = nullptr;  // nullptr: identity
  int64_t nt = 0;
  double* blk_tgt = nullptr;  // owned explicit targets
  size_t blk_tgt_cap = 0;
  double* src = nullptr;  // m x d col-major
  size_t src_cap = 0;
  int64_t m = 0;

  // pass-3 operands (kid_recon_prepare)
  int64_t r = 0;
  double* src_perm = nullptr;  // m x d, columns [skel | non-skel]
  size_t src_perm_cap = 0;
  // row-subset view (kid_select_rows): the block's targets restricted to rows of the full list
  bool sub_active = false;
  int64_t full_nt = 0;
  const int64_t* full_tidx = nullptr;
  int64_t* sub_idx = nullptr;  // composed indices, then the uploaded row list
  size_t sub_cap = 0;
  std::vector<double> src_host;       // host copies (m x d col-major) of src / src_perm: the fused
  std::vector<double> src_perm_host;  // pass carries them in its kernel parameters
  double* P2 = nullptr;        // r x meff row-major, stride = r-major padded
  std::vector<double> P2_host;  // host copy of P2 (the large-m fused pass builds its per-CTA images from it)
  size_t P2_cap = 0;
  std::vector<int64_t> nonskel;  // host: original column of each non-skeleton column
  std::vector<int64_t> skel_h;

  // scratch
  void* scratch = nullptr;
  size_t scratch_cap = 0;
  double* partial = nullptr;
  size_t partial_cap = 0;
  double* hbuf = nullptr;  // pinned host staging
  size_t hbuf_cap = 0;
  int64_t* counter = nullptr;  // device counters [8]
  int path = KID_PATH_AUTO;
  int eval_warps = 0;
  int chunk_cols = 0;
  int tile_warps = 0;     // kid_set_option(KID_OPT_TILE_WARPS): warps per CTA of the warp-tile kernel (0 auto, 8, 12)
  int tile_form = 0;      // kid_set_option(KID_OPT_TILE_FORM): warp-tile kernel form (0 auto, 1 solo, 2 cluster)
  int kernel_choice = 0;  // kid_set_option(KID_OPT_KERNEL): 0 auto, 1 k_fused, 2 k_fused_w where it applies  // kid_set_option(KID_OPT_CHUNK_COLS): K_A chunk width of the cluster kernel (0 auto)  // kid_set_option(KID_OPT_EVAL_WARPS): eval warps of the cluster kernel (0 auto, 8, 12)
  const char* last_kernel = "";  // dominant kernel of the last pass (kid_last_kernel)  // kid_set_path: which kernel family serves the Gram / leverage passes
  void* sort_tmp = nullptr;       // CUB radix-sort temporary storage (pass 1)
  size_t sort_tmp_cap = 0;

  // kernel timing (kid_profile): CUDA events on the launching stream around each pass'
  // dominant kernel, read back by kid_profile_read
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;  // pairs
  size_t prof_used = 0;
};

namespace kid {

int fail(kid_ctx* c, int code, const std::string& msg);
int cuda_fail(kid_ctx* c, cudaError_t e, const char* where);
int ensure(kid_ctx* c, void** p, size_t* cap, size_t bytes);
int ensure_pinned(kid_ctx* c, size_t bytes);
void* scratch(kid_ctx* c, size_t bytes);

#define KID_CK(ctx, call)                                       \
  do {                                                          \
    cudaError_t e_ = (call);                                    \
    if (e_ != cudaSuccess) return ::kid::cuda_fail(ctx, e_, #call); \
  } while (0)
#define KID_LAUNCHED(ctx)                                              \
  do {                                                                 \
    (ctx)->launches++;                                                 \
    cudaError_t e_ = cudaGetLastError();                               \
    if (e_ != cudaSuccess) return ::kid::cuda_fail(ctx, e_, "launch"); \
  } while (0)

// pass entry points (kid_split.cu / kid_passes.cu)
int split_candidates(kid_ctx* c, const double* center_h, int64_t n, double* cand_dist_h,
                     int64_t* cand_idx_h);
int split_finish(kid_ctx* c, const int64_t* src_idx_h, int64_t n, const double* src_pts_h, double rho,
                 double xi, int64_t* n_targets_out);
int split_device(kid_ctx* c, const double* center_h, int64_t n, double xi, int64_t* src_idx_out, double* rho_out,
                 int64_t* n_targets_out);
int row_norms_dev(kid_ctx* c, double h, double* d_w);
int gram_dev(kid_ctx* c, double h, int64_t r, double* d_out);
int leverage_dev(kid_ctx* c, double h, const double* d_W, int64_t r, double* d_scores);
int tsqr_dev(kid_ctx* c, double h, const double* d_Rin, int64_t nR, int64_t m, double* d_R);
int proj_gram_dev(kid_ctx* c, double h, const double* d_C, int64_t n, double* d_out);
// launch wrapper shared with kid_next.cu (no relocatable device code)
int launch_gram_reduce(kid_ctx* c, const double* partial, int nchunks, int LG, int n, const double* partial_sk,
                       int nparts, double* out);
int eval_rows_dev(kid_ctx* c, double h, const int64_t* d_rows, int64_t count, double* d_Ks);
int apply_skeleton_dev(kid_ctx* c, double h, const int64_t* skel, int64_t r, const double* q_skel, double* d_u);
int select_rows(kid_ctx* c, const int64_t* rows, int64_t n);
int exp_check_dev(kid_ctx* c, const double* d_x, int64_t n, double* d_y);
// large-m fused passes on a 2-CTA cluster (kid_fused.cu): D = K_B + K_A M, then D^T D or row sums of D^2
enum : int { FX_RESID = 0, FX_GRAM = 1, FX_PROJ = 2, FX_LEV = 3 };
int fused_dev(kid_ctx* c, double h, int mode, const double* M_host, int64_t n, double* d_out);
// event pair bracketing the dominant kernel of a pass (no-op unless profiling)
void prof_begin(kid_ctx* c);
void prof_end(kid_ctx* c);

}  // namespace kid
