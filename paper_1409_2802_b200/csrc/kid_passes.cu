// kid_passes.cu -- the FP64 passes over all N_T targets of K(T, S).
//
// Every pass re-evaluates its target tile of K in registers / shared memory and never
// stores K in HBM (the reference materialises it, kernel.hpp:202-208):
//   k_row_norms   w_i = ||K_i||_2                       sampling.hpp:189-196
//   k_gram        G += T^T T per 32-target tile on DMMA   lowrank.hpp:56-90 (Gram route)
//                 mode K: T = K            -> K^T K, ||K||_F^2
//                 mode D: T = K_N - K_S P2  -> D^T D, ||D||_F^2 = tr(D^T D)
//                         (compress.hpp:141-159: D = K - K[:,skel] P; the skeleton
//                          columns of D are exactly zero because P[:, skel] = I)
//   k_proj_gram   LEV mode: l_i = ||K_i W||^2              lowrank.hpp:304-305
//   k_eval_rows   K[rows, :] gathered                     compress.hpp:130-137
// The m x m accumulators live in registers (DMMA C fragments) across all tiles of a
// CTA's contiguous target chunk; partials are reduced in a fixed chunk order so results
// are bitwise reproducible run to run.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cublas_v2.h>

#include "kid_internal.cuh"

namespace kid {

__device__ double c_exp2_tab[kExpTab];  // 2^(j/64); each CTA stages it in shared memory, replicated per lane

// shared table [j][lane] (kExpTabWords doubles) for exp_neg_fast(q, tab + lane)
__device__ __forceinline__ void stage_exp_table(double* tabr, int tid, int nthr) {
  for (int e = tid; e < kExpTabWords; e += nthr) tabr[e] = c_exp2_tab[e / kExpRep];
}

int init_device_tables() {
  static thread_local int done_dev = -1;
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) return KID_E_CUDA;
  if (done_dev == dev) return KID_OK;
  double tab[kExpTab];
  for (int j = 0; j < kExpTab; ++j) tab[j] = (double)exp2l((long double)j / (long double)kExpTab);
  if (cudaMemcpyToSymbol(c_exp2_tab, tab, sizeof(tab)) != cudaSuccess) return KID_E_CUDA;
  done_dev = dev;
  return KID_OK;
}

namespace {

constexpr int kTM = 32;        // targets per tile (SYRK k-depth: 8 DMMA k-steps)
constexpr int kNT = 256;       // threads per CTA
constexpr int kNW = kNT / 32;  // warps per CTA

struct TargetView {
  const double* base;
  int64_t ld;
  const int64_t* idx;
  int64_t nt;
};

__device__ __forceinline__ double tcoord(const TargetView& tv, int64_t i, int k) {
  const int64_t row = tv.idx ? tv.idx[i] : i;
  return tv.base[row + k * tv.ld];
}

__host__ __device__ constexpr int ceil_to(int x, int a) { return (x + a - 1) / a * a; }
// row stride (in doubles) of a shared-memory tile: = 4 or 12 (mod 16), which makes the
// DMMA fragment gathers [(lane&3)*S + (lane>>2)] and [(lane>>2)*S + (lane&3)] conflict-free.
__host__ __device__ constexpr int frag_stride(int cols) { return ceil_to(cols, 8) + 4; }

// ------------------------------------------------------------------ row norms
template <int D>
__global__ void __launch_bounds__(256) k_row_norms(TargetView tv, int d_rt, const double* __restrict__ src,
                                                   int64_t m, double negc, double* __restrict__ w) {
  const int d = D ? D : d_rt;
  extern __shared__ double s_src[];  // d x m, s_src[j + k*m]
  __shared__ double s_tab[kExpTabWords];
  stage_exp_table(s_tab, threadIdx.x, blockDim.x);
  for (int64_t e = threadIdx.x; e < m * d; e += blockDim.x) s_src[e] = src[e];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tv.nt; i += (int64_t)gridDim.x * blockDim.x) {
    double t[D ? D : 1];
    if (D) {
#pragma unroll
      for (int k = 0; k < (D ? D : 1); ++k) t[k] = tcoord(tv, i, k);
    }
    double acc = 0.0;
    for (int64_t j = 0; j < m; ++j) {
      double sq = 0.0;
      if (D) {
#pragma unroll
        for (int k = 0; k < (D ? D : 1); ++k) {
          const double diff = __dsub_rn(t[k], s_src[j + k * m]);
          sq = __dadd_rn(sq, __dmul_rn(diff, diff));
        }
      } else {
        for (int k = 0; k < d; ++k) {
          const double diff = __dsub_rn(tcoord(tv, i, k), s_src[j + k * m]);
          sq = __dadd_rn(sq, __dmul_rn(diff, diff));
        }
      }
      const double kv = exp_fast(sq * negc, s_tab + (threadIdx.x & 31));
      acc = __dadd_rn(acc, __dmul_rn(kv, kv));  // sequential over j (sampling.hpp:193)
    }
    w[i] = __dsqrt_rn(acc);
  }
}

// ------------------------------------------------------------------ Gram / residual Gram
constexpr int kCSrc = 2048;  // doubles of source coordinates carried in GramArgs (16 KB)
struct GramArgs {
  TargetView tv;
  int d;
  const double* src;   // m x d col-major, columns already in [skel | non-skel] order
  int m, r, meff;      // meff = m - r
  double cscale;       // 1 / (sqrt(2) h): coordinates pre-scaled so that K = exp(-||x' - y'||^2)
  const double* P2;    // r x SP row-major, SP = frag_stride(meff) (device); nullptr when r == 0
  const int2* blist;   // [nparts][kMW][TPW] (a0, b0) first 8x8 block of each WA x 2-block warp tile, x = -1: empty
  const short* elist;  // [kEW][kEItems]: nA, nB, A items (skeleton columns), B items (4-column groups)
  int nparts;
  int64_t ntiles;
  int nchunks;
  double* partial;     // [nchunks][LG][LG]
  int LG;              // padded Gram leading dimension = ceil8(meff)
  double* partial_sk;  // [nchunks] sum K^2 (part 0), then [nparts][nchunks] partial traces of D^T D
  int dbg;             // profiling aid (KID_GRAM_DEBUG): 1 skip eval math, 2 skip the K_S P2 FMAs, 4 skip SYRK,
                       // 16 no coordinate copies (ring slots keep tile 0's targets)
  long long* trace;    // profiling aid (KID_GRAM_TRACE): [warp][tile][4] clock64 stamps of CTA 0
  // scaled source coordinates in the kernel-parameter (constant) bank: the eval warps read them
  // at warp-uniform indices, so they cost constant-cache broadcasts instead of shared-memory
  // wavefronts. [d][rS] skeleton columns, then [d][mN] non-skeleton columns (padding: far away)
  double csrc[kCSrc];
};
constexpr int kTraceTiles = 64;

// Warp-specialized pipeline (one CTA per SM), per 32-target tile:
//   warps 0..11 (kEW "eval" warps) own a host-balanced list of work items:
//     A item j      : K_S column j of the NEXT tile (exp) -> KS ring (2 slots, eval-private)
//     B item g      : non-skeleton columns 4g..4g+3 of THIS tile: K_N by exp (4 independent
//                     chains), then D = K_N - K_S P2 by DFMA against the K_S row of the target
//                     (KS ring) and -P2 rows (shared memory, LDS.128 broadcasts) -> KN stage
//     lane = target row throughout, so stores are conflict-free column-major [col][t] (stride
//     kST = 36 = 4 mod 16, which also makes the DMMA fragment gathers conflict-free);
//   warps 12..19 (kMW "MMA" warps): G += D^T D (DMMA.8x8x4) on static WA x 2-block warp tiles of
//     the upper triangle, accumulators register-resident across the CTA's whole target chunk.
// Hand-off by named barriers: FULL[s] (eval arrive, MMA sync), EMPTY[s] (MMA arrive, eval sync),
// EVAL (eval warps only: K_S of the next tile and the next coordinates are visible).
// Target coordinates stream through a 4-slot shared-memory ring by cp.async, issued three tiles
// ahead (the target index of the copy is itself loaded one tile earlier).
// DMMA and DFMA share the FP64 datapath (tools/fp64_overlap.cu): the split keeps it fed from
// both sides -- the MMA warps never wait on a GEMM phase, the eval warps fill the DMMA gaps.
constexpr int kMW = 8, kEW = 12, kGT = (kMW + kEW) * 32;  // 640 threads
constexpr int kEvalW0 = kMW, kMmaW0 = 0;
constexpr int kStages = 4;
constexpr int kST = kTM + 4;  // column-major tile stride
constexpr int kRing = 4;      // target-coordinate ring slots
constexpr int kEItems = 48;   // per eval warp: 2 counts + items
constexpr int kBarFull = 1, kBarEmpty = 1 + kStages, kBarEval = 1 + 2 * kStages;

__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// clock64 after a deferred-blocking BAR.SYNC reads the issue time; the shared-memory load and
// the dependent branch below force the stamp to be taken after the barrier has released.
#define KID_TRACE(ev)                                                                              \
  do {                                                                                             \
    if (A.trace && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0 && it < kTraceTiles) {          \
      const double probe_ = *(volatile double*)&s_tab[1];                                          \
      long long t_ = 0;                                                                            \
      if (probe_ == probe_) t_ = clock64();                                                        \
      A.trace[((size_t)warp * kTraceTiles + it) * 4 + (ev)] = t_;                                  \
    }                                                                                              \
  } while (0)

// register split: 640 threads launch with 96 registers each; setmaxnreg.inc can only take what
// the decreasing warps release: 384 (96 - E) >= 256 (M - 96)
constexpr int kEvalRegs = 72, kMmaRegs = 128;
static_assert(kGT == 640, "setmaxnreg budget below assumes 640 threads (96 registers each at launch)");
static_assert(kEW * 32 * (96 - kEvalRegs) >= kMW * 32 * (kMmaRegs - 96), "setmaxnreg.inc exceeds what .dec releases");

// SYRK over one stage for the first N warp tiles: fragments F(x) = D[k0 + fk][x*8 + fr]
// (A and B operands of D^T D use the same gather), double-buffered across the 8 k-steps.
template <int N, int TPW, int WA>
__device__ __forceinline__ void syrk_stage(double (&acc)[TPW][WA][2][2], const int (&fa0)[TPW], const int (&fb0)[TPW],
                                           const double* __restrict__ col) {
  double fa[2][N][WA], fb[2][N][2];
  auto load = [&](int buf, int k0) {
#pragma unroll
    for (int q = 0; q < N; ++q) {
#pragma unroll
      for (int u = 0; u < WA; ++u) fa[buf][q][u] = col[fa0[q] + u * 8 * kST + k0];
#pragma unroll
      for (int v = 0; v < 2; ++v) fb[buf][q][v] = col[fb0[q] + v * 8 * kST + k0];
    }
  };
  load(0, 0);
#pragma unroll
  for (int kk = 0; kk < kTM / 4; ++kk) {
    if (kk + 1 < kTM / 4) load((kk + 1) & 1, (kk + 1) * 4);
#pragma unroll
    for (int q = 0; q < N; ++q)
#pragma unroll
      for (int u = 0; u < WA; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) dmma884(acc[q][u][v][0], acc[q][u][v][1], fa[kk & 1][q][u], fb[kk & 1][q][v]);
  }
}

template <int D, int TPW, int WA>
__global__ void __launch_bounds__(kGT, 1) k_gram(const __grid_constant__ GramArgs A) {
  const int d = D ? D : A.d;
  const int m = A.m, r = A.r, meff = A.meff;
  const int NBN = ceil_to(meff, 8) / 8;
  const int r4 = ceil_to(r, 4);
  const int rS = r4, mN = NBN * 8;
  const int SPn = frag_stride(meff);  // -P2 row stride (= 4 or 12 mod 16: conflict-free B fragments)
  const int TS = (r4 > 0 ? r4 : 4) * kST, TN = ceil_to(NBN + 1, 2) * 8 * kST;  // one KS slot / one KN stage
  extern __shared__ __align__(16) double smem[];
  const double* s_srcS = A.csrc;                   // d x rS: skeleton sources, [k][j] (constant bank); pad: far away
  const double* s_srcN = A.csrc + (size_t)d * rS;  // d x mN: non-skeleton sources, [k][j]; pad: far away
  double* sP = smem;                             // r4 x SPn: -P2, row-major (pad rows / columns 0)
  double* KSb = sP + (size_t)r4 * SPn;           // 2 x (r4 x kST): K_S, column-major [k][t]; rows >= r are 0
  double* KNb = KSb + 2 * (size_t)TS;            // kStages x (.. x kST): D, column-major [col][t]
  double* ring = KNb + (size_t)kStages * TN;     // kRing x d x 32 target coordinates (unscaled)
  __shared__ double red[kEW], red_tr[kMW];
  __shared__ double s_tab[kExpTabWords];
  __shared__ short s_el[kEW * kEItems];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int chunk = blockIdx.x, part = blockIdx.y;
  stage_exp_table(s_tab, tid, kGT);
  for (int e = tid; e < kEW * kEItems; e += kGT) s_el[e] = A.elist[e];
  const int SP = frag_stride(meff);
  for (int e = tid; e < r4 * SPn; e += kGT) {
    const int k = e / SPn, n = e % SPn;
    sP[e] = (k < r && n < meff) ? -A.P2[(size_t)k * SP + n] : 0.0;
  }
  for (int e = tid; e < 2 * TS; e += kGT) KSb[e] = 0.0;
  for (int e = tid; e < kStages * TN; e += kGT) KNb[e] = 0.0;
  for (int e = tid; e < kRing * d * kTM; e += kGT) ring[e] = 0.0;
  const int64_t tile_lo = A.ntiles * chunk / A.nchunks, tile_hi = A.ntiles * (chunk + 1) / A.nchunks;
  const int ntile = (int)(tile_hi - tile_lo);
  __syncthreads();

  if (warp >= kEvalW0 && warp < kEvalW0 + kEW) {
    // ================================================================ eval warps
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kEvalRegs) : "memory");
    const int ew = warp - kEvalW0;
    const short* el = s_el + ew * kEItems;
    const int nA = el[0], nB = el[1];
    const short* itA = el + 2;
    const short* itB = el + 2 + nA;
    double sk = 0.0;
    const bool copier = ew < d && !(A.dbg & 16);  // warp ew copies coordinate dims ew, ew + kEW, ...
    const int64_t nt = A.tv.nt;
    auto trow = [&](int tl) -> int64_t {  // target row of lane in local tile tl, -1 past the end
      const int64_t i = (tile_lo + tl) * kTM + lane;
      return (tl < ntile && i < nt) ? i : -1;
    };
    auto row_of = [&](int tl) -> int64_t {
      const int64_t i = trow(tl);
      return i < 0 ? -1 : (A.tv.idx ? A.tv.idx[i] : i);
    };
    auto issue_copy = [&](int tl, int64_t prow) {  // prow: A.tv row of lane's target (or -1)
      if (prow >= 0) {
        double* slot = ring + (size_t)(tl % kRing) * d * kTM;
        for (int k = ew; k < d; k += kEW) cp_async8(slot + k * kTM + lane, A.tv.base + prow + (int64_t)k * A.tv.ld);
      }
      cp_async_commit();
    };
    // prologue: coordinates of tiles 0, 1 (visible after the barrier), 2 (in flight); the row of
    // tile 3 is loaded ahead into a register
    int64_t next_row = -1;
    if (copier) {
      issue_copy(0, row_of(0));
      issue_copy(1, row_of(1));
      cp_async_wait<0>();
      issue_copy(2, row_of(2));
      next_row = row_of(3);
    }
    nbar_sync(kBarEval, kEW * 32);

    constexpr int DR = (D > 0 && D <= 8) ? D : 1;  // coordinates held in registers per phase
    double tc[DR];
    auto load_coords = [&](int tl) {
      if constexpr (D > 0 && D <= 8) {
        const double* slot = ring + (size_t)(tl % kRing) * d * kTM;
#pragma unroll
        for (int k = 0; k < DR; ++k) tc[k] = slot[k * kTM + lane] * A.cscale;
      }
    };
    auto coord = [&](int tl, int k) -> double {
      if constexpr (D > 0 && D <= 8) return tc[k];
      else return ring[(size_t)(tl % kRing) * d * kTM + k * kTM + lane] * A.cscale;
    };
    // A items: K_S columns of local tile tl into KS slot (tl & 1); two columns per pass
    auto eval_A = [&](int tl) {
      if (tl >= ntile || nA == 0 || (A.dbg & 1)) return;
      load_coords(tl);
      const bool valid = trow(tl) >= 0;
      double* KS = KSb + (size_t)(tl & 1) * TS;
      for (int q = 0; q < nA; ++q) {  // A item: skeleton columns 4g .. 4g+3 (padding columns: K == 0)
        const int j0 = 4 * itA[q];
        double kv[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < (D ? D : 1); ++k) {
          for (int kk = k; kk < (D ? k + 1 : d); ++kk) {
            const double t = coord(tl, kk);
            const double* ss = s_srcS + kk * rS + j0;
            const double a0 = t - ss[0], a1 = t - ss[1], a2 = t - ss[2], a3 = t - ss[3];
            kv[0] = fma(a0, a0, kv[0]);
            kv[1] = fma(a1, a1, kv[1]);
            kv[2] = fma(a2, a2, kv[2]);
            kv[3] = fma(a3, a3, kv[3]);
          }
        }
        exp_neg_fast_n<4>(kv, s_tab + lane);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          kv[u] = valid ? kv[u] : 0.0;
          sk = fma(kv[u], kv[u], sk);
          KS[(j0 + u) * kST + lane] = kv[u];
        }
      }
    };
    eval_A(0);
    nbar_sync(kBarEval, kEW * 32);

    const int fr = lane >> 2, fk = lane & 3;  // DMMA fragment coordinates
    for (int it = 0; it < ntile; ++it) {
      const int s = it % kStages;
      if (copier) {  // coordinates of tile it + 3 (slot of tile it - 1, released by the last EVAL barrier)
        issue_copy(it + 3, next_row);
        next_row = row_of(it + 4);
      }
      KID_TRACE(0);
      if (it >= kStages) nbar_sync(kBarEmpty + s, kGT);  // the MMA warps released stage s
      KID_TRACE(1);
      eval_A(it + 1);
      if (!(A.dbg & 1) && nB > 0) {
        load_coords(it);
        const bool valid = trow(it) >= 0;
        const double* KS = KSb + (size_t)(it & 1) * TS;
        double* KN = KNb + (size_t)s * TN;
        for (int q = 0; q < nB; ++q) {
          // B item: columns 8nb .. 8nb+7 -- K_N by exp (two passes of four independent chains) ...
          const int j0 = 8 * itB[q];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int jh = j0 + 4 * hh;
            double kv[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int k = 0; k < (D ? D : 1); ++k) {
              for (int kk = k; kk < (D ? k + 1 : d); ++kk) {
                const double t = coord(it, kk);
                const double* sn = s_srcN + kk * mN + jh;
                const double a0 = t - sn[0], a1 = t - sn[1], a2 = t - sn[2], a3 = t - sn[3];
                kv[0] = fma(a0, a0, kv[0]);
                kv[1] = fma(a1, a1, kv[1]);
                kv[2] = fma(a2, a2, kv[2]);
                kv[3] = fma(a3, a3, kv[3]);
              }
            }
            exp_neg_fast_n<4>(kv, s_tab + lane);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              kv[u] = valid ? kv[u] : 0.0;
              sk = fma(kv[u], kv[u], sk);
              KN[(jh + u) * kST + lane] = kv[u];
            }
          }
          // ... then D = K_N - K_S P2 on DMMA over the block's four 8-target row blocks:
          // C(rb) = K_N fragment, C += K_S(rb, k-step) x (-P2)(k-step, block), back to KN
          if (r > 0 && !(A.dbg & 2)) {
            __syncwarp();
            double c[4][2];
#pragma unroll
            for (int rb = 0; rb < 4; ++rb) {
              c[rb][0] = KN[(j0 + 2 * fk) * kST + rb * 8 + fr];
              c[rb][1] = KN[(j0 + 2 * fk + 1) * kST + rb * 8 + fr];
            }
            const double* ks = KS + fk * kST + fr;
            const double* pb = sP + fk * SPn + j0 + fr;
            for (int k0 = 0; k0 < r4; k0 += 4) {
              const double b = pb[k0 * SPn];
#pragma unroll
              for (int rb = 0; rb < 4; ++rb) dmma884(c[rb][0], c[rb][1], ks[k0 * kST + rb * 8], b);
            }
            __syncwarp();
#pragma unroll
            for (int rb = 0; rb < 4; ++rb) {
              KN[(j0 + 2 * fk) * kST + rb * 8 + fr] = c[rb][0];
              KN[(j0 + 2 * fk + 1) * kST + rb * 8 + fr] = c[rb][1];
            }
          }
        }
      }
      KID_TRACE(2);
      nbar_arrive(kBarFull + s, kGT);  // stage s holds D of tile it
      if (copier) cp_async_wait<1>();  // coordinates of tile it + 2 landed (this thread's copies)
      nbar_sync(kBarEval, kEW * 32);   // ... and K_S of tile it + 1 / those coordinates are visible
      KID_TRACE(3);
    }
    if (copier) cp_async_wait<0>();
    if (part == 0) {
      sk = warp_sum(sk);
      if (lane == 0) red[ew] = sk;
    }
  } else {
    // ================================================================ MMA warps
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kMmaRegs) : "memory");
    const int mw = warp - kMmaW0;
    int2 tl[TPW];  // (a0, b0) block coordinates of WA x 2-block warp tiles; valid ones first
    int ntl = 0;
#pragma unroll
    for (int q = 0; q < TPW; ++q) {
      tl[q] = A.blist[((size_t)part * kMW + mw) * TPW + q];
      ntl += tl[q].x >= 0;
    }
    double acc[TPW][WA][2][2];
#pragma unroll
    for (int q = 0; q < TPW; ++q)
#pragma unroll
      for (int u = 0; u < WA; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) acc[q][u][v][0] = acc[q][u][v][1] = 0.0;
    const int fr = (lane >> 2), fk = (lane & 3);  // fragment coordinates
    int fa0[TPW], fb0[TPW];                       // fragment offsets of each tile's first row / column block
#pragma unroll
    for (int q = 0; q < TPW; ++q) {
      fa0[q] = (tl[q].x >= 0 ? tl[q].x : 0) * 8 * kST;
      fb0[q] = (tl[q].x >= 0 ? tl[q].y : 0) * 8 * kST;
    }
    for (int it = 0; it < ntile; ++it) {
      const int s = it % kStages;
      KID_TRACE(0);
      nbar_sync(kBarFull + s, kGT);
      KID_TRACE(1);
      // unpredicated DMMAs: a per-DMMA predicate makes ptxas wrap every DMMA in a warp-sync and
      // branch (tools/syrk_probe.cu); the tile count is instead dispatched once per stage
      const double* col = KNb + (size_t)s * TN + fr * kST + fk;
      if (!(A.dbg & 4)) {
        if (ntl == TPW) syrk_stage<TPW, TPW, WA>(acc, fa0, fb0, col);
        else if constexpr (TPW > 1) {
          if (ntl == TPW - 1) syrk_stage<TPW - 1, TPW, WA>(acc, fa0, fb0, col);
          else if constexpr (TPW > 2) {
            if (ntl == TPW - 2) syrk_stage<TPW - 2, TPW, WA>(acc, fa0, fb0, col);
          }
        }
      }
      KID_TRACE(3);
      if (it + kStages < ntile) nbar_arrive(kBarEmpty + s, kGT);  // release stage s
    }
    double* G = A.partial + (size_t)chunk * A.LG * A.LG;
    double trd = 0.0;  // this warp's share of trace(D^T D) = ||D||_F^2
#pragma unroll
    for (int q = 0; q < TPW; ++q) {
      if (tl[q].x < 0) continue;
#pragma unroll
      for (int u = 0; u < WA; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int a = tl[q].x + u, b = tl[q].y + v;
          if (a < NBN && b < NBN && a <= b) {
            const int row = a * 8 + fr, colx = b * 8 + 2 * fk;
            G[row + (size_t)colx * A.LG] = acc[q][u][v][0];
            G[row + (size_t)(colx + 1) * A.LG] = acc[q][u][v][1];
            if (row == colx) trd += acc[q][u][v][0];
            if (row == colx + 1) trd += acc[q][u][v][1];
          }
        }
    }
    trd = warp_sum(trd);
    if (lane == 0) red_tr[mw] = trd;
  }
  __syncthreads();
  if (tid == 0) {
    if (part == 0) {
      double t = 0.0;
      for (int w = 0; w < kEW; ++w) t += red[w];
      A.partial_sk[chunk] = t;
    }
    double t = 0.0;
    for (int w = 0; w < kMW; ++w) t += red_tr[w];
    A.partial_sk[(size_t)A.nchunks * (1 + part) + chunk] = t;
  }
}

// out = [sumsq_T, sumsq_K, G (meff x meff col-major, symmetric from the upper triangle)].
// Block = 32 consecutive output elements x 32 chunk groups; group g sums chunks g, g+32, ...
// in order, then the 32 group sums are combined in a fixed order: deterministic.
__global__ void __launch_bounds__(1024) k_gram_reduce(const double* __restrict__ partial, int nchunks, int LG,
                                                      int meff, const double* __restrict__ partial_sk, int nparts,
                                                      double* __restrict__ out) {
  __shared__ double part_s[32][33];
  const int64_t total = (int64_t)meff * meff;
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  double* G = out + 2;
  if (blockIdx.x == 0 && g == 31) {
    // out[0] = trace(G) and out[1] = ||K||_F^2 from the per-CTA partials (fixed order: lane-
    // strided sums, then a fixed shuffle tree) -- deterministic run to run
    double sk = 0.0, tr = 0.0;
    for (int c = lane; c < nchunks; c += 32) sk += partial_sk[c];
    for (int c = lane; c < nchunks * nparts; c += 32) tr += partial_sk[nchunks + c];
    sk = warp_sum(sk);
    tr = warp_sum(tr);
    if (lane == 0) {
      out[0] = tr;
      out[1] = sk;
    }
  }
  for (int64_t base = (int64_t)blockIdx.x * 32; base < total; base += (int64_t)gridDim.x * 32) {
    const int64_t e = base + lane;
    double s = 0.0;
    int64_t off = 0;
    if (e < total) {
      const int x = (int)(e % meff), y = (int)(e / meff);
      int ux = x, uy = y;
      if ((x >> 3) > (y >> 3) || (((x >> 3) == (y >> 3)) && x > y)) { ux = y; uy = x; }
      off = ux + (int64_t)uy * LG;
#pragma unroll 8
      for (int c = g; c < nchunks; c += 32) s += partial[(size_t)c * LG * LG + off];
    }
    part_s[g][lane] = s;
    __syncthreads();
    if (g == 0 && e < total) {
      double t = 0.0;
      for (int q = 0; q < 32; ++q) t += part_s[q][lane];
      G[e] = t;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ projected Gram
// G += (K C)^T (K C) for an arbitrary m x n coefficient matrix C, ||K C||_F^2 and ||K||_F^2.
// The compress_svd error pass (compress.hpp:243-262): with C = V_perp, an
// orthonormal basis of the complement of the sample's right singular vectors V_r,
// ||K - K V_r V_r^T||_2 = ||K V_perp||_2 = sqrt(lambda_max(G)), so the N_T x m difference the
// reference materialises and QR-factors is never formed. Per 32-target tile: K(tile, S) by exp into
// shared memory ([j][t]), D = K C on DMMA ([col][t]), G += D^T D on DMMA with the upper-triangular
// 8x8 blocks of G register-resident across the worker's contiguous chunk of tiles.
// Two warp groups ping-pong on separate K / D buffers (C shared), so one group's exps (DFMA)
// overlap the other's DMMAs; group-local named barriers, no CTA-wide sync in the loop.
struct ProjArgs {
  TargetView tv;
  int d, m, n;
  double cscale;
  const double* src;  // m x d col-major (device, unscaled)
  const double* C;    // m x n col-major (device)
  int64_t ntiles;
  int nworkers;       // gridDim.x * kPG
  double* partial;    // [nworkers][LG][LG]
  int LG;             // ceil8(n)
  double* partial_sk; // [nworkers] sum K^2, then [nworkers] tr(D^T D)
  double* scores;     // LEV mode: l_i = ||(K C)_i||^2 per target (no Gram)
};
constexpr int kPG = 2, kPW = 8, kPT = kPG * kPW * 32;
constexpr int kPMaxBlk = 17;  // SYRK blocks per warp: n <= 128 -> 136 upper blocks over 8 warps

size_t proj_smem_bytes(int m, int n, int d) {
  const int m4 = ceil_to(m, 4), n8 = ceil_to(n, 8);
  return sizeof(double) * ((size_t)m4 * frag_stride(n) + (size_t)d * m4 + (size_t)kPG * (m4 + n8) * kST);
}

// LEV: the leverage pass (lowrank.hpp:304-305) -- C = W = V_r Sigma_r^-1, per target the row sum
// of squares of K W replaces the Gram (rows of the tile summed over column blocks in order).
template <int D, bool LEV>
__global__ void __launch_bounds__(kPT, 1) k_proj_gram(const ProjArgs A) {
  const int d = D ? D : A.d;
  const int m = A.m, n = A.n;
  const int m4 = ceil_to(m, 4), NB = ceil_to(n, 8) / 8, n8 = NB * 8, SC = frag_stride(n);
  const int nblk = NB * (NB + 1) / 2;
  extern __shared__ __align__(16) double sm_pg[];
  double* sC = sm_pg;                         // m4 x SC row-major
  double* s_src = sC + (size_t)m4 * SC;       // d x m4 scaled sources (pad: far away)
  __shared__ double s_tab[kExpTabWords];
  __shared__ short2 s_blk[kPW * kPMaxBlk];
  __shared__ double red_sk[kPG][kPW], red_tr[kPG][kPW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = warp / kPW, gw = warp % kPW;
  double* sK = s_src + (size_t)d * m4 + (size_t)grp * (m4 + n8) * kST;  // [j][t], m4 x kST
  double* sD = sK + (size_t)m4 * kST;                                     // [col][t], n8 x kST
  stage_exp_table(s_tab, tid, kPT);
  for (int e = tid; e < m4 * SC; e += kPT) {
    const int j = e / SC, col = e - j * SC;
    sC[e] = (j < m && col < n) ? A.C[j + (size_t)col * m] : 0.0;
  }
  for (int e = tid; e < d * m4; e += kPT) {
    const int k = e / m4, j = e - k * m4;
    s_src[e] = j < m ? A.src[j + (size_t)k * m] * A.cscale : 1.0e4;
  }
  for (int b = tid; b < nblk; b += kPT) {  // upper-triangular block list, row-major
    int a = 0, rem = b;
    while (rem >= NB - a) { rem -= NB - a; ++a; }
    s_blk[b] = make_short2((short)a, (short)(a + rem));
  }
  __syncthreads();
  const int worker = blockIdx.x * kPG + grp;
  const int64_t tile_lo = A.ntiles * worker / A.nworkers, tile_hi = A.ntiles * (worker + 1) / A.nworkers;
  const double* tabl = s_tab + lane;
  const int bar = 1 + grp, nthr = kPW * 32;
  double acc[kPMaxBlk][2];
#pragma unroll
  for (int q = 0; q < kPMaxBlk; ++q) acc[q][0] = acc[q][1] = 0.0;
  double sk = 0.0;
  for (int64_t tile = tile_lo; tile < tile_hi; ++tile) {
    const int64_t row = tile * kTM + lane;
    const bool live = row < A.tv.nt;
    constexpr int DR = D ? D : 1;
    double t[DR];
    if constexpr (D > 0) {
#pragma unroll
      for (int k = 0; k < D; ++k) t[k] = live ? tcoord(A.tv, row, k) * A.cscale : 0.0;
    }
    // eval: lane = target, four-column groups strided over the group's warps
    for (int g = gw; g < m4 / 4; g += kPW) {
      const int j = 4 * g;
      double kv[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k = 0; k < d; ++k) {
        const double tk = D ? t[D ? k : 0] : (live ? tcoord(A.tv, row, k) * A.cscale : 0.0);
        const double* xk = s_src + (size_t)k * m4 + j;
        const double a0 = tk - xk[0], a1 = tk - xk[1], a2 = tk - xk[2], a3 = tk - xk[3];
        kv[0] = fma(a0, a0, kv[0]);
        kv[1] = fma(a1, a1, kv[1]);
        kv[2] = fma(a2, a2, kv[2]);
        kv[3] = fma(a3, a3, kv[3]);
      }
      exp_neg_fast_n<4>(kv, tabl);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double v = live ? kv[u] : 0.0;  // padding columns are exactly 0 (far-away sources)
        sK[(j + u) * kST + lane] = v;
        sk = fma(v, v, sk);
      }
    }
    nbar_sync(bar, nthr);
    // D = K C: units (column block nb, row half rh), two 8-row blocks per unit share the B fragment
    for (int u = gw; u < 2 * NB; u += kPW) {
      const int nb = u >> 1, rh = u & 1;
      double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      const double* pa = sK + (lane & 3) * kST + rh * 16 + (lane >> 2);
      const double* pb = sC + (lane & 3) * SC + nb * 8 + (lane >> 2);
      for (int k0 = 0; k0 < m4; k0 += 4) {
        const double b = pb[k0 * SC];
        dmma884(c[0][0], c[0][1], pa[k0 * kST], b);
        dmma884(c[1][0], c[1][1], pa[k0 * kST + 8], b);
      }
      if (LEV) {  // row partial over this block's 8 columns -> sD[nb][t]
#pragma unroll
        for (int rb = 0; rb < 2; ++rb) {
          double q = fma(c[rb][0], c[rb][0], c[rb][1] * c[rb][1]);
          q += __shfl_xor_sync(0xffffffffu, q, 1);
          q += __shfl_xor_sync(0xffffffffu, q, 2);
          if ((lane & 3) == 0) sD[nb * kST + rh * 16 + rb * 8 + (lane >> 2)] = q;
        }
      } else {
#pragma unroll
        for (int rb = 0; rb < 2; ++rb)
#pragma unroll
          for (int e = 0; e < 2; ++e) sD[(nb * 8 + 2 * (lane & 3) + e) * kST + rh * 16 + rb * 8 + (lane >> 2)] = c[rb][e];
      }
    }
    nbar_sync(bar, nthr);
    if (LEV) {  // warp 0 of the group: scores of the tile's 32 targets
      if (gw == 0 && live) {
        double sc = 0.0;
        for (int nb = 0; nb < NB; ++nb) sc += sD[nb * kST + lane];
        A.scores[row] = sc;
      }
      continue;
    }
    // G += D^T D over the tile's 32 targets (8 k-steps)
#pragma unroll
    for (int kk = 0; kk < kTM / 4; ++kk) {
      const int k0 = kk * 4 + (lane & 3);
#pragma unroll
      for (int q = 0; q < kPMaxBlk; ++q) {
        const int bi = gw + kPW * q;
        if (bi < nblk) {
          const short2 ab = s_blk[bi];
          const double fa = sD[(ab.x * 8 + (lane >> 2)) * kST + k0];
          const double fb = sD[(ab.y * 8 + (lane >> 2)) * kST + k0];
          dmma884(acc[q][0], acc[q][1], fa, fb);
        }
      }
    }
  }
  if (LEV) return;
  // per-worker partial: upper blocks at (a8 + row) + (b8 + col) * LG; trace from the diagonal blocks
  double tr = 0.0;
  double* P = A.partial + (size_t)worker * A.LG * A.LG;
#pragma unroll
  for (int q = 0; q < kPMaxBlk; ++q) {
    const int bi = gw + kPW * q;
    if (bi < nblk) {
      const short2 ab = s_blk[bi];
      const int x = ab.x * 8 + (lane >> 2);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int y = ab.y * 8 + 2 * (lane & 3) + e;
        P[x + (size_t)y * A.LG] = acc[q][e];
        if (x == y) tr += acc[q][e];
      }
    }
  }
  sk = warp_sum(sk);
  tr = warp_sum(tr);
  if (lane == 0) {
    red_sk[grp][gw] = sk;
    red_tr[grp][gw] = tr;
  }
  nbar_sync(bar, nthr);
  if (gw == 0 && lane == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < kPW; ++w) {
      s0 += red_sk[grp][w];
      s1 += red_tr[grp][w];
    }
    A.partial_sk[worker] = s0;
    A.partial_sk[A.nworkers + worker] = s1;
  }
}

// ------------------------------------------------------------------ TSQR
// Stable spectrum of the full K (lowrank.hpp:56-90 right_factor / singular_values of K, the
// `full_sv` of harness.hpp:176-184): the Gram route loses every sigma below
// ~sqrt(u) sigma_1, Householder QR does not. Each CTA folds its contiguous chunk of 64-row tiles
// of K into an m x m triangular factor kept in shared memory: per tile, Householder QR of the
// stacked [R; A] (A = the tile, evaluated in shared memory), whose reflector for column j touches
// only R[j, :] and A[:, j..] -- one barrier per column, column k of the update owned by warp
// k mod 16 (its dot product with the reflector is a warp-shuffle reduction over the tile rows).
// The per-CTA factors are then folded the same way (mode REDUCE: the tile rows come from a stack
// of upper-triangular factors) until one R remains. R is unique up to row signs; its singular
// values and right singular vectors are those of K.
constexpr int kQW = 16, kQThreads = kQW * 32;
constexpr int kQB = 8;  // panel width (one DMMA block)

struct TsqrArgs {
  TargetView tv;       // EVAL mode: rows of K(T, S)
  int d, m;
  double cscale;
  const double* src;   // m x d col-major (device, unscaled)
  const double* Rin;   // REDUCE mode: nR stacked m x m col-major upper factors
  int64_t nrows;       // rows to fold: nt (EVAL) or nR * m (REDUCE)
  int64_t ntiles;
  double* Rout;        // [gridDim.x][m][m] col-major
};

size_t tsqr_smem_bytes(int m, int d, int rows) {
  const int m8 = ceil_to(m, 8), m4 = ceil_to(m, 4);
  return sizeof(double) * ((size_t)m * (m + 1) / 2 + (size_t)m8 * (rows + 4) + (size_t)kQB * (rows + 4) +
                           2 * (size_t)kQB * (m8 + 4) + (size_t)d * m4);
}

// Blocked (compact-WY) Householder fold of ROWS-row tiles of K into the CTA's triangular factor.
// The reflector of column j of the stacked [R; A] touches only R[j, :] and the tile, so for a
// panel of kQB = 8 columns j0 .. j0 + 7, Y = [e_j0 .. e_j0+7 ; V] (V = the tile parts) and
// H_j0 ... H_j0+7 = I - Y T Y^T (T upper triangular, y_i^T y_j = v_i^T v_j):
//   panel   warp 0, registers only (lane = tile rows lane + 32q): the 8 reflectors, V, T;
//   W       = R[panel rows, trail] + V^T A[:, trail]   (DMMA, one 8-column block per warp);
//   W'      = T^T W;  R[panel rows, trail] -= W'         (scalar, 8 x trail);
//   A       -= V W'                                       (DMMA, 8x8 blocks over the warps).
// Four barriers per panel instead of one per column; the trailing update runs on the FP64
// tensor pipe. R is kept column-packed (R[j][k] at k(k+1)/2 + j) in shared memory.
template <int D, bool EVAL, int ROWS>
__global__ void __launch_bounds__(kQThreads, 1) k_tsqr(const TsqrArgs A) {
  constexpr int RL = ROWS / 32;   // tile rows per lane in the panel warp
  constexpr int SA = ROWS + 4;    // tile column stride (= 4 mod 16: conflict-free DMMA gathers)
  const int d = D ? D : A.d;
  const int m = A.m, m4 = ceil_to(m, 4), m8 = ceil_to(m, 8), NBm = m8 / 8;
  const int SW = m8 + 4;
  extern __shared__ __align__(16) double sm_q[];
  double* sR = sm_q;                          // packed upper triangle
  double* sA = sR + m * (m + 1) / 2;          // tile [k][t], m8 x SA (columns >= m stay 0)
  double* sV = sA + (size_t)m8 * SA;          // panel reflectors [i][t], kQB x SA
  double* sW = sV + kQB * SA;                 // W  [i][k], kQB x SW
  double* sW2 = sW + kQB * SW;                // -W' [i][k]
  double* s_src = sW2 + kQB * SW;             // d x m4 scaled sources (EVAL)
  __shared__ double s_tab[kExpTabWords];
  __shared__ double sT[kQB][kQB];             // T (upper)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fr = lane >> 2, fk = lane & 3;    // DMMA fragment coordinates
  auto rp = [](int j, int k) { return k * (k + 1) / 2 + j; };
  if (EVAL) stage_exp_table(s_tab, tid, kQThreads);
  for (int e = tid; e < m * (m + 1) / 2; e += kQThreads) sR[e] = 0.0;
  for (int e = tid; e < m8 * SA; e += kQThreads) sA[e] = 0.0;
  if (EVAL)
    for (int e = tid; e < d * m4; e += kQThreads) {
      const int k = e / m4, j = e - k * m4;
      s_src[e] = j < m ? A.src[j + (size_t)k * m] * A.cscale : 1.0e4;
    }
  const int64_t t_lo = A.ntiles * blockIdx.x / gridDim.x, t_hi = A.ntiles * (blockIdx.x + 1) / gridDim.x;
  const double* tabl = s_tab + lane;
  for (int64_t tile = t_lo; tile < t_hi; ++tile) {
    __syncthreads();  // previous tile done (and the staging above)
    const int64_t row0 = tile * ROWS;
    if (EVAL) {
      constexpr int DR = D ? D : 1;
      for (int q = 0; q < ROWS / 32; ++q) {
        const int64_t row = row0 + lane + 32 * q;
        const bool live = row < A.nrows;
        double t[DR];
        if constexpr (D > 0) {
#pragma unroll
          for (int k = 0; k < D; ++k) t[k] = live ? tcoord(A.tv, row, k) * A.cscale : 0.0;
        }
        for (int g = warp; g < m4 / 4; g += kQW) {
          const int j = 4 * g;
          double kv[4] = {0.0, 0.0, 0.0, 0.0};
          for (int k = 0; k < d; ++k) {
            const double tk = D ? t[D ? k : 0] : (live ? tcoord(A.tv, row, k) * A.cscale : 0.0);
            const double* xk = s_src + k * m4 + j;
            const double a0 = tk - xk[0], a1 = tk - xk[1], a2 = tk - xk[2], a3 = tk - xk[3];
            kv[0] = fma(a0, a0, kv[0]);
            kv[1] = fma(a1, a1, kv[1]);
            kv[2] = fma(a2, a2, kv[2]);
            kv[3] = fma(a3, a3, kv[3]);
          }
          exp_neg_fast_n<4>(kv, tabl);
#pragma unroll
          for (int u = 0; u < 4; ++u) sA[(j + u) * SA + lane + 32 * q] = live ? kv[u] : 0.0;
        }
      }
    } else {
      for (int e = tid; e < m * ROWS; e += kQThreads) {
        const int k = e / ROWS, i = e - k * ROWS;
        const int64_t gr = row0 + i;
        double v = 0.0;
        if (gr < A.nrows) {
          const int64_t b = gr / m;
          const int j = (int)(gr - b * m);
          v = k >= j ? A.Rin[(size_t)b * m * m + j + (size_t)k * m] : 0.0;
        }
        sA[k * SA + i] = v;
      }
    }
    __syncthreads();
    for (int j0 = 0; j0 < m; j0 += kQB) {
      // ---- panel: warp 0 factors columns j0 .. j0 + 7 in registers
      if (warp == 0) {
        double P[kQB][RL];
#pragma unroll
        for (int c = 0; c < kQB; ++c)
#pragma unroll
          for (int q = 0; q < RL; ++q) P[c][q] = sA[(j0 + c) * SA + lane + 32 * q];
        double tau[kQB];
#pragma unroll
        for (int j = 0; j < kQB; ++j) {
          double sq = 0.0;
#pragma unroll
          for (int q = 0; q < RL; ++q) sq = fma(P[j][q], P[j][q], sq);
          const double sig = warp_sum(sq);
          const bool col = j0 + j < m;
          const double x0 = col ? sR[rp(j0 + j, j0 + j)] : 0.0;
          double beta = x0, iv0 = 0.0;
          tau[j] = 0.0;
          if (sig != 0.0) {
            const double nrm = sqrt(fma(x0, x0, sig));
            beta = x0 >= 0.0 ? -nrm : nrm;
            const double v0 = x0 - beta;
            tau[j] = -v0 / beta;
            iv0 = 1.0 / v0;
          }
#pragma unroll
          for (int q = 0; q < RL; ++q) P[j][q] *= iv0;  // v_j
          double dot[kQB];
#pragma unroll
          for (int k = j + 1; k < kQB; ++k) {
            dot[k] = 0.0;
#pragma unroll
            for (int q = 0; q < RL; ++q) dot[k] = fma(P[j][q], P[k][q], dot[k]);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int k = j + 1; k < kQB; ++k) dot[k] += __shfl_xor_sync(0xffffffffu, dot[k], o);
#pragma unroll
          for (int k = j + 1; k < kQB; ++k) {
            const bool in = j0 + k < m;
            const double w = in ? tau[j] * (sR[rp(j0 + j, j0 + k)] + dot[k]) : 0.0;
#pragma unroll
            for (int q = 0; q < RL; ++q) P[k][q] = fma(-w, P[j][q], P[k][q]);
            __syncwarp();
            if (lane == 0 && in) sR[rp(j0 + j, j0 + k)] -= w;
          }
          __syncwarp();
          if (lane == 0 && col) sR[rp(j0 + j, j0 + j)] = beta;
        }
        // V to shared memory; T by the forward recurrence T[0:j, j] = -tau_j T[0:j, 0:j] (V^T v_j)
#pragma unroll
        for (int c = 0; c < kQB; ++c)
#pragma unroll
          for (int q = 0; q < RL; ++q) sV[c * SA + lane + 32 * q] = P[c][q];
        double g[kQB][kQB];  // g[i][j] = v_i^T v_j, i < j
#pragma unroll
        for (int j = 1; j < kQB; ++j)
#pragma unroll
          for (int i = 0; i < j; ++i) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < RL; ++q) s = fma(P[i][q], P[j][q], s);
            g[i][j] = s;
          }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int j = 1; j < kQB; ++j)
#pragma unroll
            for (int i = 0; i < j; ++i) g[i][j] += __shfl_xor_sync(0xffffffffu, g[i][j], o);
        double T[kQB][kQB];
#pragma unroll
        for (int j = 0; j < kQB; ++j) {
#pragma unroll
          for (int i = 0; i < kQB; ++i) T[i][j] = 0.0;
          T[j][j] = tau[j];
#pragma unroll
          for (int i = 0; i < j; ++i) {
            double s = 0.0;
#pragma unroll
            for (int l = i; l < j; ++l) s = fma(T[i][l], g[l][j], s);
            T[i][j] = -tau[j] * s;
          }
        }
        // lane l writes T rows l / 8 and l / 8 + 4 (compile-time register indices only)
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int i = lane / kQB + 4 * h2, j = lane % kQB;
          double tv = 0.0;
#pragma unroll
          for (int a = 0; a < kQB; ++a)
#pragma unroll
            for (int b = 0; b < kQB; ++b)
              if (a == i && b == j) tv = T[a][b];
          sT[i][j] = tv;
        }
      }
      __syncthreads();
      const int kt = j0 + kQB;  // first trailing column
      if (kt >= m) continue;
      const int NBt = (m8 - kt) / 8;
      // ---- W = R[panel rows, trail] + V^T A[:, trail]: warp w -> 8-column block w (two chains)
      for (int nb = warp; nb < NBt; nb += kQW) {
        double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
        const double* pa = sV + fr * SA + fk;
        const double* pb = sA + (size_t)(kt + nb * 8 + fr) * SA + fk;
#pragma unroll 4
        for (int k0 = 0; k0 < ROWS; k0 += 8) {
          dmma884(c0[0], c0[1], pa[k0], pb[k0]);
          dmma884(c1[0], c1[1], pa[k0 + 4], pb[k0 + 4]);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int k = kt + nb * 8 + 2 * fk + e;
          const double r = k < m ? sR[rp(j0 + fr, k)] : 0.0;
          sW[fr * SW + k] = c0[e] + c1[e] + r;
        }
      }
      __syncthreads();
      // ---- W' = T^T W; R[panel rows, trail] -= W'; sW2 = -W'
      for (int e = tid; e < kQB * (m8 - kt); e += kQThreads) {
        const int i = e / (m8 - kt), k = kt + e % (m8 - kt);
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < kQB; ++l)
          if (l <= i) s = fma(sT[l][i], sW[l * SW + k], s);
        sW2[i * SW + k] = -s;
        if (k < m && j0 + i < m) sR[rp(j0 + i, k)] -= s;
      }
      __syncthreads();
      // ---- A[:, trail] -= V W' on DMMA: (row block, column block) units over the warps
      for (int u = warp; u < (ROWS / 8) * NBt; u += kQW) {
        const int rb = u % (ROWS / 8), nb = u / (ROWS / 8);
        double* cp = sA + (size_t)(kt + nb * 8 + 2 * fk) * SA + rb * 8 + fr;
        double c[2] = {cp[0], cp[SA]};
#pragma unroll
        for (int k0 = 0; k0 < kQB; k0 += 4)
          dmma884(c[0], c[1], sV[(k0 + fk) * SA + rb * 8 + fr], sW2[(k0 + fk) * SW + kt + nb * 8 + fr]);
        cp[0] = c[0];
        cp[SA] = c[1];
      }
      __syncthreads();
    }
  }
  __syncthreads();
  double* out = A.Rout + (size_t)blockIdx.x * m * m;
  for (int e = tid; e < m * m; e += kQThreads) {
    const int k = e / m, j = e - k * m;
    out[e] = j <= k ? sR[rp(j, k)] : 0.0;
  }
}

// ------------------------------------------------------------------ gather rows
// apply_skeleton (compress.hpp:309-325): u_i = sum_j exp(-||y_i - x_j||^2 / 2h^2) q_j over the r
// skeleton points (the far-field matvec). One thread per target, four
// independent exp chains per step (exp_neg_fast_n), skeleton points (pre-scaled by 1/(sqrt2 h))
// and charges staged in shared memory [k][j] / [j] (broadcast reads; r padded to a multiple of
// four with far-away points and zero charges).
template <int D>
__global__ void __launch_bounds__(256) k_apply_skel(TargetView tv, int d_rt, const double* __restrict__ xs, int r4,
                                                    const double* __restrict__ qs, double cscale,
                                                    double* __restrict__ u) {
  const int d = D ? D : d_rt;
  extern __shared__ __align__(16) double sm_apply[];  // d x r4 points, then r4 charges
  double* s_x = sm_apply;
  double* s_q = sm_apply + (size_t)d * r4;
  __shared__ double s_tab[kExpTabWords];
  stage_exp_table(s_tab, threadIdx.x, blockDim.x);
  for (int e = threadIdx.x; e < d * r4 + r4; e += blockDim.x) s_x[e] = xs[e];
  __syncthreads();
  const double* tabl = s_tab + (threadIdx.x & 31);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tv.nt; i += (int64_t)gridDim.x * blockDim.x) {
    constexpr int DR = D ? D : 1;
    double t[DR];
    if constexpr (D > 0) {
#pragma unroll
      for (int k = 0; k < D; ++k) t[k] = tcoord(tv, i, k) * cscale;
    }
    double acc = 0.0;
    for (int j = 0; j < r4; j += 4) {
      double kv[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k = 0; k < d; ++k) {
        const double tk = D ? t[D ? k : 0] : tcoord(tv, i, k) * cscale;
        const double* xk = s_x + (size_t)k * r4 + j;
        const double a0 = tk - xk[0], a1 = tk - xk[1], a2 = tk - xk[2], a3 = tk - xk[3];
        kv[0] = fma(a0, a0, kv[0]);
        kv[1] = fma(a1, a1, kv[1]);
        kv[2] = fma(a2, a2, kv[2]);
        kv[3] = fma(a3, a3, kv[3]);
      }
      exp_neg_fast_n<4>(kv, tabl);
#pragma unroll
      for (int v = 0; v < 4; ++v) acc = fma(kv[v], s_q[j + v], acc);  // in skeleton order, as the reference
    }
    u[i] = acc;
  }
}

__global__ void k_eval_rows(TargetView tv, int d, const double* __restrict__ src, int64_t m, double denom,
                            const int64_t* __restrict__ rows, int64_t count, double* __restrict__ out) {
  const int64_t total = count * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % count, j = e / count;
    const int64_t row = rows[i];
    double sq = 0.0;
    for (int k = 0; k < d; ++k) {
      const double diff = __dsub_rn(tcoord(tv, row, k), src[j + k * m]);
      sq = __dadd_rn(sq, __dmul_rn(diff, diff));
    }
    out[i + j * count] = gauss_exact(sq, denom);
  }
}

__global__ void k_exp_check(const double* __restrict__ x, int64_t n, double* __restrict__ y) {
  __shared__ double s_tab[kExpTabWords];
  stage_exp_table(s_tab, threadIdx.x, blockDim.x);
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = exp_fast(x[i], s_tab + (threadIdx.x & 31));
}

TargetView view(const kid_ctx* c) { return TargetView{c->tbase, c->tld, c->tidx, c->nt}; }

// (WA, TPW) warp-tile layouts of the fused pass' SYRK
#define KID_LAYOUT_SWITCH(DD, M)               \
  if (WA == 1) {                               \
    switch (TPW) {                             \
      case 1: M(DD, 1, 1) break;               \
      case 2: M(DD, 2, 1) break;               \
      case 3: M(DD, 3, 1) break;               \
      case 4: M(DD, 4, 1) break;               \
      case 5: M(DD, 5, 1) break;               \
      default: M(DD, 6, 1) break;              \
    }                                          \
  } else {                                     \
    switch (TPW) {                             \
      case 1: case 2: case 3: M(DD, 3, 2) break; \
      case 4: M(DD, 4, 2) break;               \
      default: M(DD, 5, 2) break;              \
    }                                          \
  }

#define KID_DISPATCH_D(d, MACRO) \
  switch (d) {                   \
    case 1: MACRO(1); break;     \
    case 2: MACRO(2); break;     \
    case 3: MACRO(3); break;     \
    case 4: MACRO(4); break;     \
    case 5: MACRO(5); break;     \
    case 8: MACRO(8); break;     \
    case 16: MACRO(16); break;   \
    default: MACRO(0); break;    \
  }

int check_block(kid_ctx* c, double h) {
  if (!(h > 0.0)) return fail(c, KID_E_CONFIG, "Gaussian kernel requires bandwidth h > 0");
  if (!c->tbase || !c->src || c->m < 1) return fail(c, KID_E_ERROR, "no block: call kid_split or kid_set_block");
  return KID_OK;
}

}  // namespace

int row_norms_dev(kid_ctx* c, double h, double* d_w) {
  if (int rc = check_block(c, h)) return rc;
  if (c->nt == 0) return KID_OK;
  if (int rc = init_device_tables()) return fail(c, rc, "exp table upload failed");
  const double denom = -1.0 / (2.0 * h * h);
  const size_t sm = sizeof(double) * c->m * c->d;
  if (sm > 200 * 1024) return fail(c, KID_E_DIM, "row_norms: m*d too large for shared memory");
  const int blocks = (int)std::min<int64_t>((c->nt + 255) / 256, (int64_t)c->sms * 8);
#define LAUNCH(DD)                                                                              \
  {                                                                                             \
    cudaFuncSetAttribute(k_row_norms<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_row_norms<DD><<<blocks, 256, sm, c->stream>>>(view(c), c->d, c->src, c->m, denom, d_w);   \
  }
  prof_begin(c);
  KID_DISPATCH_D(c->d, LAUNCH)
  prof_end(c);
#undef LAUNCH
  KID_LAUNCHED(c);
  return KID_OK;
}

// Gram of T = K (r == 0) or T = K_N - K_S P2 (r > 0, operands from kid_recon_prepare).
// d_out = [sumsq_T, sumsq_K, G (meff x meff)].
// ------------------------------------------------------------------ large-m path
// For m - r > 128 (BASELINE c4 m=256, c5 m=512) the fused kernel's shared-memory stages do not
// fit; this path evaluates a batch of B target rows of K (columns [skel | non-skel]) into a
// transient column-major HBM buffer with the same arithmetic, then D = K_N - K_S P2 is one DGEMM
// and G += D^T D one DSYRK (cuBLAS, DMMA). ROUND-1 FALLBACK: it materialises K batch-wise,
// which the fused kernel avoids; DESIGN.md section 8 plans its replacement.
// One thread per target row (coordinates in registers, pre-scaled by 1/(sqrt2 h)), a block of
// 256 rows x a contiguous range of the m4/4 four-column groups (blockIdx.y); sources staged in
// shared memory [k][j] (scaled, padding far away -> exactly 0), four exp chains per step; the
// column-major stores Kb[i + j*B] are coalesced across the warp. ||K||_F^2 partial per block.
template <int D>
__global__ void __launch_bounds__(256) k_eval_batch(TargetView tv, int d_rt, const double* __restrict__ src, int m,
                                                    double cscale, int64_t t0, int B, double* __restrict__ Kb,
                                                    double* __restrict__ sk_part, bool staged) {
  const int d = D ? D : d_rt;
  const int m4 = ceil_to(m, 4);
  extern __shared__ __align__(16) double sm_eb[];  // d x m4 scaled sources (when staged)
  __shared__ double s_tab[kExpTabWords];
  __shared__ double red[8];
  stage_exp_table(s_tab, threadIdx.x, blockDim.x);
  if (staged)
    for (int e = threadIdx.x; e < d * m4; e += blockDim.x) {
      const int k = e / m4, j = e - k * m4;
      sm_eb[e] = j < m ? src[j + (int64_t)k * m] * cscale : 1.0e4;
    }
  __syncthreads();
  const double* tabl = s_tab + (threadIdx.x & 31);
  const int ng = m4 / 4;
  const int g_lo = (int)((int64_t)ng * blockIdx.y / gridDim.y), g_hi = (int)((int64_t)ng * (blockIdx.y + 1) / gridDim.y);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double sk = 0.0;
  if (i < B) {
    const bool live = t0 + i < tv.nt;
    constexpr int DR = D ? D : 1;
    double t[DR];
    if constexpr (D > 0) {
#pragma unroll
      for (int k = 0; k < D; ++k) t[k] = live ? tcoord(tv, t0 + i, k) * cscale : 0.0;
    }
    for (int g = g_lo; g < g_hi; ++g) {
      const int j = 4 * g;
      double kv[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k = 0; k < d; ++k) {
        const double tk = D ? t[D ? k : 0] : (live ? tcoord(tv, t0 + i, k) * cscale : 0.0);
        double x[4];
        if (staged) {
          const double* xk = sm_eb + (size_t)k * m4 + j;
#pragma unroll
          for (int u = 0; u < 4; ++u) x[u] = xk[u];
        } else {  // m * d too large for shared memory: warp-uniform L1 broadcasts
#pragma unroll
          for (int u = 0; u < 4; ++u) x[u] = j + u < m ? __ldg(src + j + u + (int64_t)k * m) * cscale : 1.0e4;
        }
        const double a0 = tk - x[0], a1 = tk - x[1], a2 = tk - x[2], a3 = tk - x[3];
        kv[0] = fma(a0, a0, kv[0]);
        kv[1] = fma(a1, a1, kv[1]);
        kv[2] = fma(a2, a2, kv[2]);
        kv[3] = fma(a3, a3, kv[3]);
      }
      exp_neg_fast_n<4>(kv, tabl);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double v = live ? kv[u] : 0.0;
        if (j + u < m) {
          Kb[i + (int64_t)(j + u) * B] = v;
          sk = fma(v, v, sk);
        }
      }
    }
  }
  sk = warp_sum(sk);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sk;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tt = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tt += red[w];
    sk_part[blockIdx.y * gridDim.x + blockIdx.x] = tt;
  }
}

// out = [tr(G), sum_K2, G] with G symmetrised from the upper triangle. Block 0 also folds the
// ||K||^2 partials: lane-strided sums, then a fixed shuffle / warp order (deterministic).
__global__ void __launch_bounds__(256) k_large_finish(double* __restrict__ G, int n, const double* __restrict__ sk_part,
                                                      int nsk, double* __restrict__ out) {
  const int64_t total = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(e % n), y = (int)(e / n);
    out[2 + e] = x <= y ? G[x + (int64_t)y * n] : G[y + (int64_t)x * n];
  }
  if (blockIdx.x == 0) {
    __shared__ double red[8];
    double sk = 0.0;
    for (int b = threadIdx.x; b < nsk; b += blockDim.x) sk += sk_part[b];
    sk = warp_sum(sk);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sk;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tr = 0.0, t = 0.0;
      for (int x = 0; x < n; ++x) tr += G[x + (int64_t)x * n];
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      out[0] = tr;
      out[1] = t;
    }
  }
}

// G (n x n, full) = D^T D (+ G when accumulate) for a tall D (rows x n, col-major, ld): cuBLAS'
// SYRK parallelises over output tiles only, which for n << rows leaves most SMs idle (one 3.5 ms
// call per 262k x 47 batch at c5); here the rows are split into nch chunks, one strided-batched
// DGEMM computes the per-chunk D_c^T D_c, and a fixed-order sum folds them (bitwise reproducible):
// 32 elements x 8 part groups per block, groups combined in order.
__global__ void __launch_bounds__(256) k_sum_partials(const double* __restrict__ part, int nparts, int64_t len,
                                                      double* __restrict__ G, bool accumulate, int rows_c, int ldG) {
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  for (int64_t base = (int64_t)blockIdx.x * 32; base < len; base += (int64_t)gridDim.x * 32) {
    const int64_t e = base + lane;
    double s = 0.0;
    if (e < len)
      for (int p = g; p < nparts; p += 8) s += part[(size_t)p * len + e];
    red[g][lane] = s;
    __syncthreads();
    if (g == 0 && e < len) {
      double t = 0.0;
      for (int q = 0; q < 8; ++q) t += red[q][lane];
      const int64_t ge = e % rows_c + (e / rows_c) * ldG;  // (rows_c x ...) block of G, leading dim ldG
      G[ge] = (accumulate ? G[ge] : 0.0) + t;
    }
    __syncthreads();
  }
}

// P2 row-major (r x SP) -> column-major (r x meff) for the DGEMM
__global__ void k_p2_colmajor(const double* __restrict__ P2, int r, int SP, int meff, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)r * meff;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e % r), nn = (int)(e / r);
    out[e] = P2[(size_t)k * SP + nn];
  }
}

int tall_syrk(kid_ctx* c, const double* D, int rows, int ld, int n, double* G, bool accumulate, double* part,
              int max_parts) {
  const double one = 1.0, zero = 0.0;
  const int nch = std::max(1, std::min(max_parts - 1, rows / 2048));
  const int chunk = rows / nch, rem = rows - nch * chunk;
  // n > 128: only the upper block triangle of 128-column blocks (the full Gram by GEMM would
  // double the flops: 10 of 16 block pairs at n = 512, 3 of 4 at n = 256)
  const int bs = n > 128 ? 128 : n;
  for (int i0 = 0; i0 < n; i0 += bs)
    for (int j0 = i0; j0 < n; j0 += bs) {
      const int ni = std::min(bs, n - i0), nj = std::min(bs, n - j0);
      const int64_t nn = (int64_t)ni * nj;
      const double* Di = D + (size_t)i0 * ld;
      const double* Dj = D + (size_t)j0 * ld;
      if (chunk > 0 &&
          cublasDgemmStridedBatched(c->blas, CUBLAS_OP_T, CUBLAS_OP_N, ni, nj, chunk, &one, Di, ld, chunk, Dj, ld, chunk,
                                    &zero, part, ni, nn, nch) != CUBLAS_STATUS_SUCCESS)
        return fail(c, KID_E_CUDA, "cublasDgemmStridedBatched failed");
      c->launches++;
      if (rem > 0) {
        if (cublasDgemm(c->blas, CUBLAS_OP_T, CUBLAS_OP_N, ni, nj, rem, &one, Di + (size_t)nch * chunk, ld,
                        Dj + (size_t)nch * chunk, ld, &zero, part + nch * nn, ni) != CUBLAS_STATUS_SUCCESS)
          return fail(c, KID_E_CUDA, "cublasDgemm failed");
        c->launches++;
      }
      k_sum_partials<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((nn + 31) / 32, c->sms * 8)), 256, 0,
                       c->stream>>>(part, nch + (rem > 0 ? 1 : 0), nn, G + i0 + (size_t)j0 * n, accumulate, ni, n);
      KID_LAUNCHED(c);
    }
  return KID_OK;
}
constexpr int kSyrkParts = 297;

int gram_dev_large(kid_ctx* c, double h, int64_t r, double* d_out) {
  const int m = (int)c->m, d = c->d, meff = (int)(m - r);
  if (!c->blas) {
    if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS) return fail(c, KID_E_CUDA, "cublasCreate failed");
  }
  if (!c->aux_stream) {
    KID_CK(c, cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 5; ++i) KID_CK(c, cudaEventCreateWithFlags(&c->aux_ev[i], cudaEventDisableTiming));
  }
  cublasSetStream(c->blas, c->stream);
  cublasSetMathMode(c->blas, CUBLAS_DEFAULT_MATH);
  const int64_t nt = c->nt;
  // batches of B target rows through two 1 GB K buffers: the eval of batch b + 1 (aux stream, FP64
  // exp) overlaps the DGEMM / Gram of batch b (launching stream, DMMA)
  const int B = (int)std::max<int64_t>(1024, std::min<int64_t>(nt, (int64_t)(1ll << 30) / (8ll * m)));
  const int64_t nbatch = (nt + B - 1) / B;
  const int ev_rows = (B + 255) / 256;
  const int ev_cols = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_to(m, 4) / 4, (4ll * c->sms + ev_rows - 1) / ev_rows));
  const int ev_blocks = ev_rows * ev_cols;
  const bool ev_staged = sizeof(double) * (size_t)d * ceil_to(m, 4) <= 160 * 1024;
  const size_t ev_smem = ev_staged ? sizeof(double) * (size_t)d * ceil_to(m, 4) : 0;
  if (int rc = init_device_tables()) return fail(c, rc, "exp table upload failed");
  // scratch: 2 K batches (B x m) | G (meff x meff) | P2 col-major (r x meff) | sk partials | Gram parts
  const size_t kb = (size_t)B * m, gb = (size_t)meff * meff, pb = (size_t)std::max<int64_t>(r, 1) * meff;
  char* base = (char*)scratch(c, sizeof(double) * (2 * kb + gb + pb + (size_t)nbatch * ev_blocks + (size_t)kSyrkParts * gb + 64));
  if (!base) return KID_E_OOM;
  double* Kbuf[2] = {(double*)base, (double*)base + kb};
  double* G = Kbuf[1] + kb;
  double* P2c = G + gb;
  double* skp = P2c + pb;
  double* gpart = skp + (size_t)nbatch * ev_blocks;
  if (r > 0) {
    k_p2_colmajor<<<(unsigned)std::min<int64_t>(((int64_t)r * meff + 255) / 256, 1024), 256, 0, c->stream>>>(
        c->P2, (int)r, frag_stride(meff), meff, P2c);
    KID_LAUNCHED(c);
  }
  const double* src = r > 0 ? c->src_perm : c->src;
  const double cscale = std::sqrt(1.0 / (2.0 * h * h));
  const double one = 1.0, mone = -1.0;
  cudaEvent_t ev_start = c->aux_ev[0], ev_eval[2] = {c->aux_ev[1], c->aux_ev[2]}, ev_free[2] = {c->aux_ev[3], c->aux_ev[4]};
  prof_begin(c);
  KID_CK(c, cudaEventRecord(ev_start, c->stream));
  KID_CK(c, cudaStreamWaitEvent(c->aux_stream, ev_start, 0));
  auto eval = [&](int64_t b) -> int {
    const int64_t t0 = b * (int64_t)B;
    const int rows = (int)std::min<int64_t>(B, nt - t0);
    if (b >= 2) KID_CK(c, cudaStreamWaitEvent(c->aux_stream, ev_free[b & 1], 0));
#define LAUNCH(DD)                                                                                         \
  {                                                                                                        \
    cudaFuncSetAttribute(k_eval_batch<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ev_smem);      \
    k_eval_batch<DD><<<dim3(ev_rows, ev_cols), 256, ev_smem, c->aux_stream>>>(view(c), d, src, m, cscale, t0, rows, \
                                                                             Kbuf[b & 1], skp + b * ev_blocks, ev_staged); \
  }
    KID_DISPATCH_D(d, LAUNCH)
#undef LAUNCH
    KID_LAUNCHED(c);
    KID_CK(c, cudaEventRecord(ev_eval[b & 1], c->aux_stream));
    return KID_OK;
  };
  if (nbatch > 0)
    if (int rc = eval(0)) return rc;
  for (int64_t b = 0; b < nbatch; ++b) {
    if (b + 1 < nbatch)
      if (int rc = eval(b + 1)) return rc;
    const int64_t t0 = b * (int64_t)B;
    const int rows = (int)std::min<int64_t>(B, nt - t0);
    double* Kb = Kbuf[b & 1];
    KID_CK(c, cudaStreamWaitEvent(c->stream, ev_eval[b & 1], 0));
    double* KN = Kb + (size_t)r * rows;  // non-skeleton columns follow the r skeleton columns
    if (r > 0) {
      if (cublasDgemm(c->blas, CUBLAS_OP_N, CUBLAS_OP_N, rows, meff, (int)r, &mone, Kb, rows, P2c, (int)r, &one, KN,
                      rows) != CUBLAS_STATUS_SUCCESS)
        return fail(c, KID_E_CUDA, "cublasDgemm failed");
      c->launches++;
    }
    if (int rc = tall_syrk(c, KN, rows, rows, meff, G, b > 0, gpart, kSyrkParts)) return rc;
    KID_CK(c, cudaEventRecord(ev_free[b & 1], c->stream));
  }
  prof_end(c);
  k_large_finish<<<std::max(1, std::min(c->sms * 4, (meff * meff + 255) / 256)), 256, 0, c->stream>>>(
      G, meff, skp, (int)(nbatch * ev_blocks), d_out);
  KID_LAUNCHED(c);
  return KID_OK;
}

int gram_dev(kid_ctx* c, double h, int64_t r, uint32_t flags, double* d_out) {
  (void)flags;
  if (int rc = check_block(c, h)) return rc;
  const int m = (int)c->m, d = c->d;
  const int meff = (int)(m - r);
  if (meff < 1) {
    // full-rank skeleton: D == 0 exactly; ||K||_F^2 still comes from a K-mode pass
    double* tmp = nullptr;
    KID_CK(c, cudaMallocAsync((void**)&tmp, sizeof(double) * (2 + (size_t)m * m), c->stream));
    int rc = gram_dev(c, h, 0, flags, tmp);
    if (!rc) {
      KID_CK(c, cudaMemsetAsync(d_out, 0, sizeof(double), c->stream));
      KID_CK(c, cudaMemcpyAsync(d_out + 1, tmp + 1, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    }
    KID_CK(c, cudaFreeAsync(tmp, c->stream));
    return rc;
  }
  const int NBN = ceil_to(meff, 8) / 8;
  const int LG = NBN * 8;
  // upper-triangular warp tiles of WA x 2 blocks (8x16 when NBN <= 12, else 16x16), row-major,
  // as (a0, b0) block coordinates; fewer padded slots than 16x16 tiles for the small-m configs
  const int WA = NBN <= 12 ? 1 : 2;
  std::vector<int2> tiles;
  if (WA == 1) {
    for (int a = 0; a < NBN; ++a)
      for (int b = a; b < NBN; b += 2) tiles.push_back(make_int2(a, b));
  } else {
    const int NBT = (NBN + 1) / 2;
    for (int a = 0; a < NBT; ++a)
      for (int b = a; b < NBT; ++b) tiles.push_back(make_int2(2 * a, 2 * b));
  }
  const int nb = (int)tiles.size();
  const int tpw_max = WA == 1 ? 6 : 5;
  int TPW = 1;
  for (int cand = 1; cand <= tpw_max; ++cand) {
    TPW = cand;
    if (nb <= kMW * cand) break;
  }
  if (WA == 2 && TPW < 3) TPW = 3;  // the instantiated 16x16 layouts (KID_LAYOUT_SWITCH)
  const int per_part = kMW * TPW;
  const int nparts = (nb + per_part - 1) / per_part;
  // per part: floor/ceil share per warp, valid tiles first; the extra tiles go to the lowest
  // warps, which sit on distinct SMSPs (warp % 4) for the first four -> SMSP-balanced DMMA work
  std::vector<int2> blist((size_t)nparts * per_part, make_int2(-1, -1));
  for (int p = 0; p < nparts; ++p) {
    const int lo = (int)((int64_t)nb * p / nparts), hi = (int)((int64_t)nb * (p + 1) / nparts);
    const int cnt = hi - lo, base_n = cnt / kMW, extra = cnt % kMW;
    int g = lo;
    for (int w = 0; w < kMW; ++w) {
      const int nw = base_n + (w < extra ? 1 : 0);
      for (int q = 0; q < nw; ++q) blist[((size_t)p * kMW + w) * TPW + q] = tiles[g++];
    }
  }
  // eval work lists: A items = groups of four skeleton columns (r4 / 4), B items = the NBN 8-column blocks of the
  // non-skeleton columns (exp + the K_S P2 DMMAs); longest-processing-time greedy over the eval
  // warps (FP64-pipe weights: a DMMA counts 8 warp DFMAs), ties broken by the load of the warp's
  // SMSP (warp % 4)
  std::vector<short> elist((size_t)kEW * kEItems, 0);
  {
    const int nBg = NBN;
    const double wA = 4.0 * (3.0 * d + 12.0), wB = 8.0 * (3.0 * d + 12.0) + 8.0 * (double)ceil_to((int)r, 4);
    std::vector<std::pair<double, int>> items;  // (weight, code): code >= 0 B block, < 0 A group -code-1
    for (int g = 0; g < nBg; ++g) items.push_back({wB, g});
    for (int j = 0; j < ceil_to((int)r, 4) / 4; ++j) items.push_back({wA, -j - 1});
    std::stable_sort(items.begin(), items.end(), [](auto& x, auto& y) { return x.first > y.first; });
    std::vector<double> wl(kEW, 0.0), sl(4, 0.0);
    std::vector<std::vector<short>> la(kEW), lb(kEW);
    for (auto& itx : items) {
      int best = 0;
      for (int w = 1; w < kEW; ++w) {
        const double key = wl[w] + 1e-3 * sl[(kEvalW0 + w) % 4], kb = wl[best] + 1e-3 * sl[(kEvalW0 + best) % 4];
        if (key < kb) best = w;
      }
      wl[best] += itx.first;
      sl[(kEvalW0 + best) % 4] += itx.first;
      if (itx.second >= 0) lb[best].push_back((short)itx.second);
      else la[best].push_back((short)(-itx.second - 1));
    }
    for (int w = 0; w < kEW; ++w) {
      if (2 + la[w].size() + lb[w].size() > (size_t)kEItems) return gram_dev_large(c, h, r, d_out);
      std::sort(la[w].begin(), la[w].end());
      std::sort(lb[w].begin(), lb[w].end());
      short* e = &elist[(size_t)w * kEItems];
      e[0] = (short)la[w].size();
      e[1] = (short)lb[w].size();
      std::copy(la[w].begin(), la[w].end(), e + 2);
      std::copy(lb[w].begin(), lb[w].end(), e + 2 + la[w].size());
    }
  }
  const int rr = (int)r, r4 = ceil_to(rr, 4);
  const int rS = r4, mN = NBN * 8;
  const int TS = (r4 > 0 ? r4 : 4) * kST, TN = ceil_to(NBN + 1, 2) * 8 * kST;
  const size_t smem = sizeof(double) * ((size_t)r4 * frag_stride(meff) + 2 * (size_t)TS + (size_t)kStages * TN +
                                        (size_t)kRing * d * kTM);
  if ((size_t)d * (rS + mN) > (size_t)kCSrc) return gram_dev_large(c, h, r, d_out);
  if (smem > 190 * 1024 || NBN > 16 || getenv("KID_FORCE_LARGE")) return gram_dev_large(c, h, r, d_out);
  const int64_t ntiles = (c->nt + kTM - 1) / kTM;
  if (int rc = init_device_tables()) return fail(c, rc, "exp table upload failed");
  int per_sm = 1;
  {
    const void* fn = nullptr;
#define PICK(DD, BB, WW) fn = (const void*)k_gram<DD, BB, WW>;
#define PICK_D(DD) KID_LAYOUT_SWITCH(DD, PICK)
    KID_DISPATCH_D(d, PICK_D)
#undef PICK_D
#undef PICK
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kGT, smem) != cudaSuccess || per_sm < 1) per_sm = 1;
  }
  int nchunks = std::max(1, c->sms * per_sm / nparts);
  nchunks = (int)std::max<int64_t>(1, std::min<int64_t>(nchunks, ntiles));
  // scratch: blist | elist | partial | partial_sk
  const size_t bl_bytes = sizeof(int2) * blist.size() + sizeof(short) * elist.size();
  const size_t part_bytes = sizeof(double) * (size_t)nchunks * LG * LG;
  char* base = (char*)scratch(c, bl_bytes + 256 + part_bytes + sizeof(double) * ((size_t)nchunks * (1 + nparts) + 8));
  if (!base) return KID_E_OOM;
  int2* d_blist = (int2*)base;
  double* partial = (double*)(base + ((bl_bytes + 255) / 256) * 256);
  double* partial_sk = partial + (size_t)nchunks * LG * LG;
  short* d_elist = (short*)(d_blist + blist.size());
  {  // pageable source: the runtime stages it before returning, so the local vector may go
    std::vector<char> hb(bl_bytes);
    std::memcpy(hb.data(), blist.data(), sizeof(int2) * blist.size());
    std::memcpy(hb.data() + sizeof(int2) * blist.size(), elist.data(), sizeof(short) * elist.size());
    KID_CK(c, cudaMemcpyAsync(d_blist, hb.data(), bl_bytes, cudaMemcpyHostToDevice, c->stream));
  }
  GramArgs A;
  A.tv = view(c);
  A.d = d;
  A.src = r > 0 ? c->src_perm : c->src;
  {
    const std::vector<double>& sh = r > 0 ? c->src_perm_host : c->src_host;
    if (sh.size() != (size_t)m * d) return fail(c, KID_E_ERROR, "gram: host copy of the sources is stale");
    const double cs = std::sqrt(1.0 / (2.0 * h * h));
    for (int k = 0; k < d; ++k) {
      for (int j = 0; j < rS; ++j) A.csrc[k * rS + j] = j < rr ? sh[(size_t)k * m + j] * cs : 1.0e4;
      for (int j = 0; j < mN; ++j)
        A.csrc[d * rS + k * mN + j] = j < meff ? sh[(size_t)k * m + rr + j] * cs : 1.0e4;  // far away: K == 0
    }
  }
  A.m = m;
  A.r = (int)r;
  A.meff = meff;
  A.cscale = std::sqrt(1.0 / (2.0 * h * h));
  A.P2 = r > 0 ? c->P2 : nullptr;
  A.blist = d_blist;
  A.elist = d_elist;
  A.nparts = nparts;
  A.ntiles = ntiles;
  A.nchunks = nchunks;
  A.partial = partial;
  A.LG = LG;
  A.partial_sk = partial_sk;
  A.dbg = getenv("KID_GRAM_DEBUG") ? atoi(getenv("KID_GRAM_DEBUG")) : 0;
  A.trace = nullptr;
  const bool tracing = getenv("KID_GRAM_TRACE") != nullptr;
  const size_t trace_n = (size_t)(kMW + kEW) * kTraceTiles * 4;
  if (tracing) {
    KID_CK(c, cudaMalloc(&A.trace, sizeof(long long) * trace_n));
    KID_CK(c, cudaMemsetAsync(A.trace, 0, sizeof(long long) * trace_n, c->stream));
  }
  dim3 grid(nchunks, nparts);
#define LAUNCH_B(DD, BB, WW)                                                                           \
  {                                                                                                    \
    cudaFuncSetAttribute(k_gram<DD, BB, WW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
    k_gram<DD, BB, WW><<<grid, kGT, smem, c->stream>>>(A);                                             \
  }
#define LAUNCH(DD) KID_LAYOUT_SWITCH(DD, LAUNCH_B)
  prof_begin(c);
  KID_DISPATCH_D(d, LAUNCH)
#undef LAUNCH
#undef LAUNCH_B
  prof_end(c);
  KID_LAUNCHED(c);
  if (tracing) {
    std::vector<long long> tr(trace_n);
    KID_CK(c, cudaMemcpyAsync(tr.data(), A.trace, sizeof(long long) * trace_n, cudaMemcpyDeviceToHost, c->stream));
    KID_CK(c, cudaStreamSynchronize(c->stream));
    cudaFree(A.trace);
    // per-phase mean cycles over tiles 4..kTraceTiles-1 (steady state): MMA warp 0, eval warp 0
    auto at = [&](int w, int it, int ev) { return tr[((size_t)w * kTraceTiles + it) * 4 + ev]; };
    double mw_full = 0, mw_syrk = 0, ew_empty = 0, ew_eval = 0, ew_bar = 0, tile = 0;
    int n = 0;
    for (int it = 4; it + 1 < kTraceTiles; ++it) {
      if (!at(kMmaW0, it + 1, 0)) break;
      mw_full += at(kMmaW0, it, 1) - at(kMmaW0, it, 0);
      mw_syrk += at(kMmaW0, it, 3) - at(kMmaW0, it, 1);
      ew_empty += at(kEvalW0, it, 1) - at(kEvalW0, it, 0);
      ew_eval += at(kEvalW0, it, 2) - at(kEvalW0, it, 1);
      ew_bar += at(kEvalW0, it, 3) - at(kEvalW0, it, 2);
      tile += at(kMmaW0, it + 1, 0) - at(kMmaW0, it, 0);
      ++n;
    }
    fprintf(stderr, "[kid trace] tile 10 eval cycles per eval warp:");
    for (int w = kEvalW0; w < kEvalW0 + kEW; ++w) fprintf(stderr, " %lld", at(w, 10, 2) - at(w, 10, 1));
    fprintf(stderr, " | syrk per MMA warp:");
    for (int w = kMmaW0; w < kMmaW0 + kMW; ++w) fprintf(stderr, " %lld", at(w, 10, 3) - at(w, 10, 1));
    fprintf(stderr, "\n");
    if (n)
      {
        double g3 = 0, g0 = 0;
        int nn = 0;
        for (int it = 4; it + 1 < kTraceTiles; ++it) {
          if (!at(kEvalW0 + kEW - 1, it + 1, 0)) break;
          g0 += at(kEvalW0, it + 1, 0) - at(kEvalW0, it, 3);
          g3 += at(kEvalW0 + kEW - 1, it + 1, 0) - at(kEvalW0 + kEW - 1, it, 3);
          ++nn;
        }
        if (nn) fprintf(stderr, "[kid trace] evalbar->next tile: copier warp %.0f, last eval warp %.0f\n", g0 / nn, g3 / nn);
      }
      fprintf(stderr, "[kid trace] cycles/tile: tile %.0f | mma: wait_full %.0f syrk %.0f | "
                      "eval: wait_empty %.0f eval %.0f arrive+evalbar %.0f (n=%d)\n",
              tile / n, mw_full / n, mw_syrk / n, ew_empty / n, ew_eval / n, ew_bar / n, n);
  }
  k_gram_reduce<<<std::max(1, std::min(c->sms * 2, (meff * meff + 31) / 32)), 1024, 0, c->stream>>>(
      partial, nchunks, LG, meff, partial_sk, nparts, d_out);
  KID_LAUNCHED(c);
  return KID_OK;
}

// G = (K C)^T (K C) for a device m x n coefficient matrix C (col-major); d_out = [||K C||_F^2,
// ||K||_F^2, G (n x n col-major)]. Fused k_proj_gram when its shared-memory footprint fits, else
// the batched path (K batch in HBM, D = K C by DGEMM, G += D^T D by DSYRK).
int proj_gram_dev(kid_ctx* c, double h, const double* d_C, int64_t n64, double* d_out) {
  if (int rc = check_block(c, h)) return rc;
  const int m = (int)c->m, d = c->d, n = (int)n64;
  if (n < 1 || n > m) return fail(c, KID_E_RANGE, "proj_gram: requires 1 <= n <= m");
  if (int rc = init_device_tables()) return fail(c, rc, "exp table upload failed");
  const double cscale = std::sqrt(1.0 / (2.0 * h * h));
  const int LG = ceil_to(n, 8);
  const size_t smem = proj_smem_bytes(m, n, d);
  if (LG <= 128 && smem <= 200 * 1024 && !getenv("KID_FORCE_LARGE")) {
    const int64_t ntiles = (c->nt + kTM - 1) / kTM;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(c->sms, (ntiles + kPG - 1) / kPG));
    const int nworkers = blocks * kPG;
    char* base = (char*)scratch(c, sizeof(double) * ((size_t)nworkers * LG * LG + 2 * (size_t)nworkers + 8));
    if (!base) return KID_E_OOM;
    ProjArgs A;
    A.tv = view(c);
    A.d = d;
    A.m = m;
    A.n = n;
    A.cscale = cscale;
    A.src = c->src;
    A.C = d_C;
    A.ntiles = ntiles;
    A.nworkers = nworkers;
    A.partial = (double*)base;
    A.LG = LG;
    A.partial_sk = A.partial + (size_t)nworkers * LG * LG;
    A.scores = nullptr;
#define LAUNCH(DD)                                                                                   \
  {                                                                                                  \
    cudaFuncSetAttribute(k_proj_gram<DD, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    k_proj_gram<DD, false><<<blocks, kPT, smem, c->stream>>>(A);                                          \
  }
    prof_begin(c);
    KID_DISPATCH_D(d, LAUNCH)
    prof_end(c);
#undef LAUNCH
    KID_LAUNCHED(c);
    k_gram_reduce<<<std::max(1, std::min(c->sms * 2, (n * n + 31) / 32)), 1024, 0, c->stream>>>(
        A.partial, nworkers, LG, n, A.partial_sk, 1, d_out);
    KID_LAUNCHED(c);
    return KID_OK;
  }
  // batched path
  if (!c->blas) {
    if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS) return fail(c, KID_E_CUDA, "cublasCreate failed");
  }
  cublasSetStream(c->blas, c->stream);
  cublasSetMathMode(c->blas, CUBLAS_DEFAULT_MATH);
  const int64_t nt = c->nt;
  const int B = (int)std::max<int64_t>(1024, std::min<int64_t>(nt, (int64_t)(1ll << 30) / (8ll * (m + n))));
  const int64_t nbatch = std::max<int64_t>(1, (nt + B - 1) / B);
  const int ev_rows = (B + 255) / 256;
  const int ev_cols = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_to(m, 4) / 4, (4ll * c->sms + ev_rows - 1) / ev_rows));
  const int ev_blocks = ev_rows * ev_cols;
  const bool ev_staged = sizeof(double) * (size_t)d * ceil_to(m, 4) <= 160 * 1024;
  const size_t ev_smem = ev_staged ? sizeof(double) * (size_t)d * ceil_to(m, 4) : 0;
  char* base = (char*)scratch(c, sizeof(double) * ((size_t)B * (m + n) + (size_t)n * n + (size_t)nbatch * ev_blocks +
                                                  (size_t)kSyrkParts * n * n + 64));
  if (!base) return KID_E_OOM;
  double* Kb = (double*)base;
  double* Db = Kb + (size_t)B * m;
  double* G = Db + (size_t)B * n;
  double* skp = G + (size_t)n * n;
  double* gpart = skp + (size_t)nbatch * ev_blocks;
  const double one = 1.0, zero = 0.0;
  if (nt == 0) {
    KID_CK(c, cudaMemsetAsync(G, 0, sizeof(double) * n * n, c->stream));
    KID_CK(c, cudaMemsetAsync(skp, 0, sizeof(double) * ev_blocks, c->stream));
  }
  prof_begin(c);
  for (int64_t b = 0; b < nbatch && nt > 0; ++b) {
    const int64_t t0 = b * (int64_t)B;
    const int rows = (int)std::min<int64_t>(B, nt - t0);
#define LAUNCH(DD)                                                                                         \
  {                                                                                                        \
    cudaFuncSetAttribute(k_eval_batch<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ev_smem);      \
    k_eval_batch<DD><<<dim3(ev_rows, ev_cols), 256, ev_smem, c->stream>>>(view(c), d, c->src, m, cscale, t0, \
                                                                         rows, Kb, skp + b * ev_blocks, ev_staged); \
  }
    KID_DISPATCH_D(d, LAUNCH)
#undef LAUNCH
    KID_LAUNCHED(c);
    if (cublasDgemm(c->blas, CUBLAS_OP_N, CUBLAS_OP_N, rows, n, m, &one, Kb, rows, d_C, m, &zero, Db, rows) !=
        CUBLAS_STATUS_SUCCESS)
      return fail(c, KID_E_CUDA, "cublasDgemm failed");
    c->launches++;
    if (int rc = tall_syrk(c, Db, rows, rows, n, G, b > 0, gpart, kSyrkParts)) return rc;
  }
  prof_end(c);
  const int nsk = nt == 0 ? ev_blocks : (int)(nbatch * ev_blocks);
  k_large_finish<<<std::max(1, std::min(c->sms * 4, (n * n + 255) / 256)), 256, 0, c->stream>>>(G, n, skp, nsk, d_out);
  KID_LAUNCHED(c);
  return KID_OK;
}

// Upper-triangular R (m x m col-major, device) with R^T R = K^T K, by TSQR over all targets
// (EVAL level: one CTA per SM over contiguous 64-row tiles; REDUCE levels: groups of up to 8
// factors folded per CTA until one remains). Rin/nR: optional extra factors to fold in first
// (kid_tsqr_combine: the factors of other ranks).
int tsqr_dev(kid_ctx* c, double h, const double* d_Rin, int64_t nR, int64_t m64, double* d_R) {
  const bool eval = d_Rin == nullptr;
  if (eval) {
    if (int rc = check_block(c, h)) return rc;
  }
  const int m = eval ? (int)c->m : (int)m64, d = eval ? c->d : 1;
  if (m < 1) return fail(c, KID_E_RANGE, "tsqr: requires m >= 1");
  if (m > 128) return fail(c, KID_E_DIM, "tsqr: m > 128 does not fit the shared-memory factor (use the Gram route)");
  // 128-row tiles where the factor and the tile fit shared memory (210 KB dynamic + 17 KB static), else 64
  const int rows = tsqr_smem_bytes(m, d, 128) <= 210 * 1024 ? 128 : 64;
  const size_t smem = tsqr_smem_bytes(m, d, rows);
  const size_t smem_red = tsqr_smem_bytes(m, 1, rows);
  if (smem > 210 * 1024) return fail(c, KID_E_DIM, "tsqr: m*d too large for shared memory");
  if (int rc = init_device_tables()) return fail(c, rc, "exp table upload failed");
  const size_t mm = (size_t)m * m;
  const int64_t nrows0 = eval ? c->nt : nR * m;
  const int64_t ntiles0 = (nrows0 + rows - 1) / rows;
  const int blocks0 = (int)std::max<int64_t>(1, std::min<int64_t>(c->sms, ntiles0));
  double* base = (double*)scratch(c, sizeof(double) * mm * (size_t)(2 * blocks0 + 2));
  if (!base) return KID_E_OOM;
  double* bufA = base;
  double* bufB = base + mm * (size_t)(blocks0 + 1);
  TsqrArgs A;
  A.tv = eval ? view(c) : TargetView{nullptr, 0, nullptr, 0};
  A.d = d;
  A.m = m;
  A.cscale = std::sqrt(1.0 / (2.0 * h * h));
  A.src = eval ? c->src : nullptr;
  A.Rin = d_Rin;
  A.nrows = nrows0;
  A.ntiles = ntiles0;
  A.Rout = bufA;
#define KID_TSQR_LAUNCH(DD, EV, RR, GRID, ARGS, SM)                                                     \
  {                                                                                                     \
    cudaFuncSetAttribute(k_tsqr<DD, EV, RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(SM));   \
    k_tsqr<DD, EV, RR><<<(GRID), kQThreads, (SM), c->stream>>>(ARGS);                                   \
  }
  prof_begin(c);
  if (eval) {
#define LAUNCH(DD)                                                     \
  if (rows == 128) KID_TSQR_LAUNCH(DD, true, 128, blocks0, A, smem)    \
  else KID_TSQR_LAUNCH(DD, true, 64, blocks0, A, smem)
    KID_DISPATCH_D(d, LAUNCH)
#undef LAUNCH
  } else {
    if (rows == 128) KID_TSQR_LAUNCH(1, false, 128, blocks0, A, smem_red)
    else KID_TSQR_LAUNCH(1, false, 64, blocks0, A, smem_red)
  }
  prof_end(c);
  KID_LAUNCHED(c);
  // fold the per-CTA factors, four per CTA per level
  int64_t nf = blocks0;
  double* cur = bufA;
  double* nxt = bufB;
  while (nf > 1) {
    const int64_t groups = (nf + 3) / 4;
    TsqrArgs Rd = A;
    Rd.Rin = cur;
    Rd.nrows = nf * m;
    Rd.ntiles = (Rd.nrows + rows - 1) / rows;
    Rd.Rout = nxt;
    if (rows == 128) KID_TSQR_LAUNCH(1, false, 128, (unsigned)groups, Rd, smem_red)
    else KID_TSQR_LAUNCH(1, false, 64, (unsigned)groups, Rd, smem_red)
    KID_LAUNCHED(c);
    nf = groups;
    std::swap(cur, nxt);
  }
#undef KID_TSQR_LAUNCH
  KID_CK(c, cudaMemcpyAsync(d_R, cur, sizeof(double) * mm, cudaMemcpyDeviceToDevice, c->stream));
  return KID_OK;
}

// scores[t0 + i] = sum_j KW[i + j * rows]^2 (KW rows x r column-major, coalesced over i)
__global__ void k_rowsq(const double* __restrict__ KW, int rows, int r, double* __restrict__ scores) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < r; ++j) {
      const double v = KW[i + (size_t)j * rows];
      s = fma(v, v, s);
    }
    scores[i] = s;
  }
}

// Leverage for W that does not fit shared memory (c4 m = 256, c5 m = 512): a 1 GB batch of K
// rows (k_eval_batch), KW = K_b W by DGEMM (W read once per batch instead of once per tile),
// row sums of squares.
int leverage_dev_large(kid_ctx* c, double h, const double* d_W, int64_t r, double* d_scores) {
  const int m = (int)c->m, d = c->d, rr = (int)r;
  if (!c->blas) {
    if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS) return fail(c, KID_E_CUDA, "cublasCreate failed");
  }
  cublasSetStream(c->blas, c->stream);
  cublasSetMathMode(c->blas, CUBLAS_DEFAULT_MATH);
  const int64_t nt = c->nt;
  const int B = (int)std::max<int64_t>(1024, std::min<int64_t>(nt, (int64_t)(1ll << 30) / (8ll * (m + rr))));
  const int64_t nbatch = (nt + B - 1) / B;
  const int ev_rows = (B + 255) / 256;
  const int ev_cols = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_to(m, 4) / 4, (4ll * c->sms + ev_rows - 1) / ev_rows));
  const int ev_blocks = ev_rows * ev_cols;
  const bool ev_staged = sizeof(double) * (size_t)d * ceil_to(m, 4) <= 160 * 1024;
  const size_t ev_smem = ev_staged ? sizeof(double) * (size_t)d * ceil_to(m, 4) : 0;
  char* base = (char*)scratch(c, sizeof(double) * ((size_t)B * (m + rr) + (size_t)ev_blocks + 64));
  if (!base) return KID_E_OOM;
  double* Kb = (double*)base;
  double* KW = Kb + (size_t)B * m;
  double* skp = KW + (size_t)B * rr;  // ||K||^2 partials (unused here)
  const double cscale = std::sqrt(1.0 / (2.0 * h * h));
  const double one = 1.0, zero = 0.0;
  prof_begin(c);
  for (int64_t b = 0; b < nbatch; ++b) {
    const int64_t t0 = b * (int64_t)B;
    const int rows = (int)std::min<int64_t>(B, nt - t0);
#define LAUNCH(DD)                                                                                         \
  {                                                                                                        \
    cudaFuncSetAttribute(k_eval_batch<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ev_smem);      \
    k_eval_batch<DD><<<dim3(ev_rows, ev_cols), 256, ev_smem, c->stream>>>(view(c), d, c->src, m, cscale, t0, \
                                                                         rows, Kb, skp, ev_staged);        \
  }
    KID_DISPATCH_D(d, LAUNCH)
#undef LAUNCH
    KID_LAUNCHED(c);
    if (cublasDgemm(c->blas, CUBLAS_OP_N, CUBLAS_OP_N, rows, rr, m, &one, Kb, rows, d_W, m, &zero, KW, rows) !=
        CUBLAS_STATUS_SUCCESS)
      return fail(c, KID_E_CUDA, "cublasDgemm failed");
    c->launches++;
    k_rowsq<<<(unsigned)std::min<int64_t>((rows + 255) / 256, (int64_t)c->sms * 8), 256, 0, c->stream>>>(KW, rows, rr,
                                                                                                      d_scores + t0);
    KID_LAUNCHED(c);
  }
  prof_end(c);
  return KID_OK;
}

int leverage_dev(kid_ctx* c, double h, const double* d_W, int64_t r, double* d_scores) {
  if (int rc = check_block(c, h)) return rc;
  if (r < 1 || r > c->m) return fail(c, KID_E_RANGE, "leverage: requires 1 <= r <= m");
  if (c->nt == 0) return KID_OK;
  if (int rc = init_device_tables()) return fail(c, rc, "exp table upload failed");
  const int m = (int)c->m, d = c->d, rr = (int)r;
  const size_t smem = proj_smem_bytes(m, rr, d);
  if (ceil_to(rr, 8) > 128 || smem > 200 * 1024 || getenv("KID_FORCE_LARGE"))
    return leverage_dev_large(c, h, d_W, r, d_scores);
  // the projected-Gram kernel in leverage mode: K tile by exp, K W on DMMA, row sums of squares
  const int64_t ntiles = (c->nt + kTM - 1) / kTM;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(c->sms, (ntiles + kPG - 1) / kPG));
  ProjArgs A{};
  A.tv = view(c);
  A.d = d;
  A.m = m;
  A.n = rr;
  A.cscale = std::sqrt(1.0 / (2.0 * h * h));
  A.src = c->src;
  A.C = d_W;
  A.ntiles = ntiles;
  A.nworkers = blocks * kPG;
  A.LG = ceil_to(rr, 8);
  A.scores = d_scores;
#define LAUNCH(DD)                                                                                       \
  {                                                                                                      \
    cudaFuncSetAttribute(k_proj_gram<DD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    k_proj_gram<DD, true><<<blocks, kPT, smem, c->stream>>>(A);                                          \
  }
  prof_begin(c);
  KID_DISPATCH_D(d, LAUNCH)
  prof_end(c);
#undef LAUNCH
  KID_LAUNCHED(c);
  return KID_OK;
}

int exp_check_dev(kid_ctx* c, const double* d_x, int64_t n, double* d_y) {
  if (int rc = init_device_tables()) return fail(c, rc, "exp table upload failed");
  k_exp_check<<<(int)std::min<int64_t>((n + 255) / 256, (int64_t)c->sms * 8), 256, 0, c->stream>>>(d_x, n, d_y);
  KID_LAUNCHED(c);
  return KID_OK;
}

int eval_rows_dev(kid_ctx* c, double h, const int64_t* d_rows, int64_t count, double* d_Ks) {
  if (int rc = check_block(c, h)) return rc;
  if (count == 0) return KID_OK;
  const int64_t total = count * c->m;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)c->sms * 16);
  k_eval_rows<<<blocks, 256, 0, c->stream>>>(view(c), c->d, c->src, c->m, 2.0 * h * h, d_rows, count, d_Ks);
  KID_LAUNCHED(c);
  return KID_OK;
}

// u = K(T, S[skel]) q_skel over the current block; x_skel / q_skel from the host (kid_apply_skeleton)
int apply_skeleton_dev(kid_ctx* c, double h, const int64_t* skel, int64_t r, const double* q_skel, double* d_u) {
  if (int rc = check_block(c, h)) return rc;
  const int d = c->d;
  const int64_t m = c->m;
  if (r < 0 || r > m) return fail(c, KID_E_RANGE, "apply_skeleton: rank out of range");
  for (int64_t j = 0; j < r; ++j)
    if (skel[j] < 0 || skel[j] >= m) return fail(c, KID_E_RANGE, "apply_skeleton: skeleton index out of range");
  if (c->src_host.size() != (size_t)m * d) return fail(c, KID_E_ERROR, "apply_skeleton: host copy of the sources is stale");
  if (c->nt == 0) return KID_OK;
  if (int rc = init_device_tables()) return fail(c, rc, "exp table upload failed");
  const int r4 = std::max(4, ceil_to((int)r, 4));
  const double cs = std::sqrt(1.0 / (2.0 * h * h));
  std::vector<double> hx((size_t)d * r4 + r4);
  for (int k = 0; k < d; ++k)
    for (int j = 0; j < r4; ++j) hx[(size_t)k * r4 + j] = j < r ? c->src_host[(size_t)k * m + skel[j]] * cs : 1.0e4;
  for (int j = 0; j < r4; ++j) hx[(size_t)d * r4 + j] = j < r ? q_skel[j] : 0.0;
  const size_t bytes = sizeof(double) * hx.size();
  if (bytes > 160 * 1024) return fail(c, KID_E_DIM, "apply_skeleton: skeleton too large for shared memory");
  double* d_x = (double*)scratch(c, bytes);
  if (!d_x) return KID_E_OOM;
  KID_CK(c, cudaMemcpyAsync(d_x, hx.data(), bytes, cudaMemcpyHostToDevice, c->stream));
  const int blocks = (int)std::min<int64_t>((c->nt + 255) / 256, (int64_t)c->sms * 8);
#define LAUNCH(DD)                                                                                  \
  {                                                                                                 \
    cudaFuncSetAttribute(k_apply_skel<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes); \
    k_apply_skel<DD><<<blocks, 256, bytes, c->stream>>>(view(c), d, d_x, r4, d_x + (size_t)d * r4, cs, d_u); \
  }
  prof_begin(c);
  KID_DISPATCH_D(d, LAUNCH)
  prof_end(c);
#undef LAUNCH
  KID_LAUNCHED(c);
  return KID_OK;
}

// Row-subset view for mc_error (compress.hpp:279-305): the block's targets become
// rows[0..n) of the full target list (indices composed on the device); n < 0 restores it.
__global__ void k_compose_rows(const int64_t* __restrict__ base_idx, const int64_t* __restrict__ rows, int64_t n,
                               int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = base_idx ? base_idx[rows[i]] : rows[i];
}

int select_rows(kid_ctx* c, const int64_t* rows, int64_t n) {
  if (!c->sub_active && n < 0) return KID_OK;
  if (!c->sub_active) {  // save the full view
    c->full_nt = c->nt;
    c->full_tidx = c->tidx;
  }
  if (n < 0) {
    c->nt = c->full_nt;
    c->tidx = c->full_tidx;
    c->sub_active = false;
    return KID_OK;
  }
  for (int64_t i = 0; i < n; ++i)
    if (rows[i] < 0 || rows[i] >= c->full_nt) return fail(c, KID_E_RANGE, "select_rows: row index out of range");
  if (ensure(c, (void**)&c->sub_idx, &c->sub_cap, sizeof(int64_t) * 2 * std::max<int64_t>(n, 1))) return KID_E_OOM;
  int64_t* d_rows = c->sub_idx + std::max<int64_t>(n, 1);
  if (n) {
    KID_CK(c, cudaMemcpyAsync(d_rows, rows, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->stream));
    k_compose_rows<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, c->stream>>>(c->full_tidx, d_rows, n,
                                                                                               c->sub_idx);
    KID_LAUNCHED(c);
  }
  c->nt = n;
  c->tidx = c->sub_idx;
  c->sub_active = true;
  return KID_OK;
}

}  // namespace kid
