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

#include "kid_device.cuh"
#include "kid_fused.cuh"

namespace kid {


namespace {


// ------------------------------------------------------------------ row norms
// w_i = ||K_i||_2 (sampling.hpp:189-196): one thread per target, four sources at a time (four independent
// exp chains, pre-scaled coordinates, the structure of k_sumsq), the squares summed in four interleaved chains.
template <int D>
__global__ void __launch_bounds__(256) k_row_norms(TargetView tv, int d_rt, const double* __restrict__ src,
                                                   int m, double cscale, double* __restrict__ w) {
  const int d = D ? D : d_rt;
  const int m4 = ceil_to(m, 4);
  extern __shared__ __align__(16) double s_src[];  // d x m4 scaled sources (padding far away: K == 0)
  __shared__ double s_tab[kExpTabWords];
  stage_exp_table(s_tab, threadIdx.x, blockDim.x);
  for (int e = threadIdx.x; e < d * m4; e += blockDim.x) {
    const int k = e / m4, j = e - k * m4;
    s_src[e] = j < m ? src[j + (int64_t)k * m] * cscale : 1.0e150;
  }
  __syncthreads();
  const double* tabl = s_tab + (threadIdx.x & 31);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tv.nt; i += (int64_t)gridDim.x * blockDim.x) {
    constexpr int DR = D ? D : 1;
    double t[DR];
    if constexpr (D > 0) {
#pragma unroll
      for (int k = 0; k < D; ++k) t[k] = tcoord(tv, i, k) * cscale;
    }
    double av[4] = {0.0, 0.0, 0.0, 0.0};  // four independent chains (sources j, j + 4, ... each)
    for (int j = 0; j < m4; j += 4) {
      double kv[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k = 0; k < d; ++k) {
        const double tk = D ? t[D ? k : 0] : tcoord(tv, i, k) * cscale;
        const double* xk = s_src + k * m4 + j;
        const double a0 = tk - xk[0], a1 = tk - xk[1], a2 = tk - xk[2], a3 = tk - xk[3];
        kv[0] = fma(a0, a0, kv[0]);
        kv[1] = fma(a1, a1, kv[1]);
        kv[2] = fma(a2, a2, kv[2]);
        kv[3] = fma(a3, a3, kv[3]);
      }
      exp_neg_fast_n<4>(kv, tabl);
#pragma unroll
      for (int u = 0; u < 4; ++u) av[u] = fma(kv[u], kv[u], av[u]);
    }
    w[i] = __dsqrt_rn((av[0] + av[1]) + (av[2] + av[3]));
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
  long long* trace;    // profiling build only (KID_GRAM_TRACE_BUILD): [warp][tile][4] clock64 stamps of CTA 0
  // scaled source coordinates in the kernel-parameter (constant) bank: the eval warps read them
  // at warp-uniform indices, so they cost constant-cache broadcasts instead of shared-memory
  // wavefronts. [d][rS] skeleton columns, then [d][mN] non-skeleton columns (padding: far away)
  double csrc[kCSrc];
};
constexpr int kTraceTiles = 64;

// Warp-specialized pipeline (one CTA per SM), per 32-target tile:
//   the kEW "eval" warps own a host-balanced list of work items:
//     A item j      : K_S column j of the NEXT tile (exp) -> KS ring (2 slots, eval-private)
//     B item g      : non-skeleton columns 4g..4g+3 of THIS tile: K_N by exp (4 independent
//                     chains), then D = K_N - K_S P2 by DFMA against the K_S row of the target
//                     (KS ring) and -P2 rows (shared memory, LDS.128 broadcasts) -> KN stage
//     lane = target row throughout, so stores are conflict-free column-major [col][t] (stride
//     kST = 36 = 4 mod 16, which also makes the DMMA fragment gathers conflict-free);
//   the kMW "MMA" warps: G += D^T D (DMMA.8x8x4) on static WA x 2-block warp tiles of
//     the upper triangle, accumulators register-resident across the CTA's whole target chunk.
// Hand-off by named barriers: FULL[s] (eval arrive, MMA sync), EMPTY[s] (MMA arrive, eval sync),
// EVAL (eval warps only: K_S of the next tile and the next coordinates are visible).
// Target coordinates stream through a 4-slot shared-memory ring by cp.async, issued three tiles
// ahead (the target index of the copy is itself loaded one tile earlier).
// DMMA and DFMA share the FP64 datapath (tools/fp64_overlap.cu): the split keeps it fed from
// both sides -- the MMA warps never wait on a GEMM phase, the eval warps fill the DMMA gaps.
constexpr int kMW = 7, kEW = 13, kGT = (kMW + kEW) * 32;  // 640 threads
constexpr int kEvalW0 = kMW, kMmaW0 = 0;
constexpr int kStages = 4;
constexpr int kRing = 4;      // target-coordinate ring slots
constexpr int kEItems = 48;   // per eval warp: 2 counts + items
constexpr int kBarFull = 1, kBarEmpty = 1 + kStages, kBarEval = 1 + 2 * kStages;

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
constexpr int kEvalRegs = 88, kMmaRegs = 104;
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
  const int r = A.r, meff = A.meff;
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
    const bool copier = ew < d;  // warp ew copies coordinate dims ew, ew + kEW, ...
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
      if (tl >= ntile || nA == 0) return;
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
      if (nB > 0) {
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
          if (r > 0) {
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
      {
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



}  // namespace

int row_norms_dev(kid_ctx* c, double h, double* d_w) {
  if (int rc = check_block(c, h)) return rc;
  if (c->nt == 0) return KID_OK;
  if (int rc = init_device_tables()) return fail(c, rc, "exp table upload failed");
  const double cscale = std::sqrt(1.0 / (2.0 * h * h));
  const size_t sm = sizeof(double) * (size_t)ceil_to((int)c->m, 4) * c->d;
  if (sm > 200 * 1024) return fail(c, KID_E_DIM, "row_norms: m*d too large for shared memory");
  const int blocks = (int)std::min<int64_t>((c->nt + 255) / 256, (int64_t)c->sms * 8);
#define LAUNCH(DD)                                                                                   \
  {                                                                                                  \
    cudaFuncSetAttribute(k_row_norms<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);      \
    k_row_norms<DD><<<blocks, 256, sm, c->stream>>>(view(c), c->d, c->src, (int)c->m, cscale, d_w);  \
  }
  prof_begin(c);
  KID_DISPATCH_D(c->d, LAUNCH)
  prof_end(c);
#undef LAUNCH
  KID_LAUNCHED(c);
  return KID_OK;
}

// ||K||_F^2 alone (the full-rank skeleton of the residual pass: D == 0): one thread per target,
// four exp chains, per-block partials folded in a fixed order. d_out = [0, ||K||_F^2].
template <int D>
__global__ void __launch_bounds__(256) k_sumsq(TargetView tv, int d_rt, const double* __restrict__ src, int m,
                                               double cscale, double* __restrict__ part) {
  const int d = D ? D : d_rt;
  const int m4 = ceil_to(m, 4);
  extern __shared__ __align__(16) double sm_sq[];  // d x m4 scaled sources
  __shared__ double s_tab[kExpTabWords];
  __shared__ double red[8];
  stage_exp_table(s_tab, threadIdx.x, blockDim.x);
  for (int e = threadIdx.x; e < d * m4; e += blockDim.x) {
    const int k = e / m4, j = e - k * m4;
    sm_sq[e] = j < m ? src[j + (int64_t)k * m] * cscale : 1.0e150;
  }
  __syncthreads();
  const double* tabl = s_tab + (threadIdx.x & 31);
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tv.nt; i += (int64_t)gridDim.x * blockDim.x) {
    constexpr int DR = D ? D : 1;
    double t[DR];
    if constexpr (D > 0) {
#pragma unroll
      for (int k = 0; k < D; ++k) t[k] = tcoord(tv, i, k) * cscale;
    }
    for (int j = 0; j < m4; j += 4) {
      double kv[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k = 0; k < d; ++k) {
        const double tk = D ? t[D ? k : 0] : tcoord(tv, i, k) * cscale;
        const double* xk = sm_sq + k * m4 + j;
        const double a0 = tk - xk[0], a1 = tk - xk[1], a2 = tk - xk[2], a3 = tk - xk[3];
        kv[0] = fma(a0, a0, kv[0]);
        kv[1] = fma(a1, a1, kv[1]);
        kv[2] = fma(a2, a2, kv[2]);
        kv[3] = fma(a3, a3, kv[3]);
      }
      exp_neg_fast_n<4>(kv, tabl);
#pragma unroll
      for (int u = 0; u < 4; ++u) acc = fma(kv[u], kv[u], acc);
    }
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

__global__ void k_sumsq_finish(const double* __restrict__ part, int n, double* __restrict__ out) {
  double s = 0.0;
  for (int b = threadIdx.x; b < n; b += 32) s += part[b];
  s = warp_sum(s);
  if (threadIdx.x == 0) {
    out[0] = 0.0;
    out[1] = s;
  }
}

int sumsq_dev(kid_ctx* c, double h, double* d_out) {
  const int m = (int)c->m, d = c->d;
  const size_t smem = sizeof(double) * (size_t)d * ceil_to(m, 4);
  if (smem > 160 * 1024) return fail(c, KID_E_DIM, "sumsq: m*d too large for shared memory");
  if (int rc = init_device_tables()) return fail(c, rc, "exp table upload failed");
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((c->nt + 255) / 256, (int64_t)c->sms * 4));
  double* part = (double*)scratch(c, sizeof(double) * (blocks + 8));
  if (!part) return KID_E_OOM;
  const double cscale = std::sqrt(1.0 / (2.0 * h * h));
  c->last_kernel = "k_sumsq";
#define LAUNCH(DD)                                                                                  \
  {                                                                                                 \
    cudaFuncSetAttribute(k_sumsq<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);      \
    k_sumsq<DD><<<blocks, 256, smem, c->stream>>>(view(c), d, c->src, m, cscale, part);             \
  }
  prof_begin(c);
  KID_DISPATCH_D(d, LAUNCH)
  prof_end(c);
#undef LAUNCH
  KID_LAUNCHED(c);
  k_sumsq_finish<<<1, 32, 0, c->stream>>>(part, blocks, d_out);
  KID_LAUNCHED(c);
  return KID_OK;
}

int gram_dev(kid_ctx* c, double h, int64_t r, double* d_out) {
  if (int rc = check_block(c, h)) return rc;
  const int m = (int)c->m, d = c->d;
  const int meff = (int)(m - r);
  if (meff < 1) return sumsq_dev(c, h, d_out);  // full-rank skeleton: D == 0 exactly, only ||K||_F^2
  const int NBN = ceil_to(meff, 8) / 8;
  const int LG = NBN * 8;
  // few D columns (n <= 32: the high-rank end of the eps sweeps): the warp-tile kernel, one CTA per SM --
  // every warp runs its own 32-row tile end to end, no producer / consumer hand-off (kid_fused_w.cu)
  if (r > 0 && NBN <= 4 && c->kernel_choice != 1 && c->path != KID_PATH_CLUSTER) {
    const int rc = fused_w_dev(c, h, FX_RESID, nullptr, 0, d_out);
    if (rc != 1) return rc;
  }
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
  const int nparts = (nb + kMW * TPW - 1) / (kMW * TPW);
  // with several parts, size the warp tile list to the part's floor/ceil share: the MMA warps
  // dispatch only tile counts TPW, TPW - 1 and TPW - 2
  TPW = std::max(WA == 2 ? 3 : 1, ((nb + nparts - 1) / nparts + kMW - 1) / kMW);
  const int per_part = kMW * TPW;
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
      if (2 + la[w].size() + lb[w].size() > (size_t)kEItems) return fused_dev(c, h, r > 0 ? FX_RESID : FX_GRAM, nullptr, 0, d_out);
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
  if ((size_t)d * (rS + mN) > (size_t)kCSrc || smem > 190 * 1024 || NBN > 16 || c->path == KID_PATH_CLUSTER)
    return fused_dev(c, h, r > 0 ? FX_RESID : FX_GRAM, nullptr, 0, d_out);
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
      for (int j = 0; j < rS; ++j) A.csrc[k * rS + j] = j < rr ? sh[(size_t)k * m + j] * cs : 1.0e150;
      for (int j = 0; j < mN; ++j)
        A.csrc[d * rS + k * mN + j] = j < meff ? sh[(size_t)k * m + rr + j] * cs : 1.0e150;  // far away: K == 0
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
  A.trace = nullptr;
#ifdef KID_GRAM_TRACE_BUILD  // profiling build only (tools/gram_probe.py): per-phase clock64 stamps of CTA 0
  const bool tracing = true;
#else
  const bool tracing = false;
#endif
  const size_t trace_n = (size_t)(kMW + kEW) * kTraceTiles * 4;
  if (tracing) {
    KID_CK(c, cudaMalloc(&A.trace, sizeof(long long) * trace_n));
    KID_CK(c, cudaMemsetAsync(A.trace, 0, sizeof(long long) * trace_n, c->stream));
  }
  dim3 grid(nchunks, nparts);
  c->last_kernel = "k_gram";
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
    for (int j = 0; j < r4; ++j) hx[(size_t)k * r4 + j] = j < r ? c->src_host[(size_t)k * m + skel[j]] * cs : 1.0e150;
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


// ------------------------------------------------------------------ launch wrappers
// (kid_next.cu launches these kernels through host functions: no relocatable device code)
int launch_gram_reduce(kid_ctx* c, const double* partial, int nchunks, int LG, int n, const double* partial_sk,
                       int nparts, double* out) {
  k_gram_reduce<<<std::max(1, std::min(c->sms * 2, (n * n + 31) / 32)), 1024, 0, c->stream>>>(partial, nchunks, LG, n,
                                                                                            partial_sk, nparts, out);
  KID_LAUNCHED(c);
  return KID_OK;
}

}  // namespace kid
