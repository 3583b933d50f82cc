// kid_next.cu -- the SURVEY.md 8(f) passes beyond the fused residual Gram:
//   k_proj_gram   G = (K C)^T (K C)      compress_svd error pass (compress.hpp:219-273)
//                 LEV mode: ||K_i W||^2    leverage scores (lowrank.hpp:296-308)
//   k_tsqr        R with R^T R = K^T K   the stable spectrum of K (lowrank.hpp:56-90)
// with their batched (K batch in HBM + cuBLAS) fallbacks for operands beyond shared memory.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>


#include "kid_device.cuh"

namespace kid {
namespace {

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
    s_src[e] = j < m ? A.src[j + (size_t)k * m] * A.cscale : 1.0e150;
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
    if constexpr (LEV) {  // warp 0 of the group: scores of the tile's 32 targets
      if (gw == 0 && live) {
        double sc = 0.0;
        for (int nb = 0; nb < NB; ++nb) sc += sD[nb * kST + lane];
        A.scores[row] = sc;
      }
    } else {
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
  }
  if constexpr (LEV) return;
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
  const int m = A.m, m4 = ceil_to(m, 4), m8 = ceil_to(m, 8);
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
      s_src[e] = j < m ? A.src[j + (size_t)k * m] * A.cscale : 1.0e150;
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

}  // namespace

// G = (K C)^T (K C) for a device m x n coefficient matrix C (col-major); d_out = [||K C||_F^2,
// ||K||_F^2, G (n x n col-major)]. Fused k_proj_gram when its shared-memory footprint fits, else
// the cluster kernel of kid_fused.cu (K never leaves the SMs in either).
int proj_gram_dev(kid_ctx* c, double h, const double* d_C, int64_t n64, double* d_out) {
  if (int rc = check_block(c, h)) return rc;
  const int m = (int)c->m, d = c->d, n = (int)n64;
  if (n < 1 || n > m) return fail(c, KID_E_RANGE, "proj_gram: requires 1 <= n <= m");
  if (int rc = init_device_tables()) return fail(c, rc, "exp table upload failed");
  const double cscale = std::sqrt(1.0 / (2.0 * h * h));
  const int LG = ceil_to(n, 8);
  const size_t smem = proj_smem_bytes(m, n, d);
  if (LG <= 128 && smem <= 200 * 1024 && c->path != KID_PATH_CLUSTER) {
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
    if (int rc = launch_gram_reduce(c, A.partial, nworkers, LG, n, A.partial_sk, 1, d_out)) return rc;
    return KID_OK;
  }
  // beyond one SM's shared memory (c4 / c5): the 2-CTA cluster kernel (kid_fused.cu) with M = C
  std::vector<double> Ch((size_t)m * n);
  KID_CK(c, cudaMemcpyAsync(Ch.data(), d_C, sizeof(double) * Ch.size(), cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  return fused_dev(c, h, FX_PROJ, Ch.data(), n, d_out);
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

// Leverage for W beyond one SM's shared memory (c4 m = 256, c5 m = 512): the cluster kernel of
// kid_fused.cu in leverage mode (K W on DMMA across the CTA pair, row sums of squares).
int leverage_dev_large(kid_ctx* c, double h, const double* d_W, int64_t r, double* d_scores) {
  const int64_t m = c->m;
  std::vector<double> Wh((size_t)m * r);
  KID_CK(c, cudaMemcpyAsync(Wh.data(), d_W, sizeof(double) * Wh.size(), cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  return fused_dev(c, h, FX_LEV, Wh.data(), r, d_scores);
}

int leverage_dev(kid_ctx* c, double h, const double* d_W, int64_t r, double* d_scores) {
  if (int rc = check_block(c, h)) return rc;
  if (r < 1 || r > c->m) return fail(c, KID_E_RANGE, "leverage: requires 1 <= r <= m");
  if (c->nt == 0) return KID_OK;
  if (int rc = init_device_tables()) return fail(c, rc, "exp table upload failed");
  const int m = (int)c->m, d = c->d, rr = (int)r;
  const size_t smem = proj_smem_bytes(m, rr, d);
  if (ceil_to(rr, 8) > 128 || smem > 200 * 1024 || c->path == KID_PATH_CLUSTER)
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

}  // namespace kid
