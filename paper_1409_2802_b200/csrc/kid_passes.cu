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
//   k_leverage    l_i = ||K_i W||^2                      lowrank.hpp:304-305
//   k_eval_rows   K[rows, :] gathered                     compress.hpp:130-137
// The m x m accumulators live in registers (DMMA C fragments) across all tiles of a
// CTA's contiguous target chunk; partials are reduced in a fixed chunk order so results
// are bitwise reproducible run to run.
#include <algorithm>
#include <cstring>
#include <vector>

#include "kid_internal.cuh"

namespace kid {
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
                                                   int64_t m, double denom, double* __restrict__ w) {
  const int d = D ? D : d_rt;
  extern __shared__ double s_src[];  // d x m, s_src[j + k*m]
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
      const double kv = gauss_exact(sq, denom);
      acc = __dadd_rn(acc, __dmul_rn(kv, kv));  // sequential over j (sampling.hpp:193)
    }
    w[i] = __dsqrt_rn(acc);
  }
}

// ------------------------------------------------------------------ Gram / residual Gram
struct GramArgs {
  TargetView tv;
  int d;
  const double* src;   // m x d col-major, columns already in [skel | non-skel] order
  int m, r, meff;      // meff = m - r
  double denom;        // (2h)h
  const double* P2;    // r x meff row-major, stride SP (device); nullptr when r == 0
  const int2* blist;   // [nparts][kNW][BPW] (a, b) block pairs, a = -1: empty slot
  int nparts;
  int64_t ntiles;
  int nchunks;
  double* partial;     // [nchunks][LG][LG]
  int LG;              // padded Gram leading dimension = ceil8(meff)
  double* partial_sk;  // [nchunks] (written by part 0)
};

template <int D, int BPW>
__global__ void __launch_bounds__(kNT) k_gram(GramArgs A) {
  const int d = D ? D : A.d;
  const int m = A.m, r = A.r, meff = A.meff;
  const int r4 = ceil_to(r, 4);
  const int SS = frag_stride(r4 > 0 ? r4 : 4);
  const int SN = frag_stride(meff);
  const int SP = SN;
  const int NBN = ceil_to(meff, 8) / 8;
  extern __shared__ __align__(16) double smem[];
  double* s_src = smem;                       // d x m
  double* s_t = s_src + (size_t)d * m;        // d x kTM
  double* KS = s_t + (size_t)d * kTM;         // kTM x SS
  double* KN = KS + (size_t)kTM * SS;         // kTM x SN
  double* sP = KN + (size_t)kTM * SN;         // r4 x SP
  __shared__ double red[kNW];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int chunk = blockIdx.x, part = blockIdx.y;
  for (int e = tid; e < m * d; e += kNT) s_src[e] = A.src[e];
  for (int e = tid; e < kTM * SS; e += kNT) KS[e] = 0.0;
  for (int e = tid; e < kTM * SN; e += kNT) KN[e] = 0.0;
  for (int e = tid; e < r4 * SP; e += kNT) {
    const int k = e / SP, n = e % SP;
    sP[e] = (k < r && n < meff) ? A.P2[(size_t)k * SP + n] : 0.0;
  }
  int2 bl[BPW];
#pragma unroll
  for (int s = 0; s < BPW; ++s) bl[s] = A.blist[((size_t)part * kNW + warp) * BPW + s];
  double acc[BPW][2];
#pragma unroll
  for (int s = 0; s < BPW; ++s) acc[s][0] = acc[s][1] = 0.0;
  double sk = 0.0;
  __syncthreads();

  const int64_t tile_lo = A.ntiles * chunk / A.nchunks, tile_hi = A.ntiles * (chunk + 1) / A.nchunks;
  for (int64_t tile = tile_lo; tile < tile_hi; ++tile) {
    const int64_t t0 = tile * kTM;
    for (int e = tid; e < kTM * d; e += kNT) {
      const int t = e % kTM, k = e / kTM;
      s_t[t + k * kTM] = (t0 + t < A.tv.nt) ? tcoord(A.tv, t0 + t, k) : 0.0;
    }
    __syncthreads();
    // (1) evaluate the 32 x m tile: columns [0, r) -> KS, [r, m) -> KN
    for (int e = tid; e < kTM * m; e += kNT) {
      const int t = e / m, j = e - t * m;
      double kv = 0.0;
      if (t0 + t < A.tv.nt) {
        double sq = 0.0;
        if (D) {
#pragma unroll
          for (int k = 0; k < (D ? D : 1); ++k) {
            const double diff = __dsub_rn(s_t[t + k * kTM], s_src[j + k * m]);
            sq = __dadd_rn(sq, __dmul_rn(diff, diff));
          }
        } else {
          for (int k = 0; k < d; ++k) {
            const double diff = __dsub_rn(s_t[t + k * kTM], s_src[j + k * m]);
            sq = __dadd_rn(sq, __dmul_rn(diff, diff));
          }
        }
        kv = gauss_exact(sq, A.denom);
      }
      sk = fma(kv, kv, sk);
      if (j < r) KS[t * SS + j] = kv;
      else KN[t * SN + (j - r)] = kv;
    }
    __syncthreads();
    // (2) D = K_N - K_S P2 on DMMA (skipped in mode K, r == 0)
    if (r > 0) {
      for (int nb = warp; nb < NBN; nb += kNW) {
        double c[kTM / 8][2];
#pragma unroll
        for (int rb = 0; rb < kTM / 8; ++rb) c[rb][0] = c[rb][1] = 0.0;
        for (int k0 = 0; k0 < r4; k0 += 4) {
          const double b = sP[(k0 + (lane & 3)) * SP + nb * 8 + (lane >> 2)];
#pragma unroll
          for (int rb = 0; rb < kTM / 8; ++rb) {
            const double a = KS[(rb * 8 + (lane >> 2)) * SS + k0 + (lane & 3)];
            dmma884(c[rb][0], c[rb][1], a, b);
          }
        }
#pragma unroll
        for (int rb = 0; rb < kTM / 8; ++rb) {
          double* p = &KN[(rb * 8 + (lane >> 2)) * SN + nb * 8 + 2 * (lane & 3)];
          p[0] = p[0] - c[rb][0];
          p[1] = p[1] - c[rb][1];
        }
      }
      __syncthreads();
    }
    // (3) G += T^T T, k = 32 targets, register-resident 8x8 blocks
#pragma unroll
    for (int k0 = 0; k0 < kTM; k0 += 4) {
      const double* row = KN + (k0 + (lane & 3)) * SN + (lane >> 2);
      int cur = -1;
      double af = 0.0;
#pragma unroll
      for (int s = 0; s < BPW; ++s) {
        if (bl[s].x >= 0) {
          if (bl[s].x != cur) {
            af = row[bl[s].x * 8];
            cur = bl[s].x;
          }
          const double bf = row[bl[s].y * 8];
          dmma884(acc[s][0], acc[s][1], af, bf);
        }
      }
    }
    __syncthreads();
  }
  // partial Gram blocks of this (chunk, part)
  double* G = A.partial + (size_t)chunk * A.LG * A.LG;
#pragma unroll
  for (int s = 0; s < BPW; ++s) {
    if (bl[s].x >= 0) {
      const int row = bl[s].x * 8 + (lane >> 2);
      const int col = bl[s].y * 8 + 2 * (lane & 3);
      G[row + (size_t)col * A.LG] = acc[s][0];
      G[row + (size_t)(col + 1) * A.LG] = acc[s][1];
    }
  }
  (void)NBN;
  if (part == 0) {
    sk = warp_sum(sk);
    if (lane == 0) red[warp] = sk;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kNW; ++w) t += red[w];
      A.partial_sk[chunk] = t;
    }
  }
}

// out = [sumsq_T, sumsq_K, G (meff x meff col-major, symmetric from the upper triangle)]
__global__ void k_gram_reduce(const double* __restrict__ partial, int nchunks, int LG, int meff,
                              const double* __restrict__ partial_sk, double* __restrict__ out) {
  const int64_t total = (int64_t)meff * meff;
  double* G = out + 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int x = (int)(e % meff), y = (int)(e / meff);
    int ux = x, uy = y;
    if ((x >> 3) > (y >> 3) || (((x >> 3) == (y >> 3)) && x > y)) { ux = y; uy = x; }
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += partial[(size_t)c * LG * LG + ux + (size_t)uy * LG];
    G[x + (size_t)y * meff] = s;
  }
}

__global__ void k_gram_finish(const double* __restrict__ partial_sk, int nchunks, int meff, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double sk = 0.0;
    for (int c = 0; c < nchunks; ++c) sk += partial_sk[c];
    double tr = 0.0;
    for (int x = 0; x < meff; ++x) tr += out[2 + x + (size_t)x * meff];
    out[0] = tr;
    out[1] = sk;
  }
}

// ------------------------------------------------------------------ leverage
struct LevArgs {
  TargetView tv;
  int d;
  const double* src;
  int m, r;
  double denom;
  const double* W;  // m x r col-major (device)
  bool w_in_smem;
  double* scores;
};

template <int D>
__global__ void __launch_bounds__(kNT) k_leverage(LevArgs A) {
  const int d = D ? D : A.d;
  const int m = A.m, r = A.r;
  const int m4 = ceil_to(m, 4);
  const int SN = frag_stride(m4);
  const int SW = frag_stride(r);
  const int NBR = ceil_to(r, 8) / 8;
  extern __shared__ __align__(16) double smem[];
  double* s_src = smem;
  double* s_t = s_src + (size_t)d * m;
  double* KN = s_t + (size_t)d * kTM;       // kTM x SN
  double* rowpart = KN + (size_t)kTM * SN;  // kTM x NBR
  double* sW = rowpart + (size_t)kTM * NBR; // m4 x SW (row-major) when w_in_smem
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < m * d; e += kNT) s_src[e] = A.src[e];
  for (int e = tid; e < kTM * SN; e += kNT) KN[e] = 0.0;
  if (A.w_in_smem)
    for (int e = tid; e < m4 * SW; e += kNT) {
      const int k = e / SW, n = e % SW;
      sW[e] = (k < m && n < r) ? A.W[k + (size_t)n * m] : 0.0;
    }
  __syncthreads();
  const int64_t ntiles = (A.tv.nt + kTM - 1) / kTM;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t t0 = tile * kTM;
    for (int e = tid; e < kTM * d; e += kNT) {
      const int t = e % kTM, k = e / kTM;
      s_t[t + k * kTM] = (t0 + t < A.tv.nt) ? tcoord(A.tv, t0 + t, k) : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < kTM * m; e += kNT) {
      const int t = e / m, j = e - t * m;
      double kv = 0.0;
      if (t0 + t < A.tv.nt) {
        double sq = 0.0;
        for (int k = 0; k < d; ++k) {
          const double diff = __dsub_rn(s_t[t + k * kTM], s_src[j + k * m]);
          sq = __dadd_rn(sq, __dmul_rn(diff, diff));
        }
        kv = gauss_exact(sq, A.denom);
      }
      KN[t * SN + j] = kv;
    }
    __syncthreads();
    for (int nb = warp; nb < NBR; nb += kNW) {
      double c[kTM / 8][2];
#pragma unroll
      for (int rb = 0; rb < kTM / 8; ++rb) c[rb][0] = c[rb][1] = 0.0;
      for (int k0 = 0; k0 < m4; k0 += 4) {
        const int kk = k0 + (lane & 3), nn = nb * 8 + (lane >> 2);
        const double b = A.w_in_smem ? sW[kk * SW + nn] : ((kk < m && nn < r) ? A.W[kk + (size_t)nn * m] : 0.0);
#pragma unroll
        for (int rb = 0; rb < kTM / 8; ++rb) {
          const double a = KN[(rb * 8 + (lane >> 2)) * SN + k0 + (lane & 3)];
          dmma884(c[rb][0], c[rb][1], a, b);
        }
      }
#pragma unroll
      for (int rb = 0; rb < kTM / 8; ++rb) {
        double q = c[rb][0] * c[rb][0] + c[rb][1] * c[rb][1];
        q += __shfl_xor_sync(0xffffffffu, q, 1);
        q += __shfl_xor_sync(0xffffffffu, q, 2);
        if ((lane & 3) == 0) rowpart[(rb * 8 + (lane >> 2)) * NBR + nb] = q;
      }
    }
    __syncthreads();
    if (tid < kTM && t0 + tid < A.tv.nt) {
      double s = 0.0;
      for (int nb = 0; nb < NBR; ++nb) s += rowpart[tid * NBR + nb];
      A.scores[t0 + tid] = s;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ gather rows
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

TargetView view(const kid_ctx* c) { return TargetView{c->tbase, c->tld, c->tidx, c->nt}; }

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
  const double denom = 2.0 * h * h;
  const size_t sm = sizeof(double) * c->m * c->d;
  if (sm > 200 * 1024) return fail(c, KID_E_DIM, "row_norms: m*d too large for shared memory");
  const int blocks = (int)std::min<int64_t>((c->nt + 255) / 256, (int64_t)c->sms * 8);
#define LAUNCH(DD)                                                                              \
  {                                                                                             \
    cudaFuncSetAttribute(k_row_norms<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k_row_norms<DD><<<blocks, 256, sm, c->stream>>>(view(c), c->d, c->src, c->m, denom, d_w);   \
  }
  KID_DISPATCH_D(c->d, LAUNCH)
#undef LAUNCH
  KID_LAUNCHED(c);
  return KID_OK;
}

// Gram of T = K (r == 0) or T = K_N - K_S P2 (r > 0, operands from kid_recon_prepare).
// d_out = [sumsq_T, sumsq_K, G (meff x meff)].
int gram_dev(kid_ctx* c, double h, int64_t r, uint32_t flags, double* d_out) {
  (void)flags;
  if (int rc = check_block(c, h)) return rc;
  const int m = (int)c->m, d = c->d;
  const int meff = (int)(m - r);
  if (meff < 1) {
    // full-rank skeleton: D == 0 exactly
    KID_CK(c, cudaMemsetAsync(d_out, 0, sizeof(double) * 2, c->stream));
    return KID_OK;
  }
  const int NBN = ceil_to(meff, 8) / 8;
  const int LG = NBN * 8;
  // upper-triangular 8x8 blocks, row-major (a <= b), grouped per warp
  std::vector<int2> blocks;
  for (int a = 0; a < NBN; ++a)
    for (int b = a; b < NBN; ++b) blocks.push_back(make_int2(a, b));
  const int nb = (int)blocks.size();
  int BPW = 4;
  for (int cand : {4, 8, 12, 16, 24}) {
    BPW = cand;
    if ((nb + kNW * cand - 1) / (kNW * cand) <= 1) break;
  }
  const int per_part = kNW * BPW;
  const int nparts = (nb + per_part - 1) / per_part;
  std::vector<int2> blist((size_t)nparts * per_part, make_int2(-1, -1));
  for (int p = 0; p < nparts; ++p)
    for (int w = 0; w < kNW; ++w)
      for (int s = 0; s < BPW; ++s) {
        // contiguous runs per warp keep the A fragment reused across consecutive slots
        const int g = p * per_part + w * BPW + s;
        if (g < nb) blist[((size_t)p * kNW + w) * BPW + s] = blocks[g];
      }
  const int r4 = ceil_to((int)r, 4);
  const int SS = frag_stride(r4 > 0 ? r4 : 4), SN = frag_stride(meff);
  const size_t smem = sizeof(double) * ((size_t)d * m + (size_t)d * kTM + (size_t)kTM * SS + (size_t)kTM * SN +
                                        (size_t)r4 * SN);
  if (smem > 220 * 1024) return fail(c, KID_E_DIM, "gram: tile does not fit shared memory (m, r too large)");
  const int64_t ntiles = (c->nt + kTM - 1) / kTM;
  int per_sm = smem <= 100 * 1024 ? 2 : 1;
  int nchunks = std::max(1, c->sms * per_sm / nparts);
  nchunks = (int)std::max<int64_t>(1, std::min<int64_t>(nchunks, ntiles));
  // scratch: blist | partial | partial_sk
  const size_t bl_bytes = sizeof(int2) * blist.size();
  const size_t part_bytes = sizeof(double) * (size_t)nchunks * LG * LG;
  char* base = (char*)scratch(c, bl_bytes + 256 + part_bytes + sizeof(double) * (nchunks + 8));
  if (!base) return KID_E_OOM;
  int2* d_blist = (int2*)base;
  double* partial = (double*)(base + ((bl_bytes + 255) / 256) * 256);
  double* partial_sk = partial + (size_t)nchunks * LG * LG;
  KID_CK(c, cudaMemcpyAsync(d_blist, blist.data(), bl_bytes, cudaMemcpyHostToDevice, c->stream));
  GramArgs A;
  A.tv = view(c);
  A.d = d;
  A.src = r > 0 ? c->src_perm : c->src;
  A.m = m;
  A.r = (int)r;
  A.meff = meff;
  A.denom = 2.0 * h * h;
  A.P2 = r > 0 ? c->P2 : nullptr;
  A.blist = d_blist;
  A.nparts = nparts;
  A.ntiles = ntiles;
  A.nchunks = nchunks;
  A.partial = partial;
  A.LG = LG;
  A.partial_sk = partial_sk;
  dim3 grid(nchunks, nparts);
#define LAUNCH_B(DD, BB)                                                                           \
  {                                                                                                \
    cudaFuncSetAttribute(k_gram<DD, BB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
    k_gram<DD, BB><<<grid, kNT, smem, c->stream>>>(A);                                             \
  }
#define LAUNCH(DD)                     \
  switch (BPW) {                       \
    case 4: LAUNCH_B(DD, 4); break;    \
    case 8: LAUNCH_B(DD, 8); break;    \
    case 12: LAUNCH_B(DD, 12); break;  \
    case 16: LAUNCH_B(DD, 16); break;  \
    default: LAUNCH_B(DD, 24); break;  \
  }
  KID_DISPATCH_D(d, LAUNCH)
#undef LAUNCH
#undef LAUNCH_B
  KID_LAUNCHED(c);
  k_gram_reduce<<<std::max(1, std::min(c->sms * 4, (meff * meff + 255) / 256)), 256, 0, c->stream>>>(
      partial, nchunks, LG, meff, partial_sk, d_out);
  KID_LAUNCHED(c);
  k_gram_finish<<<1, 32, 0, c->stream>>>(partial_sk, nchunks, meff, d_out);
  KID_LAUNCHED(c);
  return KID_OK;
}

int leverage_dev(kid_ctx* c, double h, const double* d_W, int64_t r, double* d_scores) {
  if (int rc = check_block(c, h)) return rc;
  if (r < 1 || r > c->m) return fail(c, KID_E_RANGE, "leverage: requires 1 <= r <= m");
  if (c->nt == 0) return KID_OK;
  const int m = (int)c->m, d = c->d, rr = (int)r;
  const int m4 = ceil_to(m, 4), SN = frag_stride(m4), SW = frag_stride(rr), NBR = ceil_to(rr, 8) / 8;
  size_t smem = sizeof(double) * ((size_t)d * m + (size_t)d * kTM + (size_t)kTM * SN + (size_t)kTM * NBR);
  const size_t wbytes = sizeof(double) * (size_t)m4 * SW;
  bool w_in_smem = smem + wbytes <= 200 * 1024;
  if (w_in_smem) smem += wbytes;
  if (smem > 220 * 1024) return fail(c, KID_E_DIM, "leverage: tile does not fit shared memory");
  LevArgs A{view(c), d, c->src, m, rr, 2.0 * h * h, d_W, w_in_smem, d_scores};
  const int64_t ntiles = (c->nt + kTM - 1) / kTM;
  const int blocks = (int)std::min<int64_t>(ntiles, (int64_t)c->sms * 2);
#define LAUNCH(DD)                                                                                \
  {                                                                                               \
    cudaFuncSetAttribute(k_leverage<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    k_leverage<DD><<<blocks, kNT, smem, c->stream>>>(A);                                          \
  }
  KID_DISPATCH_D(d, LAUNCH)
#undef LAUNCH
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

}  // namespace kid
