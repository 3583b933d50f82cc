// kid_resid3.cu -- the fused residual pass (compress.hpp:141-154) for blocks that fit one SM with 33 .. 128
// residual columns (m <= ~256 with r + n columns in one tile: BASELINE c1 - c3 at low and mid skeleton ranks), as
// a three-phase kernel: one CTA per SM, 12 warps, no warp specialisation.
//
// Per 64-target tile: (E) all warps evaluate K(T_tile, [S_skel | S_rest]) by exp into a shared-memory tile (lane =
// target row, four independent chains per 4-column group); one CTA barrier; (G) D = K_N - K_S P2 on DMMA in place
// over the K_N columns -- a unit is one 8-column block x two 8-row blocks, accumulator initialised from K_N, A
// fragments from K_S, B fragments from -P2 in shared memory; one CTA barrier; (S) G += D^T D on DMMA over 8 x 16
// warp tiles of the upper triangle, accumulators register-resident for the CTA's whole chunk of tiles. The tile
// is double-buffered, so two barriers per tile suffice. DFMA and DMMA share the FP64 datapath, so running the
// phases back to back loses nothing against overlapping them (kid_gram2.cu); the eval -> MMA named-barrier
// hand-offs and the unsplittable eval items of the warp-specialised k_gram are gone.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "kid_fused.cuh"

namespace kid {
namespace {

constexpr int kR3W = 12, kR3T = kR3W * 32;  // warps / threads per CTA
constexpr int kR3M = 64, kR3S = kR3M + 4;   // targets per tile (two 32-row halves: longer phases per barrier), column stride
constexpr int kR3TPW = 6;                   // 8 x 16 SYRK tiles per warp (72 tiles at 16 column blocks)

struct R3Args {
  TargetView tv;
  int d;
  double cscale;
  int64_t ntiles;
  int nchunks;
  int r4, NB, ncol, spn;  // skeleton columns (padded to 4), D column blocks, tile columns, P2 row stride
  const double* img;      // [d][ncol] scaled sources (skeleton first; padding at +far), then -P2 [r4][spn]
  const short* tiles;     // [kR3W][1 + 2 kR3TPW]: count, (a, b0) block pairs of each warp's SYRK tiles
  double* partial;        // [chunk][LG][LG]
  int LG;
  double* psk;            // [chunk] ||K||^2 partials
  double* ptr;            // [chunk] trace partials
};

__device__ __forceinline__ void r3_cp8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void r3_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void r3_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <int D>
__global__ void __launch_bounds__(kR3T, 1) k_resid3(const __grid_constant__ R3Args A) {
  const int d = D ? D : A.d;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int chunk = blockIdx.x;
  const int r4 = A.r4, NB = A.NB, ncol = A.ncol, spn = A.spn;
  extern __shared__ __align__(16) double rsm[];
  double* s_tab = rsm;                              // exp table [64][16]
  double* s_src = s_tab + kFTab;                    // [d][ncol]
  double* sP = s_src + (size_t)d * ncol;            // [r4][spn]: -P2
  double* Kt = sP + (size_t)r4 * spn;               // 2 x [ncol][kR3S]
  double* crd = Kt + 2 * (size_t)ncol * kR3S;       // 2 x [d][64] raw target coordinates, one tile ahead
  constexpr bool kReg = D > 0 && D <= 16;
  __shared__ double red_sk[kR3W], red_tr[kR3W];
  __shared__ __align__(8) uint64_t img_bar;

  for (int e = tid; e < kFTab; e += kR3T) s_tab[e] = c_exp2_tab[e / kFRep];
  if (tid == 0) {  // sources and -P2 by one TMA bulk copy (contiguous in the image)
    mbar_init(smem_u32(&img_bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t bytes = (uint32_t)(d * ncol + r4 * spn) * 8u;
    mbar_expect(smem_u32(&img_bar), bytes);
    tma_bulk_g2s(smem_u32(s_src), A.img, bytes, smem_u32(&img_bar));
  }
  for (int e = tid; e < 2 * ncol * kR3S; e += kR3T) Kt[e] = 0.0;
  __syncthreads();
  mbar_wait(smem_u32(&img_bar), 0);

  const int fr = lane >> 2, fk = lane & 3;
  // SYRK tiles of this warp: (a, b0) -> blocks (a, b0) and (a, b0 + 1); a second block past NB is padding
  const short* tl_ = A.tiles + (size_t)w * (1 + 2 * kR3TPW);
  const int ntl = tl_[0];
  int ao[kR3TPW], bo[kR3TPW], b1[kR3TPW];
#pragma unroll
  for (int q = 0; q < kR3TPW; ++q) {
    const int a = q < ntl ? tl_[1 + 2 * q] : 0, b0 = q < ntl ? tl_[2 + 2 * q] : 0;
    ao[q] = a * 8 * kR3S;
    bo[q] = b0 * 8 * kR3S;
    b1[q] = (b0 + 1 < NB ? b0 + 1 : b0) * 8 * kR3S;  // a second block past the last one: recomputed, never written
  }
  double g[kR3TPW][2][2];
#pragma unroll
  for (int q = 0; q < kR3TPW; ++q) g[q][0][0] = g[q][0][1] = g[q][1][0] = g[q][1][1] = 0.0;
  double sk = 0.0;
  const double* tabl = s_tab + (lane & (kFRep - 1));
  const int nitems = 2 * (ncol / 4), nunits = 4 * NB, nks = r4 / 4;  // (4-column group, row half); (column block, row-block pair)
  const int64_t tile_lo = A.ntiles * chunk / A.nchunks, tile_hi = A.ntiles * (chunk + 1) / A.nchunks;
  const int64_t nt = A.tv.nt;
  auto row_of = [&](int64_t tl, int half) -> int64_t {
    const int64_t row = tl * kR3M + half * 32 + lane;
    return (tl < tile_hi && row < nt) ? (A.tv.idx ? A.tv.idx[row] : row) : -1;
  };
  auto issue_crd = [&](int buf, int64_t p0, int64_t p1) {
    for (int k = w; k < d; k += kR3W) {
      double* dst = crd + ((size_t)buf * d + k) * kR3M + lane;
      if (p0 >= 0) r3_cp8(dst, A.tv.base + p0 + (int64_t)k * A.tv.ld);
      if (p1 >= 0) r3_cp8(dst + 32, A.tv.base + p1 + (int64_t)k * A.tv.ld);
    }
    r3_commit();
  };
  issue_crd(0, row_of(tile_lo, 0), row_of(tile_lo, 1));
  int64_t pn0 = row_of(tile_lo + 1, 0), pn1 = row_of(tile_lo + 1, 1);
  r3_wait_all();
  __syncthreads();
  int it = 0;
  for (int64_t tl = tile_lo; tl < tile_hi; ++tl, ++it) {
    const int buf = it & 1;
    issue_crd(buf ^ 1, pn0, pn1);
    pn0 = row_of(tl + 2, 0);
    pn1 = row_of(tl + 2, 1);
    // ---- phase E: K(T_tile, all columns), one (4-column group, 32-row half) item at a time; rows past the end
    // sit at -far (every entry exactly 0)
    double* kt = Kt + (size_t)buf * ncol * kR3S;
    for (int item = w; item < nitems; item += kR3W) {
      const int gq = item >> 1, half = item & 1;
      const bool valid = tl * kR3M + half * 32 + lane < nt;
      const double* cr = crd + (size_t)buf * d * kR3M + half * 32 + lane;
      constexpr int DR = kReg ? D : 1;
      double tc[DR];
      if constexpr (kReg) {
#pragma unroll
        for (int k = 0; k < D; ++k) tc[k] = valid ? cr[k * kR3M] * A.cscale : -kFar;
      }
      double kv[4] = {0.0, 0.0, 0.0, 0.0};
      const double* ss0 = s_src + 4 * gq;
#pragma unroll
      for (int k = 0; k < (D ? D : 1); ++k) {
        for (int kk = k; kk < (D ? k + 1 : d); ++kk) {
          double t;
          if constexpr (kReg) t = tc[kk];
          else t = valid ? cr[kk * kR3M] * A.cscale : -kFar;
          const double* ss = ss0 + (size_t)kk * ncol;
          const double a0 = t - ss[0], a1 = t - ss[1], a2 = t - ss[2], a3 = t - ss[3];
          kv[0] = fma(a0, a0, kv[0]);
          kv[1] = fma(a1, a1, kv[1]);
          kv[2] = fma(a2, a2, kv[2]);
          kv[3] = fma(a3, a3, kv[3]);
        }
      }
      exp_neg_fast_n<4, kFRep>(kv, tabl);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        kt[(4 * gq + v) * kR3S + half * 32 + lane] = kv[v];
        sk = fma(kv[v], kv[v], sk);
      }
    }
    r3_wait_all();
    __syncthreads();  // K tile complete (and the next tile's coordinates published)
    // ---- phase G: D = K_N + K_S (-P2), in place: unit = (column block cb, row-block pair rp)
    for (int u = w; u < nunits; u += kR3W) {
      const int cb = u >> 2, rp = u & 3;
      double* cp = kt + (size_t)(r4 + cb * 8 + 2 * fk) * kR3S + rp * 16 + fr;
      double c00 = cp[0], c01 = cp[kR3S], c10 = cp[8], c11 = cp[kR3S + 8];
      const double* ap = kt + fk * kR3S + rp * 16 + fr;
      const double* bp = sP + fk * spn + cb * 8 + fr;
#pragma unroll 4
      for (int ks = 0; ks < nks; ++ks) {
        const double a0 = ap[ks * 4 * kR3S], a1 = ap[ks * 4 * kR3S + 8], b = bp[ks * 4 * spn];
        dmma884(c00, c01, a0, b);
        dmma884(c10, c11, a1, b);
      }
      cp[0] = c00;
      cp[kR3S] = c01;
      cp[8] = c10;
      cp[kR3S + 8] = c11;
    }
    __syncthreads();  // D tile complete
    // ---- phase S: G += D^T D over this warp's 8 x 16 tiles (16 k-steps of 4 targets)
    const double* col = kt + (size_t)r4 * kR3S + fr * kR3S + fk;
#pragma unroll 2
    for (int kk = 0; kk < kR3M / 4; ++kk) {
#pragma unroll
      for (int q = 0; q < kR3TPW; ++q) {
        if (q >= ntl) break;
        const double a = col[ao[q] + kk * 4], f0 = col[bo[q] + kk * 4], f1 = col[b1[q] + kk * 4];
        dmma884(g[q][0][0], g[q][0][1], a, f0);
        dmma884(g[q][1][0], g[q][1][1], a, f1);
      }
    }
  }
  // ---- the warp's blocks -> partial[chunk]; trace; ||K||^2
  double trd = 0.0;
  {
    double* G = A.partial + (size_t)chunk * A.LG * A.LG;
#pragma unroll
    for (int q = 0; q < kR3TPW; ++q) {
      if (q >= ntl) break;
      const int a = tl_[1 + 2 * q];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int b = tl_[2 + 2 * q] + e;
        if (b >= NB) continue;
        const int row = a * 8 + fr, colx = b * 8 + 2 * fk;
        G[row + (size_t)colx * A.LG] = g[q][e][0];
        G[row + (size_t)(colx + 1) * A.LG] = g[q][e][1];
        if (row == colx) trd += g[q][e][0];
        if (row == colx + 1) trd += g[q][e][1];
      }
    }
  }
  trd = warp_sum(trd);
  sk = warp_sum(sk);
  if (lane == 0) {
    red_tr[w] = trd;
    red_sk[w] = sk;
  }
  __syncthreads();
  if (tid == 0) {
    double t = 0.0, k2 = 0.0;
    for (int ww = 0; ww < kR3W; ++ww) {
      t += red_tr[ww];
      k2 += red_sk[ww];
    }
    A.ptr[chunk] = t;
    A.psk[chunk] = k2;
  }
}

}  // namespace

// The residual pass of the prepared (skeleton, P) by k_resid3; d_out = [||D||_F^2, ||K||_F^2, D^T D (n x n)].
// Returns 1 when the shape does not qualify (the caller takes k_gram / the cluster kernel).
int resid3_dev(kid_ctx* c, double h, double* d_out) {
  const int m = (int)c->m, d = c->d, r = (int)c->r, n = m - r;
  if (r < 1 || n < 1) return 1;
  const int NB = (n + 7) / 8, r4 = ceil_to(r, 4);
  if (NB > 16) return 1;
  const std::vector<double>& sh = c->src_perm_host;
  if (sh.size() != (size_t)m * d) return fail(c, KID_E_ERROR, "residual pass: host copy of the sources is stale");
  if (c->P2_host.size() < (size_t)r * frag_stride(n)) return fail(c, KID_E_ERROR, "residual pass: host copy of P2 is stale");
  const int ncol = r4 + NB * 8, spn = frag_stride(NB * 8);
  const size_t smem = sizeof(double) * ((size_t)kFTab + (size_t)d * ncol + (size_t)r4 * spn + 2 * (size_t)ncol * kR3S +
                                        2 * (size_t)d * kR3M) + 64;
  if (smem > 227 * 1024 - 1024) return 1;
  // SYRK tiles (a, b0) of the upper triangle, row-major, dealt round-robin to the warps
  std::vector<short> tiles((size_t)kR3W * (1 + 2 * kR3TPW), 0);
  {
    int t = 0;
    for (int a = 0; a < NB; ++a)
      for (int b0 = a; b0 < NB; b0 += 2, ++t) {
        short* e = &tiles[(size_t)(t % kR3W) * (1 + 2 * kR3TPW)];
        if (e[0] >= kR3TPW) return 1;
        e[1 + 2 * e[0]] = (short)a;
        e[2 + 2 * e[0]] = (short)b0;
        ++e[0];
      }
  }
  const double cs = std::sqrt(1.0 / (2.0 * h * h));
  std::vector<double> img((size_t)d * ncol + (size_t)r4 * spn, 0.0);
  for (int k = 0; k < d; ++k) {
    for (int j = 0; j < r4; ++j) img[(size_t)k * ncol + j] = j < r ? sh[(size_t)k * m + j] * cs : kFar;
    for (int j = 0; j < NB * 8; ++j) img[(size_t)k * ncol + r4 + j] = j < n ? sh[(size_t)k * m + r + j] * cs : kFar;
  }
  double* Pi = img.data() + (size_t)d * ncol;
  for (int k = 0; k < r; ++k)
    for (int j = 0; j < n; ++j) Pi[(size_t)k * spn + j] = -c->P2_host[(size_t)k * frag_stride(n) + j];
  const int64_t ntiles = (c->nt + kR3M - 1) / kR3M;
  const int nchunks = (int)std::max<int64_t>(1, std::min<int64_t>(c->sms, ntiles));
  const int LG = NB * 8;
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t b_img = al(sizeof(double) * img.size()), b_tl = al(sizeof(short) * tiles.size());
  const size_t b_part = al(sizeof(double) * (size_t)nchunks * LG * LG), b_sl = al(sizeof(double) * nchunks);
  char* base = (char*)scratch(c, b_img + b_tl + b_part + 2 * b_sl);
  if (!base) return KID_E_OOM;
  {
    std::vector<char> hb(b_img + b_tl, 0);
    std::memcpy(hb.data(), img.data(), sizeof(double) * img.size());
    std::memcpy(hb.data() + b_img, tiles.data(), sizeof(short) * tiles.size());
    KID_CK(c, cudaMemcpyAsync(base, hb.data(), hb.size(), cudaMemcpyHostToDevice, c->stream));
    KID_CK(c, cudaStreamSynchronize(c->stream));  // pageable staging buffer goes out of scope
  }
  R3Args A{};
  A.tv = view(c);
  A.d = d;
  A.cscale = cs;
  A.ntiles = ntiles;
  A.nchunks = nchunks;
  A.r4 = r4;
  A.NB = NB;
  A.ncol = ncol;
  A.spn = spn;
  A.img = (const double*)base;
  A.tiles = (const short*)(base + b_img);
  A.partial = (double*)(base + b_img + b_tl);
  A.LG = LG;
  A.psk = (double*)(base + b_img + b_tl + b_part);
  A.ptr = (double*)(base + b_img + b_tl + b_part + b_sl);
  c->last_kernel = "k_resid3";
#define R3_LAUNCH(DD)                                                                              \
  {                                                                                                \
    cudaFuncSetAttribute(k_resid3<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
    k_resid3<DD><<<nchunks, kR3T, smem, c->stream>>>(A);                                           \
  }
  prof_begin(c);
  switch (d) {
    case 1: R3_LAUNCH(1) break;
    case 2: R3_LAUNCH(2) break;
    case 3: R3_LAUNCH(3) break;
    case 4: R3_LAUNCH(4) break;
    case 5: R3_LAUNCH(5) break;
    case 8: R3_LAUNCH(8) break;
    case 16: R3_LAUNCH(16) break;
    default: R3_LAUNCH(0) break;
  }
  prof_end(c);
#undef R3_LAUNCH
  KID_LAUNCHED(c);
  return launch_fx_reduce(c, A.partial, nchunks, LG, n, A.ptr, A.psk, nchunks, d_out);
}

}  // namespace kid
