// kid_gram2.cu -- K^T K for m > 128 (BASELINE c4: m = 256, c5: m = 512; lowrank.hpp:56-90, compress.hpp:156-159)
// as a two-phase kernel, one CTA per SM, no warp specialisation and no cluster exchange.
//
// The m x m Gram does not fit the registers of one SM (2080 upper 8 x 8 blocks at m = 512), so its blocks are
// grouped into parts (grid.y): column groups of 16 blocks (128 columns), one part per off-diagonal group pair
// (a 16 x 16 block square) and one per diagonal group (a triangle). A CTA owns one part over a chunk of target
// tiles. Per 32-target tile all 8 warps first evaluate the part's K columns by exp into a shared-memory tile
// (lane = target row, four independent chains; phase E), meet at one CTA barrier, then each warp runs the SYRK of
// its own two 4 x 4-block squares of the part on DMMA with the accumulators register-resident for the whole chunk
// (phase S: 16 fragment loads per 32 DMMAs; a triangle's 10 squares are spread 3 / 3 / 2 / 2 over the SM
// sub-partitions). The K tile is double-buffered, so the barrier of tile t also frees
// the buffer of tile t - 1 and one barrier per tile suffices. DFMA (exp) and DMMA share the FP64 datapath, so
// running the two phases back to back loses nothing against overlapping them; what the warp-specialised cluster
// kernel (k_fused, Gram mode) loses to its eval -> MMA hand-offs and its DSMEM exchange of D halves is gone.
// K never reaches HBM; partial Grams are reduced over the chunks in a fixed order (k_fx_reduce).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <vector>

#include "kid_fused.cuh"

namespace kid {
namespace {

constexpr int kG2W = 8, kG2T = kG2W * 32;  // warps / threads per CTA
constexpr int kG2GS = 16;                  // blocks per column group
constexpr int kG2H = 4;                    // a warp tile: two squares of kG2H x kG2H blocks
constexpr int kG2WL = 8;                   // shorts per warp: (ra0, nra, cb0, ncb) x 2 squares
constexpr int kG2Meta = 4;                 // ints per part: columns (padded), blocks, count ||K||^2 here

struct G2Args {
  TargetView tv;
  int d;
  double cscale;
  int64_t ntiles;
  int nchunks, nparts;
  const double* img;   // [part][d][ncolp_max] scaled source coordinates of the part's columns (padding at +far)
  int ncolp_max;
  const int* meta;     // [part][kG2Meta]
  const short* wlist;  // [part][kG2W][2][4]: ra0, nra, cb0, ncb of each square in local blocks (nra = 0: none)
  const int* gblk;     // [part][2 kG2GS]: global block of each local block
  double* partial;     // [chunk][LG][LG]
  int LG;
  double* psk;         // [chunk][part] ||K||^2 partials
  double* ptr;         // [chunk][part] trace partials
};

__device__ __forceinline__ void g2_cp8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void g2_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void g2_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <int D>
__global__ void __launch_bounds__(kG2T, 1) k_gram2(const __grid_constant__ G2Args A) {
  const int d = D ? D : A.d;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int part = blockIdx.y, chunk = blockIdx.x;
  const int* meta = A.meta + (size_t)part * kG2Meta;
  const int ncolp = meta[0], nblk = meta[1], count = meta[2];
  extern __shared__ __align__(16) double gsm[];
  double* s_tab = gsm;                                   // exp table [64][16]
  double* s_src = s_tab + kFTab;                         // [d][ncolp_max]
  double* Kt = s_src + (size_t)d * A.ncolp_max;          // 2 x [ncolp_max][kST]
  constexpr bool kReg = D > 0 && D <= 16;                // coordinates of the tile held in registers
  double* crd = Kt + 2 * (size_t)A.ncolp_max * kST;      // 2 x [d][32]: raw target coordinates, one tile ahead
  __shared__ double red_sk[kG2W], red_tr[kG2W];
  __shared__ __align__(8) uint64_t img_bar;

  for (int e = tid; e < kFTab; e += kG2T) s_tab[e] = c_exp2_tab[e / kFRep];
  if (tid == 0) {  // the part's source image by one TMA bulk copy
    mbar_init(smem_u32(&img_bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t bytes = (uint32_t)(d * A.ncolp_max) * 8u;
    mbar_expect(smem_u32(&img_bar), bytes);
    tma_bulk_g2s(smem_u32(s_src), A.img + (size_t)part * d * A.ncolp_max, bytes, smem_u32(&img_bar));
  }
  for (int e = tid; e < 2 * A.ncolp_max * kST; e += kG2T) Kt[e] = 0.0;
  __syncthreads();
  mbar_wait(smem_u32(&img_bar), 0);

  const short* wl = A.wlist + ((size_t)part * kG2W + w) * kG2WL;
  const int fr = lane >> 2, fk = lane & 3;
  // fragment bases of the warp's row / column blocks (out-of-range slots clamp to the last block: computed,
  // never written)
  int ra0[2], nra[2], cb0[2], ncb[2], ao[2][kG2H], bo[2][kG2H];
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    ra0[hh] = wl[4 * hh], nra[hh] = wl[4 * hh + 1], cb0[hh] = wl[4 * hh + 2], ncb[hh] = wl[4 * hh + 3];
#pragma unroll
    for (int i = 0; i < kG2H; ++i) {
      ao[hh][i] = min(ra0[hh] + i, nblk - 1) * 8 * kST;
      bo[hh][i] = min(cb0[hh] + i, nblk - 1) * 8 * kST;
    }
  }
  double acc[2][kG2H][kG2H][2];
#pragma unroll
  for (int hh = 0; hh < 2; ++hh)
#pragma unroll
    for (int i = 0; i < kG2H; ++i)
#pragma unroll
      for (int j = 0; j < kG2H; ++j) acc[hh][i][j][0] = acc[hh][i][j][1] = 0.0;
  double skv[4] = {0.0, 0.0, 0.0, 0.0};  // ||K||^2 in four independent chains
  const double* tabl = s_tab + (lane & (kFRep - 1));
  const int ngroups = ncolp / 4;
  const int64_t tile_lo = A.ntiles * chunk / A.nchunks, tile_hi = A.ntiles * (chunk + 1) / A.nchunks;
  // target coordinates stream through a 2-slot shared-memory ring by cp.async, issued one tile ahead (warp w
  // copies coordinates w, w + 8, ...); the target index of each copy is loaded one tile before that, so
  // neither latency is exposed
  const int64_t nt = A.tv.nt;
  auto row_of = [&](int64_t tl) -> int64_t {
    const int64_t row = tl * kTM + lane;
    return (tl < tile_hi && row < nt) ? (A.tv.idx ? A.tv.idx[row] : row) : -1;
  };
  auto issue_crd = [&](int buf, int64_t prow) {
    if (prow >= 0)
      for (int k = w; k < d; k += kG2W)
        g2_cp8(crd + ((size_t)buf * d + k) * kTM + lane, A.tv.base + prow + (int64_t)k * A.tv.ld);
    g2_commit();
  };
  issue_crd(0, row_of(tile_lo));
  int64_t prow_next = row_of(tile_lo + 1);
  g2_wait_all();
  __syncthreads();
  int it = 0;
  for (int64_t tl = tile_lo; tl < tile_hi; ++tl, ++it) {
    const int buf = it & 1;
    issue_crd(buf ^ 1, prow_next);
    prow_next = row_of(tl + 2);
    // ---- phase E: this warp's 4-column groups of the part's K tile (rows past the end sit at -far: K == 0)
    const bool valid = tl * kTM + lane < nt;
    constexpr int DR = kReg ? D : 1;
    double tc[DR];
    if constexpr (kReg) {
#pragma unroll
      for (int k = 0; k < D; ++k) tc[k] = valid ? crd[((size_t)buf * D + k) * kTM + lane] * A.cscale : -kFar;
    }
    const double* cr = crd + (size_t)buf * d * kTM + lane;
    double* kt = Kt + (size_t)buf * A.ncolp_max * kST;
    for (int g = w; g < ngroups; g += kG2W) {
      double kv[4] = {0.0, 0.0, 0.0, 0.0};
      const double* ss0 = s_src + 4 * g;
#pragma unroll
      for (int k = 0; k < (D ? D : 1); ++k) {
        for (int kk = k; kk < (D ? k + 1 : d); ++kk) {
          double t;
          if constexpr (kReg) t = tc[kk];
          else t = valid ? cr[kk * kTM] * A.cscale : -kFar;
          const double* ss = ss0 + (size_t)kk * A.ncolp_max;
          const double a0 = t - ss[0], a1 = t - ss[1], a2 = t - ss[2], a3 = t - ss[3];
          kv[0] = fma(a0, a0, kv[0]);
          kv[1] = fma(a1, a1, kv[1]);
          kv[2] = fma(a2, a2, kv[2]);
          kv[3] = fma(a3, a3, kv[3]);
        }
      }
      exp_neg_fast_n<4, kFRep>(kv, tabl);
#pragma unroll
      for (int v = 0; v < 4; ++v) kt[(4 * g + v) * kST + lane] = kv[v];
      if (count) {
#pragma unroll
        for (int v = 0; v < 4; ++v) skv[v] = fma(kv[v], kv[v], skv[v]);
      }
    }
    g2_wait_all();    // the next tile's coordinates have landed (this thread's copies; the barrier publishes them)
    __syncthreads();  // tile `it` is complete; every warp is past its SYRK of tile it - 1 (frees that buffer)
    // ---- phase S: G[rows of the warp, columns of the warp] += K_rows^T K_cols over the 32 targets
    const double* col = kt + fr * kST + fk;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      if (nra[hh] == 0) continue;
#pragma unroll 2
      for (int kk = 0; kk < kTM / 4; ++kk) {
        double a[kG2H], b[kG2H];
#pragma unroll
        for (int i = 0; i < kG2H; ++i) a[i] = col[ao[hh][i] + kk * 4];
#pragma unroll
        for (int j = 0; j < kG2H; ++j) b[j] = col[bo[hh][j] + kk * 4];
#pragma unroll
        for (int i = 0; i < kG2H; ++i)
#pragma unroll
          for (int j = 0; j < kG2H; ++j) dmma884(acc[hh][i][j][0], acc[hh][i][j][1], a[i], b[j]);
      }
    }
  }
  // ---- the warp's blocks -> partial[chunk] (upper blocks in global block coordinates), trace, ||K||^2
  double trd = 0.0;
  {
    double* G = A.partial + (size_t)chunk * A.LG * A.LG;
    const int* gb = A.gblk + (size_t)part * 2 * kG2GS;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh)
#pragma unroll
      for (int i = 0; i < kG2H; ++i)
#pragma unroll
        for (int j = 0; j < kG2H; ++j) {
          if (i >= nra[hh] || j >= ncb[hh]) continue;
          const int ga = gb[ra0[hh] + i], gbk = gb[cb0[hh] + j];
          if (ga > gbk) continue;
          const int row = ga * 8 + fr, colx = gbk * 8 + 2 * fk;
          G[row + (size_t)colx * A.LG] = acc[hh][i][j][0];
          G[row + (size_t)(colx + 1) * A.LG] = acc[hh][i][j][1];
          if (row == colx) trd += acc[hh][i][j][0];
          if (row == colx + 1) trd += acc[hh][i][j][1];
        }
  }
  trd = warp_sum(trd);
  const double sk = warp_sum((skv[0] + skv[1]) + (skv[2] + skv[3]));
  if (lane == 0) {
    red_tr[w] = trd;
    red_sk[w] = sk;
  }
  __syncthreads();
  if (tid == 0) {
    double t = 0.0, k2 = 0.0;
    for (int ww = 0; ww < kG2W; ++ww) {
      t += red_tr[ww];
      k2 += red_sk[ww];
    }
    A.ptr[(size_t)chunk * A.nparts + part] = t;
    A.psk[(size_t)chunk * A.nparts + part] = k2;
  }
}

}  // namespace

// K^T K of the current block by k_gram2; d_out = [tr, ||K||_F^2, G (m x m col-major)]. Returns 1 when the
// part's tile buffers do not fit shared memory (d = 64: the caller takes the cluster kernel).
int gram2_dev(kid_ctx* c, double h, double* d_out) {
  if (int rc = check_block(c, h)) return rc;
  const int m = (int)c->m, d = c->d;
  const std::vector<double>& sh = c->src_host;
  if (sh.size() != (size_t)m * d) return fail(c, KID_E_ERROR, "gram pass: host copy of the sources is stale");
  const int NB = (m + 7) / 8, LG = NB * 8;
  const int ng = (NB + kG2GS - 1) / kG2GS;
  struct Part { std::vector<int> blocks; int na, nb; bool diag; };
  std::vector<Part> parts;
  auto grp = [&](int gi) {
    std::vector<int> v;
    for (int b = gi * kG2GS; b < std::min(NB, (gi + 1) * kG2GS); ++b) v.push_back(b);
    return v;
  };
  for (int i = 0; i < ng; ++i)
    for (int j = i + 1; j < ng; ++j) {
      Part p;
      std::vector<int> gi = grp(i), gj = grp(j);
      p.na = (int)gi.size(), p.nb = (int)gj.size(), p.diag = false;
      p.blocks = gi;
      p.blocks.insert(p.blocks.end(), gj.begin(), gj.end());
      parts.push_back(p);
    }
  for (int i = 0; i < ng; ++i) {
    Part p;
    p.blocks = grp(i);
    p.na = (int)p.blocks.size(), p.nb = 0, p.diag = true;
    parts.push_back(p);
  }
  const int nparts = (int)parts.size();
  int ncolp_max = 0;
  for (auto& p : parts) ncolp_max = std::max(ncolp_max, (int)p.blocks.size() * 8);
  const size_t smem = sizeof(double) * ((size_t)kFTab + (size_t)d * ncolp_max + 2 * (size_t)ncolp_max * kST +
                                        2 * (size_t)d * kTM) + 64;
  if (smem > 227 * 1024 - 1024) return 1;
  const double cs = std::sqrt(1.0 / (2.0 * h * h));
  std::vector<double> img((size_t)nparts * d * ncolp_max, kFar);
  std::vector<int> meta((size_t)nparts * kG2Meta, 0), gblk((size_t)nparts * 2 * kG2GS, 0);
  std::vector<short> wlist((size_t)nparts * kG2W * kG2WL, 0);
  for (int pi = 0; pi < nparts; ++pi) {
    const Part& p = parts[pi];
    const int nblk = (int)p.blocks.size();
    meta[(size_t)pi * kG2Meta + 0] = nblk * 8;
    meta[(size_t)pi * kG2Meta + 1] = nblk;
    meta[(size_t)pi * kG2Meta + 2] = p.diag ? 1 : 0;  // every column lies in exactly one diagonal part
    for (int l = 0; l < nblk; ++l) {
      gblk[(size_t)pi * 2 * kG2GS + l] = p.blocks[l];
      for (int cc = 0; cc < 8; ++cc) {
        const int gc = p.blocks[l] * 8 + cc;
        if (gc < m)
          for (int k = 0; k < d; ++k) img[((size_t)pi * d + k) * ncolp_max + l * 8 + cc] = sh[(size_t)k * m + gc] * cs;
      }
    }
    // warp tiles: squares of 4 x 4 blocks, up to two per warp. Off-diagonal part: rows = group i, columns =
    // group j; triangle: rows and columns the same group, only the squares on or above the diagonal. Squares go
    // to the warp whose SM sub-partition (warp % 4) carries the least so far.
    std::vector<std::array<int, 4>> sq;
    if (!p.diag) {
      for (int r0 = 0; r0 < p.na; r0 += kG2H)
        for (int c0 = 0; c0 < p.nb; c0 += kG2H)
          sq.push_back({r0, std::min(kG2H, p.na - r0), p.na + c0, std::min(kG2H, p.nb - c0)});
    } else {
      for (int r0 = 0; r0 < p.na; r0 += kG2H)
        for (int c0 = r0; c0 < p.na; c0 += kG2H)
          sq.push_back({r0, std::min(kG2H, p.na - r0), c0, std::min(kG2H, p.na - c0)});
    }
    if ((int)sq.size() > 2 * kG2W) return fail(c, KID_E_DIM, "gram pass: more warp tiles than warp slots");
    int nsq[kG2W] = {0}, smsp[4] = {0};
    for (const auto& t : sq) {
      int best = -1;
      for (int ww = 0; ww < kG2W; ++ww) {
        if (nsq[ww] >= 2) continue;
        if (best < 0 || smsp[ww % 4] < smsp[best % 4] || (smsp[ww % 4] == smsp[best % 4] && nsq[ww] < nsq[best])) best = ww;
      }
      for (int q = 0; q < 4; ++q) wlist[((size_t)pi * kG2W + best) * kG2WL + 4 * nsq[best] + q] = (short)t[q];
      ++nsq[best];
      ++smsp[best % 4];
    }
  }
  const int64_t nt = c->nt;
  const int64_t ntiles = (nt + kTM - 1) / kTM;
  const int nchunks = (int)std::max<int64_t>(1, std::min<int64_t>(c->sms, ntiles));
  const int nslots = nchunks * nparts;
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t b_img = al(sizeof(double) * img.size()), b_meta = al(sizeof(int) * meta.size()),
               b_wl = al(sizeof(short) * wlist.size()), b_gb = al(sizeof(int) * gblk.size());
  const size_t b_part = al(sizeof(double) * (size_t)nchunks * LG * LG), b_sl = al(sizeof(double) * nslots);
  const size_t b_hdr = b_img + b_meta + b_wl + b_gb;
  char* base = (char*)scratch(c, b_hdr + b_part + 2 * b_sl);
  if (!base) return KID_E_OOM;
  {
    std::vector<char> hb(b_hdr, 0);
    std::memcpy(hb.data(), img.data(), sizeof(double) * img.size());
    std::memcpy(hb.data() + b_img, meta.data(), sizeof(int) * meta.size());
    std::memcpy(hb.data() + b_img + b_meta, wlist.data(), sizeof(short) * wlist.size());
    std::memcpy(hb.data() + b_img + b_meta + b_wl, gblk.data(), sizeof(int) * gblk.size());
    KID_CK(c, cudaMemcpyAsync(base, hb.data(), b_hdr, cudaMemcpyHostToDevice, c->stream));
    KID_CK(c, cudaStreamSynchronize(c->stream));  // pageable staging buffer goes out of scope
  }
  G2Args A{};
  A.tv = view(c);
  A.d = d;
  A.cscale = cs;
  A.ntiles = ntiles;
  A.nchunks = nchunks;
  A.nparts = nparts;
  A.img = (const double*)base;
  A.ncolp_max = ncolp_max;
  A.meta = (const int*)(base + b_img);
  A.wlist = (const short*)(base + b_img + b_meta);
  A.gblk = (const int*)(base + b_img + b_meta + b_wl);
  A.partial = (double*)(base + b_hdr);
  A.LG = LG;
  A.psk = (double*)(base + b_hdr + b_part);
  A.ptr = (double*)(base + b_hdr + b_part + b_sl);
  c->last_kernel = "k_gram2";
  const dim3 grid(nchunks, nparts, 1);
#define G2_LAUNCH(DD)                                                                              \
  {                                                                                                \
    cudaFuncSetAttribute(k_gram2<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
    k_gram2<DD><<<grid, kG2T, smem, c->stream>>>(A);                                               \
  }
  prof_begin(c);
  switch (d) {
    case 8: G2_LAUNCH(8) break;
    case 16: G2_LAUNCH(16) break;
    default: G2_LAUNCH(0) break;
  }
  prof_end(c);
#undef G2_LAUNCH
  KID_LAUNCHED(c);
  return launch_fx_reduce(c, A.partial, nchunks, LG, m, A.ptr, A.psk, nslots, d_out);
}

}  // namespace kid
