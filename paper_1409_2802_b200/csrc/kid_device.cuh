// kid_device.cuh -- device helpers shared by the FP64 passes (kid_passes.cu, kid_next.cu):
// the target view, tile geometry, the exp table, named barriers, the d dispatch.
// Each translation unit gets its own copy of the exp table (no relocatable device code).
#pragma once
#include <cmath>

#include "kid_internal.cuh"

namespace kid {
namespace {

// 2^(j/64), correctly rounded (generated from a 60-digit decimal evaluation; identical to
// exp2l(j/64) rounded to double). A static initializer: no upload, so no ordering question between
// a legacy-stream copy and the non-blocking stream the passes launch on.
__device__ const double c_exp2_tab[kExpTab] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0,
};

// shared table [j][lane] (kExpTabWords doubles) for exp_neg_fast(q, tab + lane)
__device__ __forceinline__ void stage_exp_table(double* tabr, int tid, int nthr) {
  for (int e = tid; e < kExpTabWords; e += nthr) tabr[e] = c_exp2_tab[e / kExpRep];
}

// kept for the call sites: the table needs no device-side initialisation any more
inline int init_device_tables() { return KID_OK; }

constexpr int kTM = 32;        // targets per tile (SYRK k-depth: 8 DMMA k-steps)
constexpr int kNT = 256;       // threads per CTA
constexpr int kST = kTM + 4;   // column-major tile stride

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

__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

inline TargetView view(const kid_ctx* c) { return TargetView{c->tbase, c->tld, c->tidx, c->nt}; }

inline int check_block(kid_ctx* c, double h) {
  if (!(h > 0.0)) return fail(c, KID_E_CONFIG, "Gaussian kernel requires bandwidth h > 0");
  if (!c->tbase || !c->src || c->m < 1) return fail(c, KID_E_ERROR, "no block: call kid_split or kid_set_block");
  return KID_OK;
}

}  // namespace
}  // namespace kid

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
