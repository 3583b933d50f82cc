// kid_device.cuh -- device helpers shared by the FP64 passes (kid_passes.cu, kid_next.cu):
// the target view, tile geometry, the exp table, named barriers, the d dispatch.
// Each translation unit gets its own copy of the exp table (no relocatable device code).
#pragma once
#include <cmath>

#include "kid_internal.cuh"

namespace kid {
namespace {

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
