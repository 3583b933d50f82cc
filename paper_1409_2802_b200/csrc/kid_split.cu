// kid_split.cu -- pass 1: the well-separatedness filter (split_sources_targets,
// /root/reference/proj/include/kernid/geometry.hpp:29-65) as HBM-streaming kernels.
//
//   (a) sample bound: exact distances of a strided sample of S points; the n-th smallest
//       sample key T bounds the global n-th smallest key from above (any n points at
//       distance <= T prove it), so only keys <= T can be sources;
//   (b) k_dist_cand: one coalesced pass over the N x d coordinates computing the bit-exact
//       distance (sequential sum of squared differences, no FMA, correctly-rounded sqrt;
//       geometry.hpp:36-37), storing it, and appending (key, idx) when key <= T;
//   (c) candidates sorted by (dist, idx) (two stable radix sorts) -> the exact source set of
//       nth_element with the (dist, idx) comparator (geometry.hpp:39-45);
//   (d) k_compact: single-pass decoupled look-back stable compaction of
//       {i not source : dist_i >= xi * rho} in ascending index (geometry.hpp:55-60).
// Non-negative doubles order like their bit patterns, so keys are the raw dist bits.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstring>

#include "kid_internal.cuh"

namespace kid {
namespace {

constexpr int kSampleMax = 65536;
constexpr int64_t kSampleBig = 1 << 20;
inline int64_t ceil_to64(int64_t x) { return (x + 255) / 256 * 256; }

__device__ __forceinline__ double point_dist(const double* __restrict__ pts, int64_t N, int d,
                                             int64_t i, const double* __restrict__ c) {
  double diff = __dsub_rn(pts[i], c[0]);
  double acc = __dmul_rn(diff, diff);
  for (int k = 1; k < d; ++k) {
    diff = __dsub_rn(pts[i + k * N], c[k]);
    acc = __dadd_rn(acc, __dmul_rn(diff, diff));
  }
  return __dsqrt_rn(acc);
}

// 32-bit sample keys: the distance rounded UP to float (monotone), so the n-th smallest of them,
// widened back to double, still bounds the n-th smallest sample distance from above -- half the
// radix passes of the 64-bit keys.
// The sample is S / kRun runs of kRun consecutive points spread evenly over [0, N) (coalesced reads);
// any subset gives a valid bound, the spread only keeps the candidate count near its expectation.
constexpr int kRun = 256;
__global__ void k_sample_keys32(const double* __restrict__ pts, int64_t N, int d, const double* __restrict__ center,
                                int64_t S, unsigned int* __restrict__ keys) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= S) return;
  const int64_t runs = S / kRun;
  const long long r0 = (long long)(((__int128)(j / kRun) * N) / runs);
  const int64_t i = (S == N) ? j : (int64_t)min(r0, (long long)(N - kRun)) + j % kRun;
  keys[j] = (unsigned int)__float_as_int(__double2float_ru(point_dist(pts, N, d, i, center)));
}

__global__ void k_sample_keys(const double* __restrict__ pts, int64_t N, int d,
                              const double* __restrict__ center, int64_t S,
                              unsigned long long* __restrict__ keys) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= S) return;
  const int64_t i = (S == N) ? j : (int64_t)(((__int128)j * N) / S);
  keys[j] = (unsigned long long)__double_as_longlong(point_dist(pts, N, d, i, center));
}

// (b): one thread per point, grid-stride; warp-aggregated append of candidates.
__global__ void __launch_bounds__(256) k_dist_cand(const double* __restrict__ pts, int64_t N, int d,
                                                   const double* __restrict__ center,
                                                   const unsigned long long* __restrict__ T_key,
                                                   double* __restrict__ dist,
                                                   unsigned long long* __restrict__ cand_key,
                                                   unsigned long long* __restrict__ cand_idx,
                                                   unsigned long long* __restrict__ cand_count,
                                                   int64_t cap, const unsigned int* __restrict__ T32 = nullptr) {
  __shared__ double c_s[64];
  if (threadIdx.x < d) c_s[threadIdx.x] = center[threadIdx.x];
  __syncthreads();
  const unsigned long long T =
      T32 ? (unsigned long long)__double_as_longlong((double)__int_as_float((int)*T32)) : *T_key;
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < N; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool cand = false;
    unsigned long long key = 0;
    if (i < N) {
      double diff = __dsub_rn(pts[i], c_s[0]);
      double acc = __dmul_rn(diff, diff);
      for (int k = 1; k < d; ++k) {
        diff = __dsub_rn(pts[i + k * N], c_s[k]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
      }
      const double v = __dsqrt_rn(acc);
      dist[i] = v;
      key = (unsigned long long)__double_as_longlong(v);
      cand = key <= T;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, cand);
    if (mask) {
      unsigned long long pos0 = 0;
      if (lane == 0) pos0 = atomicAdd(cand_count, (unsigned long long)__popc(mask));
      pos0 = __shfl_sync(0xffffffffu, pos0, 0);
      if (cand) {
        const unsigned long long pos = pos0 + __popc(mask & ((1u << lane) - 1u));
        if ((int64_t)pos < cap) {
          cand_key[pos] = key;
          cand_idx[pos] = (unsigned long long)i;
        }
      }
    }
  }
}

// overflow path: re-collect candidates from the stored distances (no recompute)
__global__ void k_cand_from_dist(const double* __restrict__ dist, int64_t N,
                                 const unsigned long long* __restrict__ T_key,
                                 unsigned long long* __restrict__ cand_key,
                                 unsigned long long* __restrict__ cand_idx,
                                 unsigned long long* __restrict__ cand_count) {
  const unsigned long long T = *T_key;
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < N; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    unsigned long long key = 0;
    bool cand = false;
    if (i < N) {
      key = (unsigned long long)__double_as_longlong(dist[i]);
      cand = key <= T;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, cand);
    if (mask) {
      unsigned long long pos0 = 0;
      if (lane == 0) pos0 = atomicAdd(cand_count, (unsigned long long)__popc(mask));
      pos0 = __shfl_sync(0xffffffffu, pos0, 0);
      if (cand) {
        const unsigned long long pos = pos0 + __popc(mask & ((1u << lane) - 1u));
        cand_key[pos] = key;
        cand_idx[pos] = (unsigned long long)i;
      }
    }
  }
}

__global__ void k_gather_sources(const double* __restrict__ pts, int64_t N, int d,
                                 const int64_t* __restrict__ src_local, int64_t n,
                                 double* __restrict__ src) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  for (int k = 0; k < d; ++k) src[j + k * n] = pts[src_local[j] + k * N];
}

// (d) decoupled look-back stable compaction ------------------------------------
// 256 threads x 16 items per tile; the tile's first warp resolves its exclusive prefix by a
// warp-wide look-back over up to 32 predecessors at a time (status word = 2-bit state | count).
constexpr int kCT = 256, kIPT = 16, kTile = kCT * kIPT;
constexpr unsigned long long kStAgg = 1ull << 62, kStInc = 2ull << 62, kValMask = (1ull << 62) - 1;

__device__ __forceinline__ bool is_source(const int64_t* __restrict__ s, int64_t n, int64_t i) {
  int64_t lo = 0, hi = n;  // lower_bound over the ascending local source list
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (s[mid] < i) lo = mid + 1; else hi = mid;
  }
  return lo < n && s[lo] == i;
}

__global__ void __launch_bounds__(kCT) k_compact(const double* __restrict__ dist, int64_t N, double cutoff,
                                                 double rho, const int64_t* __restrict__ src_local,
                                                 int64_t n_src, int64_t* __restrict__ out,
                                                 unsigned long long* __restrict__ tile_status,
                                                 unsigned int* __restrict__ tile_counter,
                                                 int64_t* __restrict__ total_out, int64_t ntiles,
                                                 const double* __restrict__ rho_dev, double xi) {
  if (rho_dev) {  // rho from the device-side selection; cutoff = xi * rho as on the host (geometry.hpp:57)
    rho = *rho_dev;
    cutoff = xi * rho;
  }
  __shared__ unsigned int tile_s;
  __shared__ long long warp_tot[kCT / 32];
  __shared__ long long excl_s;
  if (threadIdx.x == 0) tile_s = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const int64_t tile = tile_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // coalesced loads: item j of thread t is element tile*kTile + j*kCT + t
  const int64_t base = tile * kTile + threadIdx.x;
  unsigned flags = 0;
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    const int64_t i = base + (int64_t)j * kCT;
    if (i < N) {
      const double v = __ldcs(dist + i);
      bool f = v >= cutoff;
      if (f && v <= rho) f = !is_source(src_local, n_src, i);
      flags |= (unsigned)f << j;
    }
  }
  // per-(j) rank within the tile: items are ordered by (j, t); count flagged items of each j
  // across the block with one warp-ballot pass per j
  __shared__ int jcount[kIPT][kCT / 32];
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    const unsigned b = __ballot_sync(0xffffffffu, (flags >> j) & 1u);
    if (lane == 0) jcount[j][warp] = __popc(b);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long run = 0;
    for (int j = 0; j < kIPT; ++j)
      for (int w = 0; w < kCT / 32; ++w) {
        const int t = jcount[j][w];
        jcount[j][w] = (int)run;
        run += t;
      }
    warp_tot[0] = run;
  }
  __syncthreads();
  const long long total = warp_tot[0];
  if (warp == 0) {
    long long excl = 0;
    if (tile == 0) {
      if (lane == 0) {
        __threadfence();
        atomicExch(&tile_status[0], kStInc | (unsigned long long)total);
      }
    } else {
      if (lane == 0) {
        __threadfence();
        atomicExch(&tile_status[tile], kStAgg | (unsigned long long)total);
      }
      int64_t p = tile - 1;
      for (;;) {
        const int64_t q = p - lane;
        unsigned long long sv = kStInc;  // before tile 0: inclusive 0
        if (q >= 0) {
          do {
            sv = *((volatile unsigned long long*)&tile_status[q]);
          } while ((sv & ~kValMask) == 0);
        }
        const unsigned inc = __ballot_sync(0xffffffffu, (sv & ~kValMask) == kStInc);
        const int first = inc ? __ffs(inc) - 1 : 31;
        long long v = lane <= first ? (long long)(sv & kValMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (inc) break;
        p -= 32;
      }
      if (lane == 0) {
        __threadfence();
        atomicExch(&tile_status[tile], kStInc | (unsigned long long)(excl + total));
      }
    }
    if (lane == 0) {
      excl_s = excl;
      if (tile == ntiles - 1) *total_out = excl + total;
    }
  }
  __syncthreads();
  const long long excl = excl_s;
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    const unsigned b = __ballot_sync(0xffffffffu, (flags >> j) & 1u);
    if ((flags >> j) & 1u) out[excl + jcount[j][warp] + __popc(b & ((1u << lane) - 1u))] = base + (int64_t)j * kCT;
  }
}

// ---- fast path (kid_split on one rank): one byte per point instead of the 8-byte distance.
// T (>= rho, the sample bound) is known before the distance pass, so a point with dist > T and
// dist >= xi T is a target whatever rho turns out to be (rho <= T; xi * x rounds monotonically):
// flag 1. Every other point is "near": its exact distance is kept (a sparse 8-byte store; ~0.3% of
// the points at c5) and resolved against rho in the compaction. Traffic: 8 d N + N + 8 N_T (+ the
// near points), against the algorithmic 8 d N + 8 N_T.
__global__ void __launch_bounds__(256) k_dist_flag(const double* __restrict__ pts, int64_t N, int d,
                                                   const double* __restrict__ center,
                                                   const unsigned int* __restrict__ T32, double xi,
                                                   unsigned char* __restrict__ flag, double* __restrict__ dist,
                                                   unsigned long long* __restrict__ cand_key,
                                                   unsigned long long* __restrict__ cand_idx,
                                                   unsigned long long* __restrict__ cand_count, int64_t cap) {
  __shared__ double c_s[64];
  if (threadIdx.x < d) c_s[threadIdx.x] = center[threadIdx.x];
  __syncthreads();
  const double Td = (double)__int_as_float((int)*T32);
  const unsigned long long T = (unsigned long long)__double_as_longlong(Td);
  const double cut = xi * Td;
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < N; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool cand = false;
    unsigned long long key = 0;
    if (i < N) {
      double diff = __dsub_rn(__ldcs(pts + i), c_s[0]);
      double acc = __dmul_rn(diff, diff);
      for (int k = 1; k < d; ++k) {
        diff = __dsub_rn(__ldcs(pts + i + k * N), c_s[k]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
      }
      const double v = __dsqrt_rn(acc);
      const bool sure = v > Td && v >= cut;
      flag[i] = sure ? 1 : 0;
      if (!sure) dist[i] = v;
      key = (unsigned long long)__double_as_longlong(v);
      cand = key <= T;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, cand);
    if (mask) {
      unsigned long long pos0 = 0;
      if (lane == 0) pos0 = atomicAdd(cand_count, (unsigned long long)__popc(mask));
      pos0 = __shfl_sync(0xffffffffu, pos0, 0);
      if (cand) {
        const unsigned long long pos = pos0 + __popc(mask & ((1u << lane) - 1u));
        if ((int64_t)pos < cap) {
          cand_key[pos] = key;
          cand_idx[pos] = (unsigned long long)i;
        }
      }
    }
  }
}

// Stable compaction of the flagged points (ascending index): 256 threads x 32 consecutive points per
// tile (two 16-byte flag loads per thread), block scan, decoupled look-back over tiles, output staged
// in shared memory (64 KB) and written coalesced.
constexpr int kFIPT = 32, kFTile = kCT * kFIPT;
__global__ void __launch_bounds__(kCT) k_compact_flag(const unsigned char* __restrict__ flag,
                                                      const double* __restrict__ dist, int64_t N,
                                                      const int64_t* __restrict__ src_local, int64_t n_src,
                                                      int64_t* __restrict__ out,
                                                      unsigned long long* __restrict__ tile_status,
                                                      unsigned int* __restrict__ tile_counter,
                                                      int64_t* __restrict__ total_out, int64_t ntiles,
                                                      const double* __restrict__ rho_dev, double xi) {
  const double rho = *rho_dev, cutoff = xi * rho;  // geometry.hpp:57
  extern __shared__ int64_t stage[];  // kFTile
  __shared__ unsigned int tile_s;
  __shared__ long long wsum[kCT / 32];
  __shared__ long long excl_s, total_s;
  if (threadIdx.x == 0) tile_s = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const int64_t tile = tile_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t first = tile * kFTile + (int64_t)threadIdx.x * kFIPT;
  unsigned bits = 0;
  if (first + kFIPT <= N) {
    const uint4* f = reinterpret_cast<const uint4*>(flag + first);
    const uint4 a = __ldcs(f), b = __ldcs(f + 1);
    const unsigned w8[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int j = 0; j < kFIPT; ++j) bits |= ((w8[j >> 2] >> (8 * (j & 3))) & 1u) << j;
  } else {
    for (int j = 0; j < kFIPT; ++j)
      if (first + j < N) bits |= (unsigned)(flag[first + j] & 1) << j;
  }
  // near points: the exact distance against rho, the source list where dist <= rho
  const int64_t lim = N - first;
  unsigned near = ~bits & (lim >= kFIPT ? 0xffffffffu : ((1u << (lim > 0 ? lim : 0)) - 1u));
  while (near) {
    const int j = __ffs(near) - 1;
    near &= near - 1;
    const int64_t i = first + j;
    const double v = dist[i];
    bool f = v >= cutoff;
    if (f && v <= rho) f = !is_source(src_local, n_src, i);
    bits |= (unsigned)f << j;
  }
  // block exclusive scan of the per-thread counts
  const int cnt = __popc(bits);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long run = 0;
    for (int w = 0; w < kCT / 32; ++w) {
      const long long t = wsum[w];
      wsum[w] = run;
      run += t;
    }
    total_s = run;
  }
  __syncthreads();
  const long long total = total_s;
  const int my_off = (int)(wsum[warp] + incl - cnt);
  if (warp == 0) {
    long long excl = 0;
    if (tile == 0) {
      if (lane == 0) {
        __threadfence();
        atomicExch(&tile_status[0], kStInc | (unsigned long long)total);
      }
    } else {
      if (lane == 0) {
        __threadfence();
        atomicExch(&tile_status[tile], kStAgg | (unsigned long long)total);
      }
      int64_t p = tile - 1;
      for (;;) {
        const int64_t q = p - lane;
        unsigned long long sv = kStInc;
        if (q >= 0) {
          do {
            sv = *((volatile unsigned long long*)&tile_status[q]);
          } while ((sv & ~kValMask) == 0);
        }
        const unsigned inc = __ballot_sync(0xffffffffu, (sv & ~kValMask) == kStInc);
        const int firstinc = inc ? __ffs(inc) - 1 : 31;
        long long v = lane <= firstinc ? (long long)(sv & kValMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (inc) break;
        p -= 32;
      }
      if (lane == 0) {
        __threadfence();
        atomicExch(&tile_status[tile], kStInc | (unsigned long long)(excl + total));
      }
    }
    if (lane == 0) {
      excl_s = excl;
      if (tile == ntiles - 1) *total_out = excl + total;
    }
  }
  // stage this tile's targets in index order, then one coalesced store. Warp-transposed: in step s the 32
  // lanes place the 32 points of thread s (lane = bit), so a dense run lands on 32 consecutive words -- a thread
  // writing its own 32 points put every lane on one bank (offsets 32 doubles apart: a 32-way conflict per store)
  {
    const int64_t wfirst = tile * kFTile + (int64_t)warp * 32 * kFIPT;
#pragma unroll 4
    for (int sidx = 0; sidx < 32; ++sidx) {
      const unsigned bs = __shfl_sync(0xffffffffu, bits, sidx);
      const int os = __shfl_sync(0xffffffffu, my_off, sidx);
      if ((bs >> lane) & 1u) stage[os + __popc(bs & ((1u << lane) - 1u))] = wfirst + (int64_t)sidx * kFIPT + lane;
    }
  }
  __syncthreads();
  const long long excl = excl_s;
  for (int e = threadIdx.x; e < (int)total; e += kCT) __stcs(out + excl + e, stage[e]);
}

// Device-side selection of the n sources, in two launches (the candidate count is read on the
// device): k_split_rank -- kSelCtas CTAs each stage all <= kSelMax candidates in shared memory and
// rank their share under (dist, idx), nth_element's comparator (geometry.hpp:40-47), by counting
// (one warp per candidate, no sorting network); the n of rank < n land at sel[rank]. Then
// k_split_place (one CTA): rho = the largest of the n (geometry.hpp:52-53), the n re-ranked by index
// (geometry.hpp:50-51), the source coordinates gathered. ctrl = [rho, fallback flag (overflow or
// fewer than n candidates)].
constexpr int kSelMax = 4096, kSelT = 1024, kSelCtas = 16, kRankT = 256;
__global__ void __launch_bounds__(kRankT) k_split_rank(const unsigned long long* __restrict__ ck,
                                                      const unsigned long long* __restrict__ ci,
                                                      const unsigned long long* __restrict__ count, int64_t cap,
                                                      int nl, unsigned long long* __restrict__ sel,
                                                      double* __restrict__ ctrl) {
  extern __shared__ unsigned long long rk_sm[];  // key | idx (kSelMax each)
  unsigned long long* key = rk_sm;
  unsigned long long* idx = key + kSelMax;
  const unsigned long long total = *count;
  const unsigned long long lim = (unsigned long long)(cap < kSelMax ? cap : kSelMax);
  const bool bad = total > lim || total < (unsigned long long)nl;
  if (blockIdx.x == 0 && threadIdx.x == 0) ctrl[1] = bad ? 1.0 : 0.0;
  if (bad) return;  // uniform over the grid
  const int cnt = (int)total;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    key[i] = ck[i];
    idx[i] = ci[i];
  }
  __syncthreads();
  // one warp per candidate: the lanes stride over the others (consecutive shared-memory words), the counts are
  // summed over the warp -- cnt / 32 dependent steps per candidate instead of cnt
  const int lane = threadIdx.x & 31;
  const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), nwarps = (int)(gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < cnt; i += nwarps) {
    const unsigned long long ki = key[i], ii = idx[i];
    int rank = 0;
    for (int j = lane; j < cnt; j += 32) rank += (key[j] < ki) || (key[j] == ki && idx[j] < ii);
    rank = __reduce_add_sync(0xffffffffu, rank);
    if (lane == 0 && rank < nl) {
      sel[rank] = ki;
      sel[kSelT + rank] = ii;
    }
  }
}

__global__ void __launch_bounds__(kSelT) k_split_place(const unsigned long long* __restrict__ sel, int nl,
                                                      const double* __restrict__ pts, int64_t N, int d,
                                                      int64_t* __restrict__ src_local, double* __restrict__ src,
                                                      double* __restrict__ ctrl) {
  __shared__ unsigned long long s_idx[kSelT];
  if (ctrl[1] != 0.0) return;
  for (int i = threadIdx.x; i < nl; i += blockDim.x) s_idx[i] = sel[kSelT + i];
  __syncthreads();
  if (threadIdx.x == 0) ctrl[0] = __longlong_as_double((long long)sel[nl - 1]);  // rho: the largest of the n
  for (int i = threadIdx.x; i < nl; i += blockDim.x) {
    const unsigned long long ii = s_idx[i];
    int rank = 0;
    for (int j = 0; j < nl; ++j) rank += s_idx[j] < ii;
    const int64_t li = (int64_t)ii;
    src_local[rank] = li;
    for (int k = 0; k < d; ++k) src[rank + (int64_t)k * nl] = pts[li + k * N];
  }
}

int sort_candidates(kid_ctx* c, unsigned long long* key, unsigned long long* idx, int64_t count,
                    unsigned long long* key_alt, unsigned long long* idx_alt, int end_bit_idx) {
  // stable LSD order: by idx first, then stably by key -> (dist, idx) lexicographic
  size_t tmp1 = 0, tmp2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp1, idx, idx_alt, key, key_alt, (int)count, 0, end_bit_idx, c->stream);
  cub::DeviceRadixSort::SortPairs(nullptr, tmp2, key_alt, key, idx_alt, idx, (int)count, 0, 64, c->stream);
  const size_t need = std::max(tmp1, tmp2);
  if (ensure(c, &c->sort_tmp, &c->sort_tmp_cap, need)) return KID_E_OOM;
  void* tmp = c->sort_tmp;
  KID_CK(c, cub::DeviceRadixSort::SortPairs(tmp, tmp1, idx, idx_alt, key, key_alt, (int)count, 0, end_bit_idx, c->stream));
  c->launches += 2;
  KID_CK(c, cub::DeviceRadixSort::SortPairs(tmp, tmp2, key_alt, key, idx_alt, idx, (int)count, 0, 64, c->stream));
  c->launches += 2;
  return KID_OK;
}

}  // namespace

// Single-rank split with one host synchronisation (kid_split): sample threshold, distances and
// candidates, device-side selection (k_split_rank + k_split_place), compaction with rho read on the device.
// Returns 1 (not taken: fall back to split_candidates / split_finish) when the candidate buffer
// would exceed one CTA's sort or overflowed.
int split_device(kid_ctx* c, const double* center_h, int64_t n, double xi, int64_t* src_idx_out, double* rho_out,
                 int64_t* n_targets_out) {
  const int64_t N = c->N;
  const int d = c->d;
  if (!c->pts || N < 1 || d > 64 || n > kSelT || n > N) return 1;
  const int64_t nl = n;
  // sample size and the sample quantile used as the threshold: the k_s-th smallest of S strided
  // sample distances lets about k_s N / S points through (2.5 n + 4 N / S, a few hundred to a few
  // thousand candidates); fewer than n (rare) or more than kSelMax take the general path
  // S ~ N / 64 up to 2^20 samples (kRun-point runs): about 2.5 n + 4 N / S candidates must stay
  // below kSelMax for the one-CTA selection (at N = 1e8, m = 512: ~1700)
  const int64_t S = N <= 16384 ? N : ceil_to64(std::min<int64_t>(N, std::max<int64_t>(16384, std::min<int64_t>(kSampleBig, N / 64))));
  const int64_t ks = S == N ? nl : std::min<int64_t>(S, (int64_t)std::ceil(2.5 * (double)nl * (double)S / (double)N) + 4);
  const int64_t cap = std::min<int64_t>(kSelMax, N);
  if (ensure(c, (void**)&c->dist, &c->dist_cap, sizeof(double) * N)) return KID_E_OOM;
  if (ensure(c, (void**)&c->tgt_idx, &c->tgt_cap, sizeof(int64_t) * N)) return KID_E_OOM;
  if (ensure(c, (void**)&c->src, &c->src_cap, sizeof(double) * n * d)) return KID_E_OOM;
  const int64_t ntiles = (N + kTile - 1) / kTile;
  // scratch: center | ctrl | count | tile status | sample keys (2x) | candidates | src_local
  const size_t bytes = 512 + 64 + 16 + sizeof(unsigned long long) * (ntiles + 8) + 2 * sizeof(unsigned long long) * S +
                       2 * sizeof(unsigned long long) * cap + sizeof(int64_t) * (n + 8) +
                       2 * sizeof(unsigned long long) * kSelT;
  char* base = (char*)scratch(c, bytes);
  if (!base) return KID_E_OOM;
  double* center = (double*)base;
  double* ctrl = (double*)(base + 512);
  unsigned long long* count = (unsigned long long*)(base + 512 + 64);
  unsigned long long* status = count + 2;
  unsigned int* skeys = (unsigned int*)(status + ntiles + 8);
  unsigned int* skeys2 = skeys + S;
  unsigned long long* ck = (unsigned long long*)(skeys2 + S);  // 2S 32-bit keys: 8-byte aligned
  unsigned long long* ci = ck + cap;
  int64_t* src_local = (int64_t*)(ci + cap);
  unsigned long long* sel = (unsigned long long*)(src_local + n + 8);  // [key | idx] of the n selected
  KID_CK(c, cudaMemcpyAsync(center, center_h, sizeof(double) * d, cudaMemcpyHostToDevice, c->stream));
  KID_CK(c, cudaMemsetAsync(count, 0, sizeof(unsigned long long) * (2 + ntiles + 8), c->stream));
  KID_CK(c, cudaMemsetAsync(c->counter, 0, sizeof(int64_t) * 2, c->stream));
  k_sample_keys32<<<(unsigned)((S + 255) / 256), 256, 0, c->stream>>>(c->pts, N, d, center, S, skeys);
  KID_LAUNCHED(c);
  size_t tmpb = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmpb, skeys, skeys2, (int)S, 0, 32, c->stream);
  if (ensure(c, &c->sort_tmp, &c->sort_tmp_cap, tmpb)) return KID_E_OOM;
  KID_CK(c, cub::DeviceRadixSort::SortKeys(c->sort_tmp, tmpb, skeys, skeys2, (int)S, 0, 32, c->stream));
  c->launches += 4;
  const int64_t ftiles = (N + kFTile - 1) / kFTile;
  if (ensure(c, (void**)&c->flag, &c->flag_cap, (size_t)ftiles * kFTile)) return KID_E_OOM;
  unsigned char* flag = c->flag;
  prof_begin(c);
  k_dist_flag<<<c->sms * 8, 256, 0, c->stream>>>(c->pts, N, d, center, skeys2 + (ks - 1), xi, flag, c->dist, ck, ci,
                                                 count, cap);
  prof_end(c);
  KID_LAUNCHED(c);
  const size_t rank_smem = sizeof(unsigned long long) * 2 * kSelMax;
  cudaFuncSetAttribute(k_split_rank, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rank_smem);
  k_split_rank<<<kSelCtas, kRankT, rank_smem, c->stream>>>(ck, ci, count, cap, (int)nl, sel, ctrl);
  KID_LAUNCHED(c);
  k_split_place<<<1, kSelT, 0, c->stream>>>(sel, (int)nl, c->pts, N, d, src_local, c->src, ctrl);
  KID_LAUNCHED(c);
  prof_begin(c);
  cudaFuncSetAttribute(k_compact_flag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(int64_t) * kFTile));
  k_compact_flag<<<(unsigned)ftiles, kCT, sizeof(int64_t) * kFTile, c->stream>>>(
      flag, c->dist, N, src_local, nl, c->tgt_idx, status, (unsigned int*)c->counter, c->counter + 1, ftiles, ctrl, xi);
  prof_end(c);
  KID_LAUNCHED(c);
  // one D2H of [rho, overflow | nt | source indices | source coordinates] and one synchronisation
  const size_t hb = sizeof(double) * (2 + 1 + (size_t)n + (size_t)n * d);
  if (ensure_pinned(c, hb)) return KID_E_OOM;
  double* h = c->hbuf;
  KID_CK(c, cudaMemcpyAsync(h, ctrl, sizeof(double) * 2, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaMemcpyAsync(h + 2, c->counter + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaMemcpyAsync(h + 3, src_local, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaMemcpyAsync(h + 3 + n, c->src, sizeof(double) * n * d, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  if (h[1] != 0.0) return 1;  // candidate overflow (adversarial ordering): the general path
  int64_t nt = 0;
  std::memcpy(&nt, h + 2, sizeof(int64_t));
  const int64_t* sl = (const int64_t*)(h + 3);
  for (int64_t k = 0; k < n; ++k) src_idx_out[k] = sl[k] + c->offset;
  *rho_out = h[0];
  c->src_host.assign(h + 3 + n, h + 3 + n + (size_t)n * d);
  c->n_split_targets = nt;
  c->tbase = c->pts;
  c->tld = N;
  c->tidx = c->tgt_idx;
  c->nt = nt;
  c->m = n;
  c->r = 0;
  c->sub_active = false;
  *n_targets_out = nt;
  return KID_OK;
}

// Local n smallest (dist, idx) keys, ascending; indices are GLOBAL (offset added).
int split_candidates(kid_ctx* c, const double* center_h, int64_t n, double* cand_dist_h,
                     int64_t* cand_idx_h) {
  const int64_t N = c->N;
  const int d = c->d;
  if (!c->pts || N < 1) return fail(c, KID_E_ERROR, "kid_split: no point set");
  if (d > 64) return fail(c, KID_E_DIM, "kid_split: d > 64 unsupported");
  const int64_t nl = std::min<int64_t>(n, N);  // a shard may hold fewer than n points
  if (ensure(c, (void**)&c->dist, &c->dist_cap, sizeof(double) * N)) return KID_E_OOM;

  // scratch layout: center | T_key | count | sample keys (2x) | candidates
  const int64_t S = N <= std::max<int64_t>(kSampleMax, 4 * nl) ? N : std::max<int64_t>(kSampleMax, 4 * nl);
  int64_t cap = std::max<int64_t>(4 * nl + 1024, (int64_t)((double)N * (double)nl / (double)S * 2.0) + 4096);
  cap = std::min<int64_t>(cap, N);
  const size_t bytes = 64 * 8 + 16 + 16 + 2 * sizeof(unsigned long long) * S + 4 * sizeof(unsigned long long) * cap;
  char* base = (char*)scratch(c, bytes);
  if (!base) return KID_E_OOM;
  double* center = (double*)base;
  unsigned long long* T_key = (unsigned long long*)(base + 512);
  unsigned long long* count = (unsigned long long*)(base + 512 + 16);
  unsigned long long* skeys = (unsigned long long*)(base + 512 + 32);
  unsigned long long* skeys2 = skeys + S;
  unsigned long long* ck = skeys2 + S;
  unsigned long long* ci = ck + cap;
  unsigned long long* ck2 = ci + cap;
  unsigned long long* ci2 = ck2 + cap;

  KID_CK(c, cudaMemcpyAsync(center, center_h, sizeof(double) * d, cudaMemcpyHostToDevice, c->stream));
  KID_CK(c, cudaMemsetAsync(count, 0, sizeof(unsigned long long), c->stream));
  k_sample_keys<<<(unsigned)((S + 255) / 256), 256, 0, c->stream>>>(c->pts, N, d, center, S, skeys);
  KID_LAUNCHED(c);
  {
    size_t tmpb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tmpb, skeys, skeys2, (int)S, 0, 64, c->stream);
    if (ensure(c, &c->sort_tmp, &c->sort_tmp_cap, tmpb)) return KID_E_OOM;
    KID_CK(c, cub::DeviceRadixSort::SortKeys(c->sort_tmp, tmpb, skeys, skeys2, (int)S, 0, 64, c->stream));
    c->launches += 4;
    KID_CK(c, cudaMemcpyAsync(T_key, skeys2 + (nl - 1), sizeof(unsigned long long), cudaMemcpyDeviceToDevice,
                              c->stream));
  }
  const int blocks = c->sms * 8;
  prof_begin(c);
  k_dist_cand<<<blocks, 256, 0, c->stream>>>(c->pts, N, d, center, T_key, c->dist, ck, ci, count, cap);
  prof_end(c);
  KID_LAUNCHED(c);
  unsigned long long cnt = 0;
  KID_CK(c, cudaMemcpyAsync(&cnt, count, sizeof(cnt), cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  if ((int64_t)cnt > cap) {  // loose bound (adversarial ordering): recollect into a larger buffer
    const int64_t big = (int64_t)cnt;
    unsigned long long* buf = nullptr;
    KID_CK(c, cudaMalloc(&buf, 4 * sizeof(unsigned long long) * big));
    ck = buf; ci = ck + big; ck2 = ci + big; ci2 = ck2 + big;
    KID_CK(c, cudaMemsetAsync(count, 0, sizeof(unsigned long long), c->stream));
    k_cand_from_dist<<<blocks, 256, 0, c->stream>>>(c->dist, N, T_key, ck, ci, count);
    KID_LAUNCHED(c);
    int end_bit = 1;
    while (end_bit < 63 && (1ll << end_bit) < N) ++end_bit;
    int rc = sort_candidates(c, ck, ci, big, ck2, ci2, end_bit);
    if (!rc) {
      std::vector<unsigned long long> hk(nl), hi(nl);
      KID_CK(c, cudaMemcpy(hk.data(), ck, sizeof(unsigned long long) * nl, cudaMemcpyDeviceToHost));
      KID_CK(c, cudaMemcpy(hi.data(), ci, sizeof(unsigned long long) * nl, cudaMemcpyDeviceToHost));
      for (int64_t k = 0; k < nl; ++k) {
        std::memcpy(&cand_dist_h[k], &hk[k], 8);
        cand_idx_h[k] = (int64_t)hi[k] + c->offset;
      }
    }
    cudaFree(buf);
    return rc;
  }
  int end_bit = 1;
  while (end_bit < 63 && (1ll << end_bit) < N) ++end_bit;
  int rc = sort_candidates(c, ck, ci, (int64_t)cnt, ck2, ci2, end_bit);
  if (rc) return rc;
  std::vector<unsigned long long> hk(nl), hi(nl);
  KID_CK(c, cudaMemcpyAsync(hk.data(), ck, sizeof(unsigned long long) * nl, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaMemcpyAsync(hi.data(), ci, sizeof(unsigned long long) * nl, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  for (int64_t k = 0; k < nl; ++k) {
    std::memcpy(&cand_dist_h[k], &hk[k], 8);
    cand_idx_h[k] = (int64_t)hi[k] + c->offset;
  }
  return KID_OK;
}

// Given the global source set (ascending GLOBAL indices) and rho, compact the local targets.
// src_pts_h (n x d col-major host) may be null when every source is local.
int split_finish(kid_ctx* c, const int64_t* src_idx_h, int64_t n, const double* src_pts_h, double rho,
                 double xi, int64_t* n_targets_out) {
  const int64_t N = c->N;
  const int d = c->d;
  std::vector<int64_t> local;
  local.reserve(n);
  for (int64_t k = 0; k < n; ++k) {
    const int64_t li = src_idx_h[k] - c->offset;
    if (li >= 0 && li < N) local.push_back(li);
  }
  const int64_t nloc = (int64_t)local.size();
  const int64_t ntiles = (N + kTile - 1) / kTile;
  const size_t bytes = sizeof(int64_t) * (nloc + n + 8) + sizeof(unsigned long long) * (ntiles + 8);
  char* base = (char*)scratch(c, bytes);
  if (!base) return KID_E_OOM;
  int64_t* src_local = (int64_t*)base;
  int64_t* src_all_local = src_local + nloc;  // gather list when all sources are local
  unsigned long long* status = (unsigned long long*)(src_all_local + n + 8);
  if (ensure(c, (void**)&c->tgt_idx, &c->tgt_cap, sizeof(int64_t) * N)) return KID_E_OOM;
  if (ensure(c, (void**)&c->src, &c->src_cap, sizeof(double) * n * d)) return KID_E_OOM;
  if (nloc) KID_CK(c, cudaMemcpyAsync(src_local, local.data(), sizeof(int64_t) * nloc, cudaMemcpyHostToDevice, c->stream));
  if (src_pts_h) {
    KID_CK(c, cudaMemcpyAsync(c->src, src_pts_h, sizeof(double) * n * d, cudaMemcpyHostToDevice, c->stream));
  } else {
    if (nloc != n) return fail(c, KID_E_ERROR, "kid_split_finish: non-local sources need src_points");
    k_gather_sources<<<(unsigned)((n + 127) / 128), 128, 0, c->stream>>>(c->pts, N, d, src_local, n, c->src);
    KID_LAUNCHED(c);
  }
  KID_CK(c, cudaMemsetAsync(status, 0, sizeof(unsigned long long) * ntiles, c->stream));
  KID_CK(c, cudaMemsetAsync(c->counter, 0, sizeof(int64_t) * 2, c->stream));
  const double cutoff = xi * rho;  // geometry.hpp:57
  prof_begin(c);
  k_compact<<<(unsigned)ntiles, kCT, 0, c->stream>>>(c->dist, N, cutoff, rho, src_local, nloc, c->tgt_idx, status,
                                                     (unsigned int*)c->counter, c->counter + 1, ntiles, nullptr, 0.0);
  prof_end(c);
  KID_LAUNCHED(c);
  int64_t nt = 0;
  KID_CK(c, cudaMemcpyAsync(&nt, c->counter + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  c->src_host.resize((size_t)n * d);
  if (src_pts_h) std::memcpy(c->src_host.data(), src_pts_h, sizeof(double) * n * d);
  else KID_CK(c, cudaMemcpyAsync(c->src_host.data(), c->src, sizeof(double) * n * d, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  c->n_split_targets = nt;
  c->tbase = c->pts;
  c->tld = N;
  c->tidx = c->tgt_idx;
  c->nt = nt;
  c->m = n;
  c->r = 0;
  c->sub_active = false;
  *n_targets_out = nt;
  return KID_OK;
}

}  // namespace kid
