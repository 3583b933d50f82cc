// Throughput of the fused pass's column evaluation (distance + exp_neg_fast + sum K^2 + column-
// major store), as exps/clk/SM, by eval warps per SM and columns per pass (ILP), d = 3.
// Variants: 0 full, 1 constant table entry, 2 no store, 3 no distance (q from a register).
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
#include "../paper_1409_2802_b200/csrc/kid_internal.cuh"
__device__ double g_tab[kid::kExpTab];
constexpr int D = 3, M = 96, KST = 36;
template <int ILP, int VAR>
__global__ void k(double* out, int reps, double cs) {
  __shared__ double tab[kid::kExpTabWords];
  __shared__ __align__(16) double src[D * M];
  extern __shared__ double KN[];  // M x KST per warp-group (shared by warps: races are harmless here)
  for (int e = threadIdx.x; e < kid::kExpTabWords; e += blockDim.x) tab[e] = g_tab[e / kid::kExpRep];
  for (int e = threadIdx.x; e < D * M; e += blockDim.x) src[e] = 0.01 * (e % 97) - 0.3;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double tc[D];
  for (int k2 = 0; k2 < D; ++k2) tc[k2] = (blockIdx.x * 0.001 + lane * 0.013 + k2 * 0.1) * cs;
  double sk = 0.0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int j0 = warp * ILP; j0 < M; j0 += nw * ILP) {
      double kv[ILP];
#pragma unroll
      for (int u = 0; u < ILP; ++u) kv[u] = 0.0;
      if (VAR == 3) {
#pragma unroll
        for (int u = 0; u < ILP; ++u) kv[u] = tc[0] + 0.37 * u + j0 * 0.01;
      } else {
#pragma unroll
        for (int kk = 0; kk < D; ++kk) {
#pragma unroll
          for (int u = 0; u < ILP; u += 2) {
            const double2 s01 = *reinterpret_cast<const double2*>(&src[kk * M + j0 + u]);
            const double a0 = tc[kk] - s01.x, a1 = tc[kk] - s01.y;
            kv[u] = fma(a0, a0, kv[u]);
            if (u + 1 < ILP) kv[u + 1] = fma(a1, a1, kv[u + 1]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < ILP; ++u) {
        double e;
        if (VAR == 1) e = kid::exp_neg_fast(kv[u], tab + lane);  // (no-table variant removed)
        else e = kid::exp_neg_fast(kv[u], tab + lane);
        kv[u] = lane < 40 ? e : 0.0;
        sk = fma(kv[u], kv[u], sk);
        if (VAR != 2) KN[(j0 + u) * KST + lane] = kv[u];
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = sk;
}
template <int ILP, int VAR>
void run(int warps, double* out) {
  const int reps = 200;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const size_t sm = sizeof(double) * (M + 8) * KST;
  cudaFuncSetAttribute(k<ILP, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<ILP, VAR><<<148, warps * 32, sm>>>(out, reps, 7.0);
  cudaEventRecord(e0);
  k<ILP, VAR><<<148, warps * 32, sm>>>(out, reps, 7.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double exps = 148.0 * reps * M * 32;
  printf("{\"var\": %d, \"ilp\": %d, \"warps_per_sm\": %d, \"exp_per_clk_sm\": %.2f}\n", VAR, ILP, warps,
         exps / (ms * 1e-3) / 148 / 1.965e9);
}
int main() {
  double tab[kid::kExpTab];
  for (int j = 0; j < kid::kExpTab; ++j) tab[j] = (double)exp2l((long double)j / (long double)kid::kExpTab);
  cudaMemcpyToSymbol(g_tab, tab, sizeof(tab));
  double* out; cudaMalloc(&out, 1 << 24);
  for (int w : {8, 12, 16, 24}) {
    run<4, 0>(w, out); run<8, 0>(w, out); run<2, 0>(w, out);
    run<4, 1>(w, out); run<4, 2>(w, out); run<4, 3>(w, out);
  }
  return 0;
}
