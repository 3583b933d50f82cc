// Throughput of the FP64 passes' exp (exp_neg_fast) vs libdevice exp, by ILP and occupancy.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
#include "../paper_1409_2802_b200/csrc/kid_internal.cuh"
__device__ double g_tab[kid::kExpTab];
template <int ILP, int MODE>
__global__ void k(double* out, int iters) {
  __shared__ double tab[kid::kExpTabWords];
  for (int e = threadIdx.x; e < kid::kExpTabWords; e += blockDim.x) tab[e] = g_tab[e / kid::kExpRep];
  __syncthreads();
  double q[ILP], acc = 0;
#pragma unroll
  for (int u = 0; u < ILP; ++u) q[u] = 1.0 + 0.37 * u + threadIdx.x * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < ILP; ++u) {
      double v = MODE == 0 ? kid::exp_neg_fast(q[u], tab + (threadIdx.x & 31)) : exp(-q[u]);
      acc = fma(v, v, acc);
      q[u] += 0.001;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <int ILP, int MODE>
void run(int warps_per_sm, double* out) {
  const int threads = 32 * (warps_per_sm > 16 ? 16 : warps_per_sm), blocks = 148 * (warps_per_sm * 32 / threads);
  const int iters = 4096 / ILP;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<ILP, MODE><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e0);
  k<ILP, MODE><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double n = (double)blocks * threads * iters * ILP;
  printf("{\"mode\": \"%s\", \"ilp\": %d, \"warps_per_sm\": %d, \"gexp_s\": %.1f, \"exp_per_clk_sm\": %.2f}\n",
         MODE == 0 ? "exp_neg_fast" : "libdevice", ILP, warps_per_sm, n / ms / 1e6, n / (ms * 1e-3 * 1.965e9 * 148));
}
int main() {
  double tab[kid::kExpTab];
  for (int j = 0; j < kid::kExpTab; ++j) tab[j] = (double)exp2l((long double)j / (long double)kid::kExpTab);
  cudaMemcpyToSymbol(g_tab, tab, sizeof(tab));
  double* out; cudaMalloc(&out, 1 << 24);
  for (int w : {4, 8, 16, 32}) { run<1, 0>(w, out); run<2, 0>(w, out); run<4, 0>(w, out); run<8, 0>(w, out); }
  for (int w : {8, 32}) { run<2, 1>(w, out); run<4, 1>(w, out); }
  return 0;
}
