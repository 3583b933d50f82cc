// Dependent-chain latency (one warp) and per-SMSP throughput of DFMA / DADD / DMUL on sm_100a,
// and throughput of a dependent chain with W warps per SMSP (how many chains hide the latency).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void chain(double* out, long long* cyc, int iters, double a) {
  double x = threadIdx.x * 1e-9 + 1.0, y = x + 0.5;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (OP == 0) x = fma(x, a, 1e-3);
      if (OP == 1) x = x + a;
      if (OP == 2) x = x * a;
      if (OP == 3) { x = fma(x, a, 1e-3); y = fma(y, a, 1e-3); }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x + y;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMallocManaged(&cyc, 8);
  const char* names[] = {"dfma", "dadd", "dmul", "dfma_2chains"};
  const int iters = 1000;
  for (int op = 0; op < 4; ++op)
    for (int w : {1, 2, 4, 8, 12, 16, 24, 32}) {
      // one CTA on each SM, w warps per CTA (w/4 per SMSP)
      auto f = op == 0 ? chain<0> : op == 1 ? chain<1> : op == 2 ? chain<2> : chain<3>;
      f<<<148, 32 * w>>>(out, cyc, iters, 0.9999999);
      cudaDeviceSynchronize();
      f<<<148, 32 * w>>>(out, cyc, iters, 0.9999999);
      cudaDeviceSynchronize();
      const double ops = (double)iters * 16 * (op == 3 ? 2 : 1);
      printf("{\"op\": \"%s\", \"warps_per_sm\": %d, \"cycles_per_dep_op\": %.2f, \"warp_ops_per_clk_sm\": %.3f}\n",
             names[op], w, *cyc / ops * (op == 3 ? 2 : 1), ops * w / *cyc);
    }
  return 0;
}
