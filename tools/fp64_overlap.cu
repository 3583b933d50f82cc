// Does the FP64 tensor pipe (DMMA) run concurrently with the FP64 vector pipe (DFMA)?
// Warps [0, nd) issue DMMA.8x8x4 loops, warps [nd, 8) DFMA loops; compare with each alone.
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
__global__ void mixed(double* out, int iters_mma, int iters_fma, int n_mma_warps) {
  const int warp = threadIdx.x >> 5;
  double acc = 0;
  if (warp < n_mma_warps) {
    double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3, c[8][2] = {};
    for (int i = 0; i < iters_mma; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    for (int j = 0; j < 8; ++j) acc += c[j][0] + c[j][1];
  } else {
    double x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < iters_fma; ++i)
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], 0.999, 1e-3);
    for (int k = 0; k < 8; ++k) acc += x[k];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  double* out; cudaMalloc(&out, 1 << 24);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 4, threads = 256;
  // per-warp work: DMMA warp: iters*8 DMMA (256 FMA each, warp-wide); DFMA warp: iters*64 DFMA (32 FMA each)
  struct Cfg { const char* name; int im, ifm, nw; } cfgs[] = {
      {"dmma_only_4w", 2000, 0, 4}, {"dfma_only_4w", 0, 8000, 0}, {"mixed_4+4", 2000, 8000, 4},
      {"dmma_only_8w", 2000, 0, 8}, {"dfma_only_8w", 0, 8000, 0}};
  for (int rep = 0; rep < 2; ++rep)
    for (auto& c : cfgs) {
      int nw = c.nw;
      int tpb = threads;
      if (!strcmp(c.name, "dfma_only_4w")) tpb = 128, nw = 0;   // 4 warps, all DFMA
      if (!strcmp(c.name, "dmma_only_4w")) tpb = 128;
      mixed<<<blocks, tpb>>>(out, c.im, c.ifm, nw);
      cudaEventRecord(e0);
      mixed<<<blocks, tpb>>>(out, c.im, c.ifm, nw);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double mma_warps = (double)blocks * (nw), fma_warps = (double)blocks * (tpb / 32 - nw);
      double fl = 2.0 * (mma_warps * c.im * 8 * 256 + fma_warps * c.ifm * 64 * 32);
      printf("{\"cfg\": \"%s\", \"ms\": %.3f, \"tflops\": %.2f}\n", c.name, ms, fl / ms / 1e9);
    }
  return 0;
}
