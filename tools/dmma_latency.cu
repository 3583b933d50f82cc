// DMMA.8x8x4 latency / per-warp throughput: one warp per SMSP (4 per SM), NACC independent
// accumulator chains per warp; cycles per DMMA measured with clock64 inside the kernel.
#include <cstdio>
#include <cuda_runtime.h>
template <int NACC>
__global__ void chain(double* out, long long* cyc, int iters) {
  const int lane = threadIdx.x & 31;
  double a = lane * 1e-3, b = lane * 2e-3, c[NACC][2];
#pragma unroll
  for (int j = 0; j < NACC; ++j) c[j][0] = c[j][1] = 0.0;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < NACC; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j) s += c[j][0] + c[j][1];
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (lane == 0) cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = t1 - t0;
}
template <int NACC>
void run(int warps_per_sm, double* out, long long* cyc) {
  const int iters = 2000;
  chain<NACC><<<148, 32 * warps_per_sm>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h[32];
  cudaMemcpy(h, cyc, sizeof(long long) * warps_per_sm, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int w = 0; w < warps_per_sm; ++w) mean += h[w];
  mean /= warps_per_sm;
  printf("{\"nacc\": %d, \"warps_per_sm\": %d, \"cycles_per_dmma_per_warp\": %.1f, \"sm_dmma_per_clk\": %.3f}\n", NACC,
         warps_per_sm, mean / (iters * NACC), warps_per_sm * iters * NACC / mean);
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 22); cudaMalloc(&cyc, 1 << 16);
  for (int w : {1, 4, 8}) { run<1>(w, out, cyc); run<2>(w, out, cyc); run<4>(w, out, cyc); run<8>(w, out, cyc); run<16>(w, out, cyc); }
  return 0;
}
