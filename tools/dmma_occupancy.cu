// DMMA.8x8x4 throughput vs resident warps per SM and fragment source (registers vs shared).
#include <cstdio>
#include <cuda_runtime.h>
template <int NACC, bool FROM_SMEM>
__global__ void dmma_loop(double* out, int iters) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i * 1e-3;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double a = lane * 1e-3, b = lane * 2e-3, c[NACC][2];
#pragma unroll
  for (int j = 0; j < NACC; ++j) c[j][0] = c[j][1] = 0.0;
  int off = (threadIdx.x >> 5) * 64;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) {
      if (FROM_SMEM) {
        a = sm[(off + (lane & 3) * 36 + (lane >> 2) + j * 8) & 4095];
        b = sm[(off + 512 + (lane & 3) * 36 + (lane >> 2) + j * 8) & 4095];
      }
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
    off = (off + 4) & 1023;
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NACC, bool S>
void run(const char* name, int warps_per_sm, double* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 32 * (warps_per_sm < 8 ? warps_per_sm : 8);
  const int blocks = 148 * (warps_per_sm * 32 / threads);
  const int iters = 4000 / NACC * 8;
  dmma_loop<NACC, S><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e0);
  dmma_loop<NACC, S><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * 256 * NACC * (double)iters * blocks * (threads / 32);
  printf("{\"cfg\": \"%s\", \"warps_per_sm\": %d, \"nacc\": %d, \"smem\": %d, \"tflops\": %.2f}\n", name, warps_per_sm, NACC, (int)S, fl / ms / 1e9);
}
int main() {
  double* out; cudaMalloc(&out, 1 << 26);
  for (int w : {4, 8, 12, 16, 32}) {
    run<8, false>("reg", w, out);
    run<8, true>("smem", w, out);
    run<16, true>("smem", w, out);
    run<4, true>("smem", w, out);
  }
  return 0;
}
