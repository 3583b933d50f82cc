// Microbenchmark: FP64 vector (DFMA), FP64 tensor (DMMA) and exp(double)
// throughput on the local GPU. Used to fix P_FP64, the roofline denominator
// for the FP64 passes.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma884_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16816_loop(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = threadIdx.x * 2e-3 + k;
  double c[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void exp_loop(double* out, int iters, double step) {
  double x = -1.0 - threadIdx.x * 1e-3, acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { acc += exp(x); x -= step; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void copy_kernel(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  double* out; CK(cudaMalloc(&out, 1 << 24));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  float ms;
  for (int rep = 0; rep < 3; ++rep) {
    int iters = 4000;
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(out, iters, 0.999, 1e-3); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 64 * iters * (double)blocks * threads;
    printf("{\"kernel\": \"dfma\", \"tflops\": %.2f, \"ms\": %.3f}\n", fl / ms / 1e9, ms);

    iters = 2000;
    dmma884_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e0); dmma884_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 8 * 8 * 4 * 8 * iters * (double)blocks * (threads / 32);
    printf("{\"kernel\": \"dmma_m8n8k4\", \"tflops\": %.2f, \"ms\": %.3f}\n", fl / ms / 1e9, ms);

    iters = 500;
    dmma16816_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e0); dmma16816_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * 8 * 16 * 4 * iters * (double)blocks * (threads / 32);
    printf("{\"kernel\": \"dmma_m16n8k16\", \"tflops\": %.2f, \"ms\": %.3f}\n", fl / ms / 1e9, ms);

    iters = 500;
    exp_loop<<<blocks, threads>>>(out, iters, 1e-4);
    cudaEventRecord(e0); exp_loop<<<blocks, threads>>>(out, iters, 1e-4); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double ne = 8.0 * iters * (double)blocks * threads;
    printf("{\"kernel\": \"exp_f64\", \"gexp_per_s\": %.2f, \"ms\": %.3f}\n", ne / ms / 1e6, ms);
  }
  // sustained: back-to-back launches for ~5 s each (the clocks a seconds-long FP64 pass runs at)
  for (int kind = 0; kind < 2; ++kind) {
    const int iters = kind == 0 ? 40000 : 80000;  // ~0.1-0.2 s per launch
    double flops = 0.0, tot_ms = 0.0;
    cudaEventRecord(e0);
    int launches = 0;
    while (tot_ms < 5000.0) {
      for (int k = 0; k < 4; ++k, ++launches) {
        if (kind == 0) dmma884_loop<<<blocks, threads>>>(out, iters);
        else dfma_loop<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
        flops += kind == 0 ? 2.0 * 8 * 8 * 4 * 8 * iters * (double)blocks * (threads / 32)
                           : 2.0 * 64 * iters * (double)blocks * threads;
      }
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      tot_ms = ms;
    }
    printf("{\"kernel\": \"%s_sustained\", \"tflops\": %.2f, \"seconds\": %.2f, \"launches\": %d}\n",
           kind == 0 ? "dmma_m8n8k4" : "dfma", flops / tot_ms / 1e9, tot_ms / 1e3, launches);
  }
  size_t n = (size_t)1 << 27;  // 4 GiB per buffer in double4? no: 2^27 * 32 B = 4 GiB
  double4 *a, *b; CK(cudaMalloc(&a, n * sizeof(double4))); CK(cudaMalloc(&b, n * sizeof(double4)));
  cudaMemset(a, 0, n * sizeof(double4));
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); copy_kernel<<<sms * 16, 512>>>(a, b, n); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kernel\": \"copy\", \"gbs\": %.1f}\n", 2.0 * n * sizeof(double4) / ms / 1e6);
  }
  return 0;
}
