// Reproduces the fused pass' D = K_N - K_S P2 block loop (k_gram GEMM1) in isolation:
// 8 warps, column-major K_S / K_N stages (stride 36), row-major P2 (stride SP), r4 = 20,
// NBN = 11 column blocks x 4 row blocks = 44 DMMA blocks spread over the warps.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kST = 36, kGPW = 4;
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void probe(double* out, long long* cyc, int r4, int NBN, int SP, int reps) {
  extern __shared__ double sm[];
  double* KS = sm;
  double* KN = KS + 32 * kST;
  double* sP = KN + 96 * kST;
  for (int i = threadIdx.x; i < 32 * kST + 96 * kST + 32 * SP; i += blockDim.x) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int lane = threadIdx.x & 31, mw = threadIdx.x >> 5, fr = lane >> 2, fk = lane & 3;
  const int nblk1 = 4 * NBN, g_lo = nblk1 * mw / 8, g_hi = nblk1 * (mw + 1) / 8;
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    for (int g0 = g_lo; g0 < g_hi; g0 += kGPW) {
      double c[kGPW][2];
#pragma unroll
      for (int q = 0; q < kGPW; ++q) c[q][0] = c[q][1] = 0.0;
      for (int k0 = 0; k0 < r4; k0 += 4) {
        double a[kGPW], b[kGPW];
#pragma unroll
        for (int q = 0; q < kGPW; ++q) {
          const int g = g0 + q < g_hi ? g0 + q : g_lo;
          const int nb = g >> 2, rb = g & 3;
          if (MODE == 2) { a[q] = fk * 1e-3; b[q] = fr * 1e-3; }
          else { a[q] = KS[(k0 + fk) * kST + rb * 8 + fr]; b[q] = sP[(k0 + fk) * SP + nb * 8 + fr]; }
        }
#pragma unroll
        for (int q = 0; q < kGPW; ++q)
          if (g0 + q < g_hi) dmma884(c[q][0], c[q][1], a[q], b[q]);
      }
      if (MODE != 1) {
#pragma unroll
        for (int q = 0; q < kGPW; ++q) {
          if (g0 + q < g_hi) {
            const int g = g0 + q, nb = g >> 2, rb = g & 3;
            double* p = &KN[(nb * 8 + 2 * fk) * kST + rb * 8 + fr];
            p[0] -= c[q][0];
            p[kST] -= c[q][1];
          }
        }
      } else {
        out[threadIdx.x] += c[0][0] + c[kGPW - 1][1];
      }
    }
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 8 + mw] = (t1 - t0) / reps;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 1 << 20);
  const int SP = 92, smem = (32 * kST + 96 * kST + 32 * SP) * 8;
  long long h[8 * 148];
  auto go = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<148, 256, smem>>>(out, cyc, 20, 11, SP, 200);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0; for (int i = 0; i < 8; ++i) m += h[i]; m /= 8;
    printf("{\"variant\": \"%s\", \"cycles_per_gemm1\": %.0f, \"err\": \"%s\"}\n", name, m, cudaGetErrorString(cudaGetLastError()));
  };
  go(probe<0>, "as_in_kernel");
  go(probe<1>, "no_writeback");
  go(probe<2>, "register_operands");
  return 0;
}
