// kid_fused.cuh -- pieces shared by the cluster kernels of kid_fused.cu (k_fused) and kid_fused_w.cu
// (k_fused_w): the per-CTA meta layout, DSMEM / mbarrier / TMA helpers, the partial-Gram reduction.
#pragma once
#include "kid_device.cuh"

namespace kid {

constexpr int kFNB = 32;     // max D column blocks per part (256 columns)
constexpr int kFMeta = 16;   // ints per (part, cta)
constexpr int kFRep = 16;    // exp-table replicas (a 64-bit load is served per half-warp)
constexpr int kFTab = kExpTab * kFRep;
constexpr double kFar = 1.0e150;  // padding source coordinate: (t - far)^2 stays finite, exp -> exactly 0
enum : int { MX_ALO = 0, MX_AC, MX_ACP, MX_OWNLO, MX_OWNNB, MX_NBS, MX_SPN, MX_MSMEM, MX_NQ, MX_SKA, MX_SRCW, MX_PEERNB };

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cl_mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// DSMEM store into the peer CTA whose completion is counted (8 bytes) on the peer's mbarrier: no fence,
// the consumer's mbarrier wait sees the data (PTX st.async, sm_90+)
__device__ __forceinline__ void st_async(uint32_t a, double v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(a), "d"(v), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t a, uint32_t bytes) {  // one arrival + bytes to come
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
// TMA bulk copy global -> this CTA's shared memory (1-D, 16-byte granules), completion counted in bytes
// on an mbarrier (SASS UBLKCP): the staging of the per-CTA source / coefficient images
__device__ __forceinline__ void tma_bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t a) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nFX_WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra FX_WAIT_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// d_out = [sum tr, sum ||K||^2, G (n x n, symmetric from the upper blocks)] from the per-cluster partials,
// summed in a fixed order (k_fx_reduce, kid_fused.cu)
int launch_fx_reduce(kid_ctx* c, const double* partial, int nchunks, int LG, int n, const double* ptr,
                      const double* psk, int nslots, double* d_out);
// the warp-tile kernel for residual / projected Grams with n <= 32 D columns (kid_fused_w.cu); returns 1 when
// the shape does not qualify
int fused_w_dev(kid_ctx* c, double h, int mode, const double* Mh, int64_t n64, double* d_out);

// K^T K by the two-phase kernel k_gram2 (kid_gram2.cu); returns 1 when its tile buffers do not fit shared memory
int gram2_dev(kid_ctx* c, double h, double* d_out);

}  // namespace kid
