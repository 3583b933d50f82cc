// kid_capi.cu -- the extern "C" boundary of libkernid_cuda.so (include/kernid_cuda.h).
// Host buffers in, host buffers out; no exceptions cross the boundary; status codes map
// onto the reference exception taxonomy (proj/include/kernid/errors.hpp:11-77).
#include <algorithm>
#include <mutex>
#include <unordered_map>
#include <cstring>
#include <new>
#include <numeric>
#include <string>
#include <vector>

#include "kid_internal.cuh"

namespace kid {

int fail(kid_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

int cuda_fail(kid_ctx* c, cudaError_t e, const char* where) {
  std::string msg = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ") at " + where;
  (void)cudaGetLastError();
  return fail(c, e == cudaErrorMemoryAllocation ? KID_E_OOM : KID_E_CUDA, msg);
}

// Device allocations of the library. A -DKID_GUARD build (tools/gpu/r02_guard.sh; compute-sanitizer is closed
// on this GPU pool) brackets every allocation with 64 KB canary zones that kid_guard_check() verifies: an
// out-of-bounds global store of any kernel within 64 KB of a library buffer shows up as a corrupted canary.
#ifdef KID_GUARD
namespace {
constexpr size_t kGuardBytes = 64 * 1024;
constexpr int kGuardByte = 0xA5;
struct GuardRec { char* base; size_t bytes; };
std::mutex g_guard_mu;
std::unordered_map<void*, GuardRec> g_guard;
}  // namespace
#endif
cudaError_t dev_malloc(void** p, size_t bytes) {
#ifdef KID_GUARD
  const size_t padded = (bytes + 255) / 256 * 256;
  char* base = nullptr;
  cudaError_t e = cudaMalloc((void**)&base, padded + 2 * kGuardBytes);
  if (e != cudaSuccess) return e;
  cudaMemset(base, kGuardByte, kGuardBytes);
  cudaMemset(base + kGuardBytes + bytes, kGuardByte, padded - bytes + kGuardBytes);
  *p = base + kGuardBytes;
  std::lock_guard<std::mutex> lk(g_guard_mu);
  g_guard[*p] = GuardRec{base, bytes};
  return cudaSuccess;
#else
  return cudaMalloc(p, bytes);
#endif
}
void dev_free(void* p) {
  if (!p) return;
#ifdef KID_GUARD
  std::lock_guard<std::mutex> lk(g_guard_mu);
  auto it = g_guard.find(p);
  if (it != g_guard.end()) {
    cudaFree(it->second.base);
    g_guard.erase(it);
    return;
  }
#endif
  cudaFree(p);
}

int ensure(kid_ctx* c, void** p, size_t* cap, size_t bytes) {
  if (*p && *cap >= bytes) return KID_OK;
  if (*p) dev_free(*p);
  *p = nullptr;
  *cap = 0;
  const size_t want = std::max<size_t>(bytes, 256);
  cudaError_t e = dev_malloc(p, want);
  if (e != cudaSuccess) {
    *p = nullptr;
    cuda_fail(c, e, "cudaMalloc");
    return KID_E_OOM;
  }
  *cap = want;
  return KID_OK;
}

int ensure_pinned(kid_ctx* c, size_t bytes) {
  if (c->hbuf && c->hbuf_cap >= bytes) return KID_OK;
  if (c->hbuf) cudaFreeHost(c->hbuf);
  c->hbuf = nullptr;
  c->hbuf_cap = 0;
  cudaError_t e = cudaMallocHost((void**)&c->hbuf, std::max<size_t>(bytes, 4096));
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaMallocHost");
  c->hbuf_cap = std::max<size_t>(bytes, 4096);
  return KID_OK;
}

void* scratch(kid_ctx* c, size_t bytes) {
  if (ensure(c, &c->scratch, &c->scratch_cap, bytes)) return nullptr;
  return c->scratch;
}

void prof_begin(kid_ctx* c) {
  if (!c->prof) return;
  if (c->prof_used + 2 > c->prof_ev.size()) {
    for (int k = 0; k < 64; ++k) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return;
      c->prof_ev.push_back(e);
    }
  }
  cudaEventRecord(c->prof_ev[c->prof_used], c->stream);
}

void prof_end(kid_ctx* c) {
  if (!c->prof || c->prof_used + 2 > c->prof_ev.size()) return;
  cudaEventRecord(c->prof_ev[c->prof_used + 1], c->stream);
  c->prof_used += 2;
}

}  // namespace kid

using namespace kid;

namespace {
// per-context output buffer for the host-facing entry points (never aliases scratch)
double* out_buffer(kid_ctx* c, size_t doubles) {
  if (ensure(c, (void**)&c->partial, &c->partial_cap, sizeof(double) * doubles)) return nullptr;
  return c->partial;
}

int set_device(kid_ctx* c) {
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaSetDevice");
  return KID_OK;
}
}  // namespace

extern "C" {

int kid_abi_version(void) { return 1; }

// Page-locked host buffers for the host-buffer entry points (a pageable destination makes the
// driver stage the copy: 8 MB of target indices D2H take ~1.8 ms pageable vs ~0.2 ms pinned).
void* kid_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes ? bytes : 1) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  return p;
}

void kid_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int kid_create(kid_ctx** out, int32_t device) {
  if (!out) return KID_E_ERROR;
  *out = nullptr;
  kid_ctx* c = new (std::nothrow) kid_ctx();
  if (!c) return KID_E_OOM;
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = dev_malloc((void**)&c->counter, sizeof(int64_t) * 8);
  if (e != cudaSuccess) {
    delete c;
    (void)cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? KID_E_OOM : KID_E_CUDA;
  }
  c->stream = c->own_stream;
  *out = c;
  return KID_OK;
}

void kid_destroy(kid_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  void* bufs[] = {c->pts_own, c->dist, c->flag, c->tgt_idx, c->blk_tgt, c->src, c->src_perm, c->P2,
                  c->scratch, c->partial, c->counter, c->sort_tmp, c->sub_idx};
  for (void* p : bufs) dev_free(p);
  if (c->hbuf) cudaFreeHost(c->hbuf);
  for (cudaEvent_t e : c->prof_ev) cudaEventDestroy(e);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  delete c;
}

const char* kid_last_error(const kid_ctx* c) { return c ? c->err.c_str() : "null context"; }

int kid_set_stream(kid_ctx* c, void* s) {
  if (!c) return KID_E_ERROR;
  c->stream = s ? (cudaStream_t)s : c->own_stream;
  return KID_OK;
}

const char* kid_last_kernel(const kid_ctx* c) { return c ? c->last_kernel : ""; }

int32_t kid_device_id(const kid_ctx* c) { return c ? c->device : -1; }

void* kid_stream(kid_ctx* c) { return c ? (void*)c->stream : nullptr; }

void* kid_device_alloc(kid_ctx* c, size_t bytes) {
  if (!c || set_device(c)) return nullptr;
  void* p = nullptr;
  if (dev_malloc(&p, bytes ? bytes : 8) != cudaSuccess) {
    cuda_fail(c, cudaGetLastError(), "kid_device_alloc");
    return nullptr;
  }
  return p;
}

void kid_device_free(kid_ctx* c, void* p) {
  if (!c || !p) return;
  set_device(c);
  dev_free(p);
}

// Corrupted canary bytes around the library's live device allocations (0 = clean); -1 when the library was
// not built with -DKID_GUARD.
int64_t kid_guard_check(kid_ctx* c) {
#ifdef KID_GUARD
  if (!c || set_device(c)) return -2;
  if (cudaDeviceSynchronize() != cudaSuccess) return -2;
  std::lock_guard<std::mutex> lk(g_guard_mu);
  int64_t bad = 0;
  std::vector<unsigned char> h;
  for (auto& kv : g_guard) {
    const GuardRec& g = kv.second;
    const size_t padded = (g.bytes + 255) / 256 * 256;
    const size_t tail = padded - g.bytes + kGuardBytes;
    h.resize(kGuardBytes + tail);
    cudaMemcpy(h.data(), g.base, kGuardBytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(h.data() + kGuardBytes, g.base + kGuardBytes + g.bytes, tail, cudaMemcpyDeviceToHost);
    for (unsigned char b : h) bad += b != (unsigned char)kGuardByte;
  }
  return bad;
#else
  (void)c;
  return -1;
#endif
}

int kid_memcpy_dtoh(kid_ctx* c, void* dst, const void* src, size_t bytes) {
  if (!c || (bytes && (!dst || !src))) return KID_E_ERROR;
  if (int rc = set_device(c)) return rc;
  KID_CK(c, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  return KID_OK;
}

int kid_set_option(kid_ctx* c, int32_t key, int64_t value) {
  if (!c) return KID_E_ERROR;
  if (key == KID_OPT_EVAL_WARPS) {
    if (value != 0 && value != 8 && value != 12) return fail(c, KID_E_RANGE, "kid_set_option: eval warps must be 0, 8 or 12");
    c->eval_warps = (int)value;
    return KID_OK;
  }
  if (key == KID_OPT_CHUNK_COLS) {
    if (value != 0 && value != 32 && value != 48 && value != 64 && value != 96)
      return fail(c, KID_E_RANGE, "kid_set_option: chunk columns must be 0, 32, 48, 64 or 96");
    c->chunk_cols = (int)value;
    return KID_OK;
  }
  if (key == KID_OPT_KERNEL) {
    if (value < 0 || value > 3) return fail(c, KID_E_RANGE, "kid_set_option: kernel must be 0, 1, 2 or 3");
    c->kernel_choice = (int)value;
    return KID_OK;
  }
  if (key == KID_OPT_TILE_WARPS) {
    if (value != 0 && value != 8 && value != 12) return fail(c, KID_E_RANGE, "kid_set_option: tile warps must be 0, 8 or 12");
    c->tile_warps = (int)value;
    return KID_OK;
  }
  if (key == KID_OPT_TILE_FORM) {
    if (value < 0 || value > 2) return fail(c, KID_E_RANGE, "kid_set_option: tile form must be 0, 1 or 2");
    c->tile_form = (int)value;
    return KID_OK;
  }
  return fail(c, KID_E_RANGE, "kid_set_option: unknown option");
}

int kid_set_path(kid_ctx* c, int32_t path) {
  if (!c) return KID_E_ERROR;
  if (path != KID_PATH_AUTO && path != KID_PATH_CLUSTER) return fail(c, KID_E_RANGE, "kid_set_path: unknown path");
  c->path = path;
  return KID_OK;
}

int kid_synchronize(kid_ctx* c) {
  if (!c) return KID_E_ERROR;
  KID_CK(c, cudaStreamSynchronize(c->stream));
  return KID_OK;
}

int64_t kid_launch_count(const kid_ctx* c) { return c ? c->launches : 0; }

int kid_profile(kid_ctx* c, int32_t enable) {
  if (!c) return KID_E_ERROR;
  c->prof = enable != 0;
  c->prof_used = 0;
  return KID_OK;
}

int kid_profile_read(kid_ctx* c, double* ms_each, int64_t cap, int64_t* count) {
  if (!c || !count) return KID_E_ERROR;
  const int64_t n = (int64_t)(c->prof_used / 2);
  for (int64_t k = 0; k < n && k < cap; ++k) {
    float ms = 0.f;
    KID_CK(c, cudaEventSynchronize(c->prof_ev[2 * k + 1]));
    KID_CK(c, cudaEventElapsedTime(&ms, c->prof_ev[2 * k], c->prof_ev[2 * k + 1]));
    if (ms_each) ms_each[k] = ms;
  }
  *count = n;
  c->prof_used = 0;
  return KID_OK;
}

int kid_set_points(kid_ctx* c, const double* host_pts, int64_t N, int32_t d, int64_t index_offset) {
  if (!c || !host_pts) return KID_E_ERROR;
  if (N < 1 || d < 1) return fail(c, KID_E_RANGE, "kid_set_points: requires N >= 1 and d >= 1");
  if (int rc = set_device(c)) return rc;
  const size_t bytes = sizeof(double) * (size_t)N * d;
  if (ensure(c, (void**)&c->pts_own, &c->pts_own_cap, bytes)) return KID_E_OOM;
  KID_CK(c, cudaMemcpyAsync(c->pts_own, host_pts, bytes, cudaMemcpyHostToDevice, c->stream));
  c->pts = c->pts_own;
  c->N = N;
  c->d = d;
  c->offset = index_offset;
  c->tbase = nullptr;
  c->nt = 0;
  return KID_OK;
}

int kid_set_points_device(kid_ctx* c, const double* dev_pts, int64_t N, int32_t d, int64_t index_offset) {
  if (!c || !dev_pts) return KID_E_ERROR;
  if (N < 1 || d < 1) return fail(c, KID_E_RANGE, "kid_set_points_device: requires N >= 1 and d >= 1");
  c->pts = dev_pts;
  c->N = N;
  c->d = d;
  c->offset = index_offset;
  c->tbase = nullptr;
  c->nt = 0;
  return KID_OK;
}

int kid_split_candidates(kid_ctx* c, const double* center, int64_t n, double* cand_dist, int64_t* cand_idx) {
  if (!c || !center || !cand_dist || !cand_idx) return KID_E_ERROR;
  if (n < 1) return fail(c, KID_E_RANGE, "split_sources_targets: requires 1 <= n < N");
  if (int rc = set_device(c)) return rc;
  return split_candidates(c, center, n, cand_dist, cand_idx);
}

int kid_split_finish(kid_ctx* c, const int64_t* src_idx, int64_t n, const double* src_points, double rho,
                     double xi, int64_t* n_targets_out) {
  if (!c || !src_idx || !n_targets_out) return KID_E_ERROR;
  if (xi < 0.0) return fail(c, KID_E_RANGE, "split_sources_targets: requires xi >= 0");
  if (int rc = set_device(c)) return rc;
  return split_finish(c, src_idx, n, src_points, rho, xi, n_targets_out);
}

int kid_split(kid_ctx* c, const double* center, int64_t n, double xi, int64_t* src_idx_out, double* rho_out,
              int64_t* n_targets_out) {
  if (!c || !center || !src_idx_out || !rho_out || !n_targets_out) return KID_E_ERROR;
  if (!c->pts) return fail(c, KID_E_ERROR, "kid_split: no point set");
  if (n < 1 || n >= c->N) return fail(c, KID_E_RANGE, "split_sources_targets: requires 1 <= n < N");
  if (xi < 0.0) return fail(c, KID_E_RANGE, "split_sources_targets: requires xi >= 0");
  if (int rc = set_device(c)) return rc;
  {
    const int rc = split_device(c, center, n, xi, src_idx_out, rho_out, n_targets_out);
    if (rc == KID_OK && *n_targets_out == 0)
      return fail(c, KID_E_NO_TARGETS,
                  "split_sources_targets: no targets at separation xi = " + std::to_string(xi) + " (try a smaller xi)");
    if (rc != 1) return rc;
  }
  std::vector<double> cd(n);
  std::vector<int64_t> ci(n);
  if (int rc = split_candidates(c, center, n, cd.data(), ci.data())) return rc;
  double rho = 0.0;  // geometry.hpp:52-53
  for (int64_t k = 0; k < n; ++k) rho = std::max(rho, cd[k]);
  std::sort(ci.begin(), ci.end());  // geometry.hpp:50-51
  int64_t nt = 0;
  if (int rc = split_finish(c, ci.data(), n, nullptr, rho, xi, &nt)) return rc;
  std::memcpy(src_idx_out, ci.data(), sizeof(int64_t) * n);
  *rho_out = rho;
  *n_targets_out = nt;
  if (nt == 0)
    return fail(c, KID_E_NO_TARGETS,
                "split_sources_targets: no targets at separation xi = " + std::to_string(xi) + " (try a smaller xi)");
  return KID_OK;
}

int kid_get_targets(kid_ctx* c, int64_t* tgt_idx_out, int64_t count) {
  if (!c || (!tgt_idx_out && count)) return KID_E_ERROR;
  if (!c->tgt_idx || count > c->n_split_targets) return fail(c, KID_E_RANGE, "kid_get_targets: count exceeds N_T");
  if (count == 0) return KID_OK;
  if (int rc = set_device(c)) return rc;
  KID_CK(c, cudaMemcpyAsync(tgt_idx_out, c->tgt_idx, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  if (c->offset)
    for (int64_t k = 0; k < count; ++k) tgt_idx_out[k] += c->offset;
  return KID_OK;
}

int kid_set_block(kid_ctx* c, const double* targets, int64_t nt, const double* sources, int64_t m, int32_t d) {
  if (!c || (!targets && nt) || !sources) return KID_E_ERROR;
  if (nt < 0 || m < 1 || d < 1) return fail(c, KID_E_RANGE, "kid_set_block: requires nt >= 0, m >= 1, d >= 1");
  if (int rc = set_device(c)) return rc;
  if (ensure(c, (void**)&c->blk_tgt, &c->blk_tgt_cap, sizeof(double) * std::max<int64_t>(nt, 1) * d)) return KID_E_OOM;
  if (ensure(c, (void**)&c->src, &c->src_cap, sizeof(double) * m * d)) return KID_E_OOM;
  if (nt) KID_CK(c, cudaMemcpyAsync(c->blk_tgt, targets, sizeof(double) * nt * d, cudaMemcpyHostToDevice, c->stream));
  KID_CK(c, cudaMemcpyAsync(c->src, sources, sizeof(double) * m * d, cudaMemcpyHostToDevice, c->stream));
  c->src_host.assign(sources, sources + (size_t)m * d);
  c->sub_active = false;
  c->tbase = c->blk_tgt;
  c->tld = nt;
  c->tidx = nullptr;
  c->nt = nt;
  c->m = m;
  c->d = d;
  c->r = 0;
  return KID_OK;
}

int kid_block_shape(const kid_ctx* c, int64_t* nt, int64_t* m, int32_t* d) {
  if (!c) return KID_E_ERROR;
  if (nt) *nt = c->nt;
  if (m) *m = c->m;
  if (d) *d = c->d;
  return KID_OK;
}

int kid_row_norms_dev(kid_ctx* c, double h, double* d_w) {
  if (!c || !d_w) return KID_E_ERROR;
  return row_norms_dev(c, h, d_w);
}

int kid_row_norms(kid_ctx* c, double h, double* w_out) {
  if (!c || (!w_out && c->nt)) return KID_E_ERROR;
  if (int rc = set_device(c)) return rc;
  double* d_w = out_buffer(c, std::max<int64_t>(c->nt, 1));
  if (!d_w) return KID_E_OOM;
  if (int rc = row_norms_dev(c, h, d_w)) return rc;
  if (c->nt) KID_CK(c, cudaMemcpyAsync(w_out, d_w, sizeof(double) * c->nt, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  return KID_OK;
}

int kid_gram_dev(kid_ctx* c, double h, double* d_G, double* d_sumsq) {
  if (!c || !d_G) return KID_E_ERROR;
  // d_G receives [sumsq_K (unused slot), sumsq_K, G (m x m)] when d_sumsq is null
  (void)d_sumsq;
  return gram_dev(c, h, 0, d_G);
}

int kid_gram(kid_ctx* c, double h, double* G_out, double* sumsq_K_out) {
  if (!c || !G_out) return KID_E_ERROR;
  if (int rc = set_device(c)) return rc;
  const int64_t m = c->m;
  double* d_out = out_buffer(c, 2 + m * m);
  if (!d_out) return KID_E_OOM;
  if (int rc = gram_dev(c, h, 0, d_out)) return rc;
  std::vector<double> tmp(2);
  KID_CK(c, cudaMemcpyAsync(tmp.data(), d_out, sizeof(double) * 2, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaMemcpyAsync(G_out, d_out + 2, sizeof(double) * m * m, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  if (sumsq_K_out) *sumsq_K_out = tmp[1];
  return KID_OK;
}

int kid_tsqr_r(kid_ctx* c, double h, double* R) {
  if (!c || !R) return KID_E_ERROR;
  if (int rc = set_device(c)) return rc;
  const int64_t m = c->m;
  double* d_R = out_buffer(c, std::max<int64_t>(m * m, 1));
  if (!d_R) return KID_E_OOM;
  if (int rc = tsqr_dev(c, h, nullptr, 0, m, d_R)) return rc;
  KID_CK(c, cudaMemcpyAsync(R, d_R, sizeof(double) * m * m, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  return KID_OK;
}

int kid_tsqr_r_dev(kid_ctx* c, double h, double* d_R) {
  if (!c || !d_R) return KID_E_ERROR;
  if (int rc = set_device(c)) return rc;
  return tsqr_dev(c, h, nullptr, 0, c->m, d_R);
}

int kid_tsqr_combine(kid_ctx* c, const double* Rs, int64_t count, int64_t m, double* R) {
  if (!c || !Rs || !R) return KID_E_ERROR;
  if (count < 1 || m < 1) return fail(c, KID_E_RANGE, "tsqr_combine: requires count >= 1 and m >= 1");
  if (int rc = set_device(c)) return rc;
  double* buf = out_buffer(c, (size_t)(count + 1) * m * m);
  if (!buf) return KID_E_OOM;
  KID_CK(c, cudaMemcpyAsync(buf, Rs, sizeof(double) * count * m * m, cudaMemcpyHostToDevice, c->stream));
  double* d_R = buf + (size_t)count * m * m;
  if (int rc = tsqr_dev(c, 0.0, buf, count, m, d_R)) return rc;
  KID_CK(c, cudaMemcpyAsync(R, d_R, sizeof(double) * m * m, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  return KID_OK;
}

int kid_proj_gram_dev(kid_ctx* c, double h, const double* d_C, int64_t n, double* d_out) {
  if (!c || !d_C || !d_out) return KID_E_ERROR;
  if (int rc = set_device(c)) return rc;
  return proj_gram_dev(c, h, d_C, n, d_out);
}

int kid_proj_gram(kid_ctx* c, double h, const double* C, int64_t n, double* sumsq_D, double* sumsq_K, double* DtD) {
  if (!c || !C || !sumsq_D || !sumsq_K) return KID_E_ERROR;
  if (int rc = set_device(c)) return rc;
  const int64_t m = c->m;
  if (n < 1 || n > m) return fail(c, KID_E_RANGE, "proj_gram: requires 1 <= n <= m");
  double* buf = out_buffer(c, m * n + 2 + n * n);
  if (!buf) return KID_E_OOM;
  double* d_C = buf;
  double* d_out = buf + m * n;
  KID_CK(c, cudaMemcpyAsync(d_C, C, sizeof(double) * m * n, cudaMemcpyHostToDevice, c->stream));
  if (int rc = proj_gram_dev(c, h, d_C, n, d_out)) return rc;
  double head[2];
  KID_CK(c, cudaMemcpyAsync(head, d_out, sizeof(head), cudaMemcpyDeviceToHost, c->stream));
  if (DtD) KID_CK(c, cudaMemcpyAsync(DtD, d_out + 2, sizeof(double) * n * n, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  *sumsq_D = head[0];
  *sumsq_K = head[1];
  return KID_OK;
}

int kid_leverage_dev(kid_ctx* c, double h, const double* d_W, int64_t r, double* d_scores) {
  if (!c || !d_W || !d_scores) return KID_E_ERROR;
  return leverage_dev(c, h, d_W, r, d_scores);
}

int kid_leverage(kid_ctx* c, double h, const double* W, int64_t r, double* scores_out) {
  if (!c || !W || (!scores_out && c->nt)) return KID_E_ERROR;
  if (r < 1 || r > c->m) return fail(c, KID_E_RANGE, "row_leverage_scores: requires 1 <= r <= min(m, n)");
  if (int rc = set_device(c)) return rc;
  const int64_t m = c->m, nt = c->nt;
  double* buf = out_buffer(c, m * r + std::max<int64_t>(nt, 1));
  if (!buf) return KID_E_OOM;
  KID_CK(c, cudaMemcpyAsync(buf, W, sizeof(double) * m * r, cudaMemcpyHostToDevice, c->stream));
  if (int rc = leverage_dev(c, h, buf, r, buf + m * r)) return rc;
  if (nt) KID_CK(c, cudaMemcpyAsync(scores_out, buf + m * r, sizeof(double) * nt, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  return KID_OK;
}

int kid_recon_prepare(kid_ctx* c, const int64_t* skel, int64_t r, const double* P) {
  if (!c || (r && (!skel || !P))) return KID_E_ERROR;
  if (!c->src || c->m < 1) return fail(c, KID_E_ERROR, "no block: call kid_split or kid_set_block");
  const int64_t m = c->m;
  if (r < 0 || r > m) return fail(c, KID_E_RANGE, "compress_id: skeleton rank out of range");
  if (int rc = set_device(c)) return rc;
  std::vector<char> seen(m, 0);
  for (int64_t l = 0; l < r; ++l) {
    if (skel[l] < 0 || skel[l] >= m || seen[skel[l]])
      return fail(c, KID_E_RANGE, "compress_id: skeleton indices must be distinct columns in [0, m)");
    seen[skel[l]] = 1;
  }
  c->skel_h.assign(skel, skel + r);
  c->nonskel.clear();
  for (int64_t j = 0; j < m; ++j)
    if (!seen[j]) c->nonskel.push_back(j);
  const int64_t meff = m - r;
  const int d = c->d;
  // permuted sources [skel | non-skel]
  std::vector<double> src_h((size_t)m * d), perm_h((size_t)m * d);
  KID_CK(c, cudaMemcpyAsync(src_h.data(), c->src, sizeof(double) * m * d, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  for (int k = 0; k < d; ++k)
    for (int64_t j = 0; j < m; ++j) {
      const int64_t orig = j < r ? skel[j] : c->nonskel[j - r];
      perm_h[j + k * m] = src_h[orig + k * m];
    }
  if (ensure(c, (void**)&c->src_perm, &c->src_perm_cap, sizeof(double) * m * d)) return KID_E_OOM;
  KID_CK(c, cudaMemcpyAsync(c->src_perm, perm_h.data(), sizeof(double) * m * d, cudaMemcpyHostToDevice, c->stream));
  c->src_perm_host = perm_h;
  // P2 = P[:, non-skel], row-major r x SP (SP = frag_stride(meff), matches k_gram)
  const int64_t SP = ((meff + 7) / 8) * 8 + 4;
  std::vector<double> p2((size_t)std::max<int64_t>(r, 1) * SP, 0.0);
  for (int64_t k = 0; k < r; ++k)
    for (int64_t n = 0; n < meff; ++n) p2[k * SP + n] = P[k + c->nonskel[n] * r];
  if (ensure(c, (void**)&c->P2, &c->P2_cap, sizeof(double) * p2.size())) return KID_E_OOM;
  KID_CK(c, cudaMemcpyAsync(c->P2, p2.data(), sizeof(double) * p2.size(), cudaMemcpyHostToDevice, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  c->P2_host = std::move(p2);
  c->r = r;
  return KID_OK;
}

// d_out = [sumsq_D, sumsq_K, D^T D over the non-skeleton columns ((m-r) x (m-r))]
int kid_recon_error_dev(kid_ctx* c, double h, uint32_t flags, double* d_out) {
  if (!c || !d_out) return KID_E_ERROR;
  if (c->r == 0 && c->skel_h.empty() && c->nonskel.empty())
    return fail(c, KID_E_ERROR, "kid_recon_error_dev: call kid_recon_prepare first");
  (void)flags;
  return gram_dev(c, h, c->r, d_out);
}

int kid_recon_error(kid_ctx* c, double h, const int64_t* skel, int64_t r, const double* P, uint32_t flags,
                    double* sumsq_D, double* sumsq_K, double* DtD, double* KtK) {
  if (!c || !sumsq_D || !sumsq_K) return KID_E_ERROR;
  if (int rc = kid_recon_prepare(c, skel, r, P)) return rc;
  const int64_t m = c->m, meff = m - r;
  double* d_out = out_buffer(c, 2 + std::max<int64_t>(meff, 1) * std::max<int64_t>(meff, 1) + 2 + m * m);
  if (!d_out) return KID_E_OOM;
  if (meff == 0) {
    // full-rank skeleton: D == 0; ||K||_F^2 still needed
    if (int rc = gram_dev(c, h, 0, d_out + 2)) return rc;
    std::vector<double> t(2);
    KID_CK(c, cudaMemcpyAsync(t.data(), d_out + 2, sizeof(double) * 2, cudaMemcpyDeviceToHost, c->stream));
    if (KtK) KID_CK(c, cudaMemcpyAsync(KtK, d_out + 4, sizeof(double) * m * m, cudaMemcpyDeviceToHost, c->stream));
    KID_CK(c, cudaStreamSynchronize(c->stream));
    *sumsq_D = 0.0;
    *sumsq_K = t[1];
    if (DtD) std::fill(DtD, DtD + m * m, 0.0);
    return KID_OK;
  }
  if (int rc = gram_dev(c, h, r, d_out)) return rc;
  std::vector<double> g(2 + meff * meff);
  KID_CK(c, cudaMemcpyAsync(g.data(), d_out, sizeof(double) * g.size(), cudaMemcpyDeviceToHost, c->stream));
  double* k_out = d_out + 2 + meff * meff;
  if (flags & KID_RECON_KTK) {
    if (int rc = gram_dev(c, h, 0, k_out)) return rc;
    if (KtK) KID_CK(c, cudaMemcpyAsync(KtK, k_out + 2, sizeof(double) * m * m, cudaMemcpyDeviceToHost, c->stream));
  }
  KID_CK(c, cudaStreamSynchronize(c->stream));
  *sumsq_D = g[0];
  *sumsq_K = g[1];
  if (DtD) {
    std::fill(DtD, DtD + m * m, 0.0);
    for (int64_t y = 0; y < meff; ++y)
      for (int64_t x = 0; x < meff; ++x) DtD[c->nonskel[x] + c->nonskel[y] * m] = g[2 + x + y * meff];
  }
  return KID_OK;
}

int kid_eval_rows(kid_ctx* c, double h, const int64_t* rows, int64_t count, double* Ks_out) {
  if (!c || (count && (!rows || !Ks_out))) return KID_E_ERROR;
  if (int rc = set_device(c)) return rc;
  for (int64_t i = 0; i < count; ++i)
    if (rows[i] < 0 || rows[i] >= c->nt) return fail(c, KID_E_RANGE, "row sample index out of range");
  const int64_t m = c->m;
  double* buf = out_buffer(c, count * m + count + 1);
  if (!buf) return KID_E_OOM;
  int64_t* d_rows = (int64_t*)(buf + count * m);
  if (count) KID_CK(c, cudaMemcpyAsync(d_rows, rows, sizeof(int64_t) * count, cudaMemcpyHostToDevice, c->stream));
  if (int rc = eval_rows_dev(c, h, d_rows, count, buf)) return rc;
  if (count) KID_CK(c, cudaMemcpyAsync(Ks_out, buf, sizeof(double) * count * m, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  return KID_OK;
}

int kid_apply_skeleton_dev(kid_ctx* c, double h, const int64_t* skel, int64_t r, const double* q_skel, double* d_u) {
  if (!c || (r && (!skel || !q_skel)) || (!d_u && c->nt)) return KID_E_ERROR;
  if (int rc = set_device(c)) return rc;
  return apply_skeleton_dev(c, h, skel, r, q_skel, d_u);
}

int kid_apply_skeleton(kid_ctx* c, double h, const int64_t* skel, int64_t r, const double* P, const double* q,
                       double* u_out) {
  if (!c || (r && (!skel || !P || !q)) || (!u_out && c->nt)) return KID_E_ERROR;
  if (int rc = set_device(c)) return rc;
  const int64_t m = c->m, nt = c->nt;
  // q_skel = P q, accumulated over the m columns of P in order (Eigen's col-major GEMV)
  std::vector<double> qs((size_t)std::max<int64_t>(r, 1), 0.0);
  for (int64_t k = 0; k < m; ++k)
    for (int64_t j = 0; j < r; ++j) qs[(size_t)j] += P[j + k * r] * q[k];
  double* buf = out_buffer(c, std::max<int64_t>(nt, 1));
  if (!buf) return KID_E_OOM;
  if (int rc = apply_skeleton_dev(c, h, skel, r, qs.data(), buf)) return rc;
  if (nt) KID_CK(c, cudaMemcpyAsync(u_out, buf, sizeof(double) * nt, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  return KID_OK;
}

int kid_select_rows(kid_ctx* c, const int64_t* rows, int64_t n) {
  if (!c || (n > 0 && !rows)) return KID_E_ERROR;
  if (int rc = set_device(c)) return rc;
  return select_rows(c, rows, n);
}

int kid_exp_check(kid_ctx* c, const double* x, int64_t n, double* y) {
  if (!c || (n && (!x || !y))) return KID_E_ERROR;
  if (int rc = set_device(c)) return rc;
  double* buf = out_buffer(c, 2 * std::max<int64_t>(n, 1));
  if (!buf) return KID_E_OOM;
  if (n) KID_CK(c, cudaMemcpyAsync(buf, x, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  if (int rc = exp_check_dev(c, buf, n, buf + n)) return rc;
  if (n) KID_CK(c, cudaMemcpyAsync(y, buf + n, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  KID_CK(c, cudaStreamSynchronize(c->stream));
  return KID_OK;
}

}  // extern "C"
