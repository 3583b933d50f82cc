/*
 * kernid_oracle.c -- CPU ORACLE (test infrastructure only; see kernid_oracle.h).
 *
 * Plain-C restatement of the reference far-field path. Every function cites the
 * reference file:line it restates (paths relative to /root/reference/proj/include/kernid/).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/--impl reference
 * legs may load this library. Build: oracle/Makefile (-O2 -ffp-contract=off).
 */
#include "kernid_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------ rng.hpp */

/* rng.hpp:19-24 */
uint64_t or_splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* rng.hpp:28-33 */
uint64_t or_derive_seed(uint64_t master, uint64_t key_a, uint64_t key_b) {
  uint64_t state = master;
  state ^= or_splitmix64(&state) + key_a;
  state ^= or_splitmix64(&state) + key_b;
  return or_splitmix64(&state);
}

/* std::mt19937_64 as specified by the C++ standard ([rand.eng.mers]); rng.hpp:75 */
#define MT_N 312
#define MT_M 156
void or_rng_init(or_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
  r->has_spare = 0;
  r->spare = 0.0;
}

uint64_t or_rng_next(or_rng* r) {
  static const uint64_t UPPER = 0xFFFFFFFF80000000ull, LOWER = 0x7FFFFFFFull;
  if (r->idx >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      uint64_t x = (r->mt[i] & UPPER) | (r->mt[(i + 1) % MT_N] & LOWER);
      uint64_t xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:43 */
double or_rng_uniform01(or_rng* r) { return (double)(or_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:49-56 */
uint64_t or_rng_below(or_rng* r, uint64_t n) {
  const uint64_t limit = n * ((~(uint64_t)0) / n);
  uint64_t x;
  do {
    x = or_rng_next(r);
  } while (x >= limit);
  return x % n;
}

/* rng.hpp:59-72 */
double or_rng_normal(or_rng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  const double u1 = 1.0 - or_rng_uniform01(r);
  const double u2 = or_rng_uniform01(r);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * M_PI * u2;
  r->spare = radius * sin(angle);
  r->has_spare = 1;
  return radius * cos(angle);
}

void or_rng_dump(uint64_t seed, int64_t n, uint64_t* u64, double* unif, double* normal,
                 uint64_t below_n, uint64_t* below) {
  or_rng r;
  or_rng_init(&r, seed);
  for (int64_t i = 0; i < n; ++i) u64[i] = or_rng_next(&r);
  or_rng_init(&r, seed);
  for (int64_t i = 0; i < n; ++i) unif[i] = or_rng_uniform01(&r);
  or_rng_init(&r, seed);
  for (int64_t i = 0; i < n; ++i) normal[i] = or_rng_normal(&r);
  or_rng_init(&r, seed);
  for (int64_t i = 0; i < n; ++i) below[i] = or_rng_below(&r, below_n);
}

/* -------------------------------------------------------------- datagen.hpp */

/* datagen.hpp:35-43: ps(i, j) filled point-major into a col-major N x d matrix */
int or_gen_normal(int32_t d, int64_t N, uint64_t seed, double* out) {
  if (d < 1 || N < 1) return 1;
  or_rng r;
  or_rng_init(&r, seed);
  for (int64_t i = 0; i < N; ++i)
    for (int32_t j = 0; j < d; ++j) out[i + (int64_t)j * N] = or_rng_normal(&r);
  return 0;
}

/* --------------------------------------------------------------- kernel.hpp */

/* kernel.hpp:119-123 */
double or_silverman_bandwidth(int32_t d, int64_t N) {
  if (d < 1 || N < 1) return -1.0;
  const double e = 1.0 / ((double)d + 4.0);
  return pow(4.0 / (2.0 * d + 1.0), e) * pow((double)N, -e);
}

/* harness.hpp:95-100 */
int64_t or_random_center_index(int64_t N, uint64_t data_seed) {
  or_rng r;
  or_rng_init(&r, or_derive_seed(data_seed, 0xCE, 0));
  return (int64_t)or_rng_below(&r, (uint64_t)N);
}

/* ------------------------------------------------------------- geometry.hpp */

/* ordering (dist, idx) of geometry.hpp:39-45 */
static int key_less(double da, int64_t a, double db, int64_t b) {
  if (da != db) return da < db;
  return a < b;
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

/* geometry.hpp:29-65. dist(i) = (ps.row(i)^T - x_c).norm(): a strided row has no
 * packet access, so Eigen reduces it left to right (kernel.hpp:60-68 discipline). */
int or_split(const double* pts, int64_t N, int32_t d, const double* center, int64_t n, double xi,
             int64_t* src_idx, int64_t* tgt_idx, int64_t* n_tgt, double* rho, double* dist_out) {
  if (n < 1 || n >= N) return 1;
  if (xi < 0.0) return 1;
  double* dist = dist_out ? dist_out : (double*)malloc(sizeof(double) * (size_t)N);
  for (int64_t i = 0; i < N; ++i) {
    double diff = pts[i] - center[0];
    double acc = diff * diff;
    for (int32_t k = 1; k < d; ++k) {
      diff = pts[i + (int64_t)k * N] - center[k];
      acc += diff * diff;
    }
    dist[i] = sqrt(acc);
  }
  /* n smallest by (dist, idx): bounded max-heap (same set as nth_element, :39-45) */
  int64_t* heap = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t hs = 0;
  for (int64_t i = 0; i < N; ++i) {
    if (hs < n) {
      int64_t c = hs++;
      heap[c] = i;
      while (c > 0) {
        int64_t p = (c - 1) / 2;
        if (key_less(dist[heap[p]], heap[p], dist[heap[c]], heap[c])) {
          int64_t t = heap[p]; heap[p] = heap[c]; heap[c] = t; c = p;
        } else break;
      }
    } else if (key_less(dist[i], i, dist[heap[0]], heap[0])) {
      heap[0] = i;
      int64_t c = 0;
      for (;;) {
        int64_t l = 2 * c + 1, rr = l + 1, big = c;
        if (l < n && key_less(dist[heap[big]], heap[big], dist[heap[l]], heap[l])) big = l;
        if (rr < n && key_less(dist[heap[big]], heap[big], dist[heap[rr]], heap[rr])) big = rr;
        if (big == c) break;
        int64_t t = heap[big]; heap[big] = heap[c]; heap[c] = t; c = big;
      }
    }
  }
  memcpy(src_idx, heap, sizeof(int64_t) * (size_t)n);
  free(heap);
  qsort(src_idx, (size_t)n, sizeof(int64_t), cmp_i64); /* :50-51 */
  double r = 0.0;                                       /* :52-53 */
  for (int64_t k = 0; k < n; ++k) r = (r < dist[src_idx[k]]) ? dist[src_idx[k]] : r;
  *rho = r;
  const double cutoff = xi * r; /* :57 */
  int64_t cnt = 0, s = 0;
  for (int64_t i = 0; i < N; ++i) { /* :58-60, sources are sorted: merge-walk */
    while (s < n && src_idx[s] < i) ++s;
    const int is_source = (s < n && src_idx[s] == i);
    if (!is_source && dist[i] >= cutoff) tgt_idx[cnt++] = i;
  }
  *n_tgt = cnt;
  if (!dist_out) free(dist);
  return cnt == 0 ? 3 : 0; /* :61-63 NoTargetsError */
}

void or_gather_points(const double* pts, int64_t N, int32_t d, const int64_t* idx, int64_t count,
                      double* out) {
  for (int32_t k = 0; k < d; ++k)
    for (int64_t i = 0; i < count; ++i) out[i + (int64_t)k * count] = pts[idx[i] + (int64_t)k * N];
}

/* kernel.hpp:60-68 + 77-79 : acc from 0.0, sequential, then exp(-sq / (2.0*h*h)) */
static inline double sqdist_strided(const double* a, int64_t sa, const double* b, int64_t sb,
                                    int32_t d) {
  double acc = 0.0;
  for (int32_t k = 0; k < d; ++k) {
    const double diff = a[k * sa] - b[k * sb];
    acc += diff * diff;
  }
  return acc;
}

double or_eval_gaussian(const double* x, const double* y, int32_t d, double h) {
  return exp(-sqdist_strided(x, 1, y, 1, d) / (2.0 * h * h));
}

/* parallel_for_rows (util.hpp:21-44): fixed partition of rows into min(rows/1024, 4*hw) blocks */
typedef struct {
  const double* tgt;
  int64_t nt;
  const double* src;
  int64_t m;
  int32_t d;
  double h;
  double* K;
  int64_t nblocks;
  atomic_llong next;
} km_job;

static void km_rows(km_job* j, int64_t lo, int64_t hi) {
  /* kernel.hpp:134-146 then :164-172 fused per row (identical per-entry arithmetic) */
  for (int64_t i = lo; i < hi; ++i)
    for (int64_t c = 0; c < j->m; ++c) {
      const double sq = sqdist_strided(j->tgt + i, j->nt, j->src + c, j->m, j->d);
      j->K[i + c * j->nt] = exp(-sq / (2.0 * j->h * j->h));
    }
}

static void* km_worker(void* arg) {
  km_job* j = (km_job*)arg;
  for (;;) {
    const int64_t b = atomic_fetch_add(&j->next, 1);
    if (b >= j->nblocks) return NULL;
    km_rows(j, j->nt * b / j->nblocks, j->nt * (b + 1) / j->nblocks);
  }
}

void or_kernel_matrix(const double* tgt, int64_t nt, const double* src, int64_t m, int32_t d,
                      double h, double* K, int32_t threads) {
  long hw = threads > 0 ? threads : sysconf(_SC_NPROCESSORS_ONLN);
  if (hw < 1) hw = 1;
  int64_t nblocks = nt / 1024;
  if (nblocks > 4 * hw) nblocks = 4 * hw;
  if (nblocks < 1) nblocks = 1;
  km_job j = {tgt, nt, src, m, d, h, K, nblocks, 0};
  if (nblocks == 1 || hw == 1) {
    km_rows(&j, 0, nt);
    return;
  }
  pthread_t* pool = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)hw);
  for (long t = 0; t < hw; ++t) pthread_create(&pool[t], NULL, km_worker, &j);
  for (long t = 0; t < hw; ++t) pthread_join(pool[t], NULL);
  free(pool);
}

/* ------------------------------------------------------------- sampling.hpp */

/* sampling.hpp:68-72 */
int64_t or_sample_count(double s, int64_t m) {
  if (!(s > 0.0 && s <= 1.0)) return -1;
  int64_t c = (int64_t)ceil(s * (double)m);
  if (c > m) c = m;
  return c < 1 ? 1 : c;
}

/* sampling.hpp:189-196: strided row norm, sequential */
void or_row_norms(const double* K, int64_t nt, int64_t m, double* w) {
  for (int64_t i = 0; i < nt; ++i) {
    double acc = K[i] * K[i];
    for (int64_t j = 1; j < m; ++j) acc += K[i + j * nt] * K[i + j * nt];
    w[i] = sqrt(acc);
  }
}

/* WeightTree (sampling.hpp:78-104) */
typedef struct {
  size_t n;
  double* tree;
} wtree;
static void wt_add(wtree* t, size_t i, double delta) {
  for (size_t k = i + 1; k <= t->n; k += k & (~k + 1)) t->tree[k] += delta;
}
static size_t wt_find(const wtree* t, double u) {
  size_t pos = 0, mask = 1;
  while ((mask << 1) <= t->n) mask <<= 1;
  for (; mask > 0; mask >>= 1) {
    const size_t next = pos + mask;
    if (next <= t->n && t->tree[next] <= u) {
      u -= t->tree[next];
      pos = next;
    }
  }
  return pos < t->n - 1 ? pos : t->n - 1;
}

/* weighted_draw (sampling.hpp:108-149) */
int or_weighted_draw(const double* w, int64_t n, int64_t count, int32_t replacement, or_rng* rng,
                     int64_t* out) {
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) total += w[i];
  for (int64_t i = 0; i < n; ++i)
    if (w[i] < 0.0 || !isfinite(w[i])) return 1;
  if (!(total > 0.0)) return 5;
  if (replacement) {
    double* cum = (double*)malloc(sizeof(double) * (size_t)n);
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) cum[i] = (acc += w[i]);
    for (int64_t k = 0; k < count; ++k) {
      const double u = or_rng_uniform01(rng) * total;
      int64_t lo = 0, hi = n; /* upper_bound */
      while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (u < cum[mid]) hi = mid; else lo = mid + 1;
      }
      out[k] = lo >= n ? n - 1 : lo;
    }
    free(cum);
    return 0;
  }
  wtree t = {(size_t)n, (double*)calloc((size_t)n + 1, sizeof(double))};
  for (int64_t i = 0; i < n; ++i) wt_add(&t, (size_t)i, w[i]);
  double* live = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(live, w, sizeof(double) * (size_t)n);
  int rc = 0;
  for (int64_t k = 0; k < count; ++k) {
    const double u = or_rng_uniform01(rng) * total;
    size_t idx = wt_find(&t, u);
    if (live[idx] <= 0.0) {
      size_t probe = idx;
      while (probe + 1 < (size_t)n && live[probe] <= 0.0) ++probe;
      while (probe > 0 && live[probe] <= 0.0) --probe;
      idx = probe;
    }
    out[k] = (int64_t)idx;
    total -= live[idx];
    wt_add(&t, idx, -live[idx]);
    live[idx] = 0.0;
    if (!(total > 0.0) && k + 1 < count) { rc = 5; break; }
  }
  free(t.tree);
  free(live);
  return rc;
}

/* sample_rows (sampling.hpp:156-243) for the BASELINE schemes */
int64_t or_sample_rows(int32_t kind, int32_t replacement, int64_t m, const double* weights, double s,
                       uint64_t seed, int64_t* out) {
  if (m < 1) return -1;
  or_rng rng;
  or_rng_init(&rng, seed);
  if (kind == 1) { /* Bernoulli (sampling.hpp:183-188): out must hold m entries */
    if (!(s > 0.0 && s <= 1.0)) return -1;
    int64_t cnt = 0;
    for (int64_t i = 0; i < m; ++i)
      if (or_rng_uniform01(&rng) < s) out[cnt++] = i;
    return cnt;
  }
  const int64_t count = or_sample_count(s, m);
  if (count < 0) return -1;
  if (kind == 0) { /* :166-182 */
    if (replacement) {
      for (int64_t k = 0; k < count; ++k) out[k] = (int64_t)or_rng_below(&rng, (uint64_t)m);
    } else {
      int64_t* pool = (int64_t*)malloc(sizeof(int64_t) * (size_t)m);
      for (int64_t i = 0; i < m; ++i) pool[i] = i;
      for (int64_t k = 0; k < count; ++k) {
        const int64_t j = k + (int64_t)or_rng_below(&rng, (uint64_t)(m - k));
        int64_t t = pool[k]; pool[k] = pool[j]; pool[j] = t;
        out[k] = pool[k];
      }
      free(pool);
    }
    return count;
  }
  if (kind == 2 || kind == 4) { /* :189-196, :212-221 */
    const int rc = or_weighted_draw(weights, m, count, kind == 2 ? replacement : 0, &rng, out);
    return rc ? -(int64_t)(rc == 1 ? 1 : 5) : count;
  }
  return -1;
}

/* -------------------------------------------------------------- lowrank.hpp */

/* Householder QR (stand-in for Eigen::HouseholderQR, lowrank.hpp:60-65). A is copied. */
void or_qr_r(const double* A_in, int64_t rows, int64_t cols, double* R) {
  double* A = (double*)malloc(sizeof(double) * (size_t)(rows * cols));
  memcpy(A, A_in, sizeof(double) * (size_t)(rows * cols));
  double* v = (double*)malloc(sizeof(double) * (size_t)rows);
  for (int64_t j = 0; j < cols; ++j) {
    double* cj = A + j * rows;
    const int64_t len = rows - j;
    double nrm = 0.0;
    for (int64_t i = j; i < rows; ++i) nrm += cj[i] * cj[i];
    nrm = sqrt(nrm);
    if (nrm == 0.0) continue;
    const double alpha = cj[j];
    const double beta = alpha >= 0.0 ? -nrm : nrm;
    const double v0 = alpha - beta;
    const double tau = -v0 / beta;
    v[0] = 1.0;
    for (int64_t i = 1; i < len; ++i) v[i] = cj[j + i] / v0;
    cj[j] = beta;
    for (int64_t i = 1; i < len; ++i) cj[j + i] = 0.0;
    for (int64_t k = j + 1; k < cols; ++k) {
      double* ck = A + k * rows + j;
      double w = 0.0;
      for (int64_t i = 0; i < len; ++i) w += v[i] * ck[i];
      w *= tau;
      for (int64_t i = 0; i < len; ++i) ck[i] -= w * v[i];
    }
  }
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t r = 0; r < cols; ++r) R[r + c * cols] = (r <= c) ? A[r + c * rows] : 0.0;
  free(v);
  free(A);
}

/* One-sided Jacobi SVD (stand-in for Eigen::BDCSVD, lowrank.hpp:70-90) */
void or_jacobi_svd(const double* A_in, int64_t n, double* sv, double* V_out) {
  double* U = (double*)malloc(sizeof(double) * (size_t)(n * n));
  double* V = (double*)calloc((size_t)(n * n), sizeof(double));
  memcpy(U, A_in, sizeof(double) * (size_t)(n * n));
  for (int64_t i = 0; i < n; ++i) V[i + i * n] = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    int64_t rotated = 0;
    for (int64_t p = 0; p < n - 1; ++p)
      for (int64_t q = p + 1; q < n; ++q) {
        double* up = U + p * n;
        double* uq = U + q * n;
        double a = 0.0, b = 0.0, g = 0.0;
        for (int64_t i = 0; i < n; ++i) {
          a += up[i] * up[i];
          b += uq[i] * uq[i];
          g += up[i] * uq[i];
        }
        if (g == 0.0 || fabs(g) <= 1e-15 * sqrt(a) * sqrt(b)) continue;
        ++rotated;
        const double zeta = (b - a) / (2.0 * g);
        double t;
        if (fabs(zeta) > 1e150) t = 0.5 / zeta;
        else t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int64_t i = 0; i < n; ++i) {
          const double x = up[i], y = uq[i];
          up[i] = c * x - s * y;
          uq[i] = s * x + c * y;
        }
        double* vp = V + p * n;
        double* vq = V + q * n;
        for (int64_t i = 0; i < n; ++i) {
          const double x = vp[i], y = vq[i];
          vp[i] = c * x - s * y;
          vq[i] = s * x + c * y;
        }
      }
    if (rotated == 0) break;
  }
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  double* s = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t j = 0; j < n; ++j) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += U[i + j * n] * U[i + j * n];
    s[j] = sqrt(acc);
    order[j] = j;
  }
  for (int64_t i = 1; i < n; ++i) { /* stable insertion sort, descending */
    int64_t o = order[i], k = i - 1;
    while (k >= 0 && s[order[k]] < s[o]) { order[k + 1] = order[k]; --k; }
    order[k + 1] = o;
  }
  for (int64_t j = 0; j < n; ++j) {
    sv[j] = s[order[j]];
    if (V_out) memcpy(V_out + j * n, V + order[j] * n, sizeof(double) * (size_t)n);
  }
  free(order); free(s); free(U); free(V);
}

static void transpose(const double* A, int64_t rows, int64_t cols, double* T) {
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t r = 0; r < rows; ++r) T[c + r * cols] = A[r + c * rows];
}

/* singular_values (lowrank.hpp:70-77): QR reduction to the small side, then SVD */
void or_singular_values(const double* A, int64_t rows, int64_t cols, double* sv) {
  const int64_t k = rows < cols ? rows : cols;
  double* R = (double*)malloc(sizeof(double) * (size_t)(k * k));
  if (rows >= cols) {
    or_qr_r(A, rows, cols, R);
  } else {
    double* T = (double*)malloc(sizeof(double) * (size_t)(rows * cols));
    transpose(A, rows, cols, T);
    or_qr_r(T, cols, rows, R);
    free(T);
  }
  or_jacobi_svd(R, k, sv, NULL);
  free(R);
}

/* right_factor (lowrank.hpp:81-90), rows >= cols */
void or_right_factor(const double* A, int64_t rows, int64_t cols, double* sv, double* V) {
  double* R = (double*)malloc(sizeof(double) * (size_t)(cols * cols));
  or_qr_r(A, rows, cols, R);
  or_jacobi_svd(R, cols, sv, V);
  free(R);
}

/* epsilon_rank (lowrank.hpp:117-126) */
int64_t or_epsilon_rank(const double* sv, int64_t n, double eps, double ref_sigma1) {
  if (!(eps > 0.0 && eps < 1.0)) return -1;
  if (n == 0) return 0;
  const double ref = ref_sigma1 > 0.0 ? ref_sigma1 : sv[0];
  if (!(ref > 0.0)) return 0;
  for (int64_t r = 0; r < n; ++r)
    if (sv[r] < eps * ref) return r;
  return n;
}

/* row_leverage_scores (lowrank.hpp:296-308) */
int or_row_leverage_scores(const double* A, int64_t rows, int64_t cols, int64_t r, double* scores,
                           int32_t* degenerate_gap) {
  const int64_t mn = rows < cols ? rows : cols;
  if (r < 1 || r > mn || rows < cols) return 1;
  double* sv = (double*)malloc(sizeof(double) * (size_t)cols);
  double* V = (double*)malloc(sizeof(double) * (size_t)(cols * cols));
  or_right_factor(A, rows, cols, sv, V);
  if (!(sv[r - 1] > 0.0)) { free(sv); free(V); return 4; }
  double* W = (double*)malloc(sizeof(double) * (size_t)(cols * r)); /* :304 */
  for (int64_t j = 0; j < r; ++j)
    for (int64_t i = 0; i < cols; ++i) W[i + j * cols] = V[i + j * cols] * (1.0 / sv[j]);
  for (int64_t i = 0; i < rows; ++i) { /* :305 */
    double acc = 0.0;
    for (int64_t j = 0; j < r; ++j) {
      double t = 0.0;
      for (int64_t l = 0; l < cols; ++l) t += A[i + l * rows] * W[l + j * cols];
      acc += t * t;
    }
    scores[i] = acc;
  }
  *degenerate_gap = (r < cols) && (sv[r - 1] - sv[r] <= 1e-12 * sv[r - 1]); /* :306 */
  free(W); free(sv); free(V);
  return 0;
}

/* CpqrWorkspace (lowrank.hpp:135-198) restated with sequential reductions */
typedef struct {
  double* W;
  int64_t m, n;
  double* tau;
  int64_t* perm;
  double* colnorm2;
  double* refnorm2;
  int64_t steps;
} cpqr;

static void cpqr_init(cpqr* ws, const double* A, int64_t m, int64_t n) {
  ws->m = m; ws->n = n; ws->steps = 0;
  ws->W = (double*)malloc(sizeof(double) * (size_t)(m * n));
  memcpy(ws->W, A, sizeof(double) * (size_t)(m * n));
  const int64_t k = m < n ? m : n;
  ws->tau = (double*)calloc((size_t)(k > 0 ? k : 1), sizeof(double));
  ws->perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  ws->colnorm2 = (double*)malloc(sizeof(double) * (size_t)n);
  ws->refnorm2 = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t j = 0; j < n; ++j) {
    ws->perm[j] = j;
    double acc = 0.0;
    for (int64_t i = 0; i < m; ++i) acc += ws->W[i + j * m] * ws->W[i + j * m];
    ws->colnorm2[j] = acc;
    ws->refnorm2[j] = acc;
  }
}

static void cpqr_free(cpqr* ws) {
  free(ws->W); free(ws->tau); free(ws->perm); free(ws->colnorm2); free(ws->refnorm2);
}

static void cpqr_run(cpqr* ws, int64_t max_steps) {
  const int64_t m = ws->m, n = ws->n;
  int64_t kmax = max_steps;
  if (m < kmax) kmax = m;
  if (n < kmax) kmax = n;
  const double recompute_ratio = 2.3e-16; /* :154 */
  double* W = ws->W;
  double* v = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  double* w = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  while (ws->steps < kmax) {
    const int64_t k = ws->steps;
    int64_t piv = k; /* :157-159, ties to the lowest index */
    for (int64_t j = k + 1; j < n; ++j)
      if (ws->colnorm2[j] > ws->colnorm2[piv]) piv = j;
    if (piv != k) { /* :160-165 */
      for (int64_t i = 0; i < m; ++i) {
        const double t = W[i + k * m]; W[i + k * m] = W[i + piv * m]; W[i + piv * m] = t;
      }
      double t = ws->colnorm2[k]; ws->colnorm2[k] = ws->colnorm2[piv]; ws->colnorm2[piv] = t;
      t = ws->refnorm2[k]; ws->refnorm2[k] = ws->refnorm2[piv]; ws->refnorm2[piv] = t;
      const int64_t p = ws->perm[k]; ws->perm[k] = ws->perm[piv]; ws->perm[piv] = p;
    }
    const int64_t len = m - k;
    double normx = 0.0; /* :167 */
    for (int64_t i = k; i < m; ++i) normx += W[i + k * m] * W[i + k * m];
    normx = sqrt(normx);
    if (normx == 0.0) { /* :168-172 */
      ws->tau[k] = 0.0;
      ++ws->steps;
      continue;
    }
    const double alpha = W[k + k * m]; /* :173-178 */
    const double beta = (alpha >= 0.0) ? -normx : normx;
    const double v0 = alpha - beta;
    ws->tau[k] = -v0 / beta;
    for (int64_t i = 1; i < len; ++i) W[k + i + k * m] /= v0;
    W[k + k * m] = beta;
    if (k + 1 < n && len > 0) { /* :179-186 */
      v[0] = 1.0;
      for (int64_t i = 1; i < len; ++i) v[i] = W[k + i + k * m];
      for (int64_t j = k + 1; j < n; ++j) {
        double acc = 0.0;
        for (int64_t i = 0; i < len; ++i) acc += v[i] * W[k + i + j * m];
        w[j] = ws->tau[k] * acc;
      }
      for (int64_t j = k + 1; j < n; ++j)
        for (int64_t i = 0; i < len; ++i) W[k + i + j * m] -= v[i] * w[j];
    }
    for (int64_t j = k + 1; j < n; ++j) { /* :187-194 */
      const double t = W[k + j * m];
      ws->colnorm2[j] -= t * t;
      if (ws->colnorm2[j] < recompute_ratio * ws->refnorm2[j] || ws->colnorm2[j] < 0.0) {
        double acc = 0.0;
        for (int64_t i = k + 1; i < m; ++i) acc += W[i + j * m] * W[i + j * m];
        ws->colnorm2[j] = (m - k - 1 > 0) ? acc : 0.0;
        ws->refnorm2[j] = ws->colnorm2[j];
      }
    }
    ++ws->steps;
  }
  free(v);
  free(w);
}

/* interpolative_decomposition (lowrank.hpp:235-262) */
int or_interpolative_decomposition(const double* A, int64_t m, int64_t n, int64_t r, int64_t* skel,
                                   double* P) {
  const int64_t mn = m < n ? m : n;
  if (r < 1 || r > mn) return 1;
  cpqr ws;
  cpqr_init(&ws, A, m, n);
  cpqr_run(&ws, r);
  const double lead = fabs(ws.W[0]);
  const double tail = fabs(ws.W[(r - 1) + (r - 1) * m]);
  if (!(lead > 0.0) || tail < 10.0 * 2.220446049250313080847e-16 * lead) {
    cpqr_free(&ws);
    return 8;
  }
  for (int64_t i = 0; i < r; ++i) skel[i] = ws.perm[i];
  memset(P, 0, sizeof(double) * (size_t)(r * n));
  for (int64_t i = 0; i < r; ++i) P[i + ws.perm[i] * r] = 1.0;
  if (r < n) { /* R11 P2 = R12, column-oriented back substitution */
    double* x = (double*)malloc(sizeof(double) * (size_t)r);
    for (int64_t j = 0; j < n - r; ++j) {
      for (int64_t i = 0; i < r; ++i) x[i] = ws.W[i + (r + j) * m];
      for (int64_t i = r - 1; i >= 0; --i) {
        x[i] /= ws.W[i + i * m];
        for (int64_t k = 0; k < i; ++k) x[k] -= x[i] * ws.W[k + i * m];
      }
      const int64_t col = ws.perm[r + j];
      for (int64_t i = 0; i < r; ++i) P[i + col * r] = x[i];
    }
    free(x);
  }
  cpqr_free(&ws);
  return 0;
}

/* power_iteration_norm (lowrank.hpp:320-348) with matvec/rmatvec callbacks */
typedef void (*mv_fn)(const void* ctx, const double* x, double* y);
static double power_iteration(mv_fn mv, mv_fn rmv, const void* ctx, int64_t rows, int64_t ncols,
                              double rel_tol, int32_t max_iters) {
  double* x = (double*)malloc(sizeof(double) * (size_t)ncols);
  double* y = (double*)malloc(sizeof(double) * (size_t)rows);
  uint64_t state = 0x9E3779B97F4A7C15ull;
  for (int64_t i = 0; i < ncols; ++i) {
    state ^= state << 13;
    state ^= state >> 7;
    state ^= state << 17;
    x[i] = (double)(state >> 11) * 0x1.0p-53 - 0.5;
  }
  double nx = 0.0;
  for (int64_t i = 0; i < ncols; ++i) nx += x[i] * x[i];
  nx = sqrt(nx);
  for (int64_t i = 0; i < ncols; ++i) x[i] /= nx;
  double last = 0.0, result = 0.0;
  int done = 0;
  for (int32_t it = 0; it < max_iters && !done; ++it) {
    mv(ctx, x, y);
    double est = 0.0;
    for (int64_t i = 0; i < rows; ++i) est += y[i] * y[i];
    est = sqrt(est);
    if (est == 0.0) { result = 0.0; done = 1; break; }
    rmv(ctx, y, x);
    double xn = 0.0;
    for (int64_t i = 0; i < ncols; ++i) xn += x[i] * x[i];
    xn = sqrt(xn);
    if (xn == 0.0) { result = est; done = 1; break; }
    for (int64_t i = 0; i < ncols; ++i) x[i] /= xn;
    if (it > 0 && fabs(est - last) <= rel_tol * est) { result = est; done = 1; break; }
    last = est;
  }
  if (!done) result = last;
  free(x);
  free(y);
  return result;
}

typedef struct { const double* A; int64_t rows, cols; } dense_op;
static void dense_mv(const void* c, const double* x, double* y) {
  const dense_op* o = (const dense_op*)c;
  for (int64_t i = 0; i < o->rows; ++i) y[i] = 0.0;
  for (int64_t j = 0; j < o->cols; ++j)
    for (int64_t i = 0; i < o->rows; ++i) y[i] += o->A[i + j * o->rows] * x[j];
}
static void dense_rmv(const void* c, const double* y, double* x) {
  const dense_op* o = (const dense_op*)c;
  for (int64_t j = 0; j < o->cols; ++j) {
    double acc = 0.0;
    for (int64_t i = 0; i < o->rows; ++i) acc += o->A[i + j * o->rows] * y[i];
    x[j] = acc;
  }
}

double or_power_iteration_norm(const double* A, int64_t rows, int64_t cols, double tol, int32_t cap) {
  dense_op o = {A, rows, cols};
  return power_iteration(dense_mv, dense_rmv, &o, rows, cols, tol, cap);
}

/* spectral_norm_exact (lowrank.hpp:359) */
double or_spectral_norm_exact(const double* A, int64_t rows, int64_t cols) {
  const int64_t k = rows < cols ? rows : cols;
  double* sv = (double*)malloc(sizeof(double) * (size_t)k);
  or_singular_values(A, rows, cols, sv);
  const double s = sv[0];
  free(sv);
  return s;
}

/* ------------------------------------------------------------- compress.hpp */

/* NormPolicy::exact_allowed (compress.hpp:51-54) */
static int exact_allowed(int64_t rows, int64_t cols, double budget) {
  const int64_t mn = rows < cols ? rows : cols;
  return mn <= 1000 && (double)rows * (double)cols <= budget;
}

typedef struct {
  const double* K;
  int64_t nt, m, r;
  const int64_t* skel;
  const double* P;
  double* tmp; /* r */
} recon_op;

/* matvec x -> C (P x) - K x (compress.hpp:149) */
static void recon_mv(const void* c, const double* x, double* y) {
  const recon_op* o = (const recon_op*)c;
  for (int64_t l = 0; l < o->r; ++l) {
    double acc = 0.0;
    for (int64_t j = 0; j < o->m; ++j) acc += o->P[l + j * o->r] * x[j];
    o->tmp[l] = acc;
  }
  for (int64_t i = 0; i < o->nt; ++i) y[i] = 0.0;
  for (int64_t l = 0; l < o->r; ++l)
    for (int64_t i = 0; i < o->nt; ++i) y[i] += o->K[i + o->skel[l] * o->nt] * o->tmp[l];
  for (int64_t j = 0; j < o->m; ++j)
    for (int64_t i = 0; i < o->nt; ++i) y[i] -= o->K[i + j * o->nt] * x[j];
}
/* rmatvec y -> P^T (C^T y) - K^T y (compress.hpp:150-152) */
static void recon_rmv(const void* c, const double* y, double* x) {
  const recon_op* o = (const recon_op*)c;
  for (int64_t l = 0; l < o->r; ++l) {
    double acc = 0.0;
    for (int64_t i = 0; i < o->nt; ++i) acc += o->K[i + o->skel[l] * o->nt] * y[i];
    o->tmp[l] = acc;
  }
  for (int64_t j = 0; j < o->m; ++j) {
    double a = 0.0;
    for (int64_t l = 0; l < o->r; ++l) a += o->P[l + j * o->r] * o->tmp[l];
    double b = 0.0;
    for (int64_t i = 0; i < o->nt; ++i) b += o->K[i + j * o->nt] * y[i];
    x[j] = a - b;
  }
}

/* reconstruction_error_norm (compress.hpp:141-154) */
double or_reconstruction_error_norm(const double* K, int64_t nt, int64_t m, const int64_t* skel,
                                    int64_t r, const double* P, double budget, double tol,
                                    int32_t cap) {
  if (exact_allowed(nt, m, budget)) {
    double* diff = (double*)malloc(sizeof(double) * (size_t)(nt * m));
    for (int64_t j = 0; j < m; ++j) { /* diff = C * P; diff -= K */
      double* dj = diff + j * nt;
      for (int64_t i = 0; i < nt; ++i) dj[i] = 0.0;
      for (int64_t l = 0; l < r; ++l) {
        const double p = P[l + j * r];
        const double* cl = K + skel[l] * nt;
        for (int64_t i = 0; i < nt; ++i) dj[i] += cl[i] * p;
      }
      const double* kj = K + j * nt;
      for (int64_t i = 0; i < nt; ++i) dj[i] -= kj[i];
    }
    const double s = or_spectral_norm_exact(diff, nt, m);
    free(diff);
    return s;
  }
  double* tmp = (double*)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1));
  recon_op o = {K, nt, m, r, skel, P, tmp};
  const double s = power_iteration(recon_mv, recon_rmv, &o, nt, m, tol, cap);
  free(tmp);
  return s;
}

/* matrix_norm (compress.hpp:156-159) */
double or_matrix_norm(const double* K, int64_t nt, int64_t m, double budget, double tol, int32_t cap) {
  if (exact_allowed(nt, m, budget)) return or_spectral_norm_exact(K, nt, m);
  return or_power_iteration_norm(K, nt, m, tol, cap);
}

void or_residual_stats(const double* K, int64_t nt, int64_t m, const int64_t* skel, int64_t r,
                       const double* P, double* sumsq_D, double* sumsq_K, double* DtD, double* KtK) {
  double* D = (double*)malloc(sizeof(double) * (size_t)m);
  double* krow = (double*)malloc(sizeof(double) * (size_t)m);
  if (DtD) memset(DtD, 0, sizeof(double) * (size_t)(m * m));
  if (KtK) memset(KtK, 0, sizeof(double) * (size_t)(m * m));
  double sd = 0.0, sk = 0.0;
  for (int64_t i = 0; i < nt; ++i) {
    for (int64_t j = 0; j < m; ++j) krow[j] = K[i + j * nt];
    for (int64_t j = 0; j < m; ++j) {
      double acc = 0.0;
      for (int64_t l = 0; l < r; ++l) acc += krow[skel[l]] * P[l + j * r];
      D[j] = krow[j] - acc;
      sd += D[j] * D[j];
      sk += krow[j] * krow[j];
    }
    if (DtD)
      for (int64_t b = 0; b < m; ++b)
        for (int64_t a = 0; a < m; ++a) DtD[a + b * m] += D[a] * D[b];
    if (KtK)
      for (int64_t b = 0; b < m; ++b)
        for (int64_t a = 0; a < m; ++a) KtK[a + b * m] += krow[a] * krow[b];
  }
  *sumsq_D = sd;
  *sumsq_K = sk;
  free(D);
  free(krow);
}

/* compress.hpp:106-110 */
double or_bound_id_value(int64_t n, int64_t r, double sigma_r1) {
  const double nn = (double)n, rr = (double)r;
  return sqrt(1.0 + nn * rr * (nn - rr)) * sigma_r1;
}

/* sampling.hpp:247-266 */
double or_reconstruction_bound(int64_t m, int64_t s_count, double eps, double sigma_r1) {
  const double ratio = (double)m / (double)s_count;
  return sqrt(1.0 + ratio * (1.0 + eps) / ((1.0 - eps) * (1.0 - eps))) * sigma_r1;
}

/* compress_id (compress.hpp:168-215) */
int or_compress_id(const double* K, int64_t nt, int64_t m, const int64_t* rows, int64_t nrows,
                   double eps, int64_t fixed_r, double ref_sigma1, double k_norm, double budget,
                   double tol, int32_t cap, int64_t* rank, double* rel_error, int64_t* skel,
                   double* P, double* sigma1_sample, double* sigma_r1_sample, double* bound_id) {
  if (nrows < 1) return 1;
  double* sub = (double*)malloc(sizeof(double) * (size_t)(nrows * m)); /* gather_rows :130-137 */
  for (int64_t i = 0; i < nrows; ++i) {
    if (rows[i] < 0 || rows[i] >= nt) { free(sub); return 1; }
    for (int64_t j = 0; j < m; ++j) sub[i + j * nrows] = K[rows[i] + j * nt];
  }
  const int64_t k = nrows < m ? nrows : m;
  double* sv = (double*)malloc(sizeof(double) * (size_t)k);
  or_singular_values(sub, nrows, m, sv); /* :183 */
  int64_t r;
  if (eps > 0.0) r = or_epsilon_rank(sv, k, eps, ref_sigma1);
  else r = fixed_r < k ? fixed_r : k;
  *rank = r;
  *sigma1_sample = sv[0];
  *sigma_r1_sample = (r < k) ? sv[r] : 0.0;
  *bound_id = or_bound_id_value(m, r, *sigma_r1_sample);
  int rc = 0;
  if (r == 0) {
    *rel_error = 1.0;
  } else {
    rc = or_interpolative_decomposition(sub, nrows, m, r, skel, P);
    if (rc == 0) {
      const double num = or_reconstruction_error_norm(K, nt, m, skel, r, P, budget, tol, cap);
      const double den = k_norm > 0.0 ? k_norm : or_matrix_norm(K, nt, m, budget, tol, cap);
      *rel_error = den > 0.0 ? num / den : 0.0;
    }
  }
  free(sv);
  free(sub);
  return rc;
}

/* cyclic Jacobi eigen-solver for symmetric matrices (proj/tests/oracles.hpp:19-66 style) */
void or_jacobi_eigen(const double* A_in, int64_t n, double* evals, double* evecs) {
  double* A = (double*)malloc(sizeof(double) * (size_t)(n * n));
  double* V = (double*)calloc((size_t)(n * n), sizeof(double));
  memcpy(A, A_in, sizeof(double) * (size_t)(n * n));
  for (int64_t i = 0; i < n; ++i) V[i + i * n] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int64_t p = 0; p < n; ++p) {
      diag += A[p + p * n] * A[p + p * n];
      for (int64_t q = p + 1; q < n; ++q) off += A[p + q * n] * A[p + q * n];
    }
    if (off <= 1e-32 * diag || off == 0.0) break;
    for (int64_t p = 0; p < n; ++p)
      for (int64_t q = p + 1; q < n; ++q) {
        const double apq = A[p + q * n];
        if (apq == 0.0) continue;
        const double theta = (A[q + q * n] - A[p + p * n]) / (2.0 * apq);
        double t;
        if (fabs(theta) > 1e150) t = 0.5 / theta;
        else t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int64_t k = 0; k < n; ++k) {
          const double akp = A[k + p * n], akq = A[k + q * n];
          A[k + p * n] = c * akp - s * akq;
          A[k + q * n] = s * akp + c * akq;
        }
        for (int64_t k = 0; k < n; ++k) {
          const double apk = A[p + k * n], aqk = A[q + k * n];
          A[p + k * n] = c * apk - s * aqk;
          A[q + k * n] = s * apk + c * aqk;
        }
        for (int64_t k = 0; k < n; ++k) {
          const double vkp = V[k + p * n], vkq = V[k + q * n];
          V[k + p * n] = c * vkp - s * vkq;
          V[k + q * n] = s * vkp + c * vkq;
        }
      }
  }
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  for (int64_t i = 1; i < n; ++i) {
    int64_t o = order[i], k = i - 1;
    while (k >= 0 && A[order[k] + order[k] * n] < A[o + o * n]) { order[k + 1] = order[k]; --k; }
    order[k + 1] = o;
  }
  for (int64_t i = 0; i < n; ++i) {
    evals[i] = A[order[i] + order[i] * n];
    if (evecs) memcpy(evecs + i * n, V + order[i] * n, sizeof(double) * (size_t)n);
  }
  free(order); free(A); free(V);
}

/* -------------------------------------------------------------- compress.hpp: next rows */

/* apply_skeleton (compress.hpp:309-325): q_skel = P q (Eigen GEMV, accumulated over the m
 * columns of P in order), u_i = sum_j eval_kernel(y_i, xskel_j) q_skel_j sequentially over j
 * (mul then add: -ffp-contract=off). tgt nt x d, skel_pts r x d (col-major), P r x m col-major. */
void or_apply_skeleton(const double* tgt, int64_t nt, const double* skel_pts, int64_t r, int32_t d, double h,
                       const double* P, int64_t m, const double* q, double* u) {
  double* qs = (double*)calloc((size_t)(r > 0 ? r : 1), sizeof(double));
  for (int64_t k = 0; k < m; ++k)
    for (int64_t j = 0; j < r; ++j) qs[j] += P[j + k * r] * q[k];
  double* x = (double*)malloc(sizeof(double) * (size_t)d);
  double* y = (double*)malloc(sizeof(double) * (size_t)d);
  for (int64_t i = 0; i < nt; ++i) {
    for (int32_t k = 0; k < d; ++k) x[k] = tgt[i + k * nt];
    double acc = 0.0;
    for (int64_t j = 0; j < r; ++j) {
      for (int32_t k = 0; k < d; ++k) y[k] = skel_pts[j + k * r];
      acc += or_eval_gaussian(x, y, d, h) * qs[j];
    }
    u[i] = acc;
  }
  free(x); free(y); free(qs);
}

/* mc_error (compress.hpp:279-305) for the ID reconstruction khat_row(i) = K[i, skel] P:
 * per repetition a Bernoulli(s_mc) row draw with seed derive_seed(seed, rep) (retried once with
 * derive_seed(seed, rep, 1) when empty), num = matrix_norm(khat rows - K rows), den =
 * matrix_norm(K rows). est (n_mc). returns 0, 1 RangeError, 5 Error (empty twice). */
int or_mc_error(const double* K, int64_t nt, int64_t m, const int64_t* skel, int64_t r, const double* P,
                double s_mc, int32_t n_mc, uint64_t seed, double budget, double tol, int32_t cap, double* est) {
  if (!(s_mc > 0.0 && s_mc <= 1.0) || n_mc < 1) return 1;
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)nt);
  for (int32_t rep = 0; rep < n_mc; ++rep) {
    int64_t cnt = or_sample_rows(1, 0, nt, NULL, s_mc, or_derive_seed(seed, (uint64_t)rep, 0), rows);
    if (cnt == 0) cnt = or_sample_rows(1, 0, nt, NULL, s_mc, or_derive_seed(seed, (uint64_t)rep, 1), rows);
    if (cnt <= 0) { free(rows); return 5; }
    double* ks = (double*)malloc(sizeof(double) * (size_t)(cnt * m));
    double* diff = (double*)malloc(sizeof(double) * (size_t)(cnt * m));
    for (int64_t i = 0; i < cnt; ++i)
      for (int64_t j = 0; j < m; ++j) ks[i + j * cnt] = K[rows[i] + j * nt];
    for (int64_t i = 0; i < cnt; ++i)
      for (int64_t j = 0; j < m; ++j) {
        double acc = 0.0;  /* khat_row(i)_j = sum_l K[i, skel_l] P[l, j] */
        for (int64_t l = 0; l < r; ++l) acc += K[rows[i] + skel[l] * nt] * P[l + j * r];
        diff[i + j * cnt] = acc - ks[i + j * cnt];
      }
    const double den = or_matrix_norm(ks, cnt, m, budget, tol, cap);
    const double num = or_matrix_norm(diff, cnt, m, budget, tol, cap);
    est[rep] = den > 0.0 ? num / den : (num > 0.0 ? 1.0 / 0.0 : 0.0);
    free(ks); free(diff);
  }
  free(rows);
  return 0;
}

/* compress_svd error (compress.hpp:243-262): B = K V_r, diff = B V_r^T - K, num = spectral norm
 * (exact) of diff; returns num (the caller divides by its norm of K). Vr m x r col-major. */
double or_svd_error_norm(const double* K, int64_t nt, int64_t m, const double* Vr, int64_t r, double budget,
                         double tol, int32_t cap) {
  double* B = (double*)calloc((size_t)(nt * (r > 0 ? r : 1)), sizeof(double));
  for (int64_t k = 0; k < r; ++k)
    for (int64_t j = 0; j < m; ++j) {
      const double v = Vr[j + k * m];
      for (int64_t i = 0; i < nt; ++i) B[i + k * nt] += K[i + j * nt] * v;
    }
  double* diff = (double*)malloc(sizeof(double) * (size_t)(nt * m));
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = 0; i < nt; ++i) {
      double acc = 0.0;
      for (int64_t k = 0; k < r; ++k) acc += B[i + k * nt] * Vr[j + k * m];
      diff[i + j * nt] = acc - K[i + j * nt];
    }
  const double num = or_matrix_norm(diff, nt, m, budget, tol, cap);
  free(B); free(diff);
  return num;
}
