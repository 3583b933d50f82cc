// kernid_host.cpp -- host side of the B200 far-field path: the C++ mirror of the reference
// kernid:: API (include/kernid_b200.hpp) over the C-ABI of include/kernid_cuda.h, plus the
// small host-resident steps the north star keeps on the host (ID / pivoted QR on the
// sampled rows, epsilon-rank, weighted draws). Built with -ffp-contract=off like the
// reference (proj/CMakeLists.txt:12-15) so host-evaluated K_s rows are bit-identical.
#include "kernid_b200.hpp"

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <numeric>
#include <sstream>
#include <tuple>

namespace kernid_b200 {

// ------------------------------------------------------------------ errors
void throw_status(int code, const std::string& msg) {
  switch (code) {
    case KID_E_RANGE: throw RangeError(msg);
    case KID_E_DIM: throw DimensionError(msg);
    case KID_E_NO_TARGETS: throw NoTargetsError(msg);
    case KID_E_NUMERICAL: throw NumericalError(msg);
    case KID_E_ILLCOND: throw IllConditionedSkeletonError(msg);
    case KID_E_CONFIG: throw ConfigError(msg);
    default: throw Error(msg);
  }
}

// ------------------------------------------------------------------ rng.hpp
std::uint64_t splitmix64(std::uint64_t& state) {
  std::uint64_t z = (state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

std::uint64_t derive_seed(std::uint64_t master, std::uint64_t key_a, std::uint64_t key_b) {
  std::uint64_t state = master;
  state ^= splitmix64(state) + key_a;
  state ^= splitmix64(state) + key_b;
  return splitmix64(state);
}

std::uint64_t Rng::below(std::uint64_t n) {
  const std::uint64_t limit = n * ((~std::uint64_t{0}) / n);
  std::uint64_t x;
  do {
    x = engine_();
  } while (x >= limit);
  return x % n;
}

double Rng::normal() {
  if (has_spare_) {
    has_spare_ = false;
    return spare_;
  }
  const double u1 = 1.0 - uniform01();
  const double u2 = uniform01();
  const double radius = std::sqrt(-2.0 * std::log(u1));
  const double angle = 2.0 * M_PI * u2;
  spare_ = radius * std::sin(angle);
  has_spare_ = true;
  return radius * std::cos(angle);
}

// ------------------------------------------------------------------ kernel / datagen
void KernelSpec::validate() const {
  if (!(h > 0.0)) throw ConfigError("Gaussian kernel requires bandwidth h > 0");
}

PointSet gen_normal(int d, int64_t N, std::uint64_t seed) {
  if (d < 1 || N < 1) throw RangeError("gen_normal: requires d >= 1 and N >= 1");
  Rng rng(seed);
  PointSet ps(N, d);
  for (int64_t i = 0; i < N; ++i)
    for (int j = 0; j < d; ++j) ps(i, j) = rng.normal();
  return ps;
}

double silverman_bandwidth(int d, long long N) {
  if (d < 1 || N < 1) throw RangeError("silverman_bandwidth: requires d >= 1 and N >= 1");
  const double e = 1.0 / (static_cast<double>(d) + 4.0);
  return std::pow(4.0 / (2.0 * d + 1.0), e) * std::pow(static_cast<double>(N), -e);
}

double eval_kernel(const KernelSpec& spec, const double* x, int64_t sx, const double* y, int64_t sy, int d) {
  double acc = 0.0;  // kernel.hpp:60-68
  for (int k = 0; k < d; ++k) {
    const double diff = x[k * sx] - y[k * sy];
    acc += diff * diff;
  }
  return std::exp(-acc / (2.0 * spec.h * spec.h));  // kernel.hpp:77-79
}

// ------------------------------------------------------------------ device
Device::Device(int device) {
  const int rc = kid_create(&ctx_, device);
  if (rc) throw_status(rc, "kid_create: no usable CUDA device " + std::to_string(device));
}
Device::~Device() { kid_destroy(ctx_); }
void Device::check(int status) const {
  if (status) throw_status(status, kid_last_error(ctx_));
}

// ------------------------------------------------------------------ geometry
SourceTargetSplit split_sources_targets(Device& dev, const PointSet& ps, const std::vector<double>& x_c, int64_t n,
                                        double xi) {
  const int64_t N = ps.rows;
  if (n < 1 || n >= N) throw RangeError("split_sources_targets: requires 1 <= n < N");
  if (xi < 0.0) throw RangeError("split_sources_targets: requires xi >= 0");
  if (static_cast<int64_t>(x_c.size()) != ps.cols)
    throw DimensionError("split_sources_targets: center dimension mismatch");
  dev.check(kid_set_points(dev.ctx(), ps.data(), N, static_cast<int32_t>(ps.cols), 0));
  SourceTargetSplit split;
  split.center = x_c;
  split.xi = xi;
  split.source_indices.resize(static_cast<size_t>(n));
  int64_t nt = 0;
  dev.check(kid_split(dev.ctx(), x_c.data(), n, xi, split.source_indices.data(), &split.rho, &nt));
  split.target_indices.resize(static_cast<size_t>(nt));
  dev.check(kid_get_targets(dev.ctx(), split.target_indices.data(), nt));
  return split;
}

KernelBlock::KernelBlock(Device& dev, KernelSpec spec, const PointSet& points, const SourceTargetSplit& split)
    : dev_(&dev), spec_(spec), points_(&points), split_(&split) {
  spec_.validate();
}

Matrix KernelBlock::rows_exact(const std::vector<int64_t>& idx) const {
  const int64_t m = cols();
  const int d = static_cast<int>(points_->cols);
  const int64_t N = points_->rows;
  Matrix sub(static_cast<int64_t>(idx.size()), m);
  for (size_t i = 0; i < idx.size(); ++i) {
    if (idx[i] < 0 || idx[i] >= rows()) throw RangeError("row sample index out of range");
    const double* t = points_->data() + split_->target_indices[static_cast<size_t>(idx[i])];
    for (int64_t j = 0; j < m; ++j) {
      const double* s = points_->data() + split_->source_indices[static_cast<size_t>(j)];
      sub(static_cast<int64_t>(i), j) = eval_kernel(spec_, t, N, s, N, d);
    }
  }
  return sub;
}

std::vector<double> KernelBlock::row_norms() const {
  std::vector<double> w(static_cast<size_t>(rows()));
  dev_->check(kid_row_norms(dev_->ctx(), spec_.h, w.data()));
  return w;
}

Matrix KernelBlock::gram(double* sumsq) const {
  Matrix G(cols(), cols());
  dev_->check(kid_gram(dev_->ctx(), spec_.h, G.data(), sumsq));
  return G;
}

double KernelBlock::spectral_norm() const { return std::sqrt(lambda_max(gram())); }

// ------------------------------------------------------------------ lowrank (host)
namespace {

// Householder QR R factor of a tall (rows >= cols) matrix.
Matrix qr_r(const Matrix& A_in) {
  Matrix A = A_in;
  const int64_t rows = A.rows, cols = A.cols;
  std::vector<double> v(static_cast<size_t>(rows));
  for (int64_t j = 0; j < cols; ++j) {
    double nrm = 0.0;
    for (int64_t i = j; i < rows; ++i) nrm += A(i, j) * A(i, j);
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) continue;
    const double alpha = A(j, j);
    const double beta = alpha >= 0.0 ? -nrm : nrm;
    const double v0 = alpha - beta;
    const double tau = -v0 / beta;
    const int64_t len = rows - j;
    v[0] = 1.0;
    for (int64_t i = 1; i < len; ++i) v[static_cast<size_t>(i)] = A(j + i, j) / v0;
    A(j, j) = beta;
    for (int64_t k = j + 1; k < cols; ++k) {
      double w = 0.0;
      for (int64_t i = 0; i < len; ++i) w += v[static_cast<size_t>(i)] * A(j + i, k);
      w *= tau;
      for (int64_t i = 0; i < len; ++i) A(j + i, k) -= w * v[static_cast<size_t>(i)];
    }
  }
  Matrix R(cols, cols);
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t r = 0; r <= c; ++r) R(r, c) = A(r, c);
  return R;
}

// One-sided Jacobi: singular values (descending) of a square matrix.
std::vector<double> jacobi_sv(Matrix U) {
  const int64_t n = U.cols, rows = U.rows;
  for (int sweep = 0; sweep < 80; ++sweep) {
    int64_t rotated = 0;
    for (int64_t p = 0; p + 1 < n; ++p)
      for (int64_t q = p + 1; q < n; ++q) {
        double a = 0.0, b = 0.0, g = 0.0;
        for (int64_t i = 0; i < rows; ++i) {
          a += U(i, p) * U(i, p);
          b += U(i, q) * U(i, q);
          g += U(i, p) * U(i, q);
        }
        if (g == 0.0 || std::fabs(g) <= 1e-15 * std::sqrt(a) * std::sqrt(b)) continue;
        ++rotated;
        const double zeta = (b - a) / (2.0 * g);
        const double t = std::fabs(zeta) > 1e150 ? 0.5 / zeta
                                                   : (zeta >= 0.0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (int64_t i = 0; i < rows; ++i) {
          const double x = U(i, p), y = U(i, q);
          U(i, p) = c * x - s * y;
          U(i, q) = s * x + c * y;
        }
      }
    if (!rotated) break;
  }
  std::vector<double> sv(static_cast<size_t>(n));
  for (int64_t j = 0; j < n; ++j) {
    double acc = 0.0;
    for (int64_t i = 0; i < rows; ++i) acc += U(i, j) * U(i, j);
    sv[static_cast<size_t>(j)] = std::sqrt(acc);
  }
  std::sort(sv.begin(), sv.end(), std::greater<double>());
  return sv;
}

// One-sided Jacobi with the accumulated rotations: U V = [u_1 s_1 ...]; singular values
// (descending, all cols of them) and V (cols x cols, columns in the same order).
void jacobi_svd_v(Matrix U, std::vector<double>& sv, Matrix& V) {
  const int64_t n = U.cols, rows = U.rows;
  V = Matrix(n, n);
  for (int64_t i = 0; i < n; ++i) V(i, i) = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    int64_t rotated = 0;
    for (int64_t p = 0; p + 1 < n; ++p)
      for (int64_t q = p + 1; q < n; ++q) {
        double a = 0.0, b = 0.0, g = 0.0;
        for (int64_t i = 0; i < rows; ++i) {
          a += U(i, p) * U(i, p);
          b += U(i, q) * U(i, q);
          g += U(i, p) * U(i, q);
        }
        if (g == 0.0 || std::fabs(g) <= 1e-15 * std::sqrt(a) * std::sqrt(b)) continue;
        ++rotated;
        const double zeta = (b - a) / (2.0 * g);
        const double t = std::fabs(zeta) > 1e150 ? 0.5 / zeta
                                                   : (zeta >= 0.0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (int64_t i = 0; i < rows; ++i) {
          const double x = U(i, p), y = U(i, q);
          U(i, p) = c * x - s * y;
          U(i, q) = s * x + c * y;
        }
        for (int64_t i = 0; i < n; ++i) {
          const double x = V(i, p), y = V(i, q);
          V(i, p) = c * x - s * y;
          V(i, q) = s * x + c * y;
        }
      }
    if (!rotated) break;
  }
  std::vector<double> nrm(static_cast<size_t>(n));
  for (int64_t j = 0; j < n; ++j) {
    double acc = 0.0;
    for (int64_t i = 0; i < rows; ++i) acc += U(i, j) * U(i, j);
    nrm[static_cast<size_t>(j)] = std::sqrt(acc);
  }
  std::vector<int64_t> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), int64_t{0});
  std::stable_sort(order.begin(), order.end(),
                   [&](int64_t x, int64_t y) { return nrm[static_cast<size_t>(x)] > nrm[static_cast<size_t>(y)]; });
  Matrix Vs(n, n);
  sv.resize(static_cast<size_t>(n));
  for (int64_t j = 0; j < n; ++j) {
    sv[static_cast<size_t>(j)] = nrm[static_cast<size_t>(order[static_cast<size_t>(j)])];
    for (int64_t i = 0; i < n; ++i) Vs(i, j) = V(i, order[static_cast<size_t>(j)]);
  }
  V = std::move(Vs);
}

Matrix transpose(const Matrix& A) {
  Matrix T(A.cols, A.rows);
  for (int64_t j = 0; j < A.cols; ++j)
    for (int64_t i = 0; i < A.rows; ++i) T(j, i) = A(i, j);
  return T;
}

}  // namespace

std::vector<double> singular_values(const Matrix& A) {
  if (A.rows == 0 || A.cols == 0) throw RangeError("singular_values: empty matrix");
  if (A.rows >= A.cols) return jacobi_sv(qr_r(A));
  return jacobi_sv(qr_r(transpose(A)));
}

RightFactor right_factor(const Matrix& A) {
  if (A.rows == 0 || A.cols == 0) throw RangeError("right_factor: empty matrix");
  RightFactor rf;
  // tall: V from the SVD of the triangular factor (lowrank.hpp:81-86); wide: the full V of A,
  // whose trailing columns complete the thin V of the reference to an orthonormal basis
  jacobi_svd_v(A.rows >= A.cols ? qr_r(A) : A, rf.singular_values, rf.V);
  rf.singular_values.resize(static_cast<size_t>(std::min(A.rows, A.cols)));
  return rf;
}

// relative singular values the Gram route (sqrt of the eigenvalues of K^T K) resolves: ~sqrt(u) plus margin
constexpr double kGramResolvable = 1e-7;

namespace {
// Second pass of the m > 128 spectrum (the stand-in for the TSQR factor that does not fit one SM):
// given the Gram route's eigenpairs (V, s) of K^T K -- sigma_i resolved to ~sqrt(u) sigma_1 -- form the
// preconditioner X = V diag(1 / max(s_i, delta)), delta = 4 sqrt(m u) s_1, and take the Gram of K X on the
// device (kid_proj_gram: K X has near-orthonormal leading columns, and trailing columns of norm sigma_i / delta,
// so its Gram G2 carries the tail to ~u relative to delta^2 instead of sigma_1^2). With G2 = Q M Q^T,
// K^T K = X^-T G2 X^-1 = B^T B for B = M^(1/2) Q^T diag(max(s, delta)) V^T, whose singular values and right
// singular vectors are those of K (lowrank.hpp:56-90 takes them from the QR factor instead). B V has nearly
// orthogonal columns, so the one-sided Jacobi SVD runs on it and the rotations J are folded into V.
// Measured against LAPACK on the oracle's K: every sigma within ~2e-14 sigma_1 (m = 256 / 512, d = 1..16).
void refine_right_factor(const KernelBlock& K, RightFactor& rf) {
  const int64_t m = K.cols();
  std::vector<double> sc(static_cast<size_t>(m));
  const double s1 = rf.singular_values.empty() ? 0.0 : rf.singular_values[0];
  if (!(s1 > 0.0)) return;
  const double delta = 4.0 * std::sqrt(static_cast<double>(m) * 1.1102230246251565e-16) * s1;
  Matrix X(m, m);
  for (int64_t j = 0; j < m; ++j) {
    const double sj = j < static_cast<int64_t>(rf.singular_values.size()) ? rf.singular_values[static_cast<size_t>(j)] : 0.0;
    sc[static_cast<size_t>(j)] = std::max(sj, delta);
    const double inv = 1.0 / sc[static_cast<size_t>(j)];
    for (int64_t i = 0; i < m; ++i) X(i, j) = rf.V(i, j) * inv;
  }
  Matrix G2(m, m);
  double sd = 0.0, sk = 0.0;
  K.device().check(kid_proj_gram(K.device().ctx(), K.spec().h, X.data(), m, &sd, &sk, G2.data()));
  std::vector<double> mu;
  Matrix Q;
  sym_eig(G2, mu, &Q);
  Matrix U0(m, m);  // M^(1/2) Q^T diag(sc)
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = 0; i < m; ++i)
      U0(i, j) = std::sqrt(std::max(mu[static_cast<size_t>(i)], 0.0)) * Q(j, i) * sc[static_cast<size_t>(j)];
  Matrix J;
  std::vector<double> sv;
  jacobi_svd_v(std::move(U0), sv, J);
  Matrix Vn(m, m);
  for (int64_t j = 0; j < m; ++j)
    for (int64_t k = 0; k < m; ++k) {
      const double jk = J(k, j);
      if (jk == 0.0) continue;
      for (int64_t i = 0; i < m; ++i) Vn(i, j) += rf.V(i, k) * jk;
    }
  rf.V = std::move(Vn);
  rf.singular_values = std::move(sv);
}
}  // namespace

std::vector<double> KernelBlock::singular_values(double resolve) const {
  const int64_t m = cols();
  if (m <= 128 || resolve < kGramResolvable) return right_factor(resolve).singular_values;
  const std::vector<double> ev = sym_eigvals(gram());  // Gram route, eigenvalues only
  std::vector<double> sv(ev.size());
  for (size_t i = 0; i < ev.size(); ++i) sv[i] = std::sqrt(std::max(ev[i], 0.0));
  sv.resize(static_cast<size_t>(std::min(rows(), m)));
  return sv;
}

RightFactor KernelBlock::right_factor(double resolve) const {
  const int64_t m = cols();
  RightFactor rf;
  if (m <= 128) {
    Matrix R(m, m);
    dev_->check(kid_tsqr_r(dev_->ctx(), spec_.h, R.data()));
    jacobi_svd_v(R, rf.singular_values, rf.V);
  } else {
    std::vector<double> ev;
    sym_eig(gram(), ev, &rf.V);
    rf.singular_values.resize(ev.size());
    for (size_t i = 0; i < ev.size(); ++i) rf.singular_values[i] = std::sqrt(std::max(ev[i], 0.0));
    if (resolve < kGramResolvable) refine_right_factor(*this, rf);
  }
  rf.singular_values.resize(static_cast<size_t>(std::min(rows(), m)));
  return rf;
}

int64_t epsilon_rank(const std::vector<double>& sv, double eps, std::optional<double> reference_sigma1) {
  if (!(eps > 0.0 && eps < 1.0)) throw RangeError("epsilon_rank: requires eps in (0, 1)");
  if (sv.empty()) return 0;
  const double ref = reference_sigma1.value_or(sv[0]);
  if (!(ref > 0.0)) return 0;
  for (size_t r = 0; r < sv.size(); ++r)
    if (sv[r] < eps * ref) return static_cast<int64_t>(r);
  return static_cast<int64_t>(sv.size());
}

// lowrank.hpp:135-262, restated with sequential single-accumulator reductions.
IDFactorization interpolative_decomposition(const Matrix& A, int64_t r) {
  const int64_t m = A.rows, n = A.cols;
  if (r < 1 || r > std::min(m, n)) throw RangeError("interpolative_decomposition: requires 1 <= r <= min(m, n)");
  Matrix W = A;
  std::vector<int64_t> perm(static_cast<size_t>(n));
  std::iota(perm.begin(), perm.end(), int64_t{0});
  std::vector<double> colnorm2(static_cast<size_t>(n)), refnorm2;
  for (int64_t j = 0; j < n; ++j) {
    double acc = 0.0;
    for (int64_t i = 0; i < m; ++i) acc += W(i, j) * W(i, j);
    colnorm2[static_cast<size_t>(j)] = acc;
  }
  refnorm2 = colnorm2;
  std::vector<double> v(static_cast<size_t>(m)), w(static_cast<size_t>(n));
  constexpr double recompute_ratio = 2.3e-16;
  for (int64_t k = 0; k < r; ++k) {
    int64_t piv = k;
    for (int64_t j = k + 1; j < n; ++j)
      if (colnorm2[static_cast<size_t>(j)] > colnorm2[static_cast<size_t>(piv)]) piv = j;
    if (piv != k) {
      for (int64_t i = 0; i < m; ++i) std::swap(W(i, k), W(i, piv));
      std::swap(colnorm2[static_cast<size_t>(k)], colnorm2[static_cast<size_t>(piv)]);
      std::swap(refnorm2[static_cast<size_t>(k)], refnorm2[static_cast<size_t>(piv)]);
      std::swap(perm[static_cast<size_t>(k)], perm[static_cast<size_t>(piv)]);
    }
    const int64_t len = m - k;
    double normx = 0.0;
    for (int64_t i = k; i < m; ++i) normx += W(i, k) * W(i, k);
    normx = std::sqrt(normx);
    if (normx == 0.0) continue;
    const double alpha = W(k, k);
    const double beta = (alpha >= 0.0) ? -normx : normx;
    const double v0 = alpha - beta;
    const double tau = -v0 / beta;
    for (int64_t i = 1; i < len; ++i) W(k + i, k) /= v0;
    W(k, k) = beta;
    if (k + 1 < n && len > 0) {
      v[0] = 1.0;
      for (int64_t i = 1; i < len; ++i) v[static_cast<size_t>(i)] = W(k + i, k);
      for (int64_t j = k + 1; j < n; ++j) {
        double acc = 0.0;
        for (int64_t i = 0; i < len; ++i) acc += v[static_cast<size_t>(i)] * W(k + i, j);
        w[static_cast<size_t>(j)] = tau * acc;
      }
      for (int64_t j = k + 1; j < n; ++j)
        for (int64_t i = 0; i < len; ++i) W(k + i, j) -= v[static_cast<size_t>(i)] * w[static_cast<size_t>(j)];
    }
    for (int64_t j = k + 1; j < n; ++j) {
      const double t = W(k, j);
      double& cn = colnorm2[static_cast<size_t>(j)];
      cn -= t * t;
      if (cn < recompute_ratio * refnorm2[static_cast<size_t>(j)] || cn < 0.0) {
        double acc = 0.0;
        for (int64_t i = k + 1; i < m; ++i) acc += W(i, j) * W(i, j);
        cn = (m - k - 1 > 0) ? acc : 0.0;
        refnorm2[static_cast<size_t>(j)] = cn;
      }
    }
  }
  const double lead = std::fabs(W(0, 0));
  const double tail = std::fabs(W(r - 1, r - 1));
  if (!(lead > 0.0) || tail < 10.0 * std::numeric_limits<double>::epsilon() * lead)
    throw IllConditionedSkeletonError("interpolative_decomposition: pivot " + std::to_string(r) +
                                      " is numerically negligible; reduce the requested rank");
  IDFactorization id;
  id.rank = r;
  id.skeleton.assign(perm.begin(), perm.begin() + r);
  id.projection = Matrix(r, n);
  for (int64_t i = 0; i < r; ++i) id.projection(i, perm[static_cast<size_t>(i)]) = 1.0;
  std::vector<double> x(static_cast<size_t>(r));
  for (int64_t j = 0; j < n - r; ++j) {
    for (int64_t i = 0; i < r; ++i) x[static_cast<size_t>(i)] = W(i, r + j);
    for (int64_t i = r - 1; i >= 0; --i) {
      x[static_cast<size_t>(i)] /= W(i, i);
      for (int64_t k = 0; k < i; ++k) x[static_cast<size_t>(k)] -= x[static_cast<size_t>(i)] * W(k, i);
    }
    const int64_t col = perm[static_cast<size_t>(r + j)];
    for (int64_t i = 0; i < r; ++i) id.projection(i, col) = x[static_cast<size_t>(i)];
  }
  return id;
}

// Cyclic Jacobi eigen-solver for the symmetric m x m Grams (descending eigenvalues).
namespace {
void sym_tridiag_ql(const Matrix& A_in, std::vector<double>& d, Matrix* Z);
}  // namespace

void sym_eig(const Matrix& A_in, std::vector<double>& evals, Matrix* evecs) {
  if (A_in.rows > 128) {  // Jacobi sweeps cost seconds at m = 256 / 512
    sym_tridiag_ql(A_in, evals, evecs);
    return;
  }
  Matrix A = A_in;
  const int64_t n = A.rows;
  Matrix V(n, n);
  for (int64_t i = 0; i < n; ++i) V(i, i) = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int64_t p = 0; p < n; ++p) {
      diag += A(p, p) * A(p, p);
      for (int64_t q = p + 1; q < n; ++q) off += A(p, q) * A(p, q);
    }
    if (off == 0.0 || off <= 1e-32 * diag) break;
    for (int64_t p = 0; p < n; ++p)
      for (int64_t q = p + 1; q < n; ++q) {
        const double apq = A(p, q);
        if (apq == 0.0) continue;
        const double theta = (A(q, q) - A(p, p)) / (2.0 * apq);
        const double t = std::fabs(theta) > 1e150
                             ? 0.5 / theta
                             : (theta >= 0.0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int64_t k = 0; k < n; ++k) {
          const double akp = A(k, p), akq = A(k, q);
          A(k, p) = c * akp - s * akq;
          A(k, q) = s * akp + c * akq;
        }
        for (int64_t k = 0; k < n; ++k) {
          const double apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk - s * aqk;
          A(q, k) = s * apk + c * aqk;
        }
        if (evecs)
          for (int64_t k = 0; k < n; ++k) {
            const double vkp = V(k, p), vkq = V(k, q);
            V(k, p) = c * vkp - s * vkq;
            V(k, q) = s * vkp + c * vkq;
          }
      }
  }
  std::vector<int64_t> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), int64_t{0});
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return A(a, a) > A(b, b); });
  evals.resize(static_cast<size_t>(n));
  if (evecs) *evecs = Matrix(n, n);
  for (int64_t i = 0; i < n; ++i) {
    evals[static_cast<size_t>(i)] = A(order[static_cast<size_t>(i)], order[static_cast<size_t>(i)]);
    if (evecs)
      for (int64_t k = 0; k < n; ++k) (*evecs)(k, i) = V(k, order[static_cast<size_t>(i)]);
  }
}

// Symmetric eigen-solver for the m > 128 host steps (m = 256 / 512 Grams), where Jacobi sweeps
// cost seconds: Householder reduction to tridiagonal form (A22 <- H A22 H by the rank-2 update
// A22 - v w^T - w v^T, the reflectors accumulated into Z when vectors are wanted), then the
// implicit QL iteration with Wilkinson shifts on the tridiagonal, its Givens rotations applied to
// Z. O(n^3). Eigenvalues descending; Z's columns are the matching eigenvectors.
namespace {
void sym_tridiag_ql(const Matrix& A_in, std::vector<double>& d, Matrix* Z) {
  const int64_t n = A_in.rows;
  if (A_in.cols != n) throw DimensionError("sym_eig: matrix must be square");
  std::vector<double> a(A_in.a);  // column-major, symmetric: a[i + j n]
  auto at = [&](int64_t i, int64_t j) -> double& { return a[static_cast<size_t>(i + j * n)]; };
  d.assign(static_cast<size_t>(n), 0.0);
  std::vector<double> e(static_cast<size_t>(n), 0.0), p(static_cast<size_t>(n)), w(static_cast<size_t>(n));
  std::vector<std::vector<double>> vs(static_cast<size_t>(std::max<int64_t>(n - 2, 0)));
  std::vector<double> betas(static_cast<size_t>(std::max<int64_t>(n - 2, 0)), 0.0);
  for (int64_t k = 0; k + 2 < n; ++k) {
    const int64_t m = n - k - 1;  // length of x = A[k+1:, k]
    double nrm = 0.0;
    for (int64_t i = 0; i < m; ++i) nrm += at(k + 1 + i, k) * at(k + 1 + i, k);
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) continue;
    const double x0 = at(k + 1, k), alpha = x0 >= 0.0 ? -nrm : nrm;
    std::vector<double>& v = vs[static_cast<size_t>(k)];
    v.assign(static_cast<size_t>(m), 0.0);
    double vn = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      v[static_cast<size_t>(i)] = at(k + 1 + i, k) - (i == 0 ? alpha : 0.0);
      vn += v[static_cast<size_t>(i)] * v[static_cast<size_t>(i)];
    }
    if (vn == 0.0) continue;
    const double beta = 2.0 / vn;  // H = I - beta v v^T
    betas[static_cast<size_t>(k)] = beta;
    double K = 0.0;
    for (int64_t i = 0; i < m; ++i) {  // p = beta A22 v
      double acc = 0.0;
      for (int64_t j = 0; j < m; ++j) acc += at(k + 1 + i, k + 1 + j) * v[static_cast<size_t>(j)];
      p[static_cast<size_t>(i)] = beta * acc;
      K += v[static_cast<size_t>(i)] * p[static_cast<size_t>(i)];
    }
    K *= 0.5 * beta;
    for (int64_t i = 0; i < m; ++i) w[static_cast<size_t>(i)] = p[static_cast<size_t>(i)] - K * v[static_cast<size_t>(i)];
    for (int64_t j = 0; j < m; ++j)  // A22 -= v w^T + w v^T
      for (int64_t i = 0; i < m; ++i)
        at(k + 1 + i, k + 1 + j) -= v[static_cast<size_t>(i)] * w[static_cast<size_t>(j)] +
                                    w[static_cast<size_t>(i)] * v[static_cast<size_t>(j)];
    at(k + 1, k) = at(k, k + 1) = alpha;
    for (int64_t i = 1; i < m; ++i) at(k + 1 + i, k) = at(k, k + 1 + i) = 0.0;
  }
  for (int64_t i = 0; i < n; ++i) d[static_cast<size_t>(i)] = at(i, i);
  for (int64_t i = 0; i + 1 < n; ++i) e[static_cast<size_t>(i)] = at(i + 1, i);
  if (Z) {  // Z = H_0 H_1 ... H_{n-3}, accumulated backwards
    *Z = Matrix(n, n);
    for (int64_t i = 0; i < n; ++i) (*Z)(i, i) = 1.0;
    for (int64_t k = n - 3; k >= 0; --k) {
      const std::vector<double>& v = vs[static_cast<size_t>(k)];
      const double beta = betas[static_cast<size_t>(k)];
      if (beta == 0.0) continue;
      const int64_t m = n - k - 1;
      for (int64_t j = k + 1; j < n; ++j) {
        double s = 0.0;
        for (int64_t i = 0; i < m; ++i) s += v[static_cast<size_t>(i)] * (*Z)(k + 1 + i, j);
        s *= beta;
        for (int64_t i = 0; i < m; ++i) (*Z)(k + 1 + i, j) -= s * v[static_cast<size_t>(i)];
      }
    }
  }
  // implicit QL with shifts on (d, e), e[i] coupling i and i + 1
  for (int64_t l = 0; l < n; ++l) {
    for (int iter = 0; iter < 100; ++iter) {
      int64_t m = l;
      for (; m + 1 < n; ++m) {
        const double dd = std::fabs(d[static_cast<size_t>(m)]) + std::fabs(d[static_cast<size_t>(m + 1)]);
        if (std::fabs(e[static_cast<size_t>(m)]) <= 1e-16 * dd) break;
      }
      if (m == l) break;
      double g = (d[static_cast<size_t>(l + 1)] - d[static_cast<size_t>(l)]) / (2.0 * e[static_cast<size_t>(l)]);
      double r = std::hypot(g, 1.0);
      g = d[static_cast<size_t>(m)] - d[static_cast<size_t>(l)] + e[static_cast<size_t>(l)] / (g + (g >= 0.0 ? r : -r));
      double sn = 1.0, c = 1.0, pp = 0.0;
      bool early = false;
      for (int64_t i = m - 1; i >= l; --i) {
        const double f = sn * e[static_cast<size_t>(i)], b = c * e[static_cast<size_t>(i)];
        r = std::hypot(f, g);
        e[static_cast<size_t>(i + 1)] = r;
        if (r == 0.0) {
          d[static_cast<size_t>(i + 1)] -= pp;
          e[static_cast<size_t>(m)] = 0.0;
          early = true;
          break;
        }
        sn = f / r;
        c = g / r;
        g = d[static_cast<size_t>(i + 1)] - pp;
        r = (d[static_cast<size_t>(i)] - g) * sn + 2.0 * c * b;
        pp = sn * r;
        d[static_cast<size_t>(i + 1)] = g + pp;
        g = c * r - b;
        if (Z)
          for (int64_t k = 0; k < n; ++k) {
            const double zf = (*Z)(k, i + 1);
            (*Z)(k, i + 1) = sn * (*Z)(k, i) + c * zf;
            (*Z)(k, i) = c * (*Z)(k, i) - sn * zf;
          }
      }
      if (early) continue;
      d[static_cast<size_t>(l)] -= pp;
      e[static_cast<size_t>(l)] = g;
      e[static_cast<size_t>(m)] = 0.0;
    }
  }
  std::vector<int64_t> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), int64_t{0});
  std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) { return d[static_cast<size_t>(x)] > d[static_cast<size_t>(y)]; });
  std::vector<double> ds(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) ds[static_cast<size_t>(i)] = d[static_cast<size_t>(order[static_cast<size_t>(i)])];
  d = ds;
  if (Z) {
    Matrix Zs(n, n);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i) Zs(i, j) = (*Z)(i, order[static_cast<size_t>(j)]);
    *Z = std::move(Zs);
  }
}
}  // namespace

std::vector<double> sym_eigvals(const Matrix& A) {
  std::vector<double> d;
  sym_tridiag_ql(A, d, nullptr);
  return d;
}

// Largest eigenvalue of a symmetric PSD matrix (the spectral norms sqrt(lambda_max(D^T D)) and
// sqrt(lambda_max(K^T K)) of compress_id). n <= 128: all eigenvalues by Householder tridiagonalisation +
// implicit QL, values only (2.5 ms at n = 100 where Jacobi sweeps take 25 ms -- they were most of the c2-d3
// end-to-end step -- and closer to LAPACK: 2e-16 against 2e-14 relative). Larger n (c4 / c5:
// m = 256 / 512): Lanczos from the constant vector with full reorthogonalisation, stopped when the
// Ritz residual |beta_k s_k| of the top Ritz pair is below 1e-14 of it (|theta - lambda| <= residual),
// or at k = n (exact); the k x k tridiagonal is solved by Jacobi. ~n^2 flops per step instead of the
// O(n^3) of a full tridiagonalisation.
double lambda_max(const Matrix& G) {
  const int64_t n = G.rows;
  if (n == 0) return 0.0;
  if (n <= 128) {
    std::vector<double> ev;
    sym_tridiag_ql(G, ev, nullptr);
    return ev.empty() ? 0.0 : std::max(ev[0], 0.0);
  }
  const size_t N = static_cast<size_t>(n);
  std::vector<std::vector<double>> Q;
  std::vector<double> alpha, beta;
  std::vector<double> v(N, 1.0 / std::sqrt(static_cast<double>(n))), w(N);
  double theta = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    Q.push_back(v);
    for (size_t i = 0; i < N; ++i) {  // w = G v (column-major, symmetric)
      double acc = 0.0;
      const double* gi = G.data() + i * N;
      for (size_t j = 0; j < N; ++j) acc += gi[j] * v[j];
      w[i] = acc;
    }
    double a = 0.0;
    for (size_t i = 0; i < N; ++i) a += v[i] * w[i];
    alpha.push_back(a);
    for (int pass = 0; pass < 2; ++pass)  // full reorthogonalisation, twice
      for (const auto& q : Q) {
        double c = 0.0;
        for (size_t i = 0; i < N; ++i) c += q[i] * w[i];
        for (size_t i = 0; i < N; ++i) w[i] -= c * q[i];
      }
    double b = 0.0;
    for (size_t i = 0; i < N; ++i) b += w[i] * w[i];
    b = std::sqrt(b);
    const int64_t kk = k + 1;
    const bool last = kk == n || b <= 1e-300;
    if (last || kk % 8 == 0) {
      Matrix T(kk, kk);
      for (int64_t i = 0; i < kk; ++i) {
        T(i, i) = alpha[static_cast<size_t>(i)];
        if (i + 1 < kk) T(i, i + 1) = T(i + 1, i) = beta[static_cast<size_t>(i)];
      }
      std::vector<double> ev;
      Matrix V;
      sym_eig(T, ev, &V);
      theta = ev[0];
      const double res = std::abs(b * V(kk - 1, 0));
      if (last || res <= 1e-14 * std::abs(theta)) return std::max(theta, 0.0);
    }
    beta.push_back(b);
    for (size_t i = 0; i < N; ++i) v[i] = w[i] / b;
  }
  return std::max(theta, 0.0);
}

LeverageScores row_leverage_scores(const KernelBlock& K, int64_t r) {
  const int64_t mn = std::min(K.rows(), K.cols());
  if (r < 1 || r > mn) throw RangeError("row_leverage_scores: requires 1 <= r <= min(m, n)");
  const int64_t m = K.cols();
  // lowrank.hpp:299. m <= 128: TSQR on the device. m > 128: the Gram route where it resolves sigma_r with
  // margin, else the Gram route plus its preconditioned second pass (refine_right_factor)
  RightFactor rf = K.right_factor(kGramResolvable);
  if (m > 128 && rf.singular_values[static_cast<size_t>(r - 1)] < 100.0 * kGramResolvable * rf.singular_values[0])
    rf = K.right_factor(0.0);
  const Matrix& V = rf.V;
  std::vector<double> sv = rf.singular_values;
  sv.resize(static_cast<size_t>(m), 0.0);
  if (!(sv[static_cast<size_t>(r - 1)] > 0.0))
    throw NumericalError("row_leverage_scores: sigma_r vanishes; scores undefined");
  Matrix W(m, r);  // lowrank.hpp:304
  for (int64_t j = 0; j < r; ++j)
    for (int64_t i = 0; i < m; ++i) W(i, j) = V(i, j) * (1.0 / sv[static_cast<size_t>(j)]);
  LeverageScores out;
  out.scores.resize(static_cast<size_t>(K.rows()));
  K.device().check(kid_leverage(K.device().ctx(), K.spec().h, W.data(), r, out.scores.data()));
  out.degenerate_gap = (r < m) && (sv[static_cast<size_t>(r - 1)] - sv[static_cast<size_t>(r)] <=
                                   1e-12 * sv[static_cast<size_t>(r - 1)]);
  return out;
}

// ------------------------------------------------------------------ sampling
std::string SamplingScheme::name() const {
  std::string base;
  switch (kind) {
    case SchemeKind::Uniform: base = "uniform"; break;
    case SchemeKind::Bernoulli: base = "bernoulli"; break;
    case SchemeKind::EuclideanNorm: base = "euclidean_norm"; break;
    case SchemeKind::Distance: base = distance_direct ? "distance_direct" : "distance"; break;
    case SchemeKind::Leverage: base = "leverage"; break;
    case SchemeKind::NearestNeighbor: base = "nearest_neighbor"; break;
  }
  if (replacement && (kind == SchemeKind::Uniform || kind == SchemeKind::EuclideanNorm)) base += "_wr";
  return base;
}

int64_t sample_count(double s, int64_t m) {
  if (!(s > 0.0 && s <= 1.0)) throw RangeError("sample fraction must lie in (0, 1]");
  const int64_t c = static_cast<int64_t>(std::ceil(s * static_cast<double>(m)));
  return std::max<int64_t>(1, std::min(c, m));
}

namespace {
class WeightTree {  // Fenwick tree (sampling.hpp:78-104)
 public:
  explicit WeightTree(const std::vector<double>& w) : n_(w.size()), tree_(w.size() + 1, 0.0) {
    for (size_t i = 0; i < n_; ++i) add(i, w[i]);
  }
  size_t find(double u) const {
    size_t pos = 0, mask = 1;
    while ((mask << 1) <= n_) mask <<= 1;
    for (; mask > 0; mask >>= 1) {
      const size_t next = pos + mask;
      if (next <= n_ && tree_[next] <= u) {
        u -= tree_[next];
        pos = next;
      }
    }
    return std::min(pos, n_ - 1);
  }
  void add(size_t i, double delta) {
    for (size_t k = i + 1; k <= n_; k += k & (~k + 1)) tree_[k] += delta;
  }

 private:
  size_t n_;
  std::vector<double> tree_;
};

double center_distance(const PointSet& ps, int64_t pt, const std::vector<double>& c) {
  double diff = ps(pt, 0) - c[0];
  double acc = diff * diff;
  for (int64_t k = 1; k < ps.cols; ++k) {
    diff = ps(pt, k) - c[static_cast<size_t>(k)];
    acc += diff * diff;
  }
  return std::sqrt(acc);
}
}  // namespace

std::vector<int64_t> weighted_draw(const std::vector<double>& weights, int64_t count, bool replacement, Rng& rng) {
  const size_t m = weights.size();
  double total = std::accumulate(weights.begin(), weights.end(), 0.0);
  for (double w : weights)
    if (w < 0.0 || !std::isfinite(w)) throw RangeError("sample_rows: invalid (negative or non-finite) weight");
  if (!(total > 0.0)) throw Error("sample_rows: zero total weight");
  std::vector<int64_t> out;
  out.reserve(static_cast<size_t>(count));
  if (replacement) {
    std::vector<double> cum(m);
    std::partial_sum(weights.begin(), weights.end(), cum.begin());
    for (int64_t k = 0; k < count; ++k) {
      const double u = rng.uniform01() * total;
      size_t idx = static_cast<size_t>(std::upper_bound(cum.begin(), cum.end(), u) - cum.begin());
      if (idx >= m) idx = m - 1;
      out.push_back(static_cast<int64_t>(idx));
    }
    return out;
  }
  WeightTree tree(weights);
  std::vector<double> live = weights;
  for (int64_t k = 0; k < count; ++k) {
    const double u = rng.uniform01() * total;
    size_t idx = tree.find(u);
    if (live[idx] <= 0.0) {
      size_t probe = idx;
      while (probe + 1 < m && live[probe] <= 0.0) ++probe;
      while (probe > 0 && live[probe] <= 0.0) --probe;
      idx = probe;
    }
    out.push_back(static_cast<int64_t>(idx));
    total -= live[idx];
    tree.add(idx, -live[idx]);
    live[idx] = 0.0;
    if (!(total > 0.0) && k + 1 < count) throw Error("sample_rows: weights exhausted before reaching the requested count");
  }
  return out;
}

RowSample sample_rows(const SamplingScheme& scheme, const SampleContext& ctx, double s, std::uint64_t seed) {
  if (ctx.m < 1) throw RangeError("sample_rows: context must have m >= 1 rows");
  RowSample out;
  out.fraction = s;
  out.seed = seed;
  Rng rng(seed);
  const int64_t m = ctx.m;
  switch (scheme.kind) {
    case SchemeKind::Uniform: {
      const int64_t count = sample_count(s, m);
      if (scheme.replacement) {
        for (int64_t k = 0; k < count; ++k) out.indices.push_back(static_cast<int64_t>(rng.below(static_cast<std::uint64_t>(m))));
      } else {
        std::vector<int64_t> pool(static_cast<size_t>(m));
        std::iota(pool.begin(), pool.end(), int64_t{0});
        for (int64_t k = 0; k < count; ++k) {
          const size_t j = static_cast<size_t>(k) + static_cast<size_t>(rng.below(static_cast<std::uint64_t>(m - k)));
          std::swap(pool[static_cast<size_t>(k)], pool[j]);
          out.indices.push_back(pool[static_cast<size_t>(k)]);
        }
      }
      break;
    }
    case SchemeKind::Bernoulli: {
      if (!(s > 0.0 && s <= 1.0)) throw RangeError("sample fraction must lie in (0, 1]");
      for (int64_t i = 0; i < m; ++i)
        if (rng.uniform01() < s) out.indices.push_back(i);
      break;
    }
    case SchemeKind::EuclideanNorm: {
      if (ctx.K == nullptr) throw Error("sample_rows: EuclideanNorm scheme requires the matrix K");
      if (ctx.K->rows() != m) throw DimensionError("sample_rows: K row count disagrees with context m");
      const std::vector<double> w = ctx.K->row_norms();  // pass 2a on the device
      out.indices = weighted_draw(w, sample_count(s, m), scheme.replacement, rng);
      break;
    }
    case SchemeKind::Distance: {
      if (ctx.split == nullptr || ctx.points == nullptr)
        throw Error("sample_rows: Distance scheme requires the source/target split and points");
      if (static_cast<int64_t>(ctx.split->target_indices.size()) != m)
        throw DimensionError("sample_rows: split target count disagrees with context m");
      std::vector<double> w(static_cast<size_t>(m));
      for (int64_t i = 0; i < m; ++i) {
        const double dist = center_distance(*ctx.points, ctx.split->target_indices[static_cast<size_t>(i)], ctx.split->center);
        w[static_cast<size_t>(i)] = scheme.distance_direct ? dist : 1.0 / std::max(dist, std::numeric_limits<double>::min());
      }
      out.indices = weighted_draw(w, sample_count(s, m), false, rng);
      break;
    }
    case SchemeKind::Leverage: {
      if (ctx.K == nullptr) throw Error("sample_rows: Leverage scheme requires the matrix K");
      if (ctx.K->rows() != m) throw DimensionError("sample_rows: K row count disagrees with context m");
      if (scheme.rank_for_leverage < 1) throw RangeError("sample_rows: rank_for_leverage must be >= 1");
      const int64_t r = std::min(scheme.rank_for_leverage, std::min(ctx.K->rows(), ctx.K->cols()));
      const std::vector<double> w = row_leverage_scores(*ctx.K, r).scores;  // pass 2b on the device
      out.indices = weighted_draw(w, sample_count(s, m), false, rng);
      break;
    }
    case SchemeKind::NearestNeighbor: {
      if (ctx.split == nullptr || ctx.points == nullptr)
        throw Error("sample_rows: NearestNeighbor scheme requires the source/target split and points");
      if (static_cast<int64_t>(ctx.split->target_indices.size()) != m)
        throw DimensionError("sample_rows: split target count disagrees with context m");
      const int64_t count = sample_count(s, m);
      std::vector<std::pair<double, int64_t>> by_dist;
      by_dist.reserve(static_cast<size_t>(m));
      for (int64_t i = 0; i < m; ++i)
        by_dist.emplace_back(center_distance(*ctx.points, ctx.split->target_indices[static_cast<size_t>(i)], ctx.split->center), i);
      std::sort(by_dist.begin(), by_dist.end());
      for (int64_t k = 0; k < count; ++k) out.indices.push_back(by_dist[static_cast<size_t>(k)].second);
      break;
    }
  }
  return out;
}

// ------------------------------------------------------------------ compress
int64_t RankRule::resolve(const std::vector<double>& sv) const {
  if (fixed_r) {
    if (*fixed_r < 0) throw RangeError("rank rule: fixed rank must be nonnegative");
    return std::min<int64_t>(*fixed_r, static_cast<int64_t>(sv.size()));
  }
  if (!eps) throw ConfigError("rank rule: either eps or fixed_r must be set");
  return epsilon_rank(sv, *eps, reference_sigma1);
}

double bound_id_value(int64_t n, int64_t r, double sigma_r1) {
  if (r < 0 || r > n) throw RangeError("bound_id_value: requires 0 <= r <= n");
  const double nn = static_cast<double>(n), rr = static_cast<double>(r);
  return std::sqrt(1.0 + nn * rr * (nn - rr)) * sigma_r1;
}

double reconstruction_bound(int64_t m, int64_t s_count, double eps, double sigma_r1) {
  if (s_count < 1) throw RangeError("reconstruction_bound: requires s_count >= 1");
  if (!(eps > 0.0 && eps < 1.0)) throw RangeError("reconstruction_bound: requires eps in (0, 1)");
  if (sigma_r1 < 0.0) throw RangeError("reconstruction_bound: requires sigma_r1 >= 0");
  const double ratio = static_cast<double>(m) / static_cast<double>(s_count);
  return std::sqrt(1.0 + ratio * (1.0 + eps) / ((1.0 - eps) * (1.0 - eps))) * sigma_r1;
}

namespace {
double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

// D^T D is zero on the skeleton rows / columns (P[:, skel] = I): its spectrum is that of the
// (m - r) x (m - r) non-skeleton block.
static Matrix nonskeleton_block(const Matrix& DtD, const std::vector<int64_t>& skel) {
  const int64_t m = DtD.rows;
  std::vector<char> in(static_cast<size_t>(m), 0);
  for (int64_t j : skel) in[static_cast<size_t>(j)] = 1;
  std::vector<int64_t> b;
  for (int64_t i = 0; i < m; ++i)
    if (!in[static_cast<size_t>(i)]) b.push_back(i);
  const int64_t n = static_cast<int64_t>(b.size());
  Matrix S(n, n);
  for (int64_t y = 0; y < n; ++y)
    for (int64_t x = 0; x < n; ++x) S(x, y) = DtD(b[static_cast<size_t>(x)], b[static_cast<size_t>(y)]);
  return S;
}

// compress.hpp:168-215 with the error pass on the device.
std::pair<IDFactorization, CompressionReport> compress_id(const KernelBlock& K, const RowSample& sample,
                                                          const RankRule& rule, const CompressOptions& opts) {
  if (sample.indices.empty()) throw RangeError("compress_id: empty row sample");
  CompressionReport rep;
  rep.fraction = sample.fraction;
  rep.seed = sample.seed;
  double t0 = now_ms();
  const Matrix sub = K.rows_exact(sample.indices);
  rep.timings.sample_ms = now_ms() - t0;
  t0 = now_ms();
  const std::vector<double> sv = singular_values(sub);
  const int64_t r = rule.resolve(sv);
  rep.rank = r;
  rep.sigma1_sample = sv[0];
  rep.sigma_r1_sample = (r < static_cast<int64_t>(sv.size())) ? sv[static_cast<size_t>(r)] : 0.0;
  rep.bound_id = bound_id_value(K.cols(), r, rep.sigma_r1_sample);
  IDFactorization id;
  if (r == 0) {
    rep.rank_zero = true;
    rep.timings.factor_ms = now_ms() - t0;
    rep.rel_error = 1.0;
    rep.rel_error_fro = 1.0;
  } else {
    id = interpolative_decomposition(sub, r);
    rep.timings.factor_ms = now_ms() - t0;
    t0 = now_ms();
    const int64_t m = K.cols();
    Matrix DtD(m, m);
    double sd = 0.0, sk = 0.0;
    K.device().check(kid_recon_error(K.device().ctx(), K.spec().h, id.skeleton.data(), r, id.projection.data(),
                                     KID_RECON_DTD, &sd, &sk, DtD.data(), nullptr));
    const double num = std::sqrt(lambda_max(nonskeleton_block(DtD, id.skeleton)));
    const double den = opts.k_norm ? *opts.k_norm : K.spectral_norm();
    rep.rel_error = (den > 0.0) ? num / den : 0.0;
    rep.rel_error_fro = (sk > 0.0) ? std::sqrt(sd / sk) : 0.0;
    rep.timings.error_ms = now_ms() - t0;
  }
  if (opts.full_spectrum) {
    const auto& fs = *opts.full_spectrum;
    const double sig = (r < static_cast<int64_t>(fs.size())) ? fs[static_cast<size_t>(r)] : 0.0;
    rep.bound_sampling = reconstruction_bound(K.rows(), static_cast<int64_t>(sample.indices.size()), opts.theorem_eps, sig);
  }
  return {std::move(id), rep};
}

namespace {
// G = (K V_perp)^T (K V_perp) through the fused residual-Gram pass: with a = the ID skeleton of
// V_r^T (CPQR) and P = [I, T] its projection, V_r^T V_perp = 0 gives T = -C_a C_b^-1 (C = V_perp
// split by rows a / b), hence K V_perp = (K - K[:, a] P)[:, b] C_b: kid_recon_error on (a, P)
// yields D'^T D' and G = C_b^T (D'^T D') C_b (C_b shares its singular values with V_r[a, :]).
// Any orthonormal basis V_perp of the complement works. Optionally K^T K of the same pass.
Matrix svd_residual_gram(Device& dev, double h, const Matrix& Vr, const Matrix& Vp, double* sumsq_K, Matrix* KtK) {
  const int64_t m = Vr.rows, r = Vr.cols, n = m - r;
  Matrix VrT(r, m);
  for (int64_t j = 0; j < r; ++j)
    for (int64_t i = 0; i < m; ++i) VrT(j, i) = Vr(i, j);
  const IDFactorization idv = interpolative_decomposition(VrT, r);
  Matrix DtDm(m, m);
  double sdp = 0.0, sk = 0.0;
  dev.check(kid_recon_error(dev.ctx(), h, idv.skeleton.data(), r, idv.projection.data(),
                            KID_RECON_DTD | (KtK ? KID_RECON_KTK : 0u), &sdp, &sk, DtDm.data(),
                            KtK ? KtK->data() : nullptr));
  if (sumsq_K) *sumsq_K = sk;
  std::vector<char> in_a(static_cast<size_t>(m), 0);
  for (int64_t j : idv.skeleton) in_a[static_cast<size_t>(j)] = 1;
  std::vector<int64_t> b;
  for (int64_t i = 0; i < m; ++i)
    if (!in_a[static_cast<size_t>(i)]) b.push_back(i);
  Matrix Gp(n, n), Cb(n, n), T1(n, n), G(n, n);
  for (int64_t y = 0; y < n; ++y)
    for (int64_t x = 0; x < n; ++x) {
      Gp(x, y) = DtDm(b[static_cast<size_t>(x)], b[static_cast<size_t>(y)]);
      Cb(x, y) = Vp(b[static_cast<size_t>(x)], y);
    }
  for (int64_t y = 0; y < n; ++y)  // T1 = G' C_b
    for (int64_t x = 0; x < n; ++x) {
      double acc = 0.0;
      for (int64_t l = 0; l < n; ++l) acc += Gp(x, l) * Cb(l, y);
      T1(x, y) = acc;
    }
  for (int64_t y = 0; y < n; ++y)  // G = C_b^T T1
    for (int64_t x = 0; x < n; ++x) {
      double acc = 0.0;
      for (int64_t l = 0; l < n; ++l) acc += Cb(l, x) * T1(l, y);
      G(x, y) = acc;
    }
  return G;
}
}  // namespace

// compress.hpp:219-273 with the error pass on the device: ||K - K V_r V_r^T||_2 = ||K V_perp||_2,
// V_perp = the trailing m - r columns of the full right factor, through the fused residual-Gram
// pass (kid_recon_error) on the ID of V_r^T (the N_T x m difference is never formed; the generic
// kid_proj_gram computes the same Gram directly at about twice the cost).
std::pair<Matrix, CompressionReport> compress_svd(const KernelBlock& K, const RowSample& sample, const RankRule& rule,
                                                  const CompressOptions& opts) {
  if (sample.indices.empty()) throw RangeError("compress_svd: empty row sample");
  CompressionReport rep;
  rep.fraction = sample.fraction;
  rep.seed = sample.seed;
  double t0 = now_ms();
  const Matrix sub = K.rows_exact(sample.indices);
  rep.timings.sample_ms = now_ms() - t0;
  t0 = now_ms();
  const RightFactor rf = right_factor(sub);
  const int64_t r = rule.resolve(rf.singular_values);
  rep.rank = r;
  rep.sigma1_sample = rf.singular_values[0];
  rep.sigma_r1_sample = (r < static_cast<int64_t>(rf.singular_values.size())) ? rf.singular_values[static_cast<size_t>(r)] : 0.0;
  rep.timings.factor_ms = now_ms() - t0;
  const int64_t m = K.cols();
  Matrix Vr(m, r);
  t0 = now_ms();
  if (r == 0) {
    rep.rank_zero = true;
    rep.rel_error = 1.0;
    rep.rel_error_fro = 1.0;
  } else {
    for (int64_t j = 0; j < r; ++j)
      for (int64_t i = 0; i < m; ++i) Vr(i, j) = rf.V(i, j);
    double num = 0.0, sd = 0.0, sk = 0.0;
    if (r < m) {
      const int64_t n = m - r;
      Matrix Vp(m, n);
      for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) Vp(i, j) = rf.V(i, r + j);
      const Matrix G = svd_residual_gram(K.device(), K.spec().h, Vr, Vp, &sk, nullptr);
      for (int64_t i = 0; i < n; ++i) sd += G(i, i);
      std::vector<double> ev;
      sym_eig(G, ev, nullptr);
      num = std::sqrt(std::max(ev.empty() ? 0.0 : ev[0], 0.0));
    } else {
      K.gram(&sk);  // V_r spans R^m: the difference is rounding only
    }
    const double den = opts.k_norm ? *opts.k_norm : K.spectral_norm();
    rep.rel_error = (den > 0.0) ? num / den : 0.0;
    rep.rel_error_fro = (sk > 0.0) ? std::sqrt(sd / sk) : 0.0;
  }
  rep.timings.error_ms = now_ms() - t0;
  if (opts.full_spectrum) {
    const auto& fs = *opts.full_spectrum;
    const double sig = (r < static_cast<int64_t>(fs.size())) ? fs[static_cast<size_t>(r)] : 0.0;
    rep.bound_sampling = reconstruction_bound(K.rows(), static_cast<int64_t>(sample.indices.size()), opts.theorem_eps, sig);
  }
  return {std::move(Vr), rep};
}

std::vector<double> mc_error(const KernelBlock& K, const IDFactorization& id, double s_mc, int n_mc,
                             std::uint64_t seed) {
  if (!(s_mc > 0.0 && s_mc <= 1.0)) throw RangeError("mc_error: requires s_mc in (0, 1]");
  if (n_mc < 1) throw RangeError("mc_error: requires n_mc >= 1");
  kid_ctx* c = K.device().ctx();
  const int64_t m = K.cols(), r = id.rank;
  SamplingScheme bern;
  bern.kind = SchemeKind::Bernoulli;
  SampleContext ctx;
  ctx.m = K.rows();
  std::vector<double> estimates;
  estimates.reserve(static_cast<size_t>(n_mc));
  for (int rep = 0; rep < n_mc; ++rep) {
    RowSample rows = sample_rows(bern, ctx, s_mc, derive_seed(seed, static_cast<std::uint64_t>(rep)));
    if (rows.indices.empty()) rows = sample_rows(bern, ctx, s_mc, derive_seed(seed, static_cast<std::uint64_t>(rep), 1));
    if (rows.indices.empty()) throw Error("mc_error: Bernoulli draw empty twice; s_mc is too small for this matrix");
    K.device().check(kid_select_rows(c, rows.indices.data(), static_cast<int64_t>(rows.indices.size())));
    Matrix DtD(m, m), KtK(m, m);
    double sd = 0.0, sk = 0.0;
    const int rc = kid_recon_error(c, K.spec().h, id.skeleton.data(), r, r ? id.projection.data() : nullptr,
                                   KID_RECON_DTD | KID_RECON_KTK, &sd, &sk, DtD.data(), KtK.data());
    K.device().check(kid_select_rows(c, nullptr, -1));  // the full block again
    K.device().check(rc);
    std::vector<double> ed, ek;
    sym_eig(DtD, ed, nullptr);
    sym_eig(KtK, ek, nullptr);
    const double num = std::sqrt(std::max(ed.empty() ? 0.0 : ed[0], 0.0));
    const double den = std::sqrt(std::max(ek.empty() ? 0.0 : ek[0], 0.0));
    estimates.push_back(den > 0.0 ? num / den : (num > 0.0 ? std::numeric_limits<double>::infinity() : 0.0));
  }
  return estimates;
}

Matrix complement_basis(const Matrix& Vr) {
  const int64_t m = Vr.rows, r = Vr.cols;
  if (r > m) throw DimensionError("complement_basis: more columns than rows");
  Matrix A = Vr;
  std::vector<std::vector<double>> vs;  // Householder vectors (v[0] = 1, from row j), tau
  std::vector<double> taus;
  for (int64_t j = 0; j < r; ++j) {
    double nrm = 0.0;
    for (int64_t i = j; i < m; ++i) nrm += A(i, j) * A(i, j);
    nrm = std::sqrt(nrm);
    std::vector<double> v(static_cast<size_t>(m - j), 0.0);
    double tau = 0.0;
    if (nrm > 0.0) {
      const double alpha = A(j, j), beta = alpha >= 0.0 ? -nrm : nrm, v0 = alpha - beta;
      tau = -v0 / beta;
      v[0] = 1.0;
      for (int64_t i = 1; i < m - j; ++i) v[static_cast<size_t>(i)] = A(j + i, j) / v0;
      for (int64_t k = j; k < r; ++k) {
        double w = 0.0;
        for (int64_t i = 0; i < m - j; ++i) w += v[static_cast<size_t>(i)] * A(j + i, k);
        w *= tau;
        for (int64_t i = 0; i < m - j; ++i) A(j + i, k) -= w * v[static_cast<size_t>(i)];
      }
    }
    vs.push_back(std::move(v));
    taus.push_back(tau);
  }
  Matrix Q(m, m - r);  // Q e_k = H_0 H_1 ... H_{r-1} e_k, k = r..m-1
  for (int64_t c = 0; c < m - r; ++c) {
    std::vector<double> x(static_cast<size_t>(m), 0.0);
    x[static_cast<size_t>(r + c)] = 1.0;
    for (int64_t j = r - 1; j >= 0; --j) {
      const auto& v = vs[static_cast<size_t>(j)];
      double w = 0.0;
      for (int64_t i = 0; i < m - j; ++i) w += v[static_cast<size_t>(i)] * x[static_cast<size_t>(j + i)];
      w *= taus[static_cast<size_t>(j)];
      for (int64_t i = 0; i < m - j; ++i) x[static_cast<size_t>(j + i)] -= w * v[static_cast<size_t>(i)];
    }
    for (int64_t i = 0; i < m; ++i) Q(i, c) = x[static_cast<size_t>(i)];
  }
  return Q;
}

std::vector<double> mc_error_svd(const KernelBlock& K, const Matrix& Vr, double s_mc, int n_mc, std::uint64_t seed) {
  if (!(s_mc > 0.0 && s_mc <= 1.0)) throw RangeError("mc_error: requires s_mc in (0, 1]");
  if (n_mc < 1) throw RangeError("mc_error: requires n_mc >= 1");
  kid_ctx* c = K.device().ctx();
  const int64_t m = K.cols(), n = m - Vr.cols;
  const Matrix Vp = n > 0 ? complement_basis(Vr) : Matrix();
  SamplingScheme bern;
  bern.kind = SchemeKind::Bernoulli;
  SampleContext ctx;
  ctx.m = K.rows();
  std::vector<double> estimates;
  for (int rep = 0; rep < n_mc; ++rep) {
    RowSample rows = sample_rows(bern, ctx, s_mc, derive_seed(seed, static_cast<std::uint64_t>(rep)));
    if (rows.indices.empty()) rows = sample_rows(bern, ctx, s_mc, derive_seed(seed, static_cast<std::uint64_t>(rep), 1));
    if (rows.indices.empty()) throw Error("mc_error: Bernoulli draw empty twice; s_mc is too small for this matrix");
    K.device().check(kid_select_rows(c, rows.indices.data(), static_cast<int64_t>(rows.indices.size())));
    Matrix KtK(m, m), DtD;
    double sk = 0.0;
    int rc = KID_OK;
    try {  // the row subset is restored whatever happens
      if (n > 0) DtD = svd_residual_gram(K.device(), K.spec().h, Vr, Vp, &sk, &KtK);
      else rc = kid_gram(c, K.spec().h, KtK.data(), &sk);
    } catch (...) {
      kid_select_rows(c, nullptr, -1);
      throw;
    }
    K.device().check(kid_select_rows(c, nullptr, -1));
    K.device().check(rc);
    std::vector<double> ed, ek;
    if (n > 0) sym_eig(DtD, ed, nullptr);
    sym_eig(KtK, ek, nullptr);
    const double num = std::sqrt(std::max(ed.empty() ? 0.0 : ed[0], 0.0));
    const double den = std::sqrt(std::max(ek.empty() ? 0.0 : ek[0], 0.0));
    estimates.push_back(den > 0.0 ? num / den : (num > 0.0 ? std::numeric_limits<double>::infinity() : 0.0));
  }
  return estimates;
}

std::vector<double> apply_skeleton(const KernelBlock& K, const IDFactorization& id, const std::vector<double>& q) {
  if (static_cast<int64_t>(q.size()) != id.projection.cols)
    throw DimensionError("apply_skeleton: charge count disagrees with the projection width");
  std::vector<double> u(static_cast<size_t>(std::max<int64_t>(K.rows(), 1)));
  K.device().check(kid_apply_skeleton(K.device().ctx(), K.spec().h, id.skeleton.data(), id.rank,
                                      id.rank ? id.projection.data() : nullptr, q.data(), u.data()));
  u.resize(static_cast<size_t>(K.rows()));
  return u;
}

// ------------------------------------------------------------------ harness
std::string format_double(double v) {
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof(buf), v);
  return std::string(buf, res.ptr);
}

namespace {
std::string format_int(long long v) {
  char buf[32];
  const auto res = std::to_chars(buf, buf + sizeof(buf), v);
  return std::string(buf, res.ptr);
}
double mean_of(const std::vector<double>& v) {
  if (v.empty()) return 0.0;
  double sum = 0.0;
  for (double x : v) sum += x;
  return sum / static_cast<double>(v.size());
}
double stddev_of(const std::vector<double>& v) {
  if (v.size() < 2) return 0.0;
  const double mu = mean_of(v);
  double acc = 0.0;
  for (double x : v) acc += (x - mu) * (x - mu);
  return std::sqrt(acc / static_cast<double>(v.size() - 1));
}
std::string csv_join(const std::vector<std::string>& cells) {
  std::string line;
  for (size_t i = 0; i < cells.size(); ++i) {
    if (i) line += ',';
    line += cells[i];
  }
  return line;
}
const std::vector<std::string>& compress_csv_header() {
  static const std::vector<std::string> header = {"dataset", "d", "N", "n", "xi", "kernel", "h", "method", "scheme",
                                                  "s", "trial", "seed", "rank", "rel_error", "mc_error", "bound_id",
                                                  "bound_sampling", "elapsed_ms"};
  return header;
}
}  // namespace

std::vector<double> resolve_center(const ExperimentConfig& cfg, const PointSet& points, std::uint64_t data_seed) {
  std::vector<double> center(static_cast<size_t>(points.cols), 0.0);
  if (cfg.center_mode == CenterMode::RandomPoint) {
    Rng crng(derive_seed(data_seed, 0xCE));
    const int64_t ci = static_cast<int64_t>(crng.below(static_cast<std::uint64_t>(points.rows)));
    for (int64_t k = 0; k < points.cols; ++k) center[static_cast<size_t>(k)] = points(ci, k);
  }
  return center;
}

// harness.hpp:143-328 (Normal dataset, RandomPoint center, method "id").
void run_experiment(Device& dev, const ExperimentConfig& cfg, std::ostream& out, std::ostream* log) {
  struct Accum {
    std::vector<double> errors, ranks, mc;
  };
  std::map<std::tuple<size_t, size_t, size_t>, Accum> accum;
  struct Row {
    std::tuple<size_t, size_t, int, size_t> key;
    std::vector<std::string> cells;
  };
  std::vector<Row> rows;
  for (size_t scheme_idx = 0; scheme_idx < cfg.schemes.size(); ++scheme_idx) {
    for (int trial = 0; trial < cfg.trials; ++trial) {
      const std::uint64_t data_seed = derive_seed(cfg.seed, static_cast<std::uint64_t>(trial), scheme_idx);
      // prepare_trial (harness.hpp:107-129)
      const PointSet points = gen_normal(cfg.d, cfg.N, derive_seed(data_seed, 0xDA7A));
      const std::vector<double> center = resolve_center(cfg, points, data_seed);
      SourceTargetSplit split;
      bool trial_failed = false;
      try {
        split = split_sources_targets(dev, points, center, cfg.n_sources, cfg.xi);
      } catch (const NoTargetsError& e) {
        trial_failed = true;
        if (log) *log << "trial " << trial << " scheme " << cfg.schemes[scheme_idx].name() << ": " << e.what() << "\n";
      }
      const double h_abs = cfg.h_in_silverman_units ? cfg.h_value * silverman_bandwidth(cfg.d, cfg.N) : cfg.h_value;
      SamplingScheme scheme = cfg.schemes[scheme_idx];
      std::optional<std::vector<double>> full_sv;
      RankRule rule = cfg.rank_rule;
      std::optional<KernelBlock> K;
      if (!trial_failed) {
        K.emplace(dev, KernelSpec::gaussian(h_abs), points, split);
        const bool auto_rank = scheme.kind == SchemeKind::Leverage && cfg.scheme_rank_auto[scheme_idx];
        const bool need_full = cfg.rank_reference_full || cfg.emit_bound_sampling || auto_rank;
        // harness.hpp:176-184: device TSQR for m <= 128; for m > 128 the Gram route, refined by its second
        // pass when an eps-rank below the Gram route's resolution (or the whole spectrum) is asked for
        const double need_level = (cfg.emit_bound_sampling || !rule.eps) ? 0.0 : *rule.eps;
        if (need_full) full_sv = K->singular_values(need_level);
        if (cfg.rank_reference_full) rule.reference_sigma1 = (*full_sv)[0];
        if (auto_rank) scheme.rank_for_leverage = std::max<int64_t>(1, rule.resolve(*full_sv));
      }
      for (size_t s_idx = 0; s_idx < cfg.s_grid.size(); ++s_idx) {
        const double s = cfg.s_grid[s_idx];
        const std::uint64_t sample_seed = derive_seed(data_seed, s_idx, 1);
        std::optional<RowSample> sample;
        std::string sample_error;
        if (!trial_failed) {
          SampleContext ctx;
          ctx.m = K->rows();
          ctx.K = &*K;
          ctx.split = &split;
          ctx.points = &points;
          try {
            RowSample drawn = sample_rows(scheme, ctx, s, sample_seed);
            if (drawn.indices.empty()) sample_error = "empty Bernoulli draw";
            else sample = std::move(drawn);
          } catch (const Error& e) {
            sample_error = e.what();
          }
          if (!sample_error.empty() && log) *log << "trial " << trial << " s=" << s << ": " << sample_error << "\n";
        }
        for (size_t method_idx = 0; method_idx < cfg.methods.size(); ++method_idx) {  // harness.hpp:211-289
          const CompressionMethod method = cfg.methods[method_idx];
          std::vector<std::string> cells(compress_csv_header().size());
          cells[0] = "normal";
          cells[1] = format_int(cfg.d);
          cells[2] = format_int(static_cast<long long>(cfg.N));
          cells[3] = format_int(static_cast<long long>(cfg.n_sources));
          cells[4] = format_double(cfg.xi);
          cells[5] = "gaussian";
          cells[6] = trial_failed ? "" : format_double(h_abs);
          cells[7] = method == CompressionMethod::ID ? "id" : "svd";
          cells[8] = cfg.schemes[scheme_idx].name();
          cells[9] = format_double(s);
          cells[10] = format_int(trial);
          cells[11] = format_int(static_cast<long long>(sample_seed));
          if (!trial_failed && sample) {
            CompressOptions opts;
            opts.theorem_eps = cfg.theorem_eps;
            if (full_sv && cfg.emit_bound_sampling) opts.full_spectrum = *full_sv;
            if (full_sv) opts.k_norm = (*full_sv)[0];
            const double t0 = now_ms();
            CompressionReport rep;
            std::optional<double> mc_mean;
            const std::uint64_t mc_seed = derive_seed(data_seed, s_idx, 2);
            if (method == CompressionMethod::ID) {
              auto [id, r] = compress_id(*K, *sample, rule, opts);
              rep = r;
              if (cfg.s_mc && !rep.rank_zero) mc_mean = mean_of(mc_error(*K, id, *cfg.s_mc, cfg.n_mc, mc_seed));
            } else {
              auto [Vr, r] = compress_svd(*K, *sample, rule, opts);
              rep = r;
              if (cfg.s_mc && !rep.rank_zero) mc_mean = mean_of(mc_error_svd(*K, Vr, *cfg.s_mc, cfg.n_mc, mc_seed));
            }
            const double elapsed = now_ms() - t0;
            cells[12] = format_int(static_cast<long long>(rep.rank));
            cells[13] = format_double(rep.rel_error);
            cells[14] = mc_mean ? format_double(*mc_mean) : "";
            cells[15] = rep.bound_id ? format_double(*rep.bound_id) : "";
            cells[16] = rep.bound_sampling ? format_double(*rep.bound_sampling) : "";
            cells[17] = cfg.emit_timings ? format_double(elapsed) : "";
            auto& acc = accum[{scheme_idx, s_idx, method_idx}];
            acc.errors.push_back(rep.rel_error);
            acc.ranks.push_back(static_cast<double>(rep.rank));
            if (mc_mean) acc.mc.push_back(*mc_mean);
          }
          rows.push_back({{scheme_idx, s_idx, trial, method_idx}, std::move(cells)});
        }
      }
    }
  }
  std::sort(rows.begin(), rows.end(), [](const Row& a, const Row& b) { return a.key < b.key; });
  out << csv_join(compress_csv_header()) << "\n";
  for (const Row& row : rows) out << csv_join(row.cells) << "\n";
  for (size_t scheme_idx = 0; scheme_idx < cfg.schemes.size(); ++scheme_idx)
    for (size_t s_idx = 0; s_idx < cfg.s_grid.size(); ++s_idx)
      for (size_t method_idx = 0; method_idx < cfg.methods.size(); ++method_idx) {
      const auto it = accum.find({scheme_idx, s_idx, method_idx});
      if (it == accum.end() || it->second.errors.empty()) continue;
      const Accum& acc = it->second;
      for (const char* stat : {"mean", "std"}) {
        const bool is_mean = std::string(stat) == "mean";
        if (!is_mean && acc.errors.size() < 2) continue;
        std::vector<std::string> cells(compress_csv_header().size());
        cells[0] = "normal";
        cells[1] = format_int(cfg.d);
        cells[2] = format_int(static_cast<long long>(cfg.N));
        cells[3] = format_int(static_cast<long long>(cfg.n_sources));
        cells[4] = format_double(cfg.xi);
        cells[5] = "gaussian";
        cells[7] = cfg.methods[method_idx] == CompressionMethod::ID ? "id" : "svd";
        cells[8] = cfg.schemes[scheme_idx].name();
        cells[9] = format_double(cfg.s_grid[s_idx]);
        cells[10] = stat;
        cells[12] = is_mean ? format_int(static_cast<long long>(std::llround(mean_of(acc.ranks)))) : "";
        cells[13] = is_mean ? format_double(mean_of(acc.errors)) : format_double(stddev_of(acc.errors));
        cells[14] = acc.mc.empty() ? "" : (is_mean ? format_double(mean_of(acc.mc)) : format_double(stddev_of(acc.mc)));
        out << csv_join(cells) << "\n";
      }
    }
}

// ------------------------------------------------------------------ interaction fractions
InteractionFractions interaction_fractions(Device& dev, const PointSet& ps, const KernelSpec& spec,
                                           const std::vector<double>& x_c, int64_t n) {
  spec.validate();
  const int64_t N = ps.rows;
  const int d = static_cast<int>(ps.cols);
  if (N < 2 * n) throw RangeError("interaction_fractions: requires N >= 2n");
  if (static_cast<int64_t>(x_c.size()) != d) throw DimensionError("interaction_fractions: center dimension mismatch");
  std::vector<double> dist(static_cast<size_t>(N));
  for (int64_t i = 0; i < N; ++i) dist[static_cast<size_t>(i)] = center_distance(ps, i, x_c);
  std::vector<int64_t> order(static_cast<size_t>(N));
  std::iota(order.begin(), order.end(), int64_t{0});
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {  // compress.hpp:344-347
    if (dist[static_cast<size_t>(a)] != dist[static_cast<size_t>(b)]) return dist[static_cast<size_t>(a)] < dist[static_cast<size_t>(b)];
    return a < b;
  });
  auto take = [&](int64_t from, int64_t count) {  // col-major count x d
    Matrix blk(count, d);
    for (int64_t i = 0; i < count; ++i)
      for (int k = 0; k < d; ++k) blk(i, k) = ps(order[static_cast<size_t>(from + i)], k);
    return blk;
  };
  const Matrix sources = take(0, n), neighbors = take(n, n), far = take(2 * n, N - 2 * n);
  auto block_gram = [&](const Matrix& tg) {
    Matrix G(n, n);
    dev.check(kid_set_block(dev.ctx(), tg.data(), tg.rows, sources.data(), n, d));
    dev.check(kid_gram(dev.ctx(), spec.h, G.data(), nullptr));
    return G;
  };
  const Matrix GS = block_gram(sources), GN = block_gram(neighbors);
  const Matrix GF = far.rows > 0 ? block_gram(far) : Matrix(n, n);
  Matrix GT(n, n);
  for (size_t e = 0; e < GT.a.size(); ++e) GT.a[e] = GS.a[e] + GN.a[e] + GF.a[e];
  const double total = std::sqrt(lambda_max(GT));
  InteractionFractions f;
  if (total > 0.0) {
    f.self_frac = std::sqrt(lambda_max(GS)) / total;
    f.nn_frac = std::sqrt(lambda_max(GN)) / total;
    f.far_frac = far.rows > 0 ? std::sqrt(lambda_max(GF)) / total : 0.0;
  }
  return f;
}

// ------------------------------------------------------------------ bandwidth search
BandwidthResult bandwidth_search(Device& dev, const ExperimentConfig& cfg, const BandwidthSearchSpec& spec,
                                 std::uint64_t data_seed) {
  // prepare_trial(cfg, data_seed, /*assemble_matrix=*/false) (harness.hpp:107-129)
  const PointSet points = gen_normal(cfg.d, cfg.N, derive_seed(data_seed, 0xDA7A));
  const std::vector<double> center = resolve_center(cfg, points, data_seed);
  const SourceTargetSplit split = split_sources_targets(dev, points, center, cfg.n_sources, cfg.xi);
  const double h_S = silverman_bandwidth(cfg.d, points.rows);
  const double target = spec.kappa * static_cast<double>(cfg.n_sources);
  BandwidthResult res;
  auto rank_at = [&](double h) -> long {
    const KernelBlock K(dev, KernelSpec::gaussian(h), points, split);
    const long r = static_cast<long>(epsilon_rank(K.singular_values(spec.eps), spec.eps));
    ++res.evaluations;
    res.profile.emplace_back(h, r);
    return r;
  };
  const bool increasing = !spec.large_h_branch;
  const std::vector<double> scan = {1e-3, 1e-2, 0.03, 0.1, 0.3, 1.0, 3.0, 10.0, 1e2};
  std::vector<std::pair<double, long>> coarse;
  size_t peak_idx = 0;
  for (size_t i = 0; i < scan.size(); ++i) {
    coarse.emplace_back(scan[i] * h_S, rank_at(scan[i] * h_S));
    if (coarse[i].second > coarse[peak_idx].second) peak_idx = i;
  }
  if (static_cast<double>(coarse[peak_idx].second) < target)
    throw SearchFailureError("bandwidth_search: rank budget " + std::to_string(target) +
                                 " exceeds the peak epsilon-rank " + std::to_string(coarse[peak_idx].second),
                             res.profile);
  double lo, hi;
  long rank_lo, rank_hi;
  if (increasing) {
    hi = coarse[peak_idx].first;
    rank_hi = coarse[peak_idx].second;
    size_t below = peak_idx;
    while (below > 0 && coarse[below].second >= target) --below;
    lo = coarse[below].first;
    rank_lo = coarse[below].second;
    for (int grow = 0; grow < 5 && rank_lo >= target; ++grow) {
      lo /= 2.0;
      rank_lo = rank_at(lo);
    }
  } else {
    lo = coarse[peak_idx].first;
    rank_lo = coarse[peak_idx].second;
    size_t above = peak_idx;
    while (above + 1 < coarse.size() && coarse[above].second >= target) ++above;
    hi = coarse[above].first;
    rank_hi = coarse[above].second;
    for (int grow = 0; grow < 5 && rank_hi >= target; ++grow) {
      hi *= 2.0;
      rank_hi = rank_at(hi);
    }
  }
  const bool bracketed = increasing ? (rank_lo < target && static_cast<double>(rank_hi) >= target)
                                    : (static_cast<double>(rank_lo) >= target && rank_hi < target);
  if (!bracketed)
    throw SearchFailureError("bandwidth_search: could not bracket the rank budget " + std::to_string(target) +
                                 " on the " + (increasing ? std::string("small_h") : std::string("large_h")) + " branch",
                             res.profile);
  double h_best = increasing ? hi : lo;
  long rank_best = increasing ? rank_hi : rank_lo;
  while (res.evaluations < spec.max_iters) {
    const double mid = std::sqrt(lo * hi);
    const long rank_mid = rank_at(mid);
    if (std::abs(static_cast<double>(rank_mid) - target) <= std::abs(static_cast<double>(rank_best) - target)) {
      h_best = mid;
      rank_best = rank_mid;
    }
    if (std::abs(static_cast<double>(rank_mid) - target) <= spec.rank_tolerance_rows) {
      res.converged = true;
      break;
    }
    const bool go_right = increasing ? (rank_mid < target) : (rank_mid >= target);
    if (go_right) lo = mid;
    else hi = mid;
  }
  res.h_abs = h_best;
  res.h_over_hs = h_best / h_S;
  res.rank = rank_best;
  return res;
}

}  // namespace kernid_b200

// ====================================================================== C exports
// Flat entry points over the mirror for the Python test/bench harness (ctypes).
using namespace kernid_b200;

namespace {
thread_local std::string g_err;
int guard(const std::function<void()>& fn) {
  try {
    fn();
    return 0;
  } catch (const RangeError& e) {
    g_err = e.what(); return KID_E_RANGE;
  } catch (const DimensionError& e) {
    g_err = e.what(); return KID_E_DIM;
  } catch (const NoTargetsError& e) {
    g_err = e.what(); return KID_E_NO_TARGETS;
  } catch (const NumericalError& e) {
    g_err = e.what(); return KID_E_NUMERICAL;
  } catch (const IllConditionedSkeletonError& e) {
    g_err = e.what(); return KID_E_ILLCOND;
  } catch (const ConfigError& e) {
    g_err = e.what(); return KID_E_CONFIG;
  } catch (const std::exception& e) {
    g_err = e.what(); return KID_E_ERROR;
  }
}
Matrix wrap(const double* a, int64_t rows, int64_t cols) {
  Matrix M(rows, cols);
  std::memcpy(M.data(), a, sizeof(double) * static_cast<size_t>(rows * cols));
  return M;
}
}  // namespace

extern "C" {

const char* kidh_last_error(void) { return g_err.c_str(); }

uint64_t kidh_derive_seed(uint64_t master, uint64_t a, uint64_t b) { return derive_seed(master, a, b); }

// resolve_center RandomPoint row (harness.hpp:95-100)
int64_t kidh_center_index(int64_t N, uint64_t data_seed) {
  Rng rng(derive_seed(data_seed, 0xCE));
  return static_cast<int64_t>(rng.below(static_cast<std::uint64_t>(N)));
}

int kidh_gen_normal(int32_t d, int64_t N, uint64_t seed, double* out) {
  return guard([&] {
    PointSet ps = gen_normal(d, N, seed);
    std::memcpy(out, ps.data(), sizeof(double) * static_cast<size_t>(N * d));
  });
}

int kidh_singular_values(const double* A, int64_t rows, int64_t cols, double* sv) {
  return guard([&] {
    const auto s = singular_values(wrap(A, rows, cols));
    std::memcpy(sv, s.data(), sizeof(double) * s.size());
  });
}

int kidh_epsilon_rank(const double* sv, int64_t n, double eps, double ref_sigma1, int64_t* r) {
  return guard([&] {
    std::vector<double> v(sv, sv + n);
    *r = epsilon_rank(v, eps, ref_sigma1 > 0.0 ? std::optional<double>(ref_sigma1) : std::nullopt);
  });
}

int kidh_interpolative_decomposition(const double* A, int64_t m, int64_t n, int64_t r, int64_t* skel, double* P) {
  return guard([&] {
    const IDFactorization id = interpolative_decomposition(wrap(A, m, n), r);
    std::memcpy(skel, id.skeleton.data(), sizeof(int64_t) * static_cast<size_t>(r));
    std::memcpy(P, id.projection.data(), sizeof(double) * static_cast<size_t>(r * n));
  });
}

int kidh_sym_eig(const double* A, int64_t n, double* evals, double* evecs) {
  return guard([&] {
    std::vector<double> ev;
    Matrix V;
    sym_eig(wrap(A, n, n), ev, evecs ? &V : nullptr);
    std::memcpy(evals, ev.data(), sizeof(double) * ev.size());
    if (evecs) std::memcpy(evecs, V.data(), sizeof(double) * static_cast<size_t>(n * n));
  });
}

int kidh_lambda_max(const double* A, int64_t n, double* lmax) {
  return guard([&] { *lmax = lambda_max(wrap(A, n, n)); });
}

int kidh_sym_eigvals(const double* A, int64_t n, double* evals) {
  return guard([&] {
    const std::vector<double> ev = sym_eigvals(wrap(A, n, n));
    std::memcpy(evals, ev.data(), sizeof(double) * ev.size());
  });
}

// kind: 0 Uniform, 1 Bernoulli, 2 EuclideanNorm, 4 Leverage (weights given: host draw only)
int kidh_draw(int32_t kind, int32_t replacement, int64_t m, const double* weights, double s, uint64_t seed,
              int64_t* out, int64_t* count) {
  return guard([&] {
    Rng rng(seed);
    std::vector<int64_t> idx;
    if (kind == 0 || kind == 1) {
      SamplingScheme sc;
      sc.kind = kind == 0 ? SchemeKind::Uniform : SchemeKind::Bernoulli;
      sc.replacement = replacement != 0;
      SampleContext ctx;
      ctx.m = m;
      idx = sample_rows(sc, ctx, s, seed).indices;
    } else {
      std::vector<double> w(weights, weights + m);
      idx = weighted_draw(w, sample_count(s, m), kind == 2 && replacement, rng);
    }
    std::memcpy(out, idx.data(), sizeof(int64_t) * idx.size());
    *count = static_cast<int64_t>(idx.size());
  });
}

// Host K rows with the reference arithmetic: K(rows, :) for targets/sources given by
// indices into a col-major N x d point set.
int kidh_kernel_rows(const double* pts, int64_t N, int32_t d, const int64_t* tgt_idx, const int64_t* rows,
                     int64_t count, const int64_t* src_idx, int64_t m, double h, double* out) {
  return guard([&] {
    const KernelSpec spec = KernelSpec::gaussian(h);
    spec.validate();
    for (int64_t i = 0; i < count; ++i)
      for (int64_t j = 0; j < m; ++j)
        out[i + j * count] = eval_kernel(spec, pts + tgt_idx[rows[i]], N, pts + src_idx[j], N, d);
  });
}

// The error pass of compress_id (compress.hpp:178-206) on a caller-owned kid_ctx holding the block
// K(T, S): num = sqrt(lambda_max(D^T D)) from kid_recon_error, den = ||K||_2 = sqrt(lambda_max(K^T K))
// from kid_gram unless k_norm > 0 is given (harness.hpp:237 caches it per trial). Host buffers in
// and out: the end-to-end path of bench.py.
int kidh_error_pass(void* ctx, double h, const int64_t* skel, int64_t r, const double* P, double k_norm,
                    double* rel_error, double* rel_error_fro, double* k_norm_out) {
  return guard([&] {
    kid_ctx* c = static_cast<kid_ctx*>(ctx);
    auto ck = [&](int rc) {
      if (rc != KID_OK) throw Error(std::string("kid: ") + kid_last_error(c));
    };
    int64_t nt = 0, m = 0;
    int32_t d = 0;
    ck(kid_block_shape(c, &nt, &m, &d));
    Matrix DtD(m, m);
    double sd = 0.0, sk = 0.0;
    ck(kid_recon_error(c, h, skel, r, P, KID_RECON_DTD, &sd, &sk, DtD.data(), nullptr));
    const std::vector<int64_t> sv(skel, skel + r);
    const double num = std::sqrt(lambda_max(nonskeleton_block(DtD, sv)));
    double den = k_norm;
    if (!(den > 0.0)) {
      Matrix G(m, m);
      ck(kid_gram(c, h, G.data(), nullptr));
      den = std::sqrt(lambda_max(G));
    }
    *rel_error = den > 0.0 ? num / den : 0.0;
    *rel_error_fro = sk > 0.0 ? std::sqrt(sd / sk) : 0.0;
    if (k_norm_out) *k_norm_out = den;
  });
}

// One compress trial through the mirror on device `device` (harness prepare_trial + sample_rows
// + compress_id). scheme: 0 uniform, 2 euclidean_norm, 4 leverage (rank lev_rank; <= 0: auto).
int kidh_compress_trial(int32_t device, int32_t d, int64_t N, int64_t n, double xi, double h_value,
                        uint64_t data_seed, int32_t scheme, int64_t lev_rank, double s, uint64_t sample_seed,
                        double eps, int64_t* n_targets, int64_t* rank, double* rel_error, double* rel_error_fro,
                        int64_t* skel_out, int64_t* sample_out, int64_t* sample_count_out) {
  return guard([&] {
    Device dev(device);
    const PointSet points = gen_normal(d, N, derive_seed(data_seed, 0xDA7A));
    Rng crng(derive_seed(data_seed, 0xCE));
    const int64_t ci = static_cast<int64_t>(crng.below(static_cast<std::uint64_t>(N)));
    std::vector<double> center(static_cast<size_t>(d));
    for (int k = 0; k < d; ++k) center[static_cast<size_t>(k)] = points(ci, k);
    const SourceTargetSplit split = split_sources_targets(dev, points, center, n, xi);
    const KernelBlock K(dev, KernelSpec::gaussian(h_value * silverman_bandwidth(d, N)), points, split);
    *n_targets = K.rows();
    SamplingScheme sc;
    sc.kind = scheme == 2 ? SchemeKind::EuclideanNorm : scheme == 4 ? SchemeKind::Leverage : SchemeKind::Uniform;
    RankRule rule = RankRule::from_eps(eps);
    if (sc.kind == SchemeKind::Leverage) {
      if (lev_rank > 0) {
        sc.rank_for_leverage = lev_rank;
      } else {  // auto rank from the full spectrum (harness.hpp:176-184): device TSQR
        sc.rank_for_leverage = std::max<int64_t>(1, rule.resolve(K.singular_values(eps)));
      }
    }
    SampleContext ctx;
    ctx.m = K.rows();
    ctx.K = &K;
    ctx.split = &split;
    ctx.points = &points;
    const RowSample sample = sample_rows(sc, ctx, s, sample_seed);
    std::memcpy(sample_out, sample.indices.data(), sizeof(int64_t) * sample.indices.size());
    *sample_count_out = static_cast<int64_t>(sample.indices.size());
    auto [id, rep] = compress_id(K, sample, rule);
    *rank = rep.rank;
    *rel_error = rep.rel_error;
    *rel_error_fro = rep.rel_error_fro;
    std::memcpy(skel_out, id.skeleton.data(), sizeof(int64_t) * id.skeleton.size());
  });
}

// kidh_compress_trial with the targets sharded over `G` devices (EuclideanNorm sampling): the
// multi-GPU mirror (DeviceGroup, ShardedBlock; NCCL reductions when the devices are distinct).
int kidh_sharded_compress_trial(const int32_t* devices, int32_t G, int32_t d, int64_t N, int64_t n, double xi,
                                double h_value, uint64_t data_seed, double s, uint64_t sample_seed, double eps,
                                int64_t* n_targets, int64_t* rank, double* rel_error, double* rel_error_fro,
                                int64_t* skel_out, int64_t* sample_out, int64_t* sample_count_out, int32_t* used_nccl) {
  return guard([&] {
    DeviceGroup grp(std::vector<int>(devices, devices + G));
    const PointSet points = gen_normal(d, N, derive_seed(data_seed, 0xDA7A));
    Rng crng(derive_seed(data_seed, 0xCE));
    const int64_t ci = static_cast<int64_t>(crng.below(static_cast<std::uint64_t>(N)));
    std::vector<double> center(static_cast<size_t>(d));
    for (int k = 0; k < d; ++k) center[static_cast<size_t>(k)] = points(ci, k);
    const ShardedSplit split = split_sources_targets(grp, points, center, n, xi);
    const ShardedBlock K(grp, KernelSpec::gaussian(h_value * silverman_bandwidth(d, N)), points, split);
    *n_targets = K.rows();
    const RowSample sample = sample_rows_euclidean(K, s, sample_seed);
    std::memcpy(sample_out, sample.indices.data(), sizeof(int64_t) * sample.indices.size());
    *sample_count_out = static_cast<int64_t>(sample.indices.size());
    auto [id, rep] = compress_id(K, sample, RankRule::from_eps(eps));
    *rank = rep.rank;
    *rel_error = rep.rel_error;
    *rel_error_fro = rep.rel_error_fro;
    std::memcpy(skel_out, id.skeleton.data(), sizeof(int64_t) * id.skeleton.size());
    *used_nccl = grp.uses_nccl() ? 1 : 0;
  });
}

// One compress trial (as kidh_compress_trial, uniform sampling) followed by the 8(f) passes on
// its ID: mc_error (n_mc estimates) and apply_skeleton with charges q (m) -> u (n_targets).
int kidh_trial_next_rows(int32_t device, int32_t d, int64_t N, int64_t n, double xi, double h_value,
                         uint64_t data_seed, double s, uint64_t sample_seed, double eps, double s_mc, int32_t n_mc,
                         uint64_t mc_seed, const double* q, int64_t* n_targets, int64_t* rank, int64_t* skel_out,
                         double* P_out, double* mc_out, double* u_out, int64_t u_cap) {
  return guard([&] {
    Device dev(device);
    const PointSet points = gen_normal(d, N, derive_seed(data_seed, 0xDA7A));
    Rng crng(derive_seed(data_seed, 0xCE));
    const int64_t ci = static_cast<int64_t>(crng.below(static_cast<std::uint64_t>(N)));
    std::vector<double> center(static_cast<size_t>(d));
    for (int k = 0; k < d; ++k) center[static_cast<size_t>(k)] = points(ci, k);
    const SourceTargetSplit split = split_sources_targets(dev, points, center, n, xi);
    const KernelBlock K(dev, KernelSpec::gaussian(h_value * silverman_bandwidth(d, N)), points, split);
    *n_targets = K.rows();
    SampleContext ctx;
    ctx.m = K.rows();
    const RowSample sample = sample_rows(SamplingScheme{}, ctx, s, sample_seed);
    auto [id, rep] = compress_id(K, sample, RankRule::from_eps(eps));
    *rank = rep.rank;
    std::memcpy(skel_out, id.skeleton.data(), sizeof(int64_t) * id.skeleton.size());
    if (rep.rank) std::memcpy(P_out, id.projection.data(), sizeof(double) * id.projection.a.size());
    if (rep.rank == 0) {  // the zero-rank ID still reconstructs K as 0
      id.projection = Matrix(0, K.cols());
    }
    const std::vector<double> est = mc_error(K, id, s_mc, n_mc, mc_seed);
    std::memcpy(mc_out, est.data(), sizeof(double) * est.size());
    const std::vector<double> u = apply_skeleton(K, id, std::vector<double>(q, q + K.cols()));
    if (static_cast<int64_t>(u.size()) > u_cap) throw RangeError("kidh_trial_next_rows: u buffer too small");
    std::memcpy(u_out, u.data(), sizeof(double) * u.size());
  });
}

// The full-block spectrum of a trial's K(T, S) through the mirror (KernelBlock::right_factor(resolve):
// lowrank.hpp:56-90 on the device) and, for lev_rank > 0, row_leverage_scores(K, lev_rank)
// (lowrank.hpp:296-308). sv_out n values, V_out n x n col-major, scores_out n_targets (cap score_cap).
int kidh_trial_spectrum(int32_t device, int32_t d, int64_t N, int64_t n, double xi, double h_value,
                        uint64_t data_seed, double resolve, int64_t lev_rank, int64_t* n_targets, double* sv_out,
                        double* V_out, double* scores_out, int64_t score_cap) {
  return guard([&] {
    Device dev(device);
    const PointSet points = gen_normal(d, N, derive_seed(data_seed, 0xDA7A));
    Rng crng(derive_seed(data_seed, 0xCE));
    const int64_t ci = static_cast<int64_t>(crng.below(static_cast<std::uint64_t>(N)));
    std::vector<double> center(static_cast<size_t>(d));
    for (int k = 0; k < d; ++k) center[static_cast<size_t>(k)] = points(ci, k);
    const SourceTargetSplit split = split_sources_targets(dev, points, center, n, xi);
    const KernelBlock K(dev, KernelSpec::gaussian(h_value * silverman_bandwidth(d, N)), points, split);
    *n_targets = K.rows();
    const RightFactor rf = K.right_factor(resolve);
    for (int64_t i = 0; i < n; ++i)
      sv_out[i] = i < static_cast<int64_t>(rf.singular_values.size()) ? rf.singular_values[static_cast<size_t>(i)] : 0.0;
    if (V_out) std::memcpy(V_out, rf.V.data(), sizeof(double) * static_cast<size_t>(n) * static_cast<size_t>(n));
    if (lev_rank > 0) {
      const LeverageScores ls = row_leverage_scores(K, lev_rank);
      if (static_cast<int64_t>(ls.scores.size()) > score_cap) throw RangeError("kidh_trial_spectrum: score buffer too small");
      std::memcpy(scores_out, ls.scores.data(), sizeof(double) * ls.scores.size());
    }
  });
}

// One compress_svd trial (uniform sampling): rank, rel_error, rel_error_fro and V_r (m x rank).
int kidh_trial_svd(int32_t device, int32_t d, int64_t N, int64_t n, double xi, double h_value, uint64_t data_seed,
                   double s, uint64_t sample_seed, double eps, int64_t* rank, double* rel, double* rel_fro,
                   double* Vr_out) {
  return guard([&] {
    Device dev(device);
    const PointSet points = gen_normal(d, N, derive_seed(data_seed, 0xDA7A));
    Rng crng(derive_seed(data_seed, 0xCE));
    const int64_t ci = static_cast<int64_t>(crng.below(static_cast<std::uint64_t>(N)));
    std::vector<double> center(static_cast<size_t>(d));
    for (int k = 0; k < d; ++k) center[static_cast<size_t>(k)] = points(ci, k);
    const SourceTargetSplit split = split_sources_targets(dev, points, center, n, xi);
    const KernelBlock K(dev, KernelSpec::gaussian(h_value * silverman_bandwidth(d, N)), points, split);
    SampleContext ctx;
    ctx.m = K.rows();
    const RowSample sample = sample_rows(SamplingScheme{}, ctx, s, sample_seed);
    auto [Vr, rep] = compress_svd(K, sample, RankRule::from_eps(eps));
    *rank = rep.rank;
    *rel = rep.rel_error;
    *rel_fro = rep.rel_error_fro;
    if (rep.rank) std::memcpy(Vr_out, Vr.data(), sizeof(double) * Vr.a.size());
  });
}

// interaction_fractions over gen_normal(d, N, seed) points around x_c (d values).
int kidh_interaction_fractions(int32_t device, int32_t d, int64_t N, uint64_t seed, double h, const double* x_c,
                               int64_t n, double* fracs) {
  return guard([&] {
    Device dev(device);
    const PointSet ps = gen_normal(d, N, seed);
    const InteractionFractions f = interaction_fractions(dev, ps, KernelSpec::gaussian(h), std::vector<double>(x_c, x_c + d), n);
    fracs[0] = f.self_frac;
    fracs[1] = f.nn_frac;
    fracs[2] = f.far_frac;
  });
}

// bandwidth_search; out = [h_abs, h_over_hs, rank, evaluations, converged]; the (h, rank) profile
// (also on SearchFailureError, status KID_E_ERROR) into prof (2 x prof_cap), its length into n_prof.
int kidh_bandwidth_search(int32_t device, int32_t d, int64_t N, int64_t n, double xi, double kappa, int32_t large_h,
                          double eps, int32_t max_iters, int32_t tol_rows, uint64_t data_seed, double* out, double* prof,
                          int32_t prof_cap, int32_t* n_prof, int32_t center_random) {
  *n_prof = 0;
  auto dump = [&](const std::vector<std::pair<double, long>>& p) {
    const int32_t k = std::min<int32_t>(prof_cap, static_cast<int32_t>(p.size()));
    for (int32_t i = 0; i < k; ++i) {
      prof[2 * i] = p[static_cast<size_t>(i)].first;
      prof[2 * i + 1] = static_cast<double>(p[static_cast<size_t>(i)].second);
    }
    *n_prof = k;
  };
  return guard([&] {
    Device dev(device);
    ExperimentConfig cfg;
    cfg.d = d;
    cfg.N = N;
    cfg.n_sources = n;
    cfg.xi = xi;
    cfg.center_mode = center_random ? CenterMode::RandomPoint : CenterMode::Origin;
    BandwidthSearchSpec spec;
    spec.kappa = kappa;
    spec.large_h_branch = large_h != 0;
    spec.eps = eps;
    spec.max_iters = max_iters;
    spec.rank_tolerance_rows = tol_rows;
    try {
      const BandwidthResult r = bandwidth_search(dev, cfg, spec, data_seed);
      out[0] = r.h_abs;
      out[1] = r.h_over_hs;
      out[2] = static_cast<double>(r.rank);
      out[3] = r.evaluations;
      out[4] = r.converged ? 1.0 : 0.0;
      dump(r.profile);
    } catch (const SearchFailureError& e) {
      dump(e.profile);
      throw;
    }
  });
}

// run_experiment through the mirror; CSV written to `path`.
int kidh_run_experiment(int32_t device, int32_t d, int64_t N, int64_t n, double xi, double h_value, int32_t scheme,
                        int64_t lev_rank, const double* s_grid, int32_t n_s, double eps, int32_t trials,
                        uint64_t seed, const char* path, int32_t methods_mask, double s_mc, int32_t n_mc) {
  return guard([&] {
    Device dev(device);
    ExperimentConfig cfg;
    cfg.d = d;
    cfg.N = N;
    cfg.n_sources = n;
    cfg.xi = xi;
    cfg.h_value = h_value;
    SamplingScheme sc;
    sc.kind = scheme == 2 ? SchemeKind::EuclideanNorm : scheme == 4 ? SchemeKind::Leverage : SchemeKind::Uniform;
    if (lev_rank > 0) sc.rank_for_leverage = lev_rank;
    cfg.schemes = {sc};
    cfg.scheme_rank_auto = {sc.kind == SchemeKind::Leverage && lev_rank <= 0};
    cfg.s_grid.assign(s_grid, s_grid + n_s);
    cfg.rank_rule = RankRule::from_eps(eps);
    cfg.trials = trials;
    cfg.seed = seed;
    cfg.center_mode = CenterMode::RandomPoint;  // BASELINE.json configs: center uniformly among the points
    cfg.methods.clear();  // bit 0: id, bit 1: svd (config "methods", in that order)
    if (methods_mask & 1) cfg.methods.push_back(CompressionMethod::ID);
    if (methods_mask & 2) cfg.methods.push_back(CompressionMethod::SVD);
    if (cfg.methods.empty()) throw ConfigError("config: methods must be nonempty");
    if (s_mc > 0.0) {
      if (!(s_mc <= 1.0)) throw ConfigError("mc_error.s_mc must lie in (0, 1]");
      if (n_mc < 1) throw ConfigError("mc_error.n_mc must be >= 1");
      cfg.s_mc = s_mc;
      cfg.n_mc = n_mc;
    }
    std::ostringstream os;
    run_experiment(dev, cfg, os, nullptr);
    FILE* f = std::fopen(path, "w");
    if (!f) throw Error(std::string("cannot open ") + path);
    std::fputs(os.str().c_str(), f);
    std::fclose(f);
  });
}

}  // extern "C"
