// kernid_b200.hpp -- host C++ mirror of the reference `kernid::` API for the far-field hot
// path, running the O(N_T * m) work on the B200 through the C-ABI of kernid_cuda.h.
//
// Same names, argument meaning and error behaviour as /root/reference/proj/include/kernid/
// (namespace kernid_b200 instead of kernid). What changes:
//   * the dense Eigen::MatrixXd K of kernel_matrix() (kernel.hpp:202-208) is replaced by a
//     KernelBlock: the device-resident K(T, S) of the last split, never materialised;
//   * sample_rows / row_leverage_scores / compress_id take that block (SampleContext::K);
//   * spectral norms come from the residual Gram D^T D accumulated on the device (one pass,
//     exact up to rounding) instead of QR+SVD of a materialised difference or power
//     iteration (compress.hpp:141-159) -- NormPolicy is accepted for API parity;
//   * the tiny host steps stay on the host as in the reference: K_s rows evaluated with the
//     reference arithmetic (glibc exp, no FMA) so the ID skeleton is bit-identical, CPQR/ID,
//     epsilon-rank, weighted draws.
#pragma once
#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <ostream>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "kernid_cuda.h"

namespace kernid_b200 {

// ------------------------------------------------------------- errors.hpp:11-77
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DimensionError : public Error { public: using Error::Error; };
class NoTargetsError : public Error { public: using Error::Error; };
class RangeError : public Error { public: using Error::Error; };
class IllConditionedSkeletonError : public Error { public: using Error::Error; };
class ConfigError : public Error { public: using Error::Error; };
class NumericalError : public Error { public: using Error::Error; };
class SearchFailureError : public Error {  // errors.hpp:71-77
 public:
  SearchFailureError(const std::string& msg, std::vector<std::pair<double, long>> p) : Error(msg), profile(std::move(p)) {}
  std::vector<std::pair<double, long>> profile;
};
[[noreturn]] void throw_status(int code, const std::string& msg);

// ------------------------------------------------------------- rng.hpp:19-78
std::uint64_t splitmix64(std::uint64_t& state);
std::uint64_t derive_seed(std::uint64_t master, std::uint64_t key_a, std::uint64_t key_b = 0);
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : engine_(seed) {}
  std::uint64_t next_u64() { return engine_(); }
  double uniform01() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
  std::uint64_t below(std::uint64_t n);
  double normal();

 private:
  std::mt19937_64 engine_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

// ------------------------------------------------------------- dense host matrix
// Column-major like Eigen::MatrixXd (only what the host steps need).
struct Matrix {
  int64_t rows = 0, cols = 0;
  std::vector<double> a;
  Matrix() = default;
  Matrix(int64_t r, int64_t c, double v = 0.0) : rows(r), cols(c), a(static_cast<size_t>(r * c), v) {}
  double& operator()(int64_t i, int64_t j) { return a[static_cast<size_t>(i + j * rows)]; }
  double operator()(int64_t i, int64_t j) const { return a[static_cast<size_t>(i + j * rows)]; }
  double* data() { return a.data(); }
  const double* data() const { return a.data(); }
};

// ------------------------------------------------------------- kernel.hpp / datagen.hpp
using PointSet = Matrix;  // N x d, one point per row (kernel.hpp:14)
struct KernelSpec {       // Gaussian family only on this path (kernel.hpp:23-52)
  double h = 1.0;
  static KernelSpec gaussian(double h) { return {h}; }
  void validate() const;
};
PointSet gen_normal(int d, int64_t N, std::uint64_t seed);  // datagen.hpp:35-43
double silverman_bandwidth(int d, long long N);             // kernel.hpp:119-123
double eval_kernel(const KernelSpec& spec, const double* x, int64_t sx, const double* y, int64_t sy, int d);

// ------------------------------------------------------------- device
class Device {
 public:
  explicit Device(int device = 0);
  ~Device();
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  kid_ctx* ctx() const { return ctx_; }
  void check(int status) const;  // throws the mirrored exception

 private:
  kid_ctx* ctx_ = nullptr;
};

// ------------------------------------------------------------- geometry.hpp:21-65
struct SourceTargetSplit {
  std::vector<double> center;
  std::vector<int64_t> source_indices;
  std::vector<int64_t> target_indices;
  double rho = 0.0;
  double xi = 0.0;
};
// Uploads `ps` and runs pass 1 on the device; the block K(T, S) stays resident on `dev`.
SourceTargetSplit split_sources_targets(Device& dev, const PointSet& ps, const std::vector<double>& x_c,
                                        int64_t n, double xi);

struct RightFactor {  // lowrank.hpp:43-46
  std::vector<double> singular_values;  // min(rows, cols), nonincreasing
  Matrix V;                             // cols x cols: the reference's thin V, completed to a basis
};
// The device-resident K(T, S) of the last split (replaces the dense MatrixXd K).
class KernelBlock {
 public:
  KernelBlock(Device& dev, KernelSpec spec, const PointSet& points, const SourceTargetSplit& split);
  int64_t rows() const { return static_cast<int64_t>(split_->target_indices.size()); }
  int64_t cols() const { return static_cast<int64_t>(split_->source_indices.size()); }
  const KernelSpec& spec() const { return spec_; }
  Device& device() const { return *dev_; }
  // rows of K with the reference arithmetic (gather_rows, compress.hpp:130-137)
  Matrix rows_exact(const std::vector<int64_t>& idx) const;
  std::vector<double> row_norms() const;        // sampling.hpp:193 (device)
  Matrix gram(double* sumsq = nullptr) const;   // K^T K (device)
  double spectral_norm() const;                 // ||K||_2 = sqrt(lambda_max(K^T K))
  // right_factor(K) / singular_values(K) of the full block (lowrank.hpp:70-90). m <= 128: Householder TSQR
  // on the device (kid_tsqr_r) + a Jacobi SVD of the m x m factor -- every sigma to ~u sigma_1. m > 128
  // (the factor does not fit one SM): the Gram route (eig(K^T K), sigma resolved to ~sqrt(u) sigma_1) followed,
  // when the caller needs more, by one preconditioned second pass (kid_proj_gram on K V diag(1/sigma)) that
  // carries every sigma to ~1e-14 sigma_1. `resolve` = the relative level sigma / sigma_1 down to which the
  // caller needs the spectrum (an eps of epsilon_rank; 0 = all of it): at or above 1e-7 the Gram pass suffices.
  RightFactor right_factor(double resolve = 0.0) const;
  std::vector<double> singular_values(double resolve = 0.0) const;

 private:
  Device* dev_;
  KernelSpec spec_;
  const PointSet* points_;
  const SourceTargetSplit* split_;
};

// ------------------------------------------------------------- lowrank.hpp (host, small)
struct IDFactorization {
  std::vector<int64_t> skeleton;
  Matrix projection;  // r x n, original column order
  int64_t rank = 0;
};
struct LeverageScores {
  std::vector<double> scores;
  bool degenerate_gap = false;
};
RightFactor right_factor(const Matrix& A);                                  // lowrank.hpp:81-90
std::vector<double> singular_values(const Matrix& A);                       // lowrank.hpp:70-77
int64_t epsilon_rank(const std::vector<double>& sv, double eps,
                     std::optional<double> reference_sigma1 = std::nullopt);  // :117-126
IDFactorization interpolative_decomposition(const Matrix& A, int64_t r);     // :235-262
void sym_eig(const Matrix& A, std::vector<double>& evals, Matrix* evecs);   // Gram route (Jacobi)
std::vector<double> sym_eigvals(const Matrix& A);                           // tridiagonal + QL, values only
double lambda_max(const Matrix& G);  // largest eigenvalue of a symmetric PSD matrix (Jacobi / Lanczos)
LeverageScores row_leverage_scores(const KernelBlock& K, int64_t r);        // :296-308 (device)

// ------------------------------------------------------------- sampling.hpp
enum class SchemeKind { Uniform, Bernoulli, EuclideanNorm, Distance, Leverage, NearestNeighbor };
struct SamplingScheme {
  SchemeKind kind = SchemeKind::Uniform;
  bool replacement = false;
  int64_t rank_for_leverage = 1;
  bool distance_direct = false;
  std::string name() const;
};
struct RowSample {
  std::vector<int64_t> indices;
  double fraction = 0.0;
  std::uint64_t seed = 0;
};
struct SampleContext {
  int64_t m = 0;
  const KernelBlock* K = nullptr;
  const SourceTargetSplit* split = nullptr;
  const PointSet* points = nullptr;
};
int64_t sample_count(double s, int64_t m);
std::vector<int64_t> weighted_draw(const std::vector<double>& weights, int64_t count, bool replacement, Rng& rng);
RowSample sample_rows(const SamplingScheme& scheme, const SampleContext& ctx, double s, std::uint64_t seed);

// ------------------------------------------------------------- compress.hpp
struct RankRule {
  std::optional<double> eps;
  std::optional<int64_t> fixed_r;
  std::optional<double> reference_sigma1;
  static RankRule from_eps(double e) { return {e, std::nullopt, std::nullopt}; }
  static RankRule from_fixed(int64_t r) { return {std::nullopt, r, std::nullopt}; }
  int64_t resolve(const std::vector<double>& sv) const;
};
struct NormPolicy {
  double memory_budget_values = 2e8;
  double power_tol = 1e-6;
  int power_cap = 1000;
};
struct StageTimings {
  double sample_ms = 0.0, factor_ms = 0.0, error_ms = 0.0;
};
struct CompressionReport {
  SamplingScheme scheme;
  double fraction = 0.0;
  int64_t rank = 0;
  double rel_error = 0.0;       // ||C P - K||_2 / ||K||_2 (the reference metric)
  double rel_error_fro = 0.0;   // ||C P - K||_F / ||K||_F (north-star literal)
  std::optional<double> bound_id;
  std::optional<double> bound_sampling;
  std::uint64_t seed = 0;
  StageTimings timings;
  bool rank_zero = false;
  double sigma_r1_sample = 0.0;
  double sigma1_sample = 0.0;
};
struct CompressOptions {
  NormPolicy norms;
  std::optional<std::vector<double>> full_spectrum;
  std::optional<double> k_norm;
  double theorem_eps = 0.5;
};
double bound_id_value(int64_t n, int64_t r, double sigma_r1);
double reconstruction_bound(int64_t m, int64_t s_count, double eps, double sigma_r1);
std::pair<IDFactorization, CompressionReport> compress_id(const KernelBlock& K, const RowSample& sample,
                                                          const RankRule& rule, const CompressOptions& opts = {});

// compress.hpp:219-273: right singular basis V_r of the sample; rel_error = ||K - K V_r V_r^T||_2 / ||K||_2
// with the error pass on the device (kid_proj_gram over V_perp; the difference is never formed).
std::pair<Matrix, CompressionReport> compress_svd(const KernelBlock& K, const RowSample& sample, const RankRule& rule,
                                                  const CompressOptions& opts = {});
// compress.hpp:279-305 for the ID reconstruction (khat_row(i) = K[i, skel] P), on the device:
// each repetition draws Bernoulli(s_mc) rows with the reference seeds, restricts the block to
// them (kid_select_rows) and takes both spectral norms through the Gram route.
std::vector<double> mc_error(const KernelBlock& K, const IDFactorization& id, double s_mc, int n_mc,
                             std::uint64_t seed);
// compress.hpp:309-325 on the device: u_i = sum_j Ker(y_i, x_skel_j) (P q)_j over the block's targets.
std::vector<double> apply_skeleton(const KernelBlock& K, const IDFactorization& id, const std::vector<double>& q);

// compress.hpp:279-305 for the SVD reconstruction (khat_row(i) = V_r V_r^T K_i): num from the
// projected Gram of the row subset onto V_perp (the complement of V_r), den from its K^T K.
std::vector<double> mc_error_svd(const KernelBlock& K, const Matrix& Vr, double s_mc, int n_mc, std::uint64_t seed);
// An orthonormal basis (m x (m - r)) of the complement of the orthonormal columns of Vr (Householder).
Matrix complement_basis(const Matrix& Vr);

// ------------------------------------------------------------- harness.hpp (compress sweep)
enum class CompressionMethod { ID, SVD };  // compress.hpp:57-60
enum class CenterMode { Origin, RandomPoint };  // config.hpp:69 (the reference default is Origin)
struct ExperimentConfig {
  int d = 2;
  int64_t N = 100000;
  int64_t n_sources = 100;
  double xi = 2.0;
  double h_value = 1.0;
  bool h_in_silverman_units = true;
  std::vector<SamplingScheme> schemes{SamplingScheme{}};
  std::vector<bool> scheme_rank_auto{false};
  std::vector<double> s_grid{1e-4, 1e-3, 1e-2, 1e-1, 1.0};
  RankRule rank_rule = RankRule::from_eps(1e-2);
  bool rank_reference_full = false;
  bool emit_bound_sampling = false;
  bool emit_timings = false;
  double theorem_eps = 0.5;
  int trials = 1;
  std::uint64_t seed = 1;
  CenterMode center_mode = CenterMode::Origin;                    // config.hpp:69
  std::vector<CompressionMethod> methods{CompressionMethod::ID};  // config.hpp:79
  std::optional<double> s_mc;                                     // config.hpp:85-86 (mc_error)
  int n_mc = 1;
};
// harness.hpp:143-328 for the Normal dataset / RandomPoint center / ID method.
void run_experiment(Device& dev, const ExperimentConfig& cfg, std::ostream& out, std::ostream* log = nullptr);
// resolve_center (harness.hpp:85-101): the origin, or row below(N) of the 0xCE stream
std::vector<double> resolve_center(const ExperimentConfig& cfg, const PointSet& points, std::uint64_t data_seed);

// compress.hpp:327-378: spectral-norm fractions of the source-source, neighbour-source and
// far-field blocks of the N x n matrix of all points against the n points closest to x_c.
// The blocks are evaluated on the device (kid_set_block + kid_gram); ||.||_2 = sqrt(lambda_max)
// of the block Grams, ||K||_2 of the stack from their sum.
struct InteractionFractions {
  double self_frac = 0.0, nn_frac = 0.0, far_frac = 0.0;
};
InteractionFractions interaction_fractions(Device& dev, const PointSet& ps, const KernelSpec& spec,
                                           const std::vector<double>& x_c, int64_t n);

// harness.hpp:330-438: bisection over the Gaussian bandwidth for the h at which the eps-rank of
// K meets kappa * n; each evaluation is the device TSQR spectrum (KernelBlock::singular_values).
struct BandwidthSearchSpec {  // config.hpp:56-63
  double kappa = 0.2;
  bool large_h_branch = false;
  double eps = 1e-2;
  int max_iters = 40;
  int rank_tolerance_rows = 2;
  int seeds = 5;
};
struct BandwidthResult {
  double h_abs = 0.0, h_over_hs = 0.0;
  long rank = 0;
  int evaluations = 0;
  bool converged = false;
  std::vector<std::pair<double, long>> profile;
};
BandwidthResult bandwidth_search(Device& dev, const ExperimentConfig& cfg, const BandwidthSearchSpec& spec,
                                 std::uint64_t data_seed);
std::string format_double(double v);


// ------------------------------------------------------------- multi-GPU (kernid_multi.cpp)
// One process, G GPUs: a context per GPU, a host thread per GPU for each pass, NCCL for the Gram
// reductions (ncclCommInitAll; a group listing a device twice -- single-GPU tests -- sums on the host).
class DeviceGroup {
 public:
  explicit DeviceGroup(const std::vector<int>& devices);
  ~DeviceGroup();
  DeviceGroup(const DeviceGroup&) = delete;
  DeviceGroup& operator=(const DeviceGroup&) = delete;
  int size() const { return static_cast<int>(devs_.size()); }
  Device& dev(int g) const { return *devs_[static_cast<size_t>(g)]; }
  bool uses_nccl() const { return !comms_.empty(); }
  // sum of the per-GPU device buffers (count doubles each), read back to the host
  std::vector<double> allreduce_to_host(const std::vector<double*>& dbufs, size_t count);

 private:
  std::vector<int> ids_;
  std::vector<std::unique_ptr<Device>> devs_;
  std::vector<struct ncclComm*> comms_;
};

struct ShardedSplit {
  SourceTargetSplit global;      // identical to the single-GPU split
  std::vector<int64_t> offsets;  // G + 1 point-index boundaries of the shards
  std::vector<int64_t> nt;       // targets per shard (concatenated in GPU order = global order)
};
ShardedSplit split_sources_targets(DeviceGroup& grp, const PointSet& ps, const std::vector<double>& x_c, int64_t n,
                                   double xi);

// K(T, S) with the targets sharded over the group (the multi-GPU KernelBlock)
class ShardedBlock {
 public:
  ShardedBlock(DeviceGroup& grp, KernelSpec spec, const PointSet& points, const ShardedSplit& split);
  int64_t rows() const { return static_cast<int64_t>(split_->global.target_indices.size()); }
  int64_t cols() const { return static_cast<int64_t>(split_->global.source_indices.size()); }
  const KernelSpec& spec() const { return spec_; }
  DeviceGroup& group() const { return *grp_; }
  Matrix rows_exact(const std::vector<int64_t>& idx) const;
  std::vector<double> row_norms() const;       // global target order
  Matrix gram(double* sumsq = nullptr) const;  // K^T K, NCCL-reduced
  double spectral_norm() const;
  // [sum_0, sum_1, G (k x k)] of `pass` (writing 2 + k^2 doubles into a device buffer) over all shards
  std::vector<double> reduced_pass(int64_t k, const std::function<void(int, double*)>& pass) const;

 private:
  DeviceGroup* grp_;
  KernelSpec spec_;
  const PointSet* points_;
  const ShardedSplit* split_;
};
RowSample sample_rows_euclidean(const ShardedBlock& K, double s, std::uint64_t seed);
std::pair<IDFactorization, CompressionReport> compress_id(const ShardedBlock& K, const RowSample& sample,
                                                          const RankRule& rule, const CompressOptions& opts = {});

}  // namespace kernid_b200
