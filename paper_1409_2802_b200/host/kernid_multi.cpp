// kernid_multi.cpp -- the multi-GPU host layer of the mirror (north_star: "targets
// shard naturally across the 8 GPUs of one box; only the m x m Gram partials and scalar norms are
// combined, with an NCCL allreduce over NVLink").
//
// One process drives G GPUs: a kid_ctx per GPU, one host thread per GPU for every pass (the C-ABI is
// synchronous per context, contexts are independent), and an NCCL communicator over the group
// (ncclCommInitAll) for the reductions. The point set is split into contiguous index ranges, one per
// GPU:
//   split (geometry.hpp:29-65)  each GPU's n smallest (dist, idx) candidates -> host merge by the
//                               (dist, idx) comparator -> the global sources and rho -> every GPU
//                               compacts its own targets (kid_split_finish): bit-identical to the
//                               single-GPU split, targets in ascending global order;
//   row norms (sampling.hpp:193) per GPU, concatenated in GPU order (= global target order);
//   Grams (compress.hpp:141-159) per GPU into a device buffer, ncclAllReduce(sum) in place, read back
//                               from GPU 0. A group that lists one device more than once (tests on a
//                               single GPU) cannot form an NCCL communicator; it sums the partials on the
//                               host in GPU order instead.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <set>
#include <thread>

#include "kernid_b200.hpp"

namespace kernid_b200 {

namespace {
template <class F>
void for_each_device(int G, F&& fn) {  // one host thread per GPU; the first exception is rethrown
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(static_cast<size_t>(G));
  for (int g = 0; g < G; ++g)
    th.emplace_back([&, g] {
      try {
        fn(g);
      } catch (...) {
        err[static_cast<size_t>(g)] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}
}  // namespace

DeviceGroup::DeviceGroup(const std::vector<int>& devices) : ids_(devices) {
  if (devices.empty()) throw RangeError("DeviceGroup: no devices");
  for (int id : devices) devs_.push_back(std::make_unique<Device>(id));
  const std::set<int> distinct(devices.begin(), devices.end());
  if (distinct.size() == devices.size()) {
    comms_.resize(devices.size());
    if (ncclCommInitAll(comms_.data(), static_cast<int>(devices.size()), devices.data()) != ncclSuccess)
      comms_.clear();  // no NCCL (e.g. a driver without peer support): host reduction
  }
}

DeviceGroup::~DeviceGroup() {
  for (auto c : comms_) ncclCommDestroy(c);
}

std::vector<double> DeviceGroup::allreduce_to_host(const std::vector<double*>& dbufs, size_t count) {
  const int G = size();
  std::vector<double> out(count, 0.0);
  if (!comms_.empty()) {
    if (ncclGroupStart() != ncclSuccess) throw Error("ncclGroupStart failed");
    for (int g = 0; g < G; ++g)
      if (ncclAllReduce(dbufs[static_cast<size_t>(g)], dbufs[static_cast<size_t>(g)], count, ncclDouble, ncclSum,
                        comms_[static_cast<size_t>(g)], static_cast<cudaStream_t>(kid_stream(dev(g).ctx()))) !=
          ncclSuccess)
        throw Error("ncclAllReduce failed");
    if (ncclGroupEnd() != ncclSuccess) throw Error("ncclGroupEnd failed");
    dev(0).check(kid_memcpy_dtoh(dev(0).ctx(), out.data(), dbufs[0], sizeof(double) * count));
    for (int g = 1; g < G; ++g) dev(g).check(kid_synchronize(dev(g).ctx()));
    return out;
  }
  std::vector<double> part(count);
  for (int g = 0; g < G; ++g) {  // GPU order: deterministic
    dev(g).check(kid_memcpy_dtoh(dev(g).ctx(), part.data(), dbufs[static_cast<size_t>(g)], sizeof(double) * count));
    for (size_t i = 0; i < count; ++i) out[i] += part[i];
  }
  return out;
}

ShardedSplit split_sources_targets(DeviceGroup& grp, const PointSet& ps, const std::vector<double>& x_c, int64_t n,
                                   double xi) {
  const int64_t N = ps.rows;
  const int d = static_cast<int>(ps.cols);
  const int G = grp.size();
  if (n < 1 || n >= N) throw RangeError("split_sources_targets: requires 1 <= n < N");
  if (xi < 0.0) throw RangeError("split_sources_targets: requires xi >= 0");
  if (static_cast<int64_t>(x_c.size()) != ps.cols) throw DimensionError("split_sources_targets: center dimension mismatch");
  ShardedSplit sp;
  sp.offsets.resize(static_cast<size_t>(G) + 1);
  for (int g = 0; g <= G; ++g) sp.offsets[static_cast<size_t>(g)] = N * g / G;
  std::vector<std::vector<double>> cd(static_cast<size_t>(G));
  std::vector<std::vector<int64_t>> ci(static_cast<size_t>(G));
  for_each_device(G, [&](int g) {
    const int64_t lo = sp.offsets[static_cast<size_t>(g)], Ng = sp.offsets[static_cast<size_t>(g) + 1] - lo;
    std::vector<double> slice(static_cast<size_t>(Ng * d));  // this GPU's rows, column-major
    for (int k = 0; k < d; ++k)
      std::memcpy(slice.data() + static_cast<size_t>(k * Ng), ps.data() + static_cast<size_t>(k * N + lo),
                  sizeof(double) * static_cast<size_t>(Ng));
    Device& dv = grp.dev(g);
    dv.check(kid_set_points(dv.ctx(), slice.data(), Ng, d, lo));
    const int64_t k = std::min(n, Ng);
    cd[static_cast<size_t>(g)].resize(static_cast<size_t>(k));
    ci[static_cast<size_t>(g)].resize(static_cast<size_t>(k));
    dv.check(kid_split_candidates(dv.ctx(), x_c.data(), n, cd[static_cast<size_t>(g)].data(),
                                  ci[static_cast<size_t>(g)].data()));
  });
  // the global n smallest under (dist, idx) -- nth_element's comparator (geometry.hpp:39-45)
  std::vector<std::pair<double, int64_t>> all;
  for (int g = 0; g < G; ++g)
    for (size_t k = 0; k < cd[static_cast<size_t>(g)].size(); ++k)
      all.push_back({cd[static_cast<size_t>(g)][k], ci[static_cast<size_t>(g)][k]});
  std::sort(all.begin(), all.end());
  if (static_cast<int64_t>(all.size()) < n) throw Error("split_sources_targets: fewer than n candidates");
  SourceTargetSplit& s = sp.global;
  s.center = x_c;
  s.xi = xi;
  s.rho = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    s.rho = std::max(s.rho, all[static_cast<size_t>(k)].first);  // geometry.hpp:52-53
    s.source_indices.push_back(all[static_cast<size_t>(k)].second);
  }
  std::sort(s.source_indices.begin(), s.source_indices.end());  // geometry.hpp:50-51
  std::vector<double> src_pts(static_cast<size_t>(n * d));
  for (int k = 0; k < d; ++k)
    for (int64_t j = 0; j < n; ++j) src_pts[static_cast<size_t>(j + k * n)] = ps(s.source_indices[static_cast<size_t>(j)], k);
  sp.nt.assign(static_cast<size_t>(G), 0);
  std::vector<std::vector<int64_t>> tg(static_cast<size_t>(G));
  for_each_device(G, [&](int g) {
    Device& dv = grp.dev(g);
    int64_t nt = 0;
    dv.check(kid_split_finish(dv.ctx(), s.source_indices.data(), n, src_pts.data(), s.rho, xi, &nt));
    sp.nt[static_cast<size_t>(g)] = nt;
    tg[static_cast<size_t>(g)].resize(static_cast<size_t>(nt));
    dv.check(kid_get_targets(dv.ctx(), tg[static_cast<size_t>(g)].data(), nt));
  });
  for (int g = 0; g < G; ++g)
    s.target_indices.insert(s.target_indices.end(), tg[static_cast<size_t>(g)].begin(), tg[static_cast<size_t>(g)].end());
  if (s.target_indices.empty())
    throw NoTargetsError("split_sources_targets: no targets at separation xi = " + std::to_string(xi));
  return sp;
}

ShardedBlock::ShardedBlock(DeviceGroup& grp, KernelSpec spec, const PointSet& points, const ShardedSplit& split)
    : grp_(&grp), spec_(spec), points_(&points), split_(&split) {
  spec_.validate();
}

Matrix ShardedBlock::rows_exact(const std::vector<int64_t>& idx) const {  // gather_rows, compress.hpp:130-137
  const int64_t m = cols();
  const int d = static_cast<int>(points_->cols);
  const int64_t N = points_->rows;
  Matrix sub(static_cast<int64_t>(idx.size()), m);
  for (size_t i = 0; i < idx.size(); ++i) {
    if (idx[i] < 0 || idx[i] >= rows()) throw RangeError("row sample index out of range");
    const int64_t t = split_->global.target_indices[static_cast<size_t>(idx[i])];
    for (int64_t j = 0; j < m; ++j)
      sub(static_cast<int64_t>(i), j) = eval_kernel(spec_, points_->data() + t, N,
                                                    points_->data() + split_->global.source_indices[static_cast<size_t>(j)],
                                                    N, d);
  }
  return sub;
}

std::vector<double> ShardedBlock::row_norms() const {
  const int G = grp_->size();
  std::vector<std::vector<double>> w(static_cast<size_t>(G));
  for_each_device(G, [&](int g) {
    w[static_cast<size_t>(g)].resize(static_cast<size_t>(split_->nt[static_cast<size_t>(g)]));
    grp_->dev(g).check(kid_row_norms(grp_->dev(g).ctx(), spec_.h, w[static_cast<size_t>(g)].data()));
  });
  std::vector<double> out;
  for (auto& v : w) out.insert(out.end(), v.begin(), v.end());
  return out;
}

// [sum_0, sum_1, G (k x k)] of every GPU's shard, reduced across the group (NCCL)
std::vector<double> ShardedBlock::reduced_pass(int64_t k, const std::function<void(int, double*)>& pass) const {
  const int G = grp_->size();
  const size_t count = static_cast<size_t>(2 + k * k);
  std::vector<double*> bufs(static_cast<size_t>(G), nullptr);
  for (int g = 0; g < G; ++g) {
    bufs[static_cast<size_t>(g)] = static_cast<double*>(kid_device_alloc(grp_->dev(g).ctx(), sizeof(double) * count));
    if (!bufs[static_cast<size_t>(g)]) throw Error("kid_device_alloc failed");
  }
  std::vector<double> out;
  try {
    for_each_device(G, [&](int g) { pass(g, bufs[static_cast<size_t>(g)]); });
    out = grp_->allreduce_to_host(bufs, count);
  } catch (...) {
    for (int g = 0; g < G; ++g) kid_device_free(grp_->dev(g).ctx(), bufs[static_cast<size_t>(g)]);
    throw;
  }
  for (int g = 0; g < G; ++g) kid_device_free(grp_->dev(g).ctx(), bufs[static_cast<size_t>(g)]);
  return out;
}

Matrix ShardedBlock::gram(double* sumsq) const {
  const int64_t m = cols();
  const std::vector<double> red = reduced_pass(m, [&](int g, double* buf) {
    Device& dv = grp_->dev(g);
    dv.check(kid_gram_dev(dv.ctx(), spec_.h, buf, nullptr));
    dv.check(kid_synchronize(dv.ctx()));
  });
  if (sumsq) *sumsq = red[1];
  Matrix G(m, m);
  std::memcpy(G.data(), red.data() + 2, sizeof(double) * static_cast<size_t>(m * m));
  return G;
}

double ShardedBlock::spectral_norm() const { return std::sqrt(lambda_max(gram())); }

std::pair<IDFactorization, CompressionReport> compress_id(const ShardedBlock& K, const RowSample& sample,
                                                          const RankRule& rule, const CompressOptions& opts) {
  if (sample.indices.empty()) throw RangeError("compress_id: empty row sample");
  CompressionReport rep;
  rep.fraction = sample.fraction;
  rep.seed = sample.seed;
  const Matrix sub = K.rows_exact(sample.indices);
  const std::vector<double> sv = singular_values(sub);
  const int64_t r = rule.resolve(sv);
  rep.rank = r;
  rep.sigma1_sample = sv[0];
  rep.sigma_r1_sample = (r < static_cast<int64_t>(sv.size())) ? sv[static_cast<size_t>(r)] : 0.0;
  rep.bound_id = bound_id_value(K.cols(), r, rep.sigma_r1_sample);
  IDFactorization id;
  if (r == 0) {
    rep.rank_zero = true;
    rep.rel_error = 1.0;
    rep.rel_error_fro = 1.0;
    return {std::move(id), rep};
  }
  id = interpolative_decomposition(sub, r);
  const int64_t m = K.cols(), n = m - r;
  double sd = 0.0, sk = 0.0, num = 0.0;
  if (n > 0) {
    // the fused error pass on every shard: [||D||^2, ||K||^2, D^T D over the non-skeleton columns]
    const std::vector<double> red = K.reduced_pass(n, [&](int g, double* buf) {
      Device& dv = K.group().dev(g);
      dv.check(kid_recon_prepare(dv.ctx(), id.skeleton.data(), r, id.projection.data()));
      dv.check(kid_recon_error_dev(dv.ctx(), K.spec().h, KID_RECON_DTD, buf));
      dv.check(kid_synchronize(dv.ctx()));
    });
    sd = red[0];
    sk = red[1];
    Matrix G(n, n);
    std::memcpy(G.data(), red.data() + 2, sizeof(double) * static_cast<size_t>(n * n));
    num = std::sqrt(lambda_max(G));
  } else {
    K.gram(&sk);  // r = m: D == 0
  }
  const double den = opts.k_norm ? *opts.k_norm : K.spectral_norm();
  rep.rel_error = den > 0.0 ? num / den : 0.0;
  rep.rel_error_fro = sk > 0.0 ? std::sqrt(sd / sk) : 0.0;
  return {std::move(id), rep};
}

RowSample sample_rows_euclidean(const ShardedBlock& K, double s, std::uint64_t seed) {  // sampling.hpp:189-196
  RowSample out;
  out.fraction = s;
  out.seed = seed;
  Rng rng(seed);
  const std::vector<double> w = K.row_norms();
  out.indices = weighted_draw(w, sample_count(s, K.rows()), false, rng);
  return out;
}

}  // namespace kernid_b200
