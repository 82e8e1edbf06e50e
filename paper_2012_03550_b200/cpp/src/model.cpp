// model.cpp -- host model state, initialisation and the fp64 per-entry
// helpers.  Nothing here is on the training hot path: the epochs run on the
// device and only copy A^(n)/B^(n) in and out.
#include "sptucker/model.hpp"

#include <algorithm>
#include <atomic>
#include <limits>
#include <string>

namespace sptucker {

std::uint64_t ModelGeneration::next() {
  static std::atomic<std::uint64_t> counter{0};
  return ++counter;
}

void Ranks::validate(std::size_t order) const {
  if (J.size() != order) throw DomainError("ranks: J arity does not match tensor order");
  if (r_core < 1) throw DomainError("ranks: R_core must be >= 1");
  for (const std::uint32_t j : J) {
    if (j < 1) throw DomainError("ranks: every J_n must be >= 1");
    if (j < r_core) throw DomainError("ranks: R_core must satisfy R_core <= J_n");
  }
}

std::uint64_t Ranks::core_elems() const {
  std::uint64_t p = 1;
  for (const std::uint32_t j : J)
    p = p > std::numeric_limits<std::uint64_t>::max() / j ? std::numeric_limits<std::uint64_t>::max() : p * j;
  return p;
}

std::uint64_t Ranks::min_j() const { return *std::min_element(J.begin(), J.end()); }

std::vector<double> reconstruct_core(const std::vector<Matrix>& kruskal, const Ranks& ranks) {
  const std::size_t total = static_cast<std::size_t>(ranks.core_elems());
  std::vector<double> g(total, 0.0), term, grown;
  for (std::uint32_t r = 0; r < ranks.r_core; ++r) {
    term.resize(ranks.J[0]);
    for (std::uint32_t j = 0; j < ranks.J[0]; ++j) term[j] = kruskal[0].at(j, r);
    for (std::size_t n = 1; n < ranks.J.size(); ++n) {  // outer product, earlier modes fastest
      grown.resize(term.size() * ranks.J[n]);
      for (std::uint32_t j = 0; j < ranks.J[n]; ++j) {
        const double b = kruskal[n].at(j, r);
        for (std::size_t i = 0; i < term.size(); ++i) grown[j * term.size() + i] = b * term[i];
      }
      term.swap(grown);
    }
    for (std::size_t i = 0; i < total; ++i) g[i] += term[i];
  }
  return g;
}

Matrix unfold_dense(const std::vector<double>& flat, const std::vector<std::uint32_t>& dims, std::size_t mode) {
  std::uint64_t total = 1;
  for (const std::uint32_t d : dims) total *= d;
  if (flat.size() != total) throw InternalError("unfold_dense: size mismatch");
  Matrix out(dims[mode], static_cast<std::size_t>(total / dims[mode]));
  std::vector<std::uint32_t> at(dims.size(), 0);
  for (std::uint64_t lin = 0; lin < total; ++lin) {
    std::uint64_t col = 0, stride = 1;
    for (std::size_t k = 0; k < dims.size(); ++k) {
      if (k == mode) continue;
      col += at[k] * stride;
      stride *= dims[k];
    }
    out.at(at[mode], static_cast<std::size_t>(col)) = flat[lin];
    for (std::size_t k = 0; k < dims.size() && ++at[k] == dims[k]; ++k) at[k] = 0;
  }
  return out;
}

TuckerModel::TuckerModel(Shape shape, Ranks ranks) : shape_(std::move(shape)), ranks_(std::move(ranks)) {
  ranks_.validate(shape_.order());
  for (std::size_t n = 0; n < shape_.order(); ++n) {
    factors_.emplace_back(shape_.dim(n), ranks_.J[n]);
    kruskal_.emplace_back(ranks_.J[n], ranks_.r_core);
  }
}

TuckerModel TuckerModel::init_gaussian(const Shape& shape, const Ranks& ranks, double mean, double stddev,
                                       std::uint64_t seed) {
  if (!(stddev > 0.0)) throw DomainError("init_gaussian: stddev must be positive");
  TuckerModel m(shape, ranks);
  Rng rng(seed);
  for (Matrix& b : m.kruskal_)
    for (double& v : b.data()) v = rng.next_gaussian(mean, stddev);
  for (Matrix& a : m.factors_)
    for (double& v : a.data()) v = rng.next_gaussian(mean, stddev);
  return m;
}

void TuckerModel::refresh_core_cache() {
  core_fresh_ = false;
  gen_.bump();  // callers refresh after editing B through a held reference
}

void TuckerModel::build_core_cache() const {
  if (core_fresh_) return;
  if (ranks_.core_elems() > kMaxCoreElems)
    throw DomainError("model: dense core has " + std::to_string(ranks_.core_elems()) + " elements, cap is " +
                      std::to_string(kMaxCoreElems) + " (the device path never needs it)");
  core_dense_ = reconstruct_core(kruskal_, ranks_);
  core_unfold_.clear();
  for (std::size_t n = 0; n < order(); ++n) core_unfold_.push_back(unfold_dense(core_dense_, ranks_.J, n));
  core_fresh_ = true;
}

const std::vector<double>& TuckerModel::core_dense() const {
  build_core_cache();
  return core_dense_;
}

const Matrix& TuckerModel::core_unfolding(std::size_t n) const {
  build_core_cache();
  return core_unfold_[n];
}

void TuckerModel::kron_row_excluding(std::span<const std::uint32_t> coord, std::size_t mode,
                                     std::vector<double>& s) const {
  s.assign(1, 1.0);
  for (std::size_t k = 0; k < order(); ++k) {
    if (k == mode) continue;
    const double* a = factors_[k].row(coord[k] - 1);
    const std::size_t len = s.size(), jk = ranks_.J[k];
    s.resize(len * jk);
    for (std::size_t j = jk; j-- > 0;)  // highest block first so block 0 is read before it is overwritten
      for (std::size_t i = 0; i < len; ++i) s[j * len + i] = s[i] * a[j];
  }
}

void TuckerModel::e_column(std::span<const std::uint32_t> coord, std::size_t mode, std::vector<double>& s_scratch,
                           std::vector<double>& e) const {
  kron_row_excluding(coord, mode, s_scratch);
  const Matrix& g = core_unfolding(mode);
  e.resize(g.rows());
  for (std::size_t j = 0; j < g.rows(); ++j) e[j] = dot(g.row(j), s_scratch.data(), g.cols());
}

double TuckerModel::predict(std::span<const std::uint32_t> coord, std::vector<double>&, std::vector<double>&) const {
  return predict(coord);
}

// Kruskal route: xhat = sum_r prod_k a^(k)_{i_k} . b^(k)_{:,r} (no dense core).
double TuckerModel::predict(std::span<const std::uint32_t> coord) const {
  double x = 0.0;
  for (std::uint32_t r = 0; r < ranks_.r_core; ++r) {
    double c = 1.0;
    for (std::size_t k = 0; k < order(); ++k)
      c *= dot_strided(factors_[k].row(coord[k] - 1), kruskal_[k].data().data() + r, ranks_.r_core,
                       ranks_.J[k]);
    x += c;
  }
  return x;
}

bool TuckerModel::all_finite() const {
  for (const Matrix& a : factors_)
    if (!a.all_finite()) return false;
  for (const Matrix& b : kruskal_)
    if (!b.all_finite()) return false;
  return true;
}

}  // namespace sptucker
