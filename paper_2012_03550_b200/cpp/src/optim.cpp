// optim.cpp -- core and factor phases: the device-backed epoch calls plus the
// host fp64 per-entry helpers of the reference API.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <string>

#include "device.hpp"
#include "sptucker/core_optimizer.hpp"
#include "sptucker/factor_optimizer.hpp"

namespace sptucker {

std::size_t CoreBatchWorkspace::bytes() const {
  return batch.capacity() * sizeof(std::uint32_t) + sample_pool.capacity() * sizeof(std::uint32_t);
}

std::size_t RowBatchWorkspace::bytes() const {
  std::size_t b = 0;
  for (const std::vector<double>* v : {&s, &e, &fact1, &fact2, &grad, &gram}) b += v->capacity() * sizeof(double);
  return b;
}

// ---------------------------------------------------------------- host helpers
namespace {
// c_r = prod_{k != mode} a^(k)_{i_k} . b^(k)_{:,r}
double kruskal_coeff(const TuckerModel& m, std::span<const std::uint32_t> coord, std::size_t mode, std::size_t r) {
  double c = 1.0;
  for (std::size_t k = 0; k < m.order(); ++k) {
    if (k == mode) continue;
    const Matrix& b = m.kruskal(k);
    c *= dot_strided(m.factor(k).row(coord[k] - 1), b.data().data() + r, b.cols(), b.rows());
  }
  return c;
}

// e = B^(mode) c  (== Ghat^(mode) kron_{k != mode} a^(k)_{i_k} for a Kruskal core)
void e_kruskal(const TuckerModel& m, std::span<const std::uint32_t> coord, std::size_t mode, std::vector<double>& e) {
  const Matrix& b = m.kruskal(mode);
  e.assign(b.rows(), 0.0);
  for (std::size_t r = 0; r < b.cols(); ++r) {
    const double c = kruskal_coeff(m, coord, mode, r);
    for (std::size_t j = 0; j < b.rows(); ++j) e[j] += b.at(j, r) * c;
  }
}
}  // namespace

void compute_w_row(const TuckerModel& model, std::span<const std::uint32_t> coord, std::size_t mode, std::size_t r,
                   std::span<double> w_out) {
  const double c = kruskal_coeff(model, coord, mode, r);
  const double* a = model.factor(mode).row(coord[mode] - 1);
  for (std::size_t j = 0; j < w_out.size(); ++j) w_out[j] = c * a[j];
}

void core_residual(const TuckerModel& model, const CooTensor& t, std::span<const std::uint32_t> batch,
                   std::size_t mode, std::size_t r_exclude, std::vector<double>& out) {
  const std::size_t jn = model.ranks().J[mode], rc = model.ranks().r_core;
  const Matrix& b = model.kruskal(mode);
  std::vector<double> w(jn);
  out.resize(batch.size());
  for (std::size_t s = 0; s < batch.size(); ++s) {
    double x = t.value(batch[s]);
    for (std::size_t r = 0; r < rc; ++r) {
      if (r == r_exclude) continue;
      compute_w_row(model, t.coord(batch[s]), mode, r, w);
      x -= dot_strided(w.data(), b.data().data() + r, rc, jn);
    }
    out[s] = x;
  }
}

void grad_b(const TuckerModel& model, const CooTensor& t, std::span<const std::uint32_t> batch, std::size_t mode,
            std::size_t r, std::vector<double>& v_out, std::vector<double>* c_out) {
  const std::size_t jn = model.ranks().J[mode];
  std::vector<double> resid, w(jn), C(jn * jn, 0.0), U(jn, 0.0);
  core_residual(model, t, batch, mode, r, resid);
  for (std::size_t s = 0; s < batch.size(); ++s) {
    compute_w_row(model, t.coord(batch[s]), mode, r, w);
    for (std::size_t i = 0; i < jn; ++i) {
      U[i] += w[i] * resid[s];
      for (std::size_t j = 0; j < jn; ++j) C[i * jn + j] += w[i] * w[j];
    }
  }
  const Matrix& b = model.kruskal(mode);
  v_out.assign(jn, 0.0);
  for (std::size_t i = 0; i < jn; ++i) {
    double cb = 0.0;
    for (std::size_t j = 0; j < jn; ++j) cb += C[i * jn + j] * b.at(j, r);
    v_out[i] = cb - U[i];
  }
  if (c_out) *c_out = std::move(C);
}

void sgd_step(std::size_t m, double lambda, double gamma, std::span<double> w, std::span<const double> v) {
  if (m < 1) throw DomainError("sgd_step: batch size must be >= 1");
  if (!(gamma > 0.0)) throw DomainError("sgd_step: learning rate must be positive");
  if (lambda < 0.0) throw DomainError("sgd_step: regularization must be non-negative");
  if (w.size() != v.size()) throw InternalError("sgd_step: size mismatch");
  const double inv_m = 1.0 / static_cast<double>(m);
  for (std::size_t i = 0; i < w.size(); ++i) {
    if (!std::isfinite(w[i]) || !std::isfinite(v[i]))
      throw NumericError("sgd_step: non-finite parameter or gradient; reduce the learning rate");
    w[i] -= gamma * (v[i] * inv_m + lambda * w[i]);
    if (!std::isfinite(w[i])) throw NumericError("sgd_step: update overflowed; reduce the learning rate");
  }
}

std::vector<std::uint32_t> row_batch(const CooTensor& t, std::size_t mode, std::uint32_t i_n, double fraction,
                                     Rng& rng) {
  if (!(fraction > 0.0 && fraction <= 1.0)) throw DomainError("row_batch: fraction must lie in (0,1]");
  const auto b = t.bucket(mode, i_n);
  std::vector<std::uint32_t> out(b.begin(), b.end());
  if (fraction >= 1.0 || out.empty()) return out;
  const std::size_t keep =
      std::max<std::size_t>(1, static_cast<std::size_t>(std::llround(fraction * static_cast<double>(out.size()))));
  for (std::size_t i = 0; i < keep; ++i)
    std::swap(out[i], out[i + static_cast<std::size_t>(rng.next_below(out.size() - i))]);
  out.resize(keep);
  return out;
}

void grad_a_row(const TuckerModel& model, const CooTensor& t, std::size_t mode, std::uint32_t i_n,
                std::span<const std::uint32_t> batch, RowBatchWorkspace& ws, std::span<double> f_out) {
  const std::size_t jn = model.ranks().J[mode];
  ws.grow(ws.fact1, jn);
  ws.grow(ws.fact2, jn);
  std::fill(ws.fact1.begin(), ws.fact1.end(), 0.0);
  std::fill(ws.fact2.begin(), ws.fact2.end(), 0.0);
  const double* a = model.factor(mode).row(i_n - 1);
  for (const std::uint32_t entry : batch) {
    e_kruskal(model, t.coord(entry), mode, ws.e);
    const double p = dot(a, ws.e.data(), jn), x = t.value(entry);
    for (std::size_t j = 0; j < jn; ++j) {
      ws.fact1[j] -= x * ws.e[j];
      ws.fact2[j] += p * ws.e[j];
    }
  }
  for (std::size_t j = 0; j < jn; ++j) f_out[j] = ws.fact1[j] + ws.fact2[j];
}

void grad_a_row_gram(const TuckerModel& model, const CooTensor& t, std::size_t mode, std::uint32_t i_n,
                     std::span<const std::uint32_t> batch, RowBatchWorkspace& ws, std::span<double> f_out) {
  const std::size_t jn = model.ranks().J[mode];
  ws.grow(ws.fact1, jn);
  ws.grow(ws.gram, jn * jn);
  std::fill(ws.fact1.begin(), ws.fact1.end(), 0.0);
  std::fill(ws.gram.begin(), ws.gram.end(), 0.0);
  for (const std::uint32_t entry : batch) {
    e_kruskal(model, t.coord(entry), mode, ws.e);
    const double x = t.value(entry);
    for (std::size_t i = 0; i < jn; ++i) {
      ws.fact1[i] -= x * ws.e[i];
      for (std::size_t j = 0; j < jn; ++j) ws.gram[i * jn + j] += ws.e[i] * ws.e[j];
    }
  }
  const double* a = model.factor(mode).row(i_n - 1);
  for (std::size_t j = 0; j < jn; ++j) {
    double s = 0.0;
    for (std::size_t i = 0; i < jn; ++i) s += a[i] * ws.gram[i * jn + j];
    f_out[j] = ws.fact1[j] + s;
  }
}

// ---------------------------------------------------------------- device epochs
namespace {
// SGDT_TRACE_HOST=1: per-call host timing of the per-epoch entry points on
// stderr (diagnostics of the drop-in's host overhead; off by default).
struct HostTrace {
  bool on = [] {
    const char* e = std::getenv("SGDT_TRACE_HOST");
    return e && std::atoi(e) != 0;
  }();
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[sgdt-host] %s %.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};
}  // namespace

CoreEpochStats update_core_epoch(TuckerModel& model, const CooTensor& train, const CoreHyper& hyper,
                                 const SchedContext& sched, Rng& rng, CoreBatchWorkspace& ws) {
  if (hyper.lr < 0.0) throw DomainError("core learning rate must be non-negative");
  if (hyper.lr == 0.0) return {0, 0};
  const std::size_t nnz = train.nnz();
  const std::size_t m = hyper.batch_m == 0 ? nnz : hyper.batch_m;
  if (m > nnz) throw DomainError("core batch size exceeds training nnz");

  // device-resident across calls: the model goes up only when the host copy
  // changed since this session last synchronised it, the pool only when the
  // host vector is another buffer (device.hpp); several sampler runs per call
  // (resample_per_mode) upload the host pool every time
  HostTrace tr;
  detail::Session& s = detail::session_for(train, nullptr, model.shape(), model.ranks());
  const bool sampled = hyper.batch_m != 0;
  if (sampled && ws.sample_pool.size() != nnz) {  // sample_batch: a pool of the wrong size restarts from iota
    ws.grow(ws.sample_pool, nnz);
    std::iota(ws.sample_pool.begin(), ws.sample_pool.end(), 0u);
    s.pool_reset(ws.sample_pool);
  } else if (sampled) {
    s.sync_pool(ws.sample_pool, hyper.resample_per_mode);
  }
  const sgdt_core_hyper h{hyper.lr, hyper.reg, hyper.batch_m, hyper.resample_per_mode ? 1 : 0,
                          hyper.incremental_residual ? 1 : 0};
  ws.grow(ws.batch, m);
  for (int attempt = 0;; ++attempt) {
    s.sync_model(model);
    s.put_rng(rng);
    sgdt_core_stats st{};
    tr.mark("core: sync model/rng/pool");
    detail::check(sgdt_core_epoch(s.get(), &h, &st), "update_core_epoch");
    tr.mark("core: device epoch");
    if (!sampled) {
      std::iota(ws.batch.begin(), ws.batch.end(), 0u);
      break;
    }
    std::uint64_t len = 0;
    detail::check(sgdt_last_batch(s.get(), ws.batch.data(), &len), "update_core_epoch");
    s.d2h_bytes += m * sizeof(std::uint32_t);
    tr.mark("core: batch copy-out");
    const bool same = s.pool_apply_checked(ws.sample_pool, ws.batch);
    tr.mark("core: pool delta + host replay check");
    if (same) break;
    // the host pool was edited at a position this run read: the device ran
    // on a stale pool, so repeat the epoch from the host state (model, RNG
    // and pool are all still the pre-call ones)
    if (attempt) throw InternalError("update_core_epoch: device pool does not follow the host pool");
    s.sync_pool(ws.sample_pool, /*force=*/true);
    s.put_model(model);
  }
  s.take_model(model, /*factors=*/false, /*kruskal=*/true);  // the core phase wrote B only
  s.take_rng(rng);
  tr.mark("core: B + rng copy-out");
  std::size_t effective = 0;
  for (const Range& r : partition_even(m, sched.workers()))
    if (!r.empty()) ++effective;
  return {m, effective};
}

FactorEpochStats update_factor_epoch(TuckerModel& model, const CooTensor& train, const FactorHyper& hyper,
                                     const SchedContext& sched, Rng& rng, std::vector<RowBatchWorkspace>& per_worker) {
  if (!(hyper.row_fraction > 0.0 && hyper.row_fraction <= 1.0)) throw DomainError("row fraction must lie in (0,1]");
  if (hyper.lr < 0.0) throw DomainError("factor learning rate must be non-negative");
  if (hyper.lr == 0.0) return {};
  const std::size_t workers = sched.workers();
  if (per_worker.size() < workers) per_worker.resize(workers);
  std::uint32_t jmax = 0;
  for (const std::uint32_t j : model.ranks().J) jmax = std::max(jmax, j);
  for (RowBatchWorkspace& w : per_worker)
    for (std::vector<double>* v : {&w.e, &w.fact1, &w.fact2, &w.grad}) w.grow(*v, jmax);

  HostTrace tr;
  detail::Session& s = detail::session_for(train, nullptr, model.shape(), model.ranks());
  s.sync_model(model);
  s.put_rng(rng);
  tr.mark("factor: sync model/rng");
  const sgdt_factor_hyper h{hyper.lr, hyper.reg, hyper.row_fraction};
  const sgdt_factor_stats st = s.factor_epoch_into(model, h);  // A^(n) copied out per mode, overlapped
  s.take_rng(rng);
  tr.mark("factor: device epoch + A copy-out");

  FactorEpochStats out;
  out.rows_updated = st.rows_updated;
  out.rows_skipped = st.rows_skipped;
  if (sched.strategy == Strategy::Improved && workers > 1) {  // the reference's slice imbalance
    const std::size_t nnz = train.nnz();
    std::size_t mx = 0;
    for (const Range& r : partition_even(nnz, workers)) mx = std::max(mx, r.size());
    out.max_imbalance = static_cast<double>(mx) / (static_cast<double>(nnz) / static_cast<double>(workers)) - 1.0;
  }
  return out;
}

}  // namespace sptucker
