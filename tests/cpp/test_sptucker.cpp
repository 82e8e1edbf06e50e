// test_sptucker.cpp -- parity tests of the C++ host API (namespace sptucker,
// running on the B200 through include/sgdt.h) against the plain-C oracle
// (oracle/sgdt_oracle.c, pinned bit-for-bit to the reference by
// tests/test_oracle_pin.py).  Written in the shape of the reference's own
// suites (proj/tests/test_{sptensor,core_optimizer,factor_optimizer,eval,
// trainer}.cpp); run by tests/test_cpp_api.py with -m gpu.
//
// Bars: sampling bit-exact; per-epoch parameters rel_err <= 1e-4 with
// rel_err = |g - ref| / max(1, |ref|) (oracle.cpp:409-411); RMSE within 1e-3.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <functional>
#include <numeric>
#include <set>
#include <string>
#include <vector>

#include "sgdt_oracle.h"
#include "sptucker/core_optimizer.hpp"
#include "sptucker/eval.hpp"
#include "sptucker/factor_optimizer.hpp"
#include "sptucker/synth.hpp"
#include "sptucker/trainer.hpp"

#include <unistd.h>

using namespace sptucker;

namespace {

int g_fail = 0, g_checks = 0;
std::string g_case;

#define CHECK(cond)                                                                     \
  do {                                                                                  \
    ++g_checks;                                                                         \
    if (!(cond)) {                                                                      \
      ++g_fail;                                                                         \
      std::fprintf(stderr, "FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond); \
    }                                                                                   \
  } while (0)

template <class E, class F>
bool throws_as(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

double rel_err(double g, double ref) { return std::abs(g - ref) / std::max(1.0, std::abs(ref)); }

struct Data {
  std::vector<std::uint32_t> dims;
  std::vector<std::uint32_t> coords;
  std::vector<double> values;
};

Data planted(std::vector<std::uint32_t> dims, std::vector<std::uint32_t> tJ, std::uint32_t tR, std::size_t nnz,
             double noise, double tmean, double tsd, std::uint64_t seed) {
  Data d{dims, std::vector<std::uint32_t>(nnz * dims.size()), std::vector<double>(nnz)};
  const int rc = or_synth_planted(static_cast<int>(dims.size()), dims.data(), tJ.data(), tR, nnz, noise, tmean, tsd,
                                  seed, d.coords.data(), d.values.data());
  if (rc) std::fprintf(stderr, "oracle synth failed %d\n", rc);
  return d;
}

CooTensor to_tensor(const Data& d) { return CooTensor(Shape(d.dims), d.coords, d.values); }

struct OTensor {
  or_tensor t{};
  explicit OTensor(const Data& d) {
    or_tensor_init(&t, static_cast<int>(d.dims.size()), d.dims.data(), d.values.size(), d.coords.data(),
                   d.values.data());
  }
  ~OTensor() { or_tensor_free(&t); }
};

struct OModel {
  or_model m{};
  OModel(const std::vector<std::uint32_t>& dims, const std::vector<std::uint32_t>& J, std::uint32_t R) {
    or_model_init(&m, static_cast<int>(dims.size()), dims.data(), J.data(), R);
  }
  ~OModel() { or_model_free(&m); }
};

// Copy a host model (rounded to fp32, the device precision) into both sides.
void sync_f32(TuckerModel& tm, OModel& om) {
  for (std::size_t n = 0; n < tm.order(); ++n) {
    for (double& v : tm.factor(n).data()) v = static_cast<double>(static_cast<float>(v));
    for (double& v : tm.kruskal(n).data()) v = static_cast<double>(static_cast<float>(v));
    std::copy(tm.factor(n).data().begin(), tm.factor(n).data().end(), om.m.A[n]);
    std::copy(tm.kruskal(n).data().begin(), tm.kruskal(n).data().end(), om.m.B[n]);
  }
  tm.refresh_core_cache();
  or_model_refresh_core(&om.m);
}

double max_rel(const TuckerModel& tm, const OModel& om, bool factors) {
  double worst = 0.0;
  for (std::size_t n = 0; n < tm.order(); ++n) {
    const Matrix& x = factors ? tm.factor(n) : tm.kruskal(n);
    const double* r = factors ? om.m.A[n] : om.m.B[n];
    for (std::size_t i = 0; i < x.size(); ++i) worst = std::max(worst, rel_err(x.data()[i], r[i]));
  }
  return worst;
}

void copy_rng(const Rng& r, or_rng& o) {
  for (int i = 0; i < Rng::kWords; ++i) o.mt[i] = r.state_words()[i];
  o.idx = r.state_pos();
  o.has_spare = 0;
}

bool same_rng(const Rng& r, const or_rng& o) {
  if (r.state_pos() != o.idx) return false;
  for (int i = 0; i < Rng::kWords; ++i)
    if (r.state_words()[i] != o.mt[i]) return false;
  return true;
}

double unit_sigma(std::size_t order, std::uint32_t J, std::uint32_t R) {
  return std::pow(J * std::pow(static_cast<double>(R), 1.0 / static_cast<double>(order)), -0.25);
}

// ---------------------------------------------------------------- tests
void test_rng_engine_matches_mt19937_64() {
  Rng r(5489);
  std::uint64_t v = 0;
  for (int i = 0; i < 10000; ++i) v = r.next_u64();
  CHECK(v == 9981545732273789042ULL);  // [rand.predef]
  or_rng o;
  or_rng_seed(&o, 77);
  Rng a(77);
  bool same = true;
  for (int i = 0; i < 1000; ++i) same &= a.next_below(1000003 + i) == or_next_below(&o, 1000003 + i);
  CHECK(same);
}

void test_sample_batch_bit_exact_and_errors() {
  const Data d = planted({30, 20, 10}, {2, 2, 2}, 2, 1500, 0.0, 0.5, 0.1, 3);
  const CooTensor t = to_tensor(d);
  Rng r(11);
  or_rng o;
  copy_rng(r, o);
  std::vector<std::uint32_t> pool, out, opool(t.nnz()), oout(t.nnz());
  int ovalid = 0;
  bool same = true;
  for (const std::size_t m : {1u, 7u, 100u, 1500u, 1024u, 3u}) {
    sample_batch(t, m, r, pool, out);
    or_sample_batch(t.nnz(), m, &o, opool.data(), &ovalid, oout.data());
    same &= std::equal(out.begin(), out.end(), oout.begin());
    same &= std::equal(pool.begin(), pool.end(), opool.begin());
  }
  CHECK(same);
  CHECK(same_rng(r, o));
  std::vector<std::uint32_t> all = sample_batch(t, t.nnz(), r);
  CHECK(std::set<std::uint32_t>(all.begin(), all.end()).size() == t.nnz());
  CHECK(throws_as<DomainError>([&] { sample_batch(t, t.nnz() + 1, r); }));
  CHECK(throws_as<DomainError>([&] { sample_batch(t, 0, r); }));
  Rng r1(99), r2(99);
  CHECK(sample_batch(t, 40, r1) == sample_batch(t, 40, r2));
}

void test_epochs_teacher_forced(std::vector<std::uint32_t> dims, std::vector<std::uint32_t> J, std::uint32_t R,
                                std::size_t nnz, std::size_t batch_m, bool resample) {
  const std::size_t order = dims.size();
  const double sig = unit_sigma(order, *std::min_element(J.begin(), J.end()), R);
  const Data d = planted(dims, J, R, nnz, 0.05, 0.0, sig, 17);
  const CooTensor t = to_tensor(d);
  OTensor ot(d);
  TuckerModel tm = TuckerModel::init_gaussian(t.shape(), Ranks{J, R}, 0.0, sig, 23);
  OModel om(dims, J, R);
  sync_f32(tm, om);
  Rng rng(5);
  or_rng orng;
  copy_rng(rng, orng);
  or_core_ws ows;
  or_core_ws_init(&ows, nnz);
  CoreBatchWorkspace ws;
  std::vector<RowBatchWorkspace> rws(1);
  SchedContext sched;
  const double lr = 0.01, reg = 0.01;
  for (int epoch = 0; epoch < 2; ++epoch) {
    const CoreEpochStats cs = update_core_epoch(tm, t, CoreHyper{lr, reg, batch_m, resample, false}, sched, rng, ws);
    const or_core_hyper och{lr, reg, batch_m, resample ? 1 : 0, 0};
    CHECK(or_update_core_epoch(&om.m, &ot.t, &och, &orng, &ows) == 0);
    CHECK(cs.batch_size == (batch_m ? batch_m : nnz));
    if (batch_m) CHECK(std::equal(ws.batch.begin(), ws.batch.end(), ows.batch));
    CHECK(max_rel(tm, om, false) <= 1e-4);
    CHECK(same_rng(rng, orng));
    sync_f32(tm, om);
    const FactorEpochStats fs = update_factor_epoch(tm, t, FactorHyper{lr, reg, 1.0}, sched, rng, rws);
    const or_factor_hyper ofh{lr, reg, 1.0};
    std::size_t up = 0, sk = 0;
    CHECK(or_update_factor_epoch(&om.m, &ot.t, &ofh, &orng, &up, &sk) == 0);
    CHECK(fs.rows_updated == up && fs.rows_skipped == sk);
    CHECK(max_rel(tm, om, true) <= 1e-4);
    sync_f32(tm, om);
  }
  or_core_ws_free(&ows);
}

void test_row_fraction() {
  const std::vector<std::uint32_t> dims{6, 80, 50}, J{4, 4, 4};
  const double sig = unit_sigma(3, 4, 4);
  const Data d = planted(dims, J, 4, 4000, 0.05, 0.0, sig, 3);
  const CooTensor t = to_tensor(d);
  OTensor ot(d);
  TuckerModel tm = TuckerModel::init_gaussian(t.shape(), Ranks{J, 4}, 0.0, sig, 12);
  OModel om(dims, J, 4);
  sync_f32(tm, om);
  Rng rng(31);
  or_rng orng;
  copy_rng(rng, orng);
  std::vector<RowBatchWorkspace> rws;
  SchedContext sched;
  for (const double f : {0.5, 0.25}) {
    update_factor_epoch(tm, t, FactorHyper{0.02, 0.01, f}, sched, rng, rws);
    const or_factor_hyper h{0.02, 0.01, f};
    CHECK(or_update_factor_epoch(&om.m, &ot.t, &h, &orng, nullptr, nullptr) == 0);
    CHECK(same_rng(rng, orng));
    CHECK(max_rel(tm, om, true) <= 1e-4);
    sync_f32(tm, om);
  }
}

void test_rmse_fixed_and_perfect() {
  // zero model, values {0, 2}: RMSE sqrt(2), MAE 1 (test_eval.cpp:32-41)
  const CooTensor t(Shape({2, 1}), {1, 1, 2, 1}, {0.0, 2.0});
  const TuckerModel zero(t.shape(), Ranks{{2, 2}, 2});
  const auto [rmse, mae] = rmse_mae(zero, t);
  CHECK(std::abs(rmse - std::sqrt(2.0)) <= 1e-12);
  CHECK(std::abs(mae - 1.0) <= 1e-12);
  // planted teacher, no noise: error only from fp32 evaluation
  const Data d = planted({5, 4, 3}, {2, 2, 2}, 2, 25, 0.0, 0.5, 0.1, 5);
  const CooTensor p = to_tensor(d);
  const TuckerModel teacher = TuckerModel::init_gaussian(p.shape(), Ranks{{2, 2, 2}, 2}, 0.5, 0.1, 5);
  CHECK(rmse_mae(teacher, p).first <= 1e-6);
  // against the oracle on a noisy set
  const Data n = planted({20, 20, 10}, {3, 3, 3}, 3, 500, 0.5, 0.5, 0.1, 7);
  const CooTensor nt = to_tensor(n);
  OTensor ont(n);
  TuckerModel m = TuckerModel::init_gaussian(nt.shape(), Ranks{{3, 3, 3}, 3}, 0.5, 0.1, 999);
  OModel om({20, 20, 10}, {3, 3, 3}, 3);
  sync_f32(m, om);
  double orm = 0, oma = 0;
  or_rmse_mae(&om.m, &ont.t, &orm, &oma);
  const auto [gr, ga] = rmse_mae(m, nt);
  CHECK(rel_err(gr, orm) <= 1e-5 && rel_err(ga, oma) <= 1e-5);
}

void test_freeze_and_errors() {
  const Data d = planted({12, 10, 8}, {3, 3, 3}, 3, 300, 0.02, 0.5, 0.1, 2);
  const CooTensor t = to_tensor(d);
  TuckerModel m = TuckerModel::init_gaussian(t.shape(), Ranks{{3, 3, 3}, 3}, 0.5, 0.2, 4);
  const TuckerModel before = m;
  Rng rng(3);
  CoreBatchWorkspace ws;
  std::vector<RowBatchWorkspace> rws;
  SchedContext sched;
  const CoreEpochStats cs = update_core_epoch(m, t, CoreHyper{0.0, 0.01, 16, false, false}, sched, rng, ws);
  update_factor_epoch(m, t, FactorHyper{0.0, 0.01, 1.0}, sched, rng, rws);
  CHECK(cs.batch_size == 0);
  bool same = true;
  for (std::size_t n = 0; n < 3; ++n) same &= m.factor(n) == before.factor(n) && m.kruskal(n) == before.kruskal(n);
  CHECK(same);
  Rng fresh(3);
  CHECK(fresh.state_words() == rng.state_words() && fresh.state_pos() == rng.state_pos());
  CHECK(throws_as<DomainError>([&] { update_core_epoch(m, t, CoreHyper{0.01, 0.01, 301, false, false}, sched, rng, ws); }));
  CHECK(throws_as<DomainError>([&] { update_factor_epoch(m, t, FactorHyper{0.01, 0.01, 0.0}, sched, rng, rws); }));
  CHECK(throws_as<DomainError>([&] { sgd_step(0, 0.01, 0.1, std::span<double>(), std::span<const double>()); }));
  std::vector<double> w{2.0}, v{4.0};
  sgd_step(1, 0.0, 0.5, w, v);
  CHECK(std::abs(w[0]) <= 1e-15);  // 2 - 0.5 * 4
  CHECK(throws_as<NumericError>([&] {
    for (int i = 0; i < 50; ++i) update_factor_epoch(m, t, FactorHyper{1e30, 0.01, 1.0}, sched, rng, rws);
  }));
  CHECK(throws_as<DataError>([&] { CooTensor(Shape({2, 2}), {1, 1, 1, 1}, {1.0, 2.0}); }));  // duplicate
  CHECK(throws_as<DataError>([&] { CooTensor(Shape({2, 2}), {3, 1}, {1.0}); }));           // range
}

void test_train_end_to_end_vs_oracle() {
  const std::vector<std::uint32_t> dims{40, 30, 20};
  const Data d = planted(dims, {3, 3, 3}, 3, 3000, 0.01, 0.0, 1.0, 1);
  const CooTensor full = to_tensor(d);
  auto [tr, te] = train_test_split(full, 0.1, 1);
  HyperParams h;
  h.ranks = {3, 3, 3};
  h.r_core = 3;
  h.lr_a = h.lr_b = 0.01;
  h.reg_a = h.reg_b = 0.01;
  h.batch_m = 64;
  h.epochs = 4;
  h.seed = 1;
  auto [model, res] = train_from_scratch(tr, &te, h);
  // oracle: same split (ids from Rng(1)), same init, same batch stream
  std::vector<std::uint32_t> ids(d.values.size());
  std::size_t ntest = 0;
  or_train_test_split_ids(d.values.size(), 0.1, 1, ids.data(), &ntest);
  auto gather = [&](std::size_t b, std::size_t e) {
    Data x{dims, {}, {}};
    for (std::size_t i = b; i < e; ++i) {
      for (std::size_t k = 0; k < 3; ++k) x.coords.push_back(d.coords[ids[i] * 3 + k]);
      x.values.push_back(d.values[ids[i]]);
    }
    return x;
  };
  const Data otr = gather(ntest, ids.size()), ote = gather(0, ntest);
  CHECK(otr.values == tr.values() && ote.values == te.values());
  OTensor a(otr), b(ote);
  OModel om(dims, {3, 3, 3}, 3);
  or_model_init_gaussian(&om.m, 0.5, 0.1, 1);
  const or_hyper oh{0.01, 0.01, 0.01, 0.01, 64, 1.0, 4, 1, 0.5, 0.1, 0, 0};
  std::vector<double> met(4 * 4);
  CHECK(or_train(&om.m, &a.t, &b.t, &oh, met.data()) == 0);
  for (std::size_t e = 0; e < 4; ++e) {
    CHECK(std::abs(res.metrics[e].train_rmse - met[e * 4]) <= 1e-3);
    CHECK(std::abs(res.metrics[e].test_rmse - met[e * 4 + 2]) <= 1e-3);
  }
  const CommCost c = comm_cost_report(Ranks{h.ranks, h.r_core});
  bool cols = true;
  for (const EpochMetrics& row : res.metrics)
    cols &= row.comm_bytes == 8 * c.kruskal_params && row.peak_bytes > 0 && row.total_s == row.core_s + row.factor_s;
  CHECK(cols);
  CHECK(res.metrics.back().peak_bytes == res.metrics.front().peak_bytes);
  // no test set -> NaN test columns
  auto [m2, r2] = train_from_scratch(tr, nullptr, h);
  CHECK(std::isnan(r2.metrics.back().test_rmse));
  // determinism: identical reruns
  bool ident = true;
  for (std::size_t n = 0; n < 3; ++n) ident &= m2.factor(n) == model.factor(n) && m2.kruskal(n) == model.kruskal(n);
  CHECK(ident);
}

// Device residency of the per-epoch calls: with no host edits in between,
// K epochs through update_core_epoch / update_factor_epoch (model and pool
// kept on the device, B / A / pool deltas copied back) equal train()'s
// device loop bit for bit, and the host workspace pool equals the oracle's;
// host edits between calls (a factor row, a Kruskal column, two pool slots)
// are seen and uploaded.
void test_resident_per_epoch_calls() {
  const std::vector<std::uint32_t> dims{60, 300, 40}, J{8, 8, 8};
  const double sig = unit_sigma(3, 8, 8);
  const Data d = planted(dims, J, 8, 20000, 0.05, 0.0, sig, 5);
  const CooTensor t = to_tensor(d);
  HyperParams h;
  h.ranks = J;
  h.r_core = 8;
  h.lr_a = h.lr_b = 0.01;
  h.reg_a = h.reg_b = 0.01;
  h.batch_m = 1024;
  h.epochs = 3;
  h.seed = 4;
  h.init_mean = 0.0;
  h.init_stddev = sig;
  auto [want, res] = train_from_scratch(t, nullptr, h);
  TuckerModel tm = TuckerModel::init_gaussian(t.shape(), Ranks{J, 8}, 0.0, sig, h.seed);
  Rng rng(h.seed + 1);
  CoreBatchWorkspace ws;
  std::vector<RowBatchWorkspace> rws;
  SchedContext sched;
  OTensor ot(d);
  or_core_ws ows;
  or_core_ws_init(&ows, t.nnz());
  or_rng orng;
  copy_rng(rng, orng);
  for (std::size_t e = 0; e < h.epochs; ++e) {
    update_core_epoch(tm, t, CoreHyper{h.lr_b, h.reg_b, h.batch_m, false, false}, sched, rng, ws);
    update_factor_epoch(tm, t, FactorHyper{h.lr_a, h.reg_a, 1.0}, sched, rng, rws);
    // the oracle's sampler alone tracks the pool (no model needed for Psi)
    std::vector<std::uint32_t> psi(h.batch_m);
    or_sample_batch(t.nnz(), h.batch_m, &orng, ows.pool, &ows.pool_valid, psi.data());
    CHECK(std::equal(psi.begin(), psi.end(), ws.batch.begin()));
    CHECK(std::equal(ws.sample_pool.begin(), ws.sample_pool.end(), ows.pool));
  }
  bool ident = true;
  for (std::size_t n = 0; n < 3; ++n) ident &= tm.factor(n) == want.factor(n) && tm.kruskal(n) == want.kruskal(n);
  CHECK(ident);
  // host edits between calls: a factor entry, a Kruskal entry, two pool slots
  tm.factor(1).at(7, 3) += 0.25;
  tm.kruskal(2).at(1, 1) -= 0.125;
  tm.refresh_core_cache();
  std::swap(ws.sample_pool[3], ws.sample_pool[t.nnz() - 2]);
  std::swap(ows.pool[3], ows.pool[t.nnz() - 2]);
  TuckerModel edited = tm;
  CoreBatchWorkspace ws2;
  ws2.sample_pool = ws.sample_pool;
  Rng rng2 = rng;
  update_core_epoch(tm, t, CoreHyper{h.lr_b, h.reg_b, h.batch_m, false, false}, sched, rng, ws);
  std::vector<std::uint32_t> psi(h.batch_m);
  or_sample_batch(t.nnz(), h.batch_m, &orng, ows.pool, &ows.pool_valid, psi.data());
  CHECK(std::equal(psi.begin(), psi.end(), ws.batch.begin()));
  CHECK(std::equal(ws.sample_pool.begin(), ws.sample_pool.end(), ows.pool));
  // the same step on a fresh tensor object (new device session: everything
  // uploaded) gives the identical B
  const CooTensor t2 = to_tensor(d);
  update_core_epoch(edited, t2, CoreHyper{h.lr_b, h.reg_b, h.batch_m, false, false}, sched, rng2, ws2);
  bool same = ws2.batch == ws.batch;
  for (std::size_t n = 0; n < 3; ++n) same &= edited.kruskal(n) == tm.kruskal(n) && edited.factor(n) == tm.factor(n);
  CHECK(same);
  or_core_ws_free(&ows);
}

// Multi-GPU train() (HyperParams::devices; ranks on the same device here:
// stream-ordered barriers, no kernel waits on another): replicated and
// sharded core, 2 and 3 ranks, against the single-session train() and the
// oracle's per-epoch RMSE.
void test_train_multi_gpu() {
  const std::vector<std::uint32_t> dims{60, 50, 40};
  const double sig = unit_sigma(3, 6, 6);
  const Data d = planted(dims, {6, 6, 6}, 6, 12000, 0.05, 0.0, sig, 3);
  const CooTensor full = to_tensor(d);
  auto [tr, te] = train_test_split(full, 0.1, 1);
  HyperParams h;
  h.ranks = {6, 6, 6};
  h.r_core = 6;
  h.lr_a = h.lr_b = 0.01;
  h.reg_a = h.reg_b = 0.01;
  h.batch_m = 1500;
  h.epochs = 3;
  h.seed = 2;
  h.init_mean = 0.0;
  h.init_stddev = sig;
  auto [one, r1] = train_from_scratch(tr, &te, h);
  for (const bool sharded : {false, true})
    for (const int P : {2, 3}) {
      HyperParams hm = h;
      hm.devices.assign(P, 0);
      hm.core_sharded = sharded;
      auto [many, rp] = train_from_scratch(tr, &te, hm);
      CHECK(rp.metrics.size() == r1.metrics.size());
      for (std::size_t e = 0; e < rp.metrics.size(); ++e) {
        CHECK(std::abs(rp.metrics[e].train_rmse - r1.metrics[e].train_rmse) <= 1e-4);
        CHECK(std::abs(rp.metrics[e].test_rmse - r1.metrics[e].test_rmse) <= 1e-4);
      }
      double worst = 0.0;
      for (std::size_t n = 0; n < 3; ++n) {
        for (std::size_t i = 0; i < many.factor(n).size(); ++i)
          worst = std::max(worst, std::abs(many.factor(n).data()[i] - one.factor(n).data()[i]) /
                                      std::max(1.0, std::abs(one.factor(n).data()[i])));
        for (std::size_t i = 0; i < many.kruskal(n).size(); ++i)
          worst = std::max(worst, std::abs(many.kruskal(n).data()[i] - one.kruskal(n).data()[i]) /
                                      std::max(1.0, std::abs(one.kruskal(n).data()[i])));
      }
      CHECK(worst <= 1e-4);
    }
  HyperParams bad = h;
  bad.devices = {0, 0};
  bad.row_fraction = 0.5;
  CHECK(throws_as<ConfigError>([&] { train_from_scratch(tr, &te, bad); }));
}

void test_config_errors() {
  const Data d = planted({12, 10, 8}, {3, 3, 3}, 3, 300, 0.02, 0.5, 0.1, 2);
  const CooTensor t = to_tensor(d);
  HyperParams h;
  h.ranks = {3, 3, 3};
  h.r_core = 4;  // R > J
  CHECK(throws_as<ConfigError>([&] { train_from_scratch(t, nullptr, h); }));
  h.r_core = 3;
  h.lr_a = 0.0;
  CHECK(throws_as<ConfigError>([&] { train_from_scratch(t, nullptr, h); }));
  h.lr_a = 0.01;
  h.ranks = {3, 3};
  CHECK(throws_as<ConfigError>([&] { train_from_scratch(t, nullptr, h); }));
}

// ---------------------------------------------------------------- I/O golden
// Replays tests/golden/io/cases.txt (written by the reference itself,
// tests/golden/make_io_golden.py): the delimited reader / writer, the model
// file, the metrics CSV, synth_planted / synth_ratings and the index maps must
// give the reference's bytes, values, exception classes and messages.
std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::size_t start = 0;
  for (std::size_t i = 0; i <= s.size(); ++i)
    if (i == s.size() || s[i] == sep) {
      out.push_back(s.substr(start, i - start));
      start = i + 1;
    }
  return out;
}

std::vector<std::uint32_t> u32_list(const std::string& s) {
  std::vector<std::uint32_t> v;
  if (s == "-" || s.empty()) return v;
  for (const auto& x : split(s, ',')) v.push_back(static_cast<std::uint32_t>(std::stoull(x)));
  return v;
}

std::string slurp(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return "<missing " + path + ">";
  std::string b;
  char buf[1 << 14];
  std::size_t n;
  while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) b.append(buf, n);
  std::fclose(f);
  return b;
}

// code of the exception class (sgdt.h numbering) and its message
template <class F>
std::pair<int, std::string> outcome(F&& f) {
  try {
    f();
  } catch (const DataError& e) {  // FormatError is a DataError
    return {3, e.what()};
  } catch (const ConfigError& e) {
    return {2, e.what()};
  } catch (const NumericError& e) {
    return {4, e.what()};
  } catch (const DomainError& e) {
    return {5, e.what()};
  } catch (const std::exception& e) {
    return {1, e.what()};
  }
  return {0, ""};
}

void test_io_golden(const std::string& dir, const char* chunk_bytes) {
  if (chunk_bytes)
    setenv("SPTUCKER_LOAD_CHUNK_BYTES", chunk_bytes, 1);
  else
    unsetenv("SPTUCKER_LOAD_CHUNK_BYTES");
  char tmpl[] = "/tmp/sptucker_io_XXXXXX";
  const std::string out = mkdtemp(tmpl);
  char cwd[4096];
  CHECK(getcwd(cwd, sizeof cwd) != nullptr);
  CHECK(chdir(dir.c_str()) == 0);
  const std::string cases = slurp("cases.txt");
  int n_cases = 0;
  for (const std::string& line : split(cases, '\n')) {
    if (line.empty()) continue;
    const std::vector<std::string> f = split(line, '\t');
    ++n_cases;
    g_case = "io golden: " + f[0] + " " + f[1];
    const std::string kind = f[0];
    if (kind == "load") {
      LoadOptions o;
      o.skip_header = f[3] == "1";
      o.zero_policy = f[4] == "1" ? ZeroPolicy::Replace : ZeroPolicy::Reject;
      o.zero_replacement = std::stod(f[5]);
      o.dims_override = u32_list(f[6]);
      const std::string saved = out + "/" + f[9];
      const auto [code, msg] = outcome([&] {
        const CooTensor t = CooTensor::load_delimited(f[1], std::stoul(f[2]), o);
        CHECK(t.shape().dims() == u32_list(f[8]));
        t.save_delimited(saved);
      });
      CHECK(code == std::stoi(f[7]));
      CHECK(msg == f[10]);
      if (code == 0) CHECK(slurp(saved) == slurp(f[9]));
      if (code != std::stoi(f[7]) || msg != f[10]) std::fprintf(stderr, "  got %d '%s'\n", code, msg.c_str());
    } else if (kind == "modelgen") {
      const TuckerModel m = TuckerModel::init_gaussian(Shape(u32_list(f[1])), Ranks{u32_list(f[2]),
                                                       static_cast<std::uint32_t>(std::stoul(f[3]))},
                                                       std::stod(f[4]), std::stod(f[5]), std::stoull(f[6]));
      m.save(out + "/gen.bin");
      CHECK(slurp(out + "/gen.bin") == slurp(f[7]));
      const TuckerModel back = TuckerModel::load(f[7]);
      for (std::size_t n = 0; n < m.order(); ++n) {
        CHECK(back.factor(n) == m.factor(n));
        CHECK(back.kruskal(n) == m.kruskal(n));
      }
    } else if (kind == "model") {
      const auto [code, msg] = outcome([&] {
        const TuckerModel m = TuckerModel::load(f[1]);
        m.save(out + "/" + f[3]);
      });
      CHECK(code == std::stoi(f[2]));
      CHECK(msg == f[4]);
      if (code == 0) CHECK(slurp(out + "/" + f[3]) == slurp(f[3]));
      if (code != std::stoi(f[2]) || msg != f[4]) std::fprintf(stderr, "  got %d '%s'\n", code, msg.c_str());
    } else if (kind == "mwrite") {
      std::vector<std::string> comments = split(f[2], '|');
      std::vector<EpochMetrics> rows;
      for (const std::string& r : split(f[3], ';')) {
        std::vector<double> x;
        for (const std::string& v : split(r, ',')) x.push_back(std::strtod(v.c_str(), nullptr));
        EpochMetrics m;
        m.epoch = static_cast<std::size_t>(x[0]);
        m.core_s = x[1];
        m.factor_s = x[2];
        m.total_s = x[3];
        m.train_rmse = x[4];
        m.train_mae = x[5];
        m.test_rmse = x[6];
        m.test_mae = x[7];
        m.peak_bytes = static_cast<std::uint64_t>(x[8]);
        m.comm_bytes = static_cast<std::uint64_t>(x[9]);
        rows.push_back(m);
      }
      write_metrics_csv(out + "/m.csv", rows, comments);
      CHECK(slurp(out + "/m.csv") == slurp(f[1]));
    } else if (kind == "mparse") {
      std::vector<std::string> comments;
      std::size_t nrows = 0;
      const auto [code, msg] = outcome([&] { nrows = parse_metrics_csv(f[1], &comments).size(); });
      CHECK(code == std::stoi(f[2]));
      CHECK(msg == f[5]);
      if (code == 0) {
        CHECK(nrows == std::stoul(f[3]));
        std::string joined;
        for (std::size_t i = 0; i < comments.size(); ++i) joined += (i ? "|" : "") + comments[i];
        CHECK(joined == f[4]);
      }
    } else if (kind == "planted") {
      PlantedSpec p;
      p.shape = Shape(u32_list(f[1]));
      p.teacher_ranks = Ranks{u32_list(f[2]), static_cast<std::uint32_t>(std::stoul(f[3]))};
      p.nnz = std::stoul(f[4]);
      p.noise_stddev = std::stod(f[5]);
      p.teacher_mean = std::stod(f[6]);
      p.teacher_stddev = std::stod(f[7]);
      p.seed = std::stoull(f[8]);
      synth_planted(p).save_delimited(out + "/p.tns");
      CHECK(slurp(out + "/p.tns") == slurp(f[9]));
    } else if (kind == "ratings") {
      RatingSpec r;
      r.base.shape = Shape(u32_list(f[1]));
      r.base.teacher_ranks = Ranks{u32_list(f[2]), static_cast<std::uint32_t>(std::stoul(f[3]))};
      r.base.nnz = std::stoul(f[4]);
      r.base.teacher_mean = std::stod(f[5]);
      r.base.teacher_stddev = std::stod(f[6]);
      r.base.seed = std::stoull(f[7]);
      r.target_mean = std::stod(f[8]);
      r.target_stddev = std::stod(f[9]);
      r.noise_stddev = std::stod(f[10]);
      r.quantize_half_steps = f[11] == "1";
      r.min_value = std::stod(f[12]);
      r.max_value = std::stod(f[13]);
      synth_ratings(r).save_delimited(out + "/r.tns");
      CHECK(slurp(out + "/r.tns") == slurp(f[14]));
    } else if (kind == "index") {
      const Shape shape(u32_list(f[1]));
      const std::vector<std::uint32_t> c = u32_list(f[2]);
      const std::size_t mode = std::stoul(f[3]);
      std::uint64_t col = 0, vec = 0;
      std::vector<std::uint32_t> inv(c.size());
      const auto [code, msg] = outcome([&] {
        col = unfold_col_index(shape, c, mode);
        vec = vec_index(shape, c, mode);
        invert_vec_index(shape, vec, mode, inv);
      });
      CHECK(code == std::stoi(f[4]));
      CHECK(msg == f[8]);
      if (code == 0) {
        CHECK(col == std::stoull(f[5]));
        CHECK(vec == std::stoull(f[6]));
        CHECK(inv == u32_list(f[7]));
      }
    } else {
      CHECK(!"unknown golden case kind");
    }
  }
  CHECK(n_cases > 60);
  CHECK(chdir(cwd) == 0);
  std::filesystem::remove_all(out);
  unsetenv("SPTUCKER_LOAD_CHUNK_BYTES");
}

// save -> load round trips of the host I/O on generated data (no golden).
void test_io_round_trips() {
  char tmpl[] = "/tmp/sptucker_rt_XXXXXX";
  const std::string out = mkdtemp(tmpl);
  const Data d = planted({60, 50, 40, 3}, {3, 3, 3, 2}, 2, 5000, 0.1, 0.5, 0.1, 21);
  const CooTensor t = to_tensor(d);
  t.save_delimited(out + "/t.tns");
  setenv("SPTUCKER_LOAD_CHUNK_BYTES", "1000", 1);
  const CooTensor back = CooTensor::load_delimited(out + "/t.tns", 4);
  unsetenv("SPTUCKER_LOAD_CHUNK_BYTES");
  CHECK(back.coords() == t.coords());
  CHECK(back.values() == t.values());  // %.17g round-trips fp64 exactly
  for (std::size_t n = 0; n < 4; ++n) {
    CHECK(back.mode_perm(n) == t.mode_perm(n));
    CHECK(back.mode_offsets(n) == t.mode_offsets(n));
  }
  TuckerModel m = TuckerModel::init_gaussian(t.shape(), Ranks{{3, 3, 3, 2}, 2}, 0.0, 1.0, 4);
  m.save(out + "/m.bin");
  const TuckerModel mb = TuckerModel::load(out + "/m.bin");
  for (std::size_t n = 0; n < 4; ++n) CHECK(mb.factor(n) == m.factor(n) && mb.kruskal(n) == m.kruskal(n));
  // planted generator == the pinned oracle's, bit for bit
  PlantedSpec p;
  p.shape = Shape({60, 50, 40, 3});
  p.teacher_ranks = Ranks{{3, 3, 3, 2}, 2};
  p.nnz = 5000;
  p.noise_stddev = 0.1;
  p.seed = 21;
  const CooTensor s = synth_planted(p);
  CHECK(s.coords() == d.coords);
  CHECK(s.values() == d.values);
  std::filesystem::remove_all(out);
}

void run(const char* name, const std::function<void()>& f) {
  g_case = name;
  const int before = g_fail;
  try {
    f();
  } catch (const std::exception& e) {
    ++g_fail;
    std::fprintf(stderr, "FAIL [%s] unexpected exception: %s\n", name, e.what());
  }
  std::printf("%s %s\n", g_fail == before ? "ok  " : "FAIL", name);
}

}  // namespace

int main(int argc, char** argv) {
  bool cpu_only = false;
  std::string golden;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--cpu-only") cpu_only = true;
    if (a == "--golden" && i + 1 < argc) golden = argv[++i];
  }
  run("rng engine", test_rng_engine_matches_mt19937_64);
  run("io round trips", test_io_round_trips);
  if (!golden.empty()) {
    run("io golden (1 thread chunking)", [&] { test_io_golden(golden, nullptr); });
    run("io golden (512-byte chunks)", [&] { test_io_golden(golden, "512"); });
  }
  if (cpu_only) {  // no device in the build container
    run("config errors", test_config_errors);
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
  }
  run("sample_batch bit-exact", test_sample_batch_bit_exact_and_errors);
  run("epochs 12x10x8 R2", [] { test_epochs_teacher_forced({12, 10, 8}, {3, 3, 3}, 2, 300, 16, false); });
  run("epochs 40x30x20 R5", [] { test_epochs_teacher_forced({40, 30, 20}, {5, 5, 5}, 5, 5000, 256, false); });
  run("epochs full batch", [] { test_epochs_teacher_forced({12, 10, 8}, {3, 4, 3}, 3, 300, 0, false); });
  run("epochs order-4 resample", [] { test_epochs_teacher_forced({9, 7, 6, 5}, {2, 3, 2, 2}, 2, 400, 50, true); });
  run("epochs order-2", [] { test_epochs_teacher_forced({30, 25}, {3, 3}, 3, 220, 20, false); });
  run("epochs split rows", [] { test_epochs_teacher_forced({6, 300, 300}, {8, 8, 8}, 8, 30000, 2048, false); });
  run("epochs R10", [] { test_epochs_teacher_forced({50, 40, 30}, {10, 10, 10}, 10, 8000, 1024, false); });
  run("row fraction", test_row_fraction);
  run("rmse", test_rmse_fixed_and_perfect);
  run("freeze and errors", test_freeze_and_errors);
  run("train end to end", test_train_end_to_end_vs_oracle);
  run("resident per-epoch calls", test_resident_per_epoch_calls);
  run("multi-GPU train", test_train_multi_gpu);
  run("config errors", test_config_errors);
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
