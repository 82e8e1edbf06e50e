// ref_bridge.cpp -- TEST INFRASTRUCTURE ONLY.
//
// POD (extern "C") bridge over the UNMODIFIED reference library, compiled
// together with /root/reference/proj/src/*.cpp by oracle/Makefile into
// oracle/_ref/libsptucker_ref.so.  It lets the Python tests pin the C oracle
// against the reference itself and lets bench.py time the reference CPU path
// (`--impl reference`, `cpu_baseline.kind == "reference"`).  Nothing here is
// linked into the product library.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <span>
#include <string>
#include <cstdio>
#include <vector>

#include "sptucker/common.hpp"
#include "sptucker/core_optimizer.hpp"
#include "sptucker/eval.hpp"
#include "sptucker/factor_optimizer.hpp"
#include "sptucker/model.hpp"
#include "sptucker/scheduler.hpp"
#include "sptucker/sptensor.hpp"
#include "sptucker/synth.hpp"
#include "sptucker/trainer.hpp"

using namespace sptucker;

namespace {

// Same code map as the C-ABI (include/sgdt.h) and oracle/sgdt_oracle.h.
int code_of(const std::exception_ptr& p) {
  try {
    std::rethrow_exception(p);
  } catch (const ConfigError&) {
    return 2;
  } catch (const DataError&) {
    return 3;
  } catch (const NumericError&) {
    return 4;
  } catch (const DomainError&) {
    return 5;
  } catch (...) {
    return 1;
  }
}

#define GUARD(...)                           \
  try {                                      \
    __VA_ARGS__;                             \
    return 0;                                \
  } catch (...) {                            \
    return code_of(std::current_exception()); \
  }

struct RefTensor {
  std::unique_ptr<CooTensor> t;
};
struct RefModel {
  std::unique_ptr<TuckerModel> m;
};
struct RefRng {
  Rng rng;
  CoreBatchWorkspace core_ws;
  std::vector<RowBatchWorkspace> row_ws;
  explicit RefRng(std::uint64_t seed) : rng(seed) {}
};

Strategy strat_of(int s) {
  return s == 0 ? Strategy::Serial : (s == 1 ? Strategy::Naive : Strategy::Improved);
}

}  // namespace

extern "C" {

int ref_mt_outputs(std::uint64_t seed, std::size_t n, std::uint64_t* out) {
  GUARD({
    Rng r(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = r.next_u64();
  });
}

int ref_next_below_seq(std::uint64_t seed, std::size_t n, const std::uint64_t* bounds,
                       std::uint64_t* out) {
  GUARD({
    Rng r(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = r.next_below(bounds[i]);
  });
}

int ref_gaussian_seq(std::uint64_t seed, std::size_t n, double mean, double sd, double* out) {
  GUARD({
    Rng r(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = r.next_gaussian(mean, sd);
  });
}

int ref_synth_planted(int order, const std::uint32_t* dims, const std::uint32_t* tJ,
                      std::uint32_t tR, std::size_t nnz, double noise, double tmean,
                      double tsd, std::uint64_t seed, std::uint32_t* coords_out,
                      double* values_out) {
  GUARD({
    PlantedSpec spec;
    spec.shape = Shape(std::vector<std::uint32_t>(dims, dims + order));
    spec.teacher_ranks = Ranks{std::vector<std::uint32_t>(tJ, tJ + order), tR};
    spec.nnz = nnz;
    spec.noise_stddev = noise;
    spec.teacher_mean = tmean;
    spec.teacher_stddev = tsd;
    spec.seed = seed;
    const CooTensor t = synth_planted(spec);
    for (std::size_t e = 0; e < t.nnz(); ++e) {
      const auto c = t.coord(e);
      std::copy(c.begin(), c.end(), coords_out + e * order);
      values_out[e] = t.value(e);
    }
  });
}

void* ref_tensor_new(int order, const std::uint32_t* dims, std::size_t nnz,
                     const std::uint32_t* coords, const double* values, int* rc) {
  try {
    auto* h = new RefTensor;
    h->t = std::make_unique<CooTensor>(
        Shape(std::vector<std::uint32_t>(dims, dims + order)),
        std::vector<std::uint32_t>(coords, coords + nnz * order),
        std::vector<double>(values, values + nnz));
    *rc = 0;
    return h;
  } catch (...) {
    *rc = code_of(std::current_exception());
    return nullptr;
  }
}

void ref_tensor_free(void* h) { delete static_cast<RefTensor*>(h); }

int ref_tensor_perm(void* h, int mode, std::uint32_t* perm_out, std::uint64_t* offsets_out) {
  GUARD({
    const CooTensor& t = *static_cast<RefTensor*>(h)->t;
    const auto& p = t.mode_perm(mode);
    std::copy(p.begin(), p.end(), perm_out);
    const auto& o = t.mode_offsets(mode);
    std::copy(o.begin(), o.end(), offsets_out);
  });
}

// Split into train/test (sptensor.cpp:217-254); outputs sized by the caller:
// ntest = llround(frac * nnz).
int ref_train_test_split(void* h, double frac, std::uint64_t seed, std::uint32_t* tr_coords,
                         double* tr_values, std::uint32_t* te_coords, double* te_values) {
  GUARD({
    const CooTensor& t = *static_cast<RefTensor*>(h)->t;
    auto [tr, te] = train_test_split(t, frac, seed);
    const std::size_t order = t.order();
    for (std::size_t e = 0; e < tr.nnz(); ++e) {
      const auto c = tr.coord(e);
      std::copy(c.begin(), c.end(), tr_coords + e * order);
      tr_values[e] = tr.value(e);
    }
    for (std::size_t e = 0; e < te.nnz(); ++e) {
      const auto c = te.coord(e);
      std::copy(c.begin(), c.end(), te_coords + e * order);
      te_values[e] = te.value(e);
    }
  });
}

void* ref_model_new(int order, const std::uint32_t* dims, const std::uint32_t* J,
                    std::uint32_t R, int* rc) {
  try {
    auto* h = new RefModel;
    h->m = std::make_unique<TuckerModel>(Shape(std::vector<std::uint32_t>(dims, dims + order)),
                                         Ranks{std::vector<std::uint32_t>(J, J + order), R});
    *rc = 0;
    return h;
  } catch (...) {
    *rc = code_of(std::current_exception());
    return nullptr;
  }
}

void ref_model_free(void* h) { delete static_cast<RefModel*>(h); }

int ref_model_init_gaussian(void* h, double mean, double sd, std::uint64_t seed) {
  GUARD({
    TuckerModel& m = *static_cast<RefModel*>(h)->m;
    m = TuckerModel::init_gaussian(m.shape(), m.ranks(), mean, sd, seed);
  });
}

// Copy parameters in (dir=0) or out (dir=1); A and B are arrays of order
// pointers to row-major fp64 buffers.
int ref_model_params(void* h, int dir, double* const* A, double* const* B) {
  GUARD({
    TuckerModel& m = *static_cast<RefModel*>(h)->m;
    for (std::size_t n = 0; n < m.order(); ++n) {
      auto& a = m.factor(n).data();
      auto& b = m.kruskal(n).data();
      if (dir == 0) {
        std::copy(A[n], A[n] + a.size(), a.begin());
        std::copy(B[n], B[n] + b.size(), b.begin());
      } else {
        std::copy(a.begin(), a.end(), A[n]);
        std::copy(b.begin(), b.end(), B[n]);
      }
    }
    if (dir == 0) m.refresh_core_cache();
  });
}

double ref_model_predict(void* h, const std::uint32_t* coord) {
  const TuckerModel& m = *static_cast<RefModel*>(h)->m;
  return m.predict(std::span<const std::uint32_t>(coord, m.order()));
}

void* ref_rng_new(std::uint64_t seed) { return new RefRng(seed); }
void ref_rng_free(void* h) { delete static_cast<RefRng*>(h); }

int ref_sample_batch(void* rng, void* tensor, std::size_t m, std::uint32_t* out) {
  GUARD({
    auto* r = static_cast<RefRng*>(rng);
    const CooTensor& t = *static_cast<RefTensor*>(tensor)->t;
    std::vector<std::uint32_t> o;
    sample_batch(t, m, r->rng, r->core_ws.sample_pool, o);
    std::copy(o.begin(), o.end(), out);
  });
}

// One core epoch; the RNG handle carries the persistent sample pool.
// batch_out (nullable) receives the last Psi drawn.
int ref_core_epoch(void* model, void* tensor, void* rng, double lr, double reg,
                   std::size_t batch_m, int resample, int incremental, int strategy,
                   std::size_t threads, std::uint32_t* batch_out) {
  GUARD({
    auto* r = static_cast<RefRng*>(rng);
    TuckerModel& m = *static_cast<RefModel*>(model)->m;
    const CooTensor& t = *static_cast<RefTensor*>(tensor)->t;
    WorkerPool pool(threads);
    SchedContext sched{strat_of(strategy), BalancePolicy::Dynamic,
                       strategy == 0 ? nullptr : &pool};
    CoreHyper h{lr, reg, batch_m, resample != 0, incremental != 0};
    update_core_epoch(m, t, h, sched, r->rng, r->core_ws);
    if (batch_out) std::copy(r->core_ws.batch.begin(), r->core_ws.batch.end(), batch_out);
  });
}

int ref_factor_epoch(void* model, void* tensor, void* rng, double lr, double reg,
                     double row_fraction, int strategy, std::size_t threads,
                     std::size_t* rows_updated, std::size_t* rows_skipped) {
  GUARD({
    auto* r = static_cast<RefRng*>(rng);
    TuckerModel& m = *static_cast<RefModel*>(model)->m;
    const CooTensor& t = *static_cast<RefTensor*>(tensor)->t;
    WorkerPool pool(threads);
    SchedContext sched{strat_of(strategy), BalancePolicy::Dynamic,
                       strategy == 0 ? nullptr : &pool};
    FactorHyper h{lr, reg, row_fraction};
    const FactorEpochStats st = update_factor_epoch(m, t, h, sched, r->rng, r->row_ws);
    if (rows_updated) *rows_updated = st.rows_updated;
    if (rows_skipped) *rows_skipped = st.rows_skipped;
  });
}

int ref_rmse_mae(void* model, void* tensor, double* rmse, double* mae) {
  GUARD({
    const auto [a, b] =
        rmse_mae(*static_cast<RefModel*>(model)->m, *static_cast<RefTensor*>(tensor)->t);
    *rmse = a;
    *mae = b;
  });
}

// train_from_scratch (trainer.cpp:127-139).  metrics: epochs x 6 doubles
// {core_s, factor_s, train_rmse, train_mae, test_rmse, test_mae}.
int ref_train_from_scratch(void* train_t, void* test_t, const std::uint32_t* J,
                           std::uint32_t R, double lr_a, double lr_b, double reg_a,
                           double reg_b, std::size_t batch_m, double row_fraction,
                           std::size_t epochs, std::uint64_t seed, double init_mean,
                           double init_sd, int strategy, std::size_t threads, void* model_out,
                           double* metrics) {
  GUARD({
    const CooTensor& tr = *static_cast<RefTensor*>(train_t)->t;
    const CooTensor* te = test_t ? static_cast<RefTensor*>(test_t)->t.get() : nullptr;
    HyperParams h;
    h.ranks.assign(J, J + tr.order());
    h.r_core = R;
    h.lr_a = lr_a;
    h.lr_b = lr_b;
    h.reg_a = reg_a;
    h.reg_b = reg_b;
    h.batch_m = batch_m;
    h.row_fraction = row_fraction;
    h.epochs = epochs;
    h.seed = seed;
    h.init_mean = init_mean;
    h.init_stddev = init_sd;
    h.strategy = strat_of(strategy);
    h.threads = threads;
    auto [m, res] = train_from_scratch(tr, te, h);
    for (std::size_t e = 0; e < res.metrics.size(); ++e) {
      const auto& row = res.metrics[e];
      double* o = metrics + e * 6;
      o[0] = row.core_s;
      o[1] = row.factor_s;
      o[2] = row.train_rmse;
      o[3] = row.train_mae;
      o[4] = row.test_rmse;
      o[5] = row.test_mae;
    }
    if (model_out) *static_cast<RefModel*>(model_out)->m = std::move(m);
  });
}

// Timed epochs through the reference's own bench path (eval.cpp:201-266):
// median seconds of (core + factor) per epoch after `warmup` epochs.
int ref_bench_epoch_seconds(void* train_t, const std::uint32_t* J, std::uint32_t R,
                            double lr_a, double lr_b, double reg, std::size_t batch_m,
                            int strategy, std::size_t threads, std::size_t warmup,
                            std::size_t epochs, std::uint64_t seed, double* seconds) {
  GUARD({
    const CooTensor& tr = *static_cast<RefTensor*>(train_t)->t;
    BenchOptions o;
    o.epochs = epochs;
    o.warmup = warmup;
    o.seed = seed;
    o.lr_a = lr_a;
    o.lr_b = lr_b;
    o.reg = reg;
    o.batch_m = batch_m;
    o.strategy = strat_of(strategy);
    const auto rows = bench_speedup(tr, Ranks{std::vector<std::uint32_t>(J, J + tr.order()), R},
                                    {threads}, o);
    *seconds = rows.at(0).seconds_per_epoch;
  });
}

// timed_epochs (eval.cpp:201-223) with a configurable initialisation: the
// reference's own epoch calls, Strategy as given, `threads` workers; median
// seconds of (core + factor) over `epochs` after `warmup`.
int ref_time_epochs(void* train_t, const std::uint32_t* J, std::uint32_t R, double lr_a, double lr_b,
                    double reg, std::size_t batch_m, int strategy, std::size_t threads, std::size_t warmup,
                    std::size_t epochs, std::uint64_t seed, double init_mean, double init_sd, double* seconds) {
  GUARD({
    const CooTensor& tr = *static_cast<RefTensor*>(train_t)->t;
    TuckerModel model = TuckerModel::init_gaussian(
        tr.shape(), Ranks{std::vector<std::uint32_t>(J, J + tr.order()), R}, init_mean, init_sd, seed);
    Rng rng(seed + 1);
    WorkerPool pool(threads);
    SchedContext sched{threads <= 1 ? Strategy::Serial : strat_of(strategy), BalancePolicy::Dynamic,
                       threads <= 1 ? nullptr : &pool};
    CoreBatchWorkspace cws;
    std::vector<RowBatchWorkspace> rws(sched.workers());
    std::vector<double> secs;
    for (std::size_t e = 0; e < warmup + epochs; ++e) {
      const auto t0 = std::chrono::steady_clock::now();
      update_core_epoch(model, tr, CoreHyper{lr_b, reg, batch_m, false, false}, sched, rng, cws);
      update_factor_epoch(model, tr, FactorHyper{lr_a, reg, 1.0}, sched, rng, rws);
      const auto t1 = std::chrono::steady_clock::now();
      if (e >= warmup) secs.push_back(std::chrono::duration<double>(t1 - t0).count());
    }
    std::sort(secs.begin(), secs.end());
    const std::size_t k = secs.size();
    *seconds = k % 2 ? secs[k / 2] : 0.5 * (secs[k / 2 - 1] + secs[k / 2]);
  });
}

// timed_epochs (eval.cpp:201-223) under a wall-clock budget, for the bench's
// reference arm on full-size tensors (one config 3 epoch takes minutes on
// the CPU): the same model init, RNG seeding, workspaces and per-epoch
// (core + factor) timing, but the epoch counts are capped so the run ends
// in about budget_s.  The first epoch is a warm-up when warmup > 0 and two
// epochs fit the budget; otherwise it is the (only) timed epoch.  Then up to
// warmup - 1 more warm-ups and `epochs` timed epochs, as many as fit
// (at least one timed).  secs_out receives every timed epoch (<= epochs).
int ref_time_epochs_budget(void* train_t, const std::uint32_t* J, std::uint32_t R, double lr_a, double lr_b,
                           double reg, std::size_t batch_m, int strategy, std::size_t threads, std::size_t warmup,
                           std::size_t epochs, std::uint64_t seed, double init_mean, double init_sd,
                           double budget_s, double* secs_out, std::size_t* n_warm, std::size_t* n_timed) {
  GUARD({
    const CooTensor& tr = *static_cast<RefTensor*>(train_t)->t;
    TuckerModel model = TuckerModel::init_gaussian(
        tr.shape(), Ranks{std::vector<std::uint32_t>(J, J + tr.order()), R}, init_mean, init_sd, seed);
    Rng rng(seed + 1);
    WorkerPool pool(threads);
    SchedContext sched{threads <= 1 ? Strategy::Serial : strat_of(strategy), BalancePolicy::Dynamic,
                       threads <= 1 ? nullptr : &pool};
    CoreBatchWorkspace cws;
    std::vector<RowBatchWorkspace> rws(sched.workers());
    auto epoch = [&] {
      const auto t0 = std::chrono::steady_clock::now();
      update_core_epoch(model, tr, CoreHyper{lr_b, reg, batch_m, false, false}, sched, rng, cws);
      update_factor_epoch(model, tr, FactorHyper{lr_a, reg, 1.0}, sched, rng, rws);
      return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    *n_warm = *n_timed = 0;
    if (epochs == 0) return 0;
    const double t1 = epoch();
    double used = t1;
    if (warmup == 0 || 2.0 * t1 > budget_s) {
      secs_out[(*n_timed)++] = t1;
    } else {
      *n_warm = 1;
    }
    // more warm-ups only while the remaining timed epochs still fit
    while (*n_warm > 0 && *n_warm < warmup && used + t1 * (1.0 + static_cast<double>(epochs)) <= budget_s) {
      used += epoch();
      ++*n_warm;
    }
    while (*n_timed < epochs && (*n_timed == 0 || used + t1 <= budget_s)) {
      const double t = epoch();
      used += t;
      secs_out[(*n_timed)++] = t;
    }
  });
}

// ---- host I/O and the ratings generator (golden fixtures for the C++ host
// API: tests/golden/make_io_golden.py).  Every call stores the exception text
// for ref_last_message().
thread_local std::string g_msg;

#define GUARD_MSG(...)                                   \
  try {                                                  \
    g_msg.clear();                                       \
    __VA_ARGS__;                                         \
    return 0;                                            \
  } catch (const std::exception& ex) {                   \
    g_msg = ex.what();                                   \
    return code_of(std::current_exception());            \
  } catch (...) {                                        \
    return code_of(std::current_exception());            \
  }

const char* ref_last_message() { return g_msg.c_str(); }

// CooTensor::load_delimited (sptensor.cpp:120-195) into a new tensor handle.
void* ref_tensor_load_delimited(const char* path, std::size_t order, int skip_header, int zero_replace,
                                double zero_replacement, std::size_t n_override, const std::uint32_t* dims_override,
                                int* rc) {
  void* out = nullptr;
  *rc = [&]() -> int {
    GUARD_MSG({
      LoadOptions o;
      o.skip_header = skip_header != 0;
      o.zero_policy = zero_replace ? ZeroPolicy::Replace : ZeroPolicy::Reject;
      o.zero_replacement = zero_replacement;
      o.dims_override.assign(dims_override, dims_override + n_override);
      auto* h = new RefTensor;
      h->t = std::make_unique<CooTensor>(CooTensor::load_delimited(path, order, o));
      out = h;
    });
  }();
  return out;
}

int ref_tensor_save_delimited(void* h, const char* path) {
  GUARD_MSG({ static_cast<RefTensor*>(h)->t->save_delimited(path); });
}

// dims (order), nnz; coords/values may be null (query sizes first).
int ref_tensor_get(void* h, std::uint32_t* dims, std::size_t* nnz, std::uint32_t* coords, double* values) {
  GUARD_MSG({
    const CooTensor& t = *static_cast<RefTensor*>(h)->t;
    for (std::size_t k = 0; k < t.order(); ++k) dims[k] = t.shape().dim(k);
    *nnz = t.nnz();
    if (coords)
      for (std::size_t e = 0; e < t.nnz(); ++e) {
        const auto c = t.coord(e);
        std::copy(c.begin(), c.end(), coords + e * t.order());
      }
    if (values) std::copy(t.values().begin(), t.values().end(), values);
  });
}

int ref_model_save(void* h, const char* path) {
  GUARD_MSG({ static_cast<RefModel*>(h)->m->save(path); });
}

// TuckerModel::load (model.cpp:232-280); order/dims/J/R of the loaded model
// are written to the out-params (dims, J sized 64).
void* ref_model_load(const char* path, int* order, std::uint32_t* dims, std::uint32_t* J, std::uint32_t* R,
                     int* rc) {
  void* out = nullptr;
  *rc = [&]() -> int {
    GUARD_MSG({
      auto* h = new RefModel;
      h->m = std::make_unique<TuckerModel>(TuckerModel::load(path));
      *order = static_cast<int>(h->m->order());
      for (std::size_t n = 0; n < h->m->order(); ++n) {
        dims[n] = h->m->shape().dim(n);
        J[n] = h->m->ranks().J[n];
      }
      *R = h->m->ranks().r_core;
      out = h;
    });
  }();
  return out;
}

// write_metrics_csv (eval.cpp:78-97); rows: n x 10 doubles in column order
// (epoch, core_s, factor_s, total_s, train_rmse, train_mae, test_rmse,
// test_mae, peak_bytes, comm_bytes); comments: '\n'-separated.
int ref_write_metrics_csv(const char* path, std::size_t n, const double* rows, const char* comments) {
  GUARD_MSG({
    std::vector<EpochMetrics> r(n);
    for (std::size_t i = 0; i < n; ++i) {
      const double* x = rows + i * 10;
      r[i].epoch = static_cast<std::size_t>(x[0]);
      r[i].core_s = x[1];
      r[i].factor_s = x[2];
      r[i].total_s = x[3];
      r[i].train_rmse = x[4];
      r[i].train_mae = x[5];
      r[i].test_rmse = x[6];
      r[i].test_mae = x[7];
      r[i].peak_bytes = static_cast<std::uint64_t>(x[8]);
      r[i].comm_bytes = static_cast<std::uint64_t>(x[9]);
    }
    std::vector<std::string> c;
    std::string cur;
    for (const char* p = comments; p && *p; ++p) {
      if (*p == '\n') {
        c.push_back(cur);
        cur.clear();
      } else {
        cur += *p;
      }
    }
    if (!cur.empty()) c.push_back(cur);
    write_metrics_csv(path, r, c);
  });
}

// parse_metrics_csv (eval.cpp:99-146): rows out as n x 10 doubles (capacity
// max_rows), comments '\n'-joined into comments_out (capacity cap).
int ref_parse_metrics_csv(const char* path, std::size_t max_rows, double* rows, std::size_t* n,
                          char* comments_out, std::size_t cap) {
  GUARD_MSG({
    std::vector<std::string> c;
    const auto r = parse_metrics_csv(path, &c);
    *n = r.size();
    for (std::size_t i = 0; i < r.size() && i < max_rows; ++i) {
      double* x = rows + i * 10;
      x[0] = static_cast<double>(r[i].epoch);
      x[1] = r[i].core_s;
      x[2] = r[i].factor_s;
      x[3] = r[i].total_s;
      x[4] = r[i].train_rmse;
      x[5] = r[i].train_mae;
      x[6] = r[i].test_rmse;
      x[7] = r[i].test_mae;
      x[8] = static_cast<double>(r[i].peak_bytes);
      x[9] = static_cast<double>(r[i].comm_bytes);
    }
    std::string j;
    for (const auto& s : c) j += s + "\n";
    std::snprintf(comments_out, cap, "%s", j.c_str());
  });
}

// synth_ratings (synth.cpp:83-103).
int ref_synth_ratings(int order, const std::uint32_t* dims, const std::uint32_t* tJ, std::uint32_t tR,
                      std::size_t nnz, double tmean, double tsd, std::uint64_t seed, double target_mean,
                      double target_sd, double noise, int half_steps, double min_v, double max_v,
                      std::uint32_t* coords_out, double* values_out) {
  GUARD_MSG({
    RatingSpec spec;
    spec.base.shape = Shape(std::vector<std::uint32_t>(dims, dims + order));
    spec.base.teacher_ranks = Ranks{std::vector<std::uint32_t>(tJ, tJ + order), tR};
    spec.base.nnz = nnz;
    spec.base.teacher_mean = tmean;
    spec.base.teacher_stddev = tsd;
    spec.base.seed = seed;
    spec.target_mean = target_mean;
    spec.target_stddev = target_sd;
    spec.noise_stddev = noise;
    spec.quantize_half_steps = half_steps != 0;
    spec.min_value = min_v;
    spec.max_value = max_v;
    const CooTensor t = synth_ratings(spec);
    for (std::size_t e = 0; e < t.nnz(); ++e) {
      const auto c = t.coord(e);
      std::copy(c.begin(), c.end(), coords_out + e * order);
      values_out[e] = t.value(e);
    }
  });
}

// unfold_col_index / vec_index / invert_vec_index (sptensor.cpp:40-78).
int ref_indexing(int order, const std::uint32_t* dims, const std::uint32_t* coord, std::size_t mode,
                 std::uint64_t* col, std::uint64_t* vec, std::uint32_t* inv_coord) {
  GUARD_MSG({
    const Shape shape(std::vector<std::uint32_t>(dims, dims + order));
    const std::span<const std::uint32_t> c(coord, static_cast<std::size_t>(order));
    *col = unfold_col_index(shape, c, mode);
    *vec = vec_index(shape, c, mode);
    invert_vec_index(shape, *vec, mode, std::span<std::uint32_t>(inv_coord, static_cast<std::size_t>(order)));
  });
}

}  // extern "C"
