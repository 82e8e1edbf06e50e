// eval_trainer.cpp -- rmse_mae and train() on the device; small host utilities.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <limits>
#include <thread>

#include "device.hpp"
#include "sptucker/core_optimizer.hpp"
#include "sptucker/eval.hpp"
#include "sptucker/factor_optimizer.hpp"
#include "sptucker/trainer.hpp"

namespace sptucker {

std::pair<double, double> rmse_mae(const TuckerModel& model, const CooTensor& entries) {
  if (entries.order() != model.order()) throw DomainError("rmse_mae: order mismatch between model and data");
  for (std::size_t n = 0; n < model.order(); ++n)
    if (entries.shape().dim(n) > model.shape().dim(n))
      throw DomainError("rmse_mae: data exceeds the model's shape in mode " + std::to_string(n + 1));
  detail::Session& s = detail::session_for(entries, nullptr, model.shape(), model.ranks());
  s.sync_model(model);
  double rmse = 0.0, mae = 0.0;
  detail::check(sgdt_eval(s.get(), 0, &rmse, &mae), "rmse_mae");
  return {rmse, mae};
}

CommCost comm_cost_report(const Ranks& ranks) {
  CommCost c;
  c.dense_core_params = 1;
  for (const std::uint32_t j : ranks.J) {
    c.dense_core_params *= j;
    c.kruskal_params += static_cast<std::uint64_t>(j) * ranks.r_core;
  }
  c.ratio = static_cast<double>(c.dense_core_params) / static_cast<double>(c.kruskal_params);
  return c;
}

LinearFit fit_linear(const std::vector<double>& x, const std::vector<double>& y) {
  if (x.size() != y.size()) throw InternalError("fit_linear: length mismatch");
  LinearFit f;
  const std::size_t n = x.size();
  if (n < 2) {
    f.degenerate = true;
    return f;
  }
  double mx = 0.0, my = 0.0;
  for (std::size_t i = 0; i < n; ++i) {
    mx += x[i];
    my += y[i];
  }
  mx /= static_cast<double>(n);
  my /= static_cast<double>(n);
  double sxx = 0.0, sxy = 0.0, syy = 0.0;
  for (std::size_t i = 0; i < n; ++i) {
    sxx += (x[i] - mx) * (x[i] - mx);
    sxy += (x[i] - mx) * (y[i] - my);
    syy += (y[i] - my) * (y[i] - my);
  }
  if (sxx == 0.0) {
    f.degenerate = true;
    return f;
  }
  f.slope = sxy / sxx;
  f.intercept = my - f.slope * mx;
  f.r2 = syy == 0.0 ? 1.0 : sxy * sxy / (sxx * syy);
  return f;
}

std::vector<double> timed_epoch_seconds(const CooTensor& train, const Ranks& ranks, const BenchOptions& opts,
                                        double init_mean, double init_stddev, std::uint64_t* workspace_bytes) {
  TuckerModel model = TuckerModel::init_gaussian(train.shape(), ranks, init_mean, init_stddev, opts.seed);
  Rng rng(opts.seed + 1);
  const CoreHyper core{opts.lr_b, opts.reg, opts.batch_m, false, false};
  const FactorHyper factor{opts.lr_a, opts.reg, 1.0};
  WorkerPool pool(std::max<std::size_t>(1, opts.threads));
  const SchedContext sched{opts.threads <= 1 ? Strategy::Serial : opts.strategy, BalancePolicy::Dynamic,
                           opts.threads <= 1 ? nullptr : &pool};
  CoreBatchWorkspace core_ws;
  std::vector<RowBatchWorkspace> row_ws(sched.workers());
  std::vector<double> seconds;
  for (std::size_t ep = 0; ep < opts.warmup + opts.epochs; ++ep) {
    const auto t0 = std::chrono::steady_clock::now();
    update_core_epoch(model, train, core, sched, rng, core_ws);
    update_factor_epoch(model, train, factor, sched, rng, row_ws);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (ep >= opts.warmup) seconds.push_back(s);
  }
  if (workspace_bytes) {
    *workspace_bytes = core_ws.bytes();
    for (const auto& ws : row_ws) *workspace_bytes += ws.bytes();
  }
  return seconds;
}

namespace {
double median_of(std::vector<double> v) {
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  const std::size_t k = v.size();
  return k % 2 ? v[k / 2] : 0.5 * (v[k / 2 - 1] + v[k / 2]);
}
}  // namespace

RankScalingResult bench_rank_scaling(const CooTensor& train, const std::vector<Ranks>& grid,
                                     const std::vector<std::uint32_t>& x_values, const BenchOptions& opts) {
  if (grid.size() != x_values.size()) throw DomainError("bench_rank_scaling: grid and x values differ in length");
  RankScalingResult out;
  std::vector<double> xs, times, bytes;
  for (std::size_t i = 0; i < grid.size(); ++i) {
    std::uint64_t ws_bytes = 0;
    const double secs = median_of(timed_epoch_seconds(train, grid[i], opts, 0.5, 0.1, &ws_bytes));
    out.rows.push_back({x_values[i], secs, ws_bytes});
    xs.push_back(static_cast<double>(x_values[i]));
    times.push_back(secs);
    bytes.push_back(static_cast<double>(ws_bytes));
  }
  out.time_fit = fit_linear(xs, times);
  out.bytes_fit = fit_linear(xs, bytes);
  return out;
}

std::vector<SpeedupRow> bench_speedup(const CooTensor& train, const Ranks& ranks,
                                      const std::vector<std::size_t>& thread_grid, const BenchOptions& opts) {
  std::vector<SpeedupRow> out;
  double t1 = 0.0;
  for (const std::size_t threads : thread_grid) {
    BenchOptions o = opts;
    o.threads = threads;
    const double secs = median_of(timed_epoch_seconds(train, ranks, o, 0.5, 0.1));
    if (threads == 1 && t1 == 0.0) t1 = secs;
    SpeedupRow row;
    row.threads = threads;
    row.seconds_per_epoch = secs;
    row.speedup = (threads == 1 && secs == t1) ? 1.0 : (t1 > 0.0 ? t1 / secs : 0.0);
    row.efficiency = row.speedup / static_cast<double>(threads);
    out.push_back(row);
  }
  return out;
}

void HyperParams::validate() const {
  try {
    if (ranks.empty()) throw ConfigError("ranks must be given");
    Ranks{ranks, r_core}.validate(ranks.size());
  } catch (const DomainError& e) {
    throw ConfigError(e.what());
  }
  // The reference also caps prod J_n at kMaxCoreElems (trainer.cpp:16-18)
  // because its factor phase reads the dense core; the device path never
  // builds it, so the cap is lifted (deviations).
  if (r_core > SGDT_MAX_RCORE) throw ConfigError("R_core above 32 is not supported by the device kernels");
  if (devices.size() > 8) throw ConfigError("at most 8 devices (one node)");
  if (devices.size() > 1 && row_fraction < 1.0)
    throw ConfigError("row fraction < 1 is not supported by the multi-GPU path");
  for (const std::uint32_t j : ranks)
    if (j > SGDT_MAX_J) throw ConfigError("J_n above 64 is not supported by the device kernels");
  if (!(lr_a > 0.0) || !(lr_b > 0.0)) throw ConfigError("learning rates must be positive");
  if (reg_a < 0.0 || reg_b < 0.0) throw ConfigError("regularization must be non-negative");
  if (epochs < 1) throw ConfigError("epochs must be >= 1");
  if (!(row_fraction > 0.0 && row_fraction <= 1.0)) throw ConfigError("row fraction must lie in (0,1]");
  if (!(init_stddev > 0.0)) throw ConfigError("init stddev must be positive");
}

std::size_t HyperParams::effective_threads() const {
  if (threads > 0) return threads;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw == 0 ? 1 : hw;
}

std::vector<std::string> HyperParams::describe() const {
  auto g = [](double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%g", v);
    return std::string(b);
  };
  std::string rl;
  for (std::size_t i = 0; i < ranks.size(); ++i) rl += (i ? "," : "") + std::to_string(ranks[i]);
  return {"ranks = " + rl,
          "rcore = " + std::to_string(r_core),
          "lr-a = " + g(lr_a),
          "lr-b = " + g(lr_b),
          "reg-a = " + g(reg_a),
          "reg-b = " + g(reg_b),
          "batch-m = " + std::to_string(batch_m),
          "row-fraction = " + g(row_fraction),
          "epochs = " + std::to_string(epochs),
          "seed = " + std::to_string(seed),
          "threads = " + std::to_string(effective_threads()),
          "strategy = " + to_string(strategy),
          "balance = " + to_string(balance),
          "init-mean = " + g(init_mean),
          "init-stddev = " + g(init_stddev),
          "resample-core-batch = " + std::string(resample_core_batch ? "true" : "false"),
          "incremental-residual = " + std::string(incremental_residual ? "true" : "false"),
          "device = " + std::to_string(device),
          "devices = " + [&] {
            std::string d;
            for (std::size_t i = 0; i < devices.size(); ++i) d += (i ? "," : "") + std::to_string(devices[i]);
            return d;
          }(),
          "core-sharded = " + std::string(core_sharded ? "true" : "false")};
}

TrainResult train(TuckerModel& model, const CooTensor& train_set, const CooTensor* test_set, const HyperParams& hyper,
                  WorkerPool* /*pool: the device does the parallel work*/) {
  hyper.validate();
  if (hyper.ranks.size() != train_set.order()) throw ConfigError("ranks arity does not match tensor order");
  if (model.ranks().J != hyper.ranks || model.ranks().r_core != hyper.r_core)
    throw ConfigError("model ranks do not match the hyper-parameters");
  if (test_set) {
    if (test_set->order() != model.order()) throw DomainError("rmse_mae: order mismatch between model and data");
    for (std::size_t n = 0; n < model.order(); ++n)
      if (test_set->shape().dim(n) > model.shape().dim(n))
        throw DomainError("rmse_mae: data exceeds the model's shape in mode " + std::to_string(n + 1));
  }

  if (hyper.devices.size() > 1) return detail::train_multi_gpu(model, train_set, test_set, hyper);
  detail::Session& s = detail::session_for(train_set, test_set, model.shape(), model.ranks(), hyper.device);
  s.sync_model(model);
  Rng rng(hyper.seed + 1);  // batch stream, trainer.cpp:72
  s.put_rng(rng);
  detail::check(sgdt_reset_pool(s.get()), "train");  // fresh workspace: pool restarts from iota

  const sgdt_core_hyper ch{hyper.lr_b, hyper.reg_b, hyper.batch_m, hyper.resample_core_batch ? 1 : 0,
                           hyper.incremental_residual ? 1 : 0};
  const sgdt_factor_hyper fh{hyper.lr_a, hyper.reg_a, hyper.row_fraction};
  std::vector<double> met(hyper.epochs * 6);
  detail::check(sgdt_train(s.get(), &ch, &fh, hyper.epochs, met.data()), "train");
  s.take_model(model);

  const CommCost comm = comm_cost_report(Ranks{hyper.ranks, hyper.r_core});
  std::size_t skipped = 0;
  for (std::size_t n = 0; n < train_set.order(); ++n) {
    const auto& off = train_set.mode_offsets(n);
    for (std::size_t i = 1; i < off.size(); ++i) skipped += off[i] == off[i - 1];
  }
  TrainResult res;
  res.peak_workspace_bytes = sgdt_workspace_bytes(s.get());
  for (std::size_t e = 0; e < hyper.epochs; ++e) {
    const double* r = met.data() + e * 6;
    EpochMetrics m;
    m.epoch = e + 1;
    m.core_s = r[0];
    m.factor_s = r[1];
    m.total_s = m.core_s + m.factor_s;
    m.train_rmse = r[2];
    m.train_mae = r[3];
    m.test_rmse = test_set ? r[4] : std::numeric_limits<double>::quiet_NaN();
    m.test_mae = test_set ? r[5] : std::numeric_limits<double>::quiet_NaN();
    m.peak_bytes = res.peak_workspace_bytes;
    m.comm_bytes = 8 * comm.kruskal_params;
    res.metrics.push_back(m);
  }
  res.rows_skipped_last_epoch = skipped;
  return res;
}

std::pair<TuckerModel, TrainResult> train_from_scratch(const CooTensor& train_set, const CooTensor* test_set,
                                                       const HyperParams& hyper) {
  hyper.validate();
  if (hyper.ranks.size() != train_set.order()) throw ConfigError("ranks arity does not match tensor order");
  TuckerModel model = TuckerModel::init_gaussian(train_set.shape(), Ranks{hyper.ranks, hyper.r_core},
                                                 hyper.init_mean, hyper.init_stddev, hyper.seed);
  WorkerPool pool(1);
  TrainResult r = train(model, train_set, test_set, hyper, &pool);
  return {std::move(model), std::move(r)};
}

}  // namespace sptucker
