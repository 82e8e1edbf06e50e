// multi_gpu.cpp -- train() over several GPUs of one node from one process
// (HyperParams::devices): one sharded device session per rank, driven in
// lockstep by this host thread.  Every call below only enqueues work; the
// ranks are ordered by sgdt_stream_barrier (each stream waits on the others'
// events), so no host round trip sits between the phases and no kernel ever
// waits on another.
//
// Reference: train() (trainer.cpp:66-125) with the improved strategy's
// worker slices (factor_optimizer.cpp:209-270, scheduler.cpp:34-46) mapped
// onto ranks:
//   core phase    replicated (every rank runs the identical kernel on the
//                 identical Psi and model), or sharded (Psi sliced by
//                 partition_even(M, P); per column block the B^(n)-gradient
//                 vectors go into every rank's exchange slots and are summed
//                 in rank order -- sgdt.h "sharded core phase");
//   factor phase  each rank finalises the rows inside its slice of every
//                 mode order and stores them into every rank's A/Q (peer
//                 stores); the <= 2 cut rows per rank are merged in rank order.
// Epoch metrics use the host clock around each phase (a synchronisation per
// phase, as the reference's own timers) and rank 0's RMSE.
#include <chrono>
#include <cmath>
#include <limits>
#include <string>
#include <vector>

#include "device.hpp"
#include "sptucker/trainer.hpp"

namespace sptucker::detail {

namespace {

struct ShardGroup {
  std::vector<sgdt_session*> s;
  ~ShardGroup() {
    for (sgdt_session* x : s)
      if (x) sgdt_session_destroy(x);
  }
  void barrier() { check(sgdt_stream_barrier(s.data(), static_cast<int>(s.size())), "multi-GPU barrier"); }
  void sync() {
    for (sgdt_session* x : s) check(sgdt_synchronize(x), "multi-GPU synchronize");
  }
};

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

TrainResult train_multi_gpu(TuckerModel& model, const CooTensor& train_set, const CooTensor* test_set,
                            const HyperParams& hyper) {
  const int P = static_cast<int>(hyper.devices.size());
  const std::size_t N = model.order();
  std::vector<std::uint32_t> dims = model.shape().dims();
  std::vector<const std::uint32_t*> p1, p2;
  const sgdt_tensor_desc dtr = describe(train_set, dims, p1);
  sgdt_tensor_desc dte{};
  if (test_set) dte = describe(*test_set, dims, p2);

  check(sgdt_enable_peer_access(hyper.devices.data(), P), "multi-GPU peer access");
  ShardGroup g;
  g.s.assign(P, nullptr);
  for (int r = 0; r < P; ++r)
    check(sgdt_session_create_shard(&dtr, test_set ? &dte : nullptr, model.ranks().J.data(), model.ranks().r_core,
                                    hyper.devices[r], r, P, &g.s[r]),
          "multi-GPU session");
  // every rank's peer-visible buffers, rank-major
  const std::size_t per = 2 * N + 2;
  std::vector<void*> table(static_cast<std::size_t>(P) * per, nullptr);
  for (int r = 0; r < P; ++r) check(sgdt_peer_buffers(g.s[r], table.data() + r * per), "multi-GPU peers");
  for (int r = 0; r < P; ++r) check(sgdt_set_peers(g.s[r], const_cast<const void* const*>(table.data())), "multi-GPU peers");

  // identical model, batch stream (trainer.cpp:72) and fresh pool on every rank
  std::vector<const double*> a(N), b(N);
  for (std::size_t n = 0; n < N; ++n) {
    a[n] = model.factor(n).data().data();
    b[n] = model.kruskal(n).data().data();
  }
  const Rng rng(hyper.seed + 1);
  for (int r = 0; r < P; ++r) {
    check(sgdt_set_model(g.s[r], a.data(), b.data()), "multi-GPU model");
    check(sgdt_set_rng(g.s[r], rng.state_words().data(), rng.state_pos()), "multi-GPU rng");
    check(sgdt_reset_pool(g.s[r]), "multi-GPU pool");
  }
  g.barrier();

  const sgdt_core_hyper ch{hyper.lr_b, hyper.reg_b, hyper.batch_m, hyper.resample_core_batch ? 1 : 0,
                           hyper.incremental_residual ? 1 : 0};
  const sgdt_factor_hyper fh{hyper.lr_a, hyper.reg_a, hyper.row_fraction};
  const CommCost comm = comm_cost_report(Ranks{hyper.ranks, hyper.r_core});
  TrainResult res;
  res.peak_workspace_bytes = sgdt_workspace_bytes(g.s[0]);
  for (std::size_t e = 0; e < hyper.epochs; ++e) {
    EpochMetrics m;
    m.epoch = e + 1;
    // ---- core phase
    auto t0 = std::chrono::steady_clock::now();
    if (hyper.core_sharded) {
      std::uint32_t steps = 0, st = 0, T = 0;
      for (int r = 0; r < P; ++r) {
        check(sgdt_core_plan(g.s[r], &ch, 0, &st, &T), "update_core_epoch");
        if (r == 0) steps = st;
        if (st != steps) throw InternalError("multi-GPU: ranks planned different core steps");
      }
      for (std::uint32_t k = 0; k < steps; ++k) {
        for (int r = 0; r < P; ++r) check(sgdt_core_step(g.s[r], k), "update_core_epoch");
        if (k + 1 < steps) g.barrier();
      }
    } else {
      for (int r = 0; r < P; ++r) check(sgdt_core_epoch_async(g.s[r], &ch), "update_core_epoch");
    }
    g.sync();
    m.core_s = seconds_since(t0);
    // ---- factor phase (the leading barrier orders the peers' row stores
    // after every rank's core phase, which reads A and rewrites Q)
    t0 = std::chrono::steady_clock::now();
    g.barrier();
    for (std::size_t n = 0; n < N; ++n) {
      for (int r = 0; r < P; ++r) check(sgdt_factor_mode_p2p(g.s[r], static_cast<int>(n), &fh), "update_factor_epoch");
      g.barrier();
      for (int r = 0; r < P; ++r) check(sgdt_factor_merge_p2p(g.s[r], static_cast<int>(n), &fh), "update_factor_epoch");
      g.barrier();
    }
    for (int r = 0; r < P; ++r) {
      const int rc = sgdt_check(g.s[r]);
      if (rc == SGDT_ERR_NUMERIC)
        throw NumericError("training diverged at epoch " + std::to_string(e + 1) + "; reduce the learning rates");
      check(rc, "train");
    }
    m.factor_s = seconds_since(t0);
    m.total_s = m.core_s + m.factor_s;
    // ---- metrics on rank 0 (its A/Q hold every rank's rows)
    check(sgdt_eval(g.s[0], 0, &m.train_rmse, &m.train_mae), "rmse_mae");
    if (test_set) {
      check(sgdt_eval(g.s[0], 1, &m.test_rmse, &m.test_mae), "rmse_mae");
    } else {
      m.test_rmse = m.test_mae = std::numeric_limits<double>::quiet_NaN();
    }
    m.peak_bytes = res.peak_workspace_bytes;
    m.comm_bytes = 8 * comm.kruskal_params;
    res.metrics.push_back(m);
  }
  std::vector<double*> ao(N), bo(N);
  for (std::size_t n = 0; n < N; ++n) {
    ao[n] = model.factor(n).data().data();
    bo[n] = model.kruskal(n).data().data();
  }
  check(sgdt_get_model(g.s[0], ao.data(), bo.data()), "download model");
  model.refresh_core_cache();
  std::size_t skipped = 0;
  for (std::size_t n = 0; n < train_set.order(); ++n) {
    const auto& off = train_set.mode_offsets(n);
    for (std::size_t i = 1; i < off.size(); ++i) skipped += off[i] == off[i - 1];
  }
  res.rows_skipped_last_epoch = skipped;
  return res;
}

}  // namespace sptucker::detail
