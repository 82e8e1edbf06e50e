// bench_shim.cpp -- the bench driver's end-to-end leg through the C++ drop-in.
//
// bench.py (Python) cannot call the C++ API directly, so this small extern "C"
// entry point does what a reference caller does: it builds a
// sptucker::CooTensor from host arrays (the constructor's checks and bucket
// sorts run on the device, sgdt_tensor_layout) and runs the reference's
// timed_epochs loop (eval.cpp:201-223) -- update_core_epoch +
// update_factor_epoch on a host TuckerModel per epoch, host wall clock -- on
// libsptucker_b200.so.  It also reports the host<->device bytes the per-epoch
// calls moved during the timed epochs (model, pool and batch traffic).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../src/device.hpp"
#include "sptucker/core_optimizer.hpp"
#include "sptucker/eval.hpp"
#include "sptucker/factor_optimizer.hpp"

using namespace sptucker;

extern "C" int sptb_timed_epochs(int order, const std::uint32_t* dims, std::uint64_t nnz, const std::uint32_t* coords,
                                 const double* values, const std::uint32_t* J, std::uint32_t R, double lr_a,
                                 double lr_b, double reg, std::uint64_t batch_m, std::uint64_t warmup,
                                 std::uint64_t epochs, std::uint64_t seed, double init_mean, double init_sd,
                                 double* secs_out, std::uint64_t* h2d_bytes, std::uint64_t* d2h_bytes,
                                 double* build_s, char* err, std::size_t errlen) {
  try {
    const auto t0 = std::chrono::steady_clock::now();
    CooTensor train(Shape(std::vector<std::uint32_t>(dims, dims + order)),
                    std::vector<std::uint32_t>(coords, coords + nnz * order), std::vector<double>(values, values + nnz));
    *build_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const Ranks ranks{std::vector<std::uint32_t>(J, J + order), R};
    TuckerModel model = TuckerModel::init_gaussian(train.shape(), ranks, init_mean, init_sd, seed);
    Rng rng(seed + 1);
    const CoreHyper core{lr_b, reg, batch_m, false, false};
    const FactorHyper factor{lr_a, reg, 1.0};
    WorkerPool pool(1);
    const SchedContext sched{Strategy::Serial, BalancePolicy::Dynamic, nullptr};
    CoreBatchWorkspace core_ws;
    std::vector<RowBatchWorkspace> row_ws(1);
    std::uint64_t h0 = 0, d0 = 0;
    for (std::uint64_t ep = 0; ep < warmup + epochs; ++ep) {
      if (ep == warmup) {
        detail::Session& s = detail::session_for(train, nullptr, train.shape(), ranks);
        h0 = s.h2d_bytes;
        d0 = s.d2h_bytes;
      }
      const auto a = std::chrono::steady_clock::now();
      update_core_epoch(model, train, core, sched, rng, core_ws);
      update_factor_epoch(model, train, factor, sched, rng, row_ws);
      const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
      if (ep >= warmup) secs_out[ep - warmup] = sec;
    }
    detail::Session& s = detail::session_for(train, nullptr, train.shape(), ranks);
    *h2d_bytes = s.h2d_bytes - h0;
    *d2h_bytes = s.d2h_bytes - d0;
    return 0;
  } catch (const std::exception& e) {
    std::strncpy(err, e.what(), errlen - 1);
    err[errlen - 1] = 0;
    return 1;
  }
}
