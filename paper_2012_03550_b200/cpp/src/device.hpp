// device.hpp -- the bridge from the sptucker C++ API to the C-ABI (sgdt.h).
#pragma once

#include <memory>
#include <mutex>
#include <vector>

#include "../../../include/sgdt.h"
#include "sptucker/model.hpp"
#include "sptucker/rng.hpp"
#include "sptucker/sptensor.hpp"

namespace sptucker::detail {

// One device session = one uploaded training tensor (+ optional test tensor)
// sized for one (shape, ranks).  Owned by the tensor's DeviceCache.
class Session {
 public:
  Session(const CooTensor& train, const CooTensor* test, const Shape& shape, const Ranks& ranks, int device);
  ~Session();
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  sgdt_session* get() const { return h_; }
  bool matches(const CooTensor* test, const Shape& shape, const Ranks& ranks, int device) const;

  void put_model(const TuckerModel& m);
  void take_model(TuckerModel& m, bool factors = true, bool kruskal = true);
  void put_rng(const Rng& r);
  void take_rng(Rng& r);

  // Device residency across the per-epoch calls: the session remembers which
  // model (object and generation) its device copy equals and uploads only
  // when that changed; after a phase it downloads only what the phase wrote
  // (B after the core phase, A -- overlapped with the later modes -- after
  // the factor phase) and records the new generation.
  void sync_model(const TuckerModel& m);
  void mark_synced(const TuckerModel& m);
  // The factor epoch with the A^(n) copy-out overlapped (sgdt_factor_epoch_host).
  sgdt_factor_stats factor_epoch_into(TuckerModel& m, const sgdt_factor_hyper& h);
  // The persistent sample pool.  The device copy is the one this session
  // last wrote; it is re-uploaded when the host vector is another buffer or
  // size (or `force`).  After a single sampler run, pool_apply_checked()
  // replays the run on the host pool (the partial Fisher-Yates swaps over the
  // device's draw targets, sptensor.cpp:256-270) and compares the result with
  // the device's batch and touched positions.  A swap is a permutation of
  // positions, so equality there means the host and device pools agreed at
  // every position the run read: host edits between calls are either outside
  // the run's read set (and are checked by a later run) or detected.  On a
  // mismatch the host pool is restored and false is returned; the caller
  // uploads the host pool and repeats the call.
  void sync_pool(const std::vector<std::uint32_t>& pool, bool force = false);
  void pool_reset(const std::vector<std::uint32_t>& iota_pool);  // the host pool was just set to iota
  bool pool_apply_checked(std::vector<std::uint32_t>& pool, const std::vector<std::uint32_t>& batch);

  std::uint64_t h2d_bytes = 0, d2h_bytes = 0;  // model / pool / batch traffic of the per-epoch calls

 private:
  sgdt_session* h_ = nullptr;
  const TuckerModel* synced_model_ = nullptr;
  std::uint64_t synced_gen_ = 0;
  const std::uint32_t* pool_data_ = nullptr;
  std::size_t pool_size_ = 0;
  const CooTensor* test_ = nullptr;
  std::size_t test_nnz_ = 0;
  std::vector<std::uint32_t> dims_, J_;
  std::uint32_t R_ = 0;
  int device_ = -1;
};

struct DeviceCache {
  std::mutex mu;
  std::vector<std::unique_ptr<Session>> sessions;
};

// The C-ABI descriptor of a tensor (perms receives the per-mode orders).
sgdt_tensor_desc describe(const CooTensor& t, const std::vector<std::uint32_t>& dims,
                          std::vector<const std::uint32_t*>& perms);

}  // namespace sptucker::detail
namespace sptucker {
struct HyperParams;
struct TrainResult;
}  // namespace sptucker
namespace sptucker::detail {
// train() over HyperParams::devices (multi_gpu.cpp).
TrainResult train_multi_gpu(TuckerModel& model, const CooTensor& train_set, const CooTensor* test_set,
                            const HyperParams& hyper);

// The cached session of `train` for (test, shape, ranks), created on first use.
Session& session_for(const CooTensor& train, const CooTensor* test, const Shape& shape, const Ranks& ranks,
                     int device = -1);

}  // namespace sptucker::detail
