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

 private:
  sgdt_session* h_ = nullptr;
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

// The cached session of `train` for (test, shape, ranks), created on first use.
Session& session_for(const CooTensor& train, const CooTensor* test, const Shape& shape, const Ranks& ranks,
                     int device = -1);

}  // namespace sptucker::detail
