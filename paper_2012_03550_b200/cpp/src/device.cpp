// device.cpp -- C++ API <-> C-ABI bridge: sessions, model/RNG transfer and
// the error-code mapping (include/sgdt.h codes -> sptucker exceptions).
#include "device.hpp"

#include <algorithm>
#include <atomic>
#include <barrier>
#include <numeric>
#include <string>
#include <thread>

namespace sptucker::detail {

void throw_for(int code, const std::string& where) {
  const std::string msg = where + ": " + sgdt_last_error();
  switch (code) {
    case SGDT_ERR_CONFIG: throw ConfigError(msg);
    case SGDT_ERR_DATA: throw DataError(msg);
    case SGDT_ERR_NUMERIC: throw NumericError(msg);
    case SGDT_ERR_DOMAIN: throw DomainError(msg);
    default: throw InternalError(msg);
  }
}

sgdt_tensor_desc describe(const CooTensor& t, const std::vector<std::uint32_t>& dims,
                          std::vector<const std::uint32_t*>& perms) {
  perms.resize(t.order());
  for (std::size_t n = 0; n < t.order(); ++n) perms[n] = t.mode_perm(n).data();
  sgdt_tensor_desc d{};
  d.order = static_cast<int>(t.order());
  d.dims = dims.data();
  d.nnz = t.nnz();
  d.coords = t.coords().data();
  d.values = t.values().data();
  d.mode_perm = perms.data();
  return d;
}

namespace {
std::uint64_t model_bytes(const TuckerModel& m, bool factors, bool kruskal) {
  std::uint64_t b = 0;
  for (std::size_t n = 0; n < m.order(); ++n)
    b += (factors ? m.factor(n).size() : 0) + (kruskal ? m.kruskal(n).size() : 0);
  return b * sizeof(double);
}
}  // namespace

Session::Session(const CooTensor& train, const CooTensor* test, const Shape& shape, const Ranks& ranks,
                 int device)
    : test_(test), test_nnz_(test ? test->nnz() : 0), dims_(shape.dims()), J_(ranks.J), R_(ranks.r_core),
      device_(device) {
  std::vector<const std::uint32_t*> p1, p2;
  const sgdt_tensor_desc dtr = describe(train, dims_, p1);
  sgdt_tensor_desc dte{};
  if (test) dte = describe(*test, dims_, p2);
  check(sgdt_session_create(&dtr, test ? &dte : nullptr, J_.data(), R_, device, &h_), "device session");
}

Session::~Session() {
  if (h_) sgdt_session_destroy(h_);
}

bool Session::matches(const CooTensor* test, const Shape& shape, const Ranks& ranks, int device) const {
  return test == test_ && (test ? test->nnz() : 0) == test_nnz_ && shape.dims() == dims_ && ranks.J == J_ &&
         ranks.r_core == R_ && device == device_;
}

void Session::put_model(const TuckerModel& m) {
  std::vector<const double*> a(m.order()), b(m.order());
  for (std::size_t n = 0; n < m.order(); ++n) {
    a[n] = m.factor(n).data().data();
    b[n] = m.kruskal(n).data().data();
  }
  check(sgdt_set_model(h_, a.data(), b.data()), "upload model");
}

void Session::take_model(TuckerModel& m, bool factors, bool kruskal) {
  std::vector<double*> a(m.order()), b(m.order());
  for (std::size_t n = 0; n < m.order(); ++n) {
    if (factors) a[n] = m.factor(n).data().data();
    if (kruskal) b[n] = m.kruskal(n).data().data();
  }
  check(sgdt_get_model(h_, factors ? a.data() : nullptr, kruskal ? b.data() : nullptr), "download model");
  d2h_bytes += model_bytes(m, factors, kruskal);
  if (kruskal) m.refresh_core_cache();
  mark_synced(m);
}

void Session::sync_model(const TuckerModel& m) {
  if (synced_model_ == &m && synced_gen_ == m.generation()) return;
  put_model(m);
  h2d_bytes += model_bytes(m, true, true);
  mark_synced(m);
}

void Session::mark_synced(const TuckerModel& m) {
  synced_model_ = &m;
  synced_gen_ = m.generation();
}

sgdt_factor_stats Session::factor_epoch_into(TuckerModel& m, const sgdt_factor_hyper& h) {
  std::vector<double*> a(m.order());
  for (std::size_t n = 0; n < m.order(); ++n) a[n] = m.factor(n).data().data();
  sgdt_factor_stats st{};
  const int rc = sgdt_factor_epoch_host(h_, &h, a.data(), &st);
  if (rc == SGDT_OK || rc == SGDT_ERR_NUMERIC) {
    if (h.lr > 0.0) d2h_bytes += model_bytes(m, true, false);
    mark_synced(m);  // the host A is what the device holds, even on divergence
  }
  check(rc, "update_factor_epoch");
  return st;
}

void Session::sync_pool(const std::vector<std::uint32_t>& pool, bool force) {
  check(sgdt_set_pool_capture(h_, 1), "update_core_epoch");
  if (!force && pool.data() == pool_data_ && pool.size() == pool_size_) return;
  check(sgdt_set_pool(h_, pool.data()), "update_core_epoch");
  h2d_bytes += pool.size() * sizeof(std::uint32_t);
  pool_data_ = pool.data();
  pool_size_ = pool.size();
}

void Session::pool_reset(const std::vector<std::uint32_t>& iota_pool) {
  check(sgdt_set_pool_capture(h_, 1), "update_core_epoch");
  check(sgdt_reset_pool(h_), "update_core_epoch");
  pool_data_ = iota_pool.data();
  pool_size_ = iota_pool.size();
}

namespace {
// Runs f(thread, lo, hi) over [0, n) on up to 16 host threads; f may call
// sync() to wait for every thread (a phase barrier).  Random access into the
// pool is latency bound, so threads pay off long before bandwidth does.
class Phased {
 public:
  explicit Phased(std::size_t n)
      : n_(n), t_(std::min<std::size_t>({std::max<std::size_t>(1, std::thread::hardware_concurrency()), 16,
                                         std::max<std::size_t>(1, n / 8192)})),
        bar_(static_cast<std::ptrdiff_t>(t_)) {}
  template <class F>
  void run(F f) {
    std::vector<std::thread> th;
    th.reserve(t_ - 1);
    for (std::size_t k = 1; k < t_; ++k) th.emplace_back([&, k] { f(n_ * k / t_, n_ * (k + 1) / t_); });
    f(std::size_t{0}, n_ / t_);
    for (std::thread& x : th) x.join();
  }
  void sync() { bar_.arrive_and_wait(); }

 private:
  std::size_t n_, t_;
  std::barrier<> bar_;
};
}  // namespace

bool Session::pool_apply_checked(std::vector<std::uint32_t>& pool, const std::vector<std::uint32_t>& batch) {
  std::uint64_t n = 0;
  const std::uint32_t *pos = nullptr, *val = nullptr, *pre_j = nullptr, *pre_lo = nullptr;
  if (sgdt_pool_delta_view(h_, &pos, &val, &pre_j, &pre_lo, &n) != SGDT_OK) {
    // several runs (resample_per_mode): the pool was uploaded before the
    // call, so the device pool is the truth -- take all of it
    check(sgdt_get_pool(h_, pool.data()), "update_core_epoch");
    d2h_bytes += pool.size() * sizeof(std::uint32_t);
    pool_data_ = pool.data();
    pool_size_ = pool.size();
    return true;
  }
  d2h_bytes += 4 * n * sizeof(std::uint32_t);
  if (n != batch.size()) throw InternalError("pool delta: batch size mismatch");
  // phase 1: the host pool must hold what the device read at every read
  // position; phase 2 (only if so): the run's writes -- the touched positions
  // (a position drawn twice gets the same final value from both draws), then
  // the batch at 0..m-1
  std::atomic<bool> same{true};
  Phased ph(n);
  ph.run([&](std::size_t lo, std::size_t hi) {
    bool ok = true;
    for (std::size_t i = lo; i < hi && ok; ++i) ok = pool[i] == pre_lo[i] && pool[pos[i]] == pre_j[i];
    if (!ok) same.store(false, std::memory_order_relaxed);
    ph.sync();
    if (!same.load(std::memory_order_relaxed)) return;
    for (std::size_t i = lo; i < hi; ++i) std::atomic_ref<std::uint32_t>(pool[pos[i]]).store(val[i], std::memory_order_relaxed);
    ph.sync();
    std::copy(batch.begin() + lo, batch.begin() + hi, pool.begin() + lo);
  });
  if (!same.load()) return false;
  pool_data_ = pool.data();
  pool_size_ = pool.size();
  return true;
}

void Session::put_rng(const Rng& r) {
  check(sgdt_set_rng(h_, r.state_words().data(), r.state_pos()), "rng");
  h2d_bytes += Rng::kWords * sizeof(std::uint64_t) + sizeof(std::uint32_t);
}

void Session::take_rng(Rng& r) {
  std::uint64_t words[Rng::kWords];
  std::uint32_t pos = 0;
  check(sgdt_get_rng(h_, words, &pos), "rng");
  d2h_bytes += Rng::kWords * sizeof(std::uint64_t) + sizeof(std::uint32_t);
  r.set_state(words, pos);
}

Session& session_for(const CooTensor& train, const CooTensor* test, const Shape& shape, const Ranks& ranks,
                     int device) {
  DeviceCache& c = train.device_cache();
  std::lock_guard<std::mutex> lock(c.mu);
  for (auto& s : c.sessions)
    if (s->matches(test, shape, ranks, device)) return *s;
  c.sessions.push_back(std::make_unique<Session>(train, test, shape, ranks, device));
  return *c.sessions.back();
}

}  // namespace sptucker::detail
