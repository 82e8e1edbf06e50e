// device.cpp -- C++ API <-> C-ABI bridge: sessions, model/RNG transfer and
// the error-code mapping (include/sgdt.h codes -> sptucker exceptions).
#include "device.hpp"

#include <algorithm>
#include <numeric>
#include <string>

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
  if (!force && pool.data() == pool_data_ && pool.size() == pool_size_) return;
  check(sgdt_set_pool(h_, pool.data()), "update_core_epoch");
  h2d_bytes += pool.size() * sizeof(std::uint32_t);
  pool_data_ = pool.data();
  pool_size_ = pool.size();
}

void Session::pool_reset(const std::vector<std::uint32_t>& iota_pool) {
  check(sgdt_reset_pool(h_), "update_core_epoch");
  pool_data_ = iota_pool.data();
  pool_size_ = iota_pool.size();
}

bool Session::pool_apply_checked(std::vector<std::uint32_t>& pool, const std::vector<std::uint32_t>& batch) {
  const std::size_t m = batch.size();
  std::vector<std::uint32_t> pos(m), val(m);
  std::uint64_t n = 0;
  if (sgdt_pool_delta(h_, pos.data(), val.data(), &n) != SGDT_OK) {
    // several runs (resample_per_mode): the pool was uploaded before the
    // call, so the device pool is the truth -- take all of it
    check(sgdt_get_pool(h_, pool.data()), "update_core_epoch");
    d2h_bytes += pool.size() * sizeof(std::uint32_t);
    pool_data_ = pool.data();
    pool_size_ = pool.size();
    return true;
  }
  d2h_bytes += 2 * n * sizeof(std::uint32_t);
  for (std::size_t i = 0; i < n; ++i) std::swap(pool[i], pool[pos[i]]);
  bool same = std::equal(batch.begin(), batch.end(), pool.begin());
  for (std::size_t i = 0; same && i < n; ++i) same = pool[pos[i]] == val[i];
  if (!same) {
    for (std::size_t i = n; i-- > 0;) std::swap(pool[i], pool[pos[i]]);  // undo
    return false;
  }
  pool_data_ = pool.data();
  pool_size_ = pool.size();
  return true;
}

void Session::put_rng(const Rng& r) { check(sgdt_set_rng(h_, r.state_words().data(), r.state_pos()), "rng"); }

void Session::take_rng(Rng& r) {
  std::uint64_t words[Rng::kWords];
  std::uint32_t pos = 0;
  check(sgdt_get_rng(h_, words, &pos), "rng");
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
