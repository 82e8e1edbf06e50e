// device.cpp -- C++ API <-> C-ABI bridge: sessions, model/RNG transfer and
// the error-code mapping (include/sgdt.h codes -> sptucker exceptions).
#include "device.hpp"

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

namespace {
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
  std::vector<std::vector<double>> scratch;
  std::vector<double*> a(m.order()), b(m.order());
  for (std::size_t n = 0; n < m.order(); ++n) {
    if (factors) {
      a[n] = m.factor(n).data().data();
    } else {
      scratch.emplace_back(m.factor(n).size());
      a[n] = scratch.back().data();
    }
    if (kruskal) {
      b[n] = m.kruskal(n).data().data();
    } else {
      scratch.emplace_back(m.kruskal(n).size());
      b[n] = scratch.back().data();
    }
  }
  check(sgdt_get_model(h_, a.data(), b.data()), "download model");
  if (kruskal) m.refresh_core_cache();
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
