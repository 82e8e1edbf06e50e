// sptensor.cpp -- host construction of CooTensor (validation + per-mode
// buckets, the layout the device copies are built from) and the device-backed
// sampler entry points.
#include "sptucker/sptensor.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <string>
#include <thread>

#include "device.hpp"

namespace sptucker {

Shape::Shape(std::vector<std::uint32_t> dims) : dims_(std::move(dims)) {
  if (dims_.size() < 2) throw DomainError("shape: order must be at least 2");
  if (dims_.size() > SGDT_MAX_ORDER) throw DomainError("shape: order above 8 is not supported on the device");
  // Deviation (documented in DESIGN.md): the reference rejects shapes whose
  // element count overflows 64 bits (sptensor.cpp:34-35); nothing on the
  // device path linearises coordinates, so such shapes are accepted and
  // total_elems() saturates.
  total_ = 1;
  for (const std::uint32_t d : dims_) {
    if (d < 1) throw DomainError("shape: every dim must be >= 1");
    total_ = total_ > std::numeric_limits<std::uint64_t>::max() / d ? std::numeric_limits<std::uint64_t>::max()
                                                                     : total_ * d;
  }
}

namespace {

// Host threads for the O(nnz) construction work (a Netflix-sized tensor has
// 10^8 entries; the reference builds it on one thread).
unsigned ctor_threads(std::size_t nnz) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const std::size_t by_size = std::max<std::size_t>(1, nnz / (1u << 20));
  return static_cast<unsigned>(std::min<std::size_t>({hw, by_size, 64}));
}

template <class F>
void parallel_for(unsigned nt, std::size_t n, F&& f) {  // f(begin, end) over nt slices
  if (nt <= 1) {
    f(std::size_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < nt; ++t) pool.emplace_back([&, t] { f(n * t / nt, n * (t + 1) / nt); });
  f(std::size_t{0}, n / nt);
  for (auto& th : pool) th.join();
}

// Duplicate detection: sort (128-bit linear position, entry id) pairs.  The
// reference reports the first entry, in entry order, whose position was seen
// before (sptensor.cpp:90-99): in every group of equal positions that is the
// group's second-smallest id, and the answer is the smallest of those (or nnz
// when there is none).  The reference's 64-bit key wraps for shapes beyond
// 2^64 elements, hence the two-word key.  Slices are sorted on host threads
// and merged pairwise.
std::size_t first_duplicate(const Shape& shape, const std::vector<std::uint32_t>& coords, std::size_t nnz) {
  const std::size_t order = shape.order();
  struct Key {
    std::uint64_t hi, lo;
    std::uint32_t e;
  };
  auto less = [](const Key& a, const Key& b) {
    return a.hi != b.hi ? a.hi < b.hi : a.lo != b.lo ? a.lo < b.lo : a.e < b.e;
  };
  std::vector<Key> keys(nnz);
  const unsigned nt = ctor_threads(nnz);
  parallel_for(nt, nnz, [&](std::size_t b, std::size_t e) {
    for (std::size_t i = b; i < e; ++i) {
      unsigned __int128 key = 0, stride = 1;
      for (std::size_t k = 0; k < order; ++k) {
        key += static_cast<unsigned __int128>(coords[i * order + k] - 1) * stride;
        stride *= shape.dim(k);
      }
      keys[i] = {static_cast<std::uint64_t>(key >> 64), static_cast<std::uint64_t>(key), static_cast<std::uint32_t>(i)};
    }
    std::sort(keys.begin() + static_cast<std::ptrdiff_t>(b), keys.begin() + static_cast<std::ptrdiff_t>(e), less);
  });
  // pairwise merges of the sorted slices, a round of independent merges at a time
  std::vector<std::size_t> cut(nt + 1);
  for (unsigned t = 0; t <= nt; ++t) cut[t] = nnz * t / nt;
  for (std::size_t width = 1; width < nt; width *= 2) {
    std::vector<std::thread> pool;
    for (std::size_t t = 0; t + width < nt; t += 2 * width) {
      const std::size_t b = cut[t], m = cut[t + width], e = cut[std::min<std::size_t>(t + 2 * width, nt)];
      pool.emplace_back([&, b, m, e] {
        std::inplace_merge(keys.begin() + static_cast<std::ptrdiff_t>(b), keys.begin() + static_cast<std::ptrdiff_t>(m),
                           keys.begin() + static_cast<std::ptrdiff_t>(e), less);
      });
    }
    for (auto& th : pool) th.join();
  }
  std::size_t first = nnz;
  for (std::size_t i = 1; i < nnz; ++i) {
    const bool same = keys[i].hi == keys[i - 1].hi && keys[i].lo == keys[i - 1].lo;
    const bool second_of_group = same && (i < 2 || keys[i - 2].hi != keys[i].hi || keys[i - 2].lo != keys[i].lo);
    if (second_of_group) first = std::min<std::size_t>(first, keys[i].e);
  }
  return first;
}

}  // namespace

CooTensor::CooTensor(Shape shape, std::vector<std::uint32_t> coords, std::vector<double> values)
    : shape_(std::move(shape)), coords_(std::move(coords)), values_(std::move(values)) {
  const std::size_t order = shape_.order();
  const std::size_t nnz = values_.size();
  if (nnz == 0) throw DataError("tensor has no entries");
  if (coords_.size() != nnz * order) throw DataError("coords/values length mismatch");
  if (nnz > std::numeric_limits<std::uint32_t>::max()) throw DataError("entry count exceeds the 32-bit id space");
  mode_perm_.assign(order, std::vector<std::uint32_t>(nnz));
  mode_offsets_.assign(order, {});
  if (sgdt_device_count() > 0) {
    // on the device (sgdt_tensor_layout): range + duplicate checks by a radix
    // sort of packed coordinate keys, the N stable bucket sorts
    std::vector<std::uint32_t*> perm(order);
    std::vector<std::uint64_t*> off(order);
    for (std::size_t n = 0; n < order; ++n) {
      mode_offsets_[n].assign(static_cast<std::size_t>(shape_.dim(n)) + 1, 0);
      perm[n] = mode_perm_[n].data();
      off[n] = mode_offsets_[n].data();
    }
    const std::vector<std::uint32_t>& dims = shape_.dims();
    sgdt_tensor_desc d{};
    d.order = static_cast<int>(order);
    d.dims = dims.data();
    d.nnz = nnz;
    d.coords = coords_.data();
    d.values = values_.data();
    const int rc = sgdt_tensor_layout(&d, -1, perm.data(), off.data());
    if (rc == SGDT_ERR_DATA) throw DataError(sgdt_last_error());
    detail::check(rc, "CooTensor");
    return;
  }
  // Without a device (file tooling, the CPU test suite) the same layout is
  // built on host threads.  The reference checks entry by entry, range
  // before duplicate; the first failing entry decides the message.  Entries before the first out-of-range
  // one are all in range, so a duplicate found below it is exact.
  std::size_t bad_range = nnz;
  for (std::size_t e = 0; e < nnz && bad_range == nnz; ++e)
    for (std::size_t k = 0; k < order; ++k) {
      const std::uint32_t c = coords_[e * order + k];
      if (c < 1 || c > shape_.dim(k)) {
        bad_range = e;
        break;
      }
    }
  const std::size_t dup = first_duplicate(shape_, coords_, nnz);
  if (dup < bad_range) throw DataError("entry " + std::to_string(dup) + ": duplicate coordinate");
  if (bad_range < nnz) throw DataError("entry " + std::to_string(bad_range) + ": coordinate out of range");

  // Stable counting sort per mode: bucket i holds the entries with i_n = i in
  // ascending entry id (the order the device mode copies inherit); one host
  // thread per mode.
  auto bucket_mode = [&](std::size_t n) {
    std::vector<std::uint64_t>& off = mode_offsets_[n];
    off.assign(static_cast<std::size_t>(shape_.dim(n)) + 1, 0);
    for (std::size_t e = 0; e < nnz; ++e) ++off[coords_[e * order + n]];
    std::partial_sum(off.begin(), off.end(), off.begin());
    std::vector<std::uint64_t> next(off.begin(), off.end() - 1);
    std::vector<std::uint32_t>& perm = mode_perm_[n];
    perm.resize(nnz);
    for (std::size_t e = 0; e < nnz; ++e) perm[next[coords_[e * order + n] - 1]++] = static_cast<std::uint32_t>(e);
  };
  if (ctor_threads(nnz) > 1) {
    std::vector<std::thread> pool;
    for (std::size_t n = 1; n < order; ++n) pool.emplace_back(bucket_mode, n);
    bucket_mode(0);
    for (auto& th : pool) th.join();
  } else {
    for (std::size_t n = 0; n < order; ++n) bucket_mode(n);
  }
}

double CooTensor::mean_value() const {
  double s = 0.0;
  for (const double v : values_) s += v;
  return s / static_cast<double>(values_.size());
}

detail::DeviceCache& CooTensor::device_cache() const {
  if (!device_) device_ = std::make_shared<detail::DeviceCache>();
  return *device_;
}

std::pair<CooTensor, CooTensor> train_test_split(const CooTensor& t, double test_fraction, std::uint64_t seed) {
  if (!(test_fraction > 0.0 && test_fraction < 1.0)) throw DomainError("train_test_split: fraction must lie in (0,1)");
  const std::size_t nnz = t.nnz();
  const std::size_t ntest = static_cast<std::size_t>(std::llround(test_fraction * static_cast<double>(nnz)));
  if (ntest == 0 || ntest == nnz)
    throw DomainError("train_test_split: degenerate split (|test|=" + std::to_string(ntest) + " of " +
                      std::to_string(nnz) + ")");
  // the Fisher-Yates with Rng(seed) and the two sorts run on the device
  // (sgdt_split_ids: the sampler's swap-chain resolution, bit-exact)
  std::vector<std::uint32_t> ids(nnz);
  detail::check(sgdt_split_ids(nnz, test_fraction, seed, -1, ids.data(), ids.data() + ntest), "train_test_split");
  auto take = [&](std::size_t b, std::size_t e) {
    std::vector<std::uint32_t> c;
    std::vector<double> v;
    c.reserve((e - b) * t.order());
    v.reserve(e - b);
    for (std::size_t i = b; i < e; ++i) {
      const auto cc = t.coord(ids[i]);
      c.insert(c.end(), cc.begin(), cc.end());
      v.push_back(t.value(ids[i]));
    }
    return CooTensor(t.shape(), std::move(c), std::move(v));
  };
  CooTensor test = take(0, ntest);
  CooTensor train = take(ntest, nnz);
  return {std::move(train), std::move(test)};
}

namespace {
detail::Session& sampler_session(const CooTensor& t) {
  return detail::session_for(t, nullptr, t.shape(), Ranks{std::vector<std::uint32_t>(t.order(), 1), 1});
}
}  // namespace

void sample_batch(const CooTensor& t, std::size_t m, Rng& rng, std::vector<std::uint32_t>& pool,
                  std::vector<std::uint32_t>& out) {
  const std::size_t nnz = t.nnz();
  if (m < 1 || m > nnz) throw DomainError("sample_batch: batch size out of range");
  detail::Session& s = sampler_session(t);
  if (pool.size() != nnz) {
    pool.resize(nnz);
    std::iota(pool.begin(), pool.end(), 0u);
    s.pool_reset(pool);
  } else {
    s.sync_pool(pool);  // uploaded only if it is not the buffer this session last wrote
  }
  out.resize(m);
  for (int attempt = 0;; ++attempt) {
    s.put_rng(rng);
    detail::check(sgdt_sample_batch(s.get(), m, out.data()), "sample_batch");
    if (s.pool_apply_checked(pool, out)) break;  // replayed on the host pool and checked
    if (attempt) throw InternalError("sample_batch: device pool does not follow the host pool");
    s.sync_pool(pool, /*force=*/true);  // the host pool was edited: repeat from it
  }
  s.take_rng(rng);
}

std::vector<std::uint32_t> sample_batch(const CooTensor& t, std::size_t m, Rng& rng) {
  std::vector<std::uint32_t> pool, out;
  sample_batch(t, m, rng, pool, out);
  return out;
}

}  // namespace sptucker
