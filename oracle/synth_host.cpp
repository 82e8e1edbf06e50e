// synth_host.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Host (multi-threaded C++) restatement of the BASELINE config 2-5 generator
// sgdt_synth (paper_2012_03550_b200/csrc/sgdt_synth.cu; numpy restatement
// oracle/synth_oracle.py).  It exists so that bench.py's reference arm can
// build the SAME full-size tensor as the GPU arm without loading any product
// library or touching the GPU: the reference (oracle/_ref) then trains on it.
// tests/test_synth.py checks it against oracle/synth_oracle.py (CPU) and
// against the device generator (GPU): indices and their order bit-exact,
// values to fp64 rounding (host libm vs device log/cos/pow and FMA).
//
// Algorithm (SURVEY.md 8(d) "C2-C5 need a new generator"):
//   draw d, mode k: u = unit53(Philox4x32-10((d, d>>32, k, TAG_DRAW), seed));
//                   index = floor(u I) (uniform) or the first i with
//                   cdf[i] > u (bounded Zipf(s), blocked prefix sums);
//   first draw wins: the nnz earliest first occurrences of a linear
//                   position (mode 1 fastest), output in ascending position
//                   (synth.cpp:40);
//   teacher:        A, B ~ N(0, sigma^2), sigma = (J R^(1/N))^(-1/4);
//                   xhat = sum_r prod_k (A^(k) B^(k))[i_k, r];
//   values:         ratings round(3 + (xhat - mean)/sd) in [1, 5], or
//                   xhat + noise N(0, 1).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

namespace {

typedef unsigned __int128 u128;

struct U4 {
  uint32_t x, y, z, w;
};

inline U4 philox(U4 c, uint32_t k0, uint32_t k1) {
  for (int i = 0; i < 10; ++i) {
    if (i) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c.x;
    const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c.z;
    c = U4{static_cast<uint32_t>(p1 >> 32) ^ c.y ^ k0, static_cast<uint32_t>(p1), static_cast<uint32_t>(p0 >> 32) ^ c.w ^ k1,
           static_cast<uint32_t>(p0)};
  }
  return c;
}

inline double unit53(uint32_t hi, uint32_t lo) {
  return static_cast<double>(((static_cast<uint64_t>(hi) << 32) | lo) >> 11) * 0x1.0p-53;
}

constexpr uint32_t kTagDraw = 0x5A1F0000u, kTagTeacher = 0x7EAC0000u, kTagNoise = 0x00150000u;
constexpr uint64_t kCdfBlock = 1024, kSumChunk = 4096;

inline double normal_at(uint64_t e, uint32_t stream, uint32_t tag, uint64_t seed) {
  const U4 r = philox(U4{static_cast<uint32_t>(e), static_cast<uint32_t>(e >> 32), stream, tag}, static_cast<uint32_t>(seed),
                      static_cast<uint32_t>(seed >> 32));
  const double u1 = unit53(r.x, r.y), u2 = unit53(r.z, r.w);
  return std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(6.283185307179586 * u2);
}

template <class F>
void parallel_for(uint64_t n, int threads, F f) {  // f(begin, end, thread)
  if (n == 0) return;
  const uint64_t t = std::min<uint64_t>(threads, n);
  std::vector<std::thread> th;
  for (uint64_t i = 0; i < t; ++i) {
    const uint64_t b = n * i / t, e = n * (i + 1) / t;
    th.emplace_back([=] { f(b, e, static_cast<int>(i)); });
  }
  for (auto& x : th) x.join();
}

// dynamic work list: f(item) for item in [0, n)
template <class F>
void parallel_items(uint64_t n, int threads, F f) {
  std::atomic<uint64_t> next{0};
  std::vector<std::thread> th;
  for (int i = 0; i < threads; ++i)
    th.emplace_back([&] {
      for (uint64_t it; (it = next.fetch_add(1)) < n;) f(it);
    });
  for (auto& x : th) x.join();
}

std::vector<double> zipf_cdf(uint32_t I, double s) {
  const uint64_t nb = (I + kCdfBlock - 1) / kCdfBlock;
  std::vector<double> cdf(I), off(nb + 1);
  for (uint64_t b = 0; b < nb; ++b) {
    double acc = 0.0;
    for (uint64_t i = b * kCdfBlock; i < std::min<uint64_t>(I, (b + 1) * kCdfBlock); ++i) {
      acc += std::pow(static_cast<double>(i + 1), -s);
      cdf[i] = acc;
    }
    off[b] = acc;
  }
  double acc = 0.0;
  for (uint64_t b = 0; b < nb; ++b) {
    const double t = off[b];
    off[b] = acc;
    acc += t;
  }
  for (uint64_t i = 0; i < I; ++i) cdf[i] = (off[i / kCdfBlock] + cdf[i]) / acc;
  return cdf;
}

struct Rec {
  uint64_t hi, lo, id;
};
inline bool rec_less(const Rec& a, const Rec& b) {
  if (a.hi != b.hi) return a.hi < b.hi;
  if (a.lo != b.lo) return a.lo < b.lo;
  return a.id < b.id;
}

}  // namespace

extern "C" {

// coords_out: nnz x order (1-based, entry-major); values_out: nnz.
// Returns 0, or 5 (DomainError: bad arguments), 2 (ConfigError: index space
// too concentrated), mirroring sgdt_synth.
int sh_synth(int order, const uint32_t* dims, const double* zipf, uint64_t nnz, uint32_t J, uint32_t R, int ratings,
             double noise, uint64_t seed, int threads, uint32_t* coords_out, double* values_out) {
  if (order < 2 || order > 8 || !dims || !zipf || !coords_out || !values_out) return 5;
  long double total = 1;
  for (int k = 0; k < order; ++k) {
    if (dims[k] < 1 || zipf[k] < 0.0) return 5;
    total *= dims[k];
  }
  if (nnz == 0 || static_cast<long double>(nnz) > total / 2 || nnz > 0xFFFFFFFFull || J < 1 || R < 1) return 5;
  if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));

  std::vector<std::vector<double>> cdf(order);
  for (int k = 0; k < order; ++k)
    if (zipf[k] != 0.0) cdf[k] = zipf_cdf(dims[k], zipf[k]);
  auto draw_index = [&](int k, uint64_t d) -> uint32_t {
    const U4 r = philox(U4{static_cast<uint32_t>(d), static_cast<uint32_t>(d >> 32), static_cast<uint32_t>(k), kTagDraw},
                        static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    const double u = unit53(r.x, r.y);
    const uint32_t I = dims[k];
    if (zipf[k] == 0.0) {
      const uint64_t v = static_cast<uint64_t>(u * I);
      return static_cast<uint32_t>(v < I ? v : I - 1);
    }
    const double* c = cdf[k].data();
    uint32_t lo = 0, hi = I;
    while (lo < hi) {
      const uint32_t mid = lo + (hi - lo) / 2;
      if (c[mid] > u) hi = mid;
      else lo = mid + 1;
    }
    return lo < I ? lo : I - 1;
  };
  // bucket = the top kBucketBits of the (bit-length) key
  int keybits = 0;
  {
    u128 t = 1;
    for (int k = 0; k < order; ++k) t *= dims[k];
    t -= 1;
    while (t) {
      ++keybits;
      t >>= 1;
    }
  }
  const int bbits = std::min(keybits, 14);
  const uint64_t nbuck = 1ull << bbits;
  const int shift = keybits - bbits;
  auto bucket_of = [&](const Rec& r) -> uint64_t {
    const u128 key = (static_cast<u128>(r.hi) << 64) | r.lo;
    return static_cast<uint64_t>(key >> shift);
  };

  uint64_t cap = nnz + nnz / 4 + (1u << 20);
  std::vector<Rec> rec, tmp;
  std::vector<uint64_t> boff;
  std::vector<uint8_t> first;
  uint64_t thr = 0;
  for (int round = 0;; ++round) {
    if (round > 40) return 2;
    tmp.assign(cap, Rec{});
    parallel_for(cap, threads, [&](uint64_t b, uint64_t e, int) {
      for (uint64_t d = b; d < e; ++d) {
        u128 key = 0, stride = 1;
        for (int k = 0; k < order; ++k) {
          key += static_cast<u128>(draw_index(k, d)) * stride;
          stride *= dims[k];
        }
        tmp[d] = Rec{static_cast<uint64_t>(key >> 64), static_cast<uint64_t>(key), d};
      }
    });
    // counting sort into buckets (stable: draw order inside a bucket), then
    // each bucket sorted by (key, draw)
    std::vector<std::vector<uint64_t>> hist(threads, std::vector<uint64_t>(nbuck, 0));
    parallel_for(cap, threads, [&](uint64_t b, uint64_t e, int t) {
      for (uint64_t d = b; d < e; ++d) ++hist[t][bucket_of(tmp[d])];
    });
    boff.assign(nbuck + 1, 0);
    {
      uint64_t acc = 0;
      for (uint64_t q = 0; q < nbuck; ++q) {
        boff[q] = acc;
        for (int t = 0; t < threads; ++t) {
          const uint64_t c = hist[t][q];
          hist[t][q] = acc;
          acc += c;
        }
      }
      boff[nbuck] = acc;
    }
    rec.assign(cap, Rec{});
    parallel_for(cap, threads, [&](uint64_t b, uint64_t e, int t) {
      for (uint64_t d = b; d < e; ++d) rec[hist[t][bucket_of(tmp[d])]++] = tmp[d];
    });
    std::vector<Rec>().swap(tmp);
    parallel_items(nbuck, threads, [&](uint64_t q) { std::sort(rec.begin() + boff[q], rec.begin() + boff[q + 1], rec_less); });
    // first occurrences (the smallest draw of each key), flagged by draw id
    first.assign(cap, 0);
    parallel_items(nbuck, threads, [&](uint64_t q) {
      for (uint64_t i = boff[q]; i < boff[q + 1]; ++i)
        if (i == boff[q] || rec[i].hi != rec[i - 1].hi || rec[i].lo != rec[i - 1].lo) first[rec[i].id] = 1;
    });
    uint64_t U = 0;
    thr = cap;
    for (uint64_t d = 0; d < cap; ++d)
      if (first[d] && ++U == nnz) {
        thr = d;
        break;
      }
    if (U >= nnz) break;
    cap = cap + cap / 2;
  }
  // kept: first occurrences with draw id <= thr, in ascending key order
  std::vector<uint64_t> kept_off(nbuck + 1, 0);
  auto kept = [&](uint64_t i) { return rec[i].id <= thr && first[rec[i].id] && (i == 0 || rec[i].hi != rec[i - 1].hi || rec[i].lo != rec[i - 1].lo); };
  parallel_items(nbuck, threads, [&](uint64_t q) {
    uint64_t c = 0;
    for (uint64_t i = boff[q]; i < boff[q + 1]; ++i) c += kept(i);
    kept_off[q + 1] = c;
  });
  for (uint64_t q = 0; q < nbuck; ++q) kept_off[q + 1] += kept_off[q];
  if (kept_off[nbuck] != nnz) return 1;
  parallel_items(nbuck, threads, [&](uint64_t q) {
    uint64_t e = kept_off[q];
    for (uint64_t i = boff[q]; i < boff[q + 1]; ++i) {
      if (!kept(i)) continue;
      u128 key = (static_cast<u128>(rec[i].hi) << 64) | rec[i].lo;
      for (int k = 0; k < order; ++k) {
        coords_out[e * order + k] = static_cast<uint32_t>(key % dims[k]) + 1;
        key /= dims[k];
      }
      ++e;
    }
  });
  std::vector<Rec>().swap(rec);
  std::vector<uint8_t>().swap(first);

  // teacher Q^(k) = A^(k) B^(k), fp64, j ascending
  const double sigma = std::pow(J * std::pow(static_cast<double>(R), 1.0 / order), -0.25);
  std::vector<std::vector<double>> Q(order);
  for (int k = 0; k < order; ++k) {
    const uint64_t I = dims[k];
    std::vector<double> A(I * J), B(static_cast<uint64_t>(J) * R);
    for (uint64_t e = 0; e < B.size(); ++e) B[e] = sigma * normal_at(e, 17u + 2u * k, kTagTeacher, seed);
    parallel_for(I * J, threads, [&](uint64_t b, uint64_t e, int) {
      for (uint64_t x = b; x < e; ++x) A[x] = sigma * normal_at(x, 16u + 2u * k, kTagTeacher, seed);
    });
    Q[k].assign(I * R, 0.0);
    parallel_for(I, threads, [&](uint64_t b, uint64_t e, int) {
      for (uint64_t i = b; i < e; ++i)
        for (uint32_t r = 0; r < R; ++r) {
          double acc = 0.0;
          for (uint32_t j = 0; j < J; ++j) acc += A[i * J + j] * B[static_cast<uint64_t>(j) * R + r];
          Q[k][i * R + r] = acc;
        }
    });
  }
  parallel_for(nnz, threads, [&](uint64_t b, uint64_t e, int) {
    for (uint64_t x = b; x < e; ++x) {
      double v = 0.0;
      for (uint32_t r = 0; r < R; ++r) {
        double c = 1.0;
        for (int k = 0; k < order; ++k) c *= Q[k][static_cast<uint64_t>(coords_out[x * order + k] - 1) * R + r];
        v += c;
      }
      values_out[x] = v;
    }
  });
  if (ratings) {
    const uint64_t nc = (nnz + kSumChunk - 1) / kSumChunk;
    std::vector<double> part(nc);
    auto sums = [&](double center, bool sq) {
      parallel_for(nc, threads, [&](uint64_t b, uint64_t e, int) {
        for (uint64_t c = b; c < e; ++c) {
          double acc = 0.0;
          for (uint64_t i = c * kSumChunk; i < std::min(nnz, (c + 1) * kSumChunk); ++i) {
            const double d = values_out[i] - center;
            acc += sq ? d * d : values_out[i];
          }
          part[c] = acc;
        }
      });
      double acc = 0.0;
      for (uint64_t c = 0; c < nc; ++c) acc += part[c];
      return acc;
    };
    const double mean = sums(0.0, false) / static_cast<double>(nnz);
    const double sd = std::sqrt(sums(mean, true) / static_cast<double>(nnz - 1));
    parallel_for(nnz, threads, [&](uint64_t b, uint64_t e, int) {
      for (uint64_t x = b; x < e; ++x) {
        const double v = std::nearbyint(3.0 + (values_out[x] - mean) / sd);
        values_out[x] = v < 1.0 ? 1.0 : (v > 5.0 ? 5.0 : v);
      }
    });
  } else if (noise > 0.0) {
    parallel_for(nnz, threads, [&](uint64_t b, uint64_t e, int) {
      for (uint64_t x = b; x < e; ++x) values_out[x] += noise * normal_at(x, 99u, kTagNoise, seed);
    });
  }
  return 0;
}

// train_test_split's id partition (sptensor.cpp:217-254; the device form is
// sgdt_split_ids): Fisher-Yates of 0..nnz-1 with Rng(seed) -- j = i +
// next_below(nnz - i) for i < nnz - 1 (rng.hpp:20-25) -- the first
// llround(fraction nnz) positions are the test ids; both halves ascending.
// The swaps run with the upcoming targets prefetched (the draws do not
// depend on the array), and the halves are read off a membership flag
// instead of sorted.  Returns ntest, or 0 for a degenerate split.
uint64_t sh_split_ids(uint64_t nnz, double test_fraction, uint64_t seed, uint32_t* test_ids, uint32_t* train_ids) {
  if (!(test_fraction > 0.0 && test_fraction < 1.0)) return 0;
  const uint64_t ntest = static_cast<uint64_t>(std::llround(test_fraction * static_cast<double>(nnz)));
  if (ntest == 0 || ntest == nnz) return 0;
  std::vector<uint32_t> ids(nnz);
  for (uint64_t e = 0; e < nnz; ++e) ids[e] = static_cast<uint32_t>(e);
  std::mt19937_64 eng(seed);
  auto next_below = [&](uint64_t bound) {
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
      const uint64_t r = eng();
      if (r >= threshold) return r % bound;
    }
  };
  constexpr uint64_t kBatch = 1 << 16, kAhead = 24;
  std::vector<uint64_t> js(kBatch);
  for (uint64_t i0 = 0; i0 + 1 < nnz; i0 += kBatch) {
    const uint64_t i1 = std::min(nnz - 1, i0 + kBatch);
    for (uint64_t i = i0; i < i1; ++i) js[i - i0] = i + next_below(nnz - i);
    for (uint64_t i = i0; i < i1; ++i) {
      if (i + kAhead < i1) __builtin_prefetch(&ids[js[i + kAhead - i0]], 1);
      std::swap(ids[i], ids[js[i - i0]]);
    }
  }
  std::vector<uint8_t> in_test(nnz, 0);
  for (uint64_t i = 0; i < ntest; ++i) in_test[ids[i]] = 1;
  uint64_t a = 0, b = 0;
  for (uint64_t e = 0; e < nnz; ++e) {
    if (in_test[e]) test_ids[a++] = static_cast<uint32_t>(e);
    else train_ids[b++] = static_cast<uint32_t>(e);
  }
  return ntest;
}

}  // extern "C"
