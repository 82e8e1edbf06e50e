// io.cpp -- host I/O of the C++ API: the delimited tensor format, the binary
// model file, the metrics CSV and the unfolding / vectorisation index maps
// (SURVEY.md section 8(f) row 4).  Formats, accepted inputs and error texts
// are the reference's (sptensor.cpp:40-78,120-209, model.cpp:178-280,
// eval.cpp:47-146); the byte-for-byte pin is tests/golden/io (written by the
// reference itself, tests/golden/make_io_golden.py) checked by
// tests/cpp/test_sptucker.cpp.
//
// Nothing here is on the training hot path.  The text reader and writer are
// the only parts that scale with nnz (a Netflix-sized file is ~2.5 GB of
// text), so both split the work over host threads: the reader parses
// newline-aligned chunks independently and reports the first failing line of
// the file, exactly as the sequential reference loop would; the writer formats
// entry ranges in parallel and writes them in order.
#include <algorithm>
#include <bit>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "sptucker/eval.hpp"
#include "sptucker/model.hpp"
#include "sptucker/sptensor.hpp"

namespace sptucker {

// ---- unfolding / vectorisation indices (sptensor.cpp:40-78) ---------------

std::uint64_t unfold_col_index(const Shape& shape, std::span<const std::uint32_t> coord, std::size_t mode) {
  const std::size_t order = shape.order();
  if (mode >= order) throw DomainError("unfold_col_index: mode out of range");
  if (coord.size() != order) throw DomainError("unfold_col_index: coord arity mismatch");
  std::uint64_t col = 1, stride = 1;
  for (std::size_t k = 0; k < order; ++k) {
    if (coord[k] < 1 || coord[k] > shape.dim(k)) throw DomainError("unfold_col_index: coordinate out of range");
    if (k == mode) continue;
    col += static_cast<std::uint64_t>(coord[k] - 1) * stride;
    stride *= shape.dim(k);
  }
  return col;
}

std::uint64_t vec_index(const Shape& shape, std::span<const std::uint32_t> coord, std::size_t mode) {
  return (unfold_col_index(shape, coord, mode) - 1) * shape.dim(mode) + coord[mode];
}

void invert_vec_index(const Shape& shape, std::uint64_t k, std::size_t mode, std::span<std::uint32_t> coord) {
  const std::size_t order = shape.order();
  if (mode >= order) throw DomainError("invert_vec_index: mode out of range");
  if (coord.size() != order) throw DomainError("invert_vec_index: coord arity mismatch");
  if (k < 1 || k > shape.total_elems()) throw DomainError("invert_vec_index: position out of range");
  std::uint64_t rest = k - 1;
  coord[mode] = static_cast<std::uint32_t>(rest % shape.dim(mode)) + 1;
  rest /= shape.dim(mode);
  for (std::size_t m = 0; m < order; ++m) {
    if (m == mode) continue;
    coord[m] = static_cast<std::uint32_t>(rest % shape.dim(m)) + 1;
    rest /= shape.dim(m);
  }
}

// ---- delimited tensor text ------------------------------------------------

namespace {

std::string read_file(const std::string& path, const char* what_open) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw DataError(std::string(what_open) + " '" + path + "'");
  std::string buf;
  char tmp[1 << 16];
  std::size_t got;
  while ((got = std::fread(tmp, 1, sizeof tmp, f)) > 0) buf.append(tmp, got);
  std::fclose(f);
  return buf;
}

inline bool is_sep(char c) { return c == ' ' || c == '\t' || c == ',' || c == '\r'; }

// Fields of one line: whitespace / comma separated, empty fields dropped.
inline std::size_t split_fields(std::string_view line, std::string_view* out, std::size_t cap) {
  std::size_t n = 0, pos = 0;
  while (pos < line.size()) {
    while (pos < line.size() && is_sep(line[pos])) ++pos;
    const std::size_t start = pos;
    while (pos < line.size() && !is_sep(line[pos])) ++pos;
    if (pos > start) {
      if (n < cap) out[n] = line.substr(start, pos - start);
      ++n;
    }
  }
  return n;
}

// A line that carries data (not blank, not a '#' comment).
inline bool is_data_line(std::string_view line) {
  std::size_t pos = 0;
  while (pos < line.size() && is_sep(line[pos])) ++pos;
  return pos < line.size() && line[pos] != '#';
}

struct ChunkResult {
  std::vector<std::uint32_t> coords;
  std::vector<double> values;
  std::vector<std::uint32_t> maxima;
  std::size_t lines = 0;       // lines consumed (all of them unless failed)
  std::size_t fail_line = 0;   // 1-based inside the chunk, 0 = none
  std::string fail_what;
};

void parse_chunk(std::string_view text, std::size_t order, const LoadOptions& opts, ChunkResult& r) {
  r.maxima.assign(order, 0);
  std::vector<std::string_view> fields(order + 2);
  std::size_t pos = 0;
  while (pos < text.size()) {
    std::size_t eol = text.find('\n', pos);
    if (eol == std::string_view::npos) eol = text.size();
    const std::string_view line = text.substr(pos, eol - pos);
    pos = eol + 1;
    ++r.lines;
    auto fail = [&](std::string what) {
      r.fail_line = r.lines;
      r.fail_what = std::move(what);
    };
    const std::size_t nf = split_fields(line, fields.data(), fields.size());
    if (nf == 0 || fields[0][0] == '#') continue;
    if (nf != order + 1) {
      fail("expected " + std::to_string(order + 1) + " fields, got " + std::to_string(nf));
      return;
    }
    for (std::size_t k = 0; k < order; ++k) {
      std::uint32_t idx = 0;
      const auto f = fields[k];
      const auto [p, ec] = std::from_chars(f.data(), f.data() + f.size(), idx);
      if (ec != std::errc{} || p != f.data() + f.size() || idx < 1) {
        fail("bad index in field " + std::to_string(k + 1));
        return;
      }
      r.coords.push_back(idx);
      r.maxima[k] = std::max(r.maxima[k], idx);
    }
    double v = 0.0;
    const auto f = fields[order];
    const auto [p, ec] = std::from_chars(f.data(), f.data() + f.size(), v);
    if (ec != std::errc{} || p != f.data() + f.size() || !std::isfinite(v)) {
      fail("bad value field");
      return;
    }
    if (v == 0.0) {
      if (opts.zero_policy == ZeroPolicy::Reject) {
        fail("zero value (zero policy is reject)");
        return;
      }
      v = opts.zero_replacement;
    }
    r.values.push_back(v);
  }
}

// Smallest chunk the reader hands to a thread (4 MB; the golden replay lowers
// it with SPTUCKER_LOAD_CHUNK_BYTES to split its small files).
std::size_t min_chunk_bytes() {
  const char* e = std::getenv("SPTUCKER_LOAD_CHUNK_BYTES");
  const long long v = e ? std::atoll(e) : 0;
  return v > 0 ? static_cast<std::size_t>(v) : (4u << 20);
}

unsigned host_threads() {
  const unsigned t = std::thread::hardware_concurrency();
  return t == 0 ? 1 : std::min(t, 64u);
}

}  // namespace

CooTensor CooTensor::load_delimited(const std::string& path, std::size_t order, const LoadOptions& opts) {
  if (order < 2) throw DomainError("load_delimited: order must be >= 2");
  const std::string text = read_file(path, "cannot open");
  const std::string_view all(text);

  // The header (when skipped) is the first data-carrying line; it is consumed
  // sequentially so the chunks below only see data / blank / comment lines.
  std::size_t start = 0, head_lines = 0;
  if (opts.skip_header) {
    while (start < all.size()) {
      std::size_t eol = all.find('\n', start);
      if (eol == std::string_view::npos) eol = all.size();
      const bool data = is_data_line(all.substr(start, eol - start));
      start = eol + 1;
      ++head_lines;
      if (data) break;
    }
    start = std::min(start, all.size());
  }

  // Newline-aligned chunks of at least min_chunk_bytes, one per host thread
  // at most.
  const std::size_t body = all.size() - start;
  const std::size_t want =
      std::max<std::size_t>(1, std::min<std::size_t>(host_threads(), body / min_chunk_bytes()));
  std::vector<std::size_t> cut{start};
  for (std::size_t c = 1; c < want; ++c) {
    std::size_t at = std::max(start + body * c / want, cut.back());
    const std::size_t nl = all.find('\n', at);
    at = nl == std::string_view::npos ? all.size() : nl + 1;
    if (at > cut.back() && at < all.size()) cut.push_back(at);
  }
  cut.push_back(all.size());
  const std::size_t nchunks = cut.size() - 1;
  std::vector<ChunkResult> res(nchunks);
  {
    std::vector<std::thread> pool;
    for (std::size_t c = 1; c < nchunks; ++c)
      pool.emplace_back(parse_chunk, all.substr(cut[c], cut[c + 1] - cut[c]), order, std::cref(opts),
                        std::ref(res[c]));
    parse_chunk(all.substr(cut[0], cut[1] - cut[0]), order, opts, res[0]);
    for (auto& t : pool) t.join();
  }

  std::size_t line_base = head_lines, total = 0;
  std::vector<std::uint32_t> maxima(order, 0);
  for (const ChunkResult& r : res) {
    if (r.fail_line) throw DataError(path + ":" + std::to_string(line_base + r.fail_line) + ": " + r.fail_what);
    line_base += r.lines;
    total += r.values.size();
    for (std::size_t k = 0; k < order; ++k) maxima[k] = std::max(maxima[k], r.maxima[k]);
  }
  if (total == 0) throw DataError(path + ": no data lines (empty tensor)");

  std::vector<std::uint32_t> dims = opts.dims_override.empty() ? maxima : opts.dims_override;
  if (!opts.dims_override.empty()) {
    if (opts.dims_override.size() != order) throw DataError("dims override arity does not match order");
    for (std::size_t k = 0; k < order; ++k)
      if (maxima[k] > dims[k])
        throw DataError(path + ": index " + std::to_string(maxima[k]) + " exceeds dim " + std::to_string(dims[k]) +
                        " in mode " + std::to_string(k + 1));
  }
  std::vector<std::uint32_t> coords;
  std::vector<double> values;
  if (nchunks == 1) {
    coords = std::move(res[0].coords);
    values = std::move(res[0].values);
  } else {
    coords.reserve(total * order);
    values.reserve(total);
    for (ChunkResult& r : res) {
      coords.insert(coords.end(), r.coords.begin(), r.coords.end());
      values.insert(values.end(), r.values.begin(), r.values.end());
      r = ChunkResult{};
    }
  }
  return CooTensor(Shape(std::move(dims)), std::move(coords), std::move(values));
}

void CooTensor::save_delimited(const std::string& path) const {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw DataError("cannot write '" + path + "'");
  // "c_1 c_2 ... c_N %.17g\n" per entry (sptensor.cpp:197-209), formatted in
  // parallel blocks and written in entry order.
  const std::size_t n = nnz(), ord = order();
  const std::size_t block = 1u << 18;
  const std::size_t nblocks = (n + block - 1) / block;
  const std::size_t width = std::max<std::size_t>(1, std::min<std::size_t>(host_threads(), nblocks));
  bool ok = true;
  std::vector<std::string> out(width);
  for (std::size_t b0 = 0; b0 < nblocks && ok; b0 += width) {
    auto fmt = [&](std::size_t slot) {
      std::string& s = out[slot];
      s.clear();
      const std::size_t b = b0 + slot;
      if (b >= nblocks) return;
      const std::size_t e0 = b * block, e1 = std::min(n, e0 + block);
      s.reserve((e1 - e0) * (ord * 8 + 26));
      char buf[64];
      for (std::size_t e = e0; e < e1; ++e) {
        const std::uint32_t* c = coords_.data() + e * ord;
        for (std::size_t k = 0; k < ord; ++k) {
          const auto [p, ec] = std::to_chars(buf, buf + sizeof buf, c[k]);
          (void)ec;
          s.append(buf, p);
          s.push_back(' ');
        }
        const int len = std::snprintf(buf, sizeof buf, "%.17g", values_[e]);
        s.append(buf, static_cast<std::size_t>(len));
        s.push_back('\n');
      }
    };
    std::vector<std::thread> pool;
    for (std::size_t slot = 1; slot < width; ++slot) pool.emplace_back(fmt, slot);
    fmt(0);
    for (auto& t : pool) t.join();
    for (const std::string& s : out)
      if (!s.empty() && std::fwrite(s.data(), 1, s.size(), f) != s.size()) ok = false;
  }
  if (std::fclose(f) != 0 || !ok) throw DataError("write failed for '" + path + "'");
}

// ---- binary model file (model.cpp:178-280) --------------------------------
//
// "SPTUCKM\0", u32 version 1, u32 order, u64 dims[N], u64 J[N], u64 R, then
// B^(1..N) and A^(1..N) row-major as f64; all little-endian.

namespace {

constexpr char kModelMagic[8] = {'S', 'P', 'T', 'U', 'C', 'K', 'M', '\0'};
constexpr std::uint32_t kModelVersion = 1;

void put_le(std::string& s, std::uint64_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) s.push_back(static_cast<char>((v >> (8 * i)) & 0xFF));
}

struct Reader {
  const std::string& b;
  std::size_t at = 0;
  std::uint64_t le(int bytes) {
    if (b.size() - at < static_cast<std::size_t>(bytes)) throw FormatError("model file truncated");
    std::uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<std::uint64_t>(static_cast<unsigned char>(b[at + i])) << (8 * i);
    at += static_cast<std::size_t>(bytes);
    return v;
  }
};

}  // namespace

void TuckerModel::save(const std::string& path) const {
  std::string s(kModelMagic, sizeof kModelMagic);
  put_le(s, kModelVersion, 4);
  put_le(s, order(), 4);
  for (std::size_t n = 0; n < order(); ++n) put_le(s, shape_.dim(n), 8);
  for (std::size_t n = 0; n < order(); ++n) put_le(s, ranks_.J[n], 8);
  put_le(s, ranks_.r_core, 8);
  for (const Matrix& b : kruskal_)
    for (const double v : b.data()) put_le(s, std::bit_cast<std::uint64_t>(v), 8);
  for (const Matrix& a : factors_)
    for (const double v : a.data()) put_le(s, std::bit_cast<std::uint64_t>(v), 8);
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw DataError("cannot write '" + path + "'");
  const bool ok = std::fwrite(s.data(), 1, s.size(), f) == s.size();
  if (std::fclose(f) != 0 || !ok) throw DataError("write failed for '" + path + "'");
}

TuckerModel TuckerModel::load(const std::string& path) {
  const std::string bytes = read_file(path, "cannot open");
  if (bytes.size() < sizeof kModelMagic || std::memcmp(bytes.data(), kModelMagic, sizeof kModelMagic) != 0)
    throw FormatError("not a model file (bad magic)");
  Reader in{bytes, sizeof kModelMagic};
  const std::uint32_t version = static_cast<std::uint32_t>(in.le(4));
  if (version != kModelVersion) throw FormatError("unsupported model format version " + std::to_string(version));
  const std::uint32_t order = static_cast<std::uint32_t>(in.le(4));
  if (order < 2 || order > 64) throw FormatError("implausible tensor order");
  auto u32_field = [&](const char* what) {
    const std::uint64_t v = in.le(8);
    if (v < 1 || v > std::numeric_limits<std::uint32_t>::max()) throw FormatError(what);
    return static_cast<std::uint32_t>(v);
  };
  std::vector<std::uint32_t> dims(order);
  for (auto& d : dims) d = u32_field("dimension out of range");
  Ranks ranks;
  ranks.J.resize(order);
  for (auto& j : ranks.J) j = u32_field("rank out of range");
  ranks.r_core = u32_field("R_core out of range");
  TuckerModel m = [&] {
    try {
      return TuckerModel(Shape(dims), ranks);
    } catch (const DomainError& e) {
      throw FormatError(std::string("model file violates invariants: ") + e.what());
    }
  }();
  for (Matrix& b : m.kruskal_)
    for (double& v : b.data()) v = std::bit_cast<double>(in.le(8));
  for (Matrix& a : m.factors_)
    for (double& v : a.data()) v = std::bit_cast<double>(in.le(8));
  if (in.at != bytes.size()) throw FormatError("trailing bytes after model payload");
  if (!m.all_finite()) throw FormatError("model file holds non-finite parameters");
  m.refresh_core_cache();
  return m;
}

// ---- metrics CSV (eval.cpp:47-146) ----------------------------------------

namespace {

constexpr const char* kMetricsHeader =
    "epoch,core_s,factor_s,total_s,train_rmse,train_mae,test_rmse,test_mae,peak_bytes,comm_bytes";

std::string fmt17(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

template <class T>
T parse_field(std::string_view f, const std::string& path, std::size_t lineno, const char* what) {
  T v{};
  const auto [p, ec] = std::from_chars(f.data(), f.data() + f.size(), v);
  if (ec != std::errc{} || p != f.data() + f.size())
    throw FormatError(path + ":" + std::to_string(lineno) + ": " + what);
  return v;
}

}  // namespace

void write_metrics_csv(const std::string& path, const std::vector<EpochMetrics>& rows,
                       const std::vector<std::string>& config_comments) {
  std::string s;
  for (const std::string& c : config_comments) s += "# " + c + "\n";
  s += kMetricsHeader;
  s += '\n';
  for (const EpochMetrics& r : rows) {
    s += std::to_string(r.epoch);
    for (const double v : {r.core_s, r.factor_s, r.total_s, r.train_rmse, r.train_mae, r.test_rmse, r.test_mae})
      s += "," + fmt17(v);
    s += "," + std::to_string(r.peak_bytes) + "," + std::to_string(r.comm_bytes) + "\n";
  }
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw DataError("cannot write '" + path + "'");
  const bool ok = std::fwrite(s.data(), 1, s.size(), f) == s.size();
  if (std::fclose(f) != 0 || !ok) throw DataError("write failed for '" + path + "'");
}

std::vector<EpochMetrics> parse_metrics_csv(const std::string& path, std::vector<std::string>* comments) {
  std::ifstream in(path);
  if (!in) throw DataError("cannot open '" + path + "'");
  std::vector<EpochMetrics> rows;
  std::string line;
  std::size_t lineno = 0;
  bool header = false;
  while (std::getline(in, line)) {
    ++lineno;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty()) continue;
    if (line[0] == '#') {
      if (comments) {
        std::string c = line.substr(1);
        if (!c.empty() && c.front() == ' ') c.erase(0, 1);
        comments->push_back(std::move(c));
      }
      continue;
    }
    if (!header) {
      if (line != kMetricsHeader) throw FormatError(path + ": unexpected metrics header '" + line + "'");
      header = true;
      continue;
    }
    std::string_view f[11];
    std::size_t nf = 0, start = 0;
    const std::string_view sv(line);
    for (std::size_t i = 0; i <= sv.size(); ++i)
      if (i == sv.size() || sv[i] == ',') {
        if (nf < 11) f[nf] = sv.substr(start, i - start);
        ++nf;
        start = i + 1;
      }
    if (nf != 10) throw FormatError(path + ":" + std::to_string(lineno) + ": expected 10 fields");
    EpochMetrics r;
    r.epoch = static_cast<std::size_t>(parse_field<std::uint64_t>(f[0], path, lineno, "bad integer field"));
    double* d[7] = {&r.core_s, &r.factor_s, &r.total_s, &r.train_rmse, &r.train_mae, &r.test_rmse, &r.test_mae};
    for (int k = 0; k < 7; ++k) *d[k] = parse_field<double>(f[k + 1], path, lineno, "bad numeric field");
    r.peak_bytes = parse_field<std::uint64_t>(f[8], path, lineno, "bad integer field");
    r.comm_bytes = parse_field<std::uint64_t>(f[9], path, lineno, "bad integer field");
    rows.push_back(r);
  }
  if (!header) throw FormatError(path + ": missing metrics header");
  return rows;
}

}  // namespace sptucker
