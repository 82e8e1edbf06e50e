// sgdt_session.cu -- the C-ABI (include/sgdt.h): session setup, device
// layout build, model/RNG transfer, and the per-epoch drivers.
//
// The drivers follow the reference's control flow exactly:
//   core phase   update_core_epoch   (core_optimizer.cpp:112-257)
//   factor phase update_factor_epoch (factor_optimizer.cpp:101-273)
//   train loop   train               (trainer.cpp:66-125)
//   eval         rmse_mae            (eval.cpp:15-33)
// Every kernel is enqueued on the session stream; the public epoch calls
// synchronise once at the end to map the device divergence flag onto
// NumericError, as sgdt_step / all_finite do (core_optimizer.cpp:93-98,
// trainer.cpp:101-103).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "sgdt_internal.cuh"

struct sgdt_session : sgdt::Session {};

namespace sgdt {

namespace {
thread_local std::string g_error;

__global__ void build_entry_copy_kernel(const uint32_t* __restrict__ coords,
                                        const double* __restrict__ values, uint64_t nnz,
                                        int order, uint32_t* idx, float* val) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    for (int k = 0; k < order; ++k) idx[static_cast<uint64_t>(k) * nnz + e] = coords[e * order + k] - 1;
    val[e] = static_cast<float>(values[e]);
  }
}

// Mode-sorted copy: record q of mode n is entry perm[q] (sptensor.cpp:102-117).
// len records of the slice: record q is entry perm[q] (src copy has nnz records).
__global__ void gather_mode_copy_kernel(const uint32_t* __restrict__ src_idx,
                                        const float* __restrict__ src_val,
                                        const uint32_t* __restrict__ perm, uint64_t nnz, uint64_t len,
                                        int order, uint32_t* idx, float* val) {
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < len;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t e = perm[q];
    for (int k = 0; k < order; ++k)
      idx[static_cast<uint64_t>(k) * len + q] = src_idx[static_cast<uint64_t>(k) * nnz + e];
    val[q] = src_val[e];
  }
}

// Kept records of a row-subset epoch: record q is the mode-order record at
// position out[q] (the mode copy holds `len` records).
__global__ void gather_subset_kernel(const uint32_t* __restrict__ src_idx, const float* __restrict__ src_val,
                                     uint64_t len, const uint32_t* __restrict__ out, uint64_t T, int order,
                                     uint32_t* idx, float* val) {
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < T;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t p = out[q];
    for (int k = 0; k < order; ++k)
      idx[static_cast<uint64_t>(k) * T + q] = src_idx[static_cast<uint64_t>(k) * len + p];
    val[q] = src_val[p];
  }
}

__global__ void cast_d2f_kernel(const double* __restrict__ src, float* dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    dst[i] = static_cast<float>(src[i]);
}

__global__ void cast_f2d_kernel(const float* __restrict__ src, double* dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    dst[i] = static_cast<double>(src[i]);
}

__global__ void iota32_kernel(uint32_t* p, uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    p[i] = static_cast<uint32_t>(i);
}

unsigned grid_for(uint64_t n, int num_sms) {
  uint64_t g = (n + 255) / 256;
  const uint64_t cap = static_cast<uint64_t>(num_sms) * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<unsigned>(g);
}

// memcpy on several host threads (pinned staging -> pageable caller memory).
void parallel_copy(void* dst, const void* src, uint64_t bytes) {
  const uint64_t kMin = 4ull << 20;
  unsigned t = std::min<unsigned>(8, std::max(1u, std::thread::hardware_concurrency()));
  if (bytes < kMin * 2 || t < 2) {
    std::memcpy(dst, src, bytes);
    return;
  }
  t = static_cast<unsigned>(std::min<uint64_t>(t, bytes / kMin));
  std::vector<std::thread> th;
  for (unsigned i = 1; i < t; ++i) {
    const uint64_t b = bytes * i / t, e = bytes * (i + 1) / t;
    th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, e - b); });
  }
  std::memcpy(dst, src, bytes / t);
  for (auto& x : th) x.join();
}

// std::mt19937_64 seeding (the default engine state before set_rng).
void mt_seed(uint64_t* x, uint64_t seed) {
  x[0] = seed;
  for (uint32_t i = 1; i < 312; ++i) x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + i;
}

template <class T>
int dalloc(T** p, uint64_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  SGDT_CUDA(cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T)));
  return SGDT_OK;
}

#define TRY(x)            \
  do {                    \
    int rc_ = (x);        \
    if (rc_) return rc_;  \
  } while (0)

int validate_desc(const sgdt_tensor_desc* d, const char* what) {
  if (!d) return fail(SGDT_ERR_DOMAIN, std::string(what) + ": null tensor");
  if (d->order < 2 || d->order > kMaxOrder)
    return fail(SGDT_ERR_DOMAIN, std::string(what) + ": order must be in [2, 8]");
  if (d->nnz == 0) return fail(SGDT_ERR_DATA, std::string(what) + ": tensor has no entries");
  if (d->nnz > 0xFFFFFFFFull)
    return fail(SGDT_ERR_DATA, std::string(what) + ": entry count exceeds the 32-bit id space");
  for (int k = 0; k < d->order; ++k)
    if (d->dims[k] < 1) return fail(SGDT_ERR_DOMAIN, std::string(what) + ": every dim must be >= 1");
  // coordinate ranges are checked on the device after the upload (check_coords)
  return SGDT_OK;
}

// Row offsets of mode n (CooTensor::mode_offsets, sptensor.cpp:107-111) and,
// when no permutation is supplied, the stable counting sort itself.
void host_mode_layout(const sgdt_tensor_desc* d, int n, std::vector<uint64_t>& off,
                      std::vector<uint32_t>* perm) {
  const uint32_t dim = d->dims[n];
  const int order = d->order;
  off.assign(static_cast<size_t>(dim) + 1, 0);
  for (uint64_t e = 0; e < d->nnz; ++e) off[d->coords[e * order + n]]++;
  for (size_t i = 1; i <= dim; ++i) off[i] += off[i - 1];
  if (!perm) return;
  perm->resize(d->nnz);
  std::vector<uint64_t> cursor(off.begin(), off.end() - 1);
  for (uint64_t e = 0; e < d->nnz; ++e) (*perm)[cursor[d->coords[e * order + n] - 1]++] = static_cast<uint32_t>(e);
}

// Rows shorter than this are processed one row per lane / lane group
// (Chunk::pad = 1); 64 measured best on config 2 (16: +9%, 256: +5%).
constexpr uint64_t kShortRow = 64;

// nnz-balanced chunk schedule over the mode-sorted entries [qb, qe) (the
// whole order for a single-GPU session; this rank's partition_even slice for a
// sharded one): whole rows packed greedily up to chunk_size, longer rows cut
// into pieces of chunk_size.  A row cut by the slice edges is not finalised
// here: its pieces are summed into an export slot for the cross-rank merge
// (the rank-ordered boundary merge of factor_optimizer.cpp:247-270).  Chunk
// bounds are relative to qb.
void build_chunks(const std::vector<uint64_t>& off, uint64_t qb, uint64_t qe, uint32_t chunk_size,
                  std::vector<Chunk>& chunks, std::vector<SplitRow>& splits, uint32_t& n_pieces, ShardPlan& sp,
                  uint32_t& n_big) {
  n_big = 0;
  chunks.clear();
  splits.clear();
  n_pieces = 0;
  sp = ShardPlan{};
  sp.qb = qb;
  sp.qe = qe;
  if (qb >= qe) return;
  const size_t rows = off.size() - 1;
  // row holding position q: off[i] <= q < off[i+1]
  auto row_of = [&](uint64_t q) {
    return static_cast<size_t>(std::upper_bound(off.begin(), off.end(), q) - off.begin()) - 1;
  };
  const size_t r0 = row_of(qb), r1 = row_of(qe - 1);
  sp.row_lo = static_cast<uint32_t>(off[r0] < qb ? r0 + 1 : r0);
  sp.row_hi = static_cast<uint32_t>(r1 + 1);
  bool open = false;
  Chunk cur{0, 0, -1, 0};
  auto close = [&] {
    if (open) chunks.push_back(cur);
    open = false;
  };
  for (size_t i = r0; i <= r1 && i < rows; ++i) {
    if (off[i + 1] == off[i]) continue;
    const uint64_t b = std::max(off[i], qb) - qb, e = std::min(off[i + 1], qe) - qb, cnt = e - b;
    const bool cut = off[i] < qb || off[i + 1] > qe;
    if (cut || cnt > chunk_size) {
      close();
      SplitRow sr{static_cast<uint32_t>(i), n_pieces, 0, 0};
      if (cut) {
        sr.pad = 1 + sp.n_export;
        sp.export_rows[sp.n_export++] = static_cast<uint32_t>(i);
      }
      for (uint64_t p = b; p < e; p += chunk_size) {
        const uint64_t pe = std::min<uint64_t>(p + chunk_size, e);
        chunks.push_back(Chunk{static_cast<uint32_t>(p), static_cast<uint32_t>(pe), static_cast<int32_t>(n_pieces++), 0});
        ++sr.count;
      }
      splits.push_back(sr);
      continue;
    }
    if (open && (e - cur.begin) > chunk_size) close();
    if (!open) {
      cur = Chunk{static_cast<uint32_t>(b), static_cast<uint32_t>(e), -1, 1};
      open = true;
    } else {
      cur.end = static_cast<uint32_t>(e);
    }
    if (cnt >= kShortRow) cur.pad = 0;  // pad = 1: every row of the chunk is short
  }
  close();
  // split rows with many pieces first (one CTA each in factor_split_kernel)
  std::stable_partition(splits.begin(), splits.end(), [](const SplitRow& r) { return r.count > kSplitBig; });
  for (const SplitRow& r : splits) n_big += r.count > kSplitBig;
}

// Intra-row order of the mode-n copy.  The reference visits a row's entries in
// entry order (CooTensor::mode_perm, sptensor.cpp:102-117); the row's update
// is a sum over them, so any order is the same row update up to fp32
// summation order (inside the per-batch tolerance).  Entries of a row are
// ordered by the coordinate of a secondary mode m: the smallest other mode
// whose Q table does not fit in L1, so that a warp's gathers of Q^(m) form
// runs of equal rows (hot Zipf rows coalesce) and sweep the rest in address
// order.  Ties keep the given order (stable radix sort).  -1: keep the order.
int secondary_mode(const Session& s, int n) {
  bool largest = false;
  if (const char* e = std::getenv("SGDT_ROW_ORDER")) {  // diagnostics: entry | largest
    if (std::strcmp(e, "entry") == 0) return -1;
    largest = std::strcmp(e, "largest") == 0;
  }
  const uint64_t l1_bytes = 160 * 1024;
  int best = -1;
  for (int k = 0; k < s.order; ++k) {
    if (k == n || static_cast<uint64_t>(s.dims[k]) * s.RP * sizeof(float) <= l1_bytes) continue;
    if (best < 0 || (largest ? s.dims[k] > s.dims[best] : s.dims[k] < s.dims[best])) best = k;
  }
  return best;
}

// Sort key of entry perm[q] in the mode-n copy: i_n, then (t >= 0) the
// tiny-table coordinate i_t, then the secondary coordinate i_m:
// (i_n << 32) | (i_t * dim_m + i_m).
__global__ void row_key_kernel(const uint32_t* __restrict__ idx, uint64_t nnz, const uint32_t* __restrict__ perm,
                               uint64_t len, int n, int m, int t, uint32_t dim_m, uint64_t* __restrict__ keys) {
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < len;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t e = perm[q];
    uint32_t lo = m >= 0 ? idx[static_cast<uint64_t>(m) * nnz + e] : 0u;
    if (t >= 0) lo += idx[static_cast<uint64_t>(t) * nnz + e] * dim_m;
    keys[q] = (static_cast<uint64_t>(idx[static_cast<uint64_t>(n) * nnz + e]) << 32) | lo;
  }
}

// Inside a row, entries are ordered by the coordinate of a tiny other mode
// (<= kTinyRows rows, e.g. the 50-row fourth mode of BASELINE config 3)
// before the secondary one, so a warp's lanes share that table's rows
// (shared-memory broadcasts instead of ~15 bank-conflicted wavefronts per
// random-row LDS) while long rows keep long runs of the secondary mode.
// Config 3: modes 0-2 4.36 -> 4.18 ms.  With a 2200-row "tiny" table (config
// 2) the secondary runs break and it is slower, hence the bound.
// SGDT_ROW_ORDER=notiny turns it off (A/B runs).
constexpr uint32_t kTinyRows = 256;
int tiny_mode(const Session& s, int n, int m) {
  if (m < 0) return -1;
  if (const char* e = std::getenv("SGDT_ROW_ORDER"))
    if (std::strcmp(e, "notiny") == 0) return -1;
  int best = -1;
  for (int k = 0; k < s.order; ++k)
    if (k != n && k != m && (best < 0 || s.dims[k] < s.dims[best])) best = k;
  if (best < 0 || s.dims[best] > kTinyRows || static_cast<uint64_t>(s.dims[best]) * s.dims[m] >= (1ull << 32))
    return -1;
  return best;
}

__global__ void iota_u32_kernel(uint32_t* p, uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    p[i] = static_cast<uint32_t>(i);
}

// off[r] = first position of row r in the key-sorted order, off[dim] = len
// (CooTensor::mode_offsets, sptensor.cpp:107-111), from the sorted keys.
__global__ void row_offsets_kernel(const uint64_t* __restrict__ keys, uint64_t len, uint32_t dim,
                                   uint64_t* __restrict__ off) {
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q <= len;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int64_t cur = q < len ? static_cast<int64_t>(keys[q] >> 32) : static_cast<int64_t>(dim);
    const int64_t prev = q > 0 ? static_cast<int64_t>(keys[q - 1] >> 32) : -1;
    for (int64_t r = prev + 1; r <= cur; ++r) off[r] = q;
  }
}

struct DimList {
  uint32_t d[kMaxOrder];
};
// Coordinate ranges of an uploaded record copy (idx = coord - 1, so 0 wraps
// past every bound): the smallest offending entry id, or ~0.
__global__ void check_coords_kernel(const uint32_t* __restrict__ idx, uint64_t nnz, int order, DimList dims,
                                    unsigned long long* first_bad) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    for (int k = 0; k < order; ++k)
      if (idx[static_cast<uint64_t>(k) * nnz + e] >= dims.d[k]) atomicMin(first_bad, static_cast<unsigned long long>(e));
}

// The smallest entry id with a coordinate outside [1, I_k] (~0 if none).
int first_bad_coord(Session& s, const RecordCopy& rc, const sgdt_tensor_desc* d, uint64_t* out) {
  DimList dl{};
  for (int k = 0; k < d->order; ++k) dl.d[k] = d->dims[k];
  unsigned long long* bad = nullptr;
  TRY(dalloc(&bad, 1));
  unsigned long long h = ~0ull;
  int rc_ = SGDT_OK;
  if (cudaMemcpyAsync(bad, &h, sizeof h, cudaMemcpyHostToDevice, s.stream) != cudaSuccess) rc_ = SGDT_ERR_INTERNAL;
  if (rc_ == SGDT_OK) {
    check_coords_kernel<<<grid_for(rc.nnz, s.num_sms), 256, 0, s.stream>>>(rc.idx, rc.nnz, d->order, dl, bad);
    ++s.launches;
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(&h, bad, sizeof h, cudaMemcpyDeviceToHost, s.stream) != cudaSuccess ||
        cudaStreamSynchronize(s.stream) != cudaSuccess)
      rc_ = SGDT_ERR_INTERNAL;
  }
  cudaFree(bad);
  if (rc_ != SGDT_OK) {
    cudaGetLastError();
    return fail(SGDT_ERR_INTERNAL, "coordinate check failed");
  }
  *out = h;
  return SGDT_OK;
}

int first_duplicate(Session& s, const RecordCopy& rc, const sgdt_tensor_desc* d, uint64_t* out);

// The CooTensor constructor's checks (sptensor.cpp:80-100): entry by entry,
// range before duplicate, the first failing entry decides the DataError.
// Entries below the first out-of-range one are all in range, so a duplicate
// found below it is the reference's answer.
int check_entries(Session& s, const RecordCopy& rc, const sgdt_tensor_desc* d, const std::string& prefix) {
  uint64_t bad = ~0ull, dup = ~0ull;
  TRY(first_bad_coord(s, rc, d, &bad));
  TRY(first_duplicate(s, rc, d, &dup));
  if (dup < bad) return fail(SGDT_ERR_DATA, prefix + "entry " + std::to_string(dup) + ": duplicate coordinate");
  if (bad != ~0ull) return fail(SGDT_ERR_DATA, prefix + "entry " + std::to_string(bad) + ": coordinate out of range");
  return SGDT_OK;
}

// (An out-of-range value overflows its field and can give two different
// tuples one key; equal tuples always share a key, and a repeat that such a
// key separates from its partner lies above an out-of-range entry, which
// the reference reports first -- check_entries takes the smaller id.)
// Duplicate detection (the CooTensor constructor's hash-set pass,
// sptensor.cpp:90-100), as a sort: every entry's coordinates are packed into
// a bit string of sum_k ceil(log2 I_k) bits (equal strings <=> equal
// coordinates, no 2^64 limit), sorted least-significant word first by stable
// radix sorts of (word, entry id) pairs, and each entry equal to its sorted
// predecessor is a repeat.  The reference throws at the first entry id whose
// key was seen before; ids ascend inside a group of equal keys (iota start,
// stable passes), so that is the smallest id that is not first of its group.
struct KeyLayout {
  uint32_t shift[kMaxOrder];  // bit offset of mode k's field
};
__global__ void dup_key_word_kernel(const uint32_t* __restrict__ idx, uint64_t nnz, int order, KeyLayout kl,
                                    int word, const uint32_t* __restrict__ perm, uint64_t* __restrict__ keys) {
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < nnz;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t e = perm[q];
    uint64_t w = 0;
    for (int k = 0; k < order; ++k) {
      const uint64_t v = idx[static_cast<uint64_t>(k) * nnz + e];
      const int lo = static_cast<int>(kl.shift[k]) - 64 * word;  // field start relative to this word
      if (lo >= 0 && lo < 64) w |= v << lo;
      else if (lo < 0 && lo > -32) w |= v >> (-lo);
    }
    keys[q] = w;
  }
}

__global__ void dup_adjacent_kernel(const uint32_t* __restrict__ idx, uint64_t nnz, int order,
                                    const uint32_t* __restrict__ perm, unsigned long long* first_dup) {
  for (uint64_t q = 1 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < nnz;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t a = perm[q - 1], b = perm[q];
    bool eq = true;
    for (int k = 0; k < order && eq; ++k)
      eq = idx[static_cast<uint64_t>(k) * nnz + a] == idx[static_cast<uint64_t>(k) * nnz + b];
    if (eq) atomicMin(first_dup, static_cast<unsigned long long>(b));
  }
}

int first_duplicate(Session& s, const RecordCopy& rc, const sgdt_tensor_desc* d, uint64_t* out) {
  const uint64_t nnz = rc.nnz;
  const char* what = "duplicate check";
  *out = ~0ull;
  if (nnz < 2) return SGDT_OK;
  KeyLayout kl{};
  uint32_t total = 0;
  for (int k = 0; k < d->order; ++k) {
    kl.shift[k] = total;
    uint32_t b = 0;
    while (b < 32 && (1ull << b) < d->dims[k]) ++b;
    total += b;
  }
  const int words = std::max<int>(1, static_cast<int>((total + 63) / 64));
  uint64_t *k_in = nullptr, *k_out = nullptr;
  uint32_t *p_in = nullptr, *p_out = nullptr;
  unsigned long long* first = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  unsigned long long h = ~0ull;
  int rc_ = SGDT_OK;
  do {
    if ((rc_ = dalloc(&k_in, nnz)) || (rc_ = dalloc(&k_out, nnz)) || (rc_ = dalloc(&p_in, nnz)) ||
        (rc_ = dalloc(&p_out, nnz)) || (rc_ = dalloc(&first, 1)))
      break;
    iota_u32_kernel<<<grid_for(nnz, s.num_sms), 256, 0, s.stream>>>(p_in, nnz);
    for (int w = 0; w < words && rc_ == SGDT_OK; ++w) {
      const int bits = std::max<int>(1, std::min<int>(64, static_cast<int>(total) - 64 * w));
      dup_key_word_kernel<<<grid_for(nnz, s.num_sms), 256, 0, s.stream>>>(rc.idx, nnz, d->order, kl, w, p_in,
                                                                          k_in);
      size_t need = 0;
      if (cub::DeviceRadixSort::SortPairs(nullptr, need, k_in, k_out, p_in, p_out, static_cast<int64_t>(nnz), 0,
                                          bits, s.stream) != cudaSuccess) {
        rc_ = fail(SGDT_ERR_INTERNAL, std::string(what) + ": sort sizing failed");
        break;
      }
      if (need > tmp_bytes) {
        if (tmp) cudaFree(tmp);
        tmp = nullptr;
        if (cudaMalloc(&tmp, need) != cudaSuccess) {
          cudaGetLastError();
          rc_ = fail(SGDT_ERR_CONFIG, std::string(what) + ": out of device memory");
          break;
        }
        tmp_bytes = need;
      }
      if (cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k_in, k_out, p_in, p_out, static_cast<int64_t>(nnz), 0,
                                          bits, s.stream) != cudaSuccess) {
        rc_ = fail(SGDT_ERR_INTERNAL, std::string(what) + ": sort failed");
        break;
      }
      std::swap(p_in, p_out);
    }
    if (rc_) break;
    if (cudaMemcpyAsync(first, &h, sizeof h, cudaMemcpyHostToDevice, s.stream) != cudaSuccess) {
      rc_ = fail(SGDT_ERR_INTERNAL, "duplicate check: copy failed");
      break;
    }
    dup_adjacent_kernel<<<grid_for(nnz, s.num_sms), 256, 0, s.stream>>>(rc.idx, nnz, d->order, p_in, first);
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(&h, first, sizeof h, cudaMemcpyDeviceToHost, s.stream) != cudaSuccess ||
        cudaStreamSynchronize(s.stream) != cudaSuccess) {
      cudaGetLastError();
      rc_ = fail(SGDT_ERR_INTERNAL, std::string(what) + " failed");
    }
    s.launches += 2 + words;
  } while (false);
  for (void* p : {(void*)k_in, (void*)k_out, (void*)p_in, (void*)p_out, (void*)first, tmp})
    if (p) cudaFree(p);
  if (rc_) return rc_;
  *out = h;
  return SGDT_OK;
}

// The whole mode-n order and its row offsets on the device (CooTensor::
// mode_perm / mode_offsets, sptensor.cpp:102-117, built by a stable radix sort
// instead of the host counting sort): rows ascending by i_n; inside a row by
// the secondary mode's coordinate, ties in the given order.  host_perm: the
// caller's bucket order (or null: entry order).  off (host) receives the
// I_n + 1 offsets.  SGDT_ERR_CONFIG: nnz exceeds the sort's 31-bit item count
// (the caller falls back to the host counting sort).
int build_mode_order(Session& s, int n, const uint32_t* host_perm, uint32_t* d_perm, std::vector<uint64_t>& off) {
  const uint64_t len = s.nnz;
  if (len > static_cast<uint64_t>(INT_MAX)) return SGDT_ERR_CONFIG;
  const int m = secondary_mode(s, n);
  if (host_perm) {
    SGDT_CUDA(cudaMemcpyAsync(d_perm, host_perm, len * sizeof(uint32_t), cudaMemcpyHostToDevice, s.stream));
  } else {
    iota_u32_kernel<<<grid_for(len, s.num_sms), 256, 0, s.stream>>>(d_perm, len);
    SGDT_CUDA(cudaGetLastError());
  }
  const bool sort = !(host_perm && m < 0);  // a given bucket order needs no sort without a secondary key
  uint64_t *k_in = nullptr, *k_out = nullptr, *d_off = nullptr;
  uint32_t* p_out = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int end_bit = 32;
  while (end_bit < 64 && (1ull << (end_bit - 32)) < s.dims[n]) ++end_bit;
  const int begin_bit = m >= 0 ? 0 : 32;
  int rc = SGDT_OK;
  off.assign(static_cast<size_t>(s.dims[n]) + 1, 0);
  do {
    if ((rc = dalloc(&k_in, len)) != SGDT_OK) break;
    if ((rc = dalloc(&d_off, off.size())) != SGDT_OK) break;
    const int t = tiny_mode(s, n, m);
    row_key_kernel<<<grid_for(len, s.num_sms), 256, 0, s.stream>>>(s.train_rec.idx, s.nnz, d_perm, len, n, m, t,
                                                                    m >= 0 ? s.dims[m] : 0u, k_in);
    if (cudaGetLastError() != cudaSuccess) {
      rc = fail(SGDT_ERR_INTERNAL, "row_key_kernel launch failed");
      break;
    }
    const uint64_t* keys = k_in;
    if (sort && len > 1) {
      if ((rc = dalloc(&k_out, len)) != SGDT_OK) break;
      if ((rc = dalloc(&p_out, len)) != SGDT_OK) break;
      if (cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in, k_out, d_perm, p_out, static_cast<int>(len),
                                          begin_bit, end_bit, s.stream) != cudaSuccess ||
          cudaMalloc(&tmp, tmp_bytes) != cudaSuccess ||
          cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k_in, k_out, d_perm, p_out, static_cast<int>(len),
                                          begin_bit, end_bit, s.stream) != cudaSuccess ||
          cudaMemcpyAsync(d_perm, p_out, len * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s.stream) !=
              cudaSuccess) {
        cudaGetLastError();
        rc = fail(SGDT_ERR_INTERNAL, "mode order (radix sort) failed");
        break;
      }
      keys = k_out;
    }
    row_offsets_kernel<<<grid_for(len + 1, s.num_sms), 256, 0, s.stream>>>(keys, len, s.dims[n], d_off);
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(off.data(), d_off, off.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost, s.stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(s.stream) != cudaSuccess) {
      cudaGetLastError();
      rc = fail(SGDT_ERR_INTERNAL, "mode offsets failed");
    }
  } while (false);
  for (void* p : {(void*)k_in, (void*)k_out, (void*)d_off, (void*)p_out, tmp})
    if (p) cudaFree(p);
  return rc;
}

// This rank's export record {n_export, row0, row1, g0[RP], g1[RP]} into slot
// `rank` of every rank's record buffer (local and peers, P2P stores).
struct RecordDst {
  double* p[kMaxPeers + 1];
  int n;
};
__global__ void publish_record_kernel(const double* __restrict__ xport, uint32_t n_export, uint32_t row0,
                                      uint32_t row1, uint32_t stride, int rank, RecordDst dst) {
  for (uint32_t i = threadIdx.x; i < stride; i += blockDim.x) {
    const double v = i == 0 ? static_cast<double>(n_export)
                            : (i == 1 ? static_cast<double>(row0) : (i == 2 ? static_cast<double>(row1) : xport[i - 3]));
    for (int d = 0; d < dst.n; ++d) dst.p[d][static_cast<uint64_t>(rank) * stride + i] = v;
  }
}

// Rank-ordered merge of the records for up to 2 rows this rank finalises
// (merge_boundary of the host driver, on the device): g[i] = sum over ranks
// ascending, over their slots in order, of the partials of rows[i].
__global__ void merge_records_kernel(const double* __restrict__ rec, int world, uint32_t stride, uint32_t RP,
                                     uint32_t k, uint32_t row0, uint32_t row1, uint32_t* rows_out,
                                     double* g_out) {
  const uint32_t t = threadIdx.x;
  if (t < k) rows_out[t] = t == 0 ? row0 : row1;
  for (uint32_t x = t; x < k * RP; x += blockDim.x) {
    const uint32_t i = x / RP, r = x % RP;
    const double row = static_cast<double>(i == 0 ? row0 : row1);
    double g = 0.0;
    for (int w = 0; w < world; ++w) {
      const double* R0 = rec + static_cast<uint64_t>(w) * stride;
      const uint32_t ne = static_cast<uint32_t>(R0[0]);
      for (uint32_t q = 0; q < ne && q < 2; ++q)
        if (R0[1 + q] == row) g += R0[3 + q * RP + r];
    }
    g_out[x] = g;
  }
}

int upload_record_copy(Session& s, const sgdt_tensor_desc* d, RecordCopy& rc, uint32_t** d_coords_keep,
                       double** d_values_keep) {
  const uint64_t nnz = d->nnz;
  const int order = d->order;
  uint32_t* d_coords;
  double* d_values;
  TRY(dalloc(&d_coords, nnz * order));
  TRY(dalloc(&d_values, nnz));
  SGDT_CUDA(cudaMemcpyAsync(d_coords, d->coords, nnz * order * sizeof(uint32_t), cudaMemcpyHostToDevice,
                            s.stream));
  SGDT_CUDA(cudaMemcpyAsync(d_values, d->values, nnz * sizeof(double), cudaMemcpyHostToDevice, s.stream));
  rc.nnz = nnz;
  TRY(dalloc(&rc.idx, nnz * order));
  TRY(dalloc(&rc.val, nnz));
  build_entry_copy_kernel<<<grid_for(nnz, s.num_sms), 256, 0, s.stream>>>(d_coords, d_values, nnz, order,
                                                                           rc.idx, rc.val);
  SGDT_CUDA(cudaGetLastError());
  if (d_coords_keep) {
    *d_coords_keep = d_coords;
  } else {
    SGDT_CUDA(cudaStreamSynchronize(s.stream));
    cudaFree(d_coords);
  }
  if (d_values_keep) {
    *d_values_keep = d_values;
  } else {
    SGDT_CUDA(cudaStreamSynchronize(s.stream));
    cudaFree(d_values);
  }
  return SGDT_OK;
}

void free_session(sgdt_session* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  auto F = [](void* p) {
    if (p) cudaFree(p);
  };
  F(s->train_rec.idx);
  F(s->train_rec.val);
  F(s->test_rec.idx);
  F(s->test_rec.val);
  for (int n = 0; n < kMaxOrder; ++n) {
    F(s->mode[n].rec.idx);
    F(s->mode[n].rec.val);
    F(s->mode[n].row_ptr);
    F(s->mode[n].chunks);
    F(s->mode[n].splits);
    RowSubset& rs = s->mode[n].subset;
    for (void* p : {(void*)rs.sub_off, (void*)rs.target, (void*)rs.pos, (void*)rs.link, (void*)rs.kprev,
                    (void*)rs.lprev, (void*)rs.out, (void*)rs.rec.idx, (void*)rs.rec.val, (void*)rs.chunks,
                    (void*)rs.splits})
      F(p);
    F(s->P.A[n]);
    F(s->P.B[n]);
    F(s->P.Q[n]);
  }
  F(s->piece_partials);
  F(s->export_buf);
  F(s->xrec);
  F(s->merge_rows);
  F(s->merge_g);
  F(s->d_peers);
  F(s->mt);
  F(s->mt_out);
  F(s->mt_tent);
  F(s->mt_flag);
  F(s->jump.J);
  F(s->jump.st);
  F(s->jump.part);
  F(s->pool);
  F(s->head);
  F(s->draw_j);
  F(s->link);
  F(s->kprev);
  F(s->lprev);
  F(s->dval);
  F(s->batch);
  F(s->cs_a);
  F(s->cs_c);
  F(s->cs_xhat);
  F(s->cs_x);
  F(s->cs_part);
  F(s->core_x);
  F(s->core_part);
  F(s->core_ticket);
  F(s->pool_pre);
  F(s->d_delta);
  if (s->h_delta) cudaFreeHost(s->h_delta);
  F(s->cb_a);
  F(s->cb_c);
  F(s->cb_xh);
  F(s->cb_x);
  F(s->ev_part);
  F(s->ev_out);
  F(s->flag);
  F(s->stage);
  F(s->xfer);
  if (s->h_ev_out) cudaFreeHost(s->h_ev_out);
  if (s->h_flag) cudaFreeHost(s->h_flag);
  for (auto& e : s->ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {s->ev_start, s->ev_core, s->ev_samp, s->ev_bar})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : s->tev) cudaEventDestroy(e);
  for (cudaEvent_t e : s->ev_copy)
    if (e) cudaEventDestroy(e);
  if (s->hx) cudaFreeHost(s->hx);
  if (s->side) cudaStreamDestroy(s->side);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

int ensure_batch_capacity(Session& s, uint64_t m) {
  const uint64_t need = 2 * m * s.order;
  if (need <= s.batch_cap) return SGDT_OK;
  SGDT_CUDA(cudaStreamSynchronize(s.stream));
  SGDT_CUDA(cudaStreamSynchronize(s.side));
  auto F = [](void* p) {
    if (p) cudaFree(p);
  };
  F(s.batch);
  F(s.draw_j);
  F(s.link);
  F(s.kprev);
  F(s.lprev);
  F(s.dval);
  TRY(dalloc(&s.batch, need));
  TRY(dalloc(&s.draw_j, m));
  TRY(dalloc(&s.link, m));
  TRY(dalloc(&s.kprev, m));
  TRY(dalloc(&s.lprev, m));
  TRY(dalloc(&s.dval, m));
  s.batch_cap = need;
  s.last_batch = nullptr;
  s.last_batch_len = 0;
  return SGDT_OK;
}

int ensure_core_capacity(Session& s, uint64_t m) {
  if (m <= s.cs_cap) return SGDT_OK;
  SGDT_CUDA(cudaStreamSynchronize(s.stream));
  SGDT_CUDA(cudaStreamSynchronize(s.side));
  auto F = [](void* p) {
    if (p) cudaFree(p);
  };
  F(s.cs_a);
  F(s.cs_c);
  F(s.cs_xhat);
  F(s.cs_x);
  F(s.cs_part);
  uint32_t js = 0;
  for (int k = 0; k < s.order; ++k) js = std::max(js, s.J[k]);
  // per-CTA slices of ceil(m / grid) samples rounded up to 4; a_s in float4 groups
  const uint64_t mm = m + 4ull * s.num_sms;
  TRY(dalloc(&s.cs_a, mm * ((js + 3u) & ~3u)));
  TRY(dalloc(&s.cs_c, mm * s.RP));
  TRY(dalloc(&s.cs_xhat, mm));
  TRY(dalloc(&s.cs_x, mm));
  // stamped partials (2 x js x grid) + every CTA's own copy of the new-column words (2 x grid x js u64)
  TRY(dalloc(&s.cs_part, 3ull * s.num_sms * js));
  SGDT_CUDA(cudaMemsetAsync(s.cs_part, 0, 3ull * s.num_sms * js * sizeof(ulonglong2), s.stream));
  s.core_stamp = 0;
  s.cs_cap = m;
  return SGDT_OK;
}

int check_core_hyper(const Session& s, const sgdt_core_hyper* h, uint64_t* m_out) {
  if (!h) return fail(SGDT_ERR_DOMAIN, "core hyper is null");
  if (h->lr < 0.0) return fail(SGDT_ERR_DOMAIN, "core learning rate must be non-negative");
  if (!(h->reg >= 0.0) && h->lr > 0.0) return fail(SGDT_ERR_DOMAIN, "sgd_step: regularization must be non-negative");
  const uint64_t m = h->batch_m == 0 ? s.nnz : h->batch_m;
  if (m > s.nnz) return fail(SGDT_ERR_DOMAIN, "core batch size exceeds training nnz");
  *m_out = m;
  return SGDT_OK;
}

int check_factor_hyper(const sgdt_factor_hyper* h) {
  if (!h) return fail(SGDT_ERR_DOMAIN, "factor hyper is null");
  if (!(h->row_fraction > 0.0 && h->row_fraction <= 1.0))
    return fail(SGDT_ERR_DOMAIN, "row fraction must lie in (0,1]");
  if (h->lr < 0.0) return fail(SGDT_ERR_DOMAIN, "factor learning rate must be non-negative");
  if (h->lr > 0.0 && h->reg < 0.0) return fail(SGDT_ERR_DOMAIN, "sgd_step: regularization must be non-negative");
  return SGDT_OK;
}

// Draw the Psi of one epoch (one per mode when resampling) into `buf`.
int enqueue_sample(Session& s, const sgdt_core_hyper& h, uint64_t m, uint32_t* buf, cudaStream_t st) {
  NvtxRange range("sgdt:sample");
  const int draws = (h.resample_per_mode && h.batch_m != 0) ? s.order : 1;
  for (int n = 0; n < draws; ++n) TRY(launch_sampler(s, m, buf + static_cast<uint64_t>(n) * m, st));
  return SGDT_OK;
}

// Set up a blocked core phase over an already drawn Psi: the slice of it this
// rank reduces (sharded: partition_even(m, world)[rank], the reference's
// worker slices, scheduler.cpp:34-46; else all of it), the column-block
// width and the launch geometry (sgdt_core_blocked.cu).
int begin_core_plan(Session& s, const sgdt_core_hyper& h, uint64_t m, const uint32_t* batch, int per_mode,
                    bool sharded, uint32_t block) {
  CorePlan& pl = s.cplan;
  pl = CorePlan{};
  pl.batch = batch;
  pl.per_mode = per_mode;
  pl.m = m;
  pl.world = sharded ? s.world : 1;
  pl.rank = sharded ? s.rank : 0;
  const uint64_t base = m / pl.world, rem = m % pl.world;
  pl.lo = pl.rank * base + std::min<uint64_t>(pl.rank, rem);
  pl.hi = pl.lo + base + (static_cast<uint64_t>(pl.rank) < rem ? 1 : 0);
  pl.lr = h.lr;
  pl.reg = h.reg;
  const uint64_t len = pl.hi - pl.lo;
  const int grid_est = static_cast<int>(std::min<uint64_t>(std::max<uint64_t>((len + 255) / 256, 1), s.num_sms));
  pl.T = core_block_width(s, len, grid_est, pl.world > 1 ? 20.0 : 5.0, block);
  TRY(plan_core_geometry(s, pl));
  if (pl.T < s.R && len > s.cb_cap) {  // per-sample state kept across the blocks of a mode
    auto F = [](void* p) {
      if (p) cudaFree(p);
    };
    SGDT_CUDA(cudaStreamSynchronize(s.stream));
    F(s.cb_a);
    F(s.cb_c);
    F(s.cb_xh);
    F(s.cb_x);
    s.cb_a = s.cb_c = s.cb_xh = s.cb_x = nullptr;
    s.cb_cap = 0;
    TRY(dalloc(&s.cb_a, len * pl.js4));
    TRY(dalloc(&s.cb_c, len * s.RP));
    TRY(dalloc(&s.cb_xh, len));
    TRY(dalloc(&s.cb_x, len));
    s.cb_cap = len;
  }
  pl.valid = true;
  pl.next = 0;
  return SGDT_OK;
}

// Enqueue one core phase (no host sync).  `presampled` != nullptr: Psi was
// already drawn (run-ahead on the side stream) into that buffer.
int enqueue_core(Session& s, const sgdt_core_hyper& h, uint64_t m, const uint32_t* presampled = nullptr) {
  if (h.lr == 0.0) return SGDT_OK;  // frozen phase: bit-exact no-op, no RNG
  NvtxRange range("sgdt:core");
  TRY(ensure_batch_capacity(s, m));
  TRY(ensure_core_capacity(s, m));
  const bool per_mode = h.resample_per_mode && h.batch_m != 0;
  const uint32_t* batch = presampled;
  s.core_slot = presampled && presampled != s.batch ? 1 : 0;
  if (!batch) {
    if (h.batch_m == 0) {
      iota32_kernel<<<grid_for(m, s.num_sms), 256, 0, s.stream>>>(s.batch, m);
      SGDT_CUDA(cudaGetLastError());
      ++s.launches;
      s.last_batch = s.batch;
      s.last_batch_len = m;
    } else {
      TRY(enqueue_sample(s, h, m, s.batch, s.stream));
    }
    batch = s.batch;
  }
  if (s.core_mode == 1) {  // blocked steps, this rank alone (replicated semantics)
    TRY(begin_core_plan(s, h, m, batch, per_mode ? 1 : 0, false, 0));
    for (uint32_t k = 0; k < s.cplan.steps; ++k) TRY(launch_core_block_step(s, k));
    s.cplan.valid = false;
    return SGDT_OK;
  }
  return launch_core(s, h, batch, m, per_mode ? 1 : 0);
}

// The row-subset plan of mode n for `fraction`: keep_i = max(1,
// llround(f |bucket_i|)) per non-empty row (factor_optimizer.cpp:409-411), the
// subset row offsets and its chunk schedule.  Rebuilt only when f changes.
int ensure_subset(Session& s, int n, double fraction) {
  RowSubset& rs = s.mode[n].subset;
  if (rs.fraction == fraction) return SGDT_OK;
  SGDT_CUDA(cudaStreamSynchronize(s.stream));
  const std::vector<uint64_t>& off = s.h_row_ptr[n];
  std::vector<uint64_t> sub(off.size(), 0);
  for (size_t i = 0; i + 1 < off.size(); ++i) {
    const uint64_t bs = off[i + 1] - off[i];
    uint64_t keep = 0;
    if (bs) keep = std::max<uint64_t>(1, static_cast<uint64_t>(std::llround(fraction * static_cast<double>(bs))));
    sub[i + 1] = sub[i] + keep;
  }
  const uint64_t T = sub.back();
  auto F = [](void* p) {
    if (p) cudaFree(p);
  };
  for (void* p : {(void*)rs.sub_off, (void*)rs.target, (void*)rs.pos, (void*)rs.link, (void*)rs.kprev,
                  (void*)rs.lprev, (void*)rs.out, (void*)rs.rec.idx, (void*)rs.rec.val, (void*)rs.chunks,
                  (void*)rs.splits})
    F(p);
  rs = RowSubset{};
  rs.total = T;
  std::vector<uint32_t> sub32(sub.begin(), sub.end());
  TRY(dalloc(&rs.sub_off, sub32.size()));
  SGDT_CUDA(cudaMemcpy(rs.sub_off, sub32.data(), sub32.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
  for (uint32_t** p : {&rs.target, &rs.pos, &rs.link, &rs.kprev, &rs.lprev, &rs.out}) TRY(dalloc(p, T));
  rs.rec.nnz = T;
  TRY(dalloc(&rs.rec.idx, T * s.order));
  TRY(dalloc(&rs.rec.val, T));
  std::vector<Chunk> chunks;
  std::vector<SplitRow> splits;
  ShardPlan sp;
  build_chunks(sub, 0, T, s.chunk_size, chunks, splits, rs.n_pieces, sp, rs.n_big_splits);
  rs.n_chunks = static_cast<uint32_t>(chunks.size());
  rs.n_splits = static_cast<uint32_t>(splits.size());
  TRY(dalloc(&rs.chunks, chunks.size()));
  TRY(dalloc(&rs.splits, splits.size()));
  if (!chunks.empty())
    SGDT_CUDA(cudaMemcpy(rs.chunks, chunks.data(), chunks.size() * sizeof(Chunk), cudaMemcpyHostToDevice));
  if (!splits.empty())
    SGDT_CUDA(cudaMemcpy(rs.splits, splits.data(), splits.size() * sizeof(SplitRow), cudaMemcpyHostToDevice));
  if (rs.n_pieces > s.piece_cap) {
    F(s.piece_partials);
    s.piece_cap = rs.n_pieces;
    TRY(dalloc(&s.piece_partials, static_cast<uint64_t>(s.piece_cap) * s.RP));
  }
  rs.fraction = fraction;
  return SGDT_OK;
}

// mode_ev (nullable): events recorded before each mode's launches.
int enqueue_factor(Session& s, const sgdt_factor_hyper& h, bool time_modes, cudaEvent_t* mode_ev = nullptr) {
  if (h.lr == 0.0) return SGDT_OK;
  const bool subset = h.row_fraction < 1.0;
  if (subset && s.world > 1)
    return fail(SGDT_ERR_CONFIG, "row_fraction < 1 is not supported by the sharded (multi-GPU) factor phase");
  for (int n = 0; n < s.order; ++n) {
    NvtxRange range(nvtx_mode_name(n));
    if (time_modes) SGDT_CUDA(cudaEventRecord(s.ev[4 + n], s.stream));
    if (mode_ev) SGDT_CUDA(cudaEventRecord(mode_ev[n], s.stream));
    if (subset) {
      // the draws of mode n follow mode n-1's update in the RNG stream
      // (factor_optimizer.cpp:384-424); they do not depend on the model.
      TRY(ensure_subset(s, n, h.row_fraction));
      RowSubset& rs = s.mode[n].subset;
      TRY(launch_row_subsets(s, n, rs, s.stream));
      if (rs.total) {
        gather_subset_kernel<<<grid_for(rs.total, s.num_sms), 256, 0, s.stream>>>(
            s.mode[n].rec.idx, s.mode[n].rec.val, s.mode[n].rec.nnz, rs.out, rs.total, s.order, rs.rec.idx,
            rs.rec.val);
        SGDT_CUDA(cudaGetLastError());
        ++s.launches;
      }
    }
    TRY(launch_factor_mode(s, n, h, subset));
  }
  return SGDT_OK;
}

// A pending sgdt_sample_ahead draw: setters discard it (the state they
// install replaces the RNG/pool it advanced); other RNG consumers would draw
// out of the reference order, so they are refused until a core phase takes it.
int settle_ahead(Session& s, bool discard, const char* who) {
  if (!s.ahead_valid) return SGDT_OK;
  SGDT_CUDA(cudaStreamSynchronize(s.side));
  if (discard) {
    s.ahead_valid = false;
    return SGDT_OK;
  }
  return fail(SGDT_ERR_CONFIG, std::string(who) + ": a sgdt_sample_ahead draw is pending; run sgdt_core_epoch_async first");
}

constexpr uint64_t kTimedEpochs = 1024;

int ensure_timing_events(Session& s, uint64_t n) {
  while (s.tev.size() < n) {
    cudaEvent_t e = nullptr;
    SGDT_CUDA(cudaEventCreate(&e));
    s.tev.push_back(e);
  }
  return SGDT_OK;
}

int sync_and_flag(Session& s) {
  SGDT_CUDA(cudaMemcpyAsync(s.h_flag, s.flag, sizeof(int), cudaMemcpyDeviceToHost, s.stream));
  SGDT_CUDA(cudaStreamSynchronize(s.stream));
  if (*s.h_flag && !std::getenv("SGDT_DEBUG_IGNORE_FLAG")) {
    SGDT_CUDA(cudaMemsetAsync(s.flag, 0, sizeof(int), s.stream));
    return fail(SGDT_ERR_NUMERIC, "sgd_step: non-finite parameter or gradient; reduce the learning rate (flag " +
                                      std::to_string(*s.h_flag) + ")");
  }
  return SGDT_OK;
}

}  // namespace

void set_error(const std::string& msg) { g_error = msg; }
int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}

}  // namespace sgdt

using namespace sgdt;

extern "C" {

const char* sgdt_last_error(void) { return g_error.c_str(); }
const char* sgdt_version(void) { return "sgdt 0.2 (sm_100a)"; }

int sgdt_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void sgdt_partition_even(uint64_t count, uint64_t workers, uint64_t* begins, uint64_t* ends) {
  const uint64_t base = count / workers, rem = count % workers;
  uint64_t at = 0;
  for (uint64_t w = 0; w < workers; ++w) {
    const uint64_t len = base + (w < rem ? 1 : 0);
    begins[w] = at;
    ends[w] = at + len;
    at += len;
  }
}

__global__ void mode_key_kernel(const uint32_t* __restrict__ idx, uint64_t nnz, int n, uint32_t* __restrict__ key) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    key[e] = idx[static_cast<uint64_t>(n) * nnz + e];
}

// off[r] = first position of bucket r in the sorted coordinates (0-based
// rows; the host view is 1-based: offsets[i] = end of bucket i).
__global__ void bucket_offsets_kernel(const uint32_t* __restrict__ keys, uint64_t len, uint32_t dim,
                                      uint64_t* __restrict__ off) {
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q <= len;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int64_t cur = q < len ? static_cast<int64_t>(keys[q]) : static_cast<int64_t>(dim);
    const int64_t prev = q > 0 ? static_cast<int64_t>(keys[q - 1]) : -1;
    for (int64_t r = prev + 1; r <= cur; ++r) off[r] = q;
  }
}

int sgdt_tensor_layout(const sgdt_tensor_desc* d, int device, uint32_t* const* perm_out,
                       uint64_t* const* offsets_out) {
  TRY(validate_desc(d, "tensor"));
  if (device >= 0) SGDT_CUDA(cudaSetDevice(device));
  Session tmp;
  SGDT_CUDA(cudaGetDevice(&tmp.device));
  SGDT_CUDA(cudaDeviceGetAttribute(&tmp.num_sms, cudaDevAttrMultiProcessorCount, tmp.device));
  SGDT_CUDA(cudaStreamCreateWithFlags(&tmp.stream, cudaStreamNonBlocking));
  RecordCopy rc;
  uint32_t *key = nullptr, *key2 = nullptr, *ids = nullptr, *ids2 = nullptr;
  uint64_t* off = nullptr;
  void* scratch = nullptr;
  const uint64_t nnz = d->nnz;
  int r = [&]() -> int {
    TRY(upload_record_copy(tmp, d, rc, nullptr, nullptr));
    TRY(check_entries(tmp, rc, d, ""));
    if (!perm_out && !offsets_out) return SGDT_OK;
    TRY(dalloc(&key, nnz));
    TRY(dalloc(&key2, nnz));
    TRY(dalloc(&ids, nnz));
    TRY(dalloc(&ids2, nnz));
    size_t cap = 0;
    for (int n = 0; n < d->order; ++n) {
      const uint32_t dim = d->dims[n];
      int bits = 1;
      while (bits < 32 && (1ull << bits) < dim) ++bits;
      mode_key_kernel<<<grid_for(nnz, tmp.num_sms), 256, 0, tmp.stream>>>(rc.idx, nnz, n, key);
      iota_u32_kernel<<<grid_for(nnz, tmp.num_sms), 256, 0, tmp.stream>>>(ids, nnz);
      SGDT_CUDA(cudaGetLastError());
      size_t need = 0;
      SGDT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need, key, key2, ids, ids2, static_cast<int64_t>(nnz), 0,
                                                bits, tmp.stream));
      if (need > cap) {
        if (scratch) cudaFree(scratch);
        scratch = nullptr;
        SGDT_CUDA(cudaMalloc(&scratch, need));
        cap = need;
      }
      // stable: ids ascending inside each bucket (sptensor.cpp:102-117)
      SGDT_CUDA(cub::DeviceRadixSort::SortPairs(scratch, cap, key, key2, ids, ids2, static_cast<int64_t>(nnz), 0,
                                                bits, tmp.stream));
      if (perm_out && perm_out[n])
        SGDT_CUDA(cudaMemcpyAsync(perm_out[n], ids2, nnz * sizeof(uint32_t), cudaMemcpyDeviceToHost, tmp.stream));
      if (offsets_out && offsets_out[n]) {
        if (off) cudaFree(off);
        off = nullptr;
        TRY(dalloc(&off, static_cast<uint64_t>(dim) + 1));
        bucket_offsets_kernel<<<grid_for(nnz + 1, tmp.num_sms), 256, 0, tmp.stream>>>(key2, nnz, dim, off);
        SGDT_CUDA(cudaGetLastError());
        // host offsets[0] = 0, offsets[i] = end of bucket i (1-based rows)
        SGDT_CUDA(cudaMemcpyAsync(offsets_out[n], off, (static_cast<uint64_t>(dim) + 1) * sizeof(uint64_t),
                                  cudaMemcpyDeviceToHost, tmp.stream));
      }
      SGDT_CUDA(cudaStreamSynchronize(tmp.stream));
    }
    return SGDT_OK;
  }();
  for (void* p : {(void*)rc.idx, (void*)rc.val, (void*)key, (void*)key2, (void*)ids, (void*)ids2, (void*)off, scratch})
    if (p) cudaFree(p);
  cudaStreamDestroy(tmp.stream);
  tmp.stream = nullptr;
  return r;
}

int sgdt_session_create(const sgdt_tensor_desc* train, const sgdt_tensor_desc* test, const uint32_t* J,
                        uint32_t R, int device, sgdt_session** out) {
  return sgdt_session_create_shard(train, test, J, R, device, 0, 1, out);
}

int sgdt_session_create_shard(const sgdt_tensor_desc* train, const sgdt_tensor_desc* test, const uint32_t* J,
                              uint32_t R, int device, int rank, int world, sgdt_session** out) {
  if (!out) return fail(SGDT_ERR_DOMAIN, "out is null");
  if (world < 1 || rank < 0 || rank >= world) return fail(SGDT_ERR_DOMAIN, "shard: need 0 <= rank < world");
  *out = nullptr;
  TRY(validate_desc(train, "train"));
  if (test) {
    TRY(validate_desc(test, "test"));
    if (test->order != train->order) return fail(SGDT_ERR_DOMAIN, "rmse_mae: order mismatch between model and data");
    for (int k = 0; k < train->order; ++k)
      if (test->dims[k] > train->dims[k])
        return fail(SGDT_ERR_DOMAIN, "rmse_mae: data exceeds the model's shape in mode " + std::to_string(k + 1));
  }
  if (!J) return fail(SGDT_ERR_DOMAIN, "ranks: J is null");
  if (R < 1) return fail(SGDT_ERR_DOMAIN, "ranks: R_core must be >= 1");
  if (R > SGDT_MAX_RCORE) return fail(SGDT_ERR_CONFIG, "R_core > 32 is not supported by the device kernels");
  for (int k = 0; k < train->order; ++k) {
    if (J[k] < 1) return fail(SGDT_ERR_DOMAIN, "ranks: every J_n must be >= 1");
    if (J[k] < R) return fail(SGDT_ERR_DOMAIN, "ranks: R_core must satisfy R_core <= J_n");
    if (J[k] > SGDT_MAX_J) return fail(SGDT_ERR_CONFIG, "J_n > 64 is not supported by the device kernels");
  }
  if (device >= 0) SGDT_CUDA(cudaSetDevice(device));
  auto* s = new sgdt_session();
  SGDT_CUDA(cudaGetDevice(&s->device));
  cudaDeviceProp prop{};
  SGDT_CUDA(cudaGetDeviceProperties(&prop, s->device));
  s->num_sms = prop.multiProcessorCount;
  int rc = [&]() -> int {
    SGDT_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    // the side stream (run-ahead sampler, model copy-out) has the highest
    // priority so its short kernels are dispatched between the blocks of the
    // factor kernels instead of after them
    int prio_lo = 0, prio_hi = 0;
    SGDT_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    SGDT_CUDA(cudaStreamCreateWithPriority(&s->side, cudaStreamNonBlocking, prio_hi));
    for (auto& e : s->ev) SGDT_CUDA(cudaEventCreate(&e));
    for (cudaEvent_t* e : {&s->ev_start, &s->ev_core, &s->ev_samp, &s->ev_bar})
      SGDT_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    s->order = train->order;
    s->nnz = train->nnz;
    s->rank = rank;
    s->world = world;
    s->R = R;
    s->RP = (R + 3) & ~3u;
    // Factor chunk size: 2048 entries, 4096 for the one-entry-per-lane kernels
    // (RP <= 12) when every warp gets >= 40 chunks of 2048 (config 3: 450M
    // entries, 109.8 -> 112.4 G updates/s); longer chunks cost balance on
    // smaller tensors (config 2: 96.3 -> 93.7) and the wide kernels (config 4
    // 41.2 -> 34.4, config 5 21.7 -> 20.3).  SGDT_CHUNK_SIZE overrides.
    if (s->RP <= 12 && s->nnz / world / 2048 >= 40ull * s->num_sms * 24) s->chunk_size = 4096;
    if (const char* cs = std::getenv("SGDT_CHUNK_SIZE")) {
      const long v = std::strtol(cs, nullptr, 10);
      if (v >= 1 && v <= (1L << 24)) s->chunk_size = static_cast<uint32_t>(v);
    }
    s->P.order = s->order;
    s->P.R = R;
    s->P.RP = s->RP;
    for (int k = 0; k < s->order; ++k) {
      s->dims[k] = s->P.dims[k] = train->dims[k];
      s->J[k] = s->P.J[k] = J[k];
    }
    // records: entry order (kept for Psi gathers + train RMSE) and per mode
    TRY(upload_record_copy(*s, train, s->train_rec, nullptr, nullptr));
    TRY(check_entries(*s, s->train_rec, train, "train: "));
    uint32_t max_pieces = 0;
    std::vector<uint64_t> off;
    std::vector<uint32_t> perm;
    uint32_t* d_perm = nullptr;
    TRY(dalloc(&d_perm, s->nnz));
    for (int n = 0; n < s->order; ++n) {
      ModePlan& mp = s->mode[n];
      const uint32_t* given = (train->mode_perm && train->mode_perm[n]) ? train->mode_perm[n] : nullptr;
      {
        const int rc = build_mode_order(*s, n, given, d_perm, off);
        if (rc == SGDT_ERR_CONFIG) {  // beyond the device sort's item count: host counting sort
          host_mode_layout(train, n, off, given ? nullptr : &perm);
          if (!given) given = perm.data();
          SGDT_CUDA(cudaMemcpyAsync(d_perm, given, s->nnz * sizeof(uint32_t), cudaMemcpyHostToDevice, s->stream));
        } else if (rc != SGDT_OK) {
          cudaFree(d_perm);
          return rc;
        }
      }
      // this rank's slice of the mode-n order (partition_even, scheduler.cpp:34-46)
      uint64_t qb = 0, qe = 0;
      {
        std::vector<uint64_t> pb(world), pe(world);
        sgdt_partition_even(s->nnz, static_cast<uint64_t>(world), pb.data(), pe.data());
        qb = pb[rank];
        qe = pe[rank];
      }
      const uint64_t len = qe - qb;
      mp.rec.nnz = len;
      TRY(dalloc(&mp.rec.idx, len * s->order));
      TRY(dalloc(&mp.rec.val, len));
      if (len) {
        gather_mode_copy_kernel<<<grid_for(len, s->num_sms), 256, 0, s->stream>>>(
            s->train_rec.idx, s->train_rec.val, d_perm + qb, s->nnz, len, s->order, mp.rec.idx, mp.rec.val);
        SGDT_CUDA(cudaGetLastError());
      }
      s->h_row_ptr[n] = off;
      std::vector<uint32_t> rp(off.size());
      for (size_t i = 0; i < off.size(); ++i) rp[i] = static_cast<uint32_t>(off[i]);
      TRY(dalloc(&mp.row_ptr, rp.size()));
      SGDT_CUDA(cudaMemcpyAsync(mp.row_ptr, rp.data(), rp.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                s->stream));
      std::vector<Chunk> chunks;
      std::vector<SplitRow> splits;
      build_chunks(off, qb, qe, s->chunk_size, chunks, splits, mp.n_pieces, mp.shard, mp.n_big_splits);
      mp.rows_nonempty = 0;
      for (size_t i = 0; i + 1 < off.size(); ++i) mp.rows_nonempty += off[i + 1] > off[i];
      mp.rows_empty = s->dims[n] - mp.rows_nonempty;
      mp.n_chunks = static_cast<uint32_t>(chunks.size());
      mp.n_splits = static_cast<uint32_t>(splits.size());
      TRY(dalloc(&mp.chunks, chunks.size()));
      TRY(dalloc(&mp.splits, splits.size()));
      if (!chunks.empty())
        SGDT_CUDA(cudaMemcpyAsync(mp.chunks, chunks.data(), chunks.size() * sizeof(Chunk), cudaMemcpyHostToDevice,
                                  s->stream));
      if (!splits.empty())
        SGDT_CUDA(cudaMemcpyAsync(mp.splits, splits.data(), splits.size() * sizeof(SplitRow),
                                  cudaMemcpyHostToDevice, s->stream));
      max_pieces = std::max(max_pieces, mp.n_pieces);
      SGDT_CUDA(cudaStreamSynchronize(s->stream));  // host vectors are reused
    }
    cudaFree(d_perm);
    if (test) {
      s->nnz_test = test->nnz;
      TRY(upload_record_copy(*s, test, s->test_rec, nullptr, nullptr));
      TRY(check_entries(*s, s->test_rec, test, "test: "));
    }
    // model
    uint64_t stage = 0;
    for (int k = 0; k < s->order; ++k) {
      TRY(dalloc(&s->P.A[k], static_cast<uint64_t>(s->dims[k]) * s->J[k]));
      TRY(dalloc(&s->P.B[k], static_cast<uint64_t>(s->J[k]) * R));
      TRY(dalloc(&s->P.Q[k], static_cast<uint64_t>(s->dims[k]) * s->RP));
      SGDT_CUDA(cudaMemsetAsync(s->P.A[k], 0, static_cast<uint64_t>(s->dims[k]) * s->J[k] * sizeof(float), s->stream));
      SGDT_CUDA(cudaMemsetAsync(s->P.B[k], 0, static_cast<uint64_t>(s->J[k]) * R * sizeof(float), s->stream));
      SGDT_CUDA(cudaMemsetAsync(s->P.Q[k], 0, static_cast<uint64_t>(s->dims[k]) * s->RP * sizeof(float), s->stream));
      stage = std::max<uint64_t>(stage, static_cast<uint64_t>(s->dims[k]) * s->J[k]);
      stage = std::max<uint64_t>(stage, static_cast<uint64_t>(s->J[k]) * R);
    }
    TRY(dalloc(&s->stage, stage));
    s->stage_cap = stage;
    s->piece_cap = std::max<uint32_t>(max_pieces, 1);
    TRY(dalloc(&s->piece_partials, static_cast<uint64_t>(s->piece_cap) * s->RP));
    TRY(dalloc(&s->export_buf, 2ull * s->RP));
    s->rec_stride = 3 + 2 * s->RP;
    TRY(dalloc(&s->xrec, static_cast<uint64_t>(world) * s->rec_stride));
    TRY(dalloc(&s->merge_rows, 2));
    TRY(dalloc(&s->merge_g, 2ull * s->RP));
    TRY(dalloc(&s->d_peers, kMaxOrder));
    // blocked / sharded core phase: exchange buffer, per-CTA vectors, ticket
    s->core_x_stride = core_block_max_kstride(*s);
    TRY(dalloc(&s->core_x, 2ull * world * s->core_x_stride));
    SGDT_CUDA(cudaMemsetAsync(s->core_x, 0, 2ull * world * s->core_x_stride * sizeof(double), s->stream));
    // per-CTA vectors, then one slot per 16-CTA reduction group
    TRY(dalloc(&s->core_part, static_cast<uint64_t>(s->num_sms + s->num_sms / 16 + 1) * s->core_x_stride));
    TRY(dalloc(&s->core_ticket, 64));  // [0]: groups done, [1 + g]: CTAs of group g done
    SGDT_CUDA(cudaMemsetAsync(s->core_ticket, 0, 64 * sizeof(unsigned), s->stream));
    s->core_peer_x[rank] = s->core_x;
    if (const char* e = std::getenv("SGDT_CORE")) s->core_mode = std::strcmp(e, "blocked") == 0 ? 1 : 0;
    // sampler
    TRY(dalloc(&s->mt, 313));
    uint64_t mt[313];
    mt_seed(mt, 5489u);
    mt[312] = 312;
    SGDT_CUDA(cudaMemcpy(s->mt, mt, sizeof mt, cudaMemcpyHostToDevice));
    TRY(dalloc(&s->pool, s->nnz));
    TRY(dalloc(&s->head, s->nnz));
    SGDT_CUDA(cudaMemsetAsync(s->head, 0, s->nnz * sizeof(unsigned long long), s->stream));
    // eval + flag
    TRY(dalloc(&s->ev_part, 2ull * s->num_sms * 8));
    TRY(dalloc(&s->ev_out, 2));
    TRY(dalloc(&s->flag, 1));
    SGDT_CUDA(cudaMemsetAsync(s->flag, 0, sizeof(int), s->stream));
    SGDT_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s->h_ev_out), 2 * sizeof(double), cudaHostAllocDefault));
    SGDT_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s->h_flag), sizeof(int), cudaHostAllocDefault));
    SGDT_CUDA(cudaStreamSynchronize(s->stream));
    return SGDT_OK;
  }();
  if (rc) {
    const std::string keep = g_error;
    free_session(s);
    g_error = keep;
    return rc;
  }
  *out = s;
  return SGDT_OK;
}

void sgdt_session_destroy(sgdt_session* s) { free_session(s); }

void* sgdt_session_stream(sgdt_session* s) { return s ? static_cast<void*>(s->stream) : nullptr; }

int sgdt_set_model(sgdt_session* s, const double* const* A, const double* const* B) {
  if (!s || !A || !B) return fail(SGDT_ERR_DOMAIN, "set_model: null argument");
  SGDT_CUDA(cudaSetDevice(s->device));
  for (int k = 0; k < s->order; ++k) {
    const uint64_t na = static_cast<uint64_t>(s->dims[k]) * s->J[k];
    const uint64_t nb = static_cast<uint64_t>(s->J[k]) * s->R;
    SGDT_CUDA(cudaMemcpyAsync(s->stage, A[k], na * sizeof(double), cudaMemcpyHostToDevice, s->stream));
    cast_d2f_kernel<<<grid_for(na, s->num_sms), 256, 0, s->stream>>>(s->stage, s->P.A[k], na);
    SGDT_CUDA(cudaMemcpyAsync(s->stage, B[k], nb * sizeof(double), cudaMemcpyHostToDevice, s->stream));
    cast_d2f_kernel<<<grid_for(nb, s->num_sms), 256, 0, s->stream>>>(s->stage, s->P.B[k], nb);
    SGDT_CUDA(cudaGetLastError());
    s->launches += 2;
  }
  for (int k = 0; k < s->order; ++k) TRY(launch_q_refresh(*s, k));
  SGDT_CUDA(cudaStreamSynchronize(s->stream));
  return SGDT_OK;
}

int sgdt_get_model(sgdt_session* s, double* const* A, double* const* B) {
  if (!s || (!A && !B)) return fail(SGDT_ERR_DOMAIN, "get_model: null argument");
  SGDT_CUDA(cudaSetDevice(s->device));
  for (int k = 0; k < s->order; ++k) {
    const uint64_t na = static_cast<uint64_t>(s->dims[k]) * s->J[k];
    const uint64_t nb = static_cast<uint64_t>(s->J[k]) * s->R;
    if (A) {
      cast_f2d_kernel<<<grid_for(na, s->num_sms), 256, 0, s->stream>>>(s->P.A[k], s->stage, na);
      SGDT_CUDA(cudaMemcpyAsync(A[k], s->stage, na * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
      ++s->launches;
    }
    if (B) {
      cast_f2d_kernel<<<grid_for(nb, s->num_sms), 256, 0, s->stream>>>(s->P.B[k], s->stage, nb);
      SGDT_CUDA(cudaMemcpyAsync(B[k], s->stage, nb * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
      ++s->launches;
    }
    SGDT_CUDA(cudaGetLastError());
  }
  SGDT_CUDA(cudaStreamSynchronize(s->stream));
  return SGDT_OK;
}

int sgdt_set_rng(sgdt_session* s, const uint64_t* mt312, uint32_t pos) {
  if (!s || !mt312) return fail(SGDT_ERR_DOMAIN, "set_rng: null argument");
  if (pos > 312) return fail(SGDT_ERR_DOMAIN, "set_rng: position out of range");
  SGDT_CUDA(cudaSetDevice(s->device));
  TRY(settle_ahead(*s, true, "set_rng"));
  uint64_t st[313];
  std::memcpy(st, mt312, 312 * sizeof(uint64_t));
  st[312] = pos;
  SGDT_CUDA(cudaMemcpyAsync(s->mt, st, sizeof st, cudaMemcpyHostToDevice, s->stream));
  SGDT_CUDA(cudaStreamSynchronize(s->stream));
  return SGDT_OK;
}

int sgdt_get_rng(sgdt_session* s, uint64_t* mt312, uint32_t* pos) {
  if (!s || !mt312 || !pos) return fail(SGDT_ERR_DOMAIN, "get_rng: null argument");
  SGDT_CUDA(cudaSetDevice(s->device));
  SGDT_CUDA(cudaStreamSynchronize(s->side));
  uint64_t st[313];
  SGDT_CUDA(cudaMemcpyAsync(st, s->mt, sizeof st, cudaMemcpyDeviceToHost, s->stream));
  SGDT_CUDA(cudaStreamSynchronize(s->stream));
  std::memcpy(mt312, st, 312 * sizeof(uint64_t));
  *pos = static_cast<uint32_t>(st[312]);
  return SGDT_OK;
}

int sgdt_reset_pool(sgdt_session* s) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  TRY(settle_ahead(*s, true, "reset_pool"));
  s->pool_valid = false;
  return SGDT_OK;
}

int sgdt_set_pool(sgdt_session* s, const uint32_t* pool) {
  if (!s || !pool) return fail(SGDT_ERR_DOMAIN, "set_pool: null argument");
  SGDT_CUDA(cudaSetDevice(s->device));
  TRY(settle_ahead(*s, true, "set_pool"));
  SGDT_CUDA(cudaMemcpyAsync(s->pool, pool, s->nnz * sizeof(uint32_t), cudaMemcpyHostToDevice, s->stream));
  SGDT_CUDA(cudaStreamSynchronize(s->stream));
  s->pool_valid = true;
  return SGDT_OK;
}

int sgdt_get_pool(sgdt_session* s, uint32_t* pool) {
  if (!s || !pool) return fail(SGDT_ERR_DOMAIN, "get_pool: null argument");
  SGDT_CUDA(cudaSetDevice(s->device));
  SGDT_CUDA(cudaStreamSynchronize(s->side));
  if (!s->pool_valid) {
    for (uint64_t e = 0; e < s->nnz; ++e) pool[e] = static_cast<uint32_t>(e);
    return SGDT_OK;
  }
  SGDT_CUDA(cudaMemcpyAsync(pool, s->pool, s->nnz * sizeof(uint32_t), cudaMemcpyDeviceToHost, s->stream));
  SGDT_CUDA(cudaStreamSynchronize(s->stream));
  return SGDT_OK;
}

int sgdt_sample_batch(sgdt_session* s, uint64_t m, uint32_t* out) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  if (m < 1 || m > s->nnz) return fail(SGDT_ERR_DOMAIN, "sample_batch: batch size out of range");
  SGDT_CUDA(cudaSetDevice(s->device));
  TRY(settle_ahead(*s, false, "sample_batch"));
  s->delta_base = s->sampler_runs;
  TRY(ensure_batch_capacity(*s, m));
  TRY(launch_sampler(*s, m, s->batch, s->stream));
  if (out) SGDT_CUDA(cudaMemcpyAsync(out, s->batch, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, s->stream));
  SGDT_CUDA(cudaStreamSynchronize(s->stream));
  return SGDT_OK;
}

int sgdt_last_batch(sgdt_session* s, uint32_t* out, uint64_t* len) {
  if (!s || !len) return fail(SGDT_ERR_DOMAIN, "null argument");
  SGDT_CUDA(cudaStreamSynchronize(s->side));
  *len = s->last_batch_len;
  if (out && s->last_batch_len) {
    SGDT_CUDA(cudaMemcpyAsync(out, s->last_batch, s->last_batch_len * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                              s->stream));
    SGDT_CUDA(cudaStreamSynchronize(s->stream));
  }
  return SGDT_OK;
}

int sgdt_core_epoch(sgdt_session* s, const sgdt_core_hyper* h, sgdt_core_stats* st) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  uint64_t m = 0;
  TRY(check_core_hyper(*s, h, &m));
  SGDT_CUDA(cudaSetDevice(s->device));
  s->delta_base = s->sampler_runs;
  if (st) {
    st->batch_size = h->lr == 0.0 ? 0 : m;
    st->effective_workers = h->lr == 0.0 ? 0 : 1;
  }
  if (h->lr == 0.0) return SGDT_OK;
  TRY(settle_ahead(*s, false, "core_epoch"));
  TRY(enqueue_core(*s, *h, m));
  return sync_and_flag(*s);
}

// The reference's improved-strategy figure (factor_optimizer.cpp:209-218) with
// the ranks of a sharded session as its workers: the largest
// partition_even(nnz, world) slice over the ideal nnz / world, minus 1.  A
// single session is one worker, as the reference with threads = 1: 0.
static double rank_imbalance(const Session& s) {
  if (s.world <= 1 || s.nnz == 0) return 0.0;
  const uint64_t biggest = (s.nnz + s.world - 1) / s.world;
  return static_cast<double>(biggest) / (static_cast<double>(s.nnz) / s.world) - 1.0;
}

int sgdt_factor_epoch(sgdt_session* s, const sgdt_factor_hyper* h, sgdt_factor_stats* st) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  TRY(check_factor_hyper(h));
  SGDT_CUDA(cudaSetDevice(s->device));
  if (st) {
    *st = sgdt_factor_stats{0, 0, 0.0};
    if (h->lr > 0.0)
      for (int n = 0; n < s->order; ++n) {
        st->rows_updated += s->mode[n].rows_nonempty;
        st->rows_skipped += s->mode[n].rows_empty;
      }
    st->max_imbalance = h->lr > 0.0 ? rank_imbalance(*s) : 0.0;
  }
  if (h->lr == 0.0) return SGDT_OK;
  if (h->row_fraction < 1.0) TRY(settle_ahead(*s, false, "factor_epoch (row_fraction < 1)"));
  TRY(enqueue_factor(*s, *h, false));
  return sync_and_flag(*s);
}

__global__ void pool_delta_kernel(const uint32_t* __restrict__ draw_j, const uint32_t* __restrict__ pool, uint64_t m,
                                  uint32_t* pos, uint32_t* val) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t p = draw_j[i];
    pos[i] = p;
    val[i] = pool[p];
  }
}

int sgdt_pool_delta(sgdt_session* s, uint32_t* pos, uint32_t* val, uint64_t* n) {
  if (!s || !pos || !val || !n) return fail(SGDT_ERR_DOMAIN, "pool_delta: null argument");
  if (s->ahead_valid || s->sampler_runs != s->delta_base + 1)
    return fail(SGDT_ERR_CONFIG, "pool_delta: the last call did not make exactly one sampler run");
  SGDT_CUDA(cudaSetDevice(s->device));
  const uint64_t m = s->delta_m;
  uint32_t* d = nullptr;
  TRY(dalloc(&d, 2 * m));
  pool_delta_kernel<<<grid_for(m, s->num_sms), 256, 0, s->stream>>>(s->draw_j, s->pool, m, d, d + m);
  ++s->launches;
  int rc = SGDT_OK;
  if (cudaGetLastError() != cudaSuccess ||
      cudaMemcpyAsync(pos, d, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, s->stream) != cudaSuccess ||
      cudaMemcpyAsync(val, d + m, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, s->stream) != cudaSuccess ||
      cudaStreamSynchronize(s->stream) != cudaSuccess) {
    cudaGetLastError();
    rc = fail(SGDT_ERR_INTERNAL, "pool_delta: copy failed");
  }
  cudaFree(d);
  *n = rc == SGDT_OK ? m : 0;
  return rc;
}

int sgdt_set_pool_capture(sgdt_session* s, int on) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  s->capture_pre = on != 0;
  return SGDT_OK;
}

int sgdt_pool_delta_view(sgdt_session* s, const uint32_t** pos, const uint32_t** val, const uint32_t** pre_j,
                         const uint32_t** pre_lo, uint64_t* n) {
  if (!s || !pos || !val || !pre_j || !pre_lo || !n) return fail(SGDT_ERR_DOMAIN, "pool_delta_view: null argument");
  if (s->ahead_valid || s->sampler_runs != s->delta_base + 1)
    return fail(SGDT_ERR_CONFIG, "pool_delta: the last call did not make exactly one sampler run");
  if (!s->capture_pre || !s->pool_pre || s->delta_m > s->pool_pre_cap)
    return fail(SGDT_ERR_CONFIG, "pool_delta_view: capture is off (sgdt_set_pool_capture)");
  SGDT_CUDA(cudaSetDevice(s->device));
  const uint64_t m = s->delta_m;
  if (m > s->delta_cap) {
    if (s->d_delta) cudaFree(s->d_delta);
    if (s->h_delta) cudaFreeHost(s->h_delta);
    s->d_delta = nullptr;
    s->h_delta = nullptr;
    s->delta_cap = 0;
    TRY(dalloc(&s->d_delta, 2 * m));
    SGDT_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s->h_delta), 4 * m * sizeof(uint32_t), cudaHostAllocDefault));
    s->delta_cap = m;
  }
  pool_delta_kernel<<<grid_for(m, s->num_sms), 256, 0, s->stream>>>(s->draw_j, s->pool, m, s->d_delta,
                                                                   s->d_delta + m);
  ++s->launches;
  SGDT_CUDA(cudaGetLastError());
  SGDT_CUDA(cudaMemcpyAsync(s->h_delta, s->d_delta, 2 * m * sizeof(uint32_t), cudaMemcpyDeviceToHost, s->stream));
  SGDT_CUDA(cudaMemcpyAsync(s->h_delta + 2 * m, s->pool_pre, 2 * m * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                            s->stream));
  SGDT_CUDA(cudaStreamSynchronize(s->stream));
  *pos = s->h_delta;
  *val = s->h_delta + m;
  *pre_j = s->h_delta + 2 * m;
  *pre_lo = s->h_delta + 3 * m;
  *n = m;
  return SGDT_OK;
}

int sgdt_pool_delta_pre(sgdt_session* s, uint32_t* pos, uint32_t* val, uint32_t* pre_j, uint32_t* pre_lo,
                        uint64_t* n) {
  if (!pos || !val || !pre_j || !pre_lo || !n) return fail(SGDT_ERR_DOMAIN, "pool_delta_pre: null argument");
  const uint32_t *p, *v, *a, *b;
  TRY(sgdt_pool_delta_view(s, &p, &v, &a, &b, n));
  std::memcpy(pos, p, *n * sizeof(uint32_t));
  std::memcpy(val, v, *n * sizeof(uint32_t));
  std::memcpy(pre_j, a, *n * sizeof(uint32_t));
  std::memcpy(pre_lo, b, *n * sizeof(uint32_t));
  return SGDT_OK;
}

int sgdt_factor_epoch_host(sgdt_session* s, const sgdt_factor_hyper* h, double* const* A_out, sgdt_factor_stats* st) {
  if (!s || !A_out) return fail(SGDT_ERR_DOMAIN, "factor_epoch_host: null argument");
  TRY(check_factor_hyper(h));
  SGDT_CUDA(cudaSetDevice(s->device));
  if (st) {
    *st = sgdt_factor_stats{0, 0, 0.0};
    if (h->lr > 0.0)
      for (int n = 0; n < s->order; ++n) {
        st->rows_updated += s->mode[n].rows_nonempty;
        st->rows_skipped += s->mode[n].rows_empty;
      }
    st->max_imbalance = h->lr > 0.0 ? rank_imbalance(*s) : 0.0;
  }
  if (h->lr == 0.0) return SGDT_OK;  // A unchanged: nothing to copy
  if (h->row_fraction < 1.0) TRY(settle_ahead(*s, false, "factor_epoch_host (row_fraction < 1)"));
  uint64_t off[kMaxOrder + 1] = {0};
  for (int k = 0; k < s->order; ++k) off[k + 1] = off[k] + static_cast<uint64_t>(s->dims[k]) * s->J[k];
  if (off[s->order] > s->xfer_cap) {
    if (s->xfer) cudaFree(s->xfer);
    s->xfer = nullptr;
    s->xfer_cap = 0;
    TRY(dalloc(&s->xfer, off[s->order]));
    s->xfer_cap = off[s->order];
  }
  if (off[s->order] > s->hx_cap) {
    if (s->hx) cudaFreeHost(s->hx);
    s->hx = nullptr;
    s->hx_cap = 0;
    SGDT_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s->hx), off[s->order] * sizeof(double), cudaHostAllocDefault));
    s->hx_cap = off[s->order];
  }
  for (int n = 0; n < s->order; ++n)
    if (!s->ev_copy[n]) SGDT_CUDA(cudaEventCreateWithFlags(&s->ev_copy[n], cudaEventDisableTiming));
  // the factor passes; ev[4 + n] marks the start of mode n, ev[2] the end
  TRY(enqueue_factor(*s, *h, true));
  SGDT_CUDA(cudaEventRecord(s->ev[2], s->stream));
  // A^(n) is final once mode n's pass is done: cast + D2H on the side stream
  // while the later modes run, then the host copies it out of the pinned
  // staging while the GPU is still busy
  for (int n = 0; n < s->order; ++n) {
    SGDT_CUDA(cudaStreamWaitEvent(s->side, n + 1 < s->order ? s->ev[4 + n + 1] : s->ev[2], 0));
    const uint64_t na = off[n + 1] - off[n];
    cast_f2d_kernel<<<grid_for(na, s->num_sms), 256, 0, s->side>>>(s->P.A[n], s->xfer + off[n], na);
    SGDT_CUDA(cudaMemcpyAsync(s->hx + off[n], s->xfer + off[n], na * sizeof(double), cudaMemcpyDeviceToHost,
                              s->side));
    SGDT_CUDA(cudaEventRecord(s->ev_copy[n], s->side));
    ++s->launches;
  }
  SGDT_CUDA(cudaGetLastError());
  for (int n = 0; n < s->order; ++n) {
    SGDT_CUDA(cudaEventSynchronize(s->ev_copy[n]));
    parallel_copy(A_out[n], s->hx + off[n], (off[n + 1] - off[n]) * sizeof(double));
  }
  return sync_and_flag(*s);
}

}  // extern "C"

namespace sgdt {
namespace {
// Host destinations of the final model (sgdt_run_epochs_host); offsets into
// Session::xfer per matrix.
struct CopyOut {
  double* const* A;
  double* const* B;
  uint64_t offA[kMaxOrder], offB[kMaxOrder];
};

int run_epochs_impl(sgdt_session* s, const sgdt_core_hyper* ch, const sgdt_factor_hyper* fh, uint64_t epochs,
                    const CopyOut* out, bool first_sampled = false);
bool sample_runs_ahead(const sgdt_core_hyper* ch, const sgdt_factor_hyper* fh);
}  // namespace
}  // namespace sgdt

extern "C" {

int sgdt_run_epochs(sgdt_session* s, const sgdt_core_hyper* ch, const sgdt_factor_hyper* fh, uint64_t epochs) {
  return run_epochs_impl(s, ch, fh, epochs, nullptr);
}

int sgdt_run_epochs_host(sgdt_session* s, const sgdt_core_hyper* ch, const sgdt_factor_hyper* fh, uint64_t epochs,
                         const double* const* A_in, const double* const* B_in, double* const* A_out,
                         double* const* B_out) {
  if (!s || !A_in || !B_in || !A_out || !B_out) return fail(SGDT_ERR_DOMAIN, "run_epochs_host: null argument");
  uint64_t m = 0;
  TRY(check_core_hyper(*s, ch, &m));
  TRY(check_factor_hyper(fh));
  SGDT_CUDA(cudaSetDevice(s->device));
  CopyOut co{A_out, B_out, {}, {}};
  uint64_t total = 0;
  for (int k = 0; k < s->order; ++k) {
    co.offA[k] = total;
    total += static_cast<uint64_t>(s->dims[k]) * s->J[k];
    co.offB[k] = total;
    total += static_cast<uint64_t>(s->J[k]) * s->R;
  }
  if (total > s->xfer_cap) {
    if (s->xfer) cudaFree(s->xfer);
    s->xfer = nullptr;
    s->xfer_cap = 0;
    TRY(dalloc(&s->xfer, total));
    s->xfer_cap = total;
  }
  // Psi of the first epoch depends only on the RNG: draw it on the side
  // stream while the model is copied in
  TRY(settle_ahead(*s, false, "run_epochs_host"));
  const bool early = epochs > 0 && sample_runs_ahead(ch, fh);
  if (early) {
    TRY(ensure_batch_capacity(*s, m));
    TRY(ensure_core_capacity(*s, m));
    SGDT_CUDA(cudaEventRecord(s->ev_start, s->stream));
    SGDT_CUDA(cudaStreamWaitEvent(s->side, s->ev_start, 0));
    TRY(enqueue_sample(*s, *ch, m, s->batch, s->side));
    SGDT_CUDA(cudaEventRecord(s->ev_samp, s->side));
  }
  // load: the copies back to back, then the casts
  for (int k = 0; k < s->order; ++k) {
    const uint64_t na = static_cast<uint64_t>(s->dims[k]) * s->J[k], nb = static_cast<uint64_t>(s->J[k]) * s->R;
    SGDT_CUDA(cudaMemcpyAsync(s->xfer + co.offA[k], A_in[k], na * sizeof(double), cudaMemcpyHostToDevice,
                              s->stream));
    SGDT_CUDA(cudaMemcpyAsync(s->xfer + co.offB[k], B_in[k], nb * sizeof(double), cudaMemcpyHostToDevice,
                              s->stream));
  }
  for (int k = 0; k < s->order; ++k) {
    const uint64_t na = static_cast<uint64_t>(s->dims[k]) * s->J[k], nb = static_cast<uint64_t>(s->J[k]) * s->R;
    cast_d2f_kernel<<<grid_for(na, s->num_sms), 256, 0, s->stream>>>(s->xfer + co.offA[k], s->P.A[k], na);
    cast_d2f_kernel<<<grid_for(nb, s->num_sms), 256, 0, s->stream>>>(s->xfer + co.offB[k], s->P.B[k], nb);
    SGDT_CUDA(cudaGetLastError());
    s->launches += 2;
  }
  // Q^(k) = A^(k) B^(k) for the model just copied in: the factor phase gathers Q rows,
  // and so does the core phase's sample setup (sgdt_core.cu)
  for (int k = 0; k < s->order; ++k) TRY(launch_q_refresh(*s, k));
  if (epochs == 0) {
    SGDT_CUDA(cudaStreamSynchronize(s->stream));
    return sgdt_get_model(s, A_out, B_out);
  }
  return run_epochs_impl(s, ch, fh, epochs, &co, early);
}

}  // extern "C"

namespace sgdt {
namespace {
// Psi does not depend on the model, so epoch e+1's sampler can run on the
// side stream during epoch e (with row_fraction < 1 the factor phase also
// draws, so no run-ahead).
bool sample_runs_ahead(const sgdt_core_hyper* ch, const sgdt_factor_hyper* fh) {
  return ch->lr > 0.0 && ch->batch_m != 0 && !(fh->lr > 0.0 && fh->row_fraction < 1.0);
}

int run_epochs_impl(sgdt_session* s, const sgdt_core_hyper* ch, const sgdt_factor_hyper* fh, uint64_t epochs,
                    const CopyOut* out, bool first_sampled) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  uint64_t m = 0;
  TRY(check_core_hyper(*s, ch, &m));
  TRY(check_factor_hyper(fh));
  SGDT_CUDA(cudaSetDevice(s->device));
  TRY(settle_ahead(*s, false, "run_epochs"));
  if (epochs == 0) return SGDT_OK;
  // Psi does not depend on the model, so epoch e+1's sampler runs on the side
  // stream during epoch e's factor phase (double-buffered Psi).  The RNG
  // stream is consumed in exactly the reference order: the factor phase draws
  // nothing (row_fraction == 1).
  // (with row_fraction < 1 the factor phase also draws, so no run-ahead)
  const bool ahead = sample_runs_ahead(ch, fh);
  uint32_t* buf[2] = {nullptr, nullptr};
  if (ahead) {
    TRY(ensure_batch_capacity(*s, m));
    TRY(ensure_core_capacity(*s, m));
    buf[0] = s->batch;
    buf[1] = s->batch + static_cast<uint64_t>(s->order) * m;
    if (!first_sampled) {  // (run_epochs_host drew it before its copies)
      SGDT_CUDA(cudaEventRecord(s->ev_start, s->stream));
      SGDT_CUDA(cudaStreamWaitEvent(s->side, s->ev_start, 0));
      TRY(enqueue_sample(*s, *ch, m, buf[0], s->side));
      SGDT_CUDA(cudaEventRecord(s->ev_samp, s->side));
    }
  }
  // per-epoch phase events (the last kTimedEpochs epochs): {core start, core
  // end, mode starts[N], factor end}; sgdt_last_timing reports their means
  const int stride = s->order + 3;
  const uint64_t timed = std::min<uint64_t>(epochs, kTimedEpochs);
  TRY(ensure_timing_events(*s, timed * stride));
  for (uint64_t e = 0; e < epochs; ++e) {
    const bool last = e + 1 == epochs;
    cudaEvent_t* E = e + timed >= epochs ? &s->tev[(e + timed - epochs) * stride] : nullptr;
    if (ahead) SGDT_CUDA(cudaStreamWaitEvent(s->stream, s->ev_samp, 0));
    if (last) SGDT_CUDA(cudaEventRecord(s->ev[0], s->stream));
    if (E) SGDT_CUDA(cudaEventRecord(E[0], s->stream));
    TRY(enqueue_core(*s, *ch, m, ahead ? buf[e & 1] : nullptr));
    if (ahead && !last) {
      SGDT_CUDA(cudaEventRecord(s->ev_core, s->stream));
      SGDT_CUDA(cudaStreamWaitEvent(s->side, s->ev_core, 0));
      TRY(enqueue_sample(*s, *ch, m, buf[(e + 1) & 1], s->side));
      SGDT_CUDA(cudaEventRecord(s->ev_samp, s->side));
    }
    if (last) SGDT_CUDA(cudaEventRecord(s->ev[1], s->stream));
    if (E) SGDT_CUDA(cudaEventRecord(E[1], s->stream));
    TRY(enqueue_factor(*s, *fh, last, E ? E + 2 : nullptr));
    if (last) SGDT_CUDA(cudaEventRecord(s->ev[2], s->stream));
    if (E) SGDT_CUDA(cudaEventRecord(E[2 + s->order], s->stream));
  }
  if (out) {
    // copy-out on the side stream: B^(k) is final after the last core phase,
    // A^(n) after the last factor pass of mode n
    const bool modes = fh->lr > 0.0;
    SGDT_CUDA(cudaStreamWaitEvent(s->side, s->ev[1], 0));
    for (int k = 0; k < s->order; ++k) {
      const uint64_t nb = static_cast<uint64_t>(s->J[k]) * s->R;
      cast_f2d_kernel<<<grid_for(nb, s->num_sms), 256, 0, s->side>>>(s->P.B[k], s->xfer + out->offB[k], nb);
      SGDT_CUDA(cudaMemcpyAsync(out->B[k], s->xfer + out->offB[k], nb * sizeof(double), cudaMemcpyDeviceToHost,
                                s->side));
    }
    for (int n = 0; n < s->order; ++n) {
      const uint64_t na = static_cast<uint64_t>(s->dims[n]) * s->J[n];
      SGDT_CUDA(cudaStreamWaitEvent(s->side, modes && n + 1 < s->order ? s->ev[4 + n + 1] : s->ev[2], 0));
      cast_f2d_kernel<<<grid_for(na, s->num_sms), 256, 0, s->side>>>(s->P.A[n], s->xfer + out->offA[n], na);
      SGDT_CUDA(cudaMemcpyAsync(out->A[n], s->xfer + out->offA[n], na * sizeof(double), cudaMemcpyDeviceToHost,
                                s->side));
    }
    SGDT_CUDA(cudaGetLastError());
    s->launches += 2 * s->order;
  }
  {
    const int rc = sync_and_flag(*s);
    if (out) SGDT_CUDA(cudaStreamSynchronize(s->side));
    if (rc != SGDT_OK) return rc;
  }
  sgdt_timing t{};
  for (uint64_t e = 0; e < timed; ++e) {
    cudaEvent_t* E = &s->tev[e * stride];
    float core = 0.f, fac = 0.f;
    SGDT_CUDA(cudaEventElapsedTime(&core, E[0], E[1]));
    SGDT_CUDA(cudaEventElapsedTime(&fac, E[1], E[2 + s->order]));
    t.core_ms += core / timed;
    t.factor_ms += fac / timed;
    if (fh->lr > 0.0)
      for (int n = 0; n < s->order; ++n) {
        float x = 0.f;
        SGDT_CUDA(cudaEventElapsedTime(&x, E[2 + n], E[3 + n]));
        t.factor_mode_ms[n] += x / timed;
      }
  }
  t.epochs = static_cast<uint32_t>(timed);
  s->timing = t;
  s->timing_valid = true;
  return SGDT_OK;
}

}  // namespace
}  // namespace sgdt

extern "C" {

int sgdt_eval(sgdt_session* s, int which, double* rmse, double* mae) {
  if (!s || !rmse || !mae) return fail(SGDT_ERR_DOMAIN, "null argument");
  if (which != 0 && which != 1) return fail(SGDT_ERR_DOMAIN, "eval: which must be 0 (train) or 1 (test)");
  SGDT_CUDA(cudaSetDevice(s->device));
  return launch_eval(*s, which, rmse, mae);
}

int sgdt_train(sgdt_session* s, const sgdt_core_hyper* ch, const sgdt_factor_hyper* fh, uint64_t epochs,
               double* metrics) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  for (uint64_t e = 0; e < epochs; ++e) {
    TRY(sgdt_run_epochs(s, ch, fh, 1));
    double* row = metrics ? metrics + e * 6 : nullptr;
    if (row) {
      row[0] = s->timing.core_ms * 1e-3;
      row[1] = s->timing.factor_ms * 1e-3;
      TRY(sgdt_eval(s, 0, &row[2], &row[3]));
      if (s->nnz_test) {
        TRY(sgdt_eval(s, 1, &row[4], &row[5]));
      } else {
        row[4] = row[5] = std::nan("");
      }
    }
  }
  return SGDT_OK;
}

uint64_t sgdt_launch_count(sgdt_session* s) { return s ? s->launches : 0; }

int sgdt_get_shard_info(sgdt_session* s, int mode, sgdt_shard_info* out) {
  if (!s || !out) return fail(SGDT_ERR_DOMAIN, "null argument");
  if (mode < 0 || mode >= s->order) return fail(SGDT_ERR_DOMAIN, "shard_info: mode out of range");
  const ShardPlan& sp = s->mode[mode].shard;
  out->rank = s->rank;
  out->world = s->world;
  out->entry_begin = sp.qb;
  out->entry_end = sp.qe;
  out->row_lo = sp.row_lo;
  out->row_hi = sp.row_hi;
  out->n_export = sp.n_export;
  out->export_rows[0] = sp.export_rows[0];
  out->export_rows[1] = sp.export_rows[1];
  return SGDT_OK;
}

int sgdt_factor_mode_local(sgdt_session* s, int mode, const sgdt_factor_hyper* h, double* export_g) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  if (mode < 0 || mode >= s->order) return fail(SGDT_ERR_DOMAIN, "factor_mode_local: mode out of range");
  TRY(check_factor_hyper(h));
  if (h->lr > 0.0 && h->row_fraction < 1.0)
    return fail(SGDT_ERR_CONFIG, "row_fraction < 1 is not supported by the sharded (multi-GPU) factor phase");
  SGDT_CUDA(cudaSetDevice(s->device));
  if (h->lr == 0.0) return SGDT_OK;
  TRY(launch_factor_mode(*s, mode, *h));
  const ShardPlan& sp = s->mode[mode].shard;
  std::vector<double> buf(2ull * s->RP);
  if (sp.n_export)
    SGDT_CUDA(cudaMemcpyAsync(buf.data(), s->export_buf, sp.n_export * s->RP * sizeof(double),
                              cudaMemcpyDeviceToHost, s->stream));
  TRY(sync_and_flag(*s));
  if (export_g)
    for (uint32_t k = 0; k < sp.n_export; ++k)
      for (uint32_t r = 0; r < s->R; ++r) export_g[k * s->R + r] = buf[k * s->RP + r];
  return SGDT_OK;
}

int sgdt_factor_mode_finish(sgdt_session* s, int mode, const sgdt_factor_hyper* h, uint32_t k, const uint32_t* rows,
                            const double* g) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  if (mode < 0 || mode >= s->order) return fail(SGDT_ERR_DOMAIN, "factor_mode_finish: mode out of range");
  TRY(check_factor_hyper(h));
  SGDT_CUDA(cudaSetDevice(s->device));
  if (h->lr == 0.0 || k == 0) return SGDT_OK;
  for (uint32_t i = 0; i < k; ++i)
    if (rows[i] >= s->dims[mode]) return fail(SGDT_ERR_DOMAIN, "factor_mode_finish: row out of range");
  std::vector<double> gp(static_cast<uint64_t>(k) * s->RP, 0.0);
  for (uint32_t i = 0; i < k; ++i)
    for (uint32_t r = 0; r < s->R; ++r) gp[i * s->RP + r] = g[i * s->R + r];
  uint32_t* d_rows = nullptr;
  double* d_g = nullptr;
  TRY(dalloc(&d_rows, k));
  TRY(dalloc(&d_g, gp.size()));
  SGDT_CUDA(cudaMemcpyAsync(d_rows, rows, k * sizeof(uint32_t), cudaMemcpyHostToDevice, s->stream));
  SGDT_CUDA(cudaMemcpyAsync(d_g, gp.data(), gp.size() * sizeof(double), cudaMemcpyHostToDevice, s->stream));
  const int rc = launch_factor_finish(*s, mode, *h, k, d_rows, d_g);
  const int rc2 = sync_and_flag(*s);
  cudaFree(d_rows);
  cudaFree(d_g);
  return rc ? rc : rc2;
}

int sgdt_factor_rows(sgdt_session* s, int mode, uint32_t row_lo, uint32_t row_hi, float* buf, int to_device,
                     int buf_on_device) {
  if (!s || (!buf && row_hi > row_lo)) return fail(SGDT_ERR_DOMAIN, "null argument");
  if (mode < 0 || mode >= s->order || row_lo > row_hi || row_hi > s->dims[mode])
    return fail(SGDT_ERR_DOMAIN, "factor_rows: range out of bounds");
  SGDT_CUDA(cudaSetDevice(s->device));
  if (row_hi == row_lo) return SGDT_OK;
  float* dev = s->P.A[mode] + static_cast<uint64_t>(row_lo) * s->J[mode];
  const size_t bytes = static_cast<size_t>(row_hi - row_lo) * s->J[mode] * sizeof(float);
  const cudaMemcpyKind kind = buf_on_device ? cudaMemcpyDeviceToDevice
                                            : (to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost);
  if (to_device)
    SGDT_CUDA(cudaMemcpyAsync(dev, buf, bytes, kind, s->stream));
  else
    SGDT_CUDA(cudaMemcpyAsync(buf, dev, bytes, kind, s->stream));
  SGDT_CUDA(cudaStreamSynchronize(s->stream));
  return SGDT_OK;
}

int sgdt_factor_device_ptr(sgdt_session* s, int mode, void** ptr) {
  if (!s || !ptr) return fail(SGDT_ERR_DOMAIN, "null argument");
  if (mode < 0 || mode >= s->order) return fail(SGDT_ERR_DOMAIN, "factor_device_ptr: mode out of range");
  *ptr = s->P.A[mode];
  return SGDT_OK;
}

int sgdt_refresh_q(sgdt_session* s, int mode) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  if (mode < 0 || mode >= s->order) return fail(SGDT_ERR_DOMAIN, "refresh_q: mode out of range");
  SGDT_CUDA(cudaSetDevice(s->device));
  TRY(launch_q_refresh(*s, mode));
  SGDT_CUDA(cudaStreamSynchronize(s->stream));
  return SGDT_OK;
}

int sgdt_peer_buffers(sgdt_session* s, void** ptrs) {
  if (!s || !ptrs) return fail(SGDT_ERR_DOMAIN, "null argument");
  for (int k = 0; k < s->order; ++k) {
    ptrs[k] = s->P.A[k];
    ptrs[s->order + k] = s->P.Q[k];
  }
  ptrs[2 * s->order] = s->xrec;
  ptrs[2 * s->order + 1] = s->core_x;
  return SGDT_OK;
}

int sgdt_peer_ipc_handles(sgdt_session* s, void* handles) {
  if (!s || !handles) return fail(SGDT_ERR_DOMAIN, "null argument");
  SGDT_CUDA(cudaSetDevice(s->device));
  void* ptrs[2 * kMaxOrder + 2];
  TRY(sgdt_peer_buffers(s, ptrs));
  auto* out = static_cast<cudaIpcMemHandle_t*>(handles);
  for (int i = 0; i < 2 * s->order + 2; ++i) SGDT_CUDA(cudaIpcGetMemHandle(&out[i], ptrs[i]));
  return SGDT_OK;
}

int sgdt_ipc_open(const void* handle, int device, void** ptr) {
  if (!handle || !ptr) return fail(SGDT_ERR_DOMAIN, "null argument");
  if (device >= 0) SGDT_CUDA(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  SGDT_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return SGDT_OK;
}

int sgdt_set_peers(sgdt_session* s, const void* const* ptrs) {
  if (!s || !ptrs) return fail(SGDT_ERR_DOMAIN, "null argument");
  if (s->world - 1 > kMaxPeers) return fail(SGDT_ERR_CONFIG, "set_peers: at most 8 ranks");
  SGDT_CUDA(cudaSetDevice(s->device));
  const int per = 2 * s->order + 2;
  PeerTable tab[kMaxOrder] = {};
  int np = 0;
  for (int r = 0; r < s->world; ++r) {
    const void* const* row = ptrs + static_cast<size_t>(r) * per;
    s->core_peer_x[r] = r == s->rank ? s->core_x : static_cast<double*>(const_cast<void*>(row[2 * s->order + 1]));
    if (r == s->rank) continue;
    for (int k = 0; k < s->order; ++k) {
      tab[k].A[np] = static_cast<float*>(const_cast<void*>(row[k]));
      tab[k].Q[np] = static_cast<float*>(const_cast<void*>(row[s->order + k]));
    }
    s->peer_rec[np] = static_cast<double*>(const_cast<void*>(row[2 * s->order]));
    ++np;
  }
  for (int k = 0; k < s->order; ++k) tab[k].n = np;
  SGDT_CUDA(cudaMemcpyAsync(s->d_peers, tab, sizeof tab, cudaMemcpyHostToDevice, s->stream));
  SGDT_CUDA(cudaStreamSynchronize(s->stream));
  s->npeers = np;
  return SGDT_OK;
}

int sgdt_core_epoch_async(sgdt_session* s, const sgdt_core_hyper* h) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  uint64_t m = 0;
  TRY(check_core_hyper(*s, h, &m));
  SGDT_CUDA(cudaSetDevice(s->device));
  const int per_mode = h->resample_per_mode && h->batch_m != 0 ? 1 : 0;
  if (s->ahead_valid) {
    if (h->lr == 0.0 || s->ahead_m != m || s->ahead_per_mode != per_mode)
      return fail(SGDT_ERR_CONFIG, "core_epoch_async: hyper-parameters differ from the pending sgdt_sample_ahead");
    s->ahead_valid = false;
    SGDT_CUDA(cudaStreamWaitEvent(s->stream, s->ev_samp, 0));
    return enqueue_core(*s, *h, m, s->batch + static_cast<uint64_t>(s->ahead_slot) * s->order * m);
  }
  if (h->lr == 0.0) return SGDT_OK;
  return enqueue_core(*s, *h, m);
}

int sgdt_core_plan(sgdt_session* s, const sgdt_core_hyper* h, uint32_t block, uint32_t* steps, uint32_t* T_out) {
  if (!s || !steps) return fail(SGDT_ERR_DOMAIN, "null argument");
  uint64_t m = 0;
  TRY(check_core_hyper(*s, h, &m));
  SGDT_CUDA(cudaSetDevice(s->device));
  *steps = 0;
  if (T_out) *T_out = 0;
  const int per_mode = h->resample_per_mode && h->batch_m != 0 ? 1 : 0;
  const uint32_t* batch = nullptr;
  if (s->ahead_valid) {
    if (h->lr == 0.0 || s->ahead_m != m || s->ahead_per_mode != per_mode)
      return fail(SGDT_ERR_CONFIG, "core_plan: hyper-parameters differ from the pending sgdt_sample_ahead");
    s->ahead_valid = false;
    SGDT_CUDA(cudaStreamWaitEvent(s->stream, s->ev_samp, 0));
    batch = s->batch + static_cast<uint64_t>(s->ahead_slot) * s->order * m;
  }
  if (h->lr == 0.0) return SGDT_OK;  // frozen: no steps, no RNG
  TRY(ensure_batch_capacity(*s, m));
  s->core_slot = batch && batch != s->batch ? 1 : 0;
  if (!batch) {
    if (h->batch_m == 0) {
      iota32_kernel<<<grid_for(m, s->num_sms), 256, 0, s->stream>>>(s->batch, m);
      SGDT_CUDA(cudaGetLastError());
      ++s->launches;
      s->last_batch = s->batch;
      s->last_batch_len = m;
    } else {
      TRY(enqueue_sample(*s, *h, m, s->batch, s->stream));
    }
    batch = s->batch;
  }
  TRY(begin_core_plan(*s, *h, m, batch, per_mode, true, block));
  *steps = s->cplan.steps;
  if (T_out) *T_out = s->cplan.T;
  return SGDT_OK;
}

int sgdt_core_step(sgdt_session* s, uint32_t k) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  CorePlan& pl = s->cplan;
  if (!pl.valid) return fail(SGDT_ERR_CONFIG, "core_step: no core plan (sgdt_core_plan)");
  if (k != pl.next) return fail(SGDT_ERR_CONFIG, "core_step: steps must be launched in order");
  SGDT_CUDA(cudaSetDevice(s->device));
  {
    NvtxRange range("sgdt:core step");
    TRY(launch_core_block_step(*s, k));
  }
  if (++pl.next == pl.steps) pl.valid = false;
  return SGDT_OK;
}

int sgdt_sample_ahead(sgdt_session* s, const sgdt_core_hyper* h) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  uint64_t m = 0;
  TRY(check_core_hyper(*s, h, &m));
  SGDT_CUDA(cudaSetDevice(s->device));
  if (s->ahead_valid) return fail(SGDT_ERR_CONFIG, "sample_ahead: a draw is already pending");
  if (h->lr == 0.0 || h->batch_m == 0) return SGDT_OK;  // that core phase draws nothing
  TRY(ensure_batch_capacity(*s, m));
  TRY(ensure_core_capacity(*s, m));
  s->ahead_slot = 1 - s->core_slot;  // the slot the enqueued core phase is not reading
  SGDT_CUDA(cudaEventRecord(s->ev_core, s->stream));
  SGDT_CUDA(cudaStreamWaitEvent(s->side, s->ev_core, 0));
  TRY(enqueue_sample(*s, *h, m, s->batch + static_cast<uint64_t>(s->ahead_slot) * s->order * m, s->side));
  SGDT_CUDA(cudaEventRecord(s->ev_samp, s->side));
  s->ahead_valid = true;
  s->ahead_m = m;
  s->ahead_per_mode = h->resample_per_mode ? 1 : 0;
  return SGDT_OK;
}

int sgdt_factor_mode_p2p(sgdt_session* s, int mode, const sgdt_factor_hyper* h) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  if (mode < 0 || mode >= s->order) return fail(SGDT_ERR_DOMAIN, "factor_mode_p2p: mode out of range");
  TRY(check_factor_hyper(h));
  if (h->lr > 0.0 && h->row_fraction < 1.0)
    return fail(SGDT_ERR_CONFIG, "row_fraction < 1 is not supported by the sharded (multi-GPU) factor phase");
  if (s->world > 1 && s->npeers != s->world - 1) return fail(SGDT_ERR_CONFIG, "factor_mode_p2p: peers not set");
  SGDT_CUDA(cudaSetDevice(s->device));
  if (h->lr == 0.0) return SGDT_OK;
  TRY(launch_factor_mode(*s, mode, *h));
  const ShardPlan& sp = s->mode[mode].shard;
  RecordDst dst{};
  dst.p[0] = s->xrec;
  for (int p = 0; p < s->npeers; ++p) dst.p[1 + p] = s->peer_rec[p];
  dst.n = 1 + s->npeers;
  publish_record_kernel<<<1, 128, 0, s->stream>>>(s->export_buf, sp.n_export, sp.export_rows[0],
                                                  sp.export_rows[1], s->rec_stride, s->rank, dst);
  SGDT_CUDA(cudaGetLastError());
  ++s->launches;
  return SGDT_OK;
}

int sgdt_factor_merge_p2p(sgdt_session* s, int mode, const sgdt_factor_hyper* h) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  if (mode < 0 || mode >= s->order) return fail(SGDT_ERR_DOMAIN, "factor_merge_p2p: mode out of range");
  TRY(check_factor_hyper(h));
  SGDT_CUDA(cudaSetDevice(s->device));
  if (h->lr == 0.0) return SGDT_OK;
  // the cut row this rank publishes: an exported row inside [row_lo, row_hi)
  // (the row cut by the slice end; a row cut at the start belongs to the
  // rank where it starts, one cut at both ends likewise)
  const ShardPlan& sp = s->mode[mode].shard;
  uint32_t own[2], k = 0;
  for (uint32_t i = 0; i < sp.n_export; ++i)
    if (sp.export_rows[i] >= sp.row_lo && sp.export_rows[i] < sp.row_hi) own[k++] = sp.export_rows[i];
  if (k == 0) return SGDT_OK;
  merge_records_kernel<<<1, 128, 0, s->stream>>>(s->xrec, s->world, s->rec_stride, s->RP, k, own[0],
                                                 k > 1 ? own[1] : 0, s->merge_rows, s->merge_g);
  SGDT_CUDA(cudaGetLastError());
  ++s->launches;
  return launch_factor_finish(*s, mode, *h, k, s->merge_rows, s->merge_g);
}

int sgdt_enable_peer_access(const int* devices, int n) {
  if (!devices || n < 1) return fail(SGDT_ERR_DOMAIN, "enable_peer_access: no devices");
  int cur = 0;
  SGDT_CUDA(cudaGetDevice(&cur));
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      if (devices[i] == devices[j]) continue;
      int ok = 0;
      SGDT_CUDA(cudaDeviceCanAccessPeer(&ok, devices[i], devices[j]));
      if (!ok)
        return fail(SGDT_ERR_CONFIG, "device " + std::to_string(devices[i]) + " cannot access device " +
                                         std::to_string(devices[j]) + " (no P2P)");
      SGDT_CUDA(cudaSetDevice(devices[i]));
      const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        (void)cudaGetLastError();
      } else if (e != cudaSuccess) {
        (void)cudaGetLastError();
        cudaSetDevice(cur);
        return fail(SGDT_ERR_INTERNAL, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
      }
    }
  SGDT_CUDA(cudaSetDevice(cur));
  return SGDT_OK;
}

int sgdt_stream_barrier(sgdt_session* const* sessions, int n) {
  if (!sessions || n < 1) return fail(SGDT_ERR_DOMAIN, "stream_barrier: no sessions");
  for (int i = 0; i < n; ++i) {
    if (!sessions[i]) return fail(SGDT_ERR_DOMAIN, "stream_barrier: null session");
    SGDT_CUDA(cudaSetDevice(sessions[i]->device));
    SGDT_CUDA(cudaEventRecord(sessions[i]->ev_bar, sessions[i]->stream));
  }
  for (int i = 0; i < n; ++i) {
    SGDT_CUDA(cudaSetDevice(sessions[i]->device));
    for (int j = 0; j < n; ++j)
      if (j != i) SGDT_CUDA(cudaStreamWaitEvent(sessions[i]->stream, sessions[j]->ev_bar, 0));
  }
  return SGDT_OK;
}

int sgdt_check(sgdt_session* s) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  SGDT_CUDA(cudaSetDevice(s->device));
  SGDT_CUDA(cudaStreamSynchronize(s->side));
  return sync_and_flag(*s);
}

int sgdt_split_ids(uint64_t nnz, double test_fraction, uint64_t seed, int device, uint32_t* test_ids,
                   uint32_t* train_ids) {
  if (!(test_fraction > 0.0 && test_fraction < 1.0))
    return fail(SGDT_ERR_DOMAIN, "train_test_split: fraction must lie in (0,1)");
  const uint64_t ntest = static_cast<uint64_t>(std::llround(test_fraction * static_cast<double>(nnz)));
  if (ntest == 0 || ntest == nnz)
    return fail(SGDT_ERR_DOMAIN, "train_test_split: degenerate split (|test|=" + std::to_string(ntest) + " of " +
                                     std::to_string(nnz) + ")");
  if (nnz > 0xFFFFFFFFull || nnz > static_cast<uint64_t>(INT_MAX))
    return fail(SGDT_ERR_CONFIG, "split_ids: more entries than the device split supports");
  if ((ntest && !test_ids) || !train_ids) return fail(SGDT_ERR_DOMAIN, "split_ids: null output");
  if (device >= 0) SGDT_CUDA(cudaSetDevice(device));
  // a sampler-only session: pool = iota, Rng(seed), nnz-1 draws
  Session t;
  SGDT_CUDA(cudaGetDevice(&t.device));
  cudaDeviceProp prop{};
  SGDT_CUDA(cudaGetDeviceProperties(&prop, t.device));
  t.num_sms = prop.multiProcessorCount;
  t.nnz = nnz;
  const uint64_t m = nnz - 1;
  uint32_t *keys_out = nullptr, *batch = nullptr;
  void* tmp = nullptr;
  int rc = [&]() -> int {
    SGDT_CUDA(cudaStreamCreateWithFlags(&t.stream, cudaStreamNonBlocking));
    TRY(dalloc(&t.mt, 313));
    uint64_t mt[313];
    mt_seed(mt, seed);
    mt[312] = 312;
    SGDT_CUDA(cudaMemcpyAsync(t.mt, mt, sizeof mt, cudaMemcpyHostToDevice, t.stream));
    TRY(dalloc(&t.pool, nnz));
    TRY(dalloc(&t.head, nnz));
    SGDT_CUDA(cudaMemsetAsync(t.head, 0, nnz * sizeof(unsigned long long), t.stream));
    for (uint32_t** p : {&t.draw_j, &t.link, &t.kprev, &t.lprev, &t.dval}) TRY(dalloc(p, m));
    TRY(dalloc(&batch, m));
    TRY(launch_sampler(t, m, batch, t.stream));  // the pool is now the shuffled id array
    TRY(dalloc(&keys_out, nnz));
    size_t b1 = 0, b2 = 0;
    SGDT_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b1, t.pool, keys_out, static_cast<int>(ntest), 0, 32,
                                             t.stream));
    SGDT_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b2, t.pool + ntest, keys_out + ntest,
                                             static_cast<int>(nnz - ntest), 0, 32, t.stream));
    SGDT_CUDA(cudaMalloc(&tmp, std::max(b1, b2)));
    SGDT_CUDA(cub::DeviceRadixSort::SortKeys(tmp, b1, t.pool, keys_out, static_cast<int>(ntest), 0, 32, t.stream));
    SGDT_CUDA(cub::DeviceRadixSort::SortKeys(tmp, b2, t.pool + ntest, keys_out + ntest,
                                             static_cast<int>(nnz - ntest), 0, 32, t.stream));
    SGDT_CUDA(cudaMemcpyAsync(test_ids, keys_out, ntest * sizeof(uint32_t), cudaMemcpyDeviceToHost, t.stream));
    SGDT_CUDA(cudaMemcpyAsync(train_ids, keys_out + ntest, (nnz - ntest) * sizeof(uint32_t),
                              cudaMemcpyDeviceToHost, t.stream));
    SGDT_CUDA(cudaStreamSynchronize(t.stream));
    return SGDT_OK;
  }();
  for (void* p : {(void*)t.mt, (void*)t.pool, (void*)t.head, (void*)t.draw_j, (void*)t.link, (void*)t.kprev,
                  (void*)t.lprev, (void*)t.dval, (void*)batch, (void*)keys_out, tmp, (void*)t.mt_out,
                  (void*)t.mt_tent, (void*)t.mt_flag, (void*)t.jump.J, (void*)t.jump.st, (void*)t.jump.part})
    if (p) cudaFree(p);
  t.mt = t.mt_out = t.mt_tent = nullptr;
  t.mt_flag = nullptr;
  t.pool = t.draw_j = t.link = t.kprev = t.lprev = t.dval = nullptr;
  t.head = nullptr;
  if (t.stream) cudaStreamDestroy(t.stream);
  t.stream = nullptr;
  return rc;
}

int sgdt_synchronize(sgdt_session* s) {
  if (!s) return fail(SGDT_ERR_DOMAIN, "null session");
  SGDT_CUDA(cudaSetDevice(s->device));
  SGDT_CUDA(cudaStreamSynchronize(s->stream));
  SGDT_CUDA(cudaStreamSynchronize(s->side));
  return SGDT_OK;
}

uint64_t sgdt_workspace_bytes(sgdt_session* s) {
  if (!s) return 0;
  uint32_t js = 0;
  for (int k = 0; k < s->order; ++k) js = std::max(js, s->J[k]);
  uint64_t b = s->batch_cap * sizeof(uint32_t);
  b += s->cs_cap * (static_cast<uint64_t>(js) + s->RP + 2) * sizeof(float);
  b += 2ull * s->num_sms * js * sizeof(double);
  if (s->batch_cap) b += 5ull * (s->batch_cap / (2 * s->order)) * sizeof(uint32_t);
  uint32_t pieces = 0;
  for (int n = 0; n < s->order; ++n) pieces = std::max(pieces, s->mode[n].n_pieces);
  b += static_cast<uint64_t>(pieces) * s->RP * sizeof(double);
  return b;
}

int sgdt_last_timing(sgdt_session* s, sgdt_timing* t) {
  if (!s || !t) return fail(SGDT_ERR_DOMAIN, "null argument");
  if (!s->timing_valid) return fail(SGDT_ERR_DOMAIN, "no epoch has been timed yet");
  *t = s->timing;
  return SGDT_OK;
}

}  // extern "C"
