// sgdt_synth.cu -- the BASELINE config 2-5 generator on the device
// (it extends the reference's synth.cpp:16-103,
// which only draws uniform positions with a Gaussian teacher).
//
//   indices  per mode: bounded-support Zipf(s) by inverse CDF over 1..I_n
//            (rank 1 hottest) or uniform, from a counter-based Philox4x32-10
//            stream (key = seed, counter = (draw, mode));
//   dedup    first draw wins: a stable radix sort of the (two-word) linear
//            position keys, first occurrences kept, the nnz earliest draws
//            taken, then ascending linear position (mode 1 fastest), as the
//            reference's draw_positions sorts (synth.cpp:40);
//   teacher  A^(n), B^(n) i.i.d. N(0, sigma^2), sigma = (J R^(1/N))^(-1/4)
//            (unit-variance prediction), Box-Muller on Philox streams;
//            xhat = sum_r prod_n (A^(n) B^(n))[i_n, r] in fp64;
//   values   ratings (config 2): round(3 + (xhat - mean) / sd) clipped to
//            [1, 5], sd unbiased; else xhat + noise * N(0, 1).
//
// The numpy restatement oracle/synth_oracle.py generates the same tensor
// (tests/test_synth.py): indices bit-exact, values to fp64 rounding.
// Input preparation only -- never inside a timed region.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <string>
#include <vector>

#include "sgdt_internal.cuh"

namespace sgdt {
namespace {

// ---- Philox4x32-10 (Salmon et al., SC'11) ---------------------------------
struct U4 {
  uint32_t x, y, z, w;
};

__host__ __device__ inline U4 philox(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    if (i) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c.x;
    const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c.z;
    c = U4{static_cast<uint32_t>(p1 >> 32) ^ c.y ^ k0, static_cast<uint32_t>(p1),
           static_cast<uint32_t>(p0 >> 32) ^ c.w ^ k1, static_cast<uint32_t>(p0)};
  }
  return c;
}

// uniform in [0, 1) with 53 bits from two words
__host__ __device__ inline double unit53(uint32_t hi, uint32_t lo) {
  return static_cast<double>(((static_cast<uint64_t>(hi) << 32) | lo) >> 11) * 0x1.0p-53;
}

constexpr uint32_t kTagDraw = 0x5A1F0000u, kTagTeacher = 0x7EAC0000u, kTagNoise = 0x00150000u;

__device__ inline double normal_at(uint64_t e, uint32_t stream, uint32_t tag, uint64_t seed) {
  const U4 r = philox(U4{static_cast<uint32_t>(e), static_cast<uint32_t>(e >> 32), stream, tag},
                      static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  const double u1 = unit53(r.x, r.y), u2 = unit53(r.z, r.w);
  return sqrt(-2.0 * log(1.0 - u1)) * cos(6.283185307179586 * u2);
}

// ---- Zipf CDF: weights (i+1)^-s, blocked prefix sums ----------------------
// cdf[b * 1024 + j] = off[b] + (sequential sum of block b up to j), off[b] =
// sequential sum of the earlier block totals; then divided by the total.  The
// association is fixed, so the numpy oracle reproduces it.
constexpr int kCdfBlock = 1024;

__global__ void cdf_block_kernel(double s, uint32_t I, double* cdf, double* tot) {
  const uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t i0 = b * kCdfBlock;
  if (i0 >= I) return;
  const uint64_t i1 = i0 + kCdfBlock < I ? i0 + kCdfBlock : I;
  double acc = 0.0;
  for (uint64_t i = i0; i < i1; ++i) {
    acc += pow(static_cast<double>(i + 1), -s);
    cdf[i] = acc;
  }
  tot[b] = acc;
}

__global__ void cdf_offsets_kernel(uint64_t nb, double* tot) {  // one thread: exclusive scan, total last
  double acc = 0.0;
  for (uint64_t b = 0; b < nb; ++b) {
    const double t = tot[b];
    tot[b] = acc;
    acc += t;
  }
  tot[nb] = acc;
}

__global__ void cdf_finish_kernel(uint32_t I, const double* tot, uint64_t nb, double* cdf) {
  const double total = tot[nb];
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < I;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    cdf[i] = (tot[i / kCdfBlock] + cdf[i]) / total;
}

// ---- index draws -> two-word linear keys -----------------------------------
struct ModeTab {
  uint32_t dims[kMaxOrder];
  double s[kMaxOrder];
  const double* cdf[kMaxOrder];
  int order;
};

__device__ inline uint32_t draw_index(const ModeTab& t, int k, uint64_t d, uint64_t seed) {
  const U4 r = philox(U4{static_cast<uint32_t>(d), static_cast<uint32_t>(d >> 32), static_cast<uint32_t>(k), kTagDraw},
                      static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  const double u = unit53(r.x, r.y);
  const uint32_t I = t.dims[k];
  if (t.s[k] == 0.0) {
    const uint64_t v = static_cast<uint64_t>(u * I);
    return static_cast<uint32_t>(v < I ? v : I - 1);
  }
  const double* c = t.cdf[k];  // first i with cdf[i] > u
  uint32_t lo = 0, hi = I;
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (c[mid] > u) hi = mid; else lo = mid + 1;
  }
  return lo < I ? lo : I - 1;
}

// linear position (mode 1 fastest) as 128 bits (hi, lo)
__global__ void draw_keys_kernel(ModeTab t, uint64_t d0, uint64_t n, uint64_t seed, uint64_t* khi, uint64_t* klo,
                                 uint64_t* id) {
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t d = d0 + q;
    unsigned __int128 key = 0, stride = 1;
    for (int k = 0; k < t.order; ++k) {
      key += static_cast<unsigned __int128>(draw_index(t, k, d, seed)) * stride;
      stride *= t.dims[k];
    }
    khi[d] = static_cast<uint64_t>(key >> 64);
    klo[d] = static_cast<uint64_t>(key);
    id[d] = d;
  }
}

__global__ void first_flags_kernel(const uint64_t* khi, const uint64_t* klo, uint64_t n, unsigned char* f) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    f[i] = i == 0 || khi[i] != khi[i - 1] || klo[i] != klo[i - 1];
}

// ---- teacher and values -----------------------------------------------------
__global__ void teacher_kernel(double* out, uint64_t n, uint32_t stream, uint64_t seed, double sigma) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[e] = sigma * normal_at(e, stream, kTagTeacher, seed);
}

// Q = A B (I x J times J x R), fp64, j ascending
__global__ void q_kernel(const double* A, const double* B, uint64_t I, uint32_t J, uint32_t R, double* Q) {
  for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < I * R;
       q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = q / R;
    const uint32_t r = static_cast<uint32_t>(q % R);
    double acc = 0.0;
    for (uint32_t j = 0; j < J; ++j) acc += A[i * J + j] * B[static_cast<uint64_t>(j) * R + r];
    Q[q] = acc;
  }
}

struct QTab {
  const double* q[kMaxOrder];
  uint32_t dims[kMaxOrder];
  int order;
  uint32_t R;
};

// entries in final order: coords (1-based, entry-major) and xhat
__global__ void entries_kernel(QTab t, const uint64_t* khi, const uint64_t* klo, uint64_t n, uint32_t* coords,
                               double* xhat) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    unsigned __int128 key = (static_cast<unsigned __int128>(khi[e]) << 64) | klo[e];
    uint32_t idx[kMaxOrder];
    for (int k = 0; k < t.order; ++k) {
      idx[k] = static_cast<uint32_t>(key % t.dims[k]);
      key /= t.dims[k];
      coords[e * t.order + k] = idx[k] + 1;
    }
    double x = 0.0;
    for (uint32_t r = 0; r < t.R; ++r) {
      double c = 1.0;
      for (int k = 0; k < t.order; ++k) c *= t.q[k][static_cast<uint64_t>(idx[k]) * t.R + r];
      x += c;
    }
    xhat[e] = x;
  }
}

__global__ void noise_kernel(double* v, uint64_t n, double noise, uint64_t seed) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    v[e] += noise * normal_at(e, 99u, kTagNoise, seed);
}

// two-pass (mean, then sum of squares) fp64 sums with a fixed association:
// per-block sequential chunks of 4096, block results summed in order
constexpr int kSumChunk = 4096;
__global__ void chunk_sums_kernel(const double* v, uint64_t n, const double* center, double* part) {
  const uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t i0 = c * kSumChunk;
  if (i0 >= n) return;
  const uint64_t i1 = i0 + kSumChunk < n ? i0 + kSumChunk : n;
  const double m = center ? *center : 0.0;
  double acc = 0.0;
  for (uint64_t i = i0; i < i1; ++i) {
    const double d = v[i] - m;
    acc += center ? d * d : v[i];
  }
  part[c] = acc;
}

__global__ void sum_parts_kernel(const double* part, uint64_t nc, uint64_t n, double* out, int mode) {
  double acc = 0.0;
  for (uint64_t c = 0; c < nc; ++c) acc += part[c];
  *out = mode == 0 ? acc / static_cast<double>(n) : sqrt(acc / static_cast<double>(n - 1));
}

__global__ void ratings_kernel(double* v, uint64_t n, const double* mean, const double* sd) {
  const double m = *mean, s = *sd;
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const double x = rint(3.0 + (v[e] - m) / s);
    v[e] = x < 1.0 ? 1.0 : (x > 5.0 ? 5.0 : x);
  }
}

unsigned grid_of(uint64_t n, int sms) {
  const uint64_t g = (n + 255) / 256, cap = static_cast<uint64_t>(sms) * 32;
  return static_cast<unsigned>(g < 1 ? 1 : (g > cap ? cap : g));
}

// Device buffers freed on every exit path.
struct Bufs {
  std::vector<void*> p;
  template <class T>
  cudaError_t alloc(T** x, uint64_t n) {
    *x = nullptr;
    const cudaError_t e = cudaMalloc(reinterpret_cast<void**>(x), (n ? n : 1) * sizeof(T));
    if (e == cudaSuccess) p.push_back(*x);
    return e;
  }
  void release(void* x) {
    for (auto& q : p)
      if (q == x) {
        cudaFree(q);
        q = nullptr;
      }
  }
  ~Bufs() {
    for (void* q : p)
      if (q) cudaFree(q);
  }
};

__global__ void iota64_kernel(uint64_t* p, uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    p[i] = i;
}

__global__ void gather64_kernel(const uint64_t* src, const uint64_t* idx, uint64_t n, uint64_t* dst) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[idx[i]];
}

#define SY(x)                                   \
  do {                                          \
    const cudaError_t e_ = (x);                 \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x); \
  } while (0)

int cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();
  return fail(e == cudaErrorMemoryAllocation ? SGDT_ERR_CONFIG : SGDT_ERR_INTERNAL,
              std::string("synth: ") + what + ": " + cudaGetErrorString(e));
}

// Stable sort of the pairs (k, v) by k (64 bits), in place through scratch.
int sort_pairs(Bufs& b, uint64_t n, uint64_t* k, uint64_t* v, uint64_t* k2, uint64_t* v2, cudaStream_t st) {
  if (n <= 1) return SGDT_OK;
  if (n > static_cast<uint64_t>(INT_MAX)) return fail(SGDT_ERR_CONFIG, "synth: too many draws for one sort");
  size_t tmp = 0;
  SY(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k, k2, v, v2, static_cast<int>(n), 0, 64, st));
  void* t = nullptr;
  SY(cudaMalloc(&t, tmp));
  const cudaError_t e = cub::DeviceRadixSort::SortPairs(t, tmp, k, k2, v, v2, static_cast<int>(n), 0, 64, st);
  cudaFree(t);
  SY(e);
  SY(cudaMemcpyAsync(k, k2, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
  SY(cudaMemcpyAsync(v, v2, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
  return SGDT_OK;
}

#define SR(x)              \
  do {                     \
    const int rc_ = (x);   \
    if (rc_) return rc_;   \
  } while (0)

}  // namespace
}  // namespace sgdt

using namespace sgdt;

extern "C" int sgdt_synth(const sgdt_synth_spec* sp, int device, uint32_t* coords_out, double* values_out) {
  if (!sp || !sp->dims || !sp->zipf || !coords_out || !values_out) return fail(SGDT_ERR_DOMAIN, "synth: null argument");
  const int N = sp->order;
  if (N < 2 || N > kMaxOrder) return fail(SGDT_ERR_DOMAIN, "synth: order must be in [2, 8]");
  long double total = 1;
  for (int k = 0; k < N; ++k) {
    if (sp->dims[k] < 1) return fail(SGDT_ERR_DOMAIN, "synth: every dim must be >= 1");
    if (sp->zipf[k] < 0.0) return fail(SGDT_ERR_DOMAIN, "synth: Zipf exponents must be >= 0");
    total *= sp->dims[k];
  }
  const uint64_t nnz = sp->nnz;
  if (nnz == 0 || static_cast<long double>(nnz) > total / 2)
    return fail(SGDT_ERR_DOMAIN, "synth: nnz must lie in [1, half the index space]");
  if (nnz > 0xFFFFFFFFull) return fail(SGDT_ERR_CONFIG, "synth: entry count exceeds the 32-bit id space");
  if (sp->teacher_j < 1 || sp->teacher_r < 1) return fail(SGDT_ERR_DOMAIN, "synth: teacher ranks must be >= 1");
  if (device >= 0) SY(cudaSetDevice(device));
  int dev = 0, sms = 148;
  SY(cudaGetDevice(&dev));
  SY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaStream_t st = nullptr;
  SY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } sg{st};
  Bufs b;
  const uint64_t seed = sp->seed;
  const bool wide = total >= static_cast<long double>(18446744073709551615.0L);

  // Zipf CDFs
  ModeTab mt{};
  mt.order = N;
  for (int k = 0; k < N; ++k) {
    mt.dims[k] = sp->dims[k];
    mt.s[k] = sp->zipf[k];
    if (sp->zipf[k] == 0.0) continue;
    const uint64_t I = sp->dims[k], nb = (I + kCdfBlock - 1) / kCdfBlock;
    double *cdf = nullptr, *tot = nullptr;
    SY(b.alloc(&cdf, I));
    SY(b.alloc(&tot, nb + 1));
    cdf_block_kernel<<<static_cast<unsigned>((nb + 127) / 128), 128, 0, st>>>(sp->zipf[k], sp->dims[k], cdf, tot);
    cdf_offsets_kernel<<<1, 1, 0, st>>>(nb, tot);
    cdf_finish_kernel<<<grid_of(I, sms), 256, 0, st>>>(sp->dims[k], tot, nb, cdf);
    SY(cudaGetLastError());
    mt.cdf[k] = cdf;
  }

  // draws until nnz distinct positions: recompute from draw 0 with a larger
  // budget (draws are a pure function of their index)
  uint64_t cap = nnz + nnz / 4 + (1u << 20);
  uint64_t *khi = nullptr, *klo = nullptr, *id = nullptr, *k2 = nullptr, *v2 = nullptr, *sh = nullptr,
           *sl = nullptr, *uniq = nullptr;
  unsigned char* flag = nullptr;
  uint64_t* d_count = nullptr;
  SY(b.alloc(&d_count, 1));
  uint64_t U = 0;
  for (int round = 0;; ++round) {
    if (round > 40) return fail(SGDT_ERR_CONFIG, "synth: too few distinct positions (index space too concentrated)");
    for (void* x : {(void*)khi, (void*)klo, (void*)id, (void*)k2, (void*)v2, (void*)sh, (void*)sl, (void*)uniq,
                    (void*)flag})
      if (x) b.release(x);
    SY(b.alloc(&khi, cap));
    SY(b.alloc(&klo, cap));
    SY(b.alloc(&id, cap));
    SY(b.alloc(&k2, cap));
    SY(b.alloc(&v2, cap));
    SY(b.alloc(&sh, cap));
    SY(b.alloc(&sl, cap));
    SY(b.alloc(&uniq, cap));
    SY(b.alloc(&flag, cap));
    draw_keys_kernel<<<grid_of(cap, sms), 256, 0, st>>>(mt, 0, cap, seed, khi, klo, id);
    SY(cudaGetLastError());
    // (hi, lo) order, ties in draw order: stable by lo, then stable by hi
    SY(cudaMemcpyAsync(sl, klo, cap * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
    SR(sort_pairs(b, cap, sl, id, k2, v2, st));
    if (wide) {
      gather64_kernel<<<grid_of(cap, sms), 256, 0, st>>>(khi, id, cap, sh);
      SR(sort_pairs(b, cap, sh, id, k2, v2, st));
      gather64_kernel<<<grid_of(cap, sms), 256, 0, st>>>(klo, id, cap, sl);
    } else {
      SY(cudaMemsetAsync(sh, 0, cap * sizeof(uint64_t), st));
    }
    first_flags_kernel<<<grid_of(cap, sms), 256, 0, st>>>(sh, sl, cap, flag);
    SY(cudaGetLastError());
    size_t tmp = 0;
    SY(cub::DeviceSelect::Flagged(nullptr, tmp, id, flag, uniq, d_count, static_cast<int>(cap), st));
    void* t = nullptr;
    SY(cudaMalloc(&t, tmp));
    const cudaError_t e = cub::DeviceSelect::Flagged(t, tmp, id, flag, uniq, d_count, static_cast<int>(cap), st);
    cudaFree(t);
    SY(e);
    SY(cudaMemcpyAsync(&U, d_count, sizeof U, cudaMemcpyDeviceToHost, st));
    SY(cudaStreamSynchronize(st));
    if (U >= nnz) break;
    cap = cap + cap / 2;
  }
  // the nnz earliest first-occurrences, then ascending position
  {
    SY(cudaMemcpyAsync(k2, uniq, U * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));  // keys = draw ids
    size_t tmp = 0;
    SY(cub::DeviceRadixSort::SortKeys(nullptr, tmp, k2, v2, static_cast<int>(U), 0, 64, st));
    void* t = nullptr;
    SY(cudaMalloc(&t, tmp));
    const cudaError_t e = cub::DeviceRadixSort::SortKeys(t, tmp, k2, v2, static_cast<int>(U), 0, 64, st);
    cudaFree(t);
    SY(e);
  }
  // v2[0, nnz): the kept draw ids; their keys
  gather64_kernel<<<grid_of(nnz, sms), 256, 0, st>>>(khi, v2, nnz, sh);
  gather64_kernel<<<grid_of(nnz, sms), 256, 0, st>>>(klo, v2, nnz, sl);
  SY(cudaGetLastError());
  SR(sort_pairs(b, nnz, sl, sh, k2, id, st));  // by lo, carrying hi
  if (wide) SR(sort_pairs(b, nnz, sh, sl, k2, id, st));  // then by hi, carrying lo (stable)
  b.release(khi);
  b.release(klo);
  b.release(uniq);
  b.release(flag);
  b.release(v2);
  khi = klo = uniq = v2 = nullptr;
  flag = nullptr;

  // teacher Q^(n) = A^(n) B^(n), sigma = (J R^(1/N))^(-1/4)
  const uint32_t J = sp->teacher_j, R = sp->teacher_r;
  const double sigma = std::pow(J * std::pow(static_cast<double>(R), 1.0 / N), -0.25);
  QTab qt{};
  qt.order = N;
  qt.R = R;
  for (int k = 0; k < N; ++k) {
    const uint64_t I = sp->dims[k];
    double *A = nullptr, *B = nullptr, *Q = nullptr;
    SY(b.alloc(&A, I * J));
    SY(b.alloc(&B, static_cast<uint64_t>(J) * R));
    SY(b.alloc(&Q, I * R));
    teacher_kernel<<<grid_of(I * J, sms), 256, 0, st>>>(A, I * J, 16u + 2u * k, seed, sigma);
    teacher_kernel<<<grid_of(static_cast<uint64_t>(J) * R, sms), 256, 0, st>>>(B, static_cast<uint64_t>(J) * R,
                                                                             17u + 2u * k, seed, sigma);
    q_kernel<<<grid_of(I * R, sms), 256, 0, st>>>(A, B, I, J, R, Q);
    SY(cudaGetLastError());
    b.release(A);
    b.release(B);
    qt.q[k] = Q;
    qt.dims[k] = sp->dims[k];
  }
  uint32_t* d_coords = nullptr;
  double* d_val = nullptr;
  SY(b.alloc(&d_coords, nnz * N));
  SY(b.alloc(&d_val, nnz));
  entries_kernel<<<grid_of(nnz, sms), 256, 0, st>>>(qt, sh, sl, nnz, d_coords, d_val);
  SY(cudaGetLastError());
  if (sp->ratings) {
    const uint64_t nc = (nnz + kSumChunk - 1) / kSumChunk;
    double *part = nullptr, *stats = nullptr;
    SY(b.alloc(&part, nc));
    SY(b.alloc(&stats, 2));
    chunk_sums_kernel<<<static_cast<unsigned>((nc + 127) / 128), 128, 0, st>>>(d_val, nnz, nullptr, part);
    sum_parts_kernel<<<1, 1, 0, st>>>(part, nc, nnz, stats, 0);
    chunk_sums_kernel<<<static_cast<unsigned>((nc + 127) / 128), 128, 0, st>>>(d_val, nnz, stats, part);
    sum_parts_kernel<<<1, 1, 0, st>>>(part, nc, nnz, stats + 1, 1);
    ratings_kernel<<<grid_of(nnz, sms), 256, 0, st>>>(d_val, nnz, stats, stats + 1);
  } else if (sp->noise > 0.0) {
    noise_kernel<<<grid_of(nnz, sms), 256, 0, st>>>(d_val, nnz, sp->noise, seed);
  }
  SY(cudaGetLastError());
  SY(cudaMemcpyAsync(coords_out, d_coords, nnz * N * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  SY(cudaMemcpyAsync(values_out, d_val, nnz * sizeof(double), cudaMemcpyDeviceToHost, st));
  SY(cudaStreamSynchronize(st));
  return SGDT_OK;
}
