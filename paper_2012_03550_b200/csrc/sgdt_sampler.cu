// sgdt_sampler.cu -- K1: bit-exact device sample_batch.
//
// Reference: sample_batch (sptensor.cpp:256-270) = partial Fisher-Yates over a
// pool that persists across epochs, with draws
//   j_i = i + Rng::next_below(nnz - i)   (rng.hpp:20-25, std::mt19937_64).
//
// Device plan:
//  1. mt_draw_kernel (one CTA): the mt19937_64 state lives in shared memory;
//     a twist is two parallel half-steps of 156 lanes; each block of 312
//     tempered outputs is mapped optimistically to consecutive draws, the
//     rejection test `r < (2^64 - bound) mod bound` is evaluated per lane and
//     a block that contains a rejection is replayed sequentially by lane 0, so
//     the engine consumes exactly the outputs the host would.
//  2. The swap chain is resolved in parallel.  With V(p,i) = value at
//     position p before step i and D(i) = V(i,i):
//        out[i] = D(k)    k = max{k < i : j_k = j_i}, else pool0[j_i]
//        D(i)   = D(l)    l = max{l < i : j_l = i},   else pool0[i]
//     Draws sharing a target are linked through a stamped list head per pool
//     position (atomicExch); every predecessor query walks its (tiny) list, so
//     the result does not depend on the atomic order.  Final pool: positions
//     < m hold out[], a touched position p >= m holds D(last k with j_k = p).
#include <cuda_runtime.h>

#include "sgdt_internal.cuh"

namespace sgdt {

namespace {

constexpr int kMtN = 312;
constexpr int kMtM = 156;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ULL;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL;
constexpr uint64_t kLower = 0x000000007FFFFFFFULL;

__device__ __forceinline__ uint64_t temper(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= (z >> 43);
  return z;
}

__device__ __forceinline__ uint64_t twist_word(uint64_t cur, uint64_t nxt, uint64_t far) {
  const uint64_t y = (cur & kUpper) | (nxt & kLower);
  return far ^ (y >> 1) ^ ((y & 1ULL) ? kMtA : 0ULL);
}

// In-place twist of x[312] by 320 threads (two half-steps, reads before writes).
__device__ void mt_twist(uint64_t* x) {
  const int t = threadIdx.x;
  uint64_t v = 0;
  if (t < kMtN - kMtM) v = twist_word(x[t], x[t + 1], x[t + kMtM]);
  __syncthreads();
  if (t < kMtN - kMtM) x[t] = v;
  __syncthreads();
  if (t >= kMtN - kMtM && t < kMtN) v = twist_word(x[t], x[(t + 1) % kMtN], x[t - (kMtN - kMtM)]);
  __syncthreads();
  if (t >= kMtN - kMtM && t < kMtN) x[t] = v;
  __syncthreads();
}

// What a run of sequential next_below draws means.
//   BATCH:  draw d of sample_batch: bound = nnz - d, target = d + r % bound
//           (sptensor.cpp:265-268), position d.
//   BOUNDS: explicit u64 bounds (test hook), raw value r % bound.
//   ROWS:   row_fraction < 1 (factor_optimizer.cpp:143-165): draws are grouped
//           by row (rows ascending, sub_off = prefix sums of keep); draw q of
//           row i has bound bs_i - q, position row_ptr[i] + q and target
//           position + r % bound inside the bucket.
struct DrawPlan {
  int kind;  // 0 BATCH, 1 BOUNDS, 2 ROWS
  uint64_t nnz;
  const uint64_t* bounds;
  const uint32_t* sub_off;
  uint32_t n_rows;
  const uint32_t* row_ptr;
  uint32_t* out_target;
  uint32_t* out_pos;
  uint64_t* out64;
};

__device__ __forceinline__ uint64_t plan_bound(const DrawPlan& p, uint64_t d, uint64_t* base) {
  if (p.kind == 0) {
    *base = d;
    return p.nnz - d;
  }
  if (p.kind == 1) {
    *base = 0;
    return p.bounds[d];
  }
  uint32_t lo = 0, hi = p.n_rows;  // largest row with sub_off[row] <= d
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (p.sub_off[mid] <= d) lo = mid; else hi = mid;
  }
  const uint64_t q = d - p.sub_off[lo];
  *base = p.row_ptr[lo] + q;
  return static_cast<uint64_t>(p.row_ptr[lo + 1] - p.row_ptr[lo]) - q;
}

__device__ __forceinline__ void plan_store(const DrawPlan& p, uint64_t d, uint64_t base, uint64_t v) {
  if (p.kind == 1) {
    p.out64[d] = v;
    return;
  }
  p.out_target[d] = static_cast<uint32_t>(base + v);
  if (p.out_pos) p.out_pos[d] = static_cast<uint32_t>(base);
}

// m draws in stream order.  Each block of 312 tempered outputs is mapped
// optimistically to consecutive draws; a block containing a rejection is
// replayed by lane 0 so exactly the reference's outputs are consumed.
__global__ void __launch_bounds__(320) mt_draw_kernel(uint64_t* state, uint64_t m, DrawPlan plan) {
  __shared__ uint64_t x[kMtN];
  __shared__ uint64_t s_done, s_pos;
  const int t = threadIdx.x;
  if (t < kMtN) x[t] = state[t];
  if (t == 0) {
    s_done = 0;
    s_pos = state[kMtN];
  }
  __syncthreads();
  while (true) {
    const uint64_t done = s_done;
    uint64_t pos = s_pos;
    if (done >= m) break;
    if (pos >= kMtN) {
      mt_twist(x);
      pos = 0;
    }
    const uint64_t avail = kMtN - pos;
    const uint64_t take = (m - done) < avail ? (m - done) : avail;
    uint64_t r = 0, bound = 1, base = 0, d = done + t;
    int rej = 0;
    if (t < take) {
      r = temper(x[pos + t]);
      bound = plan_bound(plan, d, &base);
      rej = r < (0ULL - bound) % bound;
    }
    const int any = __syncthreads_or(rej);
    if (!any) {
      if (t < take) plan_store(plan, d, base, r % bound);
      __syncthreads();
      if (t == 0) {
        s_done = done + take;
        s_pos = pos + take;
      }
    } else if (t == 0) {
      uint64_t dd = done, p = pos;
      while (dd < m && p < kMtN) {
        const uint64_t rr = temper(x[p++]);
        uint64_t bb = 0;
        const uint64_t b = plan_bound(plan, dd, &bb);
        if (rr < (0ULL - b) % b) continue;
        plan_store(plan, dd, bb, rr % b);
        ++dd;
      }
      s_done = dd;
      s_pos = p;
    }
    __syncthreads();
  }
  if (t < kMtN) state[t] = x[t];
  if (t == 0) state[kMtN] = s_pos;
}

__global__ void iota_kernel(uint32_t* p, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = static_cast<uint32_t>(i);
}

__global__ void link_kernel(uint64_t m, const uint32_t* __restrict__ jd,
                            unsigned long long* head, uint32_t stamp, uint32_t* link) {
  const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const unsigned long long tag = (static_cast<unsigned long long>(stamp) << 32) | k;
  const unsigned long long old = atomicExch(&head[jd[k]], tag);
  link[k] = (old >> 32) == stamp ? static_cast<uint32_t>(old) : kNone;
}

// max element < bound of the list starting at head[p] (current stamp only)
__device__ __forceinline__ uint32_t list_max_below(const unsigned long long* head,
                                                   const uint32_t* link, uint32_t stamp,
                                                   uint32_t p, uint32_t bound) {
  const unsigned long long h = head[p];
  if ((h >> 32) != stamp) return kNone;
  uint32_t best = kNone;
  for (uint32_t k = static_cast<uint32_t>(h); k != kNone; k = link[k])
    if (k < bound && (best == kNone || k > best)) best = k;
  return best;
}

// pos: position of each draw (nullptr: draw i sits at position i).
__global__ void resolve_kernel(uint64_t m, const uint32_t* __restrict__ jd, const uint32_t* __restrict__ pos,
                               const unsigned long long* head, const uint32_t* link,
                               uint32_t stamp, uint32_t* kprev, uint32_t* lprev) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint32_t p = pos ? pos[i] : static_cast<uint32_t>(i);
  kprev[i] = list_max_below(head, link, stamp, jd[i], static_cast<uint32_t>(i));
  lprev[i] = list_max_below(head, link, stamp, p, static_cast<uint32_t>(i));
}

// D(x): value at draw x's position just before step x.  pool == nullptr:
// the initial pool is the identity (row subsets start from bucket order).
__device__ __forceinline__ uint32_t chain_value(const uint32_t* pool, const uint32_t* pos,
                                                const uint32_t* lprev, uint32_t x) {
  while (lprev[x] != kNone) x = lprev[x];
  const uint32_t p = pos ? pos[x] : x;
  return pool ? pool[p] : p;
}

__global__ void chain_kernel(uint64_t m, const uint32_t* __restrict__ pool, const uint32_t* __restrict__ pos,
                             const uint32_t* __restrict__ jd, const uint32_t* kprev,
                             const uint32_t* lprev, uint32_t* dval, uint32_t* out) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  if (dval) dval[i] = chain_value(pool, pos, lprev, static_cast<uint32_t>(i));
  const uint32_t k = kprev[i];
  out[i] = k == kNone ? (pool ? pool[jd[i]] : jd[i]) : chain_value(pool, pos, lprev, k);
}

__global__ void write_pool_kernel(uint64_t m, uint32_t* pool, const uint32_t* __restrict__ jd,
                                  const unsigned long long* head, const uint32_t* link,
                                  uint32_t stamp, const uint32_t* out, const uint32_t* dval) {
  const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  pool[k] = out[k];
  const uint32_t p = jd[k];
  if (p >= m) {
    const uint32_t owner = list_max_below(head, link, stamp, p, kNone);
    if (owner == k) pool[p] = dval[k];
  }
}

}  // namespace

int launch_sampler(Session& s, uint64_t m, uint32_t* out_batch, cudaStream_t st) {
  if (!s.pool_valid) {
    iota_kernel<<<s.num_sms * 4, 256, 0, st>>>(s.pool, s.nnz);
    ++s.launches;
    SGDT_CUDA(cudaGetLastError());
    s.pool_valid = true;
  }
  if (++s.stamp == 0) {  // stamp wrapped: clear the list heads once
    SGDT_CUDA(cudaMemsetAsync(s.head, 0, s.nnz * sizeof(unsigned long long), st));
    s.stamp = 1;
  }
  DrawPlan plan{};
  plan.kind = 0;
  plan.nnz = s.nnz;
  plan.out_target = s.draw_j;
  mt_draw_kernel<<<1, 320, 0, st>>>(s.mt, m, plan);
  SGDT_CUDA(cudaGetLastError());
  const unsigned blocks = static_cast<unsigned>((m + 255) / 256);
  link_kernel<<<blocks, 256, 0, st>>>(m, s.draw_j, s.head, s.stamp, s.link);
  resolve_kernel<<<blocks, 256, 0, st>>>(m, s.draw_j, nullptr, s.head, s.link, s.stamp, s.kprev, s.lprev);
  chain_kernel<<<blocks, 256, 0, st>>>(m, s.pool, nullptr, s.draw_j, s.kprev, s.lprev, s.dval, out_batch);
  write_pool_kernel<<<blocks, 256, 0, st>>>(m, s.pool, s.draw_j, s.head, s.link, s.stamp,
                                            out_batch, s.dval);
  SGDT_CUDA(cudaGetLastError());
  s.launches += 5;
  s.last_batch = out_batch;
  s.last_batch_len = m;
  return SGDT_OK;
}

// row_fraction < 1 for one mode: per-row partial Fisher-Yates of every
// bucket (a fresh copy each epoch, factor_optimizer.cpp:405-419), all rows'
// draws from the session RNG in row order.  out[d] (d in row i's draw range
// sub_off[i]..sub_off[i+1]) is the mode-order position of the kept entry.
int launch_row_subsets(Session& s, int n, RowSubset& rs, cudaStream_t st) {
  const uint64_t T = rs.total;
  if (T == 0) return SGDT_OK;
  if (++s.stamp == 0) {
    SGDT_CUDA(cudaMemsetAsync(s.head, 0, s.nnz * sizeof(unsigned long long), st));
    s.stamp = 1;
  }
  DrawPlan plan{};
  plan.kind = 2;
  plan.sub_off = rs.sub_off;
  plan.n_rows = s.dims[n];
  plan.row_ptr = s.mode[n].row_ptr;
  plan.out_target = rs.target;
  plan.out_pos = rs.pos;
  mt_draw_kernel<<<1, 320, 0, st>>>(s.mt, T, plan);
  SGDT_CUDA(cudaGetLastError());
  const unsigned blocks = static_cast<unsigned>((T + 255) / 256);
  link_kernel<<<blocks, 256, 0, st>>>(T, rs.target, s.head, s.stamp, rs.link);
  resolve_kernel<<<blocks, 256, 0, st>>>(T, rs.target, rs.pos, s.head, rs.link, s.stamp, rs.kprev, rs.lprev);
  chain_kernel<<<blocks, 256, 0, st>>>(T, nullptr, rs.pos, rs.target, rs.kprev, rs.lprev, nullptr, rs.out);
  SGDT_CUDA(cudaGetLastError());
  s.launches += 4;
  return SGDT_OK;
}

}  // namespace sgdt

extern "C" int sgdt_rng_next_below(const uint64_t* mt312, uint32_t pos, const uint64_t* bounds,
                                   uint64_t n, uint64_t* out, uint64_t* mt312_out,
                                   uint32_t* pos_out) {
  using namespace sgdt;
  for (uint64_t i = 0; i < n; ++i)
    if (bounds[i] == 0) return fail(SGDT_ERR_DOMAIN, "next_below: bound must be >= 1");
  uint64_t *d_state = nullptr, *d_bounds = nullptr, *d_out = nullptr;
  SGDT_CUDA(cudaMalloc(&d_state, (kMtN + 1) * sizeof(uint64_t)));
  SGDT_CUDA(cudaMalloc(&d_bounds, (n + 1) * sizeof(uint64_t)));
  SGDT_CUDA(cudaMalloc(&d_out, (n + 1) * sizeof(uint64_t)));
  uint64_t h_state[kMtN + 1];
  for (int i = 0; i < kMtN; ++i) h_state[i] = mt312[i];
  h_state[kMtN] = pos;
  SGDT_CUDA(cudaMemcpy(d_state, h_state, sizeof h_state, cudaMemcpyHostToDevice));
  SGDT_CUDA(cudaMemcpy(d_bounds, bounds, n * sizeof(uint64_t), cudaMemcpyHostToDevice));
  DrawPlan plan{};
  plan.kind = 1;
  plan.bounds = d_bounds;
  plan.out64 = d_out;
  mt_draw_kernel<<<1, 320>>>(d_state, n, plan);
  SGDT_CUDA(cudaGetLastError());
  SGDT_CUDA(cudaMemcpy(out, d_out, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  SGDT_CUDA(cudaMemcpy(h_state, d_state, sizeof h_state, cudaMemcpyDeviceToHost));
  for (int i = 0; i < kMtN; ++i) mt312_out[i] = h_state[i];
  *pos_out = static_cast<uint32_t>(h_state[kMtN]);
  cudaFree(d_state);
  cudaFree(d_bounds);
  cudaFree(d_out);
  return SGDT_OK;
}
