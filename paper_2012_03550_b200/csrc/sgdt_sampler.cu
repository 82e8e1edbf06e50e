// sgdt_sampler.cu -- K1: bit-exact device sample_batch.
//
// Reference: sample_batch (sptensor.cpp:256-270) = partial Fisher-Yates over a
// pool that persists across epochs, with draws
//   j_i = i + Rng::next_below(nnz - i)   (rng.hpp:20-25, std::mt19937_64).
//
// Device plan:
//  1. Engine outputs, then draws (launch_draws):
//     mt_gen_kernel (one CTA) only runs the engine: the state is ping-ponged
//     between two shared buffers (a twist = two parallel half-steps of 156
//     lanes, two barriers), every block of 312 outputs is tempered and stored.
//     It also records the state the engine would end in if every output were
//     accepted.  draw_map_kernel (whole grid) maps output d to draw d: bound,
//     rejection test `r < (2^64 - bound) mod bound`, r mod bound.  The
//     sequential chain is only twist + temper; the bound lookups (a binary
//     search for row subsets) and the 64-bit modulos run in parallel.  A
//     rejection (probability < bound / 2^64 per draw) shifts every later draw
//     by one output, so mt_draw_kernel then replays the whole run
//     sequentially from the unchanged state (lane 0 re-maps each block that
//     holds a rejection); otherwise it just installs the recorded state.  The
//     engine therefore consumes exactly the outputs the host would.
//     Long runs (row_fraction < 1 draws one output per kept entry: ~f nnz per
//     mode) are cut into segments of kJumpL blocks that run in parallel.  The
//     twist T is linear over GF(2) on the 312 x 64 state bits, so the start
//     of segment k is J^k (T B0) with J = T^kJumpL: J (19968 x 19968 bits,
//     50 MB, built once per session by mt_jump_build_kernel, bit-sliced: 64
//     unit-vector simulations per CTA) is applied by a cooperative kernel
//     (mt_chain_kernel), then one CTA per segment runs the engine
//     (mt_seg_gen_kernel).  The outputs are identical to the sequential run.
//  2. The swap chain is resolved in parallel.  With V(p,i) = value at
//     position p before step i and D(i) = V(i,i):
//        out[i] = D(k)    k = max{k < i : j_k = j_i}, else pool0[j_i]
//        D(i)   = D(l)    l = max{l < i : j_l = i},   else pool0[i]
//     Draws sharing a target are linked through a stamped list head per pool
//     position (atomicExch); every predecessor query walks its (tiny) list, so
//     the result does not depend on the atomic order.  Final pool: positions
//     < m hold out[], a touched position p >= m holds D(last k with j_k = p).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "sgdt_internal.cuh"

namespace sgdt {

namespace {

#define TRY_RC(x)          \
  do {                     \
    const int rc_ = (x);   \
    if (rc_) return rc_;   \
  } while (0)

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

// Raw engine outputs: n consecutive tempered outputs from the state
// (312 words + position) into out, and into tent the state after them.
__global__ void __launch_bounds__(320) mt_gen_kernel(const uint64_t* __restrict__ state, uint64_t n,
                                                     uint64_t* __restrict__ out, uint64_t* __restrict__ tent) {
  __shared__ uint64_t x[2][kMtN];
  const int t = threadIdx.x;
  if (t < kMtN) x[0][t] = state[t];
  const uint64_t pos = state[kMtN];
  __syncthreads();
  int cur = 0;
  uint64_t done = 0, endpos = kMtN;
  if (pos < kMtN) {  // the rest of the current block
    const uint64_t take = n < kMtN - pos ? n : kMtN - pos;
    if (t < take) out[t] = temper(x[0][pos + t]);
    done = take;
    endpos = pos + take;
  }
  while (done < n) {
    const int nxt = cur ^ 1;
    if (t < kMtN - kMtM) x[nxt][t] = twist_word(x[cur][t], x[cur][t + 1], x[cur][t + kMtM]);
    __syncthreads();
    if (t >= kMtN - kMtM && t < kMtN)
      x[nxt][t] = twist_word(x[cur][t], t == kMtN - 1 ? x[nxt][0] : x[cur][t + 1], x[nxt][t - (kMtN - kMtM)]);
    __syncthreads();
    cur = nxt;
    const uint64_t take = n - done < kMtN ? n - done : kMtN;
    if (t < take) out[done + t] = temper(x[cur][t]);
    done += take;
    endpos = take;
  }
  if (t < kMtN) tent[t] = x[cur][t];
  if (t == 0) tent[kMtN] = endpos;
}

// ---- jump-ahead (long runs) ------------------------------------------------

constexpr int kJumpL = 2048;             // blocks of 312 outputs per segment
constexpr int kStateBits = kMtN * 64;    // 19968
constexpr int kJumpThreads = 512;

// J = T^kJumpL, column-major: J[c * 312 + w] = word w of T^kJumpL e_c, where
// e_c has bit (c % 64) of word (c / 64) set.  CTA g simulates the 64 columns
// of word g at once, bit-sliced: P[w * 64 + b] holds bit b of word w of the
// 64 simulations (bit j = column 64 g + j).  One twist, per word i and bit b:
//   y_b = (b >= 31 ? x_i : x_{i+1})_b
//   x'_i,b = x_far,b ^ y_{b+1} (b < 63) ^ (A_b ? y_0 : 0)
// with far = i + 156 (old) for i < 156 and i - 156 (new) after, and x_{312} =
// the new x_0: two phases, each staged in registers across a barrier.
__global__ void __launch_bounds__(kJumpThreads) mt_jump_build_kernel(int L, uint64_t* __restrict__ J) {
  extern __shared__ uint64_t P[];  // 312 x 64
  const int g = blockIdx.x, t = threadIdx.x;
  for (int i = t; i < kStateBits; i += kJumpThreads) {
    const int w = i >> 6, b = i & 63;
    P[i] = w == g ? (1ULL << b) : 0ULL;
  }
  __syncthreads();
  constexpr int kHalf = (kMtN - kMtM) * 64;  // 9984 items per phase
  constexpr int kPer = (kHalf + kJumpThreads - 1) / kJumpThreads;
  for (int step = 0; step < L; ++step) {
#pragma unroll
    for (int phase = 0; phase < 2; ++phase) {
      uint64_t v[kPer];
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int it = t + q * kJumpThreads;
        v[q] = 0;
        if (it < kHalf) {
          const int i = (it >> 6) + phase * (kMtN - kMtM), b = it & 63;
          const int nx = i + 1 == kMtN ? 0 : i + 1;
          const int far = phase == 0 ? i + kMtM : i - (kMtN - kMtM);
          const uint64_t y0 = P[nx * 64];
          uint64_t r = P[far * 64 + b];
          if (b < 63) r ^= P[(b + 1 >= 31 ? i : nx) * 64 + b + 1];
          if ((kMtA >> b) & 1ULL) r ^= y0;
          v[q] = r;
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int it = t + q * kJumpThreads;
        if (it < kHalf) P[(phase * (kMtN - kMtM)) * 64 + it] = v[q];
      }
      __syncthreads();
    }
  }
  // transpose 64 x 64 bit blocks: column 64 g + j, word w
  for (int it = t; it < kStateBits; it += kJumpThreads) {
    const int j = it / kMtN, w = it % kMtN;
    uint64_t col = 0;
    for (int b = 0; b < 64; ++b) col |= ((P[w * 64 + b] >> j) & 1ULL) << b;
    J[static_cast<uint64_t>(g * 64 + j) * kMtN + w] = col;
  }
}

// Segment starts: st[0] = T B0 (B0 = the current state words), st[k] =
// J st[k-1] for k < ns.  Cooperative: per step every CTA XORs the columns of
// J selected by its share of st[k-1]'s bits into a partial, then the partials
// are reduced word by word.
__global__ void __launch_bounds__(kJumpThreads) mt_chain_kernel(const uint64_t* __restrict__ state,
                                                                const uint64_t* __restrict__ J, int ns,
                                                                uint64_t* st, uint64_t* part) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ uint64_t x[kMtN];
  const int t = threadIdx.x, nb = gridDim.x;
  if (blockIdx.x == 0) {  // st[0] = T B0 (in-place twist of a shared copy)
    if (t < kMtN) x[t] = state[t];
    __syncthreads();
    uint64_t v = 0;
    if (t < kMtN - kMtM) v = twist_word(x[t], x[t + 1], x[t + kMtM]);
    __syncthreads();
    if (t < kMtN - kMtM) x[t] = v;
    __syncthreads();
    if (t >= kMtN - kMtM && t < kMtN) v = twist_word(x[t], x[(t + 1) % kMtN], x[t - (kMtN - kMtM)]);
    __syncthreads();
    if (t >= kMtN - kMtM && t < kMtN) st[t] = v;
    if (t < kMtN - kMtM) st[t] = x[t];
  }
  grid.sync();
  // this CTA's columns, a whole number of state words: [64 w0, 64 w1)
  const int wper = (kMtN + nb - 1) / nb;
  const int w0 = min(kMtN, static_cast<int>(blockIdx.x) * wper), w1 = min(kMtN, w0 + wper);
  __shared__ uint64_t bits[kMtN];
  __shared__ uint64_t red[kJumpThreads / 32];
  for (int k = 1; k < ns; ++k) {
    const uint64_t* prev = st + static_cast<uint64_t>(k - 1) * kMtN;
    if (t < w1 - w0) bits[t] = __ldcg(prev + w0 + t);  // st/part are rewritten by other CTAs: L2 loads
    __syncthreads();
    if (t < kMtN) {
      uint64_t a = 0;
      for (int w = w0; w < w1; ++w) {
        const uint64_t m = bits[w - w0];
        const uint64_t* col = J + static_cast<uint64_t>(w) * 64 * kMtN + t;
#pragma unroll 16
        for (int b = 0; b < 64; ++b) {  // unconditional loads, masked XOR: the loads pipeline
          const uint64_t v = col[static_cast<uint64_t>(b) * kMtN];
          a ^= v & (0ULL - ((m >> b) & 1ULL));
        }
      }
      part[static_cast<uint64_t>(blockIdx.x) * kMtN + t] = a;
    }
    grid.sync();
    // word w of st[k] = XOR of the nb partials: thread b loads partial b,
    // a shuffle + shared reduction per word
    for (int w = blockIdx.x; w < kMtN; w += nb) {
      uint64_t a = t < nb ? __ldcg(part + static_cast<uint64_t>(t) * kMtN + w) : 0ULL;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a ^= __shfl_xor_sync(0xffffffffu, a, o);
      if ((t & 31) == 0) red[t >> 5] = a;
      __syncthreads();
      if (t == 0) {
        uint64_t r = 0;
        for (int i = 0; i < kJumpThreads / 32; ++i) r ^= red[i];
        st[static_cast<uint64_t>(k) * kMtN + w] = r;
      }
      __syncthreads();
    }
    grid.sync();
  }
}

// Segment k: blocks 1 + k L ... of the run (block 0 = the current state's
// remaining outputs, written by segment 0).  Output o of block bi >= 1 sits
// at head + (bi - 1) * 312 + o.  The segment holding output n - 1 records the
// end state in tent.
__global__ void __launch_bounds__(320) mt_seg_gen_kernel(const uint64_t* __restrict__ state,
                                                         const uint64_t* __restrict__ st, uint64_t n,
                                                         uint64_t* __restrict__ out, uint64_t* __restrict__ tent) {
  __shared__ uint64_t x[2][kMtN];
  const int t = threadIdx.x, k = blockIdx.x;
  const uint64_t pos0 = state[kMtN];
  const uint64_t head = pos0 < kMtN ? kMtN - pos0 : 0;
  if (k == 0 && t < head && t < n) out[t] = temper(state[pos0 + t]);
  if (k == 0 && n <= head) {  // nothing past the current block
    if (t < kMtN) tent[t] = state[t];
    if (t == 0) tent[kMtN] = pos0 + n;
    return;
  }
  if (t < kMtN) x[0][t] = st[static_cast<uint64_t>(k) * kMtN + t];
  __syncthreads();
  int cur = 0;
  for (int b = 0; b < kJumpL; ++b) {
    const uint64_t o0 = head + (static_cast<uint64_t>(k) * kJumpL + b) * kMtN;
    if (o0 >= n) break;
    if (b > 0) {
      const int nxt = cur ^ 1;
      if (t < kMtN - kMtM) x[nxt][t] = twist_word(x[cur][t], x[cur][t + 1], x[cur][t + kMtM]);
      __syncthreads();
      if (t >= kMtN - kMtM && t < kMtN)
        x[nxt][t] = twist_word(x[cur][t], t == kMtN - 1 ? x[nxt][0] : x[cur][t + 1], x[nxt][t - (kMtN - kMtM)]);
      __syncthreads();
      cur = nxt;
    }
    const uint64_t take = n - o0 < kMtN ? n - o0 : kMtN;
    if (t < take) out[o0 + t] = temper(x[cur][t]);
    if (o0 + take == n) {
      if (t < kMtN) tent[t] = x[cur][t];
      if (t == 0) tent[kMtN] = take;
    }
  }
}

// Output d -> draw d (no rejection assumed); a rejection raises *flag.
__global__ void draw_map_kernel(const uint64_t* __restrict__ out, uint64_t n, DrawPlan plan, int* flag) {
  for (uint64_t d = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; d < n;
       d += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = out[d];
    uint64_t base = 0;
    const uint64_t bound = plan_bound(plan, d, &base);
    if (r < (0ULL - bound) % bound)
      *flag = 1;
    else
      plan_store(plan, d, base, r % bound);
  }
}

// m draws in stream order.  Each block of 312 tempered outputs is mapped
// optimistically to consecutive draws; a block containing a rejection is
// replayed by lane 0 so exactly the reference's outputs are consumed.
// flag/tent (launch_draws): unless draw_map_kernel saw a rejection, only the
// recorded end state is installed.
__global__ void __launch_bounds__(320) mt_draw_kernel(uint64_t* state, uint64_t m, DrawPlan plan,
                                                      const int* flag, const uint64_t* tent) {
  __shared__ uint64_t x[kMtN];
  __shared__ uint64_t s_done, s_pos;
  const int t = threadIdx.x;
  if (flag && *flag == 0) {
    if (t <= kMtN) state[t] = tent[t];
    return;
  }
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

// n raw outputs of the engine `state` into out (+ the end state into tent):
// one CTA for short runs, parallel segments (jump-ahead) for long ones.
int launch_engine(MtJump& jp, int num_sms, const uint64_t* state, uint64_t n, uint64_t* out, uint64_t* tent,
                  cudaStream_t st, uint64_t* launches) {
  const char* env = getenv("SGDT_JUMP_MIN_BLOCKS");  // tests: force the segmented path
  const uint64_t min_blocks = env ? static_cast<uint64_t>(atoll(env)) : static_cast<uint64_t>(3 * kJumpL);
  const uint64_t blocks = n / kMtN;
  if (blocks < min_blocks || blocks < 2) {
    mt_gen_kernel<<<1, 320, 0, st>>>(state, n, out, tent);
    SGDT_CUDA(cudaGetLastError());
    ++*launches;
    return SGDT_OK;
  }
  if (!jp.J) {  // once per owner: J = T^kJumpL
    SGDT_CUDA(cudaMalloc(&jp.J, static_cast<size_t>(kStateBits) * kMtN * sizeof(uint64_t)));
    const int smem = kStateBits * static_cast<int>(sizeof(uint64_t));
    SGDT_CUDA(cudaFuncSetAttribute(mt_jump_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    mt_jump_build_kernel<<<kMtN, kJumpThreads, smem, st>>>(kJumpL, jp.J);
    SGDT_CUDA(cudaGetLastError());
    ++*launches;
  }
  // segments: enough to cover every output past the current block
  const uint64_t full = n + kMtN;  // upper bound on outputs past block 0
  const int ns = static_cast<int>((full + static_cast<uint64_t>(kJumpL) * kMtN - 1) / (static_cast<uint64_t>(kJumpL) * kMtN));
  if (jp.st_cap < static_cast<uint64_t>(ns)) {
    if (jp.st) cudaFree(jp.st);
    jp.st = nullptr;
    jp.st_cap = 0;
    SGDT_CUDA(cudaMalloc(&jp.st, static_cast<size_t>(ns) * kMtN * sizeof(uint64_t)));
    jp.st_cap = ns;
  }
  if (!jp.part) SGDT_CUDA(cudaMalloc(&jp.part, static_cast<size_t>(num_sms) * kMtN * sizeof(uint64_t)));
  {
    const uint64_t* a0 = state;
    const uint64_t* a1 = jp.J;
    int a2 = ns;
    uint64_t* a3 = jp.st;
    uint64_t* a4 = jp.part;
    void* args[] = {(void*)&a0, (void*)&a1, (void*)&a2, (void*)&a3, (void*)&a4};
    SGDT_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(mt_chain_kernel), dim3(num_sms),
                                          dim3(kJumpThreads), args, 0, st));
  }
  mt_seg_gen_kernel<<<ns, 320, 0, st>>>(state, jp.st, n, out, tent);
  SGDT_CUDA(cudaGetLastError());
  *launches += 2;
  return SGDT_OK;
}

// m draws of `plan` from the session engine (see the file header).
int launch_draws(Session& s, uint64_t m, const DrawPlan& plan, cudaStream_t st) {
  if (m == 0) return SGDT_OK;
  if (!s.mt_tent) {
    SGDT_CUDA(cudaMalloc(&s.mt_tent, (kMtN + 1) * sizeof(uint64_t)));
    SGDT_CUDA(cudaMalloc(&s.mt_flag, sizeof(int)));
  }
  if (s.mt_out_cap < m) {
    if (s.mt_out) cudaFree(s.mt_out);
    s.mt_out = nullptr;
    s.mt_out_cap = 0;
    SGDT_CUDA(cudaMalloc(&s.mt_out, m * sizeof(uint64_t)));
    s.mt_out_cap = m;
  }
  SGDT_CUDA(cudaMemsetAsync(s.mt_flag, 0, sizeof(int), st));
  TRY_RC(launch_engine(s.jump, s.num_sms, s.mt, m, s.mt_out, s.mt_tent, st, &s.launches));
  const uint64_t want = (m + 255) / 256;
  const unsigned grid = static_cast<unsigned>(want < static_cast<uint64_t>(s.num_sms) * 16 ? want
                                                                                            : s.num_sms * 16);
  draw_map_kernel<<<grid, 256, 0, st>>>(s.mt_out, m, plan, s.mt_flag);
  mt_draw_kernel<<<1, 320, 0, st>>>(s.mt, m, plan, s.mt_flag, s.mt_tent);
  SGDT_CUDA(cudaGetLastError());
  s.launches += 2;
  return SGDT_OK;
}

// The pre-run pool values at the positions a run reads (sgdt_pool_delta_pre).
__global__ void capture_pre_kernel(uint64_t m, const uint32_t* __restrict__ pool, const uint32_t* __restrict__ draw_j,
                                   uint32_t* __restrict__ pre_j, uint32_t* __restrict__ pre_lo) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    pre_j[i] = pool[draw_j[i]];
    pre_lo[i] = pool[i];
  }
}

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
  TRY_RC(launch_draws(s, m, plan, st));
  const unsigned blocks = static_cast<unsigned>((m + 255) / 256);
  link_kernel<<<blocks, 256, 0, st>>>(m, s.draw_j, s.head, s.stamp, s.link);
  resolve_kernel<<<blocks, 256, 0, st>>>(m, s.draw_j, nullptr, s.head, s.link, s.stamp, s.kprev, s.lprev);
  chain_kernel<<<blocks, 256, 0, st>>>(m, s.pool, nullptr, s.draw_j, s.kprev, s.lprev, s.dval, out_batch);
  if (s.capture_pre) {
    if (m > s.pool_pre_cap) {
      if (s.pool_pre) SGDT_CUDA(cudaFree(s.pool_pre));
      s.pool_pre = nullptr;
      s.pool_pre_cap = 0;
      SGDT_CUDA(cudaMalloc(&s.pool_pre, 2 * m * sizeof(uint32_t)));
      s.pool_pre_cap = m;
    }
    capture_pre_kernel<<<blocks, 256, 0, st>>>(m, s.pool, s.draw_j, s.pool_pre, s.pool_pre + m);
    ++s.launches;
  }
  write_pool_kernel<<<blocks, 256, 0, st>>>(m, s.pool, s.draw_j, s.head, s.link, s.stamp,
                                            out_batch, s.dval);
  SGDT_CUDA(cudaGetLastError());
  s.launches += 4;
  s.last_batch = out_batch;
  s.last_batch_len = m;
  ++s.sampler_runs;
  s.delta_m = m;
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
  TRY_RC(launch_draws(s, T, plan, st));
  const unsigned blocks = static_cast<unsigned>((T + 255) / 256);
  link_kernel<<<blocks, 256, 0, st>>>(T, rs.target, s.head, s.stamp, rs.link);
  resolve_kernel<<<blocks, 256, 0, st>>>(T, rs.target, rs.pos, s.head, rs.link, s.stamp, rs.kprev, rs.lprev);
  chain_kernel<<<blocks, 256, 0, st>>>(T, nullptr, rs.pos, rs.target, rs.kprev, rs.lprev, nullptr, rs.out);
  SGDT_CUDA(cudaGetLastError());
  s.launches += 3;
  return SGDT_OK;
}

}  // namespace sgdt

extern "C" int sgdt_rng_next_below(const uint64_t* mt312, uint32_t pos, const uint64_t* bounds,
                                   uint64_t n, uint64_t* out, uint64_t* mt312_out,
                                   uint32_t* pos_out) {
  using namespace sgdt;
  for (uint64_t i = 0; i < n; ++i)
    if (bounds[i] == 0) return fail(SGDT_ERR_DOMAIN, "next_below: bound must be >= 1");
  // the same three kernels as launch_draws (engine run, parallel map,
  // replay-or-install), so the test hook exercises the rejection fallback
  uint64_t *d_state = nullptr, *d_bounds = nullptr, *d_out = nullptr, *d_raw = nullptr, *d_tent = nullptr;
  int* d_flag = nullptr;
  SGDT_CUDA(cudaMalloc(&d_state, (kMtN + 1) * sizeof(uint64_t)));
  SGDT_CUDA(cudaMalloc(&d_tent, (kMtN + 1) * sizeof(uint64_t)));
  SGDT_CUDA(cudaMalloc(&d_flag, sizeof(int)));
  SGDT_CUDA(cudaMalloc(&d_bounds, (n + 1) * sizeof(uint64_t)));
  SGDT_CUDA(cudaMalloc(&d_out, (n + 1) * sizeof(uint64_t)));
  SGDT_CUDA(cudaMalloc(&d_raw, (n + 1) * sizeof(uint64_t)));
  uint64_t h_state[kMtN + 1];
  for (int i = 0; i < kMtN; ++i) h_state[i] = mt312[i];
  h_state[kMtN] = pos;
  SGDT_CUDA(cudaMemcpy(d_state, h_state, sizeof h_state, cudaMemcpyHostToDevice));
  SGDT_CUDA(cudaMemcpy(d_bounds, bounds, n * sizeof(uint64_t), cudaMemcpyHostToDevice));
  SGDT_CUDA(cudaMemset(d_flag, 0, sizeof(int)));
  DrawPlan plan{};
  plan.kind = 1;
  plan.bounds = d_bounds;
  plan.out64 = d_out;
  MtJump jp;
  uint64_t launches = 0;
  int num_sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (n > 0) {
    const int rc = launch_engine(jp, num_sms, d_state, n, d_raw, d_tent, 0, &launches);
    if (rc != SGDT_OK) return rc;
    draw_map_kernel<<<static_cast<unsigned>((n + 255) / 256), 256>>>(d_raw, n, plan, d_flag);
    mt_draw_kernel<<<1, 320>>>(d_state, n, plan, d_flag, d_tent);
  }
  SGDT_CUDA(cudaGetLastError());
  SGDT_CUDA(cudaMemcpy(out, d_out, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  SGDT_CUDA(cudaMemcpy(h_state, d_state, sizeof h_state, cudaMemcpyDeviceToHost));
  for (int i = 0; i < kMtN; ++i) mt312_out[i] = h_state[i];
  *pos_out = static_cast<uint32_t>(h_state[kMtN]);
  for (void* p : {(void*)d_state, (void*)d_bounds, (void*)d_out, (void*)d_raw, (void*)d_tent, (void*)d_flag,
                  (void*)jp.J, (void*)jp.st, (void*)jp.part})
    cudaFree(p);
  return SGDT_OK;
}
