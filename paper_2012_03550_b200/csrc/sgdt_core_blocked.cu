// sgdt_core_blocked.cu -- the core (Kruskal B^(n)) phase in column blocks:
// one kernel per (mode, block of T columns) plus a final kernel, so a rank
// exchanges one small vector per block instead of one per column.  This is
// the path of the sharded (multi-GPU) core phase and, with one rank, an
// alternative single-GPU core phase (SGDT_CORE=blocked|column).
//
// Reference: update_core_epoch (core_optimizer.cpp:112-257), Gauss-Seidel
// over the columns r_core of B^(n): V = -U + C b_rc (:225-250), sgd_step
// (:85-100).  With W_r[s] = c_{s,r} a_s the identity of sgdt_core.cu gives
//   V_rc = sum_s c_{s,rc} (xhat_s - x_s) a_s,
// xhat_s = sum_r c_{s,r} (a_s . b_r) kept current after every column.  For a
// block of columns [r0, r0+T), with xhat^0 the value at the block start and
// db_r the update of column r, expanding the in-block xhat updates gives
//   V_rc = V0_rc + sum_{r0 <= r' < rc} G_{rc,r'} db_r'
//   V0_rc     = sum_s c_{s,rc} (xhat^0_s - x_s) a_s              (J values)
//   G_{r,r'}  = sum_s c_{s,r} c_{s,r'} a_s a_s^T                 (J x J, symmetric)
// so one reduction over Psi per block feeds T exact Gauss-Seidel column
// steps.  Only the association of the sums changes: T = 1 is the column
// algorithm; for the reference's C (= G_{rc,rc}) and U this is the same
// algebra as the dense route.
//
// One step = one kernel, stream-ordered after the previous one:
//   prologue  every CTA loads B, sums the previous step's block vectors of
//             all ranks in rank order (fp64) and replays its T column steps
//             (identical in every CTA of every rank: B stays bit-identical
//             with no broadcast);
//   body      per tile of the CTA's Psi slice: the per-sample state (c_s, a_s,
//             xhat_s, x_s; computed at the first block of a mode, else loaded
//             from the global scratch and updated with the previous block's
//             db), then the V0 / G accumulation of this block;
//   epilogue  the CTA's vector goes to a global slot; the last CTA to finish
//             (ticket counter) sums the slots in CTA order and stores the
//             rank's vector into slot `rank` of every rank's exchange buffer
//             (NVLink P2P stores for peers), and writes B.
// The final step replays the last block and refreshes Q^(k) = A^(k) B^(k).
// Ranks need a barrier between steps (the sharded driver's stream barrier);
// one rank needs nothing beyond stream order.  No spin-waits anywhere.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "sgdt_internal.cuh"
#include "sgdt_qrows.cuh"

namespace sgdt {

namespace {

constexpr int kBlk = 512;        // threads per CTA
constexpr int kMaxTasks = kBlk;  // accumulation tasks per CTA (one per thread at most)
constexpr unsigned kGroup = 16;  // CTAs per first-level reduction group

struct BlockShape {  // one block of T columns of a mode with J = jn
  uint32_t T, jn, nt, ntp, pairs, kv, k;  // k = vector length
};

__host__ __device__ inline BlockShape block_shape(uint32_t T, uint32_t jn) {
  BlockShape b;
  b.T = T;
  b.jn = jn;
  b.nt = (jn + 3) / 4;
  b.ntp = b.nt * (b.nt + 1) / 2;
  b.pairs = T * (T - 1) / 2;
  b.kv = T * jn;
  b.k = b.kv + b.pairs * b.ntp * 16;
  return b;
}
__host__ __device__ inline uint32_t block_tasks(const BlockShape& b) { return b.T * b.nt + b.pairs * b.ntp; }

// index of tile (ta <= tb) in the packed upper triangle of nt x nt tiles
__device__ __forceinline__ uint32_t tile_index(uint32_t ta, uint32_t tb, uint32_t nt) {
  return ta * nt - ta * (ta - 1) / 2 + (tb - ta);
}
// G_{t,t'}[j][j'] (t > t') inside a block vector
__device__ __forceinline__ double g_at(const double* v, const BlockShape& b, uint32_t t, uint32_t tp, uint32_t j,
                                       uint32_t jp) {
  const uint32_t p = t * (t - 1) / 2 + tp;
  uint32_t ta = j >> 2, tb = jp >> 2, ia = j & 3, ib = jp & 3;
  if (ta > tb) {
    const uint32_t x = ta;
    ta = tb;
    tb = x;
    const uint32_t y = ia;
    ia = ib;
    ib = y;
  }
  return v[b.kv + (p * b.ntp + tile_index(ta, tb, b.nt)) * 16 + ia * 4 + ib];
}

// Words per sample row of the smem tile: a[js4] c[RP] w[T][js4] res, padded
// to 4 (mod 8) words (16-B aligned rows, conflict-free per-lane float4 writes).
__host__ __device__ inline uint32_t tile_stride(uint32_t js4, uint32_t RP, uint32_t T) {
  uint32_t s = js4 + RP + T * js4 + 1;
  s = (s + 3) & ~3u;
  if ((s & 7u) == 0) s += 4;
  return s;
}

struct BlockedArgs {
  Params P;
  const uint32_t* rec_idx;  // entry-order copy
  const float* rec_val;
  uint64_t nnz;
  const uint32_t* batch;  // Psi (m), or one per mode (order x m)
  int per_mode;
  uint64_t m;
  uint64_t lo, hi;  // this rank's slice of Psi (partition_even(m, world)[rank])
  double lr, reg, inv_m;
  int* flag;
  // this step's block (n < 0: the final step)
  int n;
  uint32_t r0, T;
  int first;       // r0 == 0: compute the per-sample state
  int keep_state;  // more blocks of mode n follow: keep the state in the global scratch
  // the previous step's block, replayed in the prologue (pn < 0: none)
  int pn;
  uint32_t pr0, pT;
  int fold;  // the previous block is of mode n: fold its db into xhat
  // exchange: this rank's buffer holds 2 slots x world x kstride fp64
  const double* xin;    // slot read: world x kstride
  double* xout[kMaxPeers + 1];  // slot written, per rank (rank `rank` at this rank's offset)
  int world, rank;
  uint32_t kstride;
  // scratch
  float* sa;    // (hi-lo) x js4   a_s
  float* sc;    // (hi-lo) x RP    c_s
  float* sxh;   // (hi-lo)
  float* sx;    // (hi-lo)
  uint32_t js4;
  double* part;  // grid x kstride
  unsigned* ticket;
  uint32_t st;   // samples per smem tile
  int q_mask;    // final step: bit k = refresh Q^(k) here (the other modes: tensor-core refresh)
};

// Replay the T column steps of a block from its summed vector v (smem):
// warp w owns j = w, w + nwarps, ...; lanes split the sum over (t', j') with a
// fixed stride and a fixed butterfly, so every CTA forms identical values.
__device__ void replay_block(const BlockedArgs& a, float* bsn, const double* v, const BlockShape& b, uint32_t r0,
                             float* dbv) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t RP = a.P.RP;
  for (uint32_t t = 0; t < b.T; ++t) {
    const uint32_t rc = r0 + t;
    for (uint32_t j = warp; j < b.jn; j += nw) {
      double V = 0.0;
      for (uint32_t q = lane; q < t * b.jn; q += 32) {
        const uint32_t tp = q / b.jn, jp = q - tp * b.jn;
        V = fma(g_at(v, b, t, tp, j, jp), static_cast<double>(dbv[tp * b.jn + jp]), V);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) V += __shfl_xor_sync(0xffffffffu, V, o);
      if (lane == 0) {
        V += v[t * b.jn + j];
        const float bold = bsn[j * RP + rc];
        double w = static_cast<double>(bold);
        int bad = (!isfinite(w) ? 1 : 0) | (!isfinite(V) ? 2 : 0);
        w -= a.lr * (V * a.inv_m + a.reg * w);
        const float bnew = static_cast<float>(w);
        bad |= !isfinite(bnew) ? 4 : 0;
        if (bad && blockIdx.x == 0) atomicOr(a.flag, bad);
        dbv[t * b.jn + j] = bnew - bold;
        bsn[j * RP + rc] = bnew;
      }
    }
    __syncthreads();
  }
}

template <int RP>
__global__ void __launch_bounds__(kBlk) core_block_kernel(BlockedArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  // ---- smem: B copy | db of the replayed block | block vector (fp64) | tile
  float* bs = reinterpret_cast<float*>(smem_raw);
  uint32_t bso[kMaxOrder];
  uint32_t off = 0;
  uint32_t js = 0;
  for (int k = 0; k < a.P.order; ++k) {
    bso[k] = off;
    off += a.P.J[k] * RP;
    js = a.P.J[k] > js ? a.P.J[k] : js;
  }
  float* dbv = bs + off;  // pT x js
  const uint32_t dbn = a.P.R * js;
  double* vec = reinterpret_cast<double*>(dbv + ((dbn + 3) & ~3u));  // kstride
  float* tile = reinterpret_cast<float*>(vec + a.kstride);

  for (int k = 0; k < a.P.order; ++k)
    for (uint32_t i = tid; i < a.P.J[k] * RP; i += blockDim.x) {
      const uint32_t j = i / RP, r = i % RP;
      bs[bso[k] + i] = r < a.P.R ? a.P.B[k][j * a.P.R + r] : 0.f;
    }

  // ---- prologue: replay the previous block from the rank-ordered sum
  if (a.pn >= 0) {
    const BlockShape pb = block_shape(a.pT, a.P.J[a.pn]);
    for (uint32_t k = tid; k < pb.k; k += blockDim.x) {
      double acc = 0.0;
      for (int r = 0; r < a.world; ++r) acc += __ldcg(a.xin + static_cast<uint64_t>(r) * a.kstride + k);
      vec[k] = acc;
    }
    __syncthreads();
    replay_block(a, bs + bso[a.pn], vec, pb, a.pr0, dbv);
  } else {
    __syncthreads();
  }

  if (a.n >= 0) {
    const int n = a.n;
    const uint32_t jn = a.P.J[n], js4 = a.js4;
    const BlockShape b = block_shape(a.T, jn);
    const uint32_t ntasks = block_tasks(b);
    const uint32_t groups = ntasks >= blockDim.x ? 1u : blockDim.x / ntasks;
    const uint32_t task = tid % ntasks, grp = tid / ntasks;
    const bool active = grp < groups;
    // task -> (kind, indices)
    bool is_v = task < b.T * b.nt;
    uint32_t t = 0, tp = 0, ta = 0, tb = 0;
    if (is_v) {
      t = task / b.nt;
      ta = task - t * b.nt;
    } else {
      const uint32_t q = task - b.T * b.nt;
      const uint32_t p = q / b.ntp;
      uint32_t ti = q - p * b.ntp;
      // pair p -> (t > tp)
      t = 1;
      while ((t + 1) * t / 2 <= p) ++t;
      tp = p - t * (t - 1) / 2;
      // packed tile ti -> (ta <= tb)
      ta = 0;
      while (ti >= b.nt - ta) {
        ti -= b.nt - ta;
        ++ta;
      }
      tb = ta + ti;
    }
    const uint32_t rc = a.r0 + t, rcp = a.r0 + tp;
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.f;

    // this CTA's share of the rank's slice
    const uint64_t len = a.hi - a.lo;
    const uint64_t base = len / gridDim.x, rem = len % gridDim.x;
    const uint64_t c0 = blockIdx.x * base + (blockIdx.x < rem ? blockIdx.x : rem);
    const uint64_t c1 = c0 + base + (blockIdx.x < rem ? 1 : 0);
    const uint32_t* batch = a.batch + (a.per_mode ? static_cast<uint64_t>(n) * a.m : 0);
    // tile row: a[js4] c[RP] w[T][js4] res pad; w_t = c_{s,r0+t} a_s and
    // res = xhat_s - x_s are all the accumulation reads.  The stride is 4 mod
    // 8 words so the per-thread float4 row writes are bank-conflict free.
    const uint32_t srow = tile_stride(js4, RP, a.T);
    const uint32_t wo = js4 + RP, ro = wo + a.T * js4;
    const float* bsn = bs + bso[n];

    for (uint64_t t0 = c0; t0 < c1; t0 += a.st) {
      const uint32_t cnt = static_cast<uint32_t>(c1 - t0 < a.st ? c1 - t0 : a.st);
      // ---- per-sample state of this tile
      for (uint32_t ls = tid; ls < cnt; ls += blockDim.x) {
        const uint64_t li = t0 + ls;  // index inside the rank's slice
        float* row = tile + static_cast<uint64_t>(ls) * srow;
        float* ra = row;
        float* rcv = row + js4;
        float xh, xv;
        if (a.first) {
          const uint32_t e = batch[a.lo + li];
          float c[RP];
#pragma unroll
          for (int r = 0; r < RP; ++r) c[r] = 1.f;
          for (int k = 0; k < a.P.order; ++k) {
            if (k == n) continue;
            const uint32_t ik = a.rec_idx[static_cast<uint64_t>(k) * a.nnz + e];
            const float* arow = a.P.A[k] + static_cast<uint64_t>(ik) * a.P.J[k];
            float d[RP];
#pragma unroll
            for (int r = 0; r < RP; ++r) d[r] = 0.f;
            for (uint32_t j = 0; j < a.P.J[k]; ++j) {
              const float av = arow[j];
#pragma unroll
              for (int r = 0; r < RP; ++r) d[r] = fmaf(av, bs[bso[k] + j * RP + r], d[r]);
            }
#pragma unroll
            for (int r = 0; r < RP; ++r) c[r] *= d[r];
          }
          const uint32_t in_ = a.rec_idx[static_cast<uint64_t>(n) * a.nnz + e];
          const float* arow = a.P.A[n] + static_cast<uint64_t>(in_) * jn;
          float p[RP];
#pragma unroll
          for (int r = 0; r < RP; ++r) p[r] = 0.f;
          for (uint32_t j = 0; j < jn; ++j) {
            const float av = arow[j];
            ra[j] = av;
#pragma unroll
            for (int r = 0; r < RP; ++r) p[r] = fmaf(av, bsn[j * RP + r], p[r]);
          }
          for (uint32_t j = jn; j < js4; ++j) ra[j] = 0.f;
          xh = 0.f;
#pragma unroll
          for (int r = 0; r < RP; ++r) {
            xh = fmaf(c[r], p[r], xh);
            rcv[r] = c[r];
          }
          xv = a.rec_val[e];
          if (a.keep_state) {
            float4* ga = reinterpret_cast<float4*>(a.sa + li * js4);
            for (uint32_t j = 0; j < js4; j += 4) ga[j / 4] = *reinterpret_cast<const float4*>(ra + j);
            float4* gc = reinterpret_cast<float4*>(a.sc + li * RP);
#pragma unroll
            for (int r = 0; r < RP; r += 4) gc[r / 4] = make_float4(c[r], c[r + 1], c[r + 2], c[r + 3]);
            a.sx[li] = xv;
          }
        } else {
          const float4* ga = reinterpret_cast<const float4*>(a.sa + li * js4);
          for (uint32_t j = 0; j < js4; j += 4) *reinterpret_cast<float4*>(ra + j) = ga[j / 4];
          const float4* gc = reinterpret_cast<const float4*>(a.sc + li * RP);
#pragma unroll
          for (int r = 0; r < RP; r += 4) *reinterpret_cast<float4*>(rcv + r) = gc[r / 4];
          xh = a.sxh[li];
          xv = a.sx[li];
          if (a.fold) {  // xhat += sum_{t'} c_{s,pr0+t'} (a_s . db_t')
            for (uint32_t q = 0; q < a.pT; ++q) {
              float d = 0.f;
              for (uint32_t j = 0; j < jn; ++j) d = fmaf(ra[j], dbv[q * jn + j], d);
              xh = fmaf(rcv[a.pr0 + q], d, xh);
            }
          }
        }
        if (a.keep_state) a.sxh[li] = xh;
        for (uint32_t q = 0; q < a.T; ++q) {
          const float cq = rcv[a.r0 + q];
          float* w = row + wo + q * js4;
          for (uint32_t j = 0; j < js4; j += 4) {
            const float4 av = *reinterpret_cast<const float4*>(ra + j);
            *reinterpret_cast<float4*>(w + j) = make_float4(cq * av.x, cq * av.y, cq * av.z, cq * av.w);
          }
        }
        row[ro] = xh - xv;
      }
      __syncthreads();
      // ---- accumulate this tile: V0 (4 outputs) or a 4 x 4 tile of G
      if (active) {
        if (is_v) {
          const uint32_t ox = wo + t * js4 + 4 * ta;
#pragma unroll 2
          for (uint32_t ls = grp; ls < cnt; ls += groups) {
            const float* row = tile + static_cast<uint64_t>(ls) * srow;
            const float r = row[ro];
            const float4 w4 = *reinterpret_cast<const float4*>(row + ox);
            acc[0] = fmaf(r, w4.x, acc[0]);
            acc[1] = fmaf(r, w4.y, acc[1]);
            acc[2] = fmaf(r, w4.z, acc[2]);
            acc[3] = fmaf(r, w4.w, acc[3]);
          }
        } else {
          const uint32_t ox = wo + t * js4 + 4 * ta, oy = wo + tp * js4 + 4 * tb;
#pragma unroll 2
          for (uint32_t ls = grp; ls < cnt; ls += groups) {
            const float* row = tile + static_cast<uint64_t>(ls) * srow;
            const float4 x4 = *reinterpret_cast<const float4*>(row + ox);
            const float4 y4 = *reinterpret_cast<const float4*>(row + oy);
            const float xx[4] = {x4.x, x4.y, x4.z, x4.w};
            const float yy[4] = {y4.x, y4.y, y4.z, y4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int k = 0; k < 4; ++k) acc[i * 4 + k] = fmaf(xx[i], yy[k], acc[i * 4 + k]);
          }
        }
      }
      __syncthreads();
    }

    // ---- CTA vector: the groups' partials summed in group order (fp64)
    for (uint32_t g = 0; g < groups; ++g) {
      if (active && grp == g) {
        if (is_v) {
          for (int i = 0; i < 4; ++i) {
            const uint32_t j = 4 * ta + i;
            if (j < jn) {
              double& d = vec[t * jn + j];
              d = (g == 0 ? 0.0 : d) + static_cast<double>(acc[i]);
            }
          }
        } else {
          const uint32_t p = t * (t - 1) / 2 + tp;
          double* d = vec + b.kv + (p * b.ntp + tile_index(ta, tb, b.nt)) * 16;
          for (int i = 0; i < 16; ++i) d[i] = (g == 0 ? 0.0 : d[i]) + static_cast<double>(acc[i]);
        }
      }
      __syncthreads();
    }
    double* mine = a.part + static_cast<uint64_t>(blockIdx.x) * a.kstride;
    for (uint32_t k = tid; k < b.k; k += blockDim.x) mine[k] = vec[k];
  }

  // ---- final step: Q^(k) = A^(k) B^(k) for every mode (from the smem B)
  if (a.n < 0) {
    const int nwarps = blockDim.x >> 5, warp = tid >> 5, lane = tid & 31;
    float* stage = tile + warp * kQStage;
    const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * nwarps + warp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * nwarps;
    for (int k = 0; k < a.P.order; ++k)
      if (a.q_mask >> k & 1)
        q_rows_tiled<RP>(a.P.A[k], a.P.Q[k], a.P.J[k], bs + bso[k], a.P.dims[k], gw, nw, stage, lane);
  }

  // ---- two-level ticket reduction (no CTA waits): the last CTA of each group
  // of kGroup CTAs sums its group's vectors (CTA order) into a group slot; the
  // last group reducer sums the group slots (group order) -> the rank vector
  // -> slot `rank` of every rank's exchange buffer; it also writes B.
  __shared__ unsigned s_last;
  const unsigned ngroups = (gridDim.x + kGroup - 1) / kGroup;
  const unsigned grp_id = blockIdx.x / kGroup;
  const unsigned g0 = grp_id * kGroup, g1 = min(gridDim.x, g0 + kGroup);
  const uint32_t K = a.n >= 0 ? block_shape(a.T, a.P.J[a.n]).k : 0;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(a.ticket + 1 + grp_id, 1u) == g1 - g0 - 1 ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  {
    double* gslot = a.part + static_cast<uint64_t>(gridDim.x + grp_id) * a.kstride;
    for (uint32_t k = tid; k < K; k += blockDim.x) {
      double acc = 0.0;
#pragma unroll 4
      for (unsigned cta = g0; cta < g1; ++cta) acc += __ldcg(a.part + static_cast<uint64_t>(cta) * a.kstride + k);
      gslot[k] = acc;
    }
    if (tid == 0) a.ticket[1 + grp_id] = 0;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(a.ticket, 1u) == ngroups - 1 ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (uint32_t k = tid; k < K; k += blockDim.x) {
    double acc = 0.0;
#pragma unroll 4
    for (unsigned g = 0; g < ngroups; ++g) acc += __ldcg(a.part + static_cast<uint64_t>(gridDim.x + g) * a.kstride + k);
    for (int r = 0; r < a.world; ++r) a.xout[r][k] = acc;
  }
  if (a.pn >= 0) {
    const int k = a.pn;
    for (uint32_t i = tid; i < a.P.J[k] * a.P.R; i += blockDim.x)
      a.P.B[k][i] = bs[bso[k] + (i / a.P.R) * RP + (i % a.P.R)];
  }
  if (tid == 0) *a.ticket = 0;
}

template <int RP>
size_t blocked_smem(const Session& s, uint32_t kstride, uint32_t st, uint32_t js4, uint32_t T) {
  size_t f = 0;
  uint32_t js = 0;
  for (int k = 0; k < s.order; ++k) {
    f += s.J[k] * RP;
    js = std::max(js, s.J[k]);
  }
  const uint32_t dbn = s.R * js;
  f += (dbn + 3) & ~3u;
  size_t bytes = f * sizeof(float) + static_cast<size_t>(kstride) * sizeof(double);
  const size_t tile = static_cast<size_t>(st) * tile_stride(js4, RP, T) * sizeof(float);
  const size_t qst = static_cast<size_t>(kBlk / 32) * kQStage * sizeof(float);
  return bytes + std::max(tile, qst);
}

template <int RP>
int blocked_launch_rp(Session& s, BlockedArgs& a, int grid, size_t smem) {
  auto kern = core_block_kernel<RP>;
  if (smem > 48 * 1024)
    SGDT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kern<<<grid, kBlk, smem, s.stream>>>(a);
  SGDT_CUDA(cudaGetLastError());
  ++s.launches;
  return SGDT_OK;
}

size_t smem_for(const Session& s, uint32_t kstride, uint32_t st, uint32_t js4, uint32_t T) {
  switch (s.RP) {
    case 4: return blocked_smem<4>(s, kstride, st, js4, T);
    case 8: return blocked_smem<8>(s, kstride, st, js4, T);
    case 12: return blocked_smem<12>(s, kstride, st, js4, T);
    case 16: return blocked_smem<16>(s, kstride, st, js4, T);
    case 20: return blocked_smem<20>(s, kstride, st, js4, T);
    case 24: return blocked_smem<24>(s, kstride, st, js4, T);
    case 28: return blocked_smem<28>(s, kstride, st, js4, T);
    case 32: return blocked_smem<32>(s, kstride, st, js4, T);
    default: return 0;
  }
}

}  // namespace

// Column-block width of the blocked core phase.  A block costs a kernel step
// (and, sharded, an exchange); its accumulation costs ~T^2 J^2 / 4 FMAs per
// sample.  T is the largest width whose task count fits one CTA and whose
// modelled time (step overhead + accumulation) is not worse than a narrower
// one; SGDT_CORE_T overrides.
uint32_t core_block_width(const Session& s, uint64_t m_local, int grid, double step_us, uint32_t requested) {
  uint32_t jmax = 0;
  for (int k = 0; k < s.order; ++k) jmax = std::max(jmax, s.J[k]);
  if (const char* e = std::getenv("SGDT_CORE_T")) {
    const int t = std::atoi(e);
    if (t >= 1) requested = static_cast<uint32_t>(t);
  }
  if (requested >= 1) {
    uint32_t T = std::min<uint32_t>(requested, s.R);
    while (T > 1 && block_tasks(block_shape(T, jmax)) > static_cast<uint32_t>(kMaxTasks)) --T;
    return T;
  }
  const double per_cta = static_cast<double>(m_local) / std::max(1, grid);
  double best = 1e300;
  uint32_t bestT = 1;
  for (uint32_t T = 1; T <= s.R; ++T) {
    const BlockShape b = block_shape(T, jmax);
    const uint32_t tasks = block_tasks(b);
    if (tasks > static_cast<uint32_t>(kMaxTasks)) break;
    const uint32_t nblk = (s.R + T - 1) / T;
    // per block: the step overhead (launch + tail; an exchange when
    // sharded), and a sweep of ~24 instructions per (sample, task) issued
    // over 4 x 32 lanes at ~1.9 GHz
    const double sweep_us = per_cta * 24.0 * tasks / 128.0 / 1.9e3;
    const double cost = nblk * (step_us + sweep_us);
    if (cost < best * 0.98) {
      best = cost;
      bestT = T;
    }
  }
  return bestT;
}

// The exchange-vector stride that fits every block width a plan may pick.
uint32_t core_block_max_kstride(const Session& s) {
  uint32_t jmax = 0, k = 2;
  for (int n = 0; n < s.order; ++n) jmax = std::max(jmax, s.J[n]);
  for (uint32_t T = 1; T <= s.R; ++T) {
    if (block_tasks(block_shape(T, jmax)) > static_cast<uint32_t>(kMaxTasks)) break;
    k = std::max(k, core_block_kstride(s, T));
  }
  return k;
}

uint32_t core_block_kstride(const Session& s, uint32_t T) {
  uint32_t k = 0;
  for (int n = 0; n < s.order; ++n) k = std::max(k, block_shape(T, s.J[n]).k);
  return (k + 1) & ~1u;
}

// One step of the blocked core plan (sgdt_internal.cuh CorePlan).  Step k < S-1
// accumulates block k; step k > 0 first replays block k-1; the last step
// (k = S-1) replays the last block and refreshes Q.
int launch_core_block_step(Session& s, uint32_t k) {
  CorePlan& pl = s.cplan;
  if (!pl.valid || k >= pl.steps) return fail(SGDT_ERR_CONFIG, "core step out of plan");
  BlockedArgs a{};
  a.P = s.P;
  a.rec_idx = s.train_rec.idx;
  a.rec_val = s.train_rec.val;
  a.nnz = s.nnz;
  a.batch = pl.batch;
  a.per_mode = pl.per_mode;
  a.m = pl.m;
  a.lo = pl.lo;
  a.hi = pl.hi;
  a.lr = pl.lr;
  a.reg = pl.reg;
  a.inv_m = 1.0 / static_cast<double>(pl.m);
  a.flag = s.flag;
  const uint32_t nb = (s.R + pl.T - 1) / pl.T;  // blocks per mode
  auto blk = [&](uint32_t i, int* n, uint32_t* r0, uint32_t* T) {
    *n = static_cast<int>(i / nb);
    *r0 = (i % nb) * pl.T;
    *T = std::min(pl.T, s.R - *r0);
  };
  if (k + 1 < pl.steps) {
    blk(k, &a.n, &a.r0, &a.T);
    a.first = a.r0 == 0;
    a.keep_state = a.r0 + a.T < s.R;
  } else {
    a.n = -1;
  }
  a.pn = -1;
  if (k > 0) {
    blk(k - 1, &a.pn, &a.pr0, &a.pT);
    a.fold = a.n >= 0 && a.pn == a.n;
  }
  a.world = pl.world;
  a.rank = pl.rank;
  a.kstride = pl.kstride;
  const uint64_t slot_elems = static_cast<uint64_t>(pl.world) * pl.kstride;
  a.xin = s.core_x + static_cast<uint64_t>((k + 1) & 1) * slot_elems;  // written by step k-1
  for (int r = 0; r < pl.world; ++r) {
    double* base = pl.world == 1 ? s.core_x : s.core_peer_x[r];
    if (!base) return fail(SGDT_ERR_CONFIG, "sharded core: peers not set (sgdt_set_peers)");
    a.xout[r] = base + static_cast<uint64_t>(k & 1) * slot_elems + static_cast<uint64_t>(pl.rank) * pl.kstride;
  }
  a.sa = s.cb_a;
  a.sc = s.cb_c;
  a.sxh = s.cb_xh;
  a.sx = s.cb_x;
  a.js4 = pl.js4;
  a.part = s.core_part;
  a.ticket = s.core_ticket;
  a.st = pl.st;
  // final step: wide modes with many rows are refreshed by the tensor-core kernel
  // after this one (it reads the B this step's last CTA writes), as in launch_core
  int tc_modes = 0;
  if (a.n < 0)
    for (int q = 0; q < s.order; ++q)
      if (q_refresh_tc_eligible(s, q)) tc_modes |= 1 << q;
  a.q_mask = ((1 << s.order) - 1) & ~tc_modes;
  int rc = SGDT_ERR_CONFIG;
  switch (s.RP) {
#define BL(RP) \
  case RP: rc = blocked_launch_rp<RP>(s, a, pl.grid, pl.smem); break;
    BL(4) BL(8) BL(12) BL(16) BL(20) BL(24) BL(28) BL(32)
#undef BL
    default: return fail(SGDT_ERR_CONFIG, "unsupported R_core");
  }
  if (rc != SGDT_OK) return rc;
  for (int q = 0; q < s.order; ++q)
    if (tc_modes >> q & 1)
      if (int r2 = launch_q_refresh_tc(s, q)) return r2;
  return SGDT_OK;
}

// Fill the launch geometry of a plan whose T, m, lo, hi are set.
int plan_core_geometry(Session& s, CorePlan& pl) {
  uint32_t js = 0;
  for (int k = 0; k < s.order; ++k) js = std::max(js, s.J[k]);
  pl.js4 = (js + 3) & ~3u;
  pl.kstride = core_block_kstride(s, pl.T);
  if (pl.kstride > s.core_x_stride) return fail(SGDT_ERR_INTERNAL, "core exchange buffer too small");
  pl.steps = static_cast<uint32_t>(s.order) * ((s.R + pl.T - 1) / pl.T) + 1;
  const uint64_t len = pl.hi - pl.lo;
  uint64_t want = (len + 255) / 256;
  uint64_t rows = 0;
  for (int k = 0; k < s.order; ++k) rows += s.dims[k];
  const uint64_t qwant = rows / (kBlk * 4);  // the final step's Q refresh
  want = std::max<uint64_t>(std::max<uint64_t>(want, qwant), 1);
  pl.grid = static_cast<int>(std::min<uint64_t>(want, static_cast<uint64_t>(s.num_sms)));
  if (const char* e = std::getenv("SGDT_CORE_GRID")) {  // diagnostics (A/B runs)
    const int g = std::atoi(e);
    if (g >= 1 && g <= s.num_sms) pl.grid = g;
  }
  for (uint32_t st : {512u, 256u, 128u, 64u}) {
    const size_t smem = smem_for(s, pl.kstride, st, pl.js4, pl.T);
    if (smem && smem <= 220 * 1024) {
      pl.st = st;
      pl.smem = smem;
      return SGDT_OK;
    }
  }
  return fail(SGDT_ERR_CONFIG, "blocked core: shared memory does not fit");
}

}  // namespace sgdt
