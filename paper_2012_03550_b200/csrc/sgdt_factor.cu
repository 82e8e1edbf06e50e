// sgdt_factor.cu -- K5: the factor (A^(n)) phase, one mode per launch.
//
// Reference: update_factor_epoch (factor_optimizer.cpp:101-273) -> step_row
// (:90-97) -> grad_a_row (:34-54) -> e_column (model.cpp:148-155) ->
// kron_row_excluding (model.cpp:124-146).  Per non-empty row i of mode n:
//   F = sum_{e in bucket(n,i)} (a . e_e - x_e) e_e,   a -= lr (F/|bucket| + reg a)
// with e_e = Ghat^(n) (kron_{k != n} a^(k)_{i_k}).  Because the core is
// Kruskal, e_e = B^(n) c_e with c_{e,r} = prod_{k != n} Q^(k)[i_k, r] and
// Q^(k) = A^(k) B^(k), and a . e_e = Q^(n)[i, :] . c_e, so
//   F = B^(n) g,   g = sum_e (p_e - x_e) c_e   (an R-vector per row).
// Per (entry, mode) unit the kernel streams one record of the mode-sorted
// copy, gathers N-1 Q rows and accumulates R values; the J x R contraction
// and the update happen once per row.  Only association changes versus the
// reference.
//
// Work decomposition: the mode-sorted entries are cut once (at session
// creation) into chunks of <= chunk_size entries holding whole rows, and rows
// longer than a chunk into pieces.  One warp streams one chunk, 32 entries
// per step (one entry per lane).  A window inside one open row accumulates
// per lane in fp32 (a chunk holds <= chunk_size entries, so <= chunk_size/32
// terms per lane); a window that crosses rows runs a segmented shuffle scan
// and every completed row is finalised in fp32 by the warp (F = B g, SGD
// step, Q^(n) row rewrite).  Pieces of split rows are written as fp64 and
// summed in fp64, in piece order, by factor_split_kernel.  No atomics on parameters, fixed
// association everywhere -> run-to-run bit identical.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "sgdt_internal.cuh"

namespace sgdt {

namespace {

constexpr unsigned kFull = 0xffffffffu;

struct FactorArgs {
  Params P;
  int n;
  const uint32_t* keys;                  // mode-n coordinates of the mode-n copy
  const float* val;                      // nnz
  const uint32_t* oidx[kMaxOrder - 1];   // other modes' coordinates (mode-n copy)
  const float* oq[kMaxOrder - 1];        // other modes' Q tables
  uint32_t orows[kMaxOrder - 1];         // their row counts
  uint64_t nnz;
  const uint32_t* row_ptr;
  const Chunk* chunks;
  uint32_t n_chunks;
  const SplitRow* splits;
  uint32_t n_splits;
  uint32_t n_big_splits;  // splits[0, n_big_splits): one CTA each; the rest one warp each
  double* piece;   // n_pieces x RP
  double* xport;   // 2 x RP: summed pieces of rows cut by this rank's slice
  uint64_t qbase;  // row_ptr value of the copy's first record (shard slice start)
  double lr, reg;
  int* flag;
  const PeerTable* peers;  // null: single device; else the peers' A^(n)/Q^(n) (stores ride along)
};

// Streamed record loads: read once, never reused -> keep them out of L1,
// which is reserved for the Q-row gathers that live on its hits.
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_stream(const float* p) {
  float v;
  asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

// B^(n) lives in shared memory with row stride RP + 1 (odd), so the
// lane-per-j pass (F_j = B[j,:] . g) and the lane-per-r pass (q_r = a . B[:,r])
// both read it without bank conflicts.  Rows are zero padded up to a multiple
// of 4 so vectorised broadcasts may run past J.
template <int RP>
__host__ __device__ constexpr int bstride() {
  return RP <= 12 ? RP : RP + 1;
}
constexpr int kWarpScratch = 96;  // floats per warp: a row (<= 64) + g (<= 32)

template <int RP>
__device__ __forceinline__ void load_bsn(const FactorArgs& a, float* bsn) {
  const uint32_t jn = a.P.J[a.n], j4 = (jn + 3) & ~3u;
  for (uint32_t i = threadIdx.x; i < j4 * bstride<RP>(); i += blockDim.x) {
    const uint32_t j = i / bstride<RP>(), r = i % bstride<RP>();
    bsn[i] = j < jn && r < a.P.R ? a.P.B[a.n][j * a.P.R + r] : 0.f;
  }
}

// What a row update needs, small enough to pass by value to the out-of-line
// finaliser (keeps the finaliser's registers out of the streaming loop).
struct RowUpdate {
  float* A;                 // A^(n)
  float* Q;                 // Q^(n)
  const uint32_t* row_ptr;  // mode-n row offsets
  const float* bsn;         // B^(n) in shared memory, J x bstride
  uint32_t jn;
  float lr, reg;
  int* flag;
  const PeerTable* peers;
};

// F = B^(n) g; a -= lr (F/cnt + reg a); Q^(n)[row] = a B^(n).  One lane, fp32
// (the parameters are fp32 on the device and F is an R-term dot product of
// an fp32 row sum).  Two passes keep only g live across the J loop.
template <int RP>
__device__ __noinline__ void finalize_row_impl(RowUpdate u, uint32_t row, const float* g) {
  const uint32_t cnt = u.row_ptr[row + 1] - u.row_ptr[row];
  const float inv = 1.0f / static_cast<float>(cnt);
  float* arow = u.A + static_cast<uint64_t>(row) * u.jn;
  float gr[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) gr[r] = g[r];
  int bad = 0;
  for (uint32_t j = 0; j < u.jn; ++j) {
    float F = 0.f;
#pragma unroll
    for (int r = 0; r < RP; ++r) F = fmaf(u.bsn[j * bstride<RP>() + r], gr[r], F);
    const float w = arow[j];
    bad |= !isfinite(w) || !isfinite(F);
    const float wn = w - u.lr * fmaf(F, inv, u.reg * w);
    bad |= !isfinite(wn);
    arow[j] = wn;
    if (u.peers)
      for (int p = 0; p < u.peers->n; ++p) u.peers->A[p][static_cast<uint64_t>(row) * u.jn + j] = wn;
  }
  float4* dst = reinterpret_cast<float4*>(u.Q + static_cast<uint64_t>(row) * RP);
#pragma unroll 1
  for (int s = 0; s < RP / 4; ++s) {
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t j = 0; j < u.jn; ++j) {
      const float wf = arow[j];
      const float* b = u.bsn + j * bstride<RP>() + 4 * s;
      q.x = fmaf(wf, b[0], q.x);
      q.y = fmaf(wf, b[1], q.y);
      q.z = fmaf(wf, b[2], q.z);
      q.w = fmaf(wf, b[3], q.w);
    }
    dst[s] = q;
    if (u.peers)
      for (int p = 0; p < u.peers->n; ++p)
        reinterpret_cast<float4*>(u.peers->Q[p] + static_cast<uint64_t>(row) * RP)[s] = q;
  }
  if (bad) atomicOr(u.flag, 8);
}

__device__ __forceinline__ RowUpdate row_update(const FactorArgs& a, const float* bsn) {
  return RowUpdate{a.P.A[a.n], a.P.Q[a.n], a.row_ptr, bsn, a.P.J[a.n], static_cast<float>(a.lr),
                   static_cast<float>(a.reg), a.flag, a.peers};
}

template <int RP, typename T>
__device__ __forceinline__ void finalize_row(const FactorArgs& a, const float* bsn, uint32_t row,
                                             const T (&g)[RP]) {
  float gf[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) gf[r] = static_cast<float>(g[r]);
  finalize_row_impl<RP>(row_update(a, bsn), row, gf);
}

// The same row update done by the whole warp, g (RP floats) in the warp's
// shared scratch: lane j updates a_j, the new row goes through the scratch
// (one store, broadcast reads) and lane r rebuilds Q^(n)[row][r].  All shared
// reads are conflict-free or broadcast.
template <int RP, typename GetG>
__device__ __forceinline__ void finalize_row_warp_core(const FactorArgs& a, const float* bsn, uint32_t row,
                                                       GetG get_g, uint32_t lane, float* wsc) {
  const uint32_t jn = a.P.J[a.n];
  const uint32_t cnt = a.row_ptr[row + 1] - a.row_ptr[row];
  const float inv = 1.0f / static_cast<float>(cnt);
  const float lr = static_cast<float>(a.lr), reg = static_cast<float>(a.reg);
  float* arow = a.P.A[a.n] + static_cast<uint64_t>(row) * jn;
  int bad = 0;
  float q = 0.f;
  for (uint32_t j0 = 0; j0 < jn; j0 += 32) {
    const uint32_t j = j0 + lane;
    float wn = 0.f;
    if (j < jn) {
      float F = 0.f;
      const float* b = bsn + j * bstride<RP>();
#pragma unroll
      for (int r = 0; r < RP; r += 4) {
        const float4 g4 = get_g(r / 4);
        F = fmaf(b[r], g4.x, F);
        F = fmaf(b[r + 1], g4.y, F);
        F = fmaf(b[r + 2], g4.z, F);
        F = fmaf(b[r + 3], g4.w, F);
      }
      const float w = arow[j];
      wn = w - lr * fmaf(F, inv, reg * w);
      bad |= !isfinite(w) || !isfinite(F) || !isfinite(wn);
      arow[j] = wn;
      if (a.peers)
        for (int p = 0; p < a.peers->n; ++p) a.peers->A[p][static_cast<uint64_t>(row) * jn + j] = wn;
    }
    if constexpr (RP <= 12) {  // narrow rows: J shuffles are cheaper than the scratch round trip
      const uint32_t jend = jn - j0 < 32 ? jn - j0 : 32;
      for (uint32_t t = 0; t < jend; ++t) {
        const float aj = __shfl_sync(0xffffffffu, wn, t);
        if (lane < RP) q = fmaf(aj, bsn[(j0 + t) * bstride<RP>() + lane], q);
      }
    } else {
      wsc[j] = wn;  // zero past jn
    }
  }
  if constexpr (RP <= 12) {
    if (lane < RP) {
      a.P.Q[a.n][static_cast<uint64_t>(row) * RP + lane] = q;
      if (a.peers)
        for (int p = 0; p < a.peers->n; ++p) a.peers->Q[p][static_cast<uint64_t>(row) * RP + lane] = q;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flag, 8);
    return;
  }
  __syncwarp();
  if (lane < RP) {
    const float4* a4 = reinterpret_cast<const float4*>(wsc);
    for (uint32_t t = 0; t < jn; t += 4) {
      const float4 w4 = a4[t / 4];
      const float* b = bsn + t * bstride<RP>() + lane;
      q = fmaf(w4.x, b[0], q);
      q = fmaf(w4.y, b[bstride<RP>()], q);
      q = fmaf(w4.z, b[2 * bstride<RP>()], q);
      q = fmaf(w4.w, b[3 * bstride<RP>()], q);
    }
    a.P.Q[a.n][static_cast<uint64_t>(row) * RP + lane] = q;
    if (a.peers)
      for (int p = 0; p < a.peers->n; ++p) a.peers->Q[p][static_cast<uint64_t>(row) * RP + lane] = q;
  }
  __syncwarp();
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flag, 8);
}

// g (RP floats) in the warp's shared scratch: broadcast reads.
template <int RP>
__device__ __forceinline__ void finalize_row_warp_all(const FactorArgs& a, const float* bsn, uint32_t row,
                                                      const float* gs, uint32_t lane, float* wsc) {
  finalize_row_warp_core<RP>(
      a, bsn, row, [gs](int s) { return reinterpret_cast<const float4*>(gs)[s]; }, lane, wsc);
}

// g held by lane `src` (one-entry-per-lane kernel, RP <= 12): shuffled into
// registers, then the warp row update.
template <int RP>
__device__ __forceinline__ void finalize_row_warp(const FactorArgs& a, const float* bsn, uint32_t row,
                                                  const float (&g)[RP], int src, uint32_t lane, float* wsc) {
  float gg[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) gg[r] = __shfl_sync(0xffffffffu, g[r], src);
  finalize_row_warp_core<RP>(
      a, bsn, row, [&gg](int s) { return make_float4(gg[4 * s], gg[4 * s + 1], gg[4 * s + 2], gg[4 * s + 3]); },
      lane, wsc);
}

template <int RP, typename T>
__device__ __forceinline__ void warp_allreduce(T (&x)[RP]) {
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    T v = x[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    x[r] = v;
  }
}

template <int RP>
constexpr int factor_min_blocks() {
  return RP <= 4 ? 4 : (RP <= 12 ? 3 : 2);
}

// One warp streams one chunk of the mode-n-sorted records (see file header).
// The next window's records are prefetched while the current window's Q rows
// are gathered; per-lane partial sums stay in fp32 (a chunk holds at most
// chunk_size entries, i.e. <= chunk_size/32 terms per lane), rows are
// finalised from the fp32 sums, and only the pieces of split rows are
// written out (and merged) in fp64.
//
// SJ >= 0: the other-mode table j == SJ (small, e.g. the 2200-row Q^(3) of
// BASELINE config 2) was staged into shared memory by the kernel and its
// gathers are LDS.128: a random-row LDG.128 costs one L1 wavefront per lane,
// an LDS.128 over 8 banks-groups about 2.6 per 8 lanes, and the L1 data pipe
// is what bounds this kernel (profiles/r01_ncu_summary.md).
template <int RP, int SJ>
__device__ __forceinline__ const float4* q_row(const FactorArgs& a, int j, uint32_t idx, const float4* qs) {
  if (j == SJ) return qs + static_cast<uint64_t>(idx) * (RP / 4);
  return reinterpret_cast<const float4*>(a.oq[j] + static_cast<uint64_t>(idx) * RP);
}
template <int RP, int SJ>
__device__ __forceinline__ float4 q_ld(const float4* p, int j) {
  if (j == SJ) return *p;
  return __ldg(p);
}
// T2: R <= RP - 2, so the last float4 of a row holds two zero pads: load it
// as a float2 (a random-row LDG.64 costs about half the L1 data-pipe
// wavefronts of an LDG.128; the product is unchanged, the pads are zero).
template <int RP, int SJ, bool T2>
__device__ __forceinline__ float4 q_ld_r(const float4* p, int j, int r) {
  if (T2 && r == RP / 4 - 1) {
    const float2* p2 = reinterpret_cast<const float2*>(p);
    const float2 v = j == SJ ? *p2 : __ldg(p2);
    return make_float4(v.x, v.y, 0.f, 0.f);
  }
  return q_ld<RP, SJ>(p, j);
}

// LM = 2: RP % 8 == 0, each global row is gathered by 256-bit loads
// (LDG.E.ENL2.256; one load per 32 B instead of two LDG.128).
__device__ __forceinline__ void ldg256(const float4* p, float4& lo, float4& hi) {
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z), "=f"(hi.w)
      : "l"(p));
}
// LM = 3: RP == 12, a 48-B row starts at 0 or 16 mod 32 and spans two
// 32-B sectors either way.  One 256-bit load covers the aligned sector
// pair's 32 B that belong to the row (floats 0..7 of an even row, 4..11 of an
// odd one) and one LDG.128 the remaining 16 B (8..11, or 0..3): two loads and
// two sector accesses per gather instead of three, with no divergence (the
// parity only selects addresses and registers).
template <int RP, int SJ, int LM>
__device__ __forceinline__ void q_ld_row(const float4* qk, int j, float4 (&g)[RP / 4]) {
  if constexpr (LM == 2 && RP % 8 == 0) {
    if (j != SJ) {
#pragma unroll
      for (int r = 0; r < RP / 4; r += 2) ldg256(qk + r, g[r], g[r + 1]);
      return;
    }
  }
  if constexpr (LM == 3 && RP == 12) {
    if (j != SJ) {
      const bool odd = (reinterpret_cast<uintptr_t>(qk) & 31u) != 0;
      float4 lo, hi;
      ldg256(odd ? qk + 1 : qk, lo, hi);
      const float4 rest = __ldg(odd ? qk : qk + 2);
      g[0] = odd ? rest : lo;
      g[1] = odd ? lo : hi;
      g[2] = odd ? hi : rest;
      return;
    }
  }
#pragma unroll
  for (int r = 0; r < RP / 4; ++r) g[r] = q_ld_r<RP, SJ, LM == 1>(qk + r, j, r);
}

template <int RP, int NO, int SJ, int LM>
__device__ __forceinline__ void chunk_body(const FactorArgs& a, const float* bsn, float* wsc, uint32_t wid,
                                           const float4* qs) {
  const uint32_t lane = threadIdx.x & 31;
  const Chunk ch = a.chunks[wid];
  const float* Qn = a.P.Q[a.n];

  if (ch.pad) {
    // A chunk of short rows (< 32 entries each): lane l owns rows r0+l,
    // r0+l+32, ... -- no cross-lane reduction; every lane finalises its own
    // rows together in SIMT.
    const uint32_t r0 = a.keys[ch.begin], r1 = a.keys[ch.end - 1];
    for (uint32_t row = r0 + lane; row <= r1; row += 32) {
      const uint32_t b = static_cast<uint32_t>(a.row_ptr[row] - a.qbase);
      const uint32_t e = static_cast<uint32_t>(a.row_ptr[row + 1] - a.qbase);
      if (b == e) continue;
      const float4* qn = reinterpret_cast<const float4*>(Qn + static_cast<uint64_t>(row) * RP);
      float4 h[RP / 4];
#pragma unroll
      for (int r = 0; r < RP / 4; ++r) h[r] = qn[r];
      float g[RP];
#pragma unroll
      for (int r = 0; r < RP; ++r) g[r] = 0.f;
      for (uint32_t q = b; q < e; ++q) {
        const float x = ld_stream(a.val + q);
        float c[RP];
#pragma unroll
        for (int r = 0; r < RP; ++r) c[r] = 1.f;
#pragma unroll
        for (int j = 0; j < NO; ++j) {
          const float4* qk = q_row<RP, SJ>(a, j, ld_stream(a.oidx[j] + q), qs);
          float4 gr[RP / 4];
          q_ld_row<RP, SJ, LM>(qk, j, gr);
#pragma unroll
          for (int r = 0; r < RP / 4; ++r) {
            const float4 t = gr[r];
            c[4 * r] *= t.x;
            c[4 * r + 1] *= t.y;
            c[4 * r + 2] *= t.z;
            c[4 * r + 3] *= t.w;
          }
        }
        float p = 0.f;
#pragma unroll
        for (int r = 0; r < RP / 4; ++r) {
          p = fmaf(h[r].x, c[4 * r], p);
          p = fmaf(h[r].y, c[4 * r + 1], p);
          p = fmaf(h[r].z, c[4 * r + 2], p);
          p = fmaf(h[r].w, c[4 * r + 3], p);
        }
        const float t = p - x;
#pragma unroll
        for (int r = 0; r < RP; ++r) g[r] = fmaf(t, c[r], g[r]);
      }
      finalize_row<RP>(a, bsn, row, g);
    }
    return;
  }

  // software pipeline: records of the next window
  uint32_t pk = kNone, pi[NO];
  float px = 0.f;
  {
    const uint32_t e = ch.begin + lane;
    if (e < ch.end) {
      pk = ld_stream(a.keys + e);
      px = ld_stream(a.val + e);
#pragma unroll
      for (int j = 0; j < NO; ++j) pi[j] = ld_stream(a.oidx[j] + e);
    }
  }
  uint32_t cur = __shfl_sync(kFull, pk, 0);
  float acc[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) acc[r] = 0.f;
  bool spread = false;  // acc spread over all lanes (else it lives in carry_lane)
  int carry_lane = 0;

  for (uint32_t base = ch.begin; base < ch.end; base += 32) {
    const uint32_t key = pk;
    const float x = px;
    uint32_t ik[NO];
#pragma unroll
    for (int j = 0; j < NO; ++j) ik[j] = pi[j];
    const bool valid = key != kNone;
    {
      const uint32_t e = base + 32 + lane;
      pk = kNone;
      if (e < ch.end) {
        pk = ld_stream(a.keys + e);
        px = ld_stream(a.val + e);
#pragma unroll
        for (int j = 0; j < NO; ++j) pi[j] = ld_stream(a.oidx[j] + e);
      }
    }
    float v[RP];
    if (valid) {
      float4 g[NO][RP / 4];
#pragma unroll
      for (int j = 0; j < NO; ++j) {
        const float4* qk = q_row<RP, SJ>(a, j, ik[j], qs);
        q_ld_row<RP, SJ, LM>(qk, j, g[j]);
      }
      const float4* qn = reinterpret_cast<const float4*>(Qn + static_cast<uint64_t>(key) * RP);
      float4 h[RP / 4];
#pragma unroll
      for (int r = 0; r < RP / 4; ++r) h[r] = qn[r];
      float p = 0.f;
#pragma unroll
      for (int r = 0; r < RP / 4; ++r) {
        float4 c = g[0][r];
#pragma unroll
        for (int j = 1; j < NO; ++j) {
          c.x *= g[j][r].x;
          c.y *= g[j][r].y;
          c.z *= g[j][r].z;
          c.w *= g[j][r].w;
        }
        v[4 * r] = c.x;
        v[4 * r + 1] = c.y;
        v[4 * r + 2] = c.z;
        v[4 * r + 3] = c.w;
        p = fmaf(h[r].x, c.x, p);
        p = fmaf(h[r].y, c.y, p);
        p = fmaf(h[r].z, c.z, p);
        p = fmaf(h[r].w, c.w, p);
      }
      const float t = p - x;
#pragma unroll
      for (int r = 0; r < RP; ++r) v[r] *= t;
    } else {
#pragma unroll
      for (int r = 0; r < RP; ++r) v[r] = 0.f;
    }
    if (__all_sync(kFull, key == cur)) {
#pragma unroll
      for (int r = 0; r < RP; ++r) acc[r] += v[r];
      spread = true;
      continue;
    }
    // ---- window crosses a row boundary
    const uint32_t pkey = __shfl_up_sync(kFull, key, 1);
    const unsigned vmask = __ballot_sync(kFull, valid);
    const unsigned heads = __ballot_sync(kFull, valid && (lane == 0 ? key != cur : key != pkey));
    if (__popc(heads) == 1) {
      // one row ends here (cur, lanes < b plus the carry) and one row starts
      // at lane b and stays open: no scan, one warp reduction.
      const int b = __ffs(heads) - 1;
      float tot[RP];
#pragma unroll
      for (int r = 0; r < RP; ++r) tot[r] = acc[r] + (static_cast<int>(lane) < b ? v[r] : 0.f);
      warp_allreduce<RP>(tot);
      finalize_row_warp<RP>(a, bsn, cur, tot, 0, lane, wsc);
      cur = __shfl_sync(kFull, key, b);
#pragma unroll
      for (int r = 0; r < RP; ++r) acc[r] = static_cast<int>(lane) >= b ? v[r] : 0.f;
      spread = true;
      continue;
    }
    float tot[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) tot[r] = acc[r];
    if (spread) {
      warp_allreduce<RP>(tot);
    } else {
#pragma unroll
      for (int r = 0; r < RP; ++r) tot[r] = __shfl_sync(kFull, tot[r], carry_lane);
    }
    // segmented inclusive scan of v by key (keys are sorted inside the window)
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t okey = __shfl_up_sync(kFull, key, d);
      const bool take = lane >= static_cast<uint32_t>(d) && okey == key;
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        const float o = __shfl_up_sync(kFull, v[r], d);
        if (take) v[r] += o;
      }
    }
    const uint32_t nkey = __shfl_down_sync(kFull, key, 1);
    const int last_valid = 31 - __clz(vmask);
    const bool seg_end = valid && (lane == 31 || nkey != key);
    const bool is_last = static_cast<int>(lane) == last_valid;
    if (key == cur) {
#pragma unroll
      for (int r = 0; r < RP; ++r) v[r] += tot[r];
    }
    const uint32_t key0 = __shfl_sync(kFull, key, 0);
    unsigned fin = __ballot_sync(kFull, seg_end && !is_last);
    if (key0 != cur) finalize_row_warp<RP>(a, bsn, cur, tot, 0, lane, wsc);  // row ended at the window edge
    if (__popc(fin) <= 4) {
      while (fin) {
        const int src = __ffs(fin) - 1;
        fin &= fin - 1;
        finalize_row_warp<RP>(a, bsn, __shfl_sync(kFull, key, src), v, src, lane, wsc);
      }
    } else if (seg_end && !is_last) {
      finalize_row<RP>(a, bsn, key, v);
    }
    cur = __shfl_sync(kFull, key, last_valid);
#pragma unroll
    for (int r = 0; r < RP; ++r) acc[r] = is_last ? v[r] : 0.f;
    spread = false;
    carry_lane = last_valid;
  }
  // ---- the open row at the chunk end
  float tot[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) tot[r] = acc[r];
  if (spread) {
    warp_allreduce<RP>(tot);
  } else {
#pragma unroll
    for (int r = 0; r < RP; ++r) tot[r] = __shfl_sync(kFull, tot[r], carry_lane);
  }
  if (ch.piece < 0) {
    finalize_row_warp<RP>(a, bsn, cur, tot, 0, lane, wsc);
  } else if (lane == 0) {
    double* dst = a.piece + static_cast<uint64_t>(ch.piece) * RP;
#pragma unroll
    for (int r = 0; r < RP; ++r) dst[r] = static_cast<double>(tot[r]);
  }
}

template <int RP, int NO, int LM>
__global__ void __launch_bounds__(256, factor_min_blocks<RP>()) factor_chunk_kernel(FactorArgs a) {
  __shared__ __align__(16) float bsn[SGDT_MAX_J * bstride<RP>()];
  __shared__ __align__(16) float wscr[8 * kWarpScratch];
  load_bsn<RP>(a, bsn);
  __syncthreads();
  const uint32_t wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid < a.n_chunks) chunk_body<RP, NO, -1, LM>(a, bsn, wscr + (threadIdx.x >> 5) * kWarpScratch, wid, nullptr);
}

// Staged variant: persistent CTAs of kStagedWarps warps copy table SJ into
// shared memory once, then stride over the chunks.
#ifndef SGDT_STAGED_WARPS
#define SGDT_STAGED_WARPS 24
#endif
constexpr int kStagedWarps = SGDT_STAGED_WARPS;
template <int RP, int NO, int SJ, int LM>
__global__ void __launch_bounds__(kStagedWarps * 32, 1) factor_staged_kernel(FactorArgs a) {
  __shared__ __align__(16) float bsn[SGDT_MAX_J * bstride<RP>()];
  __shared__ __align__(16) float wscr[kStagedWarps * kWarpScratch];
  extern __shared__ float4 qs[];
  load_bsn<RP>(a, bsn);
  if constexpr (SJ >= 0) {
    const float4* src = reinterpret_cast<const float4*>(a.oq[SJ]);
    const uint32_t n4 = a.orows[SJ] * (RP / 4);
    for (uint32_t i = threadIdx.x; i < n4; i += blockDim.x) qs[i] = __ldg(src + i);
  }
  __syncthreads();
  float* wsc = wscr + (threadIdx.x >> 5) * kWarpScratch;
  for (uint32_t wid = blockIdx.x * kStagedWarps + (threadIdx.x >> 5); wid < a.n_chunks;
       wid += gridDim.x * kStagedWarps)
    chunk_body<RP, NO, SJ, LM>(a, bsn, wsc, wid, qs);
}

// ---------------------------------------------------------------------------
// Wide rows (RP >= 16): G = RP/4 lanes cooperate on one entry, each lane owning
// a float4 slice of the R-space vectors, E = 32/G entries per warp step.  A Q
// row is gathered by one LDG.128 per lane of the group; p needs a log2(G)
// group reduction; row boundaries are a scan over E groups of float4s.  This
// keeps 4 accumulator registers per lane where the one-entry-per-lane kernel
// would carry RP of them and scan RP-wide vectors over 32 lanes.
template <int RP>
struct Lanes {
  static constexpr int G = RP / 4;
  static constexpr int E = 32 / G;
  static constexpr bool kPow2 = (G & (G - 1)) == 0;
};

template <int G, bool POW2>
__device__ __forceinline__ float group_sum(float p, int leader) {
  if constexpr (G == 1) {
    return p;
  } else if constexpr (POW2) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) p += __shfl_xor_sync(kFull, p, o);
    return p;
  } else {
    float t = 0.f;
#pragma unroll
    for (int s = 0; s < G; ++s) t += __shfl_sync(kFull, p, leader + s);
    return t;
  }
}

__device__ __forceinline__ float4 shfl4(const float4& v, int src) {
  return make_float4(__shfl_sync(kFull, v.x, src), __shfl_sync(kFull, v.y, src), __shfl_sync(kFull, v.z, src),
                     __shfl_sync(kFull, v.w, src));
}
__device__ __forceinline__ float4 shfl4_up(const float4& v, int d) {
  return make_float4(__shfl_up_sync(kFull, v.x, d), __shfl_up_sync(kFull, v.y, d),
                     __shfl_up_sync(kFull, v.z, d), __shfl_up_sync(kFull, v.w, d));
}
__device__ __forceinline__ void add4(float4& a, const float4& b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}

// Group `grp`'s RP components (a float4 per lane) into the warp's scratch.
__device__ __forceinline__ void group_row(const float4& v, int grp, int gi, int sub, float* gsc) {
  __syncwarp();
  if (gi == grp) reinterpret_cast<float4*>(gsc)[sub] = v;
  __syncwarp();
}

// MINB: resident CTAs per SM the register budget is cut for.  4 (64 registers) is the
// default.  5 (51 registers, 40 warps per SM) is used for 3-order tensors when every
// gathered Q table is far larger than the L2, i.e. the mode waits on DRAM row gathers and
// more warps in flight pay: config 5 mode 2 (two 1.28 GB tables) 7.26 -> 6.73 ms; with a
// small table among them it is slower (config 5 modes 0/1 10.25 -> 10.6 ms), and with
// more gathered rows per entry it spills (config 4, N = 5: 0.98 -> 1.65 ms per mode);
// 6 CTAs per SM (42 registers) spill as well (config 5: 10.2 -> 16.0 ms per mode).
template <int RP, int NO, int MINB>
__global__ void __launch_bounds__(256, MINB) factor_group_kernel(FactorArgs a) {
  constexpr int G = Lanes<RP>::G, E = Lanes<RP>::E;
  __shared__ __align__(16) float bsn[SGDT_MAX_J * bstride<RP>()];
  __shared__ __align__(16) float wscr[8 * kWarpScratch];
  load_bsn<RP>(a, bsn);
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  float* wsc = wscr + (threadIdx.x >> 5) * kWarpScratch;
  float* gsc = wsc + 64;
  const uint32_t wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= a.n_chunks) return;
  const Chunk ch = a.chunks[wid];
  const int gi = static_cast<int>(lane) / G, sub = static_cast<int>(lane) % G, leader = gi * G;
  const bool glane = gi < E;
  const float* Qn = a.P.Q[a.n];

  // records of the current step (key, x, ik) and the next one (pk, px, pi);
  // the current step's Q rows (t, h) were requested one step earlier, so a
  // step's gathers are in flight while the previous step is reduced
  uint32_t key = kNone, ik[NO], pk = kNone, pi[NO];
  float x = 0.f, px = 0.f;
#pragma unroll
  for (int j = 0; j < NO; ++j) ik[j] = pi[j] = 0;
  {
    const uint32_t e = ch.begin + gi;
    if (glane && e < ch.end) {
      key = ld_stream(a.keys + e);
      x = ld_stream(a.val + e);
#pragma unroll
      for (int j = 0; j < NO; ++j) ik[j] = ld_stream(a.oidx[j] + e);
    }
    const uint32_t e1 = e + E;
    if (glane && e1 < ch.end) {
      pk = ld_stream(a.keys + e1);
      px = ld_stream(a.val + e1);
#pragma unroll
      for (int j = 0; j < NO; ++j) pi[j] = ld_stream(a.oidx[j] + e1);
    }
  }
  float4 t[NO], h;
  if (key != kNone) {
#pragma unroll
    for (int j = 0; j < NO; ++j)
      t[j] = __ldg(reinterpret_cast<const float4*>(a.oq[j] + static_cast<uint64_t>(ik[j]) * RP) + sub);
    h = reinterpret_cast<const float4*>(Qn + static_cast<uint64_t>(key) * RP)[sub];
  }
  uint32_t cur = __shfl_sync(kFull, key, 0);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  bool spread = false;  // acc spread over the groups (else it lives in group carry_g)
  int carry_g = 0;

  for (uint32_t base = ch.begin; base < ch.end; base += E) {
    const uint32_t ckey = key;
    const float cx = x;
    const bool valid = ckey != kNone;
    float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
    float p = 0.f;
    if (valid) {
      c = t[0];
#pragma unroll
      for (int j = 1; j < NO; ++j) {
        c.x *= t[j].x;
        c.y *= t[j].y;
        c.z *= t[j].z;
        c.w *= t[j].w;
      }
      p = h.x * c.x;
      p = fmaf(h.y, c.y, p);
      p = fmaf(h.z, c.z, p);
      p = fmaf(h.w, c.w, p);
    }
    // advance: request the next step's Q rows, prefetch the records after it
    key = pk;
    x = px;
#pragma unroll
    for (int j = 0; j < NO; ++j) ik[j] = pi[j];
    if (key != kNone) {
#pragma unroll
      for (int j = 0; j < NO; ++j)
        t[j] = __ldg(reinterpret_cast<const float4*>(a.oq[j] + static_cast<uint64_t>(ik[j]) * RP) + sub);
      h = reinterpret_cast<const float4*>(Qn + static_cast<uint64_t>(key) * RP)[sub];
    }
    {
      const uint32_t e = base + 2 * E + gi;
      pk = kNone;
      if (glane && e < ch.end) {
        pk = ld_stream(a.keys + e);
        px = ld_stream(a.val + e);
#pragma unroll
        for (int j = 0; j < NO; ++j) pi[j] = ld_stream(a.oidx[j] + e);
      }
    }
    p = group_sum<G, Lanes<RP>::kPow2>(p, leader);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) {
      const float tt = p - cx;
      v = make_float4(tt * c.x, tt * c.y, tt * c.z, tt * c.w);
    }
    if (__all_sync(kFull, !glane || ckey == cur)) {
      add4(acc, v);
      spread = true;
      continue;
    }
    // ---- this step crosses a row boundary
    float4 tot;
    if (spread) {  // sum acc over the groups: scan, the total sits in group E-1
      float4 sc = acc;
#pragma unroll
      for (int d = 1; d < E; d <<= 1) {
        const float4 o = shfl4_up(sc, d * G);
        if (gi >= d) add4(sc, o);
      }
      tot = shfl4(sc, (E - 1) * G + sub);
    } else {
      tot = shfl4(acc, carry_g * G + sub);
    }
#pragma unroll
    for (int d = 1; d < E; d <<= 1) {  // segmented scan of v over the groups by key
      const uint32_t okey = __shfl_up_sync(kFull, ckey, d * G);
      const float4 o = shfl4_up(v, d * G);
      if (gi >= d && okey == ckey) add4(v, o);
    }
    const uint32_t nkey = __shfl_down_sync(kFull, ckey, G);
    const unsigned vmask = __ballot_sync(kFull, valid && sub == 0);
    const int last_g = (31 - __clz(vmask)) / G;
    const bool seg_end = valid && (gi == E - 1 || nkey != ckey);
    const bool is_last = gi == last_g;
    if (ckey == cur) add4(v, tot);
    const uint32_t key0 = __shfl_sync(kFull, ckey, 0);
    if (key0 != cur) {  // the open row ended exactly at the previous step
      group_row(tot, 0, gi, sub, gsc);
      finalize_row_warp_all<RP>(a, bsn, cur, gsc, lane, wsc);
    }
    unsigned fin = __ballot_sync(kFull, seg_end && !is_last && sub == 0);
    while (fin) {
      const int src = __ffs(fin) - 1;
      fin &= fin - 1;
      group_row(v, src / G, gi, sub, gsc);
      finalize_row_warp_all<RP>(a, bsn, __shfl_sync(kFull, ckey, src), gsc, lane, wsc);
    }
    cur = __shfl_sync(kFull, ckey, last_g * G);
    if (is_last) {
      acc = v;
    } else {
      acc = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    spread = false;
    carry_g = last_g;
  }
  // ---- the open row at the chunk end
  float4 tot;
  if (spread) {
    float4 sc = acc;
#pragma unroll
    for (int d = 1; d < E; d <<= 1) {
      const float4 o = shfl4_up(sc, d * G);
      if (gi >= d) add4(sc, o);
    }
    tot = shfl4(sc, (E - 1) * G + sub);
  } else {
    tot = shfl4(acc, carry_g * G + sub);
  }
  group_row(tot, 0, gi, sub, gsc);
  if (ch.piece < 0) {
    finalize_row_warp_all<RP>(a, bsn, cur, gsc, lane, wsc);
  } else if (lane < RP) {
    a.piece[static_cast<uint64_t>(ch.piece) * RP + lane] = static_cast<double>(gsc[lane]);
  }
}

// Rows longer than a chunk: sum their pieces, then finalise.  Blocks
// [0, n_big_splits) take one split row with > kSplitBig pieces each: thread t
// sums pieces t, t + 256, ... (fp64), each warp reduces with a butterfly and
// thread 0 adds the eight warp sums in warp order.  (A Zipf head row of
// BASELINE config 2 has ~6000 pieces; summing it with one warp made this
// kernel 50-70 us per mode.)  The later blocks give each warp one short split
// row (lane-strided sum, butterfly).  Fixed association either way, so the
// result is run-to-run identical.
constexpr int kSplitThreads = 256;
template <int RP>
__global__ void __launch_bounds__(kSplitThreads) factor_split_kernel(FactorArgs a) {
  __shared__ __align__(16) float bsn[SGDT_MAX_J * bstride<RP>()];
  __shared__ double part[kSplitThreads / 32][RP];
  load_bsn<RP>(a, bsn);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool big = blockIdx.x < a.n_big_splits;
  const uint32_t idx = big ? blockIdx.x : a.n_big_splits + (blockIdx.x - a.n_big_splits) * (kSplitThreads / 32) + warp;
  const bool have = idx < a.n_splits;
  SplitRow sr{};
  if (have) sr = a.splits[idx];
  double g[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) g[r] = 0.0;
  const uint32_t t0 = big ? threadIdx.x : lane, step = big ? kSplitThreads : 32;
  if (have)
    for (uint32_t p = t0; p < sr.count; p += step) {
      const double* src = a.piece + static_cast<uint64_t>(sr.first + p) * RP;
#pragma unroll
      for (int r = 0; r < RP; ++r) g[r] += src[r];
    }
  warp_allreduce<RP>(g);
  if (big) {
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < RP; ++r) part[warp][r] = g[r];
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
#pragma unroll
    for (int r = 0; r < RP; ++r) {
      double t = part[0][r];
      for (int w = 1; w < kSplitThreads / 32; ++w) t += part[w][r];
      g[r] = t;
    }
  } else {
    __syncthreads();  // bsn
    if (!have || lane != 0) return;
  }
  if (sr.pad) {  // cut by the slice edge: export for the rank-ordered merge
    double* dst = a.xport + static_cast<uint64_t>(sr.pad - 1) * RP;
#pragma unroll
    for (int r = 0; r < RP; ++r) dst[r] = g[r];
  } else {
    finalize_row<RP>(a, bsn, sr.row, g);
  }
}

// Finalise rows whose gradient was merged across ranks (g: k x RP, fp64).
template <int RP>
__global__ void __launch_bounds__(256) factor_finish_kernel(FactorArgs a, uint32_t k, const uint32_t* rows,
                                                            const double* gm) {
  __shared__ __align__(16) float bsn[SGDT_MAX_J * bstride<RP>()];
  load_bsn<RP>(a, bsn);
  __syncthreads();
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= k) return;
  double g[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) g[r] = gm[static_cast<uint64_t>(t) * RP + r];
  finalize_row<RP>(a, bsn, rows[t], g);
}

// Shared-memory staging of one other-mode table (factor_staged_kernel): the
// smallest table that fits kStageBytes, for RP <= 12 and orders 2-4.
// SGDT_STAGE=0 turns it off (A/B runs).
constexpr uint32_t kStageBytes = 104 * 1024;
template <int RP, int NO>
int staged_table(const FactorArgs& a) {
  if (RP > 12 || NO > 3) return -1;
  static const bool off = [] {
    const char* e = getenv("SGDT_STAGE");
    return e && atoi(e) == 0;
  }();
  if (off) return -1;
  int best = -1;
  for (int j = 0; j < NO; ++j)
    if (static_cast<uint64_t>(a.orows[j]) * RP * sizeof(float) <= kStageBytes &&
        (best < 0 || a.orows[j] < a.orows[best]))
      best = j;
  return best;
}

template <int RP, int NO, int SJ, int LM>
cudaError_t staged_launch_j(Session& s, const FactorArgs& a) {
  if constexpr (SJ >= NO || RP > 12 || NO > 3) {
    return cudaErrorInvalidValue;
  } else {
    const size_t smem = SJ >= 0 ? static_cast<size_t>(a.orows[SJ < 0 ? 0 : SJ]) * RP * sizeof(float) : 0;
    auto kern = factor_staged_kernel<RP, NO, SJ, LM>;
    // per device (a process may drive several), cheap host calls
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kStageBytes));
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kStagedWarps * 32, smem);
    if (e != cudaSuccess) return e;
    const int per_sm = occ < 1 ? 1 : occ;
    const uint32_t need = (a.n_chunks + kStagedWarps - 1) / kStagedWarps;
    const uint32_t grid = std::min<uint32_t>(need, static_cast<uint32_t>(per_sm) * s.num_sms);
    kern<<<grid, kStagedWarps * 32, smem, s.stream>>>(a);
    return cudaGetLastError();
  }
}

template <int RP, int NO, int LM>
cudaError_t staged_launch(Session& s, const FactorArgs& a, int sj) {
  switch (sj) {
    case -1: return staged_launch_j<RP, NO, -1, LM>(s, a);  // persistent, no staged table
    case 0: return staged_launch_j<RP, NO, 0, LM>(s, a);
    case 1: return staged_launch_j<RP, NO, 1, LM>(s, a);
    case 2: return staged_launch_j<RP, NO, 2, LM>(s, a);
    default: return cudaErrorInvalidValue;
  }
}

template <int RP, int NO>
int factor_launch(Session& s, FactorArgs& a) {
  const int block = 256, wpb = block / 32;
  if (a.n_chunks) {
    const unsigned grid = (a.n_chunks + wpb - 1) / wpb;
    static const bool force_group = [] {
      const char* e = getenv("SGDT_GROUP_KERNEL");
      return e && atoi(e) != 0;
    }();
    const int sj = RP >= 16 || force_group ? -1 : staged_table<RP, NO>(a);
    if (RP >= 16 || force_group) {
      bool dram_bound = NO == 2;  // every gathered table > 64 MB (half the L2)
      for (int k = 0; k < s.order; ++k)
        if (k != a.n && static_cast<uint64_t>(s.dims[k]) * RP * sizeof(float) <= (64ull << 20)) dram_bound = false;
      static const int minb_env = [] {  // SGDT_GROUP_MINB=4|5 forces a variant (A/B runs)
        const char* e = getenv("SGDT_GROUP_MINB");
        return e ? atoi(e) : 0;
      }();
      if (minb_env == 4) dram_bound = false;
      if (minb_env == 5) dram_bound = NO == 2;
      if constexpr (NO == 2) {
        if (dram_bound)
          factor_group_kernel<RP, NO, 5><<<grid, block, 0, s.stream>>>(a);
        else
          factor_group_kernel<RP, NO, 4><<<grid, block, 0, s.stream>>>(a);
      } else {
        factor_group_kernel<RP, NO, 4><<<grid, block, 0, s.stream>>>(a);
      }
    }
    else {
      // T2 (half-width tail loads) is instantiated for RP = 12 only (R = 9, 10)
      static const bool t2_off = [] {  // SGDT_T2=0: full-width tails (A/B runs)
        const char* e = getenv("SGDT_T2");
        return e && atoi(e) == 0;
      }();
      const bool t2 = RP == 12 && a.P.R + 2 <= RP && !t2_off;
      static const bool w256_off = [] {  // SGDT_LDG256=0: two LDG.128 per 32 B (A/B runs)
        const char* e = getenv("SGDT_LDG256");
        return e && atoi(e) == 0;
      }();
      const bool w256 = (RP % 8 == 0 || RP == 12) && !w256_off;
      static const bool persist = [] {  // SGDT_PERSIST=1: persistent launch without a staged table
        const char* e = getenv("SGDT_PERSIST");
        return e && atoi(e) != 0;
      }();
      constexpr int kLM256 = RP % 8 == 0 ? 2 : (RP == 12 ? 3 : 0);
      constexpr int kLMT2 = RP == 12 ? 1 : 0;
      if (sj >= 0 || (persist && RP <= 12 && NO <= 3)) {
        // (RP = 12 keeps the half-width tails next to a staged table: the
        // 256+128 parity loads measured 1.6-3 % slower there, 2.5 % faster
        // in the chunk kernel where both tables are global)
        const cudaError_t e = t2                ? staged_launch<RP, NO, kLMT2>(s, a, sj)
                              : w256 && RP != 12 ? staged_launch<RP, NO, kLM256>(s, a, sj)
                                                 : staged_launch<RP, NO, 0>(s, a, sj);
        SGDT_CUDA(e);
      } else if (w256) {
        factor_chunk_kernel<RP, NO, kLM256><<<grid, block, 0, s.stream>>>(a);
      } else if (t2) {
        factor_chunk_kernel<RP, NO, kLMT2><<<grid, block, 0, s.stream>>>(a);
      } else {
        factor_chunk_kernel<RP, NO, 0><<<grid, block, 0, s.stream>>>(a);
      }
    }
    SGDT_CUDA(cudaGetLastError());
    ++s.launches;
  }
  if (a.n_splits) {
    const uint32_t wpb_s = kSplitThreads / 32;
    const unsigned grid = a.n_big_splits + (a.n_splits - a.n_big_splits + wpb_s - 1) / wpb_s;
    factor_split_kernel<RP><<<grid, kSplitThreads, 0, s.stream>>>(a);
    SGDT_CUDA(cudaGetLastError());
    ++s.launches;
  }
  return SGDT_OK;
}

template <int RP>
int finish_launch(Session& s, FactorArgs& a, uint32_t k, const uint32_t* rows, const double* g) {
  factor_finish_kernel<RP><<<(k + 255) / 256, 256, 0, s.stream>>>(a, k, rows, g);
  SGDT_CUDA(cudaGetLastError());
  ++s.launches;
  return SGDT_OK;
}

template <int NO>
int factor_launch_no(Session& s, FactorArgs& a) {
  switch (s.RP) {
    case 4: return factor_launch<4, NO>(s, a);
    case 8: return factor_launch<8, NO>(s, a);
    case 12: return factor_launch<12, NO>(s, a);
    case 16: return factor_launch<16, NO>(s, a);
    case 20: return factor_launch<20, NO>(s, a);
    case 24: return factor_launch<24, NO>(s, a);
    case 28: return factor_launch<28, NO>(s, a);
    case 32: return factor_launch<32, NO>(s, a);
    default: break;
  }
  return fail(SGDT_ERR_CONFIG, "unsupported R_core");
}

FactorArgs factor_args(Session& s, int n, const sgdt_factor_hyper& h, bool subset = false) {
  const ModePlan& mp = s.mode[n];
  const RowSubset& rs = mp.subset;
  const RecordCopy& rec = subset ? rs.rec : mp.rec;
  FactorArgs a{};
  a.P = s.P;
  a.n = n;
  a.keys = rec.idx + static_cast<uint64_t>(n) * rec.nnz;
  a.val = rec.val;
  int j = 0;
  for (int k = 0; k < s.order; ++k) {
    if (k == n) continue;
    a.oidx[j] = rec.idx + static_cast<uint64_t>(k) * rec.nnz;
    a.oq[j] = s.P.Q[k];
    a.orows[j] = s.dims[k];
    ++j;
  }
  a.nnz = rec.nnz;
  a.row_ptr = subset ? rs.sub_off : mp.row_ptr;  // the batch count of a row is its kept subset
  a.chunks = subset ? rs.chunks : mp.chunks;
  a.n_chunks = subset ? rs.n_chunks : mp.n_chunks;
  a.splits = subset ? rs.splits : mp.splits;
  a.n_splits = subset ? rs.n_splits : mp.n_splits;
  a.n_big_splits = subset ? rs.n_big_splits : mp.n_big_splits;
  a.piece = s.piece_partials;
  a.xport = s.export_buf;
  a.qbase = subset ? 0 : mp.shard.qb;
  a.lr = h.lr;
  a.reg = h.reg;
  a.flag = s.flag;
  a.peers = s.npeers > 0 ? s.d_peers + n : nullptr;
  return a;
}

}  // namespace

int launch_factor_mode(Session& s, int n, const sgdt_factor_hyper& h, bool subset) {
  FactorArgs a = factor_args(s, n, h, subset);
  switch (s.order - 1) {
    case 1: return factor_launch_no<1>(s, a);
    case 2: return factor_launch_no<2>(s, a);
    case 3: return factor_launch_no<3>(s, a);
    case 4: return factor_launch_no<4>(s, a);
    case 5: return factor_launch_no<5>(s, a);
    case 6: return factor_launch_no<6>(s, a);
    case 7: return factor_launch_no<7>(s, a);
    default: break;
  }
  return fail(SGDT_ERR_CONFIG, "unsupported tensor order");
}

int launch_factor_finish(Session& s, int n, const sgdt_factor_hyper& h, uint32_t k, const uint32_t* rows,
                         const double* g) {
  if (k == 0) return SGDT_OK;
  FactorArgs a = factor_args(s, n, h);
  switch (s.RP) {
    case 4: return finish_launch<4>(s, a, k, rows, g);
    case 8: return finish_launch<8>(s, a, k, rows, g);
    case 12: return finish_launch<12>(s, a, k, rows, g);
    case 16: return finish_launch<16>(s, a, k, rows, g);
    case 20: return finish_launch<20>(s, a, k, rows, g);
    case 24: return finish_launch<24>(s, a, k, rows, g);
    case 28: return finish_launch<28>(s, a, k, rows, g);
    case 32: return finish_launch<32>(s, a, k, rows, g);
    default: break;
  }
  return fail(SGDT_ERR_CONFIG, "unsupported R_core");
}

}  // namespace sgdt
