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
// per lane in fp64; a window that crosses rows runs a segmented shuffle scan
// and every completed row is finalised by the lane that holds its sum
// (F = B g, SGD step, Q^(n) row rewrite).  Pieces of split rows are summed in
// piece order by factor_split_kernel.  No atomics on parameters, fixed
// association everywhere -> run-to-run bit identical.
#include <cuda_runtime.h>

#include "sgdt_internal.cuh"

namespace sgdt {

namespace {

constexpr unsigned kFull = 0xffffffffu;

struct FactorArgs {
  Params P;
  int n;
  const uint32_t* idx;  // mode-n copy: order x nnz (0-based)
  const float* val;     // nnz
  uint64_t nnz;
  const uint32_t* row_ptr;
  const Chunk* chunks;
  uint32_t n_chunks;
  const SplitRow* splits;
  uint32_t n_splits;
  double* piece;  // n_pieces x RP
  double lr, reg;
  int* flag;
};

template <int RP>
__device__ __forceinline__ void load_bsn(const FactorArgs& a, float* bsn) {
  const uint32_t jn = a.P.J[a.n];
  for (uint32_t i = threadIdx.x; i < jn * RP; i += blockDim.x) {
    const uint32_t j = i / RP, r = i % RP;
    bsn[i] = r < a.P.R ? a.P.B[a.n][j * a.P.R + r] : 0.f;
  }
}

// F = B^(n) g; a -= lr (F/cnt + reg a); Q^(n)[row] = a B^(n).  One lane.
template <int RP>
__device__ void finalize_row(const FactorArgs& a, const float* bsn, uint32_t row,
                             const double (&g)[RP]) {
  const uint32_t jn = a.P.J[a.n];
  const uint32_t cnt = a.row_ptr[row + 1] - a.row_ptr[row];
  const double inv = 1.0 / static_cast<double>(cnt);
  float* arow = a.P.A[a.n] + static_cast<uint64_t>(row) * jn;
  int bad = 0;
  float q[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) q[r] = 0.f;
  for (uint32_t j = 0; j < jn; ++j) {
    double F = 0.0;
#pragma unroll
    for (int r = 0; r < RP; ++r) F = fma(static_cast<double>(bsn[j * RP + r]), g[r], F);
    double w = static_cast<double>(arow[j]);
    bad |= !isfinite(w) || !isfinite(F);
    w -= a.lr * (F * inv + a.reg * w);
    const float wf = static_cast<float>(w);
    bad |= !isfinite(wf);
    arow[j] = wf;
#pragma unroll
    for (int r = 0; r < RP; ++r) q[r] = fmaf(wf, bsn[j * RP + r], q[r]);
  }
  float4* dst = reinterpret_cast<float4*>(a.P.Q[a.n] + static_cast<uint64_t>(row) * RP);
#pragma unroll
  for (int r = 0; r < RP; r += 4) dst[r / 4] = make_float4(q[r], q[r + 1], q[r + 2], q[r + 3]);
  if (bad) atomicOr(a.flag, 8);
}

template <int RP>
__device__ __forceinline__ void warp_allreduce(double (&x)[RP]) {
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    double v = x[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    x[r] = v;
  }
}

template <int RP>
__global__ void __launch_bounds__(256) factor_chunk_kernel(FactorArgs a) {
  __shared__ float bsn[SGDT_MAX_J * RP];
  load_bsn<RP>(a, bsn);
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= a.n_chunks) return;
  const Chunk ch = a.chunks[wid];
  const int n = a.n, order = a.P.order;
  const uint32_t* keys = a.idx + static_cast<uint64_t>(n) * a.nnz;
  const float* Qn = a.P.Q[n];

  uint32_t cur = keys[ch.begin];
  double acc[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) acc[r] = 0.0;
  bool spread = false;   // acc spread over all lanes (else only in carry_lane)
  int carry_lane = 0;

  for (uint32_t base = ch.begin; base < ch.end; base += 32) {
    const uint32_t e = base + lane;
    const bool valid = e < ch.end;
    uint32_t key = kNone;
    float v[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) v[r] = 0.f;
    if (valid) {
      key = __ldcs(keys + e);
      const float x = __ldcs(a.val + e);
      float c[RP];
#pragma unroll
      for (int r = 0; r < RP; ++r) c[r] = 1.f;
      for (int k = 0; k < order; ++k) {
        if (k == n) continue;
        const uint32_t ik = __ldcs(a.idx + static_cast<uint64_t>(k) * a.nnz + e);
        const float4* qk = reinterpret_cast<const float4*>(a.P.Q[k] + static_cast<uint64_t>(ik) * RP);
#pragma unroll
        for (int r = 0; r < RP; r += 4) {
          const float4 t = __ldg(qk + r / 4);
          c[r] *= t.x;
          c[r + 1] *= t.y;
          c[r + 2] *= t.z;
          c[r + 3] *= t.w;
        }
      }
      const float4* qn = reinterpret_cast<const float4*>(Qn + static_cast<uint64_t>(key) * RP);
      float p = 0.f;
#pragma unroll
      for (int r = 0; r < RP; r += 4) {
        const float4 t = qn[r / 4];
        p = fmaf(t.x, c[r], p);
        p = fmaf(t.y, c[r + 1], p);
        p = fmaf(t.z, c[r + 2], p);
        p = fmaf(t.w, c[r + 3], p);
      }
      const float t = p - x;
#pragma unroll
      for (int r = 0; r < RP; ++r) v[r] = t * c[r];
    }
    if (__all_sync(kFull, key == cur)) {
#pragma unroll
      for (int r = 0; r < RP; ++r) acc[r] += static_cast<double>(v[r]);
      spread = true;
      continue;
    }
    // ---- window crosses a row boundary
    double tot[RP];
    if (spread) {
#pragma unroll
      for (int r = 0; r < RP; ++r) tot[r] = acc[r];
      warp_allreduce<RP>(tot);
    } else {
#pragma unroll
      for (int r = 0; r < RP; ++r) tot[r] = __shfl_sync(kFull, acc[r], carry_lane);
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
    const unsigned vmask = __ballot_sync(kFull, valid);
    const int last_valid = 31 - __clz(vmask);
    const bool seg_end = valid && (lane == 31 || nkey != key);
    const bool is_last = static_cast<int>(lane) == last_valid;
    const bool first_seg = key == cur;
    double g[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) g[r] = static_cast<double>(v[r]) + (first_seg ? tot[r] : 0.0);
    if (lane == 0 && key != cur) finalize_row<RP>(a, bsn, cur, tot);  // row ended at the window edge
    if (seg_end && !is_last) finalize_row<RP>(a, bsn, key, g);
    cur = __shfl_sync(kFull, key, last_valid);
#pragma unroll
    for (int r = 0; r < RP; ++r) acc[r] = is_last ? g[r] : 0.0;
    spread = false;
    carry_lane = last_valid;
  }
  // ---- the open row at the chunk end
  double tot[RP];
  if (spread) {
#pragma unroll
    for (int r = 0; r < RP; ++r) tot[r] = acc[r];
    warp_allreduce<RP>(tot);
  } else {
#pragma unroll
    for (int r = 0; r < RP; ++r) tot[r] = __shfl_sync(kFull, acc[r], carry_lane);
  }
  if (lane == 0) {
    if (ch.piece < 0) {
      finalize_row<RP>(a, bsn, cur, tot);
    } else {
      double* dst = a.piece + static_cast<uint64_t>(ch.piece) * RP;
#pragma unroll
      for (int r = 0; r < RP; ++r) dst[r] = tot[r];
    }
  }
}

// Rows longer than a chunk: sum their pieces in piece order, then finalise.
template <int RP>
__global__ void __launch_bounds__(256) factor_split_kernel(FactorArgs a) {
  __shared__ float bsn[SGDT_MAX_J * RP];
  load_bsn<RP>(a, bsn);
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= a.n_splits) return;
  const SplitRow sr = a.splits[wid];
  double g[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) g[r] = 0.0;
  for (uint32_t p = lane; p < sr.count; p += 32) {
    const double* src = a.piece + static_cast<uint64_t>(sr.first + p) * RP;
#pragma unroll
    for (int r = 0; r < RP; ++r) g[r] += src[r];
  }
  warp_allreduce<RP>(g);
  if (lane == 0) finalize_row<RP>(a, bsn, sr.row, g);
}

template <int RP>
int factor_launch_rp(Session& s, FactorArgs& a) {
  const int block = 256, wpb = block / 32;
  if (a.n_chunks) {
    const unsigned grid = (a.n_chunks + wpb - 1) / wpb;
    factor_chunk_kernel<RP><<<grid, block, 0, s.stream>>>(a);
    SGDT_CUDA(cudaGetLastError());
    ++s.launches;
  }
  if (a.n_splits) {
    const unsigned grid = (a.n_splits + wpb - 1) / wpb;
    factor_split_kernel<RP><<<grid, block, 0, s.stream>>>(a);
    SGDT_CUDA(cudaGetLastError());
    ++s.launches;
  }
  return SGDT_OK;
}

}  // namespace

int launch_factor_mode(Session& s, int n, const sgdt_factor_hyper& h) {
  const ModePlan& mp = s.mode[n];
  FactorArgs a{};
  a.P = s.P;
  a.n = n;
  a.idx = mp.rec.idx;
  a.val = mp.rec.val;
  a.nnz = mp.rec.nnz;
  a.row_ptr = mp.row_ptr;
  a.chunks = mp.chunks;
  a.n_chunks = mp.n_chunks;
  a.splits = mp.splits;
  a.n_splits = mp.n_splits;
  a.piece = s.piece_partials;
  a.lr = h.lr;
  a.reg = h.reg;
  a.flag = s.flag;
  switch (s.RP) {
    case 4: return factor_launch_rp<4>(s, a);
    case 8: return factor_launch_rp<8>(s, a);
    case 12: return factor_launch_rp<12>(s, a);
    case 16: return factor_launch_rp<16>(s, a);
    case 20: return factor_launch_rp<20>(s, a);
    case 24: return factor_launch_rp<24>(s, a);
    case 28: return factor_launch_rp<28>(s, a);
    case 32: return factor_launch_rp<32>(s, a);
    default: break;
  }
  return fail(SGDT_ERR_CONFIG, "unsupported R_core");
}

}  // namespace sgdt
