// sgdt_core.cu -- K2/K3/K4: the core (Kruskal B^(n)) phase as one cooperative
// kernel, plus the Q^(k) = A^(k) B^(k) refresh fused at its tail.
//
// Reference: update_core_epoch (core_optimizer.cpp:112-257).  For each mode n
// (ascending) and each r_core (ascending, Gauss-Seidel over the columns):
//   resid_s = x_s - sum_{r != rc} W_r[s] . b_r          (:197-223)
//   U = sum_s W_rc[s] resid_s,  C = sum_s W_rc[s] W_rc[s]^T  (:225-243)
//   V = -U + C b_rc;  b_rc -= lr (V/M + reg b_rc)      (:246-250, sgd_step :85-100)
// with W_r[s] = c_{s,r} a^(n)_{i_n(s)} and c_{s,r} = prod_{k != n} a^(k) . b^(k)_r.
// Substituting W gives the identity used here:
//   V = sum_s c_{s,rc} (xhat_s - x_s) a^(n)_s,  xhat_s = sum_r c_{s,r} (a_s . b_r)
// so each step reduces J values instead of J^2 + J.  xhat is kept current
// after every column update (xhat_s += c_{s,rc} a_s . delta_b).
//
// Each CTA owns the contiguous sample slice partition_even(M, grid)[cta]
// (scheduler.cpp:34-46).  A step's partial V goes to a double-buffered global
// array; after grid.sync() every CTA sums the partials in CTA order (fp64) and
// applies the identical update to its shared-memory copy of B, so all CTAs
// stay bit-identical without a broadcast.  One grid barrier per (n, r_core).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "sgdt_internal.cuh"
#include "sgdt_qrows.cuh"

namespace cg = cooperative_groups;

namespace sgdt {

namespace {

struct CoreArgs {
  Params P;
  const uint32_t* rec_idx;  // entry-order copy
  const float* rec_val;
  uint64_t nnz;
  const uint32_t* batch;  // Psi (m) or one Psi per mode (order x m)
  int per_mode;
  uint64_t m;
  uint32_t js;        // sample row stride of sa (max J)
  float* sa;          // m x js      a^(n)_{i_n(s)}
  float* sc;          // m x RP      c_{s,r}
  float* sxh;         // m           xhat_s
  float* sx;          // m           x_s
  double* part;       // 2 x grid x js
  double lr, reg;
  int* flag;
  int q_refresh;      // fuse Q = A B for every mode at the end
  int local;          // per-sample state of the CTA's slice lives in shared memory
  uint32_t cap;       // samples per CTA slice (upper bound)
};

// Warp transpose-reduce: afterwards lane l holds the warp-wide sum of v[l]
// (31 shuffles for 32 values; fixed order, so every run forms the same sums).
__device__ __forceinline__ float warp_reduce32(float (&v)[32], int lane) {
#pragma unroll
  for (int h = 16; h > 0; h >>= 1) {
    const bool up = (lane & h) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const float send = up ? v[i] : v[i + h];
      const float keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  return v[0];
}

// One pass over the CTA's samples for columns j0..j0+31 of V_rcn:
//   (upd >= 0)  xhat_s += c_{s,upd} (a_s . delta_b)    -- column upd was just stepped
//   v_j += c_{s,rcn} (xhat_s - x_s) a_{s,j}
// a_s is loaded once into registers and feeds both terms.
__device__ __forceinline__ void column_pass(const float* la, const float* lc, float* lxh, const float* lx,
                                            const float* dbv, uint32_t cap, uint32_t nloc, uint32_t jn,
                                            int upd, uint32_t rcn, uint32_t j0, float (&v)[32]) {
  for (uint32_t ls = threadIdx.x; ls < nloc; ls += blockDim.x) {
    float av[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) av[q] = j0 + q < jn ? la[(j0 + q) * cap + ls] : 0.f;
    float xh = lxh[ls];
    if (upd >= 0) {
      float d = 0.f;
#pragma unroll
      for (int q = 0; q < 32; ++q) d = fmaf(av[q], dbv[q], d);
      for (uint32_t j = 32; j < jn; ++j) d = fmaf(la[j * cap + ls], dbv[j], d);
      xh = fmaf(lc[upd * cap + ls], d, xh);
      lxh[ls] = xh;
    }
    const float t = lc[rcn * cap + ls] * (xh - lx[ls]);
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = fmaf(t, av[q], v[q]);
  }
}

constexpr int kCoreBlock = 512;

template <int RP>
__global__ void __launch_bounds__(kCoreBlock) core_kernel(CoreArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ unsigned char smem_raw[];
  // Bs[k]: J_k x RP (zero padded), then per-warp partials, then delta b.
  float* bs_base = reinterpret_cast<float*>(smem_raw);
  // offsets (not pointers) so that every access stays a shared-space access
  uint32_t bso[kMaxOrder];
  uint32_t off = 0;
  for (int k = 0; k < a.P.order; ++k) {
    bso[k] = off;
    off += a.P.J[k] * RP;
  }
  const int nwarps = blockDim.x >> 5;
  double* wpart = reinterpret_cast<double*>(bs_base + ((off + 1) & ~1u));  // nwarps x js
  float* dbv = reinterpret_cast<float*>(wpart + nwarps * a.js);           // max(js, 32)
  const uint32_t dbn = a.js > 32 ? a.js : 32;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int k = 0; k < a.P.order; ++k)
    for (uint32_t i = tid; i < a.P.J[k] * RP; i += blockDim.x) {
      const uint32_t j = i / RP, r = i % RP;
      bs_base[bso[k] + i] = r < a.P.R ? a.P.B[k][j * a.P.R + r] : 0.f;
    }
  for (uint32_t j = tid; j < dbn; j += blockDim.x) dbv[j] = 0.f;
  __syncthreads();

  // this CTA's slice of Psi
  const uint64_t base = a.m / gridDim.x, rem = a.m % gridDim.x;
  const uint64_t s0 = blockIdx.x * base + (blockIdx.x < rem ? blockIdx.x : rem);
  const uint64_t s1 = s0 + base + (blockIdx.x < rem ? 1 : 0);
  const uint32_t nloc = static_cast<uint32_t>(s1 - s0);
  const double inv_m = 1.0 / static_cast<double>(a.m);
  // per-sample state of this slice (local index ls = s - s0): shared memory
  // when it fits, else the global scratch
  float *la, *lc, *lxh, *lx;
  if (a.local) {
    la = dbv + dbn;
    lc = la + static_cast<uint64_t>(a.cap) * a.js;
    lxh = lc + static_cast<uint64_t>(a.cap) * RP;
    lx = lxh + a.cap;
  } else {
    const uint64_t cb = static_cast<uint64_t>(blockIdx.x) * a.cap;
    la = a.sa + cb * a.js;
    lc = a.sc + cb * RP;
    lxh = a.sxh + cb;
    lx = a.sx + cb;
  }
  // per-sample vectors are stored transposed (la[j*cap + ls], lc[r*cap + ls])
  // so that thread-per-sample passes are coalesced / bank-conflict free
  uint32_t step = 0;

  for (int n = 0; n < a.P.order; ++n) {
    const uint32_t* batch = a.batch + (a.per_mode ? static_cast<uint64_t>(n) * a.m : 0);
    const uint32_t jn = a.P.J[n];
    for (uint32_t j = tid; j < dbn; j += blockDim.x) dbv[j] = 0.f;
    // ---- per-sample caches: c_{s,r}, a_s, xhat_s, x_s  (:158-180)
    for (uint32_t ls = tid; ls < nloc; ls += blockDim.x) {
      const uint32_t e = batch[s0 + ls];
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
          for (int r = 0; r < RP; ++r) d[r] = fmaf(av, bs_base[bso[k] + j * RP + r], d[r]);
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
        la[j * a.cap + ls] = av;
#pragma unroll
        for (int r = 0; r < RP; ++r) p[r] = fmaf(av, bs_base[bso[n] + j * RP + r], p[r]);
      }
      float xh = 0.f;
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        xh = fmaf(c[r], p[r], xh);
        lc[r * a.cap + ls] = c[r];
      }
      lxh[ls] = xh;
      lx[ls] = a.rec_val[e];
    }
    __syncthreads();

    int upd = -1;  // column whose step is still to be folded into xhat
    for (uint32_t rc = 0; rc < a.P.R; ++rc, ++step) {
      // ---- partial V over this CTA's slice: V_j = sum_s c_{s,rc} (xhat_s - x_s) a_{s,j},
      // fused with the xhat refresh for the previous column's step
      double* part = a.part + static_cast<uint64_t>(step & 1) * gridDim.x * a.js;
      for (uint32_t j0 = 0; j0 < jn; j0 += 32) {
        float v[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = 0.f;
        column_pass(la, lc, lxh, lx, dbv, a.cap, nloc, jn, j0 == 0 ? upd : -1, rc, j0, v);
        const float w = warp_reduce32(v, lane);
        if (j0 + lane < jn) wpart[warp * a.js + j0 + lane] = static_cast<double>(w);
      }
      __syncthreads();
      if (tid < static_cast<int>(jn)) {
        double acc = 0.0;
        for (int w = 0; w < nwarps; ++w) acc += wpart[w * a.js + tid];
        part[static_cast<uint64_t>(tid) * gridDim.x + blockIdx.x] = acc;  // [j][cta]
      }
      grid.sync();
      // ---- every CTA: V_j over the CTA partials (a warp per j, fixed lane
      // striding + butterfly, so every CTA forms the identical sum), then
      // sgd_step on column rc
      for (uint32_t j = warp; j < jn; j += nwarps) {
        const double* pj = part + static_cast<uint64_t>(j) * gridDim.x;
        double V = 0.0;
        for (unsigned b = lane; b < gridDim.x; b += 32) V += __ldcg(pj + b);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) V += __shfl_xor_sync(0xffffffffu, V, o);
        if (lane == 0) {
          const float bold = bs_base[bso[n] + j * RP + rc];
          double w = static_cast<double>(bold);
          int bad = (!isfinite(w) ? 1 : 0) | (!isfinite(V) ? 2 : 0);
          w -= a.lr * (V * inv_m + a.reg * w);
          const float bnew = static_cast<float>(w);
          bad |= !isfinite(bnew) ? 4 : 0;
          if (bad && blockIdx.x == 0) atomicOr(a.flag, bad);
          dbv[j] = bnew - bold;
          bs_base[bso[n] + j * RP + rc] = bnew;
        }
      }
      __syncthreads();
      upd = static_cast<int>(rc);
    }
  }

  // ---- write back B (identical in every CTA) and refresh Q^(k) = A^(k) B^(k)
  if (blockIdx.x == 0)
    for (int k = 0; k < a.P.order; ++k)
      for (uint32_t i = tid; i < a.P.J[k] * a.P.R; i += blockDim.x)
        a.P.B[k][i] = bs_base[bso[k] + (i / a.P.R) * RP + (i % a.P.R)];
  if (!a.q_refresh) return;
  float* stage = dbv + dbn + warp * kQStage;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * nwarps + warp;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * nwarps;
  for (int k = 0; k < a.P.order; ++k)
    q_rows_tiled<RP>(a.P.A[k], a.P.Q[k], a.P.J[k], bs_base + bso[k], a.P.dims[k], gw, nw, stage, lane);
}

// Standalone Q refresh (used after set_model and by the factor phase when the
// core phase is frozen).
template <int RP>
__global__ void __launch_bounds__(256) q_refresh_kernel(Params P, int k) {
  extern __shared__ float bsk[];
  const uint32_t jk = P.J[k];
  for (uint32_t i = threadIdx.x; i < jk * RP; i += blockDim.x) {
    const uint32_t j = i / RP, r = i % RP;
    bsk[i] = r < P.R ? P.B[k][j * P.R + r] : 0.f;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* stage = bsk + jk * RP + warp * kQStage;
  q_rows_tiled<RP>(P.A[k], P.Q[k], jk, bsk, P.dims[k],
                   static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) + warp,
                   static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5), stage, lane);
}

template <int RP>
int core_launch_rp(Session& s, CoreArgs& a) {
  const int block = kCoreBlock;
  size_t bs_floats = 0;
  for (int k = 0; k < s.order; ++k) bs_floats += s.J[k] * RP;
  size_t smem = ((bs_floats + 1) & ~size_t(1)) * sizeof(float) + (block / 32) * a.js * sizeof(double) +
                (a.js > 32 ? a.js : 32) * sizeof(float);
  auto kern = core_kernel<RP>;
  // one CTA per SM keeps grid.sync cheap; small batches use fewer CTAs
  uint64_t want = (a.m + 127) / 128;
  if (want < 1) want = 1;
  int grid = static_cast<int>(want < static_cast<uint64_t>(s.num_sms) ? want : s.num_sms);
  if (a.q_refresh && grid < s.num_sms) {
    uint64_t rows = 0;
    for (int k = 0; k < s.order; ++k) rows += s.dims[k];
    if (rows > static_cast<uint64_t>(grid) * block * 8) grid = s.num_sms;
  }
  if (const char* e = std::getenv("SGDT_CORE_GRID")) {  // diagnostics (A/B runs)
    const int g = std::atoi(e);
    if (g >= 1 && g <= s.num_sms) grid = g;
  }
  a.cap = static_cast<uint32_t>((a.m + grid - 1) / grid);
  const size_t local = static_cast<size_t>(a.cap) * (a.js + RP + 2) * sizeof(float);
  const size_t stage = static_cast<size_t>(block / 32) * kQStage * sizeof(float);  // tail Q refresh
  const size_t tail_local = local > stage ? local : stage;
  a.local = smem + tail_local <= 200 * 1024;
  smem += a.local ? tail_local : stage;
  if (smem > 48 * 1024)
    SGDT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  SGDT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem));
  if (per_sm < 1) return fail(SGDT_ERR_INTERNAL, "core kernel does not fit on an SM");
  s.core_grid = grid;
  void* args[] = {&a};
  SGDT_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(grid), dim3(block),
                                        args, smem, s.stream));
  ++s.launches;
  return SGDT_OK;
}

template <int RP>
int q_launch_rp(Session& s, int k) {
  const size_t smem = (s.J[k] * RP + 8 * kQStage) * sizeof(float);
  if (smem > 48 * 1024)
    SGDT_CUDA(cudaFuncSetAttribute(q_refresh_kernel<RP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  uint64_t blocks = (s.dims[k] + 255) / 256;
  if (blocks > static_cast<uint64_t>(s.num_sms) * 8) blocks = s.num_sms * 8;
  q_refresh_kernel<RP><<<static_cast<unsigned>(blocks), 256, smem, s.stream>>>(s.P, k);
  SGDT_CUDA(cudaGetLastError());
  ++s.launches;
  return SGDT_OK;
}

}  // namespace

int launch_core(Session& s, const sgdt_core_hyper& h, const uint32_t* batches, uint64_t m,
                int per_mode_batches) {
  if (m > s.cs_cap) return fail(SGDT_ERR_INTERNAL, "core scratch too small");
  CoreArgs a{};
  a.P = s.P;
  a.rec_idx = s.train_rec.idx;
  a.rec_val = s.train_rec.val;
  a.nnz = s.nnz;
  a.batch = batches;
  a.per_mode = per_mode_batches;
  a.m = m;
  uint32_t js = 0;
  for (int k = 0; k < s.order; ++k) js = s.J[k] > js ? s.J[k] : js;
  a.js = js;
  a.sa = s.cs_a;
  a.sc = s.cs_c;
  a.sxh = s.cs_xhat;
  a.sx = s.cs_x;
  a.part = s.cs_part;
  a.lr = h.lr;
  a.reg = h.reg;
  a.flag = s.flag;
  a.q_refresh = 1;
#define CORE_CALL(RP) core_launch_rp<RP>(s, a)
  switch (s.RP) {
    case 4: return CORE_CALL(4);
    case 8: return CORE_CALL(8);
    case 12: return CORE_CALL(12);
    case 16: return CORE_CALL(16);
    case 20: return CORE_CALL(20);
    case 24: return CORE_CALL(24);
    case 28: return CORE_CALL(28);
    case 32: return CORE_CALL(32);
    default: break;
  }
#undef CORE_CALL
  return fail(SGDT_ERR_CONFIG, "unsupported R_core");
}

int launch_q_refresh(Session& s, int k) {
  switch (s.RP) {
    case 4: return q_launch_rp<4>(s, k);
    case 8: return q_launch_rp<8>(s, k);
    case 12: return q_launch_rp<12>(s, k);
    case 16: return q_launch_rp<16>(s, k);
    case 20: return q_launch_rp<20>(s, k);
    case 24: return q_launch_rp<24>(s, k);
    case 28: return q_launch_rp<28>(s, k);
    case 32: return q_launch_rp<32>(s, k);
    default: break;
  }
  return fail(SGDT_ERR_CONFIG, "unsupported R_core");
}

}  // namespace sgdt
