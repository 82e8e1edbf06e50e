// sgdt_core.cu -- K2/K3/K4: the core (Kruskal B^(n)) phase as one cooperative
// kernel, plus the Q^(k) = A^(k) B^(k) refresh fused at its tail (wide modes with many
// rows go to the tensor-core refresh of sgdt_qrefresh_tc.cu, launched right after).
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
// (scheduler.cpp:34-46).  Its per-sample state (a_s in float4 groups, c_{s,r},
// xhat_s, x_s) lives in shared memory when it fits; otherwise a_s stays in shared
// memory plus one register-resident sample per thread, xhat / x in shared memory
// and c in an L2-resident scratch with a three-column cp.async ring (core_geometry).
// The setup of a mode gathers the device's current Q^(k) rows for the modes whose
// B^(k) has not been stepped yet in this phase (k > n) and for x-hat the own mode's
// row; only the modes already stepped need a^(k) B^(k) from the shared-memory B.
// A step's partial V goes to a double-buffered global
// array; column j of V belongs to one reducer warp of the grid (CTA j % grid),
// which sums the CTA partials in CTA order (fp64), takes the sgd_step on
// b_{j,rc} and publishes the new value (one shared word, or for J >= 16 one word
// per CTA so that no line is polled by every SM); every CTA then installs the identical
// column in its shared-memory copy of B.  One exchange per (n, r_core).
//
// The exchange carries its own arrival flags: a partial (one double) is stored
// as two 64-bit words {stamp:32 | half:32} and a new column value as one word
// {stamp:32 | fp32}, the stamp unique to (launch, step).  A 64-bit store is
// single-copy atomic, so a reader that sees the stamp has the payload: no fence
// and no counter.  Measured on the B200 (scripts/microbench/exchange_latency.cu):
// a store becomes visible to a polling load of another SM after ~1000 cycles, so
// the two hops cost ~2000 cycles plus the 148-way gather, against ~4800 for
// grid.sync() followed by the all-read-all of the partials (an all-read-all of
// stamped partials is one hop but its 148 x 148 polls flood the L2: slower).
// The cooperative launch is kept because it guarantees that all CTAs are
// co-resident (the polling loops need that).  Slot reuse is safe with two
// buffers: a CTA writes step s+2 only after it has taken every column of step
// s+1, which the reducers published after reading every partial of step s+1,
// which every CTA stored after taking step s.  With the per-sample state in
// global memory (large M x J) the passes dominate and grid.sync() is used
// (launch_core); SGDT_CORE_SYNC=grid|red overrides.  SGDT_CORE_TRACE=1 prints
// CTA 0's cycle counts at the phase boundaries of the first launches.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
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
  uint32_t js;        // max J
  uint32_t ja;        // js rounded up to 4: floats per sample of the a_s caches (float4 groups)
  float* sa;          // m x ja      a^(n)_{i_n(s)}
  float* sc;          // m x RP      c_{s,r}
  float* sxh;         // m           xhat_s
  float* sx;          // m           x_s
  ulonglong2* part;   // 2 x js x grid stamped partials
  unsigned long long* res;  // 2 x grid x js stamped new column values, one copy per CTA
  uint32_t stamp0;    // stamps of this launch are stamp0 + step + 1
  int grid_sync;      // exchange through grid.sync() instead of the stamps (A/B)
  long long* trace;   // SGDT_CORE_TRACE: clock64() of CTA trace_cta at the phase boundaries
  int trace_cta;      // SGDT_CORE_TRACE_CTA (default 0)
  double lr, reg;
  int* flag;
  int q_refresh;      // bit k: fuse Q^(k) = A^(k) B^(k) at the end (the other modes go to the tensor-core refresh)
  int local;          // per-sample state of the CTA's slice: 1 shared memory, 0 global scratch, 2 semi
                      // (a_s in shared memory / registers, xhat and x in shared memory, c_{s,r} global)
  uint32_t cap;       // samples per CTA slice (upper bound)
  int q_rows;         // gather the current Q^(k) rows (k > n, and the own mode's) instead of forming a^(k) B^(k)
  int res_copies;     // the new column goes to one word per CTA (wide J) instead of one shared word
  int ring;           // semi: keep a three-column ring of c in shared memory (SGDT_CORE_RING=0: A/B)
  uint32_t nsm;       // semi: samples whose a_s sit in shared memory (row stride nsm); the samples
                      // nsm + t, t < blockDim, keep a_s in the registers of thread t
};

// Warp transpose-reduce: afterwards lane l holds the warp-wide sum of v[l % JW]
// (JW - 1 shuffles for the transposition plus log2(32 / JW) butterflies; fixed
// order, so every run forms the same sums).
template <int JW>
__device__ __forceinline__ float warp_reduce(float (&v)[JW], int lane) {
#pragma unroll
  for (int h = JW / 2; h > 0; h >>= 1) {
    const bool up = (lane & h) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const float send = up ? v[i] : v[i + h];
      const float keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
#pragma unroll
  for (int o = JW; o < 32; o <<= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
  return v[0];
}

__device__ __forceinline__ void st_stamped(ulonglong2* p, double x, uint32_t stamp) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  const unsigned long long hi = static_cast<unsigned long long>(stamp) << 32;
  const unsigned long long w0 = hi | (b & 0xffffffffull), w1 = hi | (b >> 32);
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}

__device__ __forceinline__ ulonglong2 ld_stamped(const ulonglong2* p) {
  ulonglong2 w;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w.x), "=l"(w.y) : "l"(p) : "memory");
  return w;
}

// One pass over the CTA's samples for columns j0..j0+JW-1 of V_rcn:
//   (upd >= 0)  xhat_s += c_{s,upd} (a_s . delta_b)    -- column upd was just stepped
//   v_j += c_{s,rcn} (xhat_s - x_s) a_{s,j}
// a_s is loaded once into registers and feeds both terms.  The a_s cache is laid out in
// float4 groups, la4[g * capa + ls] = a_s[4g .. 4g+3] (zero past J): a thread-per-sample
// pass is conflict-free, takes J/4 128-bit loads per sample and J/4 row offsets (32-bit
// loads cost ~600 issue slots per sample at J = 32, mostly address arithmetic: config 5
// pass measured at 15.7k cycles).  la4 holds the first nla samples; with REG the sample
// nla + threadIdx.x keeps its a_s in areg (JW = 32 covers the whole row, j0 = 0).
template <int JW, bool REG>
__device__ __forceinline__ void column_pass(const float4* la4, uint32_t capa, uint32_t nla, const float* c_rcn,
                                            const float* c_upd, float* lxh, const float* lx, const float* dbv,
                                            uint32_t nloc, uint32_t jn, int upd, uint32_t j0, float (&v)[JW],
                                            const float (&areg)[32]) {
  const float4* db4 = reinterpret_cast<const float4*>(dbv);
  const uint32_t jn4 = (jn + 3) >> 2, g0 = j0 >> 2;
  for (uint32_t ls = threadIdx.x; ls < nla; ls += blockDim.x) {
    float av[JW];
#pragma unroll
    for (int g = 0; g < JW / 4; ++g) {
      const float4 t = g0 + g < jn4 ? la4[(g0 + g) * capa + ls] : make_float4(0.f, 0.f, 0.f, 0.f);
      av[4 * g] = t.x, av[4 * g + 1] = t.y, av[4 * g + 2] = t.z, av[4 * g + 3] = t.w;
    }
    float xh = lxh[ls];
    if (upd >= 0) {
      float d = 0.f;
#pragma unroll
      for (int g = 0; g < JW / 4; ++g) {  // dbv is zero past jn
        const float4 b = db4[g];
        d = fmaf(av[4 * g], b.x, d);
        d = fmaf(av[4 * g + 1], b.y, d);
        d = fmaf(av[4 * g + 2], b.z, d);
        d = fmaf(av[4 * g + 3], b.w, d);
      }
      for (uint32_t g = JW / 4; g < jn4; ++g) {
        const float4 t = la4[g * capa + ls], b = db4[g];
        d = fmaf(t.x, b.x, d);
        d = fmaf(t.y, b.y, d);
        d = fmaf(t.z, b.z, d);
        d = fmaf(t.w, b.w, d);
      }
      xh = fmaf(c_upd[ls], d, xh);
      lxh[ls] = xh;
    }
    const float t = c_rcn[ls] * (xh - lx[ls]);
#pragma unroll
    for (int q = 0; q < JW; ++q) v[q] = fmaf(t, av[q], v[q]);
  }
  if constexpr (REG) {
    static_assert(JW == 32, "register-resident samples take the whole row in one pass");
    const uint32_t ls = nla + threadIdx.x;
    if (ls < nloc) {
      float xh = lxh[ls];
      if (upd >= 0) {
        float d = 0.f;
#pragma unroll
        for (int g = 0; g < 8; ++g) {  // areg and dbv are zero past jn
          const float4 b = db4[g];
          d = fmaf(areg[4 * g], b.x, d);
          d = fmaf(areg[4 * g + 1], b.y, d);
          d = fmaf(areg[4 * g + 2], b.z, d);
          d = fmaf(areg[4 * g + 3], b.w, d);
        }
        xh = fmaf(c_upd[ls], d, xh);
        lxh[ls] = xh;
      }
      const float t = c_rcn[ls] * (xh - lx[ls]);
#pragma unroll
      for (int q = 0; q < 32; ++q) v[q] = fmaf(t, areg[q], v[q]);
    }
  }
}

// The CTA's partial of V_rcn, columns j0.. in chunks of JW, into wpart[warp][j].
template <int JW, bool REG>
__device__ __forceinline__ void column_partials(const float4* la, uint32_t capa, uint32_t nla, const float* c_rcn,
                                                const float* c_upd, float* lxh, const float* lx, const float* dbv,
                                                uint32_t nloc, uint32_t jn, int upd, double* wrow, int lane,
                                                const float (&areg)[32]) {
  for (uint32_t j0 = 0; j0 < jn; j0 += JW) {
    float v[JW];
#pragma unroll
    for (int q = 0; q < JW; ++q) v[q] = 0.f;
    column_pass<JW, REG>(la, capa, nla, c_rcn, c_upd, lxh, lx, dbv, nloc, jn, j0 == 0 ? upd : -1, j0, v, areg);
    const float w = warp_reduce<JW>(v, lane);
    if (lane < JW && j0 + lane < jn) wrow[j0 + lane] = static_cast<double>(w);
  }
}

// Values j0 .. j0+7 of a factor row (zeros past J): two 128-bit loads when the row
// is 16-B aligned (J % 4 == 0), else 8 independent scalar loads.
__device__ __forceinline__ void load_row8(const float* __restrict__ arow, uint32_t j0, uint32_t J, float (&av)[8]) {
  if ((J & 3u) == 0) {
    const float4 lo = __ldg(reinterpret_cast<const float4*>(arow + j0));
    const float4 hi = j0 + 4 < J ? __ldg(reinterpret_cast<const float4*>(arow + j0 + 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
    av[0] = lo.x, av[1] = lo.y, av[2] = lo.z, av[3] = lo.w;
    av[4] = hi.x, av[5] = hi.y, av[6] = hi.z, av[7] = hi.w;
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) av[q] = j0 + q < J ? __ldg(arow + j0 + q) : 0.f;
  }
}

constexpr int kCoreBlock = 512;
constexpr int kCoreTraceCap = 1024;

template <int RP, bool REG>
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
  double* wpart = reinterpret_cast<double*>(bs_base + ((off + 3) & ~3u));  // nwarps x js (16-B aligned)
  float* dbv = reinterpret_cast<float*>(wpart + ((nwarps * a.js + 1) & ~1u));  // max(ja, 32), 16-B aligned
  const uint32_t dbn = a.ja > 32 ? a.ja : 32;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int ti = 0;
#define CORE_TRACE()                                                    \
  do {                                                                  \
    if (a.trace && blockIdx.x == a.trace_cta && tid == 0 && ti < kCoreTraceCap) a.trace[ti++] = clock64(); \
  } while (0)
  CORE_TRACE();
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
  // (cap is a multiple of 4, so every piece below stays 16-B aligned)
  float4* la;
  float *lc, *lxh, *lx;
  // semi: a ring of three columns of c in shared memory -- column rc of this step, rc - 1
  // (its x-hat fold) and rc + 1, which cp.async fetches from the scratch during this step,
  // so no pass waits on an L2 round trip (they made the CTAs' passes uneven: 7k-15k cycles)
  float* ccol = nullptr;
  uint32_t capa = a.cap, capc = a.cap, nla = nloc;  // row strides of la / lc, samples held in la
  const uint32_t ja4 = a.ja >> 2;
  // the global scratch slice of this CTA: a_s groups [g * cap + ls]
  float4* ga = reinterpret_cast<float4*>(a.sa + static_cast<uint64_t>(blockIdx.x) * a.cap * a.ja);
  if (a.local == 1) {
    float* base = dbv + dbn;
    la = reinterpret_cast<float4*>(base);
    lc = base + static_cast<uint64_t>(a.cap) * a.ja;
    lxh = lc + static_cast<uint64_t>(a.cap) * RP;
    lx = lxh + a.cap;
  } else {
    const uint64_t cb = static_cast<uint64_t>(blockIdx.x) * a.cap;
    la = ga;
    lc = a.sc + cb * RP;
    lxh = a.sxh + cb;
    lx = a.sx + cb;
    if (a.local == 2) {  // semi: xhat, x and the first nsm samples' a_s in shared memory
      lxh = dbv + dbn;
      lx = lxh + a.cap;
      la = reinterpret_cast<float4*>(lx + a.cap);
      capa = a.nsm;
      nla = nloc < a.nsm ? nloc : a.nsm;
      if (a.ring) ccol = reinterpret_cast<float*>(la + static_cast<uint64_t>(a.nsm) * ja4);
    }
  }
  float areg[32];
#pragma unroll
  for (int q = 0; q < 32; ++q) areg[q] = 0.f;
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
      // narrow rows: all coordinates and the value first (one round trip), then the
      // rows; with RP > 16 the accumulators leave no registers for that
      constexpr bool kPre = RP <= 16;
      uint32_t ik[kMaxOrder];
      if constexpr (kPre) {
#pragma unroll
        for (int k = 0; k < kMaxOrder; ++k)
          ik[k] = k < a.P.order ? __ldg(a.rec_idx + static_cast<uint64_t>(k) * a.nnz + e) : 0u;
      }
      const float xval = __ldg(a.rec_val + e);
      float c[RP];
#pragma unroll
      for (int r = 0; r < RP; ++r) c[r] = 1.f;
      uint32_t in_ = 0;
      for (int k = 0; k < a.P.order; ++k) {
        uint32_t ikk = 0;
        if constexpr (kPre) {  // ik[k] without a dynamically indexed (local-memory) array
#pragma unroll
          for (int q = 0; q < kMaxOrder; ++q) ikk = q == k ? ik[q] : ikk;
        } else {
          ikk = a.rec_idx[static_cast<uint64_t>(k) * a.nnz + e];
        }
        if (k == n) {
          in_ = ikk;
          continue;
        }
        if (a.q_rows && k > n) {
          // B^(k) has not been stepped yet in this phase, so the device's Q^(k) row
          // (refreshed after the last core phase, rewritten by the factor finalisers)
          // is a^(k) B^(k): one row gather instead of a J x R contraction
          const float4* qrow = reinterpret_cast<const float4*>(a.P.Q[k] + static_cast<uint64_t>(ikk) * RP);
#pragma unroll
          for (int r4 = 0; r4 < RP / 4; ++r4) {
            const float4 q = __ldg(qrow + r4);
            c[4 * r4] *= q.x, c[4 * r4 + 1] *= q.y, c[4 * r4 + 2] *= q.z, c[4 * r4 + 3] *= q.w;
          }
          continue;
        }
        const float* arow = a.P.A[k] + static_cast<uint64_t>(ikk) * a.P.J[k];
        float d[RP];
#pragma unroll
        for (int r = 0; r < RP; ++r) d[r] = 0.f;
        // the row in groups of 8 values, all 8 loads issued before the FMAs (one
        // memory round trip per group instead of one per value; j ascending as before)
        for (uint32_t j0 = 0; j0 < a.P.J[k]; j0 += 8) {
          float av[8];
          load_row8(arow, j0, a.P.J[k], av);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (j0 + q < a.P.J[k]) {
#pragma unroll
              for (int r = 0; r < RP; ++r) d[r] = fmaf(av[q], bs_base[bso[k] + (j0 + q) * RP + r], d[r]);
            }
        }
#pragma unroll
        for (int r = 0; r < RP; ++r) c[r] *= d[r];
      }
      const float* arow = a.P.A[n] + static_cast<uint64_t>(in_) * jn;
      float p[RP];
      if (a.q_rows) {  // the own mode's row of Q^(n) is a_s B^(n) at the start of the mode
        const float4* qrow = reinterpret_cast<const float4*>(a.P.Q[n] + static_cast<uint64_t>(in_) * RP);
#pragma unroll
        for (int r4 = 0; r4 < RP / 4; ++r4) {
          const float4 q = __ldg(qrow + r4);
          p[4 * r4] = q.x, p[4 * r4 + 1] = q.y, p[4 * r4 + 2] = q.z, p[4 * r4 + 3] = q.w;
        }
      } else {
#pragma unroll
        for (int r = 0; r < RP; ++r) p[r] = 0.f;
      }
      for (uint32_t j0 = 0; j0 < jn; j0 += 8) {
        float av[8];
        load_row8(arow, j0, jn, av);
        {  // av is zero past jn
          float4* dst = ls < nla ? la + (j0 >> 2) * capa + ls : ga + (j0 >> 2) * a.cap + ls;
          const uint32_t dstride = ls < nla ? capa : a.cap;
          dst[0] = make_float4(av[0], av[1], av[2], av[3]);
          if (j0 + 4 < jn) dst[dstride] = make_float4(av[4], av[5], av[6], av[7]);
        }
        if (!a.q_rows) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (j0 + q < jn) {
#pragma unroll
              for (int r = 0; r < RP; ++r) p[r] = fmaf(av[q], bs_base[bso[n] + (j0 + q) * RP + r], p[r]);
            }
        }
      }
      float xh = 0.f;
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        xh = fmaf(c[r], p[r], xh);
        lc[r * capc + ls] = c[r];
      }
      if (ccol) ccol[ls] = c[0];
      lxh[ls] = xh;
      lx[ls] = xval;
    }
    __syncthreads();
    if constexpr (REG) {  // thread t takes over the a_s of sample nla + t
      const uint32_t ls = nla + tid;
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const float4 t = ls < nloc && static_cast<uint32_t>(4 * g) < jn ? ga[g * a.cap + ls]
                                                                        : make_float4(0.f, 0.f, 0.f, 0.f);
        areg[4 * g] = t.x, areg[4 * g + 1] = t.y, areg[4 * g + 2] = t.z, areg[4 * g + 3] = t.w;
      }
    }
    CORE_TRACE();  // mode setup done

    int upd = -1;  // column whose step is still to be folded into xhat
    for (uint32_t rc = 0; rc < a.P.R; ++rc, ++step) {
      // ---- partial V over this CTA's slice: V_j = sum_s c_{s,rc} (xhat_s - x_s) a_{s,j},
      // fused with the xhat refresh for the previous column's step
      ulonglong2* part = a.part + static_cast<uint64_t>(step & 1) * gridDim.x * a.js;
      const uint32_t stamp = a.stamp0 + step + 1;
      const float* c_rcn = lc + rc * capc;
      const float* c_upd = lc + (rc ? rc - 1 : 0) * capc;
      if (ccol) {
        c_rcn = ccol + (rc % 3) * a.cap;
        c_upd = ccol + ((rc + 2) % 3) * a.cap;
        if (rc + 1 < a.P.R) {
          const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(ccol + ((rc + 1) % 3) * a.cap));
          const float* src = lc + (rc + 1) * capc;
          for (uint32_t i = tid * 4; i < nloc; i += blockDim.x * 4)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + i * 4), "l"(src + i) : "memory");
          asm volatile("cp.async.commit_group;" ::: "memory");
        }
      }
      if constexpr (REG)
        column_partials<32, true>(la, capa, nla, c_rcn, c_upd, lxh, lx, dbv, nloc, jn, upd, wpart + warp * a.js,
                                  lane, areg);
      else if (jn <= 8)
        column_partials<8, false>(la, capa, nla, c_rcn, c_upd, lxh, lx, dbv, nloc, jn, upd, wpart + warp * a.js,
                                  lane, areg);
      else if (jn <= 16)
        column_partials<16, false>(la, capa, nla, c_rcn, c_upd, lxh, lx, dbv, nloc, jn, upd, wpart + warp * a.js,
                                   lane, areg);
      else
        column_partials<32, false>(la, capa, nla, c_rcn, c_upd, lxh, lx, dbv, nloc, jn, upd, wpart + warp * a.js,
                                   lane, areg);
      CORE_TRACE();  // warp partials done (warp 0)
      __syncthreads();
      CORE_TRACE();  // all warps done
      if (tid < static_cast<int>(jn)) {
        double acc = 0.0;
        for (int w = 0; w < nwarps; ++w) acc += wpart[w * a.js + tid];
        st_stamped(part + static_cast<uint64_t>(tid) * gridDim.x + blockIdx.x, acc, stamp);  // [j][cta]
      }
      CORE_TRACE();  // partial stored
      if (a.grid_sync) grid.sync();
      // ---- reducers: column j of V belongs to one warp of the grid (CTA j % grid).  It
      // sums the CTA partials in CTA order (fixed lane striding + butterfly), takes the
      // sgd_step on b_{j,rc} and publishes the new value
      // wide J: every CTA polls its own copy of the new column.  148 CTAs polling the same
      // lines serialise at their L2 slice (J = 32: store -> all-see ~6k cycles against ~1.5k
      // for a line with one reader), so the reducer stores one word per CTA; with J < 16 the
      // shared words are faster (config 2 core 0.163 vs 0.175 ms, config 3 0.364 vs 0.374)
      unsigned long long* res = a.res + static_cast<uint64_t>(step & 1) * gridDim.x * a.js;
      const uint64_t res_stride = a.res_copies ? a.js : 0;
      for (uint32_t j = blockIdx.x + warp * gridDim.x; j < jn; j += nwarps * gridDim.x) {
        const ulonglong2* pj = part + static_cast<uint64_t>(j) * gridDim.x;
        double V = 0.0;
        int rounds = 0;
        for (unsigned b0 = 0; b0 < gridDim.x; b0 += 160) {
          // up to five slots per lane in flight; a slot is ready when both of
          // its words carry this step's stamp
          ulonglong2 w[5];
          unsigned pending = 0;
#pragma unroll
          for (int q = 0; q < 5; ++q)
            if (b0 + q * 32 + lane < gridDim.x) pending |= 1u << q;
          while (pending) {
            ++rounds;
#pragma unroll
            for (int q = 0; q < 5; ++q)
              if (pending & (1u << q)) w[q] = ld_stamped(pj + b0 + q * 32 + lane);
#pragma unroll
            for (int q = 0; q < 5; ++q)
              if ((pending & (1u << q)) && static_cast<uint32_t>(w[q].x >> 32) == stamp &&
                  static_cast<uint32_t>(w[q].y >> 32) == stamp)
                pending &= ~(1u << q);
          }
#pragma unroll
          for (int q = 0; q < 5; ++q)
            if (b0 + q * 32 + lane < gridDim.x)
              V += __longlong_as_double(static_cast<long long>((w[q].y << 32) | (w[q].x & 0xffffffffull)));
        }
        if (a.trace && blockIdx.x == a.trace_cta && tid == 0 && ti < kCoreTraceCap) {
          a.trace[kCoreTraceCap + ti] = rounds;
          a.trace[ti++] = clock64();  // partials polled
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) V += __shfl_xor_sync(0xffffffffu, V, o);
        {  // every lane forms the same step (V is the warp-wide sum in all lanes)
          double w = static_cast<double>(bs_base[bso[n] + j * RP + rc]);
          int bad = (!isfinite(w) ? 1 : 0) | (!isfinite(V) ? 2 : 0);
          w -= a.lr * (V * inv_m + a.reg * w);
          const float bnew = static_cast<float>(w);
          bad |= !isfinite(bnew) ? 4 : 0;
          if (bad && lane == 0) atomicOr(a.flag, bad);
          const unsigned long long word =
              (static_cast<unsigned long long>(stamp) << 32) | static_cast<unsigned long long>(__float_as_uint(bnew));
          for (unsigned c = lane; c < (a.res_copies ? gridDim.x : 1u); c += 32)
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(res + c * res_stride + j), "l"(word) : "memory");
        }
      }
      CORE_TRACE();  // reducer role done
      // ---- every CTA: take the new column (identical everywhere) and the step delta
      if (tid < static_cast<int>(jn)) {
        unsigned long long word;
        do {
          asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];"
                       : "=l"(word)
                       : "l"(res + blockIdx.x * res_stride + tid)
                       : "memory");
        } while (static_cast<uint32_t>(word >> 32) != stamp);
        const float bnew = __uint_as_float(static_cast<uint32_t>(word));
        const float bold = bs_base[bso[n] + tid * RP + rc];
        dbv[tid] = bnew - bold;
        bs_base[bso[n] + tid * RP + rc] = bnew;
      }
      if (ccol) asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
      CORE_TRACE();  // column stepped
      upd = static_cast<int>(rc);
    }
  }

  // ---- write back B (identical in every CTA) and refresh Q^(k) = A^(k) B^(k)
  if (blockIdx.x == 0)
    for (int k = 0; k < a.P.order; ++k)
      for (uint32_t i = tid; i < a.P.J[k] * a.P.R; i += blockDim.x)
        a.P.B[k][i] = bs_base[bso[k] + (i / a.P.R) * RP + (i % a.P.R)];
  CORE_TRACE();
  if (!a.q_refresh) return;
  float* stage = dbv + dbn + warp * kQStage;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * nwarps + warp;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * nwarps;
  for (int k = 0; k < a.P.order; ++k)
    if (a.q_refresh >> k & 1)
      q_rows_tiled<RP>(a.P.A[k], a.P.Q[k], a.P.J[k], bs_base + bso[k], a.P.dims[k], gw, nw, stage, lane);
  __syncthreads();
  CORE_TRACE();
#undef CORE_TRACE
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

// Launch geometry and where the per-sample state of a CTA's slice lives:
//   local  everything in shared memory (configs 2, 3);
//   semi   a_s (J floats per sample, read by every column step) in shared memory, and when that
//          does not hold the whole slice, the a_s of up to one more sample per thread in registers
//          (J <= 32, RP >= 16 builds); xhat and x in shared memory; c_{s,r} (two columns read per
//          step) in the L2-resident global scratch (configs 4, 5: the passes were L2-bandwidth bound
//          with a_s in global memory, 226 KB per CTA and step at config 5);
//   global everything in the global scratch.
// SGDT_CORE_STATE=global|semi|local forces a choice when it fits (A/B).
struct CoreGeom {
  int grid;
  size_t smem;
  bool reg;
};

template <int RP>
int core_geometry(Session& s, CoreArgs& a, CoreGeom& g) {
  const int block = kCoreBlock;
  size_t bs_floats = 0;
  for (int k = 0; k < s.order; ++k) bs_floats += s.J[k] * RP;
  size_t smem = ((bs_floats + 3) & ~size_t(3)) * sizeof(float) +
                ((static_cast<size_t>(block / 32) * a.js + 1) & ~size_t(1)) * sizeof(double) +
                (a.ja > 32 ? a.ja : 32) * sizeof(float);
  // one CTA per SM keeps the exchange cheap; small batches use fewer CTAs
  uint64_t want = (a.m + 127) / 128;
  if (want < 1) want = 1;
  int grid = static_cast<int>(want < static_cast<uint64_t>(s.num_sms) ? want : s.num_sms);
  if (a.q_refresh && grid < s.num_sms) {
    uint64_t rows = 0;
    for (int k = 0; k < s.order; ++k)
      if (a.q_refresh >> k & 1) rows += s.dims[k];
    if (rows > static_cast<uint64_t>(grid) * block * 8) grid = s.num_sms;
  }
  if (const char* e = std::getenv("SGDT_CORE_GRID")) {  // diagnostics (A/B runs)
    const int gg = std::atoi(e);
    if (gg >= 1 && gg <= s.num_sms) grid = gg;
  }
  a.cap = (static_cast<uint32_t>((a.m + grid - 1) / grid) + 3u) & ~3u;  // float4-aligned pieces
  constexpr size_t kBudget = 200 * 1024;
  const size_t local = static_cast<size_t>(a.cap) * (a.ja + RP + 2) * sizeof(float);
  const size_t stage = static_cast<size_t>(block / 32) * kQStage * sizeof(float);  // tail Q refresh
  const char* force = std::getenv("SGDT_CORE_STATE");
  a.local = 0;
  a.nsm = 0;
  a.ring = 1;
  if (const char* e = std::getenv("SGDT_CORE_RING")) a.ring = std::atoi(e) != 0;
  // Q row gathers in the sample setup: every Q^(k) is current when a core phase starts
  // (set_model, the last core phase's refresh, the factor finalisers); SGDT_CORE_QROWS=0: A/B
  a.q_rows = 1;
  if (const char* e = std::getenv("SGDT_CORE_QROWS")) a.q_rows = std::atoi(e) != 0;
  a.res_copies = a.js >= 16;  // config 4 (J = 16): 0.463 -> 0.451 ms, config 5 (J = 32): 2.17 -> 1.96 ms
  if (const char* e = std::getenv("SGDT_CORE_RES")) a.res_copies = e[0] == 'p';  // percta | shared (A/B)
  g.reg = false;
  size_t state = stage;
  if (smem + (local > stage ? local : stage) <= kBudget && !(force && (force[0] == 'g' || force[0] == 's'))) {
    a.local = 1;
    state = local > stage ? local : stage;
  } else if (!(force && force[0] == 'g')) {
    // xhat, x and the three-column ring of c; the semi state may use all but a margin of the
    // 227 KB an SM offers one CTA
    constexpr size_t kSemiBudget = 216 * 1024;
    const size_t fixed = smem + 5 * static_cast<size_t>(a.cap) * sizeof(float);
    if (fixed < kSemiBudget) {
      uint64_t nsm = ((kSemiBudget - fixed) / (a.ja * sizeof(float))) & ~uint64_t(3);
      if (const char* e = std::getenv("SGDT_CORE_NSM")) {  // tests: force register-resident samples
        const uint64_t lim = std::strtoull(e, nullptr, 10);
        if (lim >= 1 && lim < nsm) nsm = (lim + 3) & ~uint64_t(3);
      }
      if (nsm >= a.cap) {
        nsm = a.cap;
      } else if (RP >= 16 && a.js <= 32 && nsm + block >= a.cap) {
        g.reg = true;
      } else {
        nsm = 0;
      }
      if (nsm) {
        a.local = 2;
        a.nsm = static_cast<uint32_t>(nsm);
        const size_t semi = (5 * static_cast<size_t>(a.cap) + nsm * a.ja) * sizeof(float);
        state = semi > stage ? semi : stage;
      }
    }
  }
  // exchange: stamped reducers when the passes run from shared memory (the step is
  // exchange-bound: config 2 0.186 -> 0.166 ms, config 3 0.381 -> 0.364 ms); with the
  // state in global memory the passes dominate and grid.sync() measured 1 % faster.
  // SGDT_CORE_SYNC=grid|red overrides.
  a.grid_sync = a.local == 0;
  if (const char* e = std::getenv("SGDT_CORE_SYNC")) a.grid_sync = e[0] == 'g';
  g.grid = grid;
  g.smem = smem + state;
  s.core_grid = grid;
  return SGDT_OK;
}

template <int RP, bool REG>
int core_launch_rp(Session& s, CoreArgs& a, size_t smem) {
  const int block = kCoreBlock;
  const int grid = s.core_grid;
  auto kern = core_kernel<RP, REG>;
  if (smem > 48 * 1024)
    SGDT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  SGDT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem));
  if (per_sm < 1) return fail(SGDT_ERR_INTERNAL, "core kernel does not fit on an SM");
  static long long* d_trace = nullptr;
  static int traced = 0;
  const bool trace = std::getenv("SGDT_CORE_TRACE") && traced < 4;
  if (trace && !d_trace) SGDT_CUDA(cudaMalloc(&d_trace, 2 * kCoreTraceCap * sizeof(long long)));
  a.trace = trace ? d_trace : nullptr;
  a.trace_cta = 0;
  if (const char* e = std::getenv("SGDT_CORE_TRACE_CTA")) a.trace_cta = std::atoi(e) % grid;
  if (trace) SGDT_CUDA(cudaMemsetAsync(d_trace, 0, 2 * kCoreTraceCap * sizeof(long long), s.stream));
  void* args[] = {&a};
  SGDT_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(grid), dim3(block),
                                        args, smem, s.stream));
  ++s.launches;
  if (trace) {  // diagnostics only: CTA 0's cycle counts between the phase boundaries
    static long long h[2 * kCoreTraceCap];
    SGDT_CUDA(cudaStreamSynchronize(s.stream));
    SGDT_CUDA(cudaMemcpy(h, d_trace, sizeof(h), cudaMemcpyDeviceToHost));
    ++traced;
    std::fprintf(stderr, "core trace (grid %d, state %d, nsm %u of cap %u, reg %d, sync %s, cycles since start):", grid,
                 a.local, a.nsm, a.cap, REG ? 1 : 0, a.grid_sync ? "grid" : "stamped");
    for (int i = 1; i < kCoreTraceCap && h[i]; ++i) {
      std::fprintf(stderr, " %lld", h[i] - h[0]);
      if (h[kCoreTraceCap + i]) std::fprintf(stderr, "(r%lld)", h[kCoreTraceCap + i]);
    }
    std::fprintf(stderr, "\n");
  }
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
  a.ja = (js + 3u) & ~3u;
  a.sa = s.cs_a;
  a.sc = s.cs_c;
  a.sxh = s.cs_xhat;
  a.sx = s.cs_x;
  a.part = s.cs_part;
  a.res = reinterpret_cast<unsigned long long*>(s.cs_part + 2ull * s.num_sms * js);
  {
    // stamps of this launch: core_stamp + 1 .. core_stamp + order * R; on wrap-around
    // the slots are cleared so that no stale stamp can match
    const uint32_t steps = static_cast<uint32_t>(s.order) * s.R;
    if (s.core_stamp > 0xffffffffu - steps - 1) {
      SGDT_CUDA(cudaMemsetAsync(s.cs_part, 0, 3ull * s.num_sms * js * sizeof(ulonglong2), s.stream));
      s.core_stamp = 0;
    }
    a.stamp0 = s.core_stamp;
    s.core_stamp += steps;
  }
  a.lr = h.lr;
  a.reg = h.reg;
  a.flag = s.flag;
  // wide modes with many rows are refreshed by the tensor-core kernel after the
  // cooperative kernel (sgdt_qrefresh_tc.cu); the rest at the kernel's tail
  int tc_modes = 0;
  for (int k = 0; k < s.order; ++k)
    if (q_refresh_tc_eligible(s, k)) tc_modes |= 1 << k;
  a.q_refresh = ((1 << s.order) - 1) & ~tc_modes;
  int rc = SGDT_ERR_CONFIG;
#define CORE_CALL(RP)                                                          \
  do {                                                                     \
    CoreGeom g{};                                                          \
    rc = core_geometry<RP>(s, a, g);                                       \
    if (rc == SGDT_OK) {                                                   \
      if constexpr (RP >= 16)                                              \
        rc = g.reg ? core_launch_rp<RP, true>(s, a, g.smem) : core_launch_rp<RP, false>(s, a, g.smem); \
      else                                                                 \
        rc = core_launch_rp<RP, false>(s, a, g.smem);                      \
    }                                                                      \
  } while (0)
  switch (s.RP) {
    case 4: CORE_CALL(4); break;
    case 8: CORE_CALL(8); break;
    case 12: CORE_CALL(12); break;
    case 16: CORE_CALL(16); break;
    case 20: CORE_CALL(20); break;
    case 24: CORE_CALL(24); break;
    case 28: CORE_CALL(28); break;
    case 32: CORE_CALL(32); break;
    default: return fail(SGDT_ERR_CONFIG, "unsupported R_core");
  }
#undef CORE_CALL
  if (rc != SGDT_OK) return rc;
  for (int k = 0; k < s.order; ++k)
    if (tc_modes >> k & 1)
      if (int r2 = launch_q_refresh_tc(s, k)) return r2;
  return SGDT_OK;
}

int launch_q_refresh(Session& s, int k) {
  if (q_refresh_tc_eligible(s, k)) return launch_q_refresh_tc(s, k);
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
