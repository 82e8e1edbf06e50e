// sgdt_qrefresh_tc.cu -- Q^(k) = A^(k) B^(k) for wide factors (J = 32, RP = 32)
// on the 5th-generation tensor cores: TMA tile loads, tcgen05.mma with the
// accumulator in tensor memory, a TMA tile store.
//
// Reference: the dense-core cache of TuckerModel (model.cpp:36-85,116-122) is
// replaced on the device by the Kruskal rows Q^(k) = A^(k) B^(k) (DESIGN.md
// section 3); this is the full refresh after a core phase (every B^(k) changed)
// and after a model upload.  It is the one GEMM-shaped step on the hot path:
// I_k x 32 times 32 x 32 per mode (config 5: 10M rows, 20.5 GFLOP, 2.56 GB).
//
// fp32 accuracy from TF32 products (3xTF32): every operand is split into
// hi = x with its low 13 mantissa bits cleared (exactly representable in TF32)
// and lo = x - hi (exact in fp32, at most 13 significant bits); then
//   A B ~= A_lo B_hi + A_hi B_lo + A_hi B_hi       (fp32 accumulation in TMEM)
// drops only lo x lo (2^-22 relative) and the rounding of lo to TF32 (2^-22),
// i.e. the result is within a few fp32 ulps of the fmaf chain of q_rows_tiled.
//
// One CTA = 128 threads works on tiles of 128 rows:
//   TMA load   A tile (128 x 32 fp32, 16 KB; rows are 128 B = one SWIZZLE_128B
//              span, so the tile lands in the K-major swizzled layout the MMA
//              descriptor names)
//   split      every thread splits 8 float4 in place (hi) and into a second
//              buffer (lo); the element-wise pass is layout-agnostic
//   MMA        one elected thread issues 3 x 4 tcgen05.mma.kind::tf32
//              (M = 128, N = 32, K = 8) into 32 TMEM columns, tcgen05.commit
//              arrives on an mbarrier
//   epilogue   the next tile's TMA load is issued; tcgen05.ld 32x32b.x32 gives
//              thread t row t of the tile, which it writes 128B-swizzled into
//              the (now free) lo buffer; one TMA tile store writes the 16 KB
// Several CTAs per SM (40 KB of shared memory, 32 TMEM columns each) overlap
// one another's loads, MMAs and stores; the kernel is HBM-bound (256 B per row).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "sgdt_internal.cuh"
#include "sgdt_qrows.cuh"

// the C-ABI handle is the session (as in sgdt_session.cu)
struct sgdt_session : sgdt::Session {};

namespace sgdt {

namespace {

constexpr int kTileRows = 128;
constexpr int kTcJ = 32;   // K of the product: J_k
constexpr int kTcN = 32;   // N of the product: RP
constexpr uint32_t kTileBytes = kTileRows * kTcJ * sizeof(float);  // 16 KB (A tile and Q tile)
constexpr uint32_t kTmemCols = 32;

// ---- PTX wrappers ---------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_tile(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_store_tile(const CUtensorMap* map, int c0, int c1, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"(map), "r"(c0), "r"(c1), "r"(src)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Shared-memory operand descriptor (tcgen05 matrix descriptor, K-major,
// SWIZZLE_128B): start address >> 4 in bits [0,14), leading byte offset >> 4 in
// [16,30) (not used by the swizzled K-major layouts; 1), stride byte offset >> 4
// in [32,46) (8 rows x 128 B = 1024 B between 8-row groups), descriptor version
// 1 in [46,48), layout type 2 (SWIZZLE_128B) in [61,64).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4) | (1ull << 16) | (static_cast<uint64_t>(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
// Instruction descriptor of kind::tf32: D fp32 (bits [4,6) = 1), A and B TF32
// ([7,10) = [10,13) = 2), both K-major (bits 15, 16 = 0), N >> 3 in [17,23),
// M >> 4 in [24,29).
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(kTcN >> 3) << 17) |
                            (static_cast<uint32_t>(kTileRows >> 4) << 24);

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

struct QTcSmem {
  // 1024-B aligned tiles (SWIZZLE_128B atoms are 8 rows x 128 B)
  float a_hi[kTileRows * kTcJ];  // TMA destination, split in place
  float a_lo[kTileRows * kTcJ];  // lo part; afterwards the staging of the Q tile
  float b_hi[kTcN * kTcJ];       // B^T (N x K, K-major), swizzled like a TMA tile
  float b_lo[kTcN * kTcJ];
  unsigned long long full_bar;   // TMA load landed
  unsigned long long mma_bar;    // MMAs of the tile retired
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(kTileRows) q_refresh_tc_kernel(const __grid_constant__ CUtensorMap map_a,
                                                                 const __grid_constant__ CUtensorMap map_q,
                                                                 const float* __restrict__ B, uint32_t R,
                                                                 uint32_t tiles) {
  extern __shared__ unsigned char smem_raw[];
  QTcSmem& sm = *reinterpret_cast<QTcSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t full_bar = smem_u32(&sm.full_bar), mma_bar = smem_u32(&sm.mma_bar);
  const uint32_t a_hi = smem_u32(sm.a_hi), a_lo = smem_u32(sm.a_lo);

  if (tid == 0) {
    mbar_init(full_bar, 1);
    mbar_init(mma_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // B^T split into hi / lo, element (n, k) = B[k][n] at n * 128 B + ((k / 4) ^ (n & 7)) * 16 B + (k % 4) * 4 B
  for (uint32_t i = tid; i < kTcN * kTcJ; i += kTileRows) {
    const uint32_t n = i % kTcN, k = i / kTcN;  // coalesced over n (B is J x R row-major)
    const float x = n < R ? B[k * R + n] : 0.f;
    const float hi = tf32_hi(x);
    const uint32_t o = n * kTcJ + (((k >> 2) ^ (n & 7u)) << 2) + (k & 3u);
    sm.b_hi[o] = hi;
    sm.b_lo[o] = x - hi;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  fence_async_smem();
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem_base;

  if (tid == 0 && blockIdx.x < tiles) {
    mbar_expect_tx(full_bar, kTileBytes);
    tma_load_tile(a_hi, &map_a, 0, static_cast<int>(blockIdx.x) * kTileRows, full_bar);
  }
  const uint64_t da_hi = umma_desc_sw128(a_hi), da_lo = umma_desc_sw128(a_lo);
  const uint64_t db_hi = umma_desc_sw128(smem_u32(sm.b_hi)), db_lo = umma_desc_sw128(smem_u32(sm.b_lo));

  uint32_t phase = 0;
  for (uint32_t t = blockIdx.x; t < tiles; t += gridDim.x, phase ^= 1u) {
    // the previous tile's TMA store must have read its staging (a_lo) before the split rewrites it
    if (tid == 0) tma_store_wait_read();
    mbar_wait(full_bar, phase);
    __syncthreads();
    // ---- split: hi in place, lo beside it (same offsets, so the swizzle is preserved)
    float4* h4 = reinterpret_cast<float4*>(sm.a_hi);
    float4* l4 = reinterpret_cast<float4*>(sm.a_lo);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 x = h4[tid + i * kTileRows];
      const float4 hi = make_float4(tf32_hi(x.x), tf32_hi(x.y), tf32_hi(x.z), tf32_hi(x.w));
      h4[tid + i * kTileRows] = hi;
      l4[tid + i * kTileRows] = make_float4(x.x - hi.x, x.y - hi.y, x.z - hi.z, x.w - hi.w);
    }
    fence_async_smem();  // generic-proxy writes -> the tensor core's async-proxy reads
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // K advances by 8 TF32 = 32 B inside the 128-B swizzle span: +2 in the address field.
      // The small terms first, the hi x hi term last.
#pragma unroll
      for (int k = 0; k < kTcJ / 8; ++k) umma_tf32(tmem, da_lo + 2 * k, db_hi + 2 * k, k > 0);
#pragma unroll
      for (int k = 0; k < kTcJ / 8; ++k) umma_tf32(tmem, da_hi + 2 * k, db_lo + 2 * k, 1);
#pragma unroll
      for (int k = 0; k < kTcJ / 8; ++k) umma_tf32(tmem, da_hi + 2 * k, db_hi + 2 * k, 1);
      umma_commit(mma_bar);  // implies tcgen05.fence::before_thread_sync
    }
    mbar_wait(mma_bar, phase);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // both A buffers are free: fetch the next tile while this one is written out
    if (tid == 0 && t + gridDim.x < tiles) {
      mbar_expect_tx(full_bar, kTileBytes);
      tma_load_tile(a_hi, &map_a, 0, static_cast<int>(t + gridDim.x) * kTileRows, full_bar);
    }
    // ---- epilogue: TMEM lane = tile row; warp w owns lanes 32 w .. 32 w + 31
    uint32_t q[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
          "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15]),
          "=r"(q[16]), "=r"(q[17]), "=r"(q[18]), "=r"(q[19]), "=r"(q[20]), "=r"(q[21]), "=r"(q[22]), "=r"(q[23]),
          "=r"(q[24]), "=r"(q[25]), "=r"(q[26]), "=r"(q[27]), "=r"(q[28]), "=r"(q[29]), "=r"(q[30]), "=r"(q[31])
        : "r"(tmem + (static_cast<uint32_t>(warp * 32) << 16))
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    // row tid of the Q tile, 16-B chunk c at (c ^ (row & 7)): the SWIZZLE_128B image the
    // TMA store expects; 8 consecutive lanes hit 8 different bank groups
    uint4* st4 = reinterpret_cast<uint4*>(sm.a_lo) + tid * 8;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      st4[c ^ (tid & 7)] = make_uint4(q[4 * c], q[4 * c + 1], q[4 * c + 2], q[4 * c + 3]);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    fence_async_smem();
    __syncthreads();
    if (tid == 0) tma_store_tile(&map_q, 0, static_cast<int>(t) * kTileRows, a_lo);
  }
  if (tid == 0) tma_store_wait_all();
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// rows x 32 fp32 row-major, boxes of 128 rows x 32 columns, SWIZZLE_128B
int make_row_tile_map(CUtensorMap* map, float* base, uint64_t rows) {
  EncodeTiledFn enc = encode_tiled_fn();
  if (!enc) return fail(SGDT_ERR_INTERNAL, "cuTensorMapEncodeTiled is not available from this driver");
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(kTcJ), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {kTcJ * sizeof(float)};
  const cuuint32_t box[2] = {kTcJ, kTileRows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SGDT_ERR_INTERNAL, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return SGDT_OK;
}

}  // namespace

// The tensor-core refresh serves modes with J_k = 32 and 32-wide Q rows and enough
// rows to fill the machine; SGDT_QTC=0 turns it off (A/B), SGDT_QTC=1 forces it
// for every eligible shape (tests).
bool q_refresh_tc_eligible(const Session& s, int k) {
  const char* e = std::getenv("SGDT_QTC");
  const int mode = e ? std::atoi(e) : -1;
  if (mode == 0) return false;
  if (s.J[k] != static_cast<uint32_t>(kTcJ) || s.RP != static_cast<uint32_t>(kTcN)) return false;
  if (s.dims[k] < 1 || s.dims[k] >= 0x7FFFFF00u) return false;  // TMA coordinates are int32
  return mode == 1 || s.dims[k] >= 65536u;
}

int launch_q_refresh_tc(Session& s, int k) {
  CUtensorMap map_a, map_q;
  if (int rc = make_row_tile_map(&map_a, s.P.A[k], s.dims[k])) return rc;
  if (int rc = make_row_tile_map(&map_q, s.P.Q[k], s.dims[k])) return rc;
  const uint32_t tiles = (s.dims[k] + kTileRows - 1) / kTileRows;
  const size_t smem = sizeof(QTcSmem) + 1024;
  // per device (a process may drive several), cheap host calls
  SGDT_CUDA(cudaFuncSetAttribute(q_refresh_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  SGDT_CUDA(cudaFuncSetAttribute(q_refresh_tc_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared));
  // resident CTAs per SM by shared memory (227 KB per SM, 1 KB reserved per CTA; 32 TMEM
  // columns and 64 registers x 128 threads per CTA are far from their limits)
  int per_sm = static_cast<int>((227u * 1024u) / (smem + 1024u));
  if (per_sm < 1) return fail(SGDT_ERR_INTERNAL, "tensor-core Q refresh does not fit on an SM");
  if (per_sm > 8) per_sm = 8;
  if (const char* e = std::getenv("SGDT_QTC_CTAS")) {  // diagnostics (A/B runs): resident CTAs per SM
    const int c = std::atoi(e);
    if (c >= 1 && c < per_sm) per_sm = c;
  }
  uint64_t grid = static_cast<uint64_t>(s.num_sms) * per_sm;
  if (grid > tiles) grid = tiles;
  q_refresh_tc_kernel<<<static_cast<unsigned>(grid), kTileRows, smem, s.stream>>>(map_a, map_q, s.P.B[k], s.R,
                                                                                   tiles);
  SGDT_CUDA(cudaGetLastError());
  ++s.launches;
  return SGDT_OK;
}

}  // namespace sgdt

extern "C" int sgdt_q_rows(sgdt_session* s, int mode, uint32_t row_lo, uint32_t row_hi, float* buf) {
  using namespace sgdt;
  if (!s || (!buf && row_hi > row_lo)) return fail(SGDT_ERR_DOMAIN, "null argument");
  if (mode < 0 || mode >= s->order || row_lo > row_hi || row_hi > s->dims[mode])
    return fail(SGDT_ERR_DOMAIN, "q_rows: range out of bounds");
  SGDT_CUDA(cudaSetDevice(s->device));
  if (row_hi == row_lo) return SGDT_OK;
  // device rows are RP wide (zero padded); the caller gets R_core values per row
  SGDT_CUDA(cudaMemcpy2DAsync(buf, s->R * sizeof(float), s->P.Q[mode] + static_cast<uint64_t>(row_lo) * s->RP,
                              s->RP * sizeof(float), s->R * sizeof(float), row_hi - row_lo,
                              cudaMemcpyDeviceToHost, s->stream));
  SGDT_CUDA(cudaStreamSynchronize(s->stream));
  return SGDT_OK;
}
