// sgdt_qrows.cuh -- Q^(k) = A^(k) B^(k) row tiles, shared by the core kernels
// (the fused tail refresh of both core paths and the standalone refresh).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sgdt {

// The tensor-core refresh (sgdt_qrefresh_tc.cu: TMA tiles, tcgen05.mma kind::tf32
// as 3xTF32) serves modes with J = 32, 32-wide Q rows and many rows.
struct Session;
bool q_refresh_tc_eligible(const Session& s, int mode);
int launch_q_refresh_tc(Session& s, int mode);

// Q^(k) rows = A^(k) rows x B^(k), a warp per tile of 32 rows: the tile of A
// (contiguous, row stride J) is staged through a per-warp shared buffer so
// both the A reads and the Q writes are coalesced; lane l then forms row
// i0 + l in registers (j ascending, the same fmaf order as a per-row loop).
inline constexpr int kQStage = 32 * 33;  // floats per warp


template <int RP>
__device__ __forceinline__ void q_rows_tiled(const float* __restrict__ A, float* __restrict__ Q, uint32_t J,
                                             const float* bsk, uint64_t nrows, uint64_t gw, uint64_t nw,
                                             float* stage, int lane) {
  // Full tiles with J <= 32: the 32 J floats of a tile are contiguous and 16-B
  // aligned (i0 J 4 = 128 t J bytes), read as 8 J float4 (up to 8 per lane).  The
  // next tile's loads are issued as soon as this tile's registers have been
  // scattered to the stage, so they are in flight during the FMAs and the store.
  // (RP <= 16 only: with wider rows the next tile's 32 registers spill; measured
  // config 3 core 0.372 -> 0.364 ms, config 5 3.63 -> 3.70 ms when it was on for RP = 32)
  constexpr bool kPipe = RP <= 16;
  const uint32_t n4 = 8 * J, mJ = (65536u + J - 1) / J;
  float4 v[8];
  auto load_tile = [&](uint64_t tt) {
    const float4* src4 = reinterpret_cast<const float4*>(A + tt * 32 * J);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t x = u * 32 + lane;
      v[u] = x < n4 ? __ldg(src4 + x) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  if (kPipe && J <= 32 && gw * 32 + 32 <= nrows) load_tile(gw);
  for (uint64_t t = gw; t * 32 < nrows; t += nw) {
    const uint64_t i0 = t * 32;
    const uint32_t rows = nrows - i0 < 32 ? static_cast<uint32_t>(nrows - i0) : 32u;
    float q[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) q[r] = 0.f;
    for (uint32_t j0 = 0; j0 < J; j0 += 32) {
      const uint32_t jc = J - j0 < 32 ? J - j0 : 32u;
      __syncwarp();
      if (jc == J && rows == 32) {
        if (!kPipe) load_tile(t);
        // per-element scatter (row = e / J by a 16-bit reciprocal, exact for
        // e < 1024 and J <= 32)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t x = u * 32 + lane;
          if (x < n4) {
            const float e4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t g = x * 4 + i, row = (g * mJ) >> 16;
              stage[row * 33 + (g - row * J)] = e4[i];
            }
          }
        }
        if (kPipe && (t + nw) * 32 + 32 <= nrows) load_tile(t + nw);
      } else if (jc == J) {
        const float* src = A + i0 * J;  // the whole tile is contiguous
        for (uint32_t g = lane; g < rows * jc; g += 32) {
          const uint32_t row = g / jc;
          stage[row * 33 + (g - row * jc)] = __ldg(src + g);
        }
      } else {
        for (uint32_t g = lane; g < rows * jc; g += 32) {
          const uint32_t row = g / jc, col = g - row * jc;
          stage[row * 33 + col] = __ldg(A + (i0 + row) * J + j0 + col);
        }
      }
      __syncwarp();
      if (static_cast<uint32_t>(lane) < rows)
        for (uint32_t c = 0; c < jc; ++c) {
          const float av = stage[lane * 33 + c];
          const float4* br = reinterpret_cast<const float4*>(bsk + (j0 + c) * RP);  // RP % 4 == 0
#pragma unroll
          for (int r = 0; r < RP; r += 4) {
            const float4 b = br[r / 4];
            q[r] = fmaf(av, b.x, q[r]);
            q[r + 1] = fmaf(av, b.y, q[r + 1]);
            q[r + 2] = fmaf(av, b.z, q[r + 2]);
            q[r + 3] = fmaf(av, b.w, q[r + 3]);
          }
        }
    }
    __syncwarp();
    if (static_cast<uint32_t>(lane) < rows) {
#pragma unroll
      for (int r = 0; r < RP; ++r) stage[lane * (RP + 1) + r] = q[r];
    }
    __syncwarp();
    float* dst = Q + i0 * RP;
    for (uint32_t g = lane; g < rows * RP; g += 32) {
      const uint32_t row = g / RP;
      dst[g] = stage[row * (RP + 1) + (g - row * RP)];
    }
  }
}

}  // namespace sgdt
