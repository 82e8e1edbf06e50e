// sgdt_eval.cu -- K6: RMSE / MAE over a record copy.
//
// Reference: rmse_mae (eval.cpp:15-33) with predict (model.cpp:157-167):
//   xhat = a^(1)_{i_1} . (Ghat^(1) kron_{k>1} a^(k)_{i_k}) = sum_r prod_k Q^(k)[i_k, r]
// Streaming gather over the entries; per-thread fp64 sums of err^2 and |err|,
// fixed-shape block tree, per-block partials summed in block order by a
// single-CTA second pass -> deterministic for a given launch shape.
#include <cuda_runtime.h>

#include "sgdt_internal.cuh"

namespace sgdt {

namespace {

constexpr int kEvalBlock = 256;

template <int RP>
__global__ void __launch_bounds__(kEvalBlock) eval_kernel(Params P, const uint32_t* idx,
                                                          const float* val, uint64_t nnz,
                                                          double* part) {
  double sq = 0.0, ab = 0.0;
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < nnz;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    float c[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) c[r] = 1.f;
    for (int k = 0; k < P.order; ++k) {
      const uint32_t ik = __ldcs(idx + static_cast<uint64_t>(k) * nnz + e);
      const float4* q = reinterpret_cast<const float4*>(P.Q[k] + static_cast<uint64_t>(ik) * RP);
#pragma unroll
      for (int r = 0; r < RP; r += 4) {
        const float4 t = __ldg(q + r / 4);
        c[r] *= t.x;
        c[r + 1] *= t.y;
        c[r + 2] *= t.z;
        c[r + 3] *= t.w;
      }
    }
    float xh = 0.f;
#pragma unroll
    for (int r = 0; r < RP; ++r) xh += c[r];
    const double err = static_cast<double>(__ldcs(val + e)) - static_cast<double>(xh);
    sq = fma(err, err, sq);
    ab += fabs(err);
  }
  __shared__ double s_sq[kEvalBlock], s_ab[kEvalBlock];
  s_sq[threadIdx.x] = sq;
  s_ab[threadIdx.x] = ab;
  __syncthreads();
  for (int w = kEvalBlock / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s_sq[threadIdx.x] += s_sq[threadIdx.x + w];
      s_ab[threadIdx.x] += s_ab[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s_sq[0];
    part[2 * blockIdx.x + 1] = s_ab[0];
  }
}

__global__ void eval_final_kernel(const double* part, int nblocks, uint64_t nnz, double* out) {
  if (threadIdx.x != 0) return;
  double sq = 0.0, ab = 0.0;
  for (int b = 0; b < nblocks; ++b) {
    sq += part[2 * b];
    ab += part[2 * b + 1];
  }
  const double inv = 1.0 / static_cast<double>(nnz);
  out[0] = sqrt(sq * inv);
  out[1] = ab * inv;
}

template <int RP>
int eval_launch_rp(Session& s, const RecordCopy& rc, int nblocks) {
  eval_kernel<RP><<<nblocks, kEvalBlock, 0, s.stream>>>(s.P, rc.idx, rc.val, rc.nnz, s.ev_part);
  SGDT_CUDA(cudaGetLastError());
  return SGDT_OK;
}

}  // namespace

int launch_eval(Session& s, int which, double* rmse, double* mae) {
  NvtxRange range(which ? "sgdt:eval test" : "sgdt:eval train");
  const RecordCopy& rc = which == 0 ? s.train_rec : s.test_rec;
  if (rc.nnz == 0) return fail(SGDT_ERR_DOMAIN, "rmse_mae: empty entry set");
  uint64_t want = (rc.nnz + kEvalBlock * 8 - 1) / (kEvalBlock * 8);
  const int nblocks = static_cast<int>(want < static_cast<uint64_t>(s.num_sms) * 8 ? want : s.num_sms * 8);
  int r = SGDT_ERR_CONFIG;
  switch (s.RP) {
    case 4: r = eval_launch_rp<4>(s, rc, nblocks); break;
    case 8: r = eval_launch_rp<8>(s, rc, nblocks); break;
    case 12: r = eval_launch_rp<12>(s, rc, nblocks); break;
    case 16: r = eval_launch_rp<16>(s, rc, nblocks); break;
    case 20: r = eval_launch_rp<20>(s, rc, nblocks); break;
    case 24: r = eval_launch_rp<24>(s, rc, nblocks); break;
    case 28: r = eval_launch_rp<28>(s, rc, nblocks); break;
    case 32: r = eval_launch_rp<32>(s, rc, nblocks); break;
    default: return fail(SGDT_ERR_CONFIG, "unsupported R_core");
  }
  if (r) return r;
  eval_final_kernel<<<1, 32, 0, s.stream>>>(s.ev_part, nblocks, rc.nnz, s.ev_out);
  SGDT_CUDA(cudaGetLastError());
  s.launches += 2;
  SGDT_CUDA(cudaMemcpyAsync(s.h_ev_out, s.ev_out, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                            s.stream));
  SGDT_CUDA(cudaStreamSynchronize(s.stream));
  *rmse = s.h_ev_out[0];
  *mae = s.h_ev_out[1];
  return SGDT_OK;
}

}  // namespace sgdt
