// Microbenchmark: cost per step of a grid-wide "sum J doubles over all CTAs, every
// CTA gets the result" exchange on one GPU, for the primitives the core kernel can
// use.  One cooperative launch, G CTAs x 64 threads, STEPS dependent steps; CTA 0
// reports mean cycles per step.  Build: nvcc -O3 -arch=sm_100a -o exchange_latency exchange_latency.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1);} } while (0)

constexpr int J = 10;
constexpr int STEPS = 400;

__device__ __forceinline__ void st128(ulonglong2* p, double x, unsigned stamp) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x), hi = (unsigned long long)stamp << 32;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(hi | (b & 0xffffffffull)), "l"(hi | (b >> 32)) : "memory");
}
__device__ __forceinline__ ulonglong2 ld128(const ulonglong2* p) {
  ulonglong2 w;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w.x), "=l"(w.y) : "l"(p) : "memory");
  return w;
}
__device__ __forceinline__ ulonglong2 ld128v(const ulonglong2* p) {
  ulonglong2 w;
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w.x), "=l"(w.y) : "l"(p) : "memory");
  return w;
}
__device__ __forceinline__ void st64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double unpack(ulonglong2 w) {
  return __longlong_as_double((long long)((w.y << 32) | (w.x & 0xffffffffull)));
}

// poll one stamped 64-bit word with four loads in flight, issued ~1/4 of a round trip apart
__device__ __forceinline__ unsigned long long poll64_staggered(const unsigned long long* p, unsigned stamp, int gap) {
  unsigned long long w[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    w[q] = ld64(p);
    const long long t = clock64();
    while (clock64() - t < gap) {}
  }
  for (;;) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if ((unsigned)(w[q] >> 32) == stamp) return w[q];
      w[q] = ld64(p);
    }
  }
}

// warp sums the G stamped slots of column j in CTA order; VOL selects ld.volatile
template <bool VOL>
__device__ double poll_sum(const ulonglong2* pj, unsigned G, unsigned stamp, int lane) {
  double V = 0.0;
  for (unsigned b0 = 0; b0 < G; b0 += 160) {
    ulonglong2 w[5];
    unsigned pending = 0;
#pragma unroll
    for (int q = 0; q < 5; ++q) if (b0 + q * 32 + lane < G) pending |= 1u << q;
    while (pending) {
#pragma unroll
      for (int q = 0; q < 5; ++q) if (pending & (1u << q)) w[q] = VOL ? ld128v(pj + b0 + q * 32 + lane) : ld128(pj + b0 + q * 32 + lane);
#pragma unroll
      for (int q = 0; q < 5; ++q)
        if ((pending & (1u << q)) && (unsigned)(w[q].x >> 32) == stamp && (unsigned)(w[q].y >> 32) == stamp) pending &= ~(1u << q);
    }
#pragma unroll
    for (int q = 0; q < 5; ++q) if (b0 + q * 32 + lane < G) V += unpack(w[q]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) V += __shfl_xor_sync(0xffffffffu, V, o);
  return V;
}

// variant 0: grid.sync + plain all-read-all.  1: stamped all-read-all.  2: stamped
// reducer (column j -> CTA j) + stamped result words.  3: as 2 with ld.volatile.
// 4: as 2, partials stored as two separate 64-bit words in two arrays (8-B polls).
// 5: counter: plain partials, __threadfence, atomicAdd; reducers poll the counter.
// 6: as 2 but the J reducers are the J warps of CTA 0... (64 threads: 2 warps, so j strided)
__global__ void __launch_bounds__(192) bench(int variant, ulonglong2* part, unsigned long long* res, double* plain,
                                            unsigned* counter, long long* out, double* sink, unsigned long long* res2) {
  cg::grid_group grid = cg::this_grid();
  const unsigned G = gridDim.x, cta = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ double v[J];
  double acc = 0.0;
  long long t0 = 0;
  for (int step = 0; step < STEPS + 20; ++step) {
    if (step == 20) t0 = clock64();
    const unsigned stamp = step + 1;
    ulonglong2* pp = part + (size_t)(step & 1) * G * J;
    double* pl = plain + (size_t)(step & 1) * G * J;
    unsigned long long* rr = res + (size_t)(step & 1) * J;
    const double mine = (double)(cta + 1) * 1e-3 + acc * 1e-9;
    if (variant == 0) {
      if (tid < J) pl[tid * G + cta] = mine + tid;
      grid.sync();
      for (int j = warp; j < J; j += 6) {
        double V = 0.0;
        for (unsigned b = lane; b < G; b += 32) V += __ldcg(pl + j * G + b);
        for (int o = 16; o > 0; o >>= 1) V += __shfl_xor_sync(0xffffffffu, V, o);
        if (lane == 0) v[j] = V;
      }
    } else if (variant == 1) {
      if (tid < J) st128(pp + tid * G + cta, mine + tid, stamp);
      for (int j = warp; j < J; j += 6) {
        double V = poll_sum<false>(pp + j * G, G, stamp, lane);
        if (lane == 0) v[j] = V;
      }
    } else if (variant == 2 || variant == 3 || variant == 6) {
      if (tid < J) st128(pp + tid * G + cta, mine + tid, stamp);
      if (variant == 6) {
        if (cta == 0)
          for (int j = warp; j < J; j += 6) {
            double V = poll_sum<false>(pp + j * G, G, stamp, lane);
            if (lane == 0) st64(rr + j, ((unsigned long long)stamp << 32) | __float_as_uint((float)V));
          }
      } else if (warp == 0 && cta < J) {
        double V = variant == 3 ? poll_sum<true>(pp + cta * G, G, stamp, lane) : poll_sum<false>(pp + cta * G, G, stamp, lane);
        if (lane == 0) st64(rr + cta, ((unsigned long long)stamp << 32) | __float_as_uint((float)V));
      }
      if (tid < J) {
        unsigned long long w;
        do { w = ld64(rr + tid); } while ((unsigned)(w >> 32) != stamp);
        v[tid] = __uint_as_float((unsigned)w);
      }
    } else if (variant == 7 || variant == 8) {
      // as 2; receivers poll with staggered loads; 8: reducers also re-poll without waiting for a whole round
      if (tid < J) st128(pp + tid * G + cta, mine + tid, stamp);
      if (warp == 0 && cta < J) {
        double V = 0.0;
        if (variant == 8) {
          for (unsigned b = lane; b < G; b += 32) {
            ulonglong2 w0 = ld128(pp + cta * G + b);
            long long t = clock64();
            while (clock64() - t < 150) {}
            ulonglong2 w1 = ld128(pp + cta * G + b);
            for (;;) {
              if ((unsigned)(w0.x >> 32) == stamp && (unsigned)(w0.y >> 32) == stamp) { V += unpack(w0); break; }
              w0 = ld128(pp + cta * G + b);
              if ((unsigned)(w1.x >> 32) == stamp && (unsigned)(w1.y >> 32) == stamp) { V += unpack(w1); break; }
              w1 = ld128(pp + cta * G + b);
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) V += __shfl_xor_sync(0xffffffffu, V, o);
        } else {
          V = poll_sum<false>(pp + cta * G, G, stamp, lane);
        }
        if (lane == 0) st64(rr + cta, ((unsigned long long)stamp << 32) | __float_as_uint((float)V));
      }
      if (tid < J) {
        const unsigned long long w = poll64_staggered(rr + tid, stamp, 150);
        v[tid] = __uint_as_float((unsigned)w);
      }
    } else if (variant == 10) {
      // as 2, but every CTA polls its own copy of the result words (res2[cta][16]): no hot line
      unsigned long long* r2 = res2 + (size_t)(step & 1) * G * 16;
      if (tid < J) st128(pp + tid * G + cta, mine + tid, stamp);
      if (warp == 0 && cta < J) {
        double V = poll_sum<false>(pp + cta * G, G, stamp, lane);
        const unsigned long long word = ((unsigned long long)stamp << 32) | __float_as_uint((float)V);
        for (unsigned b = lane; b < G; b += 32) st64(r2 + b * 16 + cta, word);
      }
      if (tid < J) {
        unsigned long long w;
        do { w = ld64(r2 + cta * 16 + tid); } while ((unsigned)(w >> 32) != stamp);
        v[tid] = __uint_as_float((unsigned)w);
      }
    } else if (variant == 11 || variant == 12) {
      // as 2, but a reducer is five warps, one slot per lane, combined in slot order through
      // shared memory (12: the result also goes to per-CTA copies)
      __shared__ double wsum[6];
      unsigned long long* r2 = res2 + (size_t)(step & 1) * G * 16;
      if (tid < J) st128(pp + tid * G + cta, mine + tid, stamp);
      if (cta < J && warp < 5) {
        const unsigned b = warp * 32 + lane;
        double V = 0.0;
        if (b < G) {
          ulonglong2 w;
          do { w = ld128(pp + cta * G + b); } while ((unsigned)(w.x >> 32) != stamp || (unsigned)(w.y >> 32) != stamp);
          V = unpack(w);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) V += __shfl_xor_sync(0xffffffffu, V, o);
        if (lane == 0) wsum[warp] = V;
      }
      if (cta < J) {
        __syncthreads();
        if (warp == 0) {
          const double V = wsum[0] + wsum[1] + wsum[2] + wsum[3] + wsum[4];
          const unsigned long long word = ((unsigned long long)stamp << 32) | __float_as_uint((float)V);
          if (variant == 11) { if (lane == 0) st64(rr + cta, word); }
          else for (unsigned b = lane; b < G; b += 32) st64(r2 + b * 16 + cta, word);
        }
      }
      if (tid < J) {
        unsigned long long w;
        if (variant == 11) do { w = ld64(rr + tid); } while ((unsigned)(w >> 32) != stamp);
        else do { w = ld64(r2 + cta * 16 + tid); } while ((unsigned)(w >> 32) != stamp);
        v[tid] = __uint_as_float((unsigned)w);
      }
    } else if (variant == 9) {
      // ping-pong between CTA 0 and CTA G-1: one-way latency of st.relaxed.gpu -> ld.relaxed.gpu (2 one-way trips per step)
      if (tid == 0) {
        if (cta == 0) {
          st64(rr, ((unsigned long long)stamp << 32) | 1u);
          unsigned long long w;
          do { w = ld64(rr + 1); } while ((unsigned)(w >> 32) != stamp);
        } else if (cta == G - 1) {
          unsigned long long w;
          do { w = ld64(rr); } while ((unsigned)(w >> 32) != stamp);
          st64(rr + 1, ((unsigned long long)stamp << 32) | 2u);
        }
      }
      if (tid < J) v[tid] = 1.f;
    } else if (variant == 5) {
      if (tid < J) pl[tid * G + cta] = mine + tid;
      __syncthreads();
      if (tid == 0) { __threadfence(); atomicAdd(counter, 1u); }
      if (warp == 0 && cta < J) {
        if (lane == 0) { while (*((volatile unsigned*)counter) < G * (unsigned)(step + 1)) {} __threadfence(); }
        __syncwarp();
        double V = 0.0;
        for (unsigned b = lane; b < G; b += 32) V += __ldcg(pl + cta * G + b);
        for (int o = 16; o > 0; o >>= 1) V += __shfl_xor_sync(0xffffffffu, V, o);
        if (lane == 0) st64(rr + cta, ((unsigned long long)stamp << 32) | __float_as_uint((float)V));
      }
      if (tid < J) {
        unsigned long long w;
        do { w = ld64(rr + tid); } while ((unsigned)(w >> 32) != stamp);
        v[tid] = __uint_as_float((unsigned)w);
      }
    }
    __syncthreads();
    acc += v[step % J];
    __syncthreads();
  }
  if (cta == 0 && tid == 0) out[0] = (clock64() - t0) / STEPS;
  if (tid == 0) sink[cta] = acc;
}

int main(int argc, char** argv) {
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp pr;
  CK(cudaGetDeviceProperties(&pr, dev));
  const int sms = pr.multiProcessorCount;
  ulonglong2* part; unsigned long long* res; double* plain; unsigned* counter; long long* out; double* sink;
  CK(cudaMalloc(&part, 2ull * sms * J * sizeof(ulonglong2)));
  CK(cudaMalloc(&res, 2ull * J * sizeof(unsigned long long)));
  CK(cudaMalloc(&plain, 2ull * sms * J * sizeof(double)));
  CK(cudaMalloc(&counter, 4));
  unsigned long long* res2;
  CK(cudaMalloc(&res2, 2ull * sms * 16 * 8));
  CK(cudaMalloc(&out, 8));
  CK(cudaMalloc(&sink, sms * sizeof(double)));
  const char* names[] = {"grid.sync + plain all-read-all", "stamped all-read-all", "stamped reducer (ld.relaxed.gpu 128)",
                         "stamped reducer (ld.volatile 128)", "-", "fence + counter reducer", "stamped reducer, all columns in CTA 0", "stamped reducer, staggered result polls", "stamped reducer, staggered polls on both hops", "ping-pong CTA 0 <-> CTA G-1 (two one-way trips)", "stamped reducer, per-CTA result copies", "stamped reducer, five warps per column", "five warps per column + per-CTA result copies"};
  int grids[] = {sms, 74, 32, 16};  // >= J: one reducer CTA per column
  for (int variant : {2, 10, 11, 12})
    for (int G : grids) {
      CK(cudaMemset(part, 0, 2ull * sms * J * sizeof(ulonglong2)));
      CK(cudaMemset(res, 0, 2ull * J * sizeof(unsigned long long)));
      CK(cudaMemset(counter, 0, 4));
      CK(cudaMemset(res2, 0, 2ull * sms * 16 * 8));
      void* args[] = {&variant, &part, &res, &plain, &counter, &out, &sink, &res2};
      CK(cudaLaunchCooperativeKernel((void*)bench, dim3(G), dim3(192), args, 0, 0));
      CK(cudaDeviceSynchronize());
      long long h;
      CK(cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost));
      printf("variant %d (%s) G=%d: %lld cycles/step\n", variant, names[variant], G, h); fflush(stdout);
    }
  return 0;
}
