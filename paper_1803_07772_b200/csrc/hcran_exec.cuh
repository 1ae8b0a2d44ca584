// hcran_exec.cuh -- CTA execution policy for the per-instance solver.
//
// The solver (hcran_solver.cuh) is written as CTA-cooperative code with
// uniform control flow: every thread of the CTA walks the same Dinkelbach /
// round / sweep loops, data-parallel phases split their index ranges over
// threads (or over the lanes of one warp), and every control decision is read
// from a block reduction that all threads see.  `DevEx` is the sm_100a CTA.
//
// `HostEx` runs the identical source as a single "thread" on the CPU (1 warp
// of 1 lane).  It exists ONLY for the CPU unit tests that debug the kernel
// logic in the GPU-less build container (tests/test_emu_*.py); the product
// library never contains it and refuses to run without a GPU.
#pragma once
#include <stdint.h>
#include <math.h>

#if defined(__CUDACC__)
#define HD __host__ __device__
#define HDI __host__ __device__ __forceinline__
#else
#define HD
#define HDI inline
#endif

namespace hcran {

#if defined(__CUDACC__)
struct DevEx {
  int tid, nthr, warp, lane, nwarps;
  static constexpr int WS = 32;
  double* red;  // shared scratch, >= 2 * nwarps doubles
  __device__ void init(double* scratch) {
    tid = threadIdx.x;
    nthr = blockDim.x;
    warp = tid >> 5;
    lane = tid & 31;
    nwarps = nthr >> 5;
    red = scratch;
  }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
  __device__ __forceinline__ void wsync() const { __syncwarp(); }
  __device__ __forceinline__ bool any(bool p) const { return __syncthreads_or(p) != 0; }
  // named barrier over `count` threads (a warp group); id 1..15
  __device__ __forceinline__ void named_sync(int id, int count) const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
  }
  // warp-level (all lanes receive the result; fixed butterfly order)
  __device__ __forceinline__ double wsum(double v) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  }
  __device__ __forceinline__ double wmax(double v) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  }
  __device__ __forceinline__ int wmaxi(int v) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = ::max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  }
  __device__ __forceinline__ bool wany(bool p) const { return __any_sync(0xffffffffu, p) != 0; }
  // block-level (all threads receive the result; deterministic order)
  __device__ double sum(double v) const {
    v = wsum(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < nwarps; ++w) s += red[w];
    __syncthreads();
    return s;
  }
  __device__ double max(double v) const {
    v = wmax(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = red[0];
    for (int w = 1; w < nwarps; ++w) s = fmax(s, red[w]);
    __syncthreads();
    return s;
  }
};
#endif

struct HostEx {
  int tid = 0, nthr = 1, warp = 0, lane = 0, nwarps = 1;
  static constexpr int WS = 1;
  void sync() const {}
  void wsync() const {}
  bool any(bool p) const { return p; }
  void named_sync(int, int) const {}
  double wsum(double v) const { return v; }
  double wmax(double v) const { return v; }
  int wmaxi(int v) const { return v; }
  bool wany(bool p) const { return p; }
  double sum(double v) const { return v; }
  double max(double v) const { return v; }
};

}  // namespace hcran
