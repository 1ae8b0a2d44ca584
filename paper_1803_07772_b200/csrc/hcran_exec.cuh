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
// One instance per thread group: `nthr` consecutive threads of the CTA (a
// warp group of 128, 256 threads, or the whole CTA) solve one instance, so a
// CTA keeps several independent instances in flight and the warps of one
// instance waiting at its barriers leave the SM to the others.  Group
// barriers are named barriers (id 1 + group); the whole-CTA case uses
// __syncthreads.
struct DevEx {
  int tid, nthr, warp, lane, nwarps, grp;
  static constexpr int WS = 32;
  double* red;  // shared scratch of this group, >= 2 * nwarps doubles
  __device__ void init(double* scratch, int gsize) {
    grp = threadIdx.x / gsize;
    tid = threadIdx.x - grp * gsize;
    nthr = gsize;
    warp = tid >> 5;
    lane = tid & 31;
    nwarps = nthr >> 5;
    red = scratch + grp * 2 * nwarps;
    whole = (int)blockDim.x == gsize;
  }
  bool whole;  // the instance owns the CTA (named barriers 1..15 are free)
  __device__ __forceinline__ void sync() const {
    if (nthr == (int)blockDim.x) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "r"(nthr) : "memory");
  }
  __device__ __forceinline__ void wsync() const { __syncwarp(); }
  // named barrier over `count` threads (a group of warps of one instance);
  // id 1..15 (only when the instance owns the whole CTA)
  __device__ __forceinline__ void gsync(int id, int count) const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
  }
  __device__ __forceinline__ bool any(bool p) const {
    if (nthr == (int)blockDim.x) return __syncthreads_or(p) != 0;
    const unsigned v = __any_sync(0xffffffffu, p);
    int* r = (int*)red;
    if (lane == 0) r[warp] = v ? 1 : 0;
    sync();
    int o = 0;
    for (int w = 0; w < nwarps; ++w) o |= r[w];
    sync();
    return o != 0;
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
  static __device__ __forceinline__ int fetch_add(int* p, int v) { return atomicAdd(p, v); }
  __device__ __forceinline__ int wbcast0(int v) const { return __shfl_sync(0xffffffffu, v, 0); }
  // group-level (all threads receive the result; deterministic order)
  __device__ double sum(double v) const {
    v = wsum(v);
    if (lane == 0) red[warp] = v;
    sync();
    double s = 0.0;
    for (int w = 0; w < nwarps; ++w) s += red[w];
    sync();
    return s;
  }
  __device__ double max(double v) const {
    v = wmax(v);
    if (lane == 0) red[warp] = v;
    sync();
    double s = red[0];
    for (int w = 1; w < nwarps; ++w) s = fmax(s, red[w]);
    sync();
    return s;
  }
};
#endif

struct HostEx {
  int tid = 0, nthr = 1, warp = 0, lane = 0, nwarps = 1, grp = 0;
  bool whole = false;
  double* red = nullptr;
  static constexpr int WS = 1;
  void sync() const {}
  void wsync() const {}
  void gsync(int, int) const {}
  bool any(bool p) const { return p; }
  double wsum(double v) const { return v; }
  double wmax(double v) const { return v; }
  int wmaxi(int v) const { return v; }
  bool wany(bool p) const { return p; }
  static int fetch_add(int* p, int v) { const int o = *p; *p += v; return o; }
  int wbcast0(int v) const { return v; }
  double sum(double v) const { return v; }
  double max(double v) const { return v; }
};

}  // namespace hcran
