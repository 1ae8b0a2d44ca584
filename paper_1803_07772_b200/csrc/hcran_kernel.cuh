// hcran_kernel.cuh -- the per-instance solve kernel (one template, instantiated
// per launch shape in its own translation unit so the shapes compile in
// parallel: hcran_k256.cu, hcran_k512.cu).
//
// Execution model: a persistent grid of CTAs (a multiple of the SM count),
// each pulling whole channel realisations off an atomic work queue and
// solving them start to finish (Dinkelbach outer loop, SCA rounds, sweeps,
// repair) with the state in its own workspace slot.  Instances are
// independent, so there is no inter-CTA communication beyond the queue
// counter, and per-instance work imbalance (4-21 outer iterations, 60-900
// sweeps) is absorbed by the queue.
#pragma once
#include <cuda_runtime.h>
#include <new>
#include "hcran_solver.cuh"

namespace hcran {

typedef void (*KernelFn)(View, char*, size_t, int*, int, unsigned, size_t);

// Launch shapes (threads per CTA NT, threads per instance GT): a CTA of NT
// threads runs NT / GT independent instances, one per thread group, each
// pulling instances off the shared queue.  Several instances per SM keep the
// SM busy while one instance waits at its barriers or on serial phases.

template <int NT, int GT>
__global__ void __launch_bounds__(NT, 1)
    hcran_solve_kernel(View v, char* ws, size_t per_cta, int* counter, int mode, unsigned hot,
                       size_t hot_per) {
  // pass 1 (v.dense == 0): every instance, seated-pair SIC family, flags floor ties.
  // pass 2 (v.dense == 1): only instances flagged by pass 1, dense pair family.
  constexpr int G = NT / GT;
  __shared__ double red[2 * NT / 32];
  __shared__ Ctl ctl_s[G];
  __shared__ long long next_s[G];
  // The workspace pointer table (Work, ~1 KB) and the problem view are
  // uniform over the instance's threads: one copy in shared memory (broadcast
  // loads) instead of a per-thread copy in local memory, which at 512 threads
  // is ~0.7 MB of stack per SM and misses L1 on every array base fetch.
  __shared__ __align__(16) unsigned char work_s[G][sizeof(Work)];
  __shared__ View view_s;
  DevEx ex;
  ex.init(red, GT);
  Ctl& ctl = ctl_s[ex.grp];
  Work& W = *reinterpret_cast<Work*>(work_s[ex.grp]);
  extern __shared__ __align__(16) char hot_smem[];
  if (threadIdx.x == 0) view_s = v;
  if (ex.tid == 0) {
    new (&W) Work();
    const size_t slot = (size_t)blockIdx.x * G + ex.grp;
    W.layout(ws + slot * per_cta, v.M, v.K, v.N, v.dense != 0 || v.dense_ok != 0, GT / 32);
    if (hot) W.bind_hot(hot_smem + ex.grp * hot_per, hot, v.M, v.K, v.N);  // generic pointers
  }
  __syncthreads();
  Solver<DevEx> S(ex, view_s, W, ctl);
  for (;;) {
    if (ex.tid == 0) next_s[ex.grp] = (long long)atomicAdd(counter, 1);
    ex.sync();
    const long long q = next_s[ex.grp];
    ex.sync();
    if (q >= v.B) break;
    const long long b = v.order ? (long long)v.order[q] : q;
    if (v.flag_in && !v.flag_in[b]) continue;
    S.load_instance(b);
    if (mode == 0) S.dinkelbach(b);
    else if (mode == 1) S.fixed_e(b);
    else S.report(b);
    ex.sync();
  }
}


// one getter per instantiated shape (defined in hcran_k<NT>.cu), and its
// translation unit's phase-profiler counters (-DHCRAN_PROFILE builds)
KernelFn kernel_256_256();
KernelFn kernel_512_512();
void phase_cycles_256(unsigned long long* out32, int reset);
void phase_cycles_512(unsigned long long* out32, int reset);

}  // namespace hcran
