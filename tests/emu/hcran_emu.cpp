// TEST-ONLY host emulation of the device solver (one CTA of one thread).
//
// Compiles paper_1803_07772_b200/csrc/hcran_solver.cuh with the HostEx policy
// so the CPU test-suite can debug the kernel's logic in the GPU-less build
// container and compare it with the oracle.  It is never loaded by the
// product package (which requires the sm_100a library) nor by bench.py.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include "../../paper_1803_07772_b200/csrc/hcran_solver.cuh"

using namespace hcran;

extern "C" int hcran_emu_solve(const hcran_problem_t* prob, const hcran_batch_in_t* in,
                               hcran_batch_out_t* out, int mode, int64_t first, int64_t count,
                               int dense_off) {
  Work W;
  size_t bytes = W.layout(nullptr, prob->M, prob->K, prob->N, true, 1);
  char* base = (char*)aligned_alloc(256, (bytes + 255) & ~size_t(255));
  if (!base) return -1;
  memset(base, 0, bytes);
  W.layout(base, prob->M, prob->K, prob->N, true, 1);
  View v;
  v.M = prob->M; v.K = prob->K; v.N = prob->N; v.L = prob->l_max;
  v.p_max = prob->p_max; v.mask = prob->p_mask; v.eta = prob->eta; v.w = prob->weights;
  v.sig = prob->sigma; v.static_power = prob->static_power; v.tol = prob->tol;
  v.B = in->B; v.gamma = in->gamma; v.elastic = in->elastic; v.min_rates = in->min_rates;
  v.e_fixed = in->e_fixed; v.warm_p = in->warm_p; v.out = *out;
  v.flag_int = nullptr;
  v.flag_in = nullptr;
  v.order = nullptr;
  HostEx ex;
  Ctl ctl;
  memset(&ctl, 0, sizeof(ctl));
  Solver<HostEx> S(ex, v, W, ctl);
  // seated-pair SIC family with floor ties re-run dense in place (dense_off: no
  // re-run, to expose the seated model); HCRAN_SIC_DENSE: dense everywhere
  v.dense = (prob->sic_mode == HCRAN_SIC_DENSE) ? 1 : 0;
  v.dense_ok = dense_off ? 0 : 1;
  for (int64_t b = first; b < first + count && b < in->B; ++b) {
    S.load_instance(b);
    if (mode == 0) S.dinkelbach(b);
    else if (mode == 1) S.fixed_e(b);
    else S.report(b);
  }
  free(base);
  return 0;
}
