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
  memset(&v, 0, sizeof(v));
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

// ---------------------------------------------------------------------------
// Localising harness: the device's budget multiplier on the
// reference's own `_budget_dual` inputs, with the reference's load function
// (scale.py:456-462: clip(num / (den + xi)) summed per head in numpy's pairwise
// order over the (K, N) block).
extern "C" void hcran_emu_budget(const double* num, const double* den, const double* mask,
                                 int M, int KN, const double* budget, const double* warm,
                                 double* xi_out, int* evals_out) {
  HostEx ex;
  double* buf = (double*)malloc(sizeof(double) * KN);
  for (int m = 0; m < M; ++m) {
    const double* nm = num + (size_t)m * KN;
    const double* dn = den + (size_t)m * KN;
    const double* mk = mask + (size_t)m * KN;
    auto clip = [](double n, double d, double k) -> double {
      double p = d > 0 ? n / d : k;
      if (n <= 0) return 0.0;
      return fmin(fmax(p, 0.0), k);
    };
    auto load1 = [&](double x) -> double {
      for (int i = 0; i < KN; ++i) buf[i] = clip(nm[i], dn[i] + x, mk[i]);
      return pw_sum(buf, KN);
    };
    auto load4 = [&](double x0, double x1, double x2, double x3, double& v0, double& v1,
                     double& v2, double& v3) {
      v0 = load1(x0); v1 = load1(x1); v2 = load1(x2); v3 = load1(x3);
    };
    auto aux0 = [&](double x, double& F, double& dF, double& F0) {
      double f = 0.0, df = 0.0;
      for (int i = 0; i < KN; ++i) {
        if (nm[i] <= 0) continue;
        const double d = dn[i] + x;
        if (!(d > 0)) { f += mk[i]; continue; }
        const double inv = 1.0 / d, q = nm[i] * inv;
        if (q >= mk[i]) f += mk[i];
        else { f += q; df -= q * inv; }
      }
      F = f;
      dF = df;
      F0 = load1(0.0);
    };
    int ev = 0;
    xi_out[m] = budget_multiplier(budget[m], warm[m], load1, load4, aux0, ev);
    evals_out[m] = ev;
  }
  free(buf);
  (void)ex;
}

// One sweep from a reference snapshot taken at the start of an SCA round
// (round-start powers p, carried multipliers xi / zeta / zeta_t[M][P][N] of the
// reference's oriented-pair layout): seating, bound coefficients and DC
// tangent at p, one sweep (v = 1); returns p_next, xi, zeta and the seated
// pairs' zeta_t (other entries untouched) and whether a floor tie was met.
extern "C" int hcran_emu_sweep_snapshot(const hcran_problem_t* prob, const hcran_batch_in_t* in,
                                        const double* p0, const double* xi0, const double* zeta0,
                                        double* zeta_t /* [M][P][N] in / out */, double* p_out,
                                        double* xi_out, double* zeta_out) {
  Work W;
  size_t bytes = W.layout(nullptr, prob->M, prob->K, prob->N, true, 1);
  char* base = (char*)aligned_alloc(256, (bytes + 255) & ~size_t(255));
  memset(base, 0, bytes);
  W.layout(base, prob->M, prob->K, prob->N, true, 1);
  View v;
  memset(&v, 0, sizeof(v));
  v.M = prob->M; v.K = prob->K; v.N = prob->N; v.L = prob->l_max;
  v.p_max = prob->p_max; v.mask = prob->p_mask; v.eta = prob->eta; v.w = prob->weights;
  v.sig = prob->sigma; v.static_power = prob->static_power; v.tol = prob->tol;
  v.B = in->B; v.gamma = in->gamma; v.elastic = in->elastic; v.min_rates = in->min_rates;
  v.dense = 0;
  v.dense_ok = 0;
  HostEx ex;
  Ctl ctl;
  memset(&ctl, 0, sizeof(ctl));
  Solver<HostEx> S(ex, v, W, ctl);
  const int M = prob->M, K = prob->K, N = prob->N, C = M * K * N, P = K * (K - 1) / 2;
  S.load_instance(0);
  S.ctx_setup(0.0);
  for (int c = 0; c < C; ++c) W.p[c] = p0[c];
  S.build_seating();
  S.pair_static();
  for (int m = 0; m < M; ++m) W.xi[m] = xi0[m];
  for (int k = 0; k < K; ++k) W.zeta[k] = zeta0[k];
  for (int col = 0; col < M * N; ++col) {
    const int m = col / N, n = col % N;
    for (int q = 0; q < W.npr[col]; ++q) {
      int a = W.s_user[col * SMAX + W.pr_s[col * NPAIR + q]];
      int b = W.s_user[col * SMAX + W.pr_w[col * NPAIR + q]];
      const int i = a < b ? a : b, j = a < b ? b : a;
      W.pr_zt[col * NPAIR + q] = zeta_t[((size_t)m * P + S.pair_q(i, j)) * N + n];
    }
  }
  S.round_start();
  S.sweep(1);
  for (int c = 0; c < C; ++c) p_out[c] = W.p[c];
  for (int m = 0; m < M; ++m) xi_out[m] = W.xi[m];
  for (int k = 0; k < K; ++k) zeta_out[k] = W.zeta[k];
  for (int col = 0; col < M * N; ++col) {
    const int m = col / N, n = col % N;
    for (int q = 0; q < W.npr[col]; ++q) {
      int a = W.s_user[col * SMAX + W.pr_s[col * NPAIR + q]];
      int b = W.s_user[col * SMAX + W.pr_w[col * NPAIR + q]];
      const int i = a < b ? a : b, j = a < b ? b : a;
      zeta_t[((size_t)m * P + S.pair_q(i, j)) * N + n] = W.pr_zt[col * NPAIR + q];
    }
  }
  const int fg = ctl.fg;
  free(base);
  return fg;
}
