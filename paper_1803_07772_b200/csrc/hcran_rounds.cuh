// hcran_rounds.cuh -- shared-memory-resident SCA rounds engine, sliced over
// subcarriers across a thread-block cluster (north_star).
//
// The SCA round loop of scale.py:553-615 (bound refresh, DC tangent, <= v_max
// Jacobi sweeps of analyze / budget bisection / closed form / duals, round
// rejection, stop tests) is >95% of the solve time.  Everything inside a
// sweep couples users only within one subcarrier n (interference, SIC order,
// psi terms, SIC multipliers), except three reductions: the per-RRH budget
// sums (budget bisection), the per-user surrogate rate sums (rate
// multipliers) and the per-RRH convergence maxima.  So CTA r of a cluster of
// CS owns subcarriers [r*NS, (r+1)*NS) (NS = N/CS) with all of their dense and
// seat state in its shared memory, and the three reductions are exchanged
// through distributed shared memory (double-buffered exchange slots, one
// cluster barrier per exchange).  Every CTA ends an exchange with identical
// totals, so all control decisions are replicated, never broadcast.
//
// The leader CTA (rank 0) keeps the per-instance outer logic (Dinkelbach,
// seating, repair, feasibility) on its global workspace and hands the rounds
// to the whole cluster through `run()`.  With CS = 1 the same code runs in one
// CTA; the host build (tests/emu) runs it with CS = 1.
//
// Numerics are those of hcran_solver.cuh (FP64, no FMA contraction, the
// reference's cancellation-prone forms and summation orders: column totals
// and received-power sums sequential in index order, psi_cross as A - B in
// one loop).  The decode-order prefix/suffix sums (same-RRH interference,
// psi_same) are warp scans: only the rounding of non-cancelling sums moves.
#pragma once
#include "hcran_solver.cuh"

#if defined(__CUDACC__)
#include <cooperative_groups.h>
#endif

namespace hcran {

struct ClusterHost {
  int crank = 0, csize = 1;
  void csync() const {}
  template <class T>
  T* remote(T* p, int) const { return p; }
};

#if defined(__CUDACC__)
struct ClusterDev {
  int crank, csize;
  __device__ void init() {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    crank = (int)cl.block_rank();
    csize = (int)cl.num_blocks();
  }
  __device__ __forceinline__ void csync() const {
    namespace cg = cooperative_groups;
    if (csize > 1) cg::this_cluster().sync();
    else __syncthreads();
  }
  template <class T>
  __device__ __forceinline__ T* remote(T* p, int r) const {
    namespace cg = cooperative_groups;
    return csize > 1 ? cg::this_cluster().map_shared_rank(p, r) : p;
  }
};
#endif

// warp-level exclusive prefix scan (lanes in order); host: one lane -> 0
#if defined(__CUDACC__)
__device__ __forceinline__ double wscan_excl(const DevEx&, double v, double& total) {
  double x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double t = __shfl_up_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) >= o) x += t;
  }
  total = __shfl_sync(0xffffffffu, x, 31);
  double ex = __shfl_up_sync(0xffffffffu, x, 1);
  return (threadIdx.x & 31) == 0 ? 0.0 : ex;
}
#endif
inline double wscan_excl(const HostEx&, double v, double& total) {
  total = v;
  return 0.0;
}

// shared-memory layout of one CTA's slice
struct ReMem {
  int M, K, KP, NS, L, NPL, CSL, CELLS, MNS, KNS, XN;
  // dense slice, column-contiguous [M][NS][KP] (KP = K rounded up to odd:
  // lanes over users and threads over columns both stay bank-conflict free)
  double *g, *al, *p, *u, *sig;
  uint8_t *ord, *rnk, *slot;
  double *tot, *pcr, *fterm, *colmax, *mtot;    // [M][NS]
  uint8_t *ncnt, *npr;                          // [M][NS]
  double *full, *utot, *fullm;                  // [NS][K]
  double *s_plin, *s_logplin, *s_beta, *s_pround, *s_num, *s_den, *s_psis, *s_cross, *s_inv,
      *s_rhat, *s_dlog, *s_dsA, *s_dsB, *s_nsS, *s_nsW, *s_dagg, *s_aagg, *s_mask;  // [M*NS][L]
  uint8_t* s_user;
  double *pr_zt, *pr_step, *pr_gconst, *pr_gval, *pr_brk, *pr_slack;  // [M*NS][NPL]
  uint8_t *pr_s, *pr_w;
  int16_t *useat;  // [K][NS]: local seat index (lcol*L + slot)
  int16_t* ucnt;   // [K]
  double *zeta, *xi, *eps1, *eps2, *minr, *wgt, *eta, *pmax, *ut;  // K, M, M, M, K, M*K, M, M, K
  uint8_t* el;                                                     // [K]
  double *xb0, *xb1, *xr;                                          // exchange [XN]
  double *gnum, *gden, *gmask;                                     // gathered seats of one head [N*L]
  double* tsw;                                                     // per-warp scratch [nwarps][K]

  HD static size_t al8(size_t x) { return (x + 15) & ~size_t(15); }

  HD size_t layout(char* base, int M_, int K_, int NS_, int L_, int N_, int nwarps) {
    M = M_; K = K_; NS = NS_; L = L_; NPL = L * (L - 1) / 2;
    KP = K | 1;
    CSL = M * NS * KP; CELLS = M * K * NS; MNS = M * NS; KNS = K * NS;
    XN = 2 * M + 2 * K + 8;
    const int S = MNS * L, P = MNS * (NPL > 0 ? NPL : 1);
    size_t off = 0;
    auto take = [&](size_t bytes) -> char* {
      char* r = base ? base + off : nullptr;
      off += al8(bytes);
      return r;
    };
#define RM_D(x, n) x = (double*)take(sizeof(double) * (size_t)(n))
#define RM_B(x, n) x = (uint8_t*)take((size_t)(n))
#define RM_S(x, n) x = (int16_t*)take(sizeof(int16_t) * (size_t)(n))
    RM_D(g, CSL); RM_D(al, CSL); RM_D(p, CSL); RM_D(u, CSL); RM_D(sig, CSL);
    RM_D(tot, MNS); RM_D(pcr, MNS); RM_D(fterm, MNS); RM_D(colmax, MNS); RM_D(mtot, MNS);
    RM_D(full, KNS); RM_D(utot, KNS); RM_D(fullm, KNS);
    RM_D(s_plin, S); RM_D(s_logplin, S); RM_D(s_beta, S); RM_D(s_pround, S); RM_D(s_num, S);
    RM_D(s_den, S); RM_D(s_psis, S); RM_D(s_cross, S); RM_D(s_inv, S); RM_D(s_rhat, S);
    RM_D(s_dlog, S); RM_D(s_dsA, S); RM_D(s_dsB, S); RM_D(s_nsS, S); RM_D(s_nsW, S);
    RM_D(s_dagg, S); RM_D(s_aagg, S); RM_D(s_mask, S);
    RM_D(pr_zt, P); RM_D(pr_step, P); RM_D(pr_gconst, P); RM_D(pr_gval, P); RM_D(pr_brk, P);
    RM_D(pr_slack, P);
    RM_D(zeta, K); RM_D(xi, M); RM_D(eps1, M); RM_D(eps2, M); RM_D(minr, K); RM_D(wgt, M * K);
    RM_D(eta, M); RM_D(pmax, M); RM_D(ut, K);
    RM_D(xb0, XN); RM_D(xb1, XN); RM_D(xr, XN);
    RM_D(gnum, N_ * L); RM_D(gden, N_ * L); RM_D(gmask, N_ * L);
    RM_D(tsw, nwarps * K);
    RM_B(ord, CSL); RM_B(rnk, CSL); RM_B(slot, CSL);
    RM_B(ncnt, MNS); RM_B(npr, MNS);
    RM_B(s_user, S); RM_B(pr_s, P); RM_B(pr_w, P); RM_B(el, K);
    RM_S(useat, KNS); RM_S(ucnt, K);
#undef RM_D
#undef RM_B
#undef RM_S
    return off;
  }
};

// index helpers over the hoisted locals (NS, KP_, K, N, n0, el_) of each phase
#define LC(m, k, ln) ((((m) * NS + (ln)) * KP_) + (k))
#define GC(m, k, ln) ((((m) * K + (k)) * N) + n0 + (ln))
#define ISEL(k) (el_[k] != 0)

template <class EX, class CX>
struct Rounds {
  EX& ex;
  CX& cx;
  const View& V;
  ReMem& R;
  int M, K, N, NS, L, NPL, n0;
  long long cur_b;
  const double* gam;  // instance gamma (global, [M][K][N])
  // replicated scalars
  double e, den_scale, p_ref, sic_cap, pf;
  int has_stream;
  int rounds, sweeps, evals, fg;
  double work;
  int xph;

  HD Rounds(EX& ex_, CX& cx_, const View& v, ReMem& r)
      : ex(ex_), cx(cx_), V(v), R(r), M(v.M), K(v.K), N(v.N), L(v.L) {
    NS = N / cx.csize;
    n0 = cx.crank * NS;
    NPL = L * (L - 1) / 2;
    cur_b = -1;
    gam = nullptr;
    xph = 0;
  }

  HDI int lc(int m, int k, int ln) const { return (m * NS + ln) * R.KP + k; }
  HDI int gc(int m, int k, int ln) const { return (m * K + k) * N + n0 + ln; }
  HDI bool is_el(int k) const { return R.el[k] != 0; }

  // ---------------------------------------------------------------- exchange
  HDI double* xbuf() { return xph ? R.xb1 : R.xb0; }
  // every CTA wrote xbuf()[0..n); on return xr[i] = sum (i < nsum) or max over CTAs
  HD void exchange(int nsum, int n) {
    const int M = this->M, K = this->K, N = this->N, NS = this->NS, L = this->L, NPL = this->NPL, n0 = this->n0;
    (void)M; (void)K; (void)N; (void)NS; (void)L; (void)NPL; (void)n0;
    double* __restrict__ xr_ = R.xr;

    double* mine = xbuf();
    cx.csync();
    for (int i = ex.tid; i < n; i += ex.nthr) {
      double acc = 0.0;
      for (int r = 0; r < cx.csize; ++r) {
        double v = cx.remote(mine, r)[i];
        acc = (r == 0) ? v : (i < nsum ? acc + v : fmax(acc, v));
      }
      xr_[i] = acc;
    }
    ex.sync();
    xph ^= 1;
  }

  // --------------------------------------------------------------- instance
  HD void load_instance(long long b) {
    const int M = this->M, K = this->K, N = this->N, NS = this->NS, L = this->L, NPL = this->NPL, n0 = this->n0;
    (void)M; (void)K; (void)N; (void)NS; (void)L; (void)NPL; (void)n0;
    const int CELLS_ = R.CELLS;
    const int KNS_ = R.KNS;
    const int KP_ = R.KP;
    const int MNS_ = R.MNS;
    uint8_t* __restrict__ el_ = R.el;
    double* __restrict__ eps1_ = R.eps1;
    double* __restrict__ eps2_ = R.eps2;
    double* __restrict__ eta_ = R.eta;
    double* __restrict__ fullm_ = R.fullm;
    double* __restrict__ g_ = R.g;
    double* __restrict__ minr_ = R.minr;
    double* __restrict__ mtot_ = R.mtot;
    uint8_t* __restrict__ ord_ = R.ord;
    double* __restrict__ pmax_ = R.pmax;
    uint8_t* __restrict__ rnk_ = R.rnk;
    double* __restrict__ sig_ = R.sig;
    double* __restrict__ wgt_ = R.wgt;

    gam = V.gamma + b * (long long)M * K * N;
    for (int i = ex.tid; i < CELLS_; i += ex.nthr) {
      int ln = i % NS, mk = i / NS;
      int k = mk % K, m = mk / K;
      g_[LC(m, k, ln)] = gam[GC(m, k, ln)];
      sig_[LC(m, k, ln)] = V.sig[GC(m, k, ln)];
    }
    for (int k = ex.tid; k < K; k += ex.nthr) {
      el_[k] = V.elastic[b * K + k];
      minr_[k] = V.min_rates[b * K + k];
    }
    for (int i = ex.tid; i < M * K; i += ex.nthr) wgt_[i] = V.w[i];
    for (int m = ex.tid; m < M; m += ex.nthr) {
      eta_[m] = V.eta[m];
      pmax_[m] = V.p_max[m];
      eps1_[m] = V.tol.varpi1_rel * V.p_max[m];
      eps2_[m] = V.tol.varpi2_rel * V.p_max[m];
    }
    ex.sync();
    for (int col = ex.tid; col < MNS_; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      double mt = 0.0;
      for (int k = 0; k < K; ++k) {
        double gk = g_[LC(m, k, ln)];
        int r = 0;
        for (int i = 0; i < K; ++i) {
          double gi = g_[LC(m, i, ln)];
          r += (gi > gk || (gi == gk && i < k)) ? 1 : 0;
        }
        rnk_[LC(m, k, ln)] = (uint8_t)r;
        ord_[LC(m, r, ln)] = (uint8_t)k;
        mt += V.mask[GC(m, k, ln)];
      }
      mtot_[col] = mt;
    }
    ex.sync();
    for (int kn = ex.tid; kn < KNS_; kn += ex.nthr) {
      int ln = kn / K, k = kn % K;
      double s = 0.0;
      for (int j = 0; j < M; ++j) s += mtot_[j * NS + ln] * g_[LC(j, k, ln)];
      fullm_[kn] = s;
    }
    ex.sync();
    cur_b = b;
  }

  // ------------------------------------------------------------- seating
  HD void build_seats(const double* Wp) {
    const int M = this->M, K = this->K, N = this->N, NS = this->NS, L = this->L, NPL = this->NPL, n0 = this->n0;
    (void)M; (void)K; (void)N; (void)NS; (void)L; (void)NPL; (void)n0;
    const int CELLS_ = R.CELLS;
    const int KP_ = R.KP;
    const int MNS_ = R.MNS;
    uint8_t* __restrict__ el_ = R.el;
    double* __restrict__ fullm_ = R.fullm;
    double* __restrict__ g_ = R.g;
    double* __restrict__ mtot_ = R.mtot;
    uint8_t* __restrict__ ncnt_ = R.ncnt;
    uint8_t* __restrict__ npr_ = R.npr;
    double* __restrict__ p_ = R.p;
    uint8_t* __restrict__ pr_s_ = R.pr_s;
    double* __restrict__ pr_step_ = R.pr_step;
    uint8_t* __restrict__ pr_w_ = R.pr_w;
    double* __restrict__ pr_zt_ = R.pr_zt;
    uint8_t* __restrict__ rnk_ = R.rnk;
    double* __restrict__ s_mask_ = R.s_mask;
    uint8_t* __restrict__ s_user_ = R.s_user;
    double* __restrict__ sig_ = R.sig;
    uint8_t* __restrict__ slot_ = R.slot;
    int16_t* __restrict__ ucnt_ = R.ucnt;
    int16_t* __restrict__ useat_ = R.useat;
    double* __restrict__ xi_ = R.xi;
    double* __restrict__ zeta_ = R.zeta;

    for (int i = ex.tid; i < CELLS_; i += ex.nthr) {
      int ln = i % NS, mk = i / NS;
      int k = mk % K, m = mk / K;
      p_[LC(m, k, ln)] = Wp[GC(m, k, ln)];
    }
    ex.sync();
    for (int col = ex.tid; col < MNS_; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      int cnt = 0;
      for (int k = 0; k < K; ++k) {
        int c = LC(m, k, ln);
        if (p_[c] > pf && cnt < L) {
          s_user_[col * L + cnt] = (uint8_t)k;
          s_mask_[col * L + cnt] = V.mask[GC(m, k, ln)];
          slot_[c] = (uint8_t)cnt++;
        } else {
          slot_[c] = NOSLOT;
        }
      }
      ncnt_[col] = (uint8_t)cnt;
      int np = 0;
      for (int i = 0; i < cnt; ++i)
        for (int j = i + 1; j < cnt; ++j) {
          int a = s_user_[col * L + i], bb = s_user_[col * L + j];
          bool ia = rnk_[LC(m, a, ln)] < rnk_[LC(m, bb, ln)];
          int q = col * NPL + np;
          pr_s_[q] = (uint8_t)(ia ? i : j);
          pr_w_[q] = (uint8_t)(ia ? j : i);
          pr_zt_[q] = 0.0;
          ++np;
        }
      npr_[col] = (uint8_t)np;
    }
    ex.sync();
    for (int k = ex.tid; k < K; k += ex.nthr) {
      int cnt = 0;
      for (int m = 0; m < M; ++m)
        for (int ln = 0; ln < NS; ++ln) {
          int c = LC(m, k, ln);
          if (slot_[c] != NOSLOT && cnt < NS) useat_[k * NS + cnt++] = (int16_t)((m * NS + ln) * L + slot_[c]);
        }
      ucnt_[k] = (int16_t)cnt;
      zeta_[k] = ISEL(k) ? 0.0 : 1.0;
    }
    for (int m = ex.tid; m < M; m += ex.nthr) xi_[m] = 0.0;
    // SIC multiplier steps (scale.py:701-703) for the seated pairs
    const double num = G_SIC * den_scale;
    for (int col = ex.tid; col < MNS_; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      for (int q = 0; q < npr_[col]; ++q) {
        int ss = col * L + pr_s_[col * NPL + q], sw = col * L + pr_w_[col * NPL + q];
        int a = s_user_[ss], b = s_user_[sw];
        int ca = LC(m, a, ln), cb = LC(m, b, ln);
        double g_s = g_[ca], g_w = g_[cb];
        double cm_s = fullm_[ln * K + a] - mtot_[col] * g_s;
        double cm_w = fullm_[ln * K + b] - mtot_[col] * g_w;
        double sc = g_w * sig_[ca] + g_s * sig_[cb] + g_w * cm_s + g_s * cm_w + 1e-300;
        pr_step_[col * NPL + q] = num / (p_ref * (sc * sc) * s_mask_[ss] * s_mask_[sw] + 1e-300);
      }
    }
    ex.sync();
  }

  // ------------------------------------------------------------ dense helpers
  HD void totals_full() {
    const int M = this->M, K = this->K, N = this->N, NS = this->NS, L = this->L, NPL = this->NPL, n0 = this->n0;
    (void)M; (void)K; (void)N; (void)NS; (void)L; (void)NPL; (void)n0;
    const int KNS_ = R.KNS;
    const int KP_ = R.KP;
    const int MNS_ = R.MNS;
    double* __restrict__ full_ = R.full;
    double* __restrict__ g_ = R.g;
    double* __restrict__ p_ = R.p;
    double* __restrict__ tot_ = R.tot;
  // column totals (index order) + received power per (k, n)
    for (int col = ex.tid; col < MNS_; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      double s = 0.0;
      for (int k = 0; k < K; ++k) s += p_[LC(m, k, ln)];
      tot_[col] = s;
    }
    ex.sync();
    for (int kn = ex.tid; kn < KNS_; kn += ex.nthr) {
      int ln = kn / K, k = kn % K;
      double s = 0.0;
      for (int j = 0; j < M; ++j) s += tot_[j * NS + ln] * g_[LC(j, k, ln)];
      full_[kn] = s;
    }
    ex.sync();
  }

  // bound coefficients + DC tangent at the round's start (scale.py:88-96, 726-735)
  HD void round_start() {
    const int M = this->M, K = this->K, N = this->N, NS = this->NS, L = this->L, NPL = this->NPL, n0 = this->n0;
    (void)M; (void)K; (void)N; (void)NS; (void)L; (void)NPL; (void)n0;
    const int CELLS_ = R.CELLS;
    const int KP_ = R.KP;
    const int MNS_ = R.MNS;
    double* __restrict__ al_ = R.al;
    double* __restrict__ full_ = R.full;
    double* __restrict__ g_ = R.g;
    uint8_t* __restrict__ npr_ = R.npr;
    uint8_t* __restrict__ ord_ = R.ord;
    double* __restrict__ p_ = R.p;
    double* __restrict__ pr_gconst_ = R.pr_gconst;
    double* __restrict__ pr_gval_ = R.pr_gval;
    uint8_t* __restrict__ pr_s_ = R.pr_s;
    uint8_t* __restrict__ pr_w_ = R.pr_w;
    double* __restrict__ s_beta_ = R.s_beta;
    double* __restrict__ s_cross_ = R.s_cross;
    double* __restrict__ s_logplin_ = R.s_logplin;
    double* __restrict__ s_plin_ = R.s_plin;
    double* __restrict__ s_pround_ = R.s_pround;
    uint8_t* __restrict__ s_user_ = R.s_user;
    double* __restrict__ sig_ = R.sig;
    uint8_t* __restrict__ slot_ = R.slot;
    double* __restrict__ tot_ = R.tot;

    PROF_T0
    totals_full();
    for (int col = ex.warp; col < MNS_; col += ex.nwarps) {
      int m = col / NS, ln = col % NS;
      const double tc = tot_[col];
      double carry = 0.0;
      for (int c0 = 0; c0 < K; c0 += EX::WS) {
        int r = c0 + ex.lane;
        bool act = r < K;
        int k = act ? ord_[LC(m, r, ln)] : 0;
        int c = LC(m, k, ln);
        double pc = act ? p_[c] : 0.0;
        double tot_chunk;
        double same = carry + wscan_excl(ex, pc, tot_chunk);
        if (act) {
          double g = g_[c];
          double cr = full_[ln * K + k] - tc * g;
          double z = pc * g / (sig_[c] + (g * same + cr));
          double a = 1.0, be = 0.0;
          if (z > 0) {
            a = z / (1.0 + z);
            be = log2(1.0 + z) - a * log2(z);
          }
          al_[c] = a;
          int sl = slot_[c];
          if (sl != NOSLOT) {
            int s = col * L + sl;
            s_beta_[s] = be;
            s_plin_[s] = pc;
            s_pround_[s] = pc;
            s_logplin_[s] = log(fmax(pc, ZF));
            s_cross_[s] = cr;
          }
        }
        carry = carry + tot_chunk;
      }
    }
    ex.sync();
    for (int col = ex.tid; col < MNS_; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      for (int q = 0; q < npr_[col]; ++q) {
        int pq = col * NPL + q;
        int ss = col * L + pr_s_[pq], sw = col * L + pr_w_[pq];
        double gconst = g_[LC(m, s_user_[ss], ln)] * s_plin_[ss] * s_plin_[sw];
        pr_gconst_[pq] = gconst;
        pr_gval_[pq] = gconst * s_cross_[sw];
      }
    }
    ex.sync();
    if (ex.tid == 0) work += WK_DENSE_ROUND * CELLS_ * cx.csize;
    PROF_MARK(10)
  }

  // ----------------------------------------------------------------- sweep
  HD bool sweep(int v) {
    const int M = this->M, K = this->K, N = this->N, NS = this->NS, L = this->L, NPL = this->NPL, n0 = this->n0;
    (void)M; (void)K; (void)N; (void)NS; (void)L; (void)NPL; (void)n0;
    const int CELLS_ = R.CELLS;
    const int KNS_ = R.KNS;
    const int KP_ = R.KP;
    const int MNS_ = R.MNS;
    double* __restrict__ al_ = R.al;
    double* __restrict__ colmax_ = R.colmax;
    uint8_t* __restrict__ el_ = R.el;
    double* __restrict__ eps1_ = R.eps1;
    double* __restrict__ eta_ = R.eta;
    double* __restrict__ fterm_ = R.fterm;
    double* __restrict__ full_ = R.full;
    double* __restrict__ g_ = R.g;
    double* __restrict__ minr_ = R.minr;
    uint8_t* __restrict__ ncnt_ = R.ncnt;
    uint8_t* __restrict__ npr_ = R.npr;
    uint8_t* __restrict__ ord_ = R.ord;
    double* __restrict__ p_ = R.p;
    double* __restrict__ pcr_ = R.pcr;
    double* __restrict__ pmax_ = R.pmax;
    double* __restrict__ pr_brk_ = R.pr_brk;
    double* __restrict__ pr_gconst_ = R.pr_gconst;
    double* __restrict__ pr_gval_ = R.pr_gval;
    uint8_t* __restrict__ pr_s_ = R.pr_s;
    double* __restrict__ pr_slack_ = R.pr_slack;
    double* __restrict__ pr_step_ = R.pr_step;
    uint8_t* __restrict__ pr_w_ = R.pr_w;
    double* __restrict__ pr_zt_ = R.pr_zt;
    double* __restrict__ s_aagg_ = R.s_aagg;
    double* __restrict__ s_beta_ = R.s_beta;
    double* __restrict__ s_cross_ = R.s_cross;
    double* __restrict__ s_dagg_ = R.s_dagg;
    double* __restrict__ s_den_ = R.s_den;
    double* __restrict__ s_dlog_ = R.s_dlog;
    double* __restrict__ s_dsA_ = R.s_dsA;
    double* __restrict__ s_dsB_ = R.s_dsB;
    double* __restrict__ s_inv_ = R.s_inv;
    double* __restrict__ s_logplin_ = R.s_logplin;
    double* __restrict__ s_mask_ = R.s_mask;
    double* __restrict__ s_nsS_ = R.s_nsS;
    double* __restrict__ s_nsW_ = R.s_nsW;
    double* __restrict__ s_num_ = R.s_num;
    double* __restrict__ s_plin_ = R.s_plin;
    double* __restrict__ s_psis_ = R.s_psis;
    double* __restrict__ s_rhat_ = R.s_rhat;
    uint8_t* __restrict__ s_user_ = R.s_user;
    double* __restrict__ sig_ = R.sig;
    uint8_t* __restrict__ slot_ = R.slot;
    double* __restrict__ tot_ = R.tot;
    double* __restrict__ tsw_ = R.tsw;
    double* __restrict__ u_ = R.u;
    int16_t* __restrict__ ucnt_ = R.ucnt;
    int16_t* __restrict__ useat_ = R.useat;
    double* __restrict__ utot_ = R.utot;
    double* __restrict__ wgt_ = R.wgt;
    double* __restrict__ xi_ = R.xi;
    double* __restrict__ xr_ = R.xr;
    double* __restrict__ zeta_ = R.zeta;

    PROF_T0
    totals_full();
    PROF_MARK(0)
    // decode-order pass, warp per column, lanes over ranks
    for (int col = ex.warp; col < MNS_; col += ex.nwarps) {
      int m = col / NS, ln = col % NS;
      const double tc = tot_[col];
      double* ts = tsw_ + ex.warp * K;
      double carry = 0.0;
      for (int c0 = 0; c0 < K; c0 += EX::WS) {
        int r = c0 + ex.lane;
        bool act = r < K;
        int k = act ? ord_[LC(m, r, ln)] : 0;
        int c = LC(m, k, ln);
        double pc = act ? p_[c] : 0.0;
        double tot_chunk;
        double same = carry + wscan_excl(ex, pc, tot_chunk);
        if (act) {
          double g = g_[c];
          double cr = full_[ln * K + k] - tc * g;
          double fl = sig_[c] + g * same + cr;
          double inv = 1.0 / fl;
          double zof = ISEL(k) ? 1.0 : zeta_[k];
          double crate = (wgt_[m * K + k] * zof) * al_[c];
          ts[r] = crate * g * inv / LN2;
          u_[c] = crate * inv / LN2;
          int sl = slot_[c];
          if (sl != NOSLOT) {
            s_cross_[col * L + sl] = cr;
            s_inv_[col * L + sl] = inv;
          }
        }
        carry = carry + tot_chunk;
      }
      ex.wsync();
      // suffix over weaker users: walk ranks from the weakest
      carry = 0.0;
      for (int c0 = 0; c0 < K; c0 += EX::WS) {
        int r = K - 1 - (c0 + ex.lane);
        bool act = r >= 0;
        double tv = act ? ts[r] : 0.0;
        double tot_chunk;
        double weaker = carry + wscan_excl(ex, tv, tot_chunk);
        if (act) {
          int k = ord_[LC(m, r, ln)];
          int sl = slot_[LC(m, k, ln)];
          if (sl != NOSLOT) s_psis_[col * L + sl] = weaker;
        }
        carry = carry + tot_chunk;
      }
      ex.wsync();
    }
    ex.sync();
    PROF_MARK(1)
    for (int kn = ex.tid; kn < KNS_; kn += ex.nthr) {
      int ln = kn / K, k = kn % K;
      double s = 0.0;
      for (int m = 0; m < M; ++m) s += u_[LC(m, k, ln)];
      utot_[kn] = s;
    }
    ex.sync();
    PROF_MARK(2)
    // psi_cross (A - B in one loop), seat dlog / f_term, seated-pair own terms
    for (int col = ex.tid; col < MNS_; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      double A = 0.0, Bv = 0.0;
      for (int l = 0; l < K; ++l) {
        int c = LC(m, l, ln);
        double g = g_[c];
        A += g * utot_[ln * K + l];
        Bv += g * u_[c];
      }
      pcr_[col] = A - Bv;
      double ft = 0.0;
      for (int i = 0; i < ncnt_[col]; ++i) {
        int s = col * L + i;
        s_dsA_[s] = 0.0; s_dsB_[s] = 0.0; s_nsS_[s] = 0.0; s_nsW_[s] = 0.0;
        s_dagg_[s] = 0.0; s_aagg_[s] = 0.0;
        double dl = log(fmax(p_[LC(m, s_user_[s], ln)], ZF)) - s_logplin_[s];
        s_dlog_[s] = dl;
        ft += s_plin_[s] * dl;
      }
      fterm_[col] = ft;
      for (int q = 0; q < npr_[col]; ++q) {
        int pq = col * NPL + q;
        int ss = col * L + pr_s_[pq], sw = col * L + pr_w_[pq];
        int ca = LC(m, s_user_[ss], ln), cb = LC(m, s_user_[sw], ln);
        double g_s = g_[ca], g_w = g_[cb];
        double p_s = p_[ca], p_w = p_[cb];
        double brk = g_w * sig_[ca] - g_s * sig_[cb] + g_w * s_cross_[ss];
        pr_brk_[pq] = brk;
        double zt = pr_zt_[pq];
        s_dsA_[ss] += zt * p_w * brk;
        s_dsB_[sw] += zt * p_s * brk;
        s_dagg_[ss] += zt * p_s * p_w * g_w;
        double own = zt * pr_gval_[pq];
        s_nsS_[ss] += own;
        s_nsW_[sw] += own;
        s_aagg_[sw] += zt * pr_gconst_[pq];
      }
    }
    ex.sync();
    PROF_MARK(3)
    // cross-RRH SIC aggregates, num / den, surrogate rates, SIC slack
    bool flag = false;
    for (int col = ex.tid; col < MNS_; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      double dtot = 0.0, down = 0.0, atot = 0.0, aown = 0.0;
      for (int j = 0; j < M; ++j) {
        int cj = j * NS + ln;
        for (int i = 0; i < ncnt_[cj]; ++i) {
          int s = cj * L + i;
          double g = g_[LC(m, s_user_[s], ln)];
          dtot += s_dagg_[s] * g;
          atot += s_aagg_[s] * g;
          if (j == m) { down += s_dagg_[s] * g; aown += s_aagg_[s] * g; }
        }
      }
      double dcr = dtot - down, bt = atot - aown;
      const double pc = pcr_[col];
      for (int i = 0; i < ncnt_[col]; ++i) {
        int s = col * L + i;
        int k = s_user_[s];
        int c = LC(m, k, ln);
        double zof = ISEL(k) ? 1.0 : zeta_[k];
        double crate = (wgt_[m * K + k] * zof) * al_[c];
        s_num_[s] = crate / LN2 + ((s_nsS_[s] + s_nsW_[s]) + s_plin_[s] * bt);
        double base = (e * eta_[m]) * (ISEL(k) ? 1.0 : 0.0);
        s_den_[s] = base + s_psis_[s] + pc + ((s_dsA_[s] + s_dsB_[s]) + dcr);
        double z = p_[c] * g_[c] * s_inv_[s];
        s_rhat_[s] = s_beta_[s] + al_[c] * log2(fmax(z, ZF));
        if (s_num_[s] == 0.0 && !(s_den_[s] > 0.0)) flag = true;  // floor tie
      }
      for (int q = 0; q < npr_[col]; ++q) {
        int pq = col * NPL + q;
        int ss = col * L + pr_s_[pq], sw = col * L + pr_w_[pq];
        int b = s_user_[sw];
        double hf = 0.0;
        for (int j = 0; j < M; ++j) hf += fterm_[j * NS + ln] * g_[LC(j, b, ln)];
        double hw = hf - fterm_[col] * g_[LC(m, b, ln)];
        double glin = pr_gval_[pq] * (1.0 + s_dlog_[ss] + s_dlog_[sw]) + pr_gconst_[pq] * hw;
        pr_slack_[pq] = p_[LC(m, s_user_[ss], ln)] * p_[LC(m, b, ln)] * pr_brk_[pq] - glin;
      }
    }
    flag = ex.any(flag);
    PROF_MARK(4)
    // exchange 1: budget load at xi = 0 per RRH, surrogate rate per user, floor-tie flag
    double* xb = xbuf();
    for (int m = ex.warp; m < M; m += ex.nwarps) {
      double s = 0.0;
      for (int ln = ex.lane; ln < NS; ln += EX::WS) {
        int col = m * NS + ln;
        for (int i = 0; i < ncnt_[col]; ++i) {
          int si = col * L + i;
          double num = s_num_[si], d = s_den_[si], mk = s_mask_[si];
          s += num <= 0 ? 0.0 : (d > 0 ? fmin(fmax(num / d, 0.0), mk) : mk);
        }
      }
      s = ex.wsum(s);
      if (ex.lane == 0) xb[m] = s;
    }
    for (int k = ex.tid; k < K; k += ex.nthr) {
      double r = 0.0;
      for (int t = 0; t < ucnt_[k]; ++t) {
        int s = useat_[k * NS + t];
        r += wgt_[(s / L / NS) * K + k] * s_rhat_[s];
      }
      xb[M + k] = r;
    }
    if (ex.tid == 0) xb[M + K] = flag ? 1.0 : 0.0;
    ex.sync();
    exchange(M + K + 1, M + K + 1);
    PROF_MARK(5)
    if (xr_[M + K] != 0.0) fg = 1;
    // per-RRH budget multipliers: exact bisection (scale.py:444-475).  One warp
    // group per tight RRH holds that RRH's seats from every CTA of the cluster
    // in registers; every CTA runs the same bisection on the same data in the
    // same order, so xi comes out identical everywhere without a broadcast.
    const double damp = 1.0 / sqrt((double)(v > 1 ? v : 1));
    int ev_total = 0;
    bool any_tight = false;
    for (int m = 0; m < M; ++m) any_tight |= (xr_[m] > pmax_[m]);
    if (!any_tight) {
      for (int m = ex.tid; m < M; m += ex.nthr) xi_[m] = 0.0;
      ev_total = M;
    } else {
      constexpr int SPL = EX::WS == 1 ? 4096 : 8;  // seats per lane (registers on the device)
      const int wph = ex.nwarps / M >= 1 ? ex.nwarps / M : 1;
      const int groups = ex.nwarps / wph;
      const int gsz = EX::WS * wph;
      const int grp = ex.warp / wph, gl = (ex.warp % wph) * EX::WS + ex.lane;
      for (int m0 = 0; m0 < M; m0 += groups) {
        const int m = m0 + grp;
        const bool mine = grp < groups && m < M;
        const bool tight = mine && xr_[m] > pmax_[m];
        if (mine && !tight && gl == 0) { xi_[m] = 0.0; colmax_[m] = 1.0; }
        if (tight) {
          double nm[SPL], dn[SPL], mk[SPL];
          int cnt = 0;
          for (int q = gl; q < N; q += gsz) {
            const int r = q / NS, col = m * NS + q % NS;
            const uint8_t nc = cx.remote(ncnt_, r)[col];
            const double* rn = cx.remote(s_num_, r) + col * L;
            const double* rd = cx.remote(s_den_, r) + col * L;
            const double* rk = cx.remote(s_mask_, r) + col * L;
            for (int i = 0; i < nc && cnt < SPL; ++i, ++cnt) {
              nm[cnt] = rn[i];
              dn[cnt] = rd[i];
              mk[cnt] = rk[i];
            }
          }
          const double budget = pmax_[m];
          int evals_m = 1;
          auto load = [&](double x) -> double {
            double acc = 0.0;
            for (int i = 0; i < cnt; ++i) {
              double d = dn[i] + x;
              acc += nm[i] <= 0 ? 0.0 : (d > 0 ? fmin(fmax(nm[i] / d, 0.0), mk[i]) : mk[i]);
            }
            acc = ex.wsum(acc);
            if (wph > 1) {  // combine the group's warps in order
              double* red = tsw_;
              if (ex.lane == 0) red[ex.warp * K] = acc;
              ex.named_sync(1 + grp, gsz);
              acc = 0.0;
              for (int w = grp * wph; w < (grp + 1) * wph; ++w) acc += red[w * K];
              ex.named_sync(1 + grp, gsz);
            }
            ++evals_m;
            return acc;
          };
          double hi = fmax(4.0 * xi_[m], 1e-6);
          for (int it = 0; it < 80; ++it) {
            if (load(hi) > budget) hi *= 8.0;
            else break;
          }
          double lo = 0.0;
          for (int it = 0; it < 42; ++it) {
            double mid = 0.5 * (lo + hi);
            if (load(mid) > budget) lo = mid;
            else hi = mid;
          }
          if (gl == 0) { xi_[m] = hi; colmax_[m] = (double)evals_m; }
        }
      }
      ex.sync();
      for (int m = 0; m < M; ++m) ev_total += (int)colmax_[m];
      ex.sync();
    }
    PROF_MARK(6)
    // rate multipliers (replicated)
    for (int k = ex.tid; k < K; k += ex.nthr) {
      if (ISEL(k)) continue;
      double sl = fmin(fmax(minr_[k] - xr_[M + k], -2.0 * RATE_SCALE), 2.0 * RATE_SCALE);
      double z = zeta_[k] + damp * (G_RATE / RATE_SCALE) * sl;
      zeta_[k] = fmin(fmax(z, 0.0), V.tol.dual_cap);
    }
    // closed form, SIC multipliers, per-RRH movement
    for (int col = ex.tid; col < MNS_; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      for (int q = 0; q < npr_[col]; ++q) {
        int pq = col * NPL + q;
        double zt = pr_zt_[pq] + damp * pr_step_[pq] * pr_slack_[pq];
        pr_zt_[pq] = fmin(fmax(zt, 0.0), sic_cap);
      }
      double dmax = 0.0;
      const double xm = xi_[m];
      for (int i = 0; i < ncnt_[col]; ++i) {
        int s = col * L + i;
        int c = LC(m, s_user_[s], ln);
        double num = s_num_[s], d = s_den_[s] + xm, mk = s_mask_[s];
        double raw = d > 0 ? num / d : mk;
        if (num <= 0) raw = 0.0;
        double pn = fmax(fmin(fmax(raw, 0.0), mk), pf);
        dmax = fmax(dmax, fabs(pn - p_[c]));
        p_[c] = pn;
      }
      colmax_[col] = dmax;
    }
    ex.sync();
    PROF_MARK(7)
    xb = xbuf();
    for (int m = ex.warp; m < M; m += ex.nwarps) {
      double d = 0.0;
      for (int ln = ex.lane; ln < NS; ln += EX::WS) d = fmax(d, colmax_[m * NS + ln]);
      d = ex.wmax(d);
      if (ex.lane == 0) xb[m] = d;
    }
    ex.sync();
    exchange(0, M);
    PROF_MARK(8)
    bool still = true;
    for (int m = 0; m < M; ++m)
      if (!(xr_[m] < eps1_[m])) still = false;
    // work counter (whole instance): dense cells, seats, budget evaluations
    if (ex.tid == 0) {
      int nseat = 0;
      for (int col = 0; col < MNS_; ++col) nseat += ncnt_[col];
      nseat *= cx.csize;  // approximately uniform slices
      const double np_ = 3.0 * nseat / (L > 1 ? L : 1);
      work += WK_DENSE_SWEEP * CELLS_ * cx.csize + WK_SEAT_SWEEP * nseat +
              WK_SEAT_EVAL * nseat * ((double)ev_total / M) + (WK_PAIR_SWEEP + 2.0 * M) * np_;
      evals += ev_total;
      sweeps += 1;
    }
    ex.sync();
    return still;
  }

  // ---------------------------------------------------------- round end
  HDI double val(int c, int col, int src) const {
    int sl = R.slot[c];
    if (src == 1 && sl != NOSLOT) return R.s_pround[col * L + sl];
    return R.p[c];
  }
  // surrogate partials for source `src` into xb[o], xb[o+1]; seat rates into s_dsA
  HD void surrogate_part(int src, double* xb, int o) {
    const int M = this->M, K = this->K, N = this->N, NS = this->NS, L = this->L, NPL = this->NPL, n0 = this->n0;
    (void)M; (void)K; (void)N; (void)NS; (void)L; (void)NPL; (void)n0;
    const int KP_ = R.KP;
    const int MNS_ = R.MNS;
    double* __restrict__ al_ = R.al;
    uint8_t* __restrict__ el_ = R.el;
    double* __restrict__ eta_ = R.eta;
    double* __restrict__ g_ = R.g;
    uint8_t* __restrict__ ncnt_ = R.ncnt;
    uint8_t* __restrict__ ord_ = R.ord;
    uint8_t* __restrict__ rnk_ = R.rnk;
    double* __restrict__ s_beta_ = R.s_beta;
    double* __restrict__ s_dsA_ = R.s_dsA;
    uint8_t* __restrict__ s_user_ = R.s_user;
    double* __restrict__ sig_ = R.sig;
    double* __restrict__ tot_ = R.tot;
    double* __restrict__ wgt_ = R.wgt;

    for (int col = ex.tid; col < MNS_; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      double s = 0.0;
      for (int k = 0; k < K; ++k) s += val(LC(m, k, ln), col, src);
      tot_[col] = s;
    }
    ex.sync();
    double rs = 0.0, ps = 0.0;
    for (int col = ex.tid; col < MNS_; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      for (int i = 0; i < ncnt_[col]; ++i) {
        int s = col * L + i;
        int k = s_user_[s];
        int c = LC(m, k, ln);
        double g = g_[c];
        double full = 0.0;
        for (int j = 0; j < M; ++j) full += tot_[j * NS + ln] * g_[LC(j, k, ln)];
        double cr = full - tot_[col] * g;
        double same = 0.0;
        for (int r = 0; r < rnk_[c]; ++r) same += val(LC(m, ord_[LC(m, r, ln)], ln), col, src);
        double pv = val(c, col, src);
        double z = pv * g / (sig_[c] + (g * same + cr));
        double rh = z > 0 ? s_beta_[s] + al_[c] * log2(fmax(z, ZF)) : 0.0;
        s_dsA_[s] = rh;
        if (ISEL(k)) {
          rs += rh * wgt_[m * K + k];
          ps += eta_[m] * pv;
        }
      }
    }
    rs = ex.sum(rs);
    ps = ex.sum(ps);
    if (ex.tid == 0) { xb[o] = rs; xb[o + 1] = ps; }
  }

  HD int round_end(int s) {
    const int M = this->M, K = this->K, N = this->N, NS = this->NS, L = this->L, NPL = this->NPL, n0 = this->n0;
    (void)M; (void)K; (void)N; (void)NS; (void)L; (void)NPL; (void)n0;
    const int KP_ = R.KP;
    const int MNS_ = R.MNS;
    double* __restrict__ colmax_ = R.colmax;
    uint8_t* __restrict__ el_ = R.el;
    double* __restrict__ eps2_ = R.eps2;
    double* __restrict__ minr_ = R.minr;
    uint8_t* __restrict__ ncnt_ = R.ncnt;
    double* __restrict__ p_ = R.p;
    double* __restrict__ s_dsA_ = R.s_dsA;
    double* __restrict__ s_pround_ = R.s_pround;
    uint8_t* __restrict__ s_user_ = R.s_user;
    int16_t* __restrict__ ucnt_ = R.ucnt;
    int16_t* __restrict__ useat_ = R.useat;
    double* __restrict__ wgt_ = R.wgt;
    double* __restrict__ xr_ = R.xr;
    double* __restrict__ zeta_ = R.zeta;
  // returns 1 to stop the round loop
    PROF_T0
    double* xb = xbuf();
    surrogate_part(1, xb, 0);
    surrogate_part(0, xb, 2);
    ex.sync();
    for (int k = ex.tid; k < K; k += ex.nthr) {
      double r = 0.0;
      for (int t = 0; t < ucnt_[k]; ++t) {
        int q = useat_[k * NS + t];
        r += wgt_[(q / L / NS) * K + k] * s_dsA_[q];
      }
      xb[4 + k] = r;
    }
    for (int col = ex.tid; col < MNS_; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      double d = 0.0;
      for (int i = 0; i < ncnt_[col]; ++i) {
        int q = col * L + i;
        d = fmax(d, fabs(p_[LC(m, s_user_[q], ln)] - s_pround_[q]));
      }
      colmax_[col] = d;
    }
    ex.sync();
    for (int m = ex.warp; m < M; m += ex.nwarps) {
      double d = 0.0;
      for (int ln = ex.lane; ln < NS; ln += EX::WS) d = fmax(d, colmax_[m * NS + ln]);
      d = ex.wmax(d);
      if (ex.lane == 0) xb[4 + K + m] = d;
    }
    ex.sync();
    exchange(4 + K, 4 + K + M);
    PROF_MARK(11)
    if (ex.tid == 0) rounds += 1;
    const double sp = V.static_power;
    double old_obj = xr_[0] - e * (sp + xr_[1]);
    double new_obj = xr_[2] - e * (sp + xr_[3]);
    if (new_obj < old_obj) {  // rejected round: restore its start (scale.py:595-601)
      for (int col = ex.tid; col < MNS_; col += ex.nthr) {
        int m = col / NS, ln = col % NS;
        for (int i = 0; i < ncnt_[col]; ++i) {
          int q = col * L + i;
          p_[LC(m, s_user_[q], ln)] = s_pround_[q];
        }
      }
      ex.sync();
      return 1;
    }
    const double capz = V.tol.dual_cap * (1 - 1e-9);
    for (int k = 0; k < K; ++k)
      if (!ISEL(k) && zeta_[k] >= capz && xr_[4 + k] < minr_[k] - V.tol.c13_rate_tol) return 1;
    if (s > 0) {
      bool settled = true;
      for (int m = 0; m < M; ++m)
        if (!(xr_[4 + K + m] < eps2_[m])) settled = false;
      if (settled) return 1;
    }
    return 0;
  }

  // ---------------------------------------------------------------- driver
  // All CTAs of the cluster call run() with the same command.  Returns with
  // the slice powers written back to Wp (global, [M][K][N]) and the counters set.
  HD void run(const ReCmd& cmd, double* Wp) {
    const int M = this->M, K = this->K, N = this->N, NS = this->NS, L = this->L, NPL = this->NPL, n0 = this->n0;
    (void)M; (void)K; (void)N; (void)NS; (void)L; (void)NPL; (void)n0;
    const int CELLS_ = R.CELLS;
    const int KP_ = R.KP;
    double* __restrict__ p_ = R.p;

    PROF_T0
    if (cmd.b != cur_b) load_instance(cmd.b);
    e = cmd.e; den_scale = cmd.den_scale; p_ref = cmd.p_ref; sic_cap = cmd.sic_cap;
    pf = cmd.p_floor; has_stream = cmd.has_stream;
    rounds = sweeps = evals = fg = 0;
    work = 0.0;
    build_seats(Wp);
    PROF_MARK(12)
    for (int s = 0; s < V.tol.s_max; ++s) {
      round_start();
      for (int v = 1; v <= V.tol.v_max; ++v) {
        bool still = sweep(v);
        if (v >= 8 && still) break;
      }
      if (round_end(s)) break;
    }
    for (int i = ex.tid; i < CELLS_; i += ex.nthr) {
      int ln = i % NS, mk = i / NS;
      int k = mk % K, m = mk / K;
      Wp[GC(m, k, ln)] = p_[LC(m, k, ln)];
    }
#if defined(__CUDA_ARCH__)
    __threadfence();
#endif
    cx.csync();
  }
};

}  // namespace hcran
