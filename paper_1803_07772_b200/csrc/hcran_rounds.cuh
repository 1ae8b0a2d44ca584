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
  int M, K, NS, L, NPL, CSL, MNS, KNS, XN;
  double *g, *al, *p, *u, *sig;                 // [M][K][NS]
  uint8_t *ord, *rnk, *slot;                    // [M][K][NS]
  double *tot, *pcr, *fterm, *colmax, *mtot;    // [M][NS]
  uint8_t *ncnt, *npr;                          // [M][NS]
  double *full, *utot, *fullm;                  // [K][NS]
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
    CSL = M * K * NS; MNS = M * NS; KNS = K * NS;
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

  HDI int lc(int m, int k, int ln) const { return (m * K + k) * NS + ln; }
  HDI int gc(int m, int k, int ln) const { return (m * K + k) * N + n0 + ln; }
  HDI bool is_el(int k) const { return R.el[k] != 0; }

  // ---------------------------------------------------------------- exchange
  HDI double* xbuf() { return xph ? R.xb1 : R.xb0; }
  // every CTA wrote xbuf()[0..n); on return xr[i] = sum (i < nsum) or max over CTAs
  HD void exchange(int nsum, int n) {
    double* mine = xbuf();
    cx.csync();
    for (int i = ex.tid; i < n; i += ex.nthr) {
      double acc = 0.0;
      for (int r = 0; r < cx.csize; ++r) {
        double v = cx.remote(mine, r)[i];
        acc = (r == 0) ? v : (i < nsum ? acc + v : fmax(acc, v));
      }
      R.xr[i] = acc;
    }
    ex.sync();
    xph ^= 1;
  }

  // --------------------------------------------------------------- instance
  HD void load_instance(long long b) {
    gam = V.gamma + b * (long long)M * K * N;
    for (int i = ex.tid; i < R.CSL; i += ex.nthr) {
      int ln = i % NS, mk = i / NS;
      int k = mk % K, m = mk / K;
      R.g[i] = gam[gc(m, k, ln)];
      R.sig[i] = V.sig[gc(m, k, ln)];
    }
    for (int k = ex.tid; k < K; k += ex.nthr) {
      R.el[k] = V.elastic[b * K + k];
      R.minr[k] = V.min_rates[b * K + k];
    }
    for (int i = ex.tid; i < M * K; i += ex.nthr) R.wgt[i] = V.w[i];
    for (int m = ex.tid; m < M; m += ex.nthr) {
      R.eta[m] = V.eta[m];
      R.pmax[m] = V.p_max[m];
      R.eps1[m] = V.tol.varpi1_rel * V.p_max[m];
      R.eps2[m] = V.tol.varpi2_rel * V.p_max[m];
    }
    ex.sync();
    for (int col = ex.tid; col < R.MNS; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      double mt = 0.0;
      for (int k = 0; k < K; ++k) {
        double gk = R.g[lc(m, k, ln)];
        int r = 0;
        for (int i = 0; i < K; ++i) {
          double gi = R.g[lc(m, i, ln)];
          r += (gi > gk || (gi == gk && i < k)) ? 1 : 0;
        }
        R.rnk[lc(m, k, ln)] = (uint8_t)r;
        R.ord[lc(m, r, ln)] = (uint8_t)k;
        mt += V.mask[gc(m, k, ln)];
      }
      R.mtot[col] = mt;
    }
    ex.sync();
    for (int kn = ex.tid; kn < R.KNS; kn += ex.nthr) {
      int k = kn / NS, ln = kn % NS;
      double s = 0.0;
      for (int j = 0; j < M; ++j) s += R.mtot[j * NS + ln] * R.g[lc(j, k, ln)];
      R.fullm[kn] = s;
    }
    ex.sync();
    cur_b = b;
  }

  // ------------------------------------------------------------- seating
  HD void build_seats(const double* Wp) {
    for (int i = ex.tid; i < R.CSL; i += ex.nthr) {
      int ln = i % NS, mk = i / NS;
      int k = mk % K, m = mk / K;
      R.p[i] = Wp[gc(m, k, ln)];
    }
    ex.sync();
    for (int col = ex.tid; col < R.MNS; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      int cnt = 0;
      for (int k = 0; k < K; ++k) {
        int c = lc(m, k, ln);
        if (R.p[c] > pf && cnt < L) {
          R.s_user[col * L + cnt] = (uint8_t)k;
          R.s_mask[col * L + cnt] = V.mask[gc(m, k, ln)];
          R.slot[c] = (uint8_t)cnt++;
        } else {
          R.slot[c] = NOSLOT;
        }
      }
      R.ncnt[col] = (uint8_t)cnt;
      int np = 0;
      for (int i = 0; i < cnt; ++i)
        for (int j = i + 1; j < cnt; ++j) {
          int a = R.s_user[col * L + i], bb = R.s_user[col * L + j];
          bool ia = R.rnk[lc(m, a, ln)] < R.rnk[lc(m, bb, ln)];
          int q = col * NPL + np;
          R.pr_s[q] = (uint8_t)(ia ? i : j);
          R.pr_w[q] = (uint8_t)(ia ? j : i);
          R.pr_zt[q] = 0.0;
          ++np;
        }
      R.npr[col] = (uint8_t)np;
    }
    ex.sync();
    for (int k = ex.tid; k < K; k += ex.nthr) {
      int cnt = 0;
      for (int m = 0; m < M; ++m)
        for (int ln = 0; ln < NS; ++ln) {
          int c = lc(m, k, ln);
          if (R.slot[c] != NOSLOT && cnt < NS) R.useat[k * NS + cnt++] = (int16_t)((m * NS + ln) * L + R.slot[c]);
        }
      R.ucnt[k] = (int16_t)cnt;
      R.zeta[k] = is_el(k) ? 0.0 : 1.0;
    }
    for (int m = ex.tid; m < M; m += ex.nthr) R.xi[m] = 0.0;
    // SIC multiplier steps (scale.py:701-703) for the seated pairs
    const double num = G_SIC * den_scale;
    for (int col = ex.tid; col < R.MNS; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      for (int q = 0; q < R.npr[col]; ++q) {
        int ss = col * L + R.pr_s[col * NPL + q], sw = col * L + R.pr_w[col * NPL + q];
        int a = R.s_user[ss], b = R.s_user[sw];
        int ca = lc(m, a, ln), cb = lc(m, b, ln);
        double g_s = R.g[ca], g_w = R.g[cb];
        double cm_s = R.fullm[a * NS + ln] - R.mtot[col] * g_s;
        double cm_w = R.fullm[b * NS + ln] - R.mtot[col] * g_w;
        double sc = g_w * R.sig[ca] + g_s * R.sig[cb] + g_w * cm_s + g_s * cm_w + 1e-300;
        R.pr_step[col * NPL + q] = num / (p_ref * (sc * sc) * R.s_mask[ss] * R.s_mask[sw] + 1e-300);
      }
    }
    ex.sync();
  }

  // ------------------------------------------------------------ dense helpers
  HD void totals_full() {  // column totals (index order) + received power per (k, n)
    for (int col = ex.tid; col < R.MNS; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      double s = 0.0;
      for (int k = 0; k < K; ++k) s += R.p[lc(m, k, ln)];
      R.tot[col] = s;
    }
    ex.sync();
    for (int kn = ex.tid; kn < R.KNS; kn += ex.nthr) {
      int k = kn / NS, ln = kn % NS;
      double s = 0.0;
      for (int j = 0; j < M; ++j) s += R.tot[j * NS + ln] * R.g[lc(j, k, ln)];
      R.full[kn] = s;
    }
    ex.sync();
  }

  // bound coefficients + DC tangent at the round's start (scale.py:88-96, 726-735)
  HD void round_start() {
    totals_full();
    for (int col = ex.warp; col < R.MNS; col += ex.nwarps) {
      int m = col / NS, ln = col % NS;
      const double tc = R.tot[col];
      double carry = 0.0;
      for (int c0 = 0; c0 < K; c0 += EX::WS) {
        int r = c0 + ex.lane;
        bool act = r < K;
        int k = act ? R.ord[lc(m, r, ln)] : 0;
        int c = lc(m, k, ln);
        double pc = act ? R.p[c] : 0.0;
        double tot_chunk;
        double same = carry + wscan_excl(ex, pc, tot_chunk);
        if (act) {
          double g = R.g[c];
          double cr = R.full[k * NS + ln] - tc * g;
          double z = pc * g / (R.sig[c] + (g * same + cr));
          double a = 1.0, be = 0.0;
          if (z > 0) {
            a = z / (1.0 + z);
            be = log2(1.0 + z) - a * log2(z);
          }
          R.al[c] = a;
          int sl = R.slot[c];
          if (sl != NOSLOT) {
            int s = col * L + sl;
            R.s_beta[s] = be;
            R.s_plin[s] = pc;
            R.s_pround[s] = pc;
            R.s_logplin[s] = log(fmax(pc, ZF));
            R.s_cross[s] = cr;
          }
        }
        carry = carry + tot_chunk;
      }
    }
    ex.sync();
    for (int col = ex.tid; col < R.MNS; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      for (int q = 0; q < R.npr[col]; ++q) {
        int pq = col * NPL + q;
        int ss = col * L + R.pr_s[pq], sw = col * L + R.pr_w[pq];
        double gconst = R.g[lc(m, R.s_user[ss], ln)] * R.s_plin[ss] * R.s_plin[sw];
        R.pr_gconst[pq] = gconst;
        R.pr_gval[pq] = gconst * R.s_cross[sw];
      }
    }
    ex.sync();
    if (ex.tid == 0) work += WK_DENSE_ROUND * R.CSL * cx.csize;
  }

  // ----------------------------------------------------------------- sweep
  HD bool sweep(int v) {
    totals_full();
    // decode-order pass, warp per column, lanes over ranks
    for (int col = ex.warp; col < R.MNS; col += ex.nwarps) {
      int m = col / NS, ln = col % NS;
      const double tc = R.tot[col];
      double* ts = R.tsw + ex.warp * K;
      double carry = 0.0;
      for (int c0 = 0; c0 < K; c0 += EX::WS) {
        int r = c0 + ex.lane;
        bool act = r < K;
        int k = act ? R.ord[lc(m, r, ln)] : 0;
        int c = lc(m, k, ln);
        double pc = act ? R.p[c] : 0.0;
        double tot_chunk;
        double same = carry + wscan_excl(ex, pc, tot_chunk);
        if (act) {
          double g = R.g[c];
          double cr = R.full[k * NS + ln] - tc * g;
          double fl = R.sig[c] + g * same + cr;
          double inv = 1.0 / fl;
          double zof = is_el(k) ? 1.0 : R.zeta[k];
          double crate = (R.wgt[m * K + k] * zof) * R.al[c];
          ts[r] = crate * g * inv / LN2;
          R.u[c] = crate * inv / LN2;
          int sl = R.slot[c];
          if (sl != NOSLOT) {
            R.s_cross[col * L + sl] = cr;
            R.s_inv[col * L + sl] = inv;
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
          int k = R.ord[lc(m, r, ln)];
          int sl = R.slot[lc(m, k, ln)];
          if (sl != NOSLOT) R.s_psis[col * L + sl] = weaker;
        }
        carry = carry + tot_chunk;
      }
      ex.wsync();
    }
    ex.sync();
    for (int kn = ex.tid; kn < R.KNS; kn += ex.nthr) {
      int k = kn / NS, ln = kn % NS;
      double s = 0.0;
      for (int m = 0; m < M; ++m) s += R.u[lc(m, k, ln)];
      R.utot[kn] = s;
    }
    ex.sync();
    // psi_cross (A - B in one loop), seat dlog / f_term, seated-pair own terms
    for (int col = ex.tid; col < R.MNS; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      double A = 0.0, Bv = 0.0;
      for (int l = 0; l < K; ++l) {
        int c = lc(m, l, ln);
        double g = R.g[c];
        A += g * R.utot[l * NS + ln];
        Bv += g * R.u[c];
      }
      R.pcr[col] = A - Bv;
      double ft = 0.0;
      for (int i = 0; i < R.ncnt[col]; ++i) {
        int s = col * L + i;
        R.s_dsA[s] = 0.0; R.s_dsB[s] = 0.0; R.s_nsS[s] = 0.0; R.s_nsW[s] = 0.0;
        R.s_dagg[s] = 0.0; R.s_aagg[s] = 0.0;
        double dl = log(fmax(R.p[lc(m, R.s_user[s], ln)], ZF)) - R.s_logplin[s];
        R.s_dlog[s] = dl;
        ft += R.s_plin[s] * dl;
      }
      R.fterm[col] = ft;
      for (int q = 0; q < R.npr[col]; ++q) {
        int pq = col * NPL + q;
        int ss = col * L + R.pr_s[pq], sw = col * L + R.pr_w[pq];
        int ca = lc(m, R.s_user[ss], ln), cb = lc(m, R.s_user[sw], ln);
        double g_s = R.g[ca], g_w = R.g[cb];
        double p_s = R.p[ca], p_w = R.p[cb];
        double brk = g_w * R.sig[ca] - g_s * R.sig[cb] + g_w * R.s_cross[ss];
        R.pr_brk[pq] = brk;
        double zt = R.pr_zt[pq];
        R.s_dsA[ss] += zt * p_w * brk;
        R.s_dsB[sw] += zt * p_s * brk;
        R.s_dagg[ss] += zt * p_s * p_w * g_w;
        double own = zt * R.pr_gval[pq];
        R.s_nsS[ss] += own;
        R.s_nsW[sw] += own;
        R.s_aagg[sw] += zt * R.pr_gconst[pq];
      }
    }
    ex.sync();
    // cross-RRH SIC aggregates, num / den, surrogate rates, SIC slack
    bool flag = false;
    for (int col = ex.tid; col < R.MNS; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      double dtot = 0.0, down = 0.0, atot = 0.0, aown = 0.0;
      for (int j = 0; j < M; ++j) {
        int cj = j * NS + ln;
        for (int i = 0; i < R.ncnt[cj]; ++i) {
          int s = cj * L + i;
          double g = R.g[lc(m, R.s_user[s], ln)];
          dtot += R.s_dagg[s] * g;
          atot += R.s_aagg[s] * g;
          if (j == m) { down += R.s_dagg[s] * g; aown += R.s_aagg[s] * g; }
        }
      }
      double dcr = dtot - down, bt = atot - aown;
      const double pc = R.pcr[col];
      for (int i = 0; i < R.ncnt[col]; ++i) {
        int s = col * L + i;
        int k = R.s_user[s];
        int c = lc(m, k, ln);
        double zof = is_el(k) ? 1.0 : R.zeta[k];
        double crate = (R.wgt[m * K + k] * zof) * R.al[c];
        R.s_num[s] = crate / LN2 + ((R.s_nsS[s] + R.s_nsW[s]) + R.s_plin[s] * bt);
        double base = (e * R.eta[m]) * (is_el(k) ? 1.0 : 0.0);
        R.s_den[s] = base + R.s_psis[s] + pc + ((R.s_dsA[s] + R.s_dsB[s]) + dcr);
        double z = R.p[c] * R.g[c] * R.s_inv[s];
        R.s_rhat[s] = R.s_beta[s] + R.al[c] * log2(fmax(z, ZF));
        if (R.s_num[s] == 0.0 && R.s_den[s] == 0.0) flag = true;
      }
      for (int q = 0; q < R.npr[col]; ++q) {
        int pq = col * NPL + q;
        int ss = col * L + R.pr_s[pq], sw = col * L + R.pr_w[pq];
        int b = R.s_user[sw];
        double hf = 0.0;
        for (int j = 0; j < M; ++j) hf += R.fterm[j * NS + ln] * R.g[lc(j, b, ln)];
        double hw = hf - R.fterm[col] * R.g[lc(m, b, ln)];
        double glin = R.pr_gval[pq] * (1.0 + R.s_dlog[ss] + R.s_dlog[sw]) + R.pr_gconst[pq] * hw;
        R.pr_slack[pq] = R.p[lc(m, R.s_user[ss], ln)] * R.p[lc(m, b, ln)] * R.pr_brk[pq] - glin;
      }
    }
    flag = ex.any(flag);
    // exchange 1: budget load at xi = 0 per RRH, surrogate rate per user, floor-tie flag
    double* xb = xbuf();
    for (int m = ex.warp; m < M; m += ex.nwarps) {
      double s = 0.0;
      for (int ln = ex.lane; ln < NS; ln += EX::WS) {
        int col = m * NS + ln;
        for (int i = 0; i < R.ncnt[col]; ++i) {
          int si = col * L + i;
          double num = R.s_num[si], d = R.s_den[si], mk = R.s_mask[si];
          s += num <= 0 ? 0.0 : (d > 0 ? fmin(fmax(num / d, 0.0), mk) : mk);
        }
      }
      s = ex.wsum(s);
      if (ex.lane == 0) xb[m] = s;
    }
    for (int k = ex.tid; k < K; k += ex.nthr) {
      double r = 0.0;
      for (int t = 0; t < R.ucnt[k]; ++t) {
        int s = R.useat[k * NS + t];
        r += R.wgt[(s / L / NS) * K + k] * R.s_rhat[s];
      }
      xb[M + k] = r;
    }
    if (ex.tid == 0) xb[M + K] = flag ? 1.0 : 0.0;
    ex.sync();
    exchange(M + K + 1, M + K + 1);
    if (R.xr[M + K] != 0.0) fg = 1;
    // per-RRH budget multipliers (exact bisection on the gathered seats of tight heads)
    const double damp = 1.0 / sqrt((double)(v > 1 ? v : 1));
    int ev_total = 0;
    for (int m = 0; m < M; ++m) {
      const double budget = R.pmax[m];
      if (!(R.xr[m] > budget)) {
        if (ex.tid == 0) R.xi[m] = 0.0;
        ev_total += 1;
        continue;
      }
      // gather head m's seats from every CTA, in (rank, subcarrier, slot) order
      if (ex.warp == 0) {
        int cnt = 0;
        for (int r = 0; r < cx.csize; ++r) {
          uint8_t* rc = cx.remote(R.ncnt, r);
          double* rn = cx.remote(R.s_num, r);
          double* rd = cx.remote(R.s_den, r);
          double* rk = cx.remote(R.s_mask, r);
          for (int ln = 0; ln < NS; ++ln) {
            int col = m * NS + ln;
            int nc = rc[col];
            for (int i = ex.lane; i < nc; i += EX::WS) {
              R.gnum[cnt + i] = rn[col * L + i];
              R.gden[cnt + i] = rd[col * L + i];
              R.gmask[cnt + i] = rk[col * L + i];
            }
            cnt += nc;
          }
        }
        ex.wsync();
        int evals_m = 0;
        auto load = [&](double x) -> double {
          double s = 0.0;
          for (int i = ex.lane; i < cnt; i += EX::WS) {
            double num = R.gnum[i], d = R.gden[i] + x, mk = R.gmask[i];
            s += num <= 0 ? 0.0 : (d > 0 ? fmin(fmax(num / d, 0.0), mk) : mk);
          }
          ++evals_m;
          return ex.wsum(s);
        };
        double hi = fmax(4.0 * R.xi[m], 1e-6);
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
        ex.wsync();
        if (ex.lane == 0) { R.xi[m] = hi; R.colmax[0] = (double)(evals_m + 1); }
      }
      ex.sync();
      ev_total += (int)R.colmax[0];
      ex.sync();
    }
    // rate multipliers (replicated)
    for (int k = ex.tid; k < K; k += ex.nthr) {
      if (is_el(k)) continue;
      double sl = fmin(fmax(R.minr[k] - R.xr[M + k], -2.0 * RATE_SCALE), 2.0 * RATE_SCALE);
      double z = R.zeta[k] + damp * (G_RATE / RATE_SCALE) * sl;
      R.zeta[k] = fmin(fmax(z, 0.0), V.tol.dual_cap);
    }
    // closed form, SIC multipliers, per-RRH movement
    for (int col = ex.tid; col < R.MNS; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      for (int q = 0; q < R.npr[col]; ++q) {
        int pq = col * NPL + q;
        double zt = R.pr_zt[pq] + damp * R.pr_step[pq] * R.pr_slack[pq];
        R.pr_zt[pq] = fmin(fmax(zt, 0.0), sic_cap);
      }
      double dmax = 0.0;
      const double xm = R.xi[m];
      for (int i = 0; i < R.ncnt[col]; ++i) {
        int s = col * L + i;
        int c = lc(m, R.s_user[s], ln);
        double num = R.s_num[s], d = R.s_den[s] + xm, mk = R.s_mask[s];
        double raw = d > 0 ? num / d : mk;
        if (num <= 0) raw = 0.0;
        double pn = fmax(fmin(fmax(raw, 0.0), mk), pf);
        dmax = fmax(dmax, fabs(pn - R.p[c]));
        R.p[c] = pn;
      }
      R.colmax[col] = dmax;
    }
    ex.sync();
    xb = xbuf();
    for (int m = ex.warp; m < M; m += ex.nwarps) {
      double d = 0.0;
      for (int ln = ex.lane; ln < NS; ln += EX::WS) d = fmax(d, R.colmax[m * NS + ln]);
      d = ex.wmax(d);
      if (ex.lane == 0) xb[m] = d;
    }
    ex.sync();
    exchange(0, M);
    bool still = true;
    for (int m = 0; m < M; ++m)
      if (!(R.xr[m] < R.eps1[m])) still = false;
    // work counter (whole instance): dense cells, seats, budget evaluations
    if (ex.tid == 0) {
      int nseat = 0;
      for (int col = 0; col < R.MNS; ++col) nseat += R.ncnt[col];
      nseat *= cx.csize;  // approximately uniform slices
      const double np_ = 3.0 * nseat / (L > 1 ? L : 1);
      work += WK_DENSE_SWEEP * R.CSL * cx.csize + WK_SEAT_SWEEP * nseat +
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
    for (int col = ex.tid; col < R.MNS; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      double s = 0.0;
      for (int k = 0; k < K; ++k) s += val(lc(m, k, ln), col, src);
      R.tot[col] = s;
    }
    ex.sync();
    double rs = 0.0, ps = 0.0;
    for (int col = ex.tid; col < R.MNS; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      for (int i = 0; i < R.ncnt[col]; ++i) {
        int s = col * L + i;
        int k = R.s_user[s];
        int c = lc(m, k, ln);
        double g = R.g[c];
        double full = 0.0;
        for (int j = 0; j < M; ++j) full += R.tot[j * NS + ln] * R.g[lc(j, k, ln)];
        double cr = full - R.tot[col] * g;
        double same = 0.0;
        for (int r = 0; r < R.rnk[c]; ++r) same += val(lc(m, R.ord[lc(m, r, ln)], ln), col, src);
        double pv = val(c, col, src);
        double z = pv * g / (R.sig[c] + (g * same + cr));
        double rh = z > 0 ? R.s_beta[s] + R.al[c] * log2(fmax(z, ZF)) : 0.0;
        R.s_dsA[s] = rh;
        if (is_el(k)) {
          rs += rh * R.wgt[m * K + k];
          ps += R.eta[m] * pv;
        }
      }
    }
    rs = ex.sum(rs);
    ps = ex.sum(ps);
    if (ex.tid == 0) { xb[o] = rs; xb[o + 1] = ps; }
  }

  HD int round_end(int s) {  // returns 1 to stop the round loop
    double* xb = xbuf();
    surrogate_part(1, xb, 0);
    surrogate_part(0, xb, 2);
    ex.sync();
    for (int k = ex.tid; k < K; k += ex.nthr) {
      double r = 0.0;
      for (int t = 0; t < R.ucnt[k]; ++t) {
        int q = R.useat[k * NS + t];
        r += R.wgt[(q / L / NS) * K + k] * R.s_dsA[q];
      }
      xb[4 + k] = r;
    }
    for (int col = ex.tid; col < R.MNS; col += ex.nthr) {
      int m = col / NS, ln = col % NS;
      double d = 0.0;
      for (int i = 0; i < R.ncnt[col]; ++i) {
        int q = col * L + i;
        d = fmax(d, fabs(R.p[lc(m, R.s_user[q], ln)] - R.s_pround[q]));
      }
      R.colmax[col] = d;
    }
    ex.sync();
    for (int m = ex.warp; m < M; m += ex.nwarps) {
      double d = 0.0;
      for (int ln = ex.lane; ln < NS; ln += EX::WS) d = fmax(d, R.colmax[m * NS + ln]);
      d = ex.wmax(d);
      if (ex.lane == 0) xb[4 + K + m] = d;
    }
    ex.sync();
    exchange(4 + K, 4 + K + M);
    if (ex.tid == 0) rounds += 1;
    const double sp = V.static_power;
    double old_obj = R.xr[0] - e * (sp + R.xr[1]);
    double new_obj = R.xr[2] - e * (sp + R.xr[3]);
    if (new_obj < old_obj) {  // rejected round: restore its start (scale.py:595-601)
      for (int col = ex.tid; col < R.MNS; col += ex.nthr) {
        int m = col / NS, ln = col % NS;
        for (int i = 0; i < R.ncnt[col]; ++i) {
          int q = col * L + i;
          R.p[lc(m, R.s_user[q], ln)] = R.s_pround[q];
        }
      }
      ex.sync();
      return 1;
    }
    const double capz = V.tol.dual_cap * (1 - 1e-9);
    for (int k = 0; k < K; ++k)
      if (!is_el(k) && R.zeta[k] >= capz && R.xr[4 + k] < R.minr[k] - V.tol.c13_rate_tol) return 1;
    if (s > 0) {
      bool settled = true;
      for (int m = 0; m < M; ++m)
        if (!(R.xr[4 + K + m] < R.eps2[m])) settled = false;
      if (settled) return 1;
    }
    return 0;
  }

  // ---------------------------------------------------------------- driver
  // All CTAs of the cluster call run() with the same command.  Returns with
  // the slice powers written back to Wp (global, [M][K][N]) and the counters set.
  HD void run(const ReCmd& cmd, double* Wp) {
    if (cmd.b != cur_b) load_instance(cmd.b);
    e = cmd.e; den_scale = cmd.den_scale; p_ref = cmd.p_ref; sic_cap = cmd.sic_cap;
    pf = cmd.p_floor; has_stream = cmd.has_stream;
    rounds = sweeps = evals = fg = 0;
    work = 0.0;
    build_seats(Wp);
    for (int s = 0; s < V.tol.s_max; ++s) {
      round_start();
      for (int v = 1; v <= V.tol.v_max; ++v) {
        bool still = sweep(v);
        if (v >= 8 && still) break;
      }
      if (round_end(s)) break;
    }
    for (int i = ex.tid; i < R.CSL; i += ex.nthr) {
      int ln = i % NS, mk = i / NS;
      int k = mk % K, m = mk / K;
      Wp[gc(m, k, ln)] = R.p[i];
    }
#if defined(__CUDA_ARCH__)
    __threadfence();
#endif
    cx.csync();
  }
};

}  // namespace hcran
