// hcran_work.cuh -- per-CTA workspace layout (one instance in flight per CTA).
//
// Dense per-cell state is [m][k][n] (cell c = (m*K + k)*N + n, the
// reference's index order, model.py:8-11), so a (m, n) column is strided by
// N and consecutive threads of a column phase touch consecutive n.
// Seat-compressed state: every (m, n) column holds at most SMAX seated users
// (exclusive seating, scale.py:561-566, 1007-1014), slots sorted by user
// index; the SIC multiplier family lives only on seated pairs (SURVEY.md
// 7.3-2, probe A.9: bit-identical to the dense family).
#pragma once
#include <stddef.h>
#include <stdint.h>
#include "hcran_exec.cuh"

namespace hcran {

constexpr int SMAX = 4;                       // seats per column (l_max <= 4)
constexpr int NPAIR = SMAX * (SMAX - 1) / 2;  // seated pairs per column
constexpr uint8_t NOSLOT = 0xFF;
// products-active multiplier families (scale.py:761-775, 835-840, 861-895):
// sparse rows, live only for non-exclusive seatings
constexpr int TQMAX = 64;    // materialised tuple rows (theta'), per inner solve
constexpr int THMAX = 1024;  // cross-head seat pairs of one user (theta)
constexpr int RMAX = 64;     // SCA rounds per inner solve (Tolerances.s_max <= RMAX)

struct Work {
  // dense [C], reference order [m][k][n]
  double *p, *pacc, *alpha, *u;  // alpha: bound slope per round; u: scratch copy of p
  uint8_t *ord, *rnk, *slot, *flag;  // rnk: decode rank (# stronger users on (m, n))
  // column tables of the analysis: seat ranks ascending [MN][SMAX], prefix
  // sums of the seat powers in that order [MN][SMAX + 1]
  uint8_t* cs_r;
  double* cs_q;
  // columns [MN]
  double *tot, *pcross, *fterm, *dcross, *bterm, *mtot, *colmax;
  uint8_t *ncnt, *npr;
  // [KN]
  double *full, *utot, *fullm;
  // seats [MN * SMAX]
  double *s_plin, *s_logplin, *s_num, *s_den, *s_psis, *s_cross, *s_inv, *s_rhat, *s_dlog,
      *s_beta, *s_dsA, *s_dsB, *s_nsS, *s_nsW, *s_dagg, *s_aagg, *s_pround,
      *s_mask,   // s_mask: the seat's per-cell power cap (mask), set with the seating
      *s_alpha,  // the seat's bound slope (per round)
      *s_p,      // the seat's power (mirrors p at its cell during the rounds)
      *s_g;      // the seat cell's gain (static per seating)
  int32_t* s_cell;  // the seat's cell index (static per seating)
  uint8_t* s_rk;    // the seat's decode rank (static per seating)
  uint8_t* s_user;
  // pairs [MN * NPAIR]
  double *pr_zt, *pr_step, *pr_gconst, *pr_gval, *pr_brk, *pr_slack;
  uint8_t *pr_s, *pr_w;  // slot indices of strong / weak member
  // users
  double *zeta, *minr, *score, *urate;  // score [M*K]
  uint8_t *elastic, *hsort, *best;      // hsort [K*M]: heads by score, descending; best [K]
  int32_t *tried, *needy;               // boost bookkeeping [K]
  double* dtmp;                         // [K]
  int32_t *useat, *ucnt;                // useat [K*N]: seat id = col*SMAX + slot
  // heads
  double *xi, *delta, *eps1, *eps2, *mtmp;
  int32_t* mev;  // budget-load evaluations per head (work counter)
  // repair scratch
  double *tb, *tX, *tY, *tS, *leaf;  // [MN] x4, leaf [C/64 + 64]
  int32_t* perm;                     // [N]
  int32_t* tlist;                    // [MN + 64] trim: each lane's active columns (strided by the warp size)
  uint8_t *dmask, *tie;              // [N] subcarriers on the dense SIC family / with a floor tie
  // repair: the nonzero cells of each column (<= l_max after the top-l cut),
  // users in index order (nzu) and in decode order (nzr); nzc 255 = not sparse
  uint8_t *nzu, *nzr, *nzc;
  int32_t* dlist;                    // [N] the dense subcarriers, compacted
  // dense SIC pair family (exact mode for floor-tie instances) -- bound when dense
  double *cx, *cxl, *dA, *dB, *nS, *nW, *dg, *ag;  // [C]
  double *pd_zt, *pd_step;                         // [K(K-1)/2][MN] (pair-major)
  uint8_t *pq_i, *pq_j;                            // [K(K-1)/2] members of pair q
  // products-active families: tuple rows (column, slot mask) and cross-head seat pairs
  int32_t *tq_col, *th_a, *th_b;                   // [TQMAX], [THMAX] x2 (seat ids)
  uint8_t* tq_sm;                                  // [TQMAX] member slots (bit mask)
  double *tq_val, *tq_step, *tq_slack;             // [TQMAX]
  double *th_val, *th_step, *th_slack;             // [THMAX]
  double *s_ppair, *s_ptup;                        // [S] per-seat pair / tuple pressure
  double* pbest;                                   // [C] multistart: best start's end point
  double *robj, *robj_best;                        // [RMAX] round objectives (current / accepted start)

  double* wleaf;    // [nw][wlstride]: leaf sums of the warp-parallel pairwise sums
  int32_t* wleafi;  // [nw][wlstride]: their offsets (PwCache)
  int wlstride;
  int nwarps = 1;
  double* gam_hot = nullptr;  // shared-memory copy of the instance's gains (bound by the kernel, else null)

  HD static size_t align(size_t x) { return (x + 255) & ~size_t(255); }
  // seats per user the per-user lists hold: a user may sit on several heads
  // only in small instances (multistart / external warm starts)
  HD static int useat_cap(int M, int K, int N) {
    return size_t(M) * K * N <= 4096 ? M * N : N;
  }

  // Arrays that may live in shared memory instead of the global slot, in
  // priority order: the analysis' column / row tables (read for every cell in
  // every sweep), then the per-cell streams.  `hot` is a bit mask over this
  // list; returns the bytes and rebinds the pointers when base != nullptr.
  enum { HOT_CSR, HOT_CSQ, HOT_TOT, HOT_FULL, HOT_UTOT, HOT_RNK, HOT_GAM, HOT_ALPHA, HOT_U,
         HOT_SLOT, HOT_P, HOT_N };
  HD static size_t hot_bytes(int i, size_t M, size_t K, size_t N) {
    const size_t C = M * K * N;
    switch (i) {
      case HOT_CSR: return M * N * SMAX;
      case HOT_CSQ: return 8 * M * N * (SMAX + 1);
      case HOT_TOT: return 8 * M * N;
      case HOT_FULL: case HOT_UTOT: return 8 * K * N;
      case HOT_RNK: case HOT_SLOT: return C;
      default: return 8 * C;
    }
  }
  HD size_t bind_hot(char* base, unsigned hot, int M, int K, int N) {
    size_t off = 0;
    for (int i = 0; i < HOT_N; ++i) {
      if (!(hot & (1u << i))) continue;
      char* q = base ? base + off : nullptr;
      off += (hot_bytes(i, M, K, N) + 15) & ~size_t(15);
      if (!base) continue;
      switch (i) {
        case HOT_CSR: cs_r = (uint8_t*)q; break;
        case HOT_CSQ: cs_q = (double*)q; break;
        case HOT_TOT: tot = (double*)q; break;
        case HOT_FULL: full = (double*)q; break;
        case HOT_UTOT: utot = (double*)q; break;
        case HOT_RNK: rnk = (uint8_t*)q; break;
        case HOT_GAM: gam_hot = (double*)q; break;
        case HOT_ALPHA: alpha = (double*)q; break;
        case HOT_U: u = (double*)q; break;
        case HOT_SLOT: slot = (uint8_t*)q; break;
        case HOT_P: p = (double*)q; break;
      }
    }
    return off;
  }

  // returns bytes; binds pointers when base != nullptr
  HD size_t layout(char* base, int M, int K, int N, bool dense = false, int nw = 16) {
    const size_t C = size_t(M) * K * N, MN = size_t(M) * N, KN = size_t(K) * N;
    nwarps = nw;
    wlstride = K * N / 64 + 8;
    const size_t S = MN * SMAX, PP = MN * NPAIR;
    size_t off = 0;
    auto take = [&](size_t bytes) -> char* {
      char* r = base ? base + off : nullptr;
      off += align(bytes);
      return r;
    };
#define HC_D(name, n) name = (double*)take(sizeof(double) * (n))
#define HC_B(name, n) name = (uint8_t*)take(n)
#define HC_I(name, n) name = (int32_t*)take(sizeof(int32_t) * (n))
    HC_D(p, C); HC_D(pacc, C); HC_D(alpha, C); HC_D(u, C);
    HC_B(ord, C); HC_B(rnk, C); HC_B(slot, C); HC_B(flag, C);
    HC_B(cs_r, MN * SMAX); HC_D(cs_q, MN * (SMAX + 1));
    HC_D(wleaf, size_t(nw) * wlstride); HC_I(wleafi, size_t(nw) * wlstride);
    HC_D(tot, MN); HC_D(pcross, MN); HC_D(fterm, MN); HC_D(dcross, MN); HC_D(bterm, MN);
    HC_D(mtot, MN); HC_D(colmax, MN);
    HC_B(ncnt, MN); HC_B(npr, MN);
    HC_D(full, KN); HC_D(utot, KN); HC_D(fullm, KN);
    HC_D(s_plin, S); HC_D(s_logplin, S); HC_D(s_num, S); HC_D(s_den, S); HC_D(s_psis, S);
    HC_D(s_cross, S); HC_D(s_inv, S); HC_D(s_rhat, S); HC_D(s_dlog, S); HC_D(s_beta, S);
    HC_D(s_dsA, S); HC_D(s_dsB, S); HC_D(s_nsS, S); HC_D(s_nsW, S); HC_D(s_dagg, S);
    HC_D(s_aagg, S); HC_D(s_pround, S); HC_D(s_mask, S); HC_D(s_alpha, S);
    HC_D(s_p, S); HC_D(s_g, S); HC_I(s_cell, S); HC_B(s_rk, S);
    HC_B(s_user, S);
    HC_D(pr_zt, PP); HC_D(pr_step, PP); HC_D(pr_gconst, PP); HC_D(pr_gval, PP);
    HC_D(pr_brk, PP); HC_D(pr_slack, PP);
    HC_B(pr_s, PP); HC_B(pr_w, PP);
    HC_D(zeta, K); HC_D(minr, K); HC_D(score, size_t(M) * K); HC_D(urate, K);
    HC_B(elastic, K); HC_B(hsort, size_t(K) * M); HC_B(best, K);
    HC_I(tried, K); HC_I(needy, K); HC_D(dtmp, K);
    HC_I(useat, size_t(K) * useat_cap(M, K, N)); HC_I(ucnt, K);
    HC_D(xi, M); HC_D(delta, M); HC_D(eps1, M); HC_D(eps2, M); HC_D(mtmp, M);
    HC_I(mev, M);
    HC_D(tb, MN); HC_D(tX, MN); HC_D(tY, MN); HC_D(tS, MN); HC_D(leaf, C / 64 + 64);
    HC_I(perm, N); HC_I(tlist, MN + 64);
    HC_B(dmask, N); HC_B(tie, N); HC_I(dlist, N);
    HC_B(nzu, MN * SMAX); HC_B(nzr, MN * SMAX); HC_B(nzc, MN);
    HC_I(tq_col, TQMAX); HC_B(tq_sm, TQMAX); HC_D(tq_val, TQMAX); HC_D(tq_step, TQMAX);
    HC_D(tq_slack, TQMAX);
    HC_I(th_a, THMAX); HC_I(th_b, THMAX); HC_D(th_val, THMAX); HC_D(th_step, THMAX);
    HC_D(th_slack, THMAX);
    HC_D(s_ppair, S); HC_D(s_ptup, S);
    HC_D(pbest, C <= 4096 ? C : 1);
    HC_D(robj, RMAX); HC_D(robj_best, RMAX);
    if (dense) {
      const size_t PD = MN * (size_t(K) * (K - 1) / 2);
      HC_D(cx, C); HC_D(cxl, C); HC_D(dA, C); HC_D(dB, C); HC_D(nS, C); HC_D(nW, C);
      HC_D(dg, C); HC_D(ag, C);
      HC_D(pd_zt, PD); HC_D(pd_step, PD);
      HC_B(pq_i, PD / MN + 1); HC_B(pq_j, PD / MN + 1);
    } else {
      cx = cxl = dA = dB = nS = nW = dg = ag = pd_zt = pd_step = nullptr;
      pq_i = pq_j = nullptr;
    }
#undef HC_D
#undef HC_B
#undef HC_I
    return off;
  }
};

}  // namespace hcran
