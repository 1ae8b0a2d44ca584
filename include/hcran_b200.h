/*
 * hcran_b200.h -- C ABI of the B200 batched EE solver (libhcran_b200.so).
 *
 * Drop-in boundary for the reference's hot path.  The
 * reference (hcran-noma, pure Python) has no native ABI; these entry points
 * replace, for a whole batch of independent channel realisations at once:
 *
 *   hcran_b200_solve_batch          <- dinkelbach.solve(ch, cfg, ScaleSolver())
 *                                      /root/reference/pkg/src/hcran_noma/dinkelbach.py:65-112
 *                                      fanned out by scenarios.run_sweep / run_draw
 *                                      (scenarios.py:237-296)
 *   hcran_b200_solve_fixed_e_batch  <- ScaleSolver.solve_fixed_e(ch, cfg, e, warm_start)
 *                                      (scale.py:506-551; the InnerSolver protocol,
 *                                      dinkelbach.py:28-33)
 *   hcran_b200_plan                 <- (no reference counterpart: workspace sizing)
 *   hcran_b200_version              <- hcran_noma.__version__ (__init__.py:36)
 *
 * Conventions: plain C types only; every array pointer is DEVICE memory owned
 * by the caller; arrays are row-major with the reference's [m][k][n] =
 * (RRH, user, subcarrier) index order (model.py:8-11).  Calls are
 * stream-ordered (`stream` is a cudaStream_t, NULL = legacy default), never
 * allocate, never synchronise the host, and are thread-safe across distinct
 * (stream, workspace) pairs.  Return value: 0 on success, a negative
 * HCRAN_E_* code on argument errors (nothing is launched then).  Per-instance
 * outcomes are reported through `status` (HCRAN_ST_*), mirroring the
 * reference's DinkelbachTrace.status / InnerResult.status / InfeasibleProblemError.
 */
#ifndef HCRAN_B200_H
#define HCRAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HCRAN_B200_ABI_VERSION 1

/* error codes (return values) */
#define HCRAN_OK 0
#define HCRAN_E_ARG (-1)        /* null pointer / bad dimension */
#define HCRAN_E_SIZE (-2)       /* M,K,N or l_max outside the supported range */
#define HCRAN_E_WORKSPACE (-3)  /* workspace too small (see hcran_b200_plan) */
#define HCRAN_E_LAUNCH (-4)     /* CUDA launch failure */

/* per-instance status codes */
#define HCRAN_ST_CONVERGED 0   /* Dinkelbach surplus <= xi            (dinkelbach.py:93-97)  */
#define HCRAN_ST_CAP 1         /* outer_max reached                   (dinkelbach.py:104-106) */
#define HCRAN_ST_STALLED 2     /* ee <= e, or a later inner infeasible (dinkelbach.py:82-102) */
#define HCRAN_ST_INFEASIBLE 3  /* first inner solve infeasible -> InfeasibleProblemError
                                  (dinkelbach.py:81-86); fixed-e: InnerResult "infeasible" */
#define HCRAN_ST_OK 0          /* fixed-e: InnerResult "ok" */
#define HCRAN_ST_UNSUPPORTED 4 /* device state capacity exceeded: more than 4 seats on one
                                  (m, n), > 64 tuple rows or > 1024 cross-head seat pairs
                                  (products-active families, scale.py:566, 861-895) */

/* Tolerances (model.py:59-80); rho1/rho2 already resolved from the mask. */
typedef struct hcran_tolerances {
  double xi;           /* Dinkelbach surplus stop                    */
  double varpi1_rel;   /* sweep stop, relative to p_max[m]           */
  double varpi2_rel;   /* round stop, relative to p_max[m]           */
  int32_t s_max;       /* SCA rounds                                 */
  int32_t v_max;       /* sweeps per round                           */
  int32_t outer_max;   /* Dinkelbach iterations                      */
  double rho1, rho2;   /* C10 / C11 product slack levels             */
  double dual_cap;     /* multiplier cap                             */
  double c13_rate_tol; /* streaming rate band                        */
  double c14_rel_tol;  /* SIC margin band                            */
  double box_rel_tol;  /* mask / budget band                         */
} hcran_tolerances_t;

/* Network configuration shared by every instance of a batch (NetworkConfig,
 * model.py:83-185).  All arrays are device pointers. */
typedef struct hcran_problem {
  int32_t M, K, N;        /* RRHs, users, subcarriers                         */
  int32_t l_max;          /* users per subcarrier (SIC cluster size)          */
  const double* p_max;    /* [M]        per-RRH budget, W                     */
  const double* p_mask;   /* [M][K][N]  spectral mask, W                      */
  const double* eta;      /* [M]        amplifier inefficiency                */
  const double* weights;  /* [M][K]     rate weights in [0, 1]                */
  const double* sigma;    /* [M][K][N]  noise power, W                        */
  double static_power;    /* fibre + circuit floor, W (model.py:173-176)      */
  hcran_tolerances_t tol;
  int32_t sic_mode;       /* HCRAN_SIC_SEATED (default), _DENSE or _SEATED_FAST */
} hcran_problem_t;

/* SIC multiplier family (scale.py:668-723, 776-819).  DENSE tracks a
 * multiplier for every oriented user pair on every (RRH, subcarrier), exactly
 * as the reference.  SEATED tracks the pairs whose members are both seated and
 * re-solves with DENSE any instance in which a seat's numerator vanishes while
 * its denominator is not positive (a "floor tie": the
 * reference then decides the seat from the floor-level (~1e-75) multipliers of
 * unseated pairs); ~7x faster than DENSE at config[1]. */
#define HCRAN_SIC_SEATED 0      /* default: exact on every golden draw        */
#define HCRAN_SIC_DENSE 1       /* dense family for every inner solve                     */
#define HCRAN_SIC_SEATED_FAST 2 /* seated family, floor ties NOT re-run (opt-in, inexact) */

/* Per-instance inputs. */
typedef struct hcran_batch_in {
  int64_t B;                /* instances                                      */
  const double* gamma;      /* [B][M][K][N] channel power gains (ChannelState.gamma) */
  const uint8_t* elastic;   /* [B][K] 1 = elastic user, 0 = streaming          */
  const double* min_rates;  /* [B][K] minimum rate, bits/s/Hz (0 for elastic)   */
  const double* e_fixed;    /* [B] fixed-e solves only (else ignored)          */
  const double* warm_p;     /* [B][M][K][N] fixed-e warm start or NULL         */
} hcran_batch_in_t;

/* Per-instance outputs (any pointer may be NULL to skip that output). */
typedef struct hcran_batch_out {
  double* p;             /* [B][M][K][N] PowerAllocation.p, W                  */
  uint8_t* rho;          /* [B][M][K][N] PowerAllocation.rho                   */
  uint8_t* a;            /* [B][M][K]    PowerAllocation.a                     */
  double* ee;            /* [B] EnergyReport.ee of the final allocation        */
  double* sum_rate;      /* [B] EnergyReport.sum_rate                          */
  double* total_power;   /* [B] EnergyReport.total_power                       */
  double* final_e;       /* [B] DinkelbachTrace.final_e (fixed-e: e)           */
  double* objective;     /* [B] R - e P of the returned allocation (true objective) */
  int32_t* outer_iters;  /* [B] len(DinkelbachTrace.iterations)                */
  int32_t* rounds;       /* [B] SCA rounds, summed over outer iterations       */
  int32_t* sweeps;       /* [B] power sweeps, summed over outer iterations     */
  int32_t* bisect_evals; /* [B] budget-multiplier load evaluations (work counter) */
  int8_t* status;        /* [B] HCRAN_ST_*                                     */
  uint8_t* feasible;     /* [B] check_feasibility(final).ok                    */
  double* xi;            /* [B][M] budget multipliers at the last sweep        */
  double* zeta;          /* [B][K] rate multipliers at the last sweep          */
  double* e_trace;       /* [B][outer_max] Dinkelbach e per iteration (nan-padded) */
  double* surplus_trace; /* [B][outer_max] surplus per iteration               */
  int32_t* rounds_trace; /* [B][outer_max] rounds per outer iteration          */
  int32_t* sweeps_trace; /* [B][outer_max] sweeps per outer iteration          */
  uint8_t* flags;        /* [B] HCRAN_FLAG_* diagnostics                        */
  double* work;          /* [B] algorithmic FP64 work, flop-equivalents */
  /* SolveStats of the last inner solve (scale.py:405-418) */
  double* round_obj;     /* [B][tol.s_max] surrogate objective per SCA round (nan-padded) */
  double* fp_residual;   /* [B] fixed-point residual |p - update(p)| / p_max at exit;
                            computed only when this pointer is set (one extra sweep) */
  double* max_dual;      /* [B] largest multiplier entry                         */
  int32_t* floor_hits;   /* [B] seated cells with den <= 1e-12 den_scale and num > 0 */
} hcran_batch_out_t;

/* flags: a seat met num == 0 with den <= 0 in the seated-pair SIC model, i.e.
 * the reference would decide it from floor-level multipliers of unseated pairs
 * (the instance is re-solved with the dense pair family). */
#define HCRAN_FLAG_FLOOR_TIE 1
#define HCRAN_FLAG_DENSE_RESOLVED 2 /* result comes from the dense-pair re-solve */

/* Workspace sizing: number of CTAs the solver will keep resident for this
 * problem on `device` and the device workspace bytes it needs. */
int hcran_b200_plan(const hcran_problem_t* prob, int64_t B, int device,
                    int32_t* grid_out, size_t* ws_bytes_out);

/* Full Dinkelbach solve of every instance (device-side outer loop). */
int hcran_b200_solve_batch(const hcran_problem_t* prob, const hcran_batch_in_t* in,
                           hcran_batch_out_t* out, void* workspace, size_t ws_bytes,
                           void* stream);

/* Energy report of given allocations (warm_p, [B][M][K][N]): sum rate, total
 * power, EE, objective at e_fixed (or 0), feasibility, rho / a -- the
 * reference's model.energy_efficiency / check_feasibility / derive_binaries
 * (model.py:338-341, 404-521).  Used by the host-driven Dinkelbach loop over
 * an arbitrary InnerSolver (dinkelbach.py:65-112). */
int hcran_b200_report_batch(const hcran_problem_t* prob, const hcran_batch_in_t* in,
                            hcran_batch_out_t* out, void* workspace, size_t ws_bytes,
                            void* stream);

/* Device-side channel synthesis: the instance loader of scenarios.py:84-153
 * (build_config's user drop + gen_channel) restated for the device.  Users are
 * uniform in a disc of radius `disc_radius` around the origin (r = R sqrt(U),
 * theta = 2 pi U), gains gamma[m][k][n] = Exp(1) * d(m,k)^-pathloss_exp.
 * Draw d uses Philox4x32-10 keyed by (seed, d): the reference's distributions,
 * not its numpy (PCG64) numbers -- parity fixtures use host-generated draws. */
typedef struct hcran_synth {
  int32_t M, K, N;
  const double* rrh_xy;  /* [M][2] RRH positions, metres (device)          */
  double disc_radius;    /* 500 m (scenarios.py DISC_RADIUS_M)             */
  double pathloss_exp;   /* 3                                              */
  uint64_t seed;
} hcran_synth_t;

/* Writes gamma_out[B][M][K][N] (device) for draws first_draw .. first_draw+B-1. */
int hcran_b200_synth_gamma(const hcran_synth_t* sp, int64_t first_draw, int64_t B,
                           double* gamma_out, void* stream);

/* One fixed-e inner solve per instance (InnerSolver conformance). */
int hcran_b200_solve_fixed_e_batch(const hcran_problem_t* prob, const hcran_batch_in_t* in,
                                   hcran_batch_out_t* out, void* workspace,
                                   size_t ws_bytes, void* stream);

/* Which engine the solver picks for this problem: engine 1 = shared-memory
 * rounds engine on a thread-block cluster of `cluster` CTAs (smem bytes per
 * CTA), engine 0 = global-workspace engine (shapes whose slices do not fit). */
int hcran_b200_engine(const hcran_problem_t* prob, int64_t B, int device, int32_t* engine,
                      int32_t* cluster, size_t* smem);

/* Kernel launches issued by the last successful call on this thread. */
int32_t hcran_b200_last_launches(void);

const char* hcran_b200_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HCRAN_B200_H */
