// hcran_kernel.cu -- C ABI of libhcran_b200.so (include/hcran_b200.h): launch
// planning, workspace layout, queue ordering, device channel synthesis.  The
// solve kernel itself is hcran_kernel.cuh (instantiated in hcran_k*.cu).
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include "hcran_kernel.cuh"

using namespace hcran;

struct Shape {
  int nt, gt;
};
// default shape per instance size (cells); HCRAN_SHAPE=NT:GT overrides
static Shape shape_of(const hcran_problem_t* p) {
  const char* e = getenv("HCRAN_SHAPE");
  if (e) {
    Shape s{0, 0};
    if (sscanf(e, "%d:%d", &s.nt, &s.gt) == 2) return s;
  }
  const int64_t cells = (int64_t)p->M * p->K * p->N;
  if (cells >= 16384) return Shape{512, 512};
  return Shape{256, 256};
}

// ---------------------------------------------------------------- queue order
// Per-instance work varies ~10x and the persistent queue
// hands instances out in order, so a costly instance popped late sets the
// makespan.  The queue is ordered by a predicted cost, longest first: the
// spread (standard deviation over users) of log10 of each user's best channel
// gain, which correlates with the instance's work (0.44-0.48 on independent
// c1 samples).  Counting sort over ORDER_NB buckets; the order inside a bucket
// is arbitrary -- results depend only on the instance.
#define ORDER_NB 256
#define ORDER_KEY_MAX 4.0

static __global__ void __launch_bounds__(256) hcran_order_key(View v, int32_t* bucket,
                                                              int32_t* hist) {
  __shared__ double lg[256];
  const int b = blockIdx.x, K = v.K, MN = v.M * v.N, N = v.N;
  const double* g = v.gamma + (size_t)b * v.M * K * N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = warp; k < K; k += blockDim.x >> 5) {
    double mx = 0.0;
    for (int c = lane; c < MN; c += 32) {
      const int m = c / N, n = c - m * N;
      mx = fmax(mx, g[((size_t)m * K + k) * N + n]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) lg[k] = log10(fmax(mx, 1e-300));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mean = 0.0, var = 0.0;
    for (int k = 0; k < K; ++k) mean += lg[k];
    mean /= K;
    for (int k = 0; k < K; ++k) var += (lg[k] - mean) * (lg[k] - mean);
    const double key = sqrt(var / K);
    int q = (int)(key * (ORDER_NB / ORDER_KEY_MAX));
    q = q < 0 ? 0 : (q >= ORDER_NB ? ORDER_NB - 1 : q);
    const int bk = ORDER_NB - 1 - q;  // bucket 0 = largest predicted cost
    bucket[b] = bk;
    atomicAdd(&hist[bk], 1);
  }
}

static __global__ void hcran_order_scan(int32_t* hist) {  // exclusive scan in place, 1 thread
  if (threadIdx.x == 0) {
    int32_t acc = 0;
    for (int i = 0; i < ORDER_NB; ++i) {
      const int32_t h = hist[i];
      hist[i] = acc;
      acc += h;
    }
  }
}

static __global__ void hcran_order_scatter(const int32_t* bucket, int32_t* offs, int32_t* order,
                                           int64_t B) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) order[atomicAdd(&offs[bucket[b]], 1)] = (int32_t)b;
}

static thread_local int32_t g_last_launches = 0;
// workspace: [0, HEADER) queue counters + order histogram (zeroed per launch),
// then flags [B], order + bucket [B] int32, then the CTA slots
static const size_t HEADER = 4096;
static const size_t HIST_OFF = 1024;

static int check_problem(const hcran_problem_t* p) {
  if (!p) return HCRAN_E_ARG;
  if (p->M < 1 || p->K < 1 || p->N < 1) return HCRAN_E_SIZE;
  if (p->K > 255 || p->N > 256 || p->M > 31) return HCRAN_E_SIZE;
  if (p->l_max < 1 || p->l_max > SMAX) return HCRAN_E_SIZE;
  if (p->sic_mode < HCRAN_SIC_SEATED || p->sic_mode > HCRAN_SIC_SEATED_FAST) return HCRAN_E_ARG;
  if (!p->p_max || !p->p_mask || !p->eta || !p->weights || !p->sigma) return HCRAN_E_ARG;
  return HCRAN_OK;
}

// workspace bytes of one instance slot
static size_t per_cta_bytes(const hcran_problem_t* p, bool dense = false) {
  Work w;
  return w.layout(nullptr, p->M, p->K, p->N, dense, shape_of(p).gt / 32);
}

static size_t flags_bytes(int64_t B) { return ((size_t)B + 255) & ~(size_t)255; }
static size_t order_bytes(int64_t B) { return 2 * (((size_t)B * 4 + 255) & ~(size_t)255); }

// CTAs for the dense re-solve pass: a few per SM at most, bounded to ~4 GiB of state
static int64_t dense_ctas(const hcran_problem_t* p, int64_t B, int64_t grid1) {
  size_t per = per_cta_bytes(p, true) * (shape_of(p).nt / shape_of(p).gt);
  int64_t g = (int64_t)(((size_t)4 << 30) / per);
  if (g > grid1) g = grid1;
  if (g > B) g = B;
  if (g < 1) g = 1;
  return g;
}

static KernelFn kernel_of(Shape s) {
  if (s.nt == 256 && s.gt == 256) return kernel_256_256();
  if (s.nt == 512 && s.gt == 512) return kernel_512_512();
  return nullptr;
}

// resident CTAs (one per SM: the kernels are register-bound at NT threads)
static int resident_ctas(int device, Shape sh, size_t smem) {
  int sms = 148, per_sm = 1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) sms = 148;
  const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel_of(sh), sh.nt, smem);
  if (e != cudaSuccess || per_sm < 1) per_sm = 1;
  if (per_sm > 8) per_sm = 8;  // state lives in the workspace: bound its footprint
  return sms * per_sm;
}

struct Plan {
  int64_t grid;      // CTAs of pass 1
  int64_t slots;     // pass-1 workspace slots (one per CTA)
  size_t per;        // bytes per slot
  int64_t grid2;     // CTAs of pass 2 (dense SIC family)
  size_t perd;
  size_t total;
  unsigned hot;      // Work::HOT_* arrays bound to dynamic shared memory
  size_t hot_smem;   // their bytes per CTA
  size_t hot_per;    // ... per instance (thread group)
  Shape sh;          // launch shape
  int groups;        // instances per CTA
  int dense_all;     // 1: every instance runs the dense SIC pair family in pass 1
  int dense_ok;      // 1: pass-1 slots carry the dense family (floor ties re-run in place)
};

// Shared-memory residency: the per-sweep streams of the analysis (decode
// ranks, gains, bound slopes, ...) are bound to dynamic shared memory in
// Work::HOT_* priority order while they fit the instance's share of
// HCRAN_HOT_KB (per CTA); an array that does not fit is skipped, the rest stay
// in the L1/L2-cached slot.
#ifndef HCRAN_HOT_KB_DEFAULT
#define HCRAN_HOT_KB_DEFAULT 16
#endif
static void choose_hot(const hcran_problem_t* prob, int maxsm, Plan* P) {
  const char* e = getenv("HCRAN_HOT_KB");
  size_t budget = (size_t)(e ? atoi(e) : HCRAN_HOT_KB_DEFAULT) * 1024;
  const size_t cap = (size_t)maxsm - 8192;  // static shared memory of the kernel
  if (budget > cap) budget = cap;
  budget /= P->groups;
  P->hot = 0;
  P->hot_per = 0;
  const char* mk = getenv("HCRAN_HOT_MASK");  // explicit Work::HOT_* bit mask (tuning sweeps)
  const unsigned want = mk ? (unsigned)strtoul(mk, nullptr, 0) : ~0u;
  for (int i = 0; i < Work::HOT_N; ++i) {
    if (!(want & (1u << i))) continue;
    const size_t b = (Work::hot_bytes(i, prob->M, prob->K, prob->N) + 15) & ~size_t(15);
    if (P->hot_per + b > budget) continue;
    P->hot |= 1u << i;
    P->hot_per += b;
  }
  P->hot_smem = P->hot_per * P->groups;
  if (P->hot_smem) cudaFuncSetAttribute(kernel_of(P->sh), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)P->hot_smem);
}

static int make_plan(const hcran_problem_t* prob, int64_t B, int device, Plan* P) {
  P->hot = 0;
  P->hot_smem = 0;
  P->sh = shape_of(prob);
  if (!kernel_of(P->sh)) return HCRAN_E_ARG;
  P->groups = P->sh.nt / P->sh.gt;
  const int64_t Bp = B > 0 ? B : 1;
  int maxsm = 0;
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (maxsm <= 0) maxsm = 232448;
  P->perd = per_cta_bytes(prob, true);
  P->dense_ok = 0;
  const char* dn = getenv("HCRAN_DENSE");
  P->dense_all = prob->sic_mode == HCRAN_SIC_DENSE ? 1 : 0;
  if (dn) P->dense_all = atoi(dn);
  choose_hot(prob, maxsm, P);
  int64_t g = resident_ctas(device, P->sh, P->hot_smem);
  const int64_t gneed = (Bp + P->groups - 1) / P->groups;
  if (g > gneed) g = gneed;
  P->grid = g;
  P->slots = g * P->groups;
  // floor ties are re-run in place when every slot can carry the dense family
  P->dense_ok = (!P->dense_all && prob->sic_mode != HCRAN_SIC_SEATED_FAST &&
                 (size_t)P->slots * P->perd <= ((size_t)24 << 30)) ? 1 : 0;
  P->per = per_cta_bytes(prob, P->dense_all != 0 || P->dense_ok != 0);
  P->grid2 = (P->dense_all || P->dense_ok || prob->sic_mode == HCRAN_SIC_SEATED_FAST)
                 ? 0 : dense_ctas(prob, Bp, P->grid);
  P->total = HEADER + flags_bytes(Bp) + order_bytes(Bp) + (size_t)P->slots * P->per +
             (size_t)P->grid2 * P->groups * P->perd;
  return HCRAN_OK;
}

extern "C" int hcran_b200_plan(const hcran_problem_t* prob, int64_t B, int device,
                               int32_t* grid_out, size_t* ws_bytes_out) {
  int rc = check_problem(prob);
  if (rc) return rc;
  if (B < 0 || !grid_out || !ws_bytes_out) return HCRAN_E_ARG;
  Plan P;
  make_plan(prob, B, device, &P);
  *grid_out = (int32_t)P.grid;
  *ws_bytes_out = P.total;
  return HCRAN_OK;
}

static int launch(const hcran_problem_t* prob, const hcran_batch_in_t* in, hcran_batch_out_t* out,
                  void* workspace, size_t ws_bytes, void* stream, int mode) {
  g_last_launches = 0;
  int rc = check_problem(prob);
  if (rc) return rc;
  if (!in || !out || !workspace || !in->gamma || !in->elastic || !in->min_rates) return HCRAN_E_ARG;
  if (mode == 1 && !in->e_fixed) return HCRAN_E_ARG;
  if (mode == 2 && !in->warm_p) return HCRAN_E_ARG;
  if (prob->tol.s_max > RMAX) return HCRAN_E_SIZE;
  if (in->B <= 0) return HCRAN_OK;
  int device = 0;
  cudaGetDevice(&device);
  Plan P;
  rc = make_plan(prob, in->B, device, &P);
  if (rc) return rc;
  if (ws_bytes < P.total) return HCRAN_E_WORKSPACE;
  View v;
  v.M = prob->M; v.K = prob->K; v.N = prob->N; v.L = prob->l_max;
  v.p_max = prob->p_max; v.mask = prob->p_mask; v.eta = prob->eta; v.w = prob->weights;
  v.sig = prob->sigma; v.static_power = prob->static_power; v.tol = prob->tol;
  v.B = in->B; v.gamma = in->gamma; v.elastic = in->elastic; v.min_rates = in->min_rates;
  v.e_fixed = in->e_fixed; v.warm_p = in->warm_p; v.out = *out;
  cudaStream_t s = (cudaStream_t)stream;
  char* base = (char*)workspace;
  uint8_t* flags = (uint8_t*)(base + HEADER);
  int32_t* order = (int32_t*)(base + HEADER + flags_bytes(in->B));
  int32_t* bucket = order + order_bytes(in->B) / 8;
  char* slots1 = base + HEADER + flags_bytes(in->B) + order_bytes(in->B);
  char* slots2 = slots1 + (size_t)P.slots * P.per;
  if (cudaMemsetAsync(base, 0, HEADER, s) != cudaSuccess) return HCRAN_E_LAUNCH;
  // pass-1 floor-tie flags only when a second pass will re-solve the flagged instances
  v.dense = P.dense_all ? 1 : 0; v.dense_ok = P.dense_ok; v.flag_int = P.grid2 ? flags : nullptr;
  v.flag_in = nullptr;
  v.order = nullptr;
  int launches = 0;
  const char* ord_env = getenv("HCRAN_ORDER");
  if (in->B > P.slots && !(ord_env && atoi(ord_env) == 0)) {  // queue order matters past one wave
    int32_t* hist = (int32_t*)(base + HIST_OFF);
    hcran_order_key<<<(unsigned)in->B, 256, 0, s>>>(v, bucket, hist);
    hcran_order_scan<<<1, 32, 0, s>>>(hist);
    hcran_order_scatter<<<(unsigned)((in->B + 255) / 256), 256, 0, s>>>(bucket, hist, order, in->B);
    if (cudaGetLastError() != cudaSuccess) return HCRAN_E_LAUNCH;
    v.order = order;
    launches = 3;
  }
  const KernelFn kfn = kernel_of(P.sh);
  kfn<<<(unsigned)P.grid, P.sh.nt, P.hot_smem, s>>>(v, slots1, P.per, (int*)base, mode, P.hot, P.hot_per);
  if (cudaGetLastError() != cudaSuccess) return HCRAN_E_LAUNCH;
  if (P.grid2 == 0) {  // pass 1 already settled every floor tie (or the fast model ignores them)
    g_last_launches = launches + 1;
    return HCRAN_OK;
  }
  v.dense = 1; v.dense_ok = 0; v.flag_int = nullptr; v.flag_in = flags;
  kfn<<<(unsigned)P.grid2, P.sh.nt, P.hot_smem, s>>>(v, slots2, P.perd, (int*)base + 1, mode, P.hot,
                                                     P.hot_per);
  if (cudaGetLastError() != cudaSuccess) return HCRAN_E_LAUNCH;
  g_last_launches = launches + 2;
  return HCRAN_OK;
}

extern "C" int hcran_b200_engine(const hcran_problem_t* prob, int64_t B, int device,
                                 int32_t* engine, int32_t* cluster, size_t* smem) {
  int rc = check_problem(prob);
  if (rc) return rc;
  Plan P;
  make_plan(prob, B, device, &P);
  if (engine) *engine = 0;   // one CTA per instance (the cluster engine of round 1 is gone)
  if (cluster) *cluster = 1;
  if (smem) *smem = P.hot_smem;
  return HCRAN_OK;
}

extern "C" int hcran_b200_solve_batch(const hcran_problem_t* prob, const hcran_batch_in_t* in,
                                      hcran_batch_out_t* out, void* workspace, size_t ws_bytes,
                                      void* stream) {
  return launch(prob, in, out, workspace, ws_bytes, stream, 0);
}

extern "C" int hcran_b200_solve_fixed_e_batch(const hcran_problem_t* prob,
                                              const hcran_batch_in_t* in, hcran_batch_out_t* out,
                                              void* workspace, size_t ws_bytes, void* stream) {
  return launch(prob, in, out, workspace, ws_bytes, stream, 1);
}

extern "C" int hcran_b200_report_batch(const hcran_problem_t* prob, const hcran_batch_in_t* in,
                                       hcran_batch_out_t* out, void* workspace, size_t ws_bytes,
                                       void* stream) {
  return launch(prob, in, out, workspace, ws_bytes, stream, 2);
}

extern "C" int32_t hcran_b200_last_launches(void) { return g_last_launches; }

// phase profiler readout (only meaningful in a -DHCRAN_PROFILE build)
extern "C" int hcran_b200_phase_cycles(unsigned long long* out32, int reset) {
#if defined(HCRAN_PROFILE)
  // each kernel translation unit has its own counters: sum them
  unsigned long long a[32], b[32];
  phase_cycles_256(a, reset);
  phase_cycles_512(b, reset);
  for (int i = 0; i < 32; ++i) out32[i] = a[i] + b[i];
  return 0;
#else
  for (int i = 0; i < 32; ++i) out32[i] = 0;
  (void)reset;
  return -1;
#endif
}

extern "C" const char* hcran_b200_version(void) {
  return "hcran_b200 0.1.0 (abi 1, sm_100a, fp64 core)";
}

// --------------------------------------------------------- channel synthesis
// Device-side instance loader (scenarios.py:84-153, restated): users uniform
// in the coverage disc (r = R sqrt(U), theta = 2 pi U), gains Exp(1) * d^-3 per
// (RRH, user, subcarrier), written straight into the solver's input layout so
// a large batch (config[3]: ~4 MiB of gains per instance) never exists on the
// host.  Counter-based Philox4x32-10 keyed by (seed, draw): every draw is
// reproducible on any GPU and any shard, and shards are disjoint by draw index.
namespace {
struct Philox {
  __device__ static void round(uint32_t c[4], uint32_t k[2]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
    const uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
    const uint32_t o0 = hi1 ^ c[1] ^ k[0], o1 = lo1, o2 = hi0 ^ c[3] ^ k[1], o3 = lo0;
    c[0] = o0; c[1] = o1; c[2] = o2; c[3] = o3;
  }
  // 4 x 32 random bits for (seed, draw, index)
  __device__ static void gen(uint64_t seed, uint64_t draw, uint64_t idx, uint32_t out[4]) {
    uint32_t c[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), (uint32_t)draw, (uint32_t)(draw >> 32)};
    uint32_t k[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      round(c, k);
      k[0] += 0x9E3779B9u;
      k[1] += 0xBB67AE85u;
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
  }
  // uniform double in [0, 1) from 64 bits (53-bit mantissa)
  __device__ static double u01(uint32_t a, uint32_t b) {
    const uint64_t v = (((uint64_t)a << 32) | b) >> 11;
    return (double)v * 0x1p-53;
  }
};
}  // namespace

static __global__ void __launch_bounds__(256) hcran_synth_kernel(hcran_synth_t sp, int64_t first,
                                                                 int64_t B, double* gamma) {
  extern __shared__ double dpl[];  // [M][K]: d^-pathloss
  const int M = sp.M, K = sp.K, N = sp.N;
  const int64_t b = blockIdx.x;
  if (b >= B) return;
  const uint64_t draw = (uint64_t)(first + b);
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    uint32_t r4[4];
    Philox::gen(sp.seed, draw, (uint64_t)k, r4);
    const double r = sp.disc_radius * sqrt(Philox::u01(r4[0], r4[1]));
    const double th = 2.0 * 3.141592653589793 * Philox::u01(r4[2], r4[3]);
    const double x = r * cos(th), y = r * sin(th);
    for (int m = 0; m < M; ++m) {
      const double dx = sp.rrh_xy[2 * m] - x, dy = sp.rrh_xy[2 * m + 1] - y;
      dpl[m * K + k] = pow(sqrt(dx * dx + dy * dy), -sp.pathloss_exp);
    }
  }
  __syncthreads();
  const int64_t C = (int64_t)M * K * N;
  double* g = gamma + b * C;
  for (int64_t c2 = threadIdx.x; 2 * c2 < C; c2 += blockDim.x) {  // two cells per draw of 4 words
    uint32_t r4[4];
    Philox::gen(sp.seed, draw, (uint64_t)K + (uint64_t)c2, r4);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t c = 2 * c2 + h;
      if (c >= C) break;
      const double chi = -log1p(-Philox::u01(r4[2 * h], r4[2 * h + 1]));  // Exp(1)
      g[c] = chi * dpl[c / N];  // [m][k][n]: (m * K + k) = c / N
    }
  }
}

extern "C" int hcran_b200_synth_gamma(const hcran_synth_t* sp, int64_t first_draw, int64_t B,
                                      double* gamma_out, void* stream) {
  if (!sp || !gamma_out || !sp->rrh_xy) return HCRAN_E_ARG;
  if (sp->M < 1 || sp->K < 1 || sp->N < 1 || (size_t)sp->M * sp->K * 8 > 48 * 1024) return HCRAN_E_SIZE;
  if (B <= 0) return HCRAN_OK;
  hcran_synth_kernel<<<(unsigned)B, 256, (size_t)sp->M * sp->K * sizeof(double), (cudaStream_t)stream>>>(
      *sp, first_draw, B, gamma_out);
  return cudaGetLastError() == cudaSuccess ? HCRAN_OK : HCRAN_E_LAUNCH;
}
