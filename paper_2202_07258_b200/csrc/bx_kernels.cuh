// bx_kernels.cuh -- sm_100a kernels of the screened box-constrained LS iteration.
//
// Hot path:
//   k_pass     one streamed pass over the preserved columns A_act.  Each CTA
//              owns a contiguous range of columns, stages them whole into a
//              shared-memory ring with cp.async.bulk (TMA bulk engine,
//              mbarrier completion) and, per column j,
//                 g_j   = a_j . v            (dot; v = residual / extrapolated residual)
//                 x_j'  = clip(y_j - eta g_j, l_j, u_j)    (PG / FISTA update)
//                 acc  += a_j x_j'           (the next residual's partial A x')
//              so ONE read of A serves both products of a projected-gradient
//              step (solvers.py:109-116 does two GEMV passes).  Each thread
//              owns R row chunks of 16-byte vectors, R the smallest count
//              covering m, so chunks 0..R-2 run without row guards (the pass
//              is issue-limited under the board power cap).  Modes cover
//              the screening pass (dot + epsilon partial), power iteration
//              (solvers.py:78-85) and plain A x (refresh, certified gap).
//   k_reduce   sums the per-CTA partial rows in a fixed order (deterministic),
//              adds the offset z - y, and in its last CTA finalises the
//              objective, the StepSizeTooLarge guard (solvers.py:111-114) or
//              the FISTA restart test.
//   k_dual     dual translation/scaling + reduced dual + gap clamp + radius +
//              slack (driver.py:183-201, 213-219; duality.py:154-156).
//   k_sphere / k_scan / k_compact / k_gather
//              gap-safe sphere test (screening.py:60-69) with warp-ballot /
//              block prefix-sum compaction of the preserved set and the
//              physical rewrite of A_act (solvers.py:57).
#pragma once
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <stdint.h>
#include <math.h>

namespace bx {

#ifndef BX_NT
#define BX_NT 512
#endif
constexpr int NT = BX_NT;          // k_pass block size
constexpr int RMAX = 12 * 512 / NT;  // register-resident envelope: R * NT * V covers m <= 12288 fp64 / 24576 fp32
constexpr int NWARPS = NT / 32;
constexpr int CMAX = 8;            // columns per ring slot (max)
constexpr int SMAX = 8;            // ring slots (max)
constexpr int RT = 256;            // block size of the vector kernels
constexpr int PASS_STAGED = 7;     // per-column state arrays a pass may stage in shared memory

// device-resident round records (small-round kernel, graph rounds): primal,
// dual, gap, eps, radius, momentum, restarts, %globaltimer at the round's
// end (ns), gap-evaluation time excluded so far in the batch (ns, screening
// off: the reference's offline-gap convention, driver.py:180-181)
constexpr int TRACE_W = 10;

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_stamp(unsigned long long* slot) { *slot = globaltimer(); }

template <typename T> struct V16;
template <> struct V16<double> { using type = double2; static constexpr int n = 2; };
template <> struct V16<float> { using type = float4; static constexpr int n = 4; };

enum PassUpd : int {
  U_DOT = 0,    // g_j = a_j . v ; epsilon partial over infinite-upper columns
  U_PG_G = 1,   // x_j' = clip(x_j - eta g_j) with the stored g (no dot)
  U_PG = 2,     // dot + PG update
  U_APG = 3,    // dot on r_y = r + beta (r - r_prev), FISTA update
  U_POWER = 4,  // w_j = a_j . u ; acc += a_j w_j ; sum w_j^2
  U_AX = 5      // acc += a_j c_j (c = coef or x)
};

enum ReduceMode : int { R_PLAIN = 0, R_SET = 1, R_PG = 2, R_APG = 3, R_POWER = 4, R_CERT = 5 };
// or-ed into R_PG / R_APG for the speculative round-boundary step: the
// objective / momentum before the step are kept (bak_*) and a step error is
// recorded in err_spec, because the step is undone when the round's
// screening event changes the problem it was taken on
constexpr int R_SPEC = 16;

enum DevErr : int {
  DE_NONE = 0, DE_STEP_TOO_LARGE = 4, DE_INTERNAL_CONSISTENCY = 5, DE_POWER_ZERO = 64, DE_PEER_TIMEOUT = 65
};

// Scalars shared by the kernels of one context (device memory).
struct DualOut {
  double primal, dual, gap, gap_raw, eps, radius, slack, thr, th_norm2;
};

struct DevScalars {
  double eta;       // step in force
  double P;         // 0.5 ||r||^2 of the current residual
  double P_prev;    // objective before the last pass (error reporting)
  double mom_t;     // FISTA momentum scalar t_k
  double nw;        // power iteration ||w||
  double sigma;     // sqrt(nw)
  double cert_P;    // 0.5 ||A x - y||^2 on the full problem
  DualOut act;      // reduced-problem dual point of this round
  DualOut cert;     // certified (full-problem) dual point
  double rise_rel;  // StepSizeTooLarge tolerance: 1e-9 + rise_rel * P (0 for fp64, solvers.py:112)
  double rs_f;      // FISTA restart slacks (1e-12 fp64; fp32 values sized to fp32 round-off)
  double rs_g;
  double err_v1, err_v2;  // objective values at a StepSizeTooLarge event
  // state before the speculative round-boundary step (restored on undo)
  double bak_P, bak_mom_t;
  double spec_v1, spec_v2;  // objective values of a speculative StepSizeTooLarge
  // this rank's sphere-test counts; n_dirty = screened columns whose iterate
  // around the speculative step is off the bound (the step must be undone)
  int64_t n_keep, n_lo, n_up, n_dirty;
  int64_t g_keep, g_lo, g_up, g_dirty;  // summed over ranks (== local on one GPU)
  int32_t err;
  int32_t restarts;
  int32_t bak_restarts;
  int32_t err_spec;  // StepSizeTooLarge raised by the speculative step
  unsigned int counters[8];
};

template <typename T>
struct PassArgs {
  const T* A;              // column base
  int64_t ld;              // column stride (elements)
  const int32_t* colmap;   // column p lives at A + colmap[p]*ld (NULL: p)
  int64_t k;               // columns in this pass
  int64_t m;               // rows
  // every vector is fp64; only A (and the per-CTA partial rows) has the
  // storage type T -- fp32 storage halves the streamed bytes without
  // lowering the precision of the iterate ("fp32")
  const double* vin;       // dot vector (residual / power vector)
  const double* vin_prev;  // row-blocked dot with an extrapolated vector (unused by the fused modes)
  double* x;               // iterate (updated in place)
  double* xprev;           // FISTA previous iterate (PG speculative step: x before the step)
  double* gprev;           // FISTA: gradient at the previous iterate (read g_{k-1}, written g_k)
  const double* lo;
  const double* hi;
  double* g;               // gradient A'v (written by dot modes, read by U_PG_G)
  const double* att;       // A't for the epsilon partial
  const double* nrm;       // ||a_j|| (FISTA restart slack)
  const double* coef;      // U_AX coefficients (NULL: x)
  T* part;                 // [gridDim.x][ldp] partial rows of A x' (fp32 accumulation for T = float)
  int64_t ldp;
  double* bpart;           // [gridDim.x] block scalar partial (eps max / sum w^2)
  DevScalars* sc;
  int upd;
  int has_inf;
  int C;                   // columns per ring slot
  int S;                   // ring slots
  uint32_t colbytes;       // bytes moved per column (multiple of 16)
  uint32_t colstride;      // smem bytes per column in a slot
  int pre;                 // >= columns per CTA: the CTA's per-column state is staged in smem (0: off)
  int accumulate;          // U_DOT over a row block: g[p] = (accumulate ? g[p] : 0) + block dot, no epsilon
  int extrap;              // dot with the FISTA extrapolated residual r + beta (r - r_prev)
  // speculative round-boundary step (U_PG / U_APG): the pass's dot is also
  // the round's screening gradient -- g[p] = g_k, epsilon partial -> epart;
  // FISTA keeps x_{k-1} / g_{k-1} in xbak / gbak for an undo
  int spec;
  int zskip;               // skip the axpy of zero coefficients (0 only with env BX_NO_ZSKIP: exactness test)
  double* xbak;
  double* gbak;
  double* epart;           // [gridDim.x] epsilon partial (block max)
  // fused reduce (PG / FISTA step on one GPU, cooperative launch): after the
  // stream, the CTAs reduce the partial rows themselves -- rout = sum of
  // partials + roff, rsave = rout's previous contents (speculative step) --
  // and the last CTA folds the objective / restart test (rmode, as k_reduce)
  int fuse;
  const double* roff;
  double* rout;
  double* rsave;
  double* rpart;           // [gridDim.x] per-CTA ||r||^2 partials
  int rmode;
  int rcounter;
};

template <typename T>
__device__ void pass_fused_reduce(const PassArgs<T>& a, unsigned char* scratch);

// ----------------------------------------------------------------------------
// PTX helpers: mbarrier + bulk copy (TMA bulk engine, SASS UBLKCP)
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void set_err(DevScalars* sc, int code) { atomicCAS(&sc->err, 0, code); }

// numpy-order scalar helpers (no FMA contraction, so the update matches
// `np.clip(x - eta * g, lo, hi)` operation by operation)
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
// np.clip(v, lo, hi) == minimum(maximum(v, lo), hi) for non-NaN input
template <typename T>
__device__ __forceinline__ T clip(T v, T lo, T hi) {
  const T a = v < lo ? lo : v;
  return a > hi ? hi : a;
}

template <typename T>
__device__ __forceinline__ void unpack(const typename V16<T>::type& v, T* o);
template <>
__device__ __forceinline__ void unpack<double>(const double2& v, double* o) {
  o[0] = v.x;
  o[1] = v.y;
}
template <>
__device__ __forceinline__ void unpack<float>(const float4& v, float* o) {
  o[0] = v.x;
  o[1] = v.y;
  o[2] = v.z;
  o[3] = v.w;
}
template <typename T>
__device__ __forceinline__ typename V16<T>::type pack(const T* o);
template <>
__device__ __forceinline__ double2 pack<double>(const double* o) {
  return make_double2(o[0], o[1]);
}
template <>
__device__ __forceinline__ float4 pack<float>(const float* o) {
  return make_float4(o[0], o[1], o[2], o[3]);
}

// packed fp32 FMA, SASS FFMA2 (sm_100a): d = a * b + c on two lanes, each
// lane rounded exactly like a scalar fma.rn.f32
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n.reg .b64 ra, rb, rc, rd;\nmov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\nmov.b64 rc, {%6, %7};\n"
      "fma.rn.f32x2 rd, ra, rb, rc;\nmov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
// acc[e] += a[e] * v[e], e < 4
__device__ __forceinline__ void fma2_acc(float* acc, const float* a, const float* v) {
  const float2 lo = ffma2(make_float2(a[0], a[1]), make_float2(v[0], v[1]), make_float2(acc[0], acc[1]));
  const float2 hi = ffma2(make_float2(a[2], a[3]), make_float2(v[2], v[3]), make_float2(acc[2], acc[3]));
  acc[0] = lo.x; acc[1] = lo.y; acc[2] = hi.x; acc[3] = hi.y;
}
// acc[e] += a[e] * c, e < 4
__device__ __forceinline__ void fma2_axpy(float* acc, const float* a, float c) {
  const float2 cc = make_float2(c, c);
  const float2 lo = ffma2(make_float2(a[0], a[1]), cc, make_float2(acc[0], acc[1]));
  const float2 hi = ffma2(make_float2(a[2], a[3]), cc, make_float2(acc[2], acc[3]));
  acc[0] = lo.x; acc[1] = lo.y; acc[2] = hi.x; acc[3] = hi.y;
}

// V consecutive fp64 values -> registers of type T (16-byte vector loads)
template <typename T>
__device__ __forceinline__ void load_rows(const double* p, double* o) {
  constexpr int V = V16<T>::n;
#pragma unroll
  for (int h = 0; h < V / 2; ++h) {
    const double2 q = *reinterpret_cast<const double2*>(p + 2 * h);
    o[2 * h] = q.x;
    o[2 * h + 1] = q.y;
  }
}

// columns per slot as a function of R (rows-per-thread chunks)
__host__ __device__ constexpr int cols_per_slot(int R) { return R >= 6 ? 1 : (R >= 4 ? 2 : (R >= 2 ? 4 : 8)); }

// ----------------------------------------------------------------------------
// k_pass: one streamed pass over k columns (see header comment)
// ----------------------------------------------------------------------------
// AT: accumulation type of the dot vector, the dots and the partial rows --
// T for the hot passes; double for fp32 storage in the rare certificate
// passes (then a.part holds fp64 partial rows)
template <typename T, int R, bool DOT, bool AXPY, typename AT = T>
__global__ void __launch_bounds__(NT, 1) k_pass(const PassArgs<T> a) {
  using VT = typename V16<T>::type;
  constexpr int V = V16<T>::n;
  constexpr int C = cols_per_slot(R);
  extern __shared__ __align__(1024) unsigned char smem[];
  const int tid = threadIdx.x;
  const int m = static_cast<int>(a.m);
  const int row0 = tid * V;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int64_t G = gridDim.x;
  const int64_t b = blockIdx.x;
  const int64_t p0 = a.k * b / G;
  const int64_t p1 = a.k * (b + 1) / G;
  const int ncol = static_cast<int>(p1 - p0);
  const int S = a.S;
  const int ngroups = (ncol + C - 1) / C;
  const uint32_t slot_bytes = C * a.colstride;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * slot_bytes);
  double* red = reinterpret_cast<double*>(bars + SMAX);  // [NWARPS][C]
  double* cf = red + NWARPS * CMAX;                      // [C] axpy coefficients
  double* bscr = cf + CMAX;                              // [3][CMAX] block scalar scratch
  double* s_step = bscr + 3 * CMAX;                      // [2] step eta, FISTA momentum coefficient
  double* stg = s_step + 2;                              // [PASS_STAGED][pre] staged per-column state

  // step eta and FISTA's momentum coefficient, computed once per CTA and read
  // by the per-column epilogue from shared memory (short epilogue chain, and
  // no registers held across the streaming loop)
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    s_step[0] = a.sc->eta;
    const double t = a.sc->mom_t;
    const double tn = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
    s_step[1] = (t - 1.0) / tn;
  }
  __syncthreads();

  uint64_t pol = 0;
  if (tid == 0) {
    pol = policy_evict_first();
    const int pre = ngroups < S ? ngroups : S;
    for (int gi = 0; gi < pre; ++gi) {
      const int cg = min(C, ncol - gi * C);
      mbar_expect_tx(&bars[gi], cg * a.colbytes);
      for (int c = 0; c < cg; ++c) {
        const int64_t p = p0 + (int64_t)gi * C + c;
        const int64_t col = a.colmap ? (int64_t)a.colmap[p] : p;
        bulk_g2s(smem + gi * slot_bytes + c * a.colstride, a.A + col * a.ld, a.colbytes, &bars[gi], pol);
      }
    }
  }

  // the dot vector, register resident: thread owns rows (i*NT + tid)*V + e.
  // FISTA dots the plain residual r_k: the extrapolated gradient is formed
  // per column by linearity, g_y = g_k + beta (g_k - g_{k-1}),
  // so the dot is also the gradient at x_k -- the round's screening gradient
  AT vr[DOT ? R : 1][V];
  double beta = 0.0;   // extrapolation of the dot vector (row-blocked dots only)
  auto step_eta = [&]() { return s_step[0]; };
  auto momentum_beta = [&]() { return s_step[1]; };
  if (DOT) {
    if (a.extrap) {
      const double t = a.sc->mom_t;
      const double tn = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
      beta = (t - 1.0) / tn;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int row = row0 + i * (NT * V);
#pragma unroll
      for (int e = 0; e < V; ++e) vr[i][e] = AT(0);
      if (row < m) {
        double cur[V];
        load_rows<T>(a.vin + row, cur);
        if (beta != 0.0) {
          double prv[V];
          load_rows<T>(a.vin_prev + row, prv);
#pragma unroll
          for (int e = 0; e < V; ++e) cur[e] = add_rn(cur[e], mul_rn(beta, sub_rn(cur[e], prv[e])));
        }
#pragma unroll
        for (int e = 0; e < V; ++e) vr[i][e] = (row + e < m) ? static_cast<AT>(cur[e]) : AT(0);
      }
    }
  }

  AT acc[AXPY ? R : 1][V];
#pragma unroll
  for (int i = 0; i < (AXPY ? R : 1); ++i)
#pragma unroll
    for (int e = 0; e < V; ++e) acc[i][e] = AT(0);

  double run = 0.0;   // block-scalar running value (threads tid < C)
  double run2 = 0.0;  // second block scalar (FISTA restart slack)
  double run3 = 0.0;  // speculative step: epsilon partial (max)

  // Stage this CTA's per-column state in shared memory once (coalesced), so
  // the per-column update between the two barriers never waits on HBM.
  const bool staged = a.pre >= ncol && a.pre > 0;
  // slots: U_DOT hi, att | U_PG_G x, lo, hi, g | U_PG x, lo, hi, -, -, -, att |
  // U_APG x, lo, hi, x_prev, ||a||, g_prev, att | U_AX coef
  // (no pointer per slot: the epilogue indexes stg directly -- fewer live
  // registers in the R = 10..12 instantiations)
#define BX_STG(f) stg[(f) * a.pre + ql]
  const bool want_att = a.spec && a.has_inf;
  if (staged) {
    const double* src[PASS_STAGED] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    switch (a.upd) {
      case U_DOT: src[0] = a.hi; src[1] = a.att; break;
      case U_PG_G: src[0] = a.x; src[1] = a.lo; src[2] = a.hi; src[3] = a.g; break;
      case U_PG: src[0] = a.x; src[1] = a.lo; src[2] = a.hi; if (want_att) src[6] = a.att; break;
      case U_APG:
        src[0] = a.x; src[1] = a.lo; src[2] = a.hi; src[3] = a.xprev; src[4] = a.nrm; src[5] = a.gprev;
        if (want_att) src[6] = a.att;
        break;
      case U_AX: src[0] = a.coef ? a.coef : a.x; break;
      default: break;
    }
    for (int f = 0; f < PASS_STAGED; ++f)
      if (src[f])
        for (int q = tid; q < ncol; q += NT) stg[f * a.pre + q] = src[f][p0 + q];
    __syncthreads();
  }

  // ring slot / mbarrier phase of group gi: a running counter (no integer
  // division per column; A/B on the B200 with the unguarded chunk loops:
  // ~2% faster for fp64 under the power cap, ~5% for fp32)
  int s_run = 0;
  uint32_t ph_run = 0;
  for (int gi = 0; gi < ngroups; ++gi) {
    const int s = s_run;
    const uint32_t ph = ph_run;
    const int cg = min(C, ncol - gi * C);
    mbar_wait(&bars[s], ph);
    const unsigned char* slot = smem + s * slot_bytes;
    if (DOT) {
      AT d[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        d[c] = AT(0);
        if (c < cg) {
          const T* col = reinterpret_cast<const T*>(slot + c * a.colstride);
          if constexpr (sizeof(T) == 8) {
            // fp64: one chain per thread (measured faster than split sums
            // here); chunks 0 .. R-2 are full (see the fp32 path): no guards
#pragma unroll
            for (int i = 0; i < R - 1; ++i) {
              T av[V];
              unpack<T>(*reinterpret_cast<const VT*>(col + row0 + i * (NT * V)), av);
#pragma unroll
              for (int e = 0; e < V; ++e) d[c] += av[e] * vr[i][e];
            }
            {
              const int row = row0 + (R - 1) * (NT * V);
              if (row < m) {
                T av[V];
                unpack<T>(*reinterpret_cast<const VT*>(col + row), av);
#pragma unroll
                for (int e = 0; e < V; ++e) d[c] += ((row + e < m) ? av[e] : T(0)) * vr[R - 1][e];
              }
            }
          } else if constexpr (sizeof(AT) == 8) {
            // fp32 storage, fp64 accumulation (certificate passes)
            double dd[V];
#pragma unroll
            for (int e = 0; e < V; ++e) dd[e] = 0.0;
#pragma unroll
            for (int i = 0; i < R; ++i) {
              const int row = row0 + i * (NT * V);
              if (row < m) {
                T av[V];
                unpack<T>(*reinterpret_cast<const VT*>(col + row), av);
#pragma unroll
                for (int e = 0; e < V; ++e)
                  if (row + e < m) dd[e] += static_cast<double>(av[e]) * vr[i][e];
              }
            }
            d[c] = dd[0];
#pragma unroll
            for (int e = 1; e < V; ++e) d[c] += dd[e];
          } else {
          // fp32 (twice the elements per byte): V independent partial sums
          // (short dependency chains) combined in a fixed order; only the
          // vector holding row m-1 needs a guard
          T dd[V];
#pragma unroll
          for (int e = 0; e < V; ++e) dd[e] = T(0);
          // chunks 0 .. R-2 are full for every thread (R is the smallest
          // with R * NT * V >= m): no row guards, no divergence bookkeeping
#pragma unroll
          for (int i = 0; i < R - 1; ++i) {
            T av[V];
            unpack<T>(*reinterpret_cast<const VT*>(col + row0 + i * (NT * V)), av);
            // packed fp32 FMA (FFMA2): same per-element fma.rn as the
            // scalar chains, half the issue slots
            fma2_acc(dd, av, vr[i]);
          }
#pragma unroll
          for (int i = R - 1; i < R; ++i) {
            const int row = row0 + i * (NT * V);
            if (row + V <= m) {
              T av[V];
              unpack<T>(*reinterpret_cast<const VT*>(col + row), av);
              fma2_acc(dd, av, vr[i]);
            } else if (row < m) {
              T av[V];
              unpack<T>(*reinterpret_cast<const VT*>(col + row), av);
#pragma unroll
              for (int e = 0; e < V; ++e)
                if (row + e < m) dd[e] += av[e] * vr[i][e];
            }
          }
          d[c] = dd[0];
#pragma unroll
          for (int e = 1; e < V; ++e) d[c] += dd[e];
          }
        }
        d[c] = warp_sum<AT>(d[c]);
      }
      if (lane == 0) {
#pragma unroll
        for (int c = 0; c < C; ++c) red[warp * CMAX + c] = static_cast<double>(d[c]);
      }
      __syncthreads();
      if (tid < cg) {
        double gsum = 0.0;
#pragma unroll
        for (int w = 0; w < NWARPS; ++w) gsum += red[w * CMAX + tid];
        const double gj = gsum;
        const int ql = gi * C + tid;  // local column index
        const int64_t p = p0 + ql;
        double coef = 0.0;
        switch (a.upd) {
          case U_DOT: {
            if (a.accumulate >= 0) {  // row-blocked path: partial dot of this row block
              a.g[p] = a.accumulate ? add_rn(a.g[p], gj) : gj;
              break;
            }
            a.g[p] = gj;
            const double hj = staged ? BX_STG(0) : a.hi[p];
            if (a.has_inf && isinf(hj)) {
              const double ratio = fmax(-gj, 0.0) / fabs(staged ? BX_STG(1) : a.att[p]);
              run = fmax(run, ratio);
            }
          } break;
          case U_PG: {
            const double eta = step_eta();
            a.g[p] = gj;
            const double xo = staged ? BX_STG(0) : a.x[p];
            const double hj = staged ? BX_STG(2) : a.hi[p];
            const double xn = clip<double>(sub_rn(xo, mul_rn(eta, gj)), staged ? BX_STG(1) : a.lo[p], hj);
            if (a.spec) {
              a.xprev[p] = xo;  // x_k, for an undo
              if (a.has_inf && isinf(hj)) run3 = fmax(run3, fmax(-gj, 0.0) / fabs(staged ? BX_STG(6) : a.att[p]));
            }
            a.x[p] = xn;
            coef = xn;
          } break;
          case U_APG: {
            // FISTA step by gradient linearity: the dot is g_k
            const double eta = step_eta();
            const double mbeta = momentum_beta();
            const double xo = staged ? BX_STG(0) : a.x[p];
            const double xp = staged ? BX_STG(3) : a.xprev[p];
            const double gp = staged ? BX_STG(5) : a.gprev[p];
            const double hj = staged ? BX_STG(2) : a.hi[p];
            double yv = xo, gy = gj;
            if (mbeta != 0.0) {
              yv = add_rn(xo, mul_rn(mbeta, sub_rn(xo, xp)));
              gy = add_rn(gj, mul_rn(mbeta, sub_rn(gj, gp)));
            }
            const double xn = clip<double>(sub_rn(yv, mul_rn(eta, gy)), staged ? BX_STG(1) : a.lo[p], hj);
            if (a.spec) {
              a.xbak[p] = xp;  // x_{k-1}, g_{k-1}: an undo restores them
              a.gbak[p] = gp;
              a.g[p] = gj;     // the round's screening gradient (g at x_k)
              if (a.has_inf && isinf(hj)) run3 = fmax(run3, fmax(-gj, 0.0) / fabs(staged ? BX_STG(6) : a.att[p]));
            }
            a.xprev[p] = xo;
            a.gprev[p] = gj;
            a.x[p] = xn;
            coef = xn;
            // gradient restart test g_y'(x+ - x) and its round-off scale
            // sum ||a_j|| |x+ - x| (FISTA)
            const double dxj = xn - xo;
            run += gy * dxj;
            run2 += (staged ? BX_STG(4) : a.nrm[p]) * fabs(dxj);
          } break;
          case U_POWER: {
            coef = gj;
            run += coef * coef;
          } break;
          default:
            break;
        }
        cf[tid] = coef;
      }
      __syncthreads();
    } else {
      if (tid < cg) {
        const int ql = gi * C + tid;
        const int64_t p = p0 + ql;
        double coef = 0.0;
        if (a.upd == U_PG_G) {
          const double eta = step_eta();
          const double xo = staged ? BX_STG(0) : a.x[p];
          const double xn = clip<double>(sub_rn(xo, mul_rn(eta, staged ? BX_STG(3) : a.g[p])),
                                         staged ? BX_STG(1) : a.lo[p], staged ? BX_STG(2) : a.hi[p]);
          a.x[p] = xn;
          coef = xn;
        } else {
          coef = staged ? BX_STG(0) : (a.coef ? a.coef[p] : a.x[p]);
        }
        cf[tid] = coef;
      }
      __syncthreads();
    }
    if constexpr (AXPY && sizeof(T) == 8) {
      // fp64: chunks 0 .. R-2 unguarded; the last chunk's rows >= m only
      // reach the padding of the partial row, which k_reduce never reads
#pragma unroll
      for (int c = 0; c < C; ++c) {
        // a column whose coefficient is zero (most of an NNLS iterate sits on
        // its bound) adds exactly nothing: skip its shared-memory reads and
        // FMAs (CTA-uniform branch)
        if (c < cg && (cf[c] != 0.0 || !a.zskip)) {
          const AT cc = static_cast<AT>(cf[c]);
          const T* col = reinterpret_cast<const T*>(slot + c * a.colstride);
#pragma unroll
          for (int i = 0; i < R - 1; ++i) {
            T av[V];
            unpack<T>(*reinterpret_cast<const VT*>(col + row0 + i * (NT * V)), av);
#pragma unroll
            for (int e = 0; e < V; ++e) acc[i][e] += av[e] * cc;
          }
          if (row0 + (R - 1) * (NT * V) < m) {
            T av[V];
            unpack<T>(*reinterpret_cast<const VT*>(col + row0 + (R - 1) * (NT * V)), av);
#pragma unroll
            for (int e = 0; e < V; ++e) acc[R - 1][e] += av[e] * cc;
          }
        }
      }
    } else if constexpr (AXPY && sizeof(T) == 4 && sizeof(AT) == 4) {
      // fp32: chunks 0 .. R-2 unguarded (see the dot); rows >= m of the last
      // vector only reach the padding of the partial row, which k_reduce never
      // reads
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (c < cg && (cf[c] != 0.0 || !a.zskip)) {
          const AT cc = static_cast<AT>(cf[c]);
          const T* col = reinterpret_cast<const T*>(slot + c * a.colstride);
#pragma unroll
          for (int i = 0; i < R - 1; ++i) {
            T av[V];
            unpack<T>(*reinterpret_cast<const VT*>(col + row0 + i * (NT * V)), av);
            fma2_axpy(acc[i], av, cc);
          }
          if (row0 + (R - 1) * (NT * V) < m) {
            T av[V];
            unpack<T>(*reinterpret_cast<const VT*>(col + row0 + (R - 1) * (NT * V)), av);
            fma2_axpy(acc[R - 1], av, cc);
          }
        }
      }
    } else if (AXPY) {
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (c < cg && (cf[c] != 0.0 || !a.zskip)) {
          const AT cc = static_cast<AT>(cf[c]);
          const T* col = reinterpret_cast<const T*>(slot + c * a.colstride);
#pragma unroll
          for (int i = 0; i < R; ++i) {
            const int row = row0 + i * (NT * V);
            if (row < m) {
              T av[V];
              unpack<T>(*reinterpret_cast<const VT*>(col + row), av);
              if constexpr (sizeof(T) == 8) {
#pragma unroll
                for (int e = 0; e < V; ++e) acc[i][e] += ((row + e < m) ? av[e] : T(0)) * cc;
              } else if constexpr (sizeof(AT) == 8) {
#pragma unroll
                for (int e = 0; e < V; ++e) acc[i][e] += static_cast<double>(av[e]) * cc;
              } else {
                // rows >= m of the last vector only reach the padding of the
                // partial row, which k_reduce never reads: no per-element guard
                fma2_axpy(acc[i], av, cc);
              }
            }
          }
        }
      }
    }
    __syncthreads();  // every thread is done with slot s
    if (++s_run == S) {
      s_run = 0;
      ph_run ^= 1u;
    }
    if (tid == 0 && gi + S < ngroups) {
      const int gn = gi + S;
      const int cgn = min(C, ncol - gn * C);
      fence_proxy_async_smem();
      mbar_expect_tx(&bars[s], cgn * a.colbytes);
      for (int c = 0; c < cgn; ++c) {
        const int64_t p = p0 + (int64_t)gn * C + c;
        const int64_t col = a.colmap ? (int64_t)a.colmap[p] : p;
        bulk_g2s(smem + s * slot_bytes + c * a.colstride, a.A + col * a.ld, a.colbytes, &bars[s], pol);
      }
    }
  }

  if (AXPY) {
    if constexpr (sizeof(AT) == sizeof(T)) {
      T* out = a.part + b * a.ldp;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int row = row0 + i * (NT * V);
        if (row < m) *reinterpret_cast<VT*>(out + row) = pack<T>(acc[i]);
      }
    } else {
      AT* out = reinterpret_cast<AT*>(a.part) + b * a.ldp;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int row = row0 + i * (NT * V);
#pragma unroll
        for (int e = 0; e < V; ++e)
          if (row + e < m) out[row + e] = acc[i][e];
      }
    }
  }
#undef BX_STG
  if (a.bpart || a.epart) {
    if (tid < C) {
      bscr[tid] = run;
      bscr[CMAX + tid] = run2;
      bscr[2 * CMAX + tid] = run3;
    }
    __syncthreads();
    if (tid == 0) {
      double v = bscr[0], v2 = bscr[CMAX], v3 = bscr[2 * CMAX];
      for (int c = 1; c < C; ++c) {
        v = (a.upd == U_DOT) ? fmax(v, bscr[c]) : v + bscr[c];
        v2 += bscr[CMAX + c];
        v3 = fmax(v3, bscr[2 * CMAX + c]);
      }
      if (a.bpart) {
        if (a.upd == U_APG) {
          a.bpart[2 * b] = v;
          a.bpart[2 * b + 1] = v2;
        } else {
          a.bpart[b] = v;
        }
      }
      if (a.epart) a.epart[b] = v3;
    }
  }
  if constexpr (AXPY && sizeof(AT) == sizeof(T)) {
    // (the ring is drained: its shared memory is the reduce's scratch)
    if (a.fuse) pass_fused_reduce<T>(a, smem);
  }
}

// ----------------------------------------------------------------------------
// k_reduce: out_i = sum_b part[b][i] (+ off_i) ; block partial of ||out||^2 ;
// last block finalises the objective bookkeeping.
// ----------------------------------------------------------------------------
__device__ __forceinline__ double block_sum_rt(double v, double* sh) {
  v = warp_sum<double>(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
  }
  __syncthreads();
  return t;  // valid in thread 0
}

// Blocks own RB = 32*V consecutive rows; the 8 warps split the G partial rows
// (warp w sums partials w, w+8, ...), then the 8 slice sums are combined in
// warp order -- a fixed summation order, so results are deterministic.
constexpr int RED_SLICES = RT / 32;
constexpr int RED_ONESHOT = 20;  // partial rows per slice loaded in one go (G <= 160)

template <typename T>
__device__ __forceinline__ void finalize_objective(DevScalars* sc, int mode, double Pn, double scale_div,
                                                   double gdot, double gscale) {
  if (mode & R_SPEC) {
    // speculative round-boundary step: keep what an undo restores
    sc->bak_P = sc->P;
    sc->bak_mom_t = sc->mom_t;
    sc->bak_restarts = sc->restarts;
  }
  switch (mode & ~R_SPEC) {
    case R_SET:
      sc->P = Pn;
      break;
    case R_PG:
      if (Pn > sc->P + 1e-9 + sc->rise_rel * fabs(sc->P)) {  // solvers.py:111-114
        if (mode & R_SPEC) {
          // raised only if the step stands (the round neither converges nor
          // undoes it): the reference raises it in the next round's pg_step
          if (sc->err_spec == 0) {
            sc->spec_v1 = sc->P;
            sc->spec_v2 = Pn;
          }
          atomicCAS(&sc->err_spec, 0, DE_STEP_TOO_LARGE);
        } else {
          if (sc->err == 0) {
            sc->err_v1 = sc->P;
            sc->err_v2 = Pn;
          }
          set_err(sc, DE_STEP_TOO_LARGE);
        }
      }
      sc->P = Pn;
      break;
    case R_APG: {
      const double t = sc->mom_t;
      const double tn = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
      const double s_f = sc->rs_f * fmax(1.0, fabs(sc->P));
      const double s_g = sc->rs_g * sqrt(2.0 * sc->P) * gscale;
      if (Pn > sc->P + s_f || gdot > s_g) {  // function / gradient restart (FISTA)
        sc->mom_t = 1.0;
        sc->restarts += 1;
      } else {
        sc->mom_t = tn;
      }
      sc->P = Pn;
    } break;
    case R_POWER:
      sc->nw = scale_div;
      sc->sigma = sqrt(scale_div);
      if (scale_div == 0.0) set_err(sc, DE_POWER_ZERO);
      break;
    case R_CERT:
      sc->cert_P = Pn;
      break;
    default:
      break;
  }
}

// save (speculative step, may be NULL): the previous contents of out
template <typename T>
__global__ void __launch_bounds__(RT) k_reduce(const T* __restrict__ part, int64_t ldp, int G, int64_t m,
                                               const double* off, double* out,
                                               DevScalars* sc, double* bpart, const double* wpart,
                                               int Gw, int mode, int counter, double* __restrict__ save) {
  using VT = typename V16<T>::type;
  constexpr int V = V16<T>::n;
  constexpr int RB = 32 * V;
  __shared__ double sl[RED_SLICES][RB];
  __shared__ double sh[RT / 32];
  __shared__ double s_div;
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int base = mode & ~R_SPEC;
  if (base == R_POWER && warp == 0) {
    double nw2 = 0.0;
    for (int b = lane; b < Gw; b += 32) nw2 += wpart[b];
    // fixed-shape tree: deterministic
    nw2 = warp_sum<double>(nw2);
    if (lane == 0) s_div = sqrt(nw2);
  }
  double sq = 0.0;
  static_assert(RB <= RT, "one output row per thread");
  for (int64_t r0 = (int64_t)blockIdx.x * RB; r0 < m; r0 += (int64_t)gridDim.x * RB) {
    const int64_t row = r0 + lane * V;
    // the offset row this thread adds below, requested in the same L2 round
    // trip as the partial rows (off may alias out: read before it is written)
    const int64_t orow = r0 + threadIdx.x;
    const double offv = (off && threadIdx.x < RB && orow < m) ? off[orow] : 0.0;
    double acc[V];  // partial rows summed in fp64 (fixed order)
#pragma unroll
    for (int e = 0; e < V; ++e) acc[e] = 0.0;
    if (row < m && G <= RED_ONESHOT * RED_SLICES) {
      // every partial row of this lane's slice in flight at once: one L2 round
      // trip (G = one per CTA of the pass, <= 160 on a 148-SM part); absent
      // rows read as zero, the fixed pairwise tree keeps the order fixed
      T q[RED_ONESHOT][V];
#pragma unroll
      for (int u = 0; u < RED_ONESHOT; ++u) {
        const int b = warp + u * RED_SLICES;
        if (b < G) {
          unpack<T>(*reinterpret_cast<const VT*>(part + (int64_t)b * ldp + row), q[u]);
        } else {
#pragma unroll
          for (int e = 0; e < V; ++e) q[u][e] = T(0);
        }
      }
#pragma unroll
      for (int e = 0; e < V; ++e) {
        double s[RED_ONESHOT];
#pragma unroll
        for (int u = 0; u < RED_ONESHOT; ++u) s[u] = static_cast<double>(q[u][e]);
#pragma unroll
        for (int w = 1; w < RED_ONESHOT; w *= 2)
#pragma unroll
          for (int u = 0; u + w < RED_ONESHOT; u += 2 * w) s[u] += s[u + w];
        acc[e] = s[0];
      }
    } else if (row < m) {
      int bb = warp;
      // eight partial rows in flight per lane (the loop is L2-latency bound)
      for (; bb + 7 * RED_SLICES < G; bb += 8 * RED_SLICES) {
        T q[8][V];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          unpack<T>(*reinterpret_cast<const VT*>(part + (int64_t)(bb + u * RED_SLICES) * ldp + row), q[u]);
#pragma unroll
        for (int e = 0; e < V; ++e)
          acc[e] += ((static_cast<double>(q[0][e]) + static_cast<double>(q[1][e])) +
                     (static_cast<double>(q[2][e]) + static_cast<double>(q[3][e]))) +
                    ((static_cast<double>(q[4][e]) + static_cast<double>(q[5][e])) +
                     (static_cast<double>(q[6][e]) + static_cast<double>(q[7][e])));
      }
      for (; bb + 3 * RED_SLICES < G; bb += 4 * RED_SLICES) {
        T q0[V], q1[V], q2[V], q3[V];
        unpack<T>(*reinterpret_cast<const VT*>(part + (int64_t)bb * ldp + row), q0);
        unpack<T>(*reinterpret_cast<const VT*>(part + (int64_t)(bb + RED_SLICES) * ldp + row), q1);
        unpack<T>(*reinterpret_cast<const VT*>(part + (int64_t)(bb + 2 * RED_SLICES) * ldp + row), q2);
        unpack<T>(*reinterpret_cast<const VT*>(part + (int64_t)(bb + 3 * RED_SLICES) * ldp + row), q3);
#pragma unroll
        for (int e = 0; e < V; ++e)
          acc[e] += (static_cast<double>(q0[e]) + static_cast<double>(q1[e])) +
                    (static_cast<double>(q2[e]) + static_cast<double>(q3[e]));
      }
      for (; bb < G; bb += RED_SLICES) {
        T q[V];
        unpack<T>(*reinterpret_cast<const VT*>(part + (int64_t)bb * ldp + row), q);
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] += static_cast<double>(q[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < V; ++e) sl[warp][lane * V + e] = acc[e];
    __syncthreads();  // also publishes s_div (R_POWER) to every thread
    for (int q = threadIdx.x; q < RB; q += RT) {
      const int64_t i = r0 + q;
      if (i < m) {
        double s = sl[0][q];
#pragma unroll
        for (int w = 1; w < RED_SLICES; ++w) s += sl[w][q];
        if (off) s = add_rn(s, offv);
        if (base == R_POWER) s = s / s_div;
        if (save) save[i] = out[i];
        out[i] = s;
        sq += s * s;
      }
    }
    __syncthreads();
  }
  if (base == R_PLAIN) return;
  const double tot = block_sum_rt(sq, sh);
  if (threadIdx.x == 0) {
    bpart[blockIdx.x] = tot;
    __threadfence();
    const unsigned prev = atomicAdd(&sc->counters[counter], 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!last || warp != 0) return;
  __threadfence();
  // last block: warp 0 folds the block partials (lane-strided + fixed tree)
  double total = 0.0, gdot = 0.0, gscale = 0.0;
  for (int b = lane; b < (int)gridDim.x; b += 32) total += __ldcg(&bpart[b]);
  if (base == R_APG && wpart)
    for (int b = lane; b < Gw; b += 32) {
      gdot += __ldcg(&wpart[2 * b]);
      gscale += __ldcg(&wpart[2 * b + 1]);
    }
  total = warp_sum<double>(total);
  gdot = warp_sum<double>(gdot);
  gscale = warp_sum<double>(gscale);
  if (lane != 0) return;
  finalize_objective<T>(sc, mode, 0.5 * total, base == R_POWER ? s_div : 0.0, gdot, gscale);
  sc->counters[counter] = 0u;
}

// The reduce of k_pass's fused mode (one cooperative grid, every CTA
// resident): grid-wide sync once every partial row is written, then CTA b
// sums rows [b*per, (b+1)*per) over the G partials (8 groups of partial rows
// per 64-row chunk, combined in group order: deterministic), adds the offset,
// and the last CTA to finish folds the per-CTA ||r||^2 and restart partials
// in a fixed order and takes the StepSizeTooLarge / restart decision --
// k_reduce's arithmetic, without its launch and without a second pass over
// the partial rows' launch boundary.
template <typename T>
__device__ void pass_fused_reduce(const PassArgs<T>& a, unsigned char* scratch) {
  constexpr int FR = 64;        // rows per chunk
  constexpr int FQ = NT / FR;   // partial-row groups
  constexpr int FONESHOT = (160 + FQ - 1) / FQ;  // partials per thread loaded in one go (G <= 160)
  double* sm = reinterpret_cast<double*>(scratch);  // [FQ][FR] (+ [NWARPS] + flag)
  double* swarp = sm + FQ * FR;
  int* slast = reinterpret_cast<int*>(swarp + NWARPS);
  __threadfence();
  cooperative_groups::this_grid().sync();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t m = a.m;
  const int64_t per = (m + G - 1) / G;
  const int64_t r0 = b * per < m ? b * per : m;
  const int64_t r1 = r0 + per < m ? r0 + per : m;
  const int rr = tid % FR, q = tid / FR;
  double sq = 0.0;
  for (int64_t base = r0; base < r1; base += FR) {
    const int64_t i = base + rr;
    double s = 0.0;
    if (i < r1) {
      if (G <= FQ * FONESHOT) {
        // every partial of this thread in flight at once (one L2 round trip)
        T v[FONESHOT];
#pragma unroll
        for (int u = 0; u < FONESHOT; ++u) {
          const int64_t bb = q + (int64_t)u * FQ;
          v[u] = bb < G ? __ldcg(a.part + bb * a.ldp + i) : T(0);
        }
#pragma unroll
        for (int u = 0; u < FONESHOT; ++u) s += static_cast<double>(v[u]);
      } else {
        for (int64_t bb = q; bb < G; bb += FQ) s += static_cast<double>(__ldcg(a.part + bb * a.ldp + i));
      }
    }
    sm[q * FR + rr] = s;
    __syncthreads();
    if (tid < FR && i < r1) {
      double t = sm[rr];
#pragma unroll
      for (int h = 1; h < FQ; ++h) t += sm[h * FR + rr];
      t = add_rn(t, a.roff[i]);
      if (a.rsave) a.rsave[i] = a.rout[i];
      a.rout[i] = t;
      sq += t * t;
    }
    __syncthreads();
  }
  sq = warp_sum<double>(sq);
  if (lane == 0) swarp[warp] = sq;
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0;
    for (int w = 0; w < NWARPS; ++w) tot += swarp[w];
    a.rpart[b] = tot;
    __threadfence();
    const unsigned prev = atomicAdd(&a.sc->counters[a.rcounter], 1u);
    *slast = (prev == (unsigned)G - 1) ? 1 : 0;
  }
  __syncthreads();
  if (!*slast || warp != 0) return;
  __threadfence();
  double total = 0.0, gdot = 0.0, gscale = 0.0;
  for (int64_t bb = lane; bb < G; bb += 32) total += __ldcg(&a.rpart[bb]);
  if ((a.rmode & ~R_SPEC) == R_APG && a.bpart)
    for (int64_t bb = lane; bb < G; bb += 32) {
      gdot += __ldcg(&a.bpart[2 * bb]);
      gscale += __ldcg(&a.bpart[2 * bb + 1]);
    }
  total = warp_sum<double>(total);
  gdot = warp_sum<double>(gdot);
  gscale = warp_sum<double>(gscale);
  if (lane != 0) return;
  finalize_objective<T>(a.sc, a.rmode, 0.5 * total, 0.0, gdot, gscale);
  a.sc->counters[a.rcounter] = 0u;
}

// ----------------------------------------------------------------------------
// k_dual: dual point, reduced dual objective, clamped gap, radius, slack
// ----------------------------------------------------------------------------
// _reduced_dual (driver.py:120-128) / eval_dual (duality.py:103-124), clamp_gap
// (duality.py:154), radius (screening.py:11-15), slack (driver.py:219)
__device__ __forceinline__ void dual_finalize(DevScalars* sc, int which, double t1, double t2, double t3, double t4,
                                              double eps, double slack_scale, double alpha) {
  // which: 0 reduced problem, 1 certificate (full problem), 2 reduced problem
  // at the iterate before a speculative round-boundary step (its objective
  // was kept in bak_P)
  DualOut* out = (which == 1) ? &sc->cert : &sc->act;
  double dual = t1 - 0.5 * t2;
  dual -= t3;
  dual -= t4;
  const double primal = (which == 1) ? sc->cert_P : (which == 2 ? sc->bak_P : sc->P);
  const double raw = primal - dual;
  if (raw < -1e-9) set_err(sc, DE_INTERNAL_CONSISTENCY);
  const double gap = fmax(raw, 0.0);
  out->primal = primal;
  out->dual = dual;
  out->gap_raw = raw;
  out->gap = gap;
  out->eps = eps;
  out->th_norm2 = t2;
  out->radius = sqrt(2.0 * gap / alpha);
  out->slack = slack_scale * fmax(1.0, sqrt(t2));
  out->thr = out->radius + out->slack;
}

template <typename T>
__global__ void __launch_bounds__(RT) k_dual(const T* __restrict__ r, const T* __restrict__ t,
                                             const T* __restrict__ tgt, T* __restrict__ theta, int64_t m,
                                             const T* __restrict__ g, const T* __restrict__ att,
                                             const T* __restrict__ lo, const T* __restrict__ hi,
                                             T* __restrict__ v, int64_t k, const double* eps_part, int Ge,
                                             int has_inf, DevScalars* sc, int which, double* bpart,
                                             double slack_scale, double alpha, int counter, double* sums_out) {
  __shared__ double sh[RT / 32][4];
  __shared__ double s_eps;
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    double e = 0.0;
    if (has_inf)
      for (int b = lane; b < Ge; b += 32) e = fmax(e, eps_part[b]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
    if (lane == 0) s_eps = e;  // max is order independent: exact
  }
  __syncthreads();
  const double eps = s_eps;
  const T te = static_cast<T>(eps);
  double s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
  const int64_t stride = (int64_t)gridDim.x * RT;
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < m; i += stride) {
    T th = -r[i];  // driver.py:184
    if (eps > 0.0) th = add_rn(th, mul_rn(te, t[i]));  // driver.py:194-195
    theta[i] = th;
    s1 += static_cast<double>(th) * static_cast<double>(tgt[i]);
    s2 += static_cast<double>(th) * static_cast<double>(th);
  }
  for (int64_t j = (int64_t)blockIdx.x * RT + threadIdx.x; j < k; j += stride) {
    T vj = -g[j];  // driver.py:185
    if (has_inf) vj = add_rn(vj, mul_rn(te, att[j]));  // driver.py:196
    v[j] = vj;
    const double vd = static_cast<double>(vj);
    s3 += static_cast<double>(lo[j]) * fmin(vd, 0.0);
    if (!isinf(static_cast<double>(hi[j]))) s4 += static_cast<double>(hi[j]) * fmax(vd, 0.0);
  }
  s1 = warp_sum<double>(s1);
  s2 = warp_sum<double>(s2);
  s3 = warp_sum<double>(s3);
  s4 = warp_sum<double>(s4);
  if (lane == 0) {
    sh[warp][0] = s1;
    sh[warp][1] = s2;
    sh[warp][2] = s3;
    sh[warp][3] = s4;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double a = 0.0;
    for (int w = 0; w < RT / 32; ++w) a += sh[w][threadIdx.x];
    bpart[4 * blockIdx.x + threadIdx.x] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&sc->counters[counter], 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!last || warp != 0) return;
  __threadfence();
  double t1 = 0.0, t2 = 0.0, t3 = 0.0, t4 = 0.0;
  for (int b = lane; b < (int)gridDim.x; b += 32) {
    t1 += __ldcg(&bpart[4 * b + 0]);
    t2 += __ldcg(&bpart[4 * b + 1]);
    t3 += __ldcg(&bpart[4 * b + 2]);
    t4 += __ldcg(&bpart[4 * b + 3]);
  }
  t1 = warp_sum<double>(t1);
  t2 = warp_sum<double>(t2);
  t3 = warp_sum<double>(t3);
  t4 = warp_sum<double>(t4);
  if (lane != 0) return;
  sc->counters[counter] = 0u;
  if (sums_out) {
    // column-sharded: the bound terms t3, t4 are this rank's share; the host
    // allreduces them and k_dual_fin finalises (t1, t2 come from the
    // replicated residual and are identical on every rank)
    sums_out[0] = t1;
    sums_out[1] = t2;
    sums_out[2] = t3;
    sums_out[3] = t4;
    sums_out[4] = eps;
    return;
  }
  dual_finalize(sc, which, t1, t2, t3, t4, eps, slack_scale, alpha);
}

__global__ void k_dual_fin(const double* sums, DevScalars* sc, int which, double slack_scale, double alpha) {
  if (threadIdx.x == 0 && blockIdx.x == 0)
    dual_finalize(sc, which, sums[0], sums[1], sums[2], sums[3], sums[4], slack_scale, alpha);
}

// ----------------------------------------------------------------------------
// sphere test + compaction (warp ballot + block prefix sums)
// flags: 0 keep, 1 lower, 2 upper
// ----------------------------------------------------------------------------
// Speculative round boundary: with sx0 != NULL the iterate
// has already taken the next round's first step; a screened coordinate is
// "dirty" when any of the iterates the step touched -- sx0 (after), sx1
// (the round's final x), sx2 (FISTA: the one before) -- is off the bound it
// is screened at.  Any dirty column means the step used a residual the
// screening changes: the host undoes it (k_spec_undo) and takes it again.
template <typename T>
__global__ void __launch_bounds__(RT) k_sphere(const T* __restrict__ v, const T* __restrict__ nrm,
                                               const T* __restrict__ lo, const T* __restrict__ hi, int64_t k,
                                               const DevScalars* sc, uint8_t* __restrict__ flags,
                                               int32_t* __restrict__ bcnt, const double* __restrict__ sx0,
                                               const double* __restrict__ sx1, const double* __restrict__ sx2) {
  __shared__ int32_t wc[RT / 32][4];
  const int64_t j = (int64_t)blockIdx.x * RT + threadIdx.x;
  int f = -1;
  bool dirty = false;
  if (j < k) {
    const double thr = sc->act.thr * static_cast<double>(nrm[j]);
    const double vj = static_cast<double>(v[j]);
    f = 0;
    if (vj < -thr)
      f = 1;
    else if (vj > thr && !isinf(static_cast<double>(hi[j])))
      f = 2;
    flags[j] = static_cast<uint8_t>(f);
    if (f > 0 && sx0) {
      const double bnd = static_cast<double>(f == 1 ? lo[j] : hi[j]);
      dirty = sx0[j] != bnd || sx1[j] != bnd || (sx2 && sx2[j] != bnd);
    }
  }
  const unsigned bk = __ballot_sync(0xffffffffu, f == 0);
  const unsigned bl = __ballot_sync(0xffffffffu, f == 1);
  const unsigned bu = __ballot_sync(0xffffffffu, f == 2);
  const unsigned bd = __ballot_sync(0xffffffffu, dirty);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    wc[warp][0] = __popc(bk);
    wc[warp][1] = __popc(bl);
    wc[warp][2] = __popc(bu);
    wc[warp][3] = __popc(bd);
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    int s = 0;
    for (int w = 0; w < RT / 32; ++w) s += wc[w][threadIdx.x];
    bcnt[4 * blockIdx.x + threadIdx.x] = s;
  }
}

// single block: exclusive scan of the per-block (keep, lower, upper, dirty)
// counts in place; totals to sc->n_keep / n_lo / n_up / n_dirty
__global__ void __launch_bounds__(1024) k_scan(int32_t* bcnt, int nb, DevScalars* sc) {
  __shared__ int64_t wsum[32][4];
  __shared__ int64_t carry[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 4) carry[threadIdx.x] = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    int64_t c[4] = {0, 0, 0, 0};
    if (i < nb) {
      c[0] = bcnt[4 * i + 0];
      c[1] = bcnt[4 * i + 1];
      c[2] = bcnt[4 * i + 2];
      c[3] = bcnt[4 * i + 3];
    }
    int64_t inc[4] = {c[0], c[1], c[2], c[3]};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t nb_ = __shfl_up_sync(0xffffffffu, inc[q], o);
        if (lane >= o) inc[q] += nb_;
      }
      if (lane == 31) wsum[warp][q] = inc[q];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int64_t w = wsum[lane][q];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int64_t nb_ = __shfl_up_sync(0xffffffffu, w, o);
          if (lane >= o) w += nb_;
        }
        wsum[lane][q] = w;  // inclusive over warps
      }
    }
    __syncthreads();
    if (i < nb) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t wex = warp ? wsum[warp - 1][q] : 0;
        bcnt[4 * i + q] = static_cast<int32_t>(carry[q] + wex + inc[q] - c[q]);
      }
    }
    __syncthreads();
    if (threadIdx.x < 4) carry[threadIdx.x] += wsum[31][threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    sc->n_keep = sc->g_keep = carry[0];
    sc->n_lo = sc->g_lo = carry[1];
    sc->n_up = sc->g_up = carry[2];
    sc->n_dirty = sc->g_dirty = carry[3];
  }
}

// scatter by flag: kept columns -> compacted per-column state (order kept);
// screened -> x_full snapped to its bound, the (column, bound) list for the
// z update, and the global sat_lower / sat_upper lists (screening.py:84-94)
template <typename T>
struct ColState {
  int32_t* idx;
  T* x;
  T* xprev;
  T* gprev;  // FISTA gradient at x_prev (NULL: not carried)
  T* xbak;   // a standing speculative step's x_{k-1} / g_{k-1} (NULL: not carried)
  T* gbak;
  T* lo;
  T* hi;
  T* nrm;
  T* att;
  int32_t* pos;  // physical column in the compacted buffer (src NULL: identity)
};

template <typename T>
__global__ void __launch_bounds__(RT) k_compact(const uint8_t* __restrict__ flags, const int32_t* __restrict__ boff,
                                                int64_t k, ColState<T> src, ColState<T> dst, T* __restrict__ x_full,
                                                int32_t* __restrict__ scr_idx, T* __restrict__ scr_val, int64_t n_lo_total,
                                                int64_t* __restrict__ sat_lo, int64_t* __restrict__ sat_up,
                                                int64_t col_offset, T* __restrict__ scr_dx, T* __restrict__ scr_dxp) {
  __shared__ int32_t woff[RT / 32][3];
  const int64_t j = (int64_t)blockIdx.x * RT + threadIdx.x;
  const int f = (j < k) ? flags[j] : 3;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const unsigned bq[3] = {__ballot_sync(0xffffffffu, f == 0), __ballot_sync(0xffffffffu, f == 1),
                          __ballot_sync(0xffffffffu, f == 2)};
  if (lane == 0) {
    woff[warp][0] = __popc(bq[0]);
    woff[warp][1] = __popc(bq[1]);
    woff[warp][2] = __popc(bq[2]);
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    int run = 0;
    for (int w = 0; w < RT / 32; ++w) {
      const int x = woff[w][threadIdx.x];
      woff[w][threadIdx.x] = run;
      run += x;
    }
  }
  __syncthreads();
  if (f > 2) return;
  const int64_t pos = (int64_t)boff[4 * blockIdx.x + f] + woff[warp][f] + __popc(bq[f] & lt);
  const int32_t id = src.idx[j];
  if (f == 0) {
    dst.idx[pos] = id;
    if (dst.pos) dst.pos[pos] = src.pos ? src.pos[j] : static_cast<int32_t>(j);
    dst.x[pos] = src.x[j];
    if (src.xprev) dst.xprev[pos] = src.xprev[j];
    if (src.gprev) dst.gprev[pos] = src.gprev[j];
    if (src.xbak) dst.xbak[pos] = src.xbak[j];
    if (src.gbak) dst.gbak[pos] = src.gbak[j];
    dst.lo[pos] = src.lo[j];
    dst.hi[pos] = src.hi[j];
    dst.nrm[pos] = src.nrm[j];
    dst.att[pos] = src.att[j];
  } else {
    // screened: x snapped to its bound; (b - x) and (b - x_prev) drive the
    // incremental residual refresh r += A_S (b - x_S)
    const T b = (f == 1) ? src.lo[j] : src.hi[j];
    const int64_t q = (f == 1) ? pos : n_lo_total + pos;
    x_full[id] = b;
    scr_idx[q] = id;
    scr_val[q] = b;
    scr_dx[q] = sub_rn(b, src.x[j]);
    scr_dxp[q] = src.xprev ? sub_rn(b, src.xprev[j]) : T(0);
    if (f == 1)
      sat_lo[pos] = col_offset + id;
    else
      sat_up[pos] = col_offset + id;
  }
}

// physical column rewrite: B[:, p] = A[:, idx[p]]  (solvers.py:57)
template <typename T>
__global__ void __launch_bounds__(RT) k_gather(const T* __restrict__ A, int64_t lda, const int32_t* __restrict__ idx,
                                               int64_t k, int64_t m, T* __restrict__ B, int64_t ldb) {
  using VT = typename V16<T>::type;
  constexpr int V = V16<T>::n;
  for (int64_t p = blockIdx.x; p < k; p += gridDim.x) {
    const VT* s = reinterpret_cast<const VT*>(A + (int64_t)idx[p] * lda);
    VT* d = reinterpret_cast<VT*>(B + p * ldb);
    const int64_t nv = (m + V - 1) / V;
    for (int64_t i = threadIdx.x; i < nv; i += RT) d[i] = __ldcs(s + i);
  }
}

// per-column statistics of the original matrix: ||a_j|| (model.py:89-92) and
// a_j' t (duality.py:52); flags zero columns and non-interior t
template <typename T>
__global__ void __launch_bounds__(RT) k_colstats(const T* __restrict__ A, int64_t lda, int64_t n, int64_t m,
                                                 const double* __restrict__ t, double* __restrict__ nrm,
                                                 double* __restrict__ att,
                                                 int check_interior, int* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * RT + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * RT) >> 5;
  for (int64_t j = w; j < n; j += nw) {
    const T* col = A + j * lda;
    double ss = 0.0, st = 0.0;
    for (int64_t i = lane; i < m; i += 32) {
      const double a = static_cast<double>(col[i]);
      ss += a * a;
      st += a * t[i];
    }
    ss = warp_sum<double>(ss);
    st = warp_sum<double>(st);
    if (lane == 0) {
      const double nj = sqrt(ss);
      nrm[j] = nj;
      att[j] = st;
      if (nj == 0.0) atomicOr(&flags[0], 1);
      if (check_interior && !(st < -1e-10 * nj)) atomicOr(&flags[0], 2);
    }
  }
}

template <typename T>
__global__ void k_init_cols(int64_t n, const T* __restrict__ lo, const T* __restrict__ hi, T* __restrict__ x_full,
                            int32_t* __restrict__ idx, T* __restrict__ x, T* __restrict__ lo2, T* __restrict__ hi2,
                            const T* __restrict__ nrm, T* __restrict__ nrm2, const T* __restrict__ att,
                            T* __restrict__ att2) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const T x0 = clip<T>(T(0), lo[j], hi[j]);  // driver.py:149
    x_full[j] = x0;
    x[j] = x0;
    idx[j] = static_cast<int32_t>(j);
    lo2[j] = lo[j];
    hi2[j] = hi[j];
    nrm2[j] = nrm[j];
    att2[j] = att[j];
  }
}

// bx_set_state: the per-column state of a given preserved set (Workspace,
// solvers.py:51-63): x, bounds, norms and A't gathered from the full arrays
__global__ void k_gather_state(int64_t k, const int64_t* __restrict__ pres, int32_t* __restrict__ idx,
                               const double* __restrict__ xf, const double* __restrict__ lof,
                               const double* __restrict__ hif, const double* __restrict__ nrmf,
                               const double* __restrict__ attf, double* __restrict__ x, double* __restrict__ lo,
                               double* __restrict__ hi, double* __restrict__ nrm, double* __restrict__ att,
                               double* __restrict__ xprev, double* __restrict__ gprev) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < k; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = pres[p];
    idx[p] = static_cast<int32_t>(j);
    x[p] = xf[j];
    xprev[p] = xf[j];
    gprev[p] = 0.0;
    lo[p] = lof[j];
    hi[p] = hif[j];
    nrm[p] = nrmf[j];
    att[p] = attf[j];
  }
}

// sphere test on caller-given inner products (screening.py:60-69):
// thr_j = (radius + slack) ||a_j||, strict comparisons, upper only for
// finite u_j
__global__ void k_sphere_given(const double* __restrict__ v, const double* __restrict__ nrm,
                               const double* __restrict__ hi, const int32_t* __restrict__ pres, int64_t k,
                               double radius, double slack, uint8_t* __restrict__ flags) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < k; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = pres[p];
    const double thr = (radius + slack) * nrm[j];
    const double vj = v[j];
    uint8_t f = 0;
    if (vj < -thr)
      f = 1;
    else if (vj > thr && !isinf(hi[j]))
      f = 2;
    flags[p] = f;
  }
}

template <typename T>
__global__ void k_offsets(int64_t m, const T* __restrict__ y, const T* __restrict__ z, T* __restrict__ off,
                          T* __restrict__ tgt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    off[i] = sub_rn(z[i], y[i]);  // solvers.py:62
    tgt[i] = sub_rn(y[i], z[i]);  // solvers.py:63
  }
}

template <typename T>
__global__ void k_scatter_x(int64_t k, const int32_t* __restrict__ idx, const T* __restrict__ x, T* __restrict__ x_full) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < k; p += (int64_t)gridDim.x * blockDim.x)
    x_full[idx[p]] = x[p];
}

template <typename T>
__global__ void k_fill(int64_t n, T* __restrict__ d, T v) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) d[p] = v;
}

template <typename T>
__global__ void k_neg(int64_t n, const T* __restrict__ s, T* __restrict__ d) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) d[p] = -s[p];
}

// bound structure probe: bit0 some lower != 0, bit1 some finite upper != 0,
// bit2 some upper infinite, bit3 lower not finite, bit4 lower >= upper, bit5 NaN
template <typename T>
__global__ void k_bounds_probe(int64_t n, const T* __restrict__ lo, const T* __restrict__ hi, int* __restrict__ out) {
  int f = 0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double l = static_cast<double>(lo[j]), u = static_cast<double>(hi[j]);
    if (l != 0.0) f |= 1;
    if (!isinf(u) && u != 0.0) f |= 2;
    if (isinf(u)) f |= 4;
    if (!isfinite(l)) f |= 8;
    if (!(l < u)) f |= 16;
    if (isnan(l) || isnan(u)) f |= 32;
  }
  if (f) atomicOr(out, f);
}

// Row-blocked path (m beyond the register-resident envelope): after the dot
// has been accumulated over all row blocks, the per-column update of the mode
// (the same arithmetic as k_pass's epilogue) and its block scalar partials.
// Writes coef (the axpy coefficients of the following A x blocks).
// FISTA: g holds g_k (the dot at r_k); the extrapolated gradient is formed by
// linearity from gprev (g_{k-1}), which is then replaced by g_k.  spec: the
// speculative round-boundary step (x_k -> xprev / x_{k-1}, g_{k-1} -> xbak,
// gbak for an undo; epsilon partial of g_k -> epart).
__global__ void __launch_bounds__(RT) k_colupdate(int upd, int64_t k, double* __restrict__ x, double* __restrict__ xprev,
                                                  const double* __restrict__ lo, const double* __restrict__ hi,
                                                  const double* __restrict__ g, const double* __restrict__ att,
                                                  const double* __restrict__ nrm, double* __restrict__ coef,
                                                  double* __restrict__ bpart, int has_inf, const DevScalars* sc,
                                                  double* __restrict__ gprev, int spec, double* __restrict__ xbak,
                                                  double* __restrict__ gbak, double* __restrict__ epart) {
  __shared__ double sh[RT / 32][3];
  const double eta = sc->eta;
  double beta = 0.0;
  if (upd == U_APG) {
    const double t = sc->mom_t;
    const double tn = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
    beta = (t - 1.0) / tn;
  }
  double r1 = 0.0, r2 = 0.0, r3 = 0.0;
  for (int64_t p = (int64_t)blockIdx.x * RT + threadIdx.x; p < k; p += (int64_t)gridDim.x * RT) {
    const double gj = g[p];
    if (spec && has_inf && isinf(hi[p])) r3 = fmax(r3, fmax(-gj, 0.0) / fabs(att[p]));
    switch (upd) {
      case U_DOT:
        if (has_inf && isinf(hi[p])) r1 = fmax(r1, fmax(-gj, 0.0) / fabs(att[p]));
        break;
      case U_PG:
      case U_PG_G: {
        const double xo = x[p];
        const double xn = clip<double>(sub_rn(xo, mul_rn(eta, gj)), lo[p], hi[p]);
        if (spec) xprev[p] = xo;
        x[p] = xn;
        coef[p] = xn;
      } break;
      case U_APG: {
        const double xo = x[p], xp = xprev[p], gp = gprev[p];
        double yv = xo, gy = gj;
        if (beta != 0.0) {
          yv = add_rn(xo, mul_rn(beta, sub_rn(xo, xp)));
          gy = add_rn(gj, mul_rn(beta, sub_rn(gj, gp)));
        }
        const double xn = clip<double>(sub_rn(yv, mul_rn(eta, gy)), lo[p], hi[p]);
        if (spec) {
          xbak[p] = xp;
          gbak[p] = gp;
        }
        xprev[p] = xo;
        gprev[p] = gj;
        x[p] = xn;
        coef[p] = xn;
        const double dx = xn - xo;
        r1 += gy * dx;
        r2 += nrm[p] * fabs(dx);
      } break;
      case U_POWER:
        coef[p] = gj;
        r1 += gj * gj;
        break;
      default:
        break;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (upd == U_DOT) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r1 = fmax(r1, __shfl_xor_sync(0xffffffffu, r1, o));
  } else {
    r1 = warp_sum<double>(r1);
    r2 = warp_sum<double>(r2);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r3 = fmax(r3, __shfl_xor_sync(0xffffffffu, r3, o));
  if (lane == 0) {
    sh[warp][0] = r1;
    sh[warp][1] = r2;
    sh[warp][2] = r3;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double v1 = sh[0][0], v2 = sh[0][1], v3 = sh[0][2];
    for (int w = 1; w < RT / 32; ++w) {
      v1 = (upd == U_DOT) ? fmax(v1, sh[w][0]) : v1 + sh[w][0];
      v2 += sh[w][1];
      v3 = fmax(v3, sh[w][2]);
    }
    if (bpart) {
      if (upd == U_APG) {
        bpart[2 * blockIdx.x] = v1;
        bpart[2 * blockIdx.x + 1] = v2;
      } else {
        bpart[blockIdx.x] = v1;
      }
    }
    if (spec && epart) epart[blockIdx.x] = v3;
  }
}

// Undo of the speculative round-boundary step (the round's screening event
// changed the problem the step was taken on, or the step size changes):
// x <- x_k, and for FISTA x_prev <- x_{k-1}, g_prev <- g_{k-1}; the residual
// r_k (saved by the step's reduce) and the scalars before the step.
__global__ void k_spec_undo(int64_t k, int apg, double* __restrict__ x, double* __restrict__ xprev,
                            const double* __restrict__ xbak, double* __restrict__ gprev,
                            const double* __restrict__ gbak, int64_t m, double* __restrict__ r,
                            const double* __restrict__ rbak, DevScalars* sc) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t p = i0; p < k; p += stride) {
    x[p] = xprev[p];
    if (apg) {
      xprev[p] = xbak[p];
      gprev[p] = gbak[p];
    }
  }
  for (int64_t i = i0; i < m; i += stride) r[i] = rbak[i];
  if (i0 == 0) {
    sc->P = sc->bak_P;
    sc->mom_t = sc->bak_mom_t;
    sc->restarts = sc->bak_restarts;
    sc->err_spec = 0;
  }
}

// column-sharded helpers -----------------------------------------------------
// fold per-block scalar partials into out[0..stride): sum (op 0) or max (op 1),
// lane-strided + fixed-shape tree (deterministic)
__global__ void k_fold(const double* __restrict__ in, int G, int stride, int op, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int q = 0; q < stride; ++q) {
    double v = 0.0;
    for (int b = lane; b < G; b += 32) {
      const double x = __ldcg(&in[b * stride + q]);
      v = op ? fmax(v, x) : v + x;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, v, o);
      v = op ? fmax(v, y) : v + y;
    }
    if (lane == 0) out[q] = v;
  }
}

// in-process rank group (tests on one GPU): out = reduce over ranks of
// ptrs[r][0..count) in rank order.  dtype: 0 f64, 1 f32, 2 i64, 3 i32; op: 0 sum, 1 max
__global__ void k_group_reduce(void* __restrict__ out, const void* const* __restrict__ ptrs, int n, int64_t count,
                               int dtype, int op) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    if (dtype == 0) {
      double v = static_cast<const double*>(ptrs[0])[i];
      for (int r = 1; r < n; ++r) {
        const double x = static_cast<const double*>(ptrs[r])[i];
        v = op ? fmax(v, x) : v + x;
      }
      static_cast<double*>(out)[i] = v;
    } else if (dtype == 1) {
      float v = static_cast<const float*>(ptrs[0])[i];
      for (int r = 1; r < n; ++r) {
        const float x = static_cast<const float*>(ptrs[r])[i];
        v = op ? fmaxf(v, x) : v + x;
      }
      static_cast<float*>(out)[i] = v;
    } else if (dtype == 2) {
      long long v = static_cast<const long long*>(ptrs[0])[i];
      for (int r = 1; r < n; ++r) {
        const long long x = static_cast<const long long*>(ptrs[r])[i];
        v = op ? (x > v ? x : v) : v + x;
      }
      static_cast<long long*>(out)[i] = v;
    } else {
      int v = static_cast<const int*>(ptrs[0])[i];
      for (int r = 1; r < n; ++r) {
        const int x = static_cast<const int*>(ptrs[r])[i];
        v = op ? (x > v ? x : v) : v + x;
      }
      static_cast<int*>(out)[i] = v;
    }
  }
}

}  // namespace bx
