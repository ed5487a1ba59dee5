// bx_small.cuh -- one PG / FISTA round of a small problem in ONE cooperative
// launch (BASELINE config 1: A_act is 16 MB, it fits in the aggregate shared
// memory of the 148 SMs).
//
// The streamed path (k_pass + k_reduce, two launches per step) is latency
// bound at this size: ~21 us per step for 16 MB.  Here every CTA loads its
// contiguous block of preserved columns into shared memory ONCE per round and
// keeps it there; each step is
//     dots of the local columns (one warp per column) with the residual
//     staged in shared memory -> each column's x update by the lane that
//     holds its dot -> local partial A x+ rows  -> grid barrier
//     -> CTA b reduces rows [b*mb, (b+1)*mb) over all partials in a fixed order
//        (+ z - y), and its share of ||r||^2 and the restart partials
//     -> grid barrier -> every CTA loads the next step's residual rows and
//        folds the per-CTA scalars in the same L2 round trip (same order, same
//        value everywhere) and takes the same StepSizeTooLarge / restart
//        decision
// and the round ends with the screening dot pass (g = A'r, epsilon partials)
// consumed by k_dual.  The arithmetic is the streamed path's: same per-column
// update, same deterministic reductions (different summation grouping).
#pragma once
#include "bx_kernels.cuh"

namespace bx {

constexpr int SM_NT = 512;
constexpr int SM_CMAX = 48;  // max resident columns per CTA

struct SmallArgs {
  const void* A;
  int64_t ld;
  const int32_t* colmap;  // column p at A + colmap[p] * ld (NULL: p)
  int64_t k;
  int m;
  double* x;
  double* xprev;
  double* gprev;   // FISTA: gradient at x_prev
  const double* lo;
  const double* hi;
  const double* nrm;
  const double* att;
  double* g;
  double* r[2];
  const double* off;
  double* part;    // [G][ldp] partial rows (fp64)
  int64_t ldp;
  double* bpart;   // [G][4] per-CTA scalars
  double* epart;   // [G] epsilon partials for k_dual
  DevScalars* sc;
  unsigned* bar;   // [G] per-CTA barrier epochs
  int passes;
  int kind;        // 0 PG, 2 APG
  int g_valid;     // PG: the first step may use the stored gradient
  int has_inf;
  int do_dot;      // end the round with the screening dot pass
  int rc;          // r[rc] holds the current residual
  int colstride;   // smem elements per column
  int ncmax;       // resident columns per CTA (smem sized for it)
  // device-resident round loop (max_rounds > 1): after each round the kernel
  // evaluates the dual point, the gap, the stop test and the sphere test
  // itself, and returns to the host only at an event (something screened, a
  // convergence candidate, an error) or after max_rounds.
  int max_rounds;
  const double* t;    // translation vector (rows)
  const double* tgt;  // y - z (rows)
  double* theta;      // dual point (rows)
  double* dpart;      // [G][8] dual / count partials
  double* trace;      // [max_rounds][TRACE_W] per completed round
  unsigned long long* stamp0;  // %globaltimer at the kernel's start
  int* done;          // [2]: completed event-free rounds, event flag
  double tol;
  int relative_gap;
  int screening;
  double slack_scale;
  double alpha;
  int zskip;          // skip zero coefficients in the partial-row loop (0 only with env BX_NO_ZSKIP)
  unsigned long long* dbg;  // BX_SMALL_DEBUG: per-phase clock sums of CTA 0 (null otherwise)
};

// Grid barrier: one monotonic arrival counter per launch (zeroed by the host
// before the launch); the n-th barrier of the launch completes when the
// counter reaches n * gridDim.x.  Arrival is a fire-and-forget release
// reduction and the wait polls with acquire loads -- no
// generation word to read first and no reset inside the kernel (one L2 round
// trip less per barrier than a sense-reversal barrier).  All CTAs are
// co-resident (cooperative launch).
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& nbar) {
  __syncthreads();
  ++nbar;
  if (threadIdx.x == 0) {
    // release-reduction: orders this CTA's prior writes (made visible to
    // thread 0 by the CTA barrier) before the arrival, without a full fence
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    const unsigned target = nbar * gridDim.x;
    while (ld_acquire_gpu(bar) < target) {
    }
  }
  __syncthreads();
}

template <typename T, int R>
__global__ void __launch_bounds__(SM_NT, 1) k_round_small(const SmallArgs a) {
  using VT = typename V16<T>::type;
  constexpr int V = V16<T>::n;
  constexpr int NW = SM_NT / 32;
  extern __shared__ __align__(1024) unsigned char smem[];
  T* cols = reinterpret_cast<T*>(smem);
  double* red = reinterpret_cast<double*>(smem + (((size_t)a.ncmax * a.colstride * sizeof(T) + 127) / 128) * 128);
  double* gcol = red + NW * SM_CMAX;   // [SM_CMAX] reduced dots
  double* cf = gcol + SM_CMAX;         // [SM_CMAX] axpy coefficients
  double* rsx = cf + SM_CMAX;          // [2][SM_NT] restart partials
  double* sc4 = rsx + 2 * SM_NT;       // [8] block scalars
  double* cx = sc4 + 8;                // [SM_CMAX] resident x
  double* cxp = cx + SM_CMAX;          // [SM_CMAX] x_prev
  double* clo = cxp + SM_CMAX;         // bounds, norms, A't, stored gradient
  double* chi = clo + SM_CMAX;
  double* cnr = chi + SM_CMAX;
  double* cat = cnr + SM_CMAX;
  double* cg = cat + SM_CMAX;          // gradient at the current x (when gv)
  double* cgp = cg + SM_CMAX;          // FISTA: gradient at x_prev
  double* coff = cgp + SM_CMAX;        // [SM_NT] z - y of the rows this CTA reduces
  double* rv = coff + SM_NT;           // [m, padded] the dot vector of this step
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m = a.m;
  const int G = gridDim.x, b = blockIdx.x;
  const int64_t p0 = a.k * b / G, p1 = a.k * (b + 1) / G;
  const int ncol = (int)(p1 - p0);
  const int row0 = tid * V;

  // resident columns (read once per round)
  {
    const int nv = (m + V - 1) / V;
    const T* A = static_cast<const T*>(a.A);
    for (int q = tid; q < ncol * nv; q += SM_NT) {
      const int c = q / nv, v = q - c * nv;
      const int64_t col = a.colmap ? (int64_t)a.colmap[p0 + c] : (p0 + c);
      *reinterpret_cast<VT*>(cols + (size_t)c * a.colstride + v * V) =
          *reinterpret_cast<const VT*>(A + col * a.ld + v * V);
    }
  }
  if (tid < ncol) {
    const int64_t p = p0 + tid;
    cx[tid] = a.x[p];
    cxp[tid] = a.kind == 2 ? a.xprev[p] : 0.0;
    clo[tid] = a.lo[p];
    chi[tid] = a.hi[p];
    cnr[tid] = a.nrm[p];
    cat[tid] = a.att[p];
    cg[tid] = a.g[p];
    cgp[tid] = a.kind == 2 ? a.gprev[p] : 0.0;
  }
  __syncthreads();

  double eta = a.sc->eta;
  unsigned nbar = 0;  // grid barriers passed in this launch
  double t_mom = a.sc->mom_t;
  double P = a.sc->P;
  int rc = a.rc;
  int gv = a.g_valid;
  // rows of the reduce phase owned by this CTA
  const int mb = (m + G - 1) / G;
  const int r_lo = min(m, b * mb), r_hi = min(m, r_lo + mb);
  const int nrow = r_hi - r_lo;
  if (tid < nrow) coff[tid] = a.off[r_lo + tid];

  // dots of the local columns with rv (shared memory): one warp per column,
  // lanes over 16-byte row vectors with two independent chains, then one
  // butterfly -- no cross-warp fold
  // warp-level dot of local column c with rv (shared memory): lanes over
  // 16-byte row vectors with two independent chains, one butterfly (every
  // lane ends with the sum)
  const int nv = m / V;  // full vectors; the m % V tail goes to lane 0
  auto col_dot = [&](int c) {
    const T* col = cols + (size_t)c * a.colstride;
    double s0 = 0.0, s1 = 0.0;
    int vi = lane;
    for (; vi + 32 < nv; vi += 64) {
      T av[V], aw[V];
      double rr[V], rw[V];
      unpack<T>(*reinterpret_cast<const VT*>(col + vi * V), av);
      unpack<T>(*reinterpret_cast<const VT*>(col + (vi + 32) * V), aw);
      load_rows<T>(rv + vi * V, rr);
      load_rows<T>(rv + (vi + 32) * V, rw);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        s0 += static_cast<double>(av[e]) * rr[e];
        s1 += static_cast<double>(aw[e]) * rw[e];
      }
    }
    if (vi < nv) {
      T av[V];
      double rr[V];
      unpack<T>(*reinterpret_cast<const VT*>(col + vi * V), av);
      load_rows<T>(rv + vi * V, rr);
#pragma unroll
      for (int e = 0; e < V; ++e) s0 += static_cast<double>(av[e]) * rr[e];
    }
    if (lane == 0)
      for (int row = nv * V; row < m; ++row) s1 += static_cast<double>(col[row]) * rv[row];
    return warp_sum<double>(s0 + s1);
  };
  // dots of all local columns into gout (one warp per column)
  auto dots = [&](double* gout) {
    for (int c = warp; c < ncol; c += NW) {
      const double sum = col_dot(c);
      if (lane == 0) gout[c] = sum;
    }
    __syncthreads();
  };

  int done_rounds = 0, event = 0;
  const bool timed = a.dbg && b == 0 && tid == 0;
  long long tsm[7] = {0, 0, 0, 0, 0, 0, 0};
  long long tsx[4] = {0, 0, 0, 0};
  bool perr = false;
  if (b == 0 && tid == 0 && a.stamp0) *a.stamp0 = globaltimer();
  double excl_ns = 0.0;  // dual-point time of this launch (block 0's view; screening off)
  // this thread's rows (tid + q * SM_NT) of the current residual, loaded
  // right after the barrier that completes them -- in the same L2 round trip
  // as the objective fold instead of one after it
  constexpr int PR = R * V;
  double pr[PR];
  bool have_pre = false;
  for (int rnd = 0; rnd < a.max_rounds; ++rnd) {
  for (int pass = 0; pass < a.passes; ++pass) {
    const long long tp0 = timed ? clock64() : 0;
    const double* rcur = a.r[rc];
    const double tn = (1.0 + sqrt(1.0 + 4.0 * t_mom * t_mom)) / 2.0;
    const double beta = (a.kind == 2) ? (t_mom - 1.0) / tn : 0.0;
    // the gradient at x is known (the previous round's screening dot): the
    // round's first step needs no dot
    const bool use_stored = (gv && pass == 0);
    // column update (PG / FISTA), done by the lane that holds the column's
    // dot -- no CTA barrier between the dots and the updates.  FISTA forms
    // the extrapolated gradient by linearity:
    // g_y = g_k + beta (g_k - g_{k-1})
    auto update_col = [&](int c, double gj) {
      const double xo = cx[c];
      double xn;
      if (a.kind == 2) {
        const double xp = cxp[c];
        double yv = xo, gy = gj;
        if (beta != 0.0) {
          yv = add_rn(xo, mul_rn(beta, sub_rn(xo, xp)));
          gy = add_rn(gj, mul_rn(beta, sub_rn(gj, cgp[c])));
        }
        xn = clip<double>(sub_rn(yv, mul_rn(eta, gy)), clo[c], chi[c]);
        cxp[c] = xo;
        cgp[c] = gj;
        const double dx = xn - xo;
        rsx[c] = gy * dx;                  // restart partials of this CTA
        rsx[SM_NT + c] = cnr[c] * fabs(dx);
      } else {
        cg[c] = gj;
        xn = clip<double>(sub_rn(xo, mul_rn(eta, gj)), clo[c], chi[c]);
      }
      cx[c] = xn;
      cf[c] = xn;
    };
    if (!use_stored) {
      // residual -> shared memory; written by other CTAs before the barrier:
      // read through L2
      if (have_pre) {
#pragma unroll
        for (int q = 0; q < PR; ++q) {
          const int row = tid + q * SM_NT;
          if (row < m) rv[row] = pr[q];
        }
      } else {
        for (int row = tid; row < m; row += SM_NT) rv[row] = __ldcg(&rcur[row]);
      }
      __syncthreads();
      const long long td0 = timed ? clock64() : 0;
      for (int c = warp; c < ncol; c += NW) {
        const double gj = col_dot(c);
        const long long td1 = timed ? clock64() : 0;
        if (lane == 0) update_col(c, gj);
        if (timed) {
          tsx[1] += td1 - td0;        // warp 0's column dot
          tsx[2] += clock64() - td1;  // its update
        }
      }
      if (timed) tsx[0] += td0 - tp0;  // residual to shared memory + barrier
    } else {
      for (int c = warp; c < ncol; c += NW)
        if (lane == 0) update_col(c, cg[c]);
    }
    __syncthreads();
    const long long tp1 = timed ? clock64() : 0;
    // restart partials of this CTA (fixed order: lane-strided, then one
    // butterfly in warp 0; lane 0 = thread 0 also publishes them below)
    if (warp == 0 && a.kind == 2) {
      double s1 = 0.0, s2 = 0.0;
      for (int c = lane; c < ncol; c += 32) {
        s1 += rsx[c];
        s2 += rsx[SM_NT + c];
      }
      s1 = warp_sum<double>(s1);
      s2 = warp_sum<double>(s2);
      if (lane == 0) {
        sc4[0] = s1;
        sc4[1] = s2;
      }
    }
    // local partial rows of A x+
    {
      double acc[R][V];
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int e = 0; e < V; ++e) acc[i][e] = 0.0;
      for (int c = 0; c < ncol; ++c) {
        const double xc = cf[c];
        if (xc == 0.0 && a.zskip) continue;  // a coordinate on its zero bound adds exactly nothing (CTA-uniform)
        const T* col = cols + (size_t)c * a.colstride;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const int row = row0 + i * (SM_NT * V);
          if (row < m) {
            T av[V];
            unpack<T>(*reinterpret_cast<const VT*>(col + row), av);
#pragma unroll
            for (int e = 0; e < V; ++e) acc[i][e] += static_cast<double>(av[e]) * xc;
          }
        }
      }
      if (timed) tsx[3] += clock64() - tp1;  // restart fold + the partial-row loop
      double* out = a.part + (int64_t)b * a.ldp;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int row = row0 + i * (SM_NT * V);
#pragma unroll
        for (int e = 0; e < V; ++e)
          if (row + e < m) out[row + e] = acc[i][e];
      }
    }
    // thread 0 wrote sc4 itself (warp 0's fold); the grid barrier's entry
    // CTA barrier orders every thread's partial rows before the arrival
    if (tid == 0 && a.kind == 2) {
      a.bpart[4 * b + 1] = sc4[0];
      a.bpart[4 * b + 2] = sc4[1];
    }
    const long long tp2 = timed ? clock64() : 0;
    grid_barrier(a.bar, nbar);
    const long long tp3 = timed ? clock64() : 0;
    // distributed reduce of this CTA's rows: one warp per row, lanes over
    // the G partials (independent L2 loads), one butterfly
    double sq = 0.0;
    for (int rr = warp; rr < nrow; rr += NW) {
      double s = 0.0;
      for (int q = lane; q < G; q += 32) s += __ldcg(&a.part[(int64_t)q * a.ldp + r_lo + rr]);
      s = warp_sum<double>(s);
      const double v = add_rn(s, coff[rr]);
      if (lane == 0) a.r[rc ^ 1][r_lo + rr] = v;
      sq += v * v;
    }
    if (lane == 0) red[warp] = sq;
    __syncthreads();
    // fold of the NW warp sums: one butterfly in warp 0 (fixed order)
    if (warp == 0) {
      const double s = warp_sum<double>(lane < NW ? red[lane] : 0.0);
      if (lane == 0) a.bpart[4 * b + 0] = s;
    }
    const long long tp4 = timed ? clock64() : 0;
    grid_barrier(a.bar, nbar);
    const long long tp5 = timed ? clock64() : 0;
    // the next step's residual rows (r just completed, r[rc ^ 1]), issued
    // before the fold below
#pragma unroll
    for (int q = 0; q < PR; ++q) {
      const int row = tid + q * SM_NT;
      if (row < m) pr[q] = __ldcg(&a.r[rc ^ 1][row]);
    }
    have_pre = true;
    // every CTA folds the same values in the same order -> same decision
    if (warp == 0) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      if (a.kind == 2) {
        for (int q = lane; q < G; q += 32) {
          s0 += __ldcg(&a.bpart[4 * q + 0]);
          s1 += __ldcg(&a.bpart[4 * q + 1]);
          s2 += __ldcg(&a.bpart[4 * q + 2]);
        }
        s1 = warp_sum<double>(s1);
        s2 = warp_sum<double>(s2);
      } else {
        for (int q = lane; q < G; q += 32) s0 += __ldcg(&a.bpart[4 * q + 0]);
      }
      s0 = warp_sum<double>(s0);
      if (lane == 0) {
        sc4[4] = s0;
        sc4[5] = s1;
        sc4[6] = s2;
      }
    }
    __syncthreads();
    const double Pn = 0.5 * sc4[4];
    if (a.kind == 2) {
      const double s_f = a.sc->rs_f * fmax(1.0, fabs(P));
      const double s_g = a.sc->rs_g * sqrt(2.0 * P) * sc4[6];
      const bool restart = (Pn > P + s_f) || (sc4[5] > s_g);
      if (b == 0 && tid == 0 && restart) a.sc->restarts += 1;
      t_mom = restart ? 1.0 : tn;
    } else {
      if (Pn > P + 1e-9 + a.sc->rise_rel * fabs(P)) {
        perr = true;
        if (b == 0 && tid == 0) {
          if (a.sc->err == 0) {
            a.sc->err_v1 = P;
            a.sc->err_v2 = Pn;
          }
          set_err(a.sc, DE_STEP_TOO_LARGE);
        }
      }
    }
    P = Pn;
    rc ^= 1;
    gv = 0;
    if (timed) {
      const long long tp6 = clock64();
      tsm[0] += tp1 - tp0;  // residual to shared memory, dots, column updates
      tsm[1] += tp2 - tp1;  // local partial rows of A x+
      tsm[2] += tp3 - tp2;  // grid barrier 1
      tsm[3] += tp4 - tp3;  // distributed row reduce
      tsm[4] += tp5 - tp4;  // grid barrier 2
      tsm[5] += tp6 - tp5;  // next residual rows + scalar fold
      ++tsm[6];
    }
    // no CTA barrier here: every shared-memory reuse of the next step (rv,
    // sc4, cf / rsx) is already separated from this step's reads by the
    // barriers above
  }
  // screening dot pass at the final x: g = A'r and the epsilon partial
  double ep = 0.0;
  if (a.do_dot) {
    if (have_pre) {
#pragma unroll
      for (int q = 0; q < PR; ++q)
        if (tid + q * SM_NT < m) rv[tid + q * SM_NT] = pr[q];
    } else {
      for (int row = tid; row < m; row += SM_NT) rv[row] = __ldcg(&a.r[rc][row]);
    }
    __syncthreads();
    dots(gcol);
    if (tid < ncol) {
      const double gj = gcol[tid];
      cg[tid] = gj;
      if (a.has_inf && isinf(chi[tid])) ep = fmax(-gj, 0.0) / fabs(cat[tid]);
    }
    // max is order independent
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ep = fmax(ep, __shfl_xor_sync(0xffffffffu, ep, o));
    if (lane == 0) red[warp] = ep;
    __syncthreads();
    if (tid == 0) {
      double e = 0.0;
      for (int w = 0; w < NW; ++w) e = fmax(e, red[w]);
      a.epart[b] = e;
    }
  }
  if (a.max_rounds <= 1) break;
  if (perr) {
    event = 1;
    break;
  }
  // ---- device dual point (driver.py:183-201), gap, stop and sphere tests ----
  grid_barrier(a.bar, nbar);
  const unsigned long long t_dual0 = (b == 0 && tid == 0) ? globaltimer() : 0ull;
  if (warp == 0) {
    double e = 0.0;
    for (int q = lane; q < G; q += 32) e = fmax(e, __ldcg(&a.epart[q]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
    if (lane == 0) sc4[2] = e;
  }
  __syncthreads();
  const double eps = a.has_inf ? sc4[2] : 0.0;
  {
    double s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
    for (int i = r_lo + tid; i < r_hi; i += SM_NT) {
      double th = -__ldcg(&a.r[rc][i]);
      if (eps > 0.0) th = add_rn(th, mul_rn(eps, a.t[i]));
      a.theta[i] = th;
      s1 += th * a.tgt[i];
      s2 += th * th;
    }
    if (tid < ncol) {
      double vj = -cg[tid];
      if (a.has_inf) vj = add_rn(vj, mul_rn(eps, cat[tid]));
      gcol[tid] = vj;  // v for the sphere test
      s3 = clo[tid] * fmin(vj, 0.0);
      if (!isinf(chi[tid])) s4 = chi[tid] * fmax(vj, 0.0);
    }
    s1 = warp_sum<double>(s1);
    s2 = warp_sum<double>(s2);
    s3 = warp_sum<double>(s3);
    s4 = warp_sum<double>(s4);
    if (lane == 0) {
      rsx[4 * warp + 0] = s1;
      rsx[4 * warp + 1] = s2;
      rsx[4 * warp + 2] = s3;
      rsx[4 * warp + 3] = s4;
    }
    __syncthreads();
    if (tid < 4) {
      double acc = 0.0;
      for (int w = 0; w < NW; ++w) acc += rsx[4 * w + tid];
      a.dpart[8 * b + tid] = acc;
    }
  }
  grid_barrier(a.bar, nbar);
  if (warp == 0) {
    double t1 = 0.0, t2 = 0.0, t3 = 0.0, t4 = 0.0;
    for (int q = lane; q < G; q += 32) {
      t1 += __ldcg(&a.dpart[8 * q + 0]);
      t2 += __ldcg(&a.dpart[8 * q + 1]);
      t3 += __ldcg(&a.dpart[8 * q + 2]);
      t4 += __ldcg(&a.dpart[8 * q + 3]);
    }
    t1 = warp_sum<double>(t1);
    t2 = warp_sum<double>(t2);
    t3 = warp_sum<double>(t3);
    t4 = warp_sum<double>(t4);
    if (lane == 0) {
      double dual = t1 - 0.5 * t2;
      dual -= t3;
      dual -= t4;
      sc4[3] = dual;
      sc4[4] = t2;
    }
  }
  __syncthreads();
  const double dual = sc4[3];
  const double raw = P - dual;
  const double gap = fmax(raw, 0.0);
  const double radius = sqrt(2.0 * gap / a.alpha);
  const double thr = radius + a.slack_scale * fmax(1.0, sqrt(sc4[4]));
  const double tol_r = a.relative_gap ? a.tol * fmax(1.0, fabs(P)) : a.tol;
  // events the host must handle: weak-duality violation, a convergence
  // candidate (certified gap), anything screened
  bool ev = (raw < -1e-9) || (gap < tol_r);
  int nscr = 0;
  if (a.screening && tid < ncol) {
    const double vj = gcol[tid];
    const double tj = thr * cnr[tid];
    nscr = (vj < -tj) || (vj > tj && !isinf(chi[tid]));
  }
  nscr = __syncthreads_count(nscr);
  if (tid == 0) a.dpart[8 * b + 4] = (double)nscr;
  grid_barrier(a.bar, nbar);
  if (warp == 0) {
    double c = 0.0;
    for (int q = lane; q < G; q += 32) c += __ldcg(&a.dpart[8 * q + 4]);
    c = warp_sum<double>(c);
    if (lane == 0) sc4[5] = c;
  }
  __syncthreads();
  ev = ev || (sc4[5] > 0.0);
  if (ev) {
    event = 1;
    break;
  }
  if (b == 0 && tid == 0) {
    const unsigned long long t_end = globaltimer();
    if (!a.screening) excl_ns += (double)(t_end - t_dual0);
    double* tr = a.trace + TRACE_W * rnd;
    tr[0] = P;
    tr[1] = dual;
    tr[2] = gap;
    tr[3] = eps;
    tr[4] = radius;
    tr[5] = t_mom;
    tr[6] = (double)a.sc->restarts;
    tr[7] = (double)t_end;
    tr[8] = excl_ns;
  }
  ++done_rounds;
  gv = 1;  // the next round starts from this round's screening gradient
  __syncthreads();
  }  // rounds
  if (timed)
    for (int q = 0; q < 7; ++q) atomicAdd(a.dbg + q, (unsigned long long)tsm[q]);
  if (timed)
    for (int q = 0; q < 4; ++q) atomicAdd(a.dbg + 8 + q, (unsigned long long)tsx[q]);
  // write back the resident per-column state
  if (tid < ncol) {
    const int64_t p = p0 + tid;
    a.x[p] = cx[tid];
    if (a.kind == 2) {
      a.xprev[p] = cxp[tid];
      a.gprev[p] = cgp[tid];
    }
    a.g[p] = cg[tid];
  }
  if (b == 0 && tid == 0) {
    a.sc->P = P;
    a.sc->mom_t = t_mom;
    if (a.done) {
      a.done[0] = done_rounds;
      a.done[1] = event;
      a.done[2] = rc;
    }
  }
}

}  // namespace bx
