// bx_batched.cuh -- batched many-right-hand-side FISTA with per-problem
// Gap-safe screening on fp64 tensor cores (BASELINE config 5; semantics in
// oracle/batched_oracle.py).
//
// K NNLS problems share one dictionary A (m x n, m <= 208).  A persistent CTA
// (16 warps: 8 tiles of 8 problems x 2 coordinate / row halves) owns a tile of
// 64 problems and runs whole rounds for it with no grid-wide
// dependency (problems are independent).  Per FISTA step it streams A in
// chunks J of 16 columns (A is L2 resident: 8 MB at config 5) together with
// the tile's x / x_prev chunk (HBM), and per chunk
//     G_J  = A_J' R_y                       (16 x 64, K = m)   DMMA m8n8k4
//     X+_J = max(Y_J - eta G_J, 0) on the active set  (epilogue, registers)
//     R+  += A_J X+_J                       (m x 64,  K = 16)  DMMA m8n8k4
// so the gradient matrix never reaches HBM.  R+ lives in registers (each warp
// 8 problems x half the rows); the per-problem restart tests, objective, dual point,
// gap, radius and the sphere test are all tile-local.
#pragma once
#include "bx_kernels.cuh"
#include "bx_cd.cuh"  // cp.async helpers

namespace bx {

constexpr int BT_NT = 512;    // threads (16 warps: 8 problem tiles x 2 halves)
constexpr int BT_TILE = 64;   // problems per tile (8 per warp column)
constexpr int BT_CH = 16;     // dictionary columns per chunk
constexpr int BT_MT = 26;     // max m8 row tiles (m <= 208)
constexpr int BT_MH = 13;     // row tiles per warp half (GEMM2 accumulators)
constexpr int BT_SX = 20;     // smem stride of x tiles (== 4 mod 16: conflict-free fragments)

struct BatchArgs {
  const double* A;     // m x n, column stride lda
  int64_t lda;
  int m, n, K;         // K = number of problems (multiple of BT_TILE)
  int sa;              // smem stride of A chunks / residual tiles (>= m8, == 4 mod 16)
  const double* Y;     // m x K, stride ldy
  int64_t ldy;
  double* X[2];        // n x K ping-pong (stride ldx)
  double* R[2];        // m x K ping-pong (stride ldy)
  int64_t ldx;
  uint32_t* mask;      // active bits: word k * nw + j / 32
  int nw;
  const double* nrm;   // ||a_j||
  const double* att;   // a_j' t (t = -1)
  double* mom;         // per-problem FISTA t
  double* P;           // per-problem objective 0.5 ||r||^2 at x
  double* stats;       // per problem: [primal, dual, gap, eps, preserved] (5 x K)
  double eta;
  int passes;
  int par;             // buffer parity at entry: X[par], R[par] hold x, r; X[1-par], R[1-par] hold x_prev, r_prev
  int screening;
  double rs_f, rs_g, slack_scale;
  // second schedule (bx_batched2.cuh): the dictionary packed chunk by chunk
  // in the ring's stage layout (k_b2_pack), a whole number of 16-column chunks
  const double* Ap;
  int nch;             // chunks
  int tile0, tile1;    // tile range of this launch (second schedule)
  // rounds per launch (second schedule): units (round, tile) in round-major
  // order; round0 = rounds completed before this launch; per-octet completed
  // round flags; per-octet round summaries [osum_rounds][K / 8][4]
  int nrl, round0;
  unsigned* oct_round;
  double* osum;
  int osum_rounds;
  int64_t K_user;
  double gap_tol;
  double att_max, nrm_min;        // max_j |a_j't|, min_j ||a_j|| over the real columns (sphere-test bound)
  int bound_skip;                 // 1: skip the per-coordinate sphere sweep of tiles the bound clears
  unsigned long long* sweeps2;    // tiles that ran the per-coordinate sweep (counter; may be null)
  unsigned long long* dbg;  // BX_BT_DEBUG: per-warp wait counters of the second schedule (null otherwise)
  int sa2;             // column stride of the second schedule's tiles (>= m8, == 4 mod 8)
};

// not volatile: a pure function of its operands, so the compiler may
// schedule it freely
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct BatchSmem {
  double* rys;   // [64][sa]   residual (or extrapolated residual) of the tile
  double* abuf;  // [2][16][sa] dictionary chunks
  double* xs;    // [2][64][SX] x chunk
  double* xps;   // [2][64][SX] x_prev chunk
  double* xns;   // [64][SX]   new x chunk
  uint32_t* mk;  // [2][64]    mask words of the chunk
  double* red;   // scratch [8][64]
  double* beta;  // [64]
};

// This thread's 16-byte pieces of a dictionary chunk (16 columns x m rows),
// decomposed once per kernel: the (column, row) split of a piece index is the
// same for every chunk, so the per-chunk copy loop has no integer division.
__host__ __device__ constexpr int bt_pmax(int nt) { return (BT_CH * (BT_MT * 8 / 2) + nt - 1) / nt; }
template <int NTH>
struct BtPlan {
  static constexpr int PM = bt_pmax(NTH);
  int jj[PM];    // column within the chunk (BT_CH: no piece)
  int soff[PM];  // smem offset (doubles)
  int goff[PM];  // global offset from the chunk's first column (doubles)
};
template <int NTH>
__device__ __forceinline__ BtPlan<NTH> bt_plan(const BatchArgs& a) {
  BtPlan<NTH> pl;
  const int mv = (a.m + 1) / 2;
#pragma unroll
  for (int i = 0; i < BtPlan<NTH>::PM; ++i) {
    const int q = threadIdx.x + i * NTH;
    const int jj = q < BT_CH * mv ? q / mv : BT_CH;
    const int v = q - jj * mv;
    pl.jj[i] = jj;
    pl.soff[i] = jj * a.sa + 2 * v;
    pl.goff[i] = (int)(jj * a.lda) + 2 * v;
  }
  return pl;
}

template <int TILE>
__device__ __forceinline__ void bt_prefetch(const BatchArgs& a, const BtPlan<TILE * 8>& pl, const BatchSmem& s,
                                            int buf, int c, int k0, const double* X, const double* Xp, bool with_x) {
  constexpr int NT_ = TILE * 8;
  const int j0 = c * BT_CH;
  const int nj = min(BT_CH, a.n - j0);
  // A chunk: 16 columns x m rows (16-byte pieces)
  double* ab = s.abuf + buf * BT_CH * a.sa;
  const double* ag = a.A + (int64_t)j0 * a.lda;
#pragma unroll
  for (int i = 0; i < BtPlan<NT_>::PM; ++i) {
    if (pl.jj[i] < nj)
      cp_async16(ab + pl.soff[i], ag + pl.goff[i]);
    else if (pl.jj[i] < BT_CH)
      *reinterpret_cast<double2*>(ab + pl.soff[i]) = make_double2(0.0, 0.0);
  }
  if (with_x) {
    // x / x_prev chunks: TILE problems x 16 coordinates
    double* xs = s.xs + buf * TILE * BT_SX;
    double* xp = s.xps + buf * TILE * BT_SX;
    for (int q = threadIdx.x; q < TILE * 8; q += NT_) {
      const int nn = q >> 3, v = q & 7;
      if (2 * v < nj) {
        cp_async16(xs + nn * BT_SX + 2 * v, X + (int64_t)(k0 + nn) * a.ldx + j0 + 2 * v);
        if (Xp) cp_async16(xp + nn * BT_SX + 2 * v, Xp + (int64_t)(k0 + nn) * a.ldx + j0 + 2 * v);
      }
    }
  }
  if (threadIdx.x < TILE) {
    const int w = j0 >> 5;
    s.mk[buf * TILE + threadIdx.x] = a.mask[(int64_t)(k0 + threadIdx.x) * a.nw + w];
  }
  cp_async_commit();
}

// G tile (coords 8 mh + g, problems n0 + 2 tig + e) = A_J' Ry: one 8x8 output
// tile per warp, K = m in steps of 4.  Four independent accumulator sets
// (k-steps interleaved) keep 4 DMMA chains in flight per warp (a single chain
// is DMMA-latency bound); they are summed in a fixed order (deterministic).
__device__ __forceinline__ void bt_gemm1(const BatchArgs& a, const double* ab, const double* rys, int n0, int mh,
                                         int g, int tig, double (&gt)[2]) {
  double acc[4][2];
#pragma unroll
  for (int u = 0; u < 4; ++u) acc[u][0] = acc[u][1] = 0.0;
  const int m4 = (a.m + 3) / 4;
  const double* rb = rys + (n0 + g) * a.sa + tig;
  const double* a0 = ab + (8 * mh + g) * a.sa + tig;
  int kk = 0;
  for (; kk + 4 <= m4; kk += 4) {
    double b[4], x0[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      b[u] = rb[4 * (kk + u)];
      x0[u] = a0[4 * (kk + u)];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(acc[u][0], acc[u][1], x0[u], b[u]);
  }
  // remainder (m4 % 4 k-steps): warp-uniform, unrolled per count so no
  // DMMA sits in a data-dependent loop
  switch (m4 - kk) {
    case 3: dmma(acc[2][0], acc[2][1], a0[4 * (kk + 2)], rb[4 * (kk + 2)]);  // fallthrough
    case 2: dmma(acc[1][0], acc[1][1], a0[4 * (kk + 1)], rb[4 * (kk + 1)]);  // fallthrough
    case 1: dmma(acc[0][0], acc[0][1], a0[4 * kk], rb[4 * kk]); break;
    default: break;
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) gt[e] = (acc[0][e] + acc[1][e]) + (acc[2][e] + acc[3][e]);
}

// acc (rows 8 (mlo + q) + g, problems n0 + 2 tig + e) += A_J X_J over this
// warp's row half [mlo, mlo + NQ); K = 16 coordinates.  NQ is a compile-time
// tile count: an unguarded, fully unrolled DMMA sequence (a per-tile guard
// makes every DMMA predicated, and the compiler then brackets each one with
// WARPSYNC + NOP)
template <int NQ>
__device__ __forceinline__ void bt_gemm2_n(const BatchArgs& a, const double* ab, const double* xns, int n0, int g,
                                           int tig, double (&acc)[BT_MH][2], int mlo) {
  const double* ag = ab + 8 * mlo + g;
#pragma unroll
  for (int kk = 0; kk < BT_CH / 4; ++kk) {
    const int j = 4 * kk + tig;
    const double b = xns[(n0 + g) * BT_SX + j];
    const double* aj = ag + j * a.sa;
#pragma unroll
    for (int q = 0; q < NQ; ++q) dmma(acc[q][0], acc[q][1], aj[8 * q], b);
  }
}
__device__ __forceinline__ void bt_gemm2(const BatchArgs& a, const double* ab, const double* xns, int n0, int g,
                                         int tig, double (&acc)[BT_MH][2], int mlo, int mhi) {
  // warp-uniform dispatch on the tile count of this row half
  switch (mhi - mlo) {
    case 13: bt_gemm2_n<13>(a, ab, xns, n0, g, tig, acc, mlo); break;
    case 12: bt_gemm2_n<12>(a, ab, xns, n0, g, tig, acc, mlo); break;
    case 11: bt_gemm2_n<11>(a, ab, xns, n0, g, tig, acc, mlo); break;
    case 10: bt_gemm2_n<10>(a, ab, xns, n0, g, tig, acc, mlo); break;
    case 9: bt_gemm2_n<9>(a, ab, xns, n0, g, tig, acc, mlo); break;
    case 8: bt_gemm2_n<8>(a, ab, xns, n0, g, tig, acc, mlo); break;
    case 7: bt_gemm2_n<7>(a, ab, xns, n0, g, tig, acc, mlo); break;
    case 6: bt_gemm2_n<6>(a, ab, xns, n0, g, tig, acc, mlo); break;
    case 5: bt_gemm2_n<5>(a, ab, xns, n0, g, tig, acc, mlo); break;
    case 4: bt_gemm2_n<4>(a, ab, xns, n0, g, tig, acc, mlo); break;
    case 3: bt_gemm2_n<3>(a, ab, xns, n0, g, tig, acc, mlo); break;
    case 2: bt_gemm2_n<2>(a, ab, xns, n0, g, tig, acc, mlo); break;
    case 1: bt_gemm2_n<1>(a, ab, xns, n0, g, tig, acc, mlo); break;
    default: break;
  }
}

// TILE = 64: 16 warps, double-buffered dictionary chunks, one CTA per SM;
// TILE = 32: 8 warps, single-buffered chunks, two CTAs per SM (each CTA's
// chunk-copy waits and barriers overlap the other CTA's DMMA work)
template <int TILE>
__global__ void __launch_bounds__(TILE * 8, 512 / (TILE * 8)) k_batched_round(const BatchArgs a) {
  constexpr int NT_ = TILE * 8;
  constexpr int NTW = TILE / 8;             // problem tiles (of 8) per CTA
  constexpr int NB = TILE == 64 ? 2 : 1;    // dictionary chunk buffers
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int nt = warp % NTW, mh = warp / NTW;  // problem tile of this warp, coordinate / row half
  const int n0 = nt * 8;
  BatchSmem s;
  {
    double* p = reinterpret_cast<double*>(smem_raw);
    s.rys = p;
    p += TILE * a.sa;
    s.abuf = p;
    p += NB * BT_CH * a.sa;
    s.xs = p;
    p += NB * TILE * BT_SX;
    s.xps = p;
    p += NB * TILE * BT_SX;
    s.xns = p;
    p += TILE * BT_SX;
    s.red = p;  // [8][64]: per-problem partials of the two warp halves
    p += 8 * TILE;
    s.beta = p;
    p += TILE;
    s.mk = reinterpret_cast<uint32_t*>(p);
  }
  const BtPlan<NT_> pl = bt_plan<NT_>(a);
  const int mt_n = (a.m + 7) / 8;
  const int mlo = mh ? BT_MH : 0, mhi = mh ? mt_n : min(BT_MH, mt_n);
  const int nch = (a.n + BT_CH - 1) / BT_CH;
  const int ntiles = a.K / TILE;
  // zero both dictionary buffers once: rows in [m, sa) and columns past n are
  // never written by the chunk copies and must multiply as exact zeros
  for (int q = tid; q < NB * BT_CH * a.sa; q += NT_) s.abuf[q] = 0.0;
  __syncthreads();

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int k0 = tile * TILE;
    int par = a.par;
    // ---------------- FISTA steps ----------------
    for (int pass = 0; pass < a.passes; ++pass) {
      const double* X = a.X[par];
      double* Xp = a.X[1 - par];  // read as x_prev, then overwritten by x+
      const double* R = a.R[par];
      double* Rp = a.R[1 - par];
      if (tid < TILE) {
        const double t = a.mom[k0 + tid];
        const double tn = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
        s.beta[tid] = (t - 1.0) / tn;
      }
      __syncthreads();
      // R_y = R + beta (R - R_prev)  (rows >= m zero padded)
      for (int q = tid; q < TILE * a.sa; q += NT_) {
        const int nn = q / a.sa, i = q - nn * a.sa;
        double v = 0.0;
        if (i < a.m) {
          const double r = R[(int64_t)(k0 + nn) * a.ldy + i];
          const double bt = s.beta[nn];
          v = r;
          if (bt != 0.0) v = add_rn(r, mul_rn(bt, sub_rn(r, Rp[(int64_t)(k0 + nn) * a.ldy + i])));
        }
        s.rys[q] = v;
      }
      double acc[BT_MH][2];
#pragma unroll
      for (int q = 0; q < BT_MH; ++q) acc[q][0] = acc[q][1] = 0.0;
      double gdot[2] = {0.0, 0.0}, gsc[2] = {0.0, 0.0};
      const double bt0 = s.beta[n0 + 2 * tig], bt1 = s.beta[n0 + 2 * tig + 1];
      bt_prefetch<TILE>(a, pl, s, 0, 0, k0, X, Xp, true);
      for (int c = 0; c < nch; ++c) {
        if (NB == 1 && c > 0) {  // the single buffer is free once every warp left chunk c-1
          __syncthreads();
          bt_prefetch<TILE>(a, pl, s, 0, c, k0, X, Xp, true);
        }
        const int buf = NB == 2 ? (c & 1) : 0;
        cp_async_wait_all();
        __syncthreads();
        if (NB == 2 && c + 1 < nch) bt_prefetch<TILE>(a, pl, s, buf ^ 1, c + 1, k0, X, Xp, true);
        const double* ab = s.abuf + buf * BT_CH * a.sa;
        const double* xs = s.xs + buf * TILE * BT_SX;
        const double* xps = s.xps + buf * TILE * BT_SX;
        const uint32_t* mk = s.mk + buf * TILE;
        double gt[2];
        bt_gemm1(a, ab, s.rys, n0, mh, g, tig, gt);
        // epilogue: the FISTA update of this lane's two elements
        const int j0 = c * BT_CH;
        {
          const int jj = 8 * mh + g;
          const int j = j0 + jj;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int nn = n0 + 2 * tig + e;
            double xn = 0.0;
            if (j < a.n) {
              const bool act = (mk[nn] >> (j & 31)) & 1u;
              const double x = xs[nn * BT_SX + jj], xp = xps[nn * BT_SX + jj];
              const double bt = e ? bt1 : bt0;
              double yv = x;
              if (bt != 0.0) yv = add_rn(x, mul_rn(bt, sub_rn(x, xp)));
              if (act) {
                xn = sub_rn(yv, mul_rn(a.eta, gt[e]));
                xn = xn < 0.0 ? 0.0 : xn;
              }
              const double dx = xn - x;
              gdot[e] += gt[e] * dx;
              gsc[e] += a.nrm[j] * fabs(dx);
            }
            s.xns[nn * BT_SX + jj] = xn;
          }
        }
        // only the warp pair of problem tile nt shares these xns rows: a
        // named barrier per pair instead of a CTA barrier, so pairs drift and
        // one pair's epilogue overlaps another's DMMA work
        asm volatile("bar.sync %0, 64;" ::"r"(1 + nt) : "memory");
        // x+ chunk -> global (the x_prev slot, already consumed for this chunk)
        {
          const int nj = min(BT_CH, a.n - j0);
          for (int q = mh * 32 + lane; q < 8 * BT_CH; q += 64) {
            const int nn = n0 + q / BT_CH, jj = q % BT_CH;
            if (jj < nj) Xp[(int64_t)(k0 + nn) * a.ldx + j0 + jj] = s.xns[nn * BT_SX + jj];
          }
        }
        bt_gemm2(a, ab, s.xns, n0, g, tig, acc, mlo, mhi);
      }
      // r+ = A x+ - y  (into the r_prev slot), objective, restart test
      double sq[2] = {0.0, 0.0};
#pragma unroll
      for (int q = 0; q < BT_MH; ++q) {
        const int i = 8 * (mlo + q) + g;
        if (mlo + q < mhi && i < a.m) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int nn = n0 + 2 * tig + e;
            const double r = acc[q][e] - a.Y[(int64_t)(k0 + nn) * a.ldy + i];
            Rp[(int64_t)(k0 + nn) * a.ldy + i] = r;
            sq[e] += r * r;
          }
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          sq[e] += __shfl_xor_sync(0xffffffffu, sq[e], o);
          gdot[e] += __shfl_xor_sync(0xffffffffu, gdot[e], o);
          gsc[e] += __shfl_xor_sync(0xffffffffu, gsc[e], o);
        }
      }
      if (g == 0) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int nn = n0 + 2 * tig + e;
          s.red[(0 + mh) * TILE + nn] = sq[e];
          s.red[(2 + mh) * TILE + nn] = gdot[e];
          s.red[(4 + mh) * TILE + nn] = gsc[e];
        }
      }
      __syncthreads();
      if (tid < TILE) {
        const int k = k0 + tid;
        const double Pn = 0.5 * (s.red[tid] + s.red[TILE + tid]);
        const double gd = s.red[2 * TILE + tid] + s.red[3 * TILE + tid];
        const double gs = s.red[4 * TILE + tid] + s.red[5 * TILE + tid];
        const double P = a.P[k];
        const double t = a.mom[k];
        const double tn = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
        const double s_f = a.rs_f * fmax(1.0, fabs(P));
        const double s_g = a.rs_g * sqrt(2.0 * P) * gs;
        a.mom[k] = (Pn > P + s_f || gd > s_g) ? 1.0 : tn;
        a.P[k] = Pn;
      }
      par ^= 1;
      __syncthreads();
    }
    // ---------------- dual point, gap, sphere test at x ----------------
    {
      const double* X = a.X[par];
      double* Xq = a.X[1 - par];
      const double* R = a.R[par];
      // r at x into smem
      for (int q = tid; q < TILE * a.sa; q += NT_) {
        const int nn = q / a.sa, i = q - nn * a.sa;
        s.rys[q] = (i < a.m) ? R[(int64_t)(k0 + nn) * a.ldy + i] : 0.0;
      }
      // sweep 1: epsilon_k = max_j (v_jk)+ / |a_j't|, v = -A'r
      double emax[2] = {0.0, 0.0};
      bt_prefetch<TILE>(a, pl, s, 0, 0, k0, X, nullptr, false);
      for (int c = 0; c < nch; ++c) {
        if (NB == 1 && c > 0) {  // the single buffer is free once every warp left chunk c-1
          __syncthreads();
          bt_prefetch<TILE>(a, pl, s, 0, c, k0, X, nullptr, false);
        }
        const int buf = NB == 2 ? (c & 1) : 0;
        cp_async_wait_all();
        __syncthreads();
        if (NB == 2 && c + 1 < nch) bt_prefetch<TILE>(a, pl, s, buf ^ 1, c + 1, k0, X, nullptr, false);
        double gt[2];
        bt_gemm1(a, s.abuf + buf * BT_CH * a.sa, s.rys, n0, mh, g, tig, gt);
        const int j = c * BT_CH + 8 * mh + g;
        if (j < a.n) {
          const double inv = 1.0 / fabs(a.att[j]);
#pragma unroll
          for (int e = 0; e < 2; ++e) emax[e] = fmax(emax[e], fmax(-gt[e], 0.0) * inv);
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) emax[e] = fmax(emax[e], __shfl_xor_sync(0xffffffffu, emax[e], o));
      if (g == 0) {
        s.red[mh * TILE + n0 + 2 * tig] = emax[0];
        s.red[mh * TILE + n0 + 2 * tig + 1] = emax[1];
      }
      __syncthreads();
      if (tid < TILE) s.beta[tid] = fmax(s.red[tid], s.red[TILE + tid]);  // eps per problem
      __syncthreads();
      // dual objective per problem: theta = -r + eps t (t = -1): theta_i = -r_i - eps
      for (int pb = warp; pb < TILE; pb += NT_ / 32) {
        const double eps = s.beta[pb];
        double s1 = 0.0, s2 = 0.0;
        for (int i = lane; i < a.m; i += 32) {
          double th = -s.rys[pb * a.sa + i];
          if (eps > 0.0) th = add_rn(th, mul_rn(eps, -1.0));
          s1 += th * a.Y[(int64_t)(k0 + pb) * a.ldy + i];
          s2 += th * th;
        }
        s1 = warp_sum<double>(s1);
        s2 = warp_sum<double>(s2);
        if (lane == 0) {
          const int k = k0 + pb;
          const double P = a.P[k];
          const double D = s1 - 0.5 * s2;
          const double gap = fmax(P - D, 0.0);
          double* st = a.stats;
          st[k] = P;
          st[a.K + k] = D;
          st[2 * a.K + k] = gap;
          st[3 * a.K + k] = eps;
          s.red[6 * TILE + pb] = sqrt(2.0 * gap) + a.slack_scale * fmax(1.0, sqrt(s2));  // radius + slack
        }
      }
      __syncthreads();
      // sweep 2: v = -g + eps a't ; screen v < -(radius + slack) ||a_j||
      __shared__ int dirty;
      if (tid == 0) dirty = 0;
      if (a.screening) {
        bt_prefetch<TILE>(a, pl, s, 0, 0, k0, X, nullptr, false);
        for (int c = 0; c < nch; ++c) {
          if (NB == 1 && c > 0) {  // the single buffer is free once every warp left chunk c-1
            __syncthreads();
            bt_prefetch<TILE>(a, pl, s, 0, c, k0, X, nullptr, false);
          }
          const int buf = NB == 2 ? (c & 1) : 0;
          cp_async_wait_all();
          __syncthreads();
          if (NB == 2 && c + 1 < nch) bt_prefetch<TILE>(a, pl, s, buf ^ 1, c + 1, k0, X, nullptr, false);
          double gt[2];
          bt_gemm1(a, s.abuf + buf * BT_CH * a.sa, s.rys, n0, mh, g, tig, gt);
          const uint32_t* mk = s.mk + buf * TILE;
          const int j = c * BT_CH + 8 * mh + g;
          if (j < a.n) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int nn = n0 + 2 * tig + e;
              const bool act = (mk[nn] >> (j & 31)) & 1u;
              const double v = add_rn(-gt[e], mul_rn(s.beta[nn], a.att[j]));
              if (act && v < -s.red[6 * TILE + nn] * a.nrm[j]) {
                const int64_t k = k0 + nn;
                atomicAnd(&a.mask[k * a.nw + (j >> 5)], ~(1u << (j & 31)));
                const_cast<double*>(X)[k * a.ldx + j] = 0.0;
                Xq[k * a.ldx + j] = 0.0;
                dirty = 1;
              }
            }
          }
        }
      }
      __syncthreads();
      if (dirty) {
        // refresh r = A x - y and r_prev = A x_prev - y (screened x snapped to 0)
        for (int which = 0; which < 2; ++which) {
          const double* Xw = which ? Xq : X;
          double* Rw = a.R[which ? 1 - par : par];
          double acc[BT_MH][2];
#pragma unroll
          for (int q = 0; q < BT_MH; ++q) acc[q][0] = acc[q][1] = 0.0;
          bt_prefetch<TILE>(a, pl, s, 0, 0, k0, Xw, nullptr, true);
          for (int c = 0; c < nch; ++c) {
            if (NB == 1 && c > 0) {  // the single buffer is free once every warp left chunk c-1
              __syncthreads();
              bt_prefetch<TILE>(a, pl, s, 0, c, k0, Xw, nullptr, true);
            }
            const int buf = NB == 2 ? (c & 1) : 0;
            cp_async_wait_all();
            __syncthreads();
            if (NB == 2 && c + 1 < nch) bt_prefetch<TILE>(a, pl, s, buf ^ 1, c + 1, k0, Xw, nullptr, true);
            // stage the chunk in the conflict-free layout of xns
            const double* xs = s.xs + buf * TILE * BT_SX;
            const int nj = min(BT_CH, a.n - c * BT_CH);
            for (int q = tid; q < TILE * BT_CH; q += NT_) {
              const int nn = q / BT_CH, jj = q - nn * BT_CH;
              s.xns[nn * BT_SX + jj] = (jj < nj) ? xs[nn * BT_SX + jj] : 0.0;
            }
            __syncthreads();
            bt_gemm2(a, s.abuf + buf * BT_CH * a.sa, s.xns, n0, g, tig, acc, mlo, mhi);
          }
          double sq[2] = {0.0, 0.0};
#pragma unroll
          for (int q = 0; q < BT_MH; ++q) {
            const int i = 8 * (mlo + q) + g;
            if (mlo + q < mhi && i < a.m) {
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int nn = n0 + 2 * tig + e;
                const double r = acc[q][e] - a.Y[(int64_t)(k0 + nn) * a.ldy + i];
                Rw[(int64_t)(k0 + nn) * a.ldy + i] = r;
                sq[e] += r * r;
              }
            }
          }
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) sq[e] += __shfl_xor_sync(0xffffffffu, sq[e], o);
          if (g == 0) {
            s.red[mh * TILE + n0 + 2 * tig] = sq[0];
            s.red[mh * TILE + n0 + 2 * tig + 1] = sq[1];
          }
          __syncthreads();
          if (which == 0 && tid < TILE) a.P[k0 + tid] = 0.5 * (s.red[tid] + s.red[TILE + tid]);
          __syncthreads();
        }
      }
      // preserved counts
      for (int pb = warp; pb < TILE; pb += NT_ / 32) {
        int cnt = 0;
        for (int w = lane; w < a.nw; w += 32) cnt += __popc(a.mask[(int64_t)(k0 + pb) * a.nw + w]);
        cnt = warp_sum<int>(cnt);
        if (lane == 0) a.stats[4 * a.K + k0 + pb] = cnt;
      }
      __syncthreads();
    }
  }
}

// initial state: x = x_prev = 0, r = r_prev = -y, P = 0.5||y||^2, t = 1, all active
__global__ void k_batched_init(BatchArgs a) {
  const int64_t tot = (int64_t)a.K * a.ldy;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < tot; q += (int64_t)gridDim.x * blockDim.x) {
    const double v = -a.Y[q];
    a.R[0][q] = v;
    a.R[1][q] = v;
  }
  const int64_t totx = (int64_t)a.K * a.ldx;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < totx; q += (int64_t)gridDim.x * blockDim.x) {
    a.X[0][q] = 0.0;
    a.X[1][q] = 0.0;
  }
  const int64_t totm = (int64_t)a.K * a.nw;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < totm; q += (int64_t)gridDim.x * blockDim.x) {
    const int w = (int)(q % a.nw);
    const int lo = w * 32;
    const int nb = min(32, a.n - lo);
    a.mask[q] = nb >= 32 ? 0xffffffffu : ((1u << nb) - 1u);
  }
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < a.K; k += (int64_t)gridDim.x * blockDim.x) {
    a.mom[k] = 1.0;
    double s = 0.0;
    for (int i = 0; i < a.m; ++i) {
      const double y = a.Y[k * a.ldy + i];
      s += y * y;
    }
    a.P[k] = 0.5 * s;
  }
}

}  // namespace bx
