// bx_batched2.cuh -- batched many-right-hand-side FISTA, second schedule
// (BASELINE config 5; semantics in oracle/batched_oracle.py, the same as
// bx_batched.cuh's first schedule, which stays selectable with BX_BT_V1=1).
//
// One warp owns a problem octet outright: both products of a FISTA step,
// the update between them and every per-problem reduction stay inside the
// warp, so a step has no CTA barrier and no cross-warp traffic at all.  The
// eight warps of a CTA share only the dictionary stream: 16-column chunks of
// A (L2 resident) land in a 4-stage shared-memory ring by cp.async.bulk (TMA
// bulk engine, mbarrier completion); a stage is refilled by whichever warp
// releases it last (a counter per stage), so there is no producer warp and
// no warp ever waits for a slower one except through the ring's depth.
//
// Per chunk J and octet (m8n8k4 fp64 MMA = SASS DMMA.8x8x4):
//     G'_J = R_y' A_J      (8 problems x 16 coords, K = m)   R_y' is the A operand
//     X+_J = max(Y_J - eta G'_J, 0) on the active set         registers only
//     R+  += A_J X+_J      (m rows x 8 problems, K = 16)
// Computing the gradient tile transposed puts a lane's two outputs on ONE
// problem and two neighbouring coordinates, which (a) is exactly the B
// fragment GEMM2 needs when its K index runs over (tile, parity) pairs, so
// x+ never leaves registers between the two products, and (b) makes the
// x / x_prev loads and the x+ store 16-byte vectors (64 contiguous bytes per
// problem per quad) straight from / to HBM with no staging.  Operand loads:
// GEMM1 1.5 LDS.64 per DMMA (one R_y fragment feeds both coordinate tiles),
// GEMM2 1 (the x+ fragment is in registers), against 2 and 1.08 before.
// Chunk columns sit in the ring under a slot permutation that keeps both
// products' fragment loads bank-conflict free with one column stride.
#pragma once
#include "bx_batched.cuh"

namespace bx {

constexpr int B2_NW = 8;                 // warps per CTA = problem octets per tile
constexpr int B2_NT = 32 * B2_NW;
constexpr int B2_NST = 4;                // ring stages
constexpr int B2_MT = BT_MT;             // max m8 row tiles

// ring slot of chunk column c (0..15): within each 8-column tile the upper
// four columns swap pairwise, so that {c, c+2, c+4, c+6} and {0..3}, {4..7}
// all hit distinct residues mod 4 (times a stride == 4 mod 16 doubles)
__host__ __device__ constexpr int b2_slot(int c) { return (c & 8) | ((c & 7) ^ ((c >> 2) & 1)); }

struct B2Ring {
  double* stage;   // [NST][16][sa]: column slots; rows sa - 2, sa - 1 of a slot hold ||a_j||, a_j't
  uint64_t* full;  // [NST] mbarriers (tx-count completion)
  int* cnt;        // [NST] warps that released the stage
  int it;          // chunks consumed so far (the same sequence in every warp)
  int sa;          // column stride (doubles), == 4 mod 8
  int sstride;     // stage stride (doubles) = 16 sa
};

// chunk (q mod nch) -> stage (q mod NST).  The packed dictionary (k_b2_pack)
// stores every chunk exactly as it sits in a stage, so a refill is ONE bulk
// copy (16 sa doubles) issued by one lane.
__device__ __forceinline__ void b2_issue(const BatchArgs& a, const B2Ring& rg, int q, int lane, uint64_t pol) {
  if (lane == 0) {
    const int s = q % B2_NST;
    const int c = q % a.nch;
    const uint32_t bytes = (uint32_t)(rg.sstride * 8);
    mbar_expect_tx(&rg.full[s], bytes);
    bulk_g2s(rg.stage + (size_t)s * rg.sstride, a.Ap + (int64_t)c * rg.sstride, bytes, &rg.full[s], pol);
  }
}

__device__ __forceinline__ const double* b2_acquire(const BatchArgs& a, const B2Ring& rg) {
  const int s = rg.it % B2_NST;
  mbar_wait(&rg.full[s], (uint32_t)((rg.it / B2_NST) & 1));
  return rg.stage + (size_t)s * rg.sstride;
}

// stage of chunk q (anywhere ahead in the sequence: waiting does not consume)
__device__ __forceinline__ const double* b2_acquire_at(const B2Ring& rg, int q) {
  const int s = q % B2_NST;
  mbar_wait(&rg.full[s], (uint32_t)((q / B2_NST) & 1));
  return rg.stage + (size_t)s * rg.sstride;
}

// This warp is done with the current stage.  Split in two so that nobody
// waits for the counter's round trip: _begin posts the arrival (lane 0's
// return value stays in flight), _end -- called a chunk later -- looks at it,
// and the last of the CTA's warps to have arrived refills the stage with the
// chunk NST ahead.
__device__ __forceinline__ int b2_release_begin(B2Ring& rg, int lane) {
  const int s = rg.it % B2_NST;
  __syncwarp();
  int old = 0;
  if (lane == 0)
    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(&rg.cnt[s])) : "memory");
  ++rg.it;
  return old;
}
// q = the chunk index the arrival was for
__device__ __forceinline__ void b2_release_end(const BatchArgs& a, const B2Ring& rg, int old, int q, int lane,
                                               uint64_t pol) {
  const int last = __shfl_sync(0xffffffffu, old == B2_NW - 1, 0);
  if (last) {
    if (lane == 0) {
      rg.cnt[q % B2_NST] = 0;
      fence_proxy_async_smem();
    }
    b2_issue(a, rg, q + B2_NST, lane, pol);
  }
}
__device__ __forceinline__ void b2_release(const BatchArgs& a, B2Ring& rg, int lane, uint64_t pol) {
  const int q = rg.it;
  const int old = b2_release_begin(rg, lane);
  b2_release_end(a, rg, old, q, lane, pol);
}

__device__ __forceinline__ double2 b2_ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// d[t][e] (problem g, coordinate 8 t + 2 tig + e of the chunk) = sum_i Ry[i][g] A_J[i][.]
// ry = warp's R_y + g * sa ; b0 = stage + slot(g) * sa.  The K index is a
// summation index, so which rows form a k-step is free: within a 16-row block
// lane tig takes the row pairs at ro = 2 (tig & 1) + 8 (tig >> 1) and ro + 4,
// one LDS.128 per operand for two k-steps (bank-conflict free for a column
// stride == 4 mod 8: a quarter warp's eight 16-byte units are distinct mod
// 8).  Chains: (pair element, coordinate tile) = 4 independent.
template <int MTC>
__device__ __forceinline__ void b2_gemm1(const double* __restrict__ ry, const double* __restrict__ b0, int sa8, int mt_n,
                                         int tig, double (&d)[2][2]) {
  double acc[2][2][2];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int t = 0; t < 2; ++t) acc[u][t][0] = acc[u][t][1] = 0.0;
  const int ro = 2 * (tig & 1) + 8 * (tig >> 1);
  const double* b1 = b0 + sa8;
  auto step2 = [&](int off) {
    const double2 ra = b2_ld2(ry + off), x0 = b2_ld2(b0 + off), x1 = b2_ld2(b1 + off);
    dmma(acc[0][0][0], acc[0][0][1], ra.x, x0.x);
    dmma(acc[0][1][0], acc[0][1][1], ra.x, x1.x);
    dmma(acc[1][0][0], acc[1][0][1], ra.y, x0.y);
    dmma(acc[1][1][0], acc[1][1][1], ra.y, x1.y);
  };
  // the 8 rows an odd row-tile count leaves: two plain k-steps (rows tig and
  // 4 + tig), 8-byte loads (16-byte pairs would conflict 2-way here)
  auto tail = [&](int off) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double ra = ry[off + 4 * h + tig];
      dmma(acc[h][0][0], acc[h][0][1], ra, b0[off + 4 * h + tig]);
      dmma(acc[h][1][0], acc[h][1][1], ra, b1[off + 4 * h + tig]);
    }
  };
  if constexpr (MTC > 0) {
#pragma unroll
    for (int b = 0; b < MTC / 2; ++b) {
      step2(16 * b + ro);
      step2(16 * b + ro + 4);
    }
    if constexpr (MTC & 1) tail(16 * (MTC / 2));
  } else {
    const int nb = mt_n >> 1;
#pragma unroll 2
    for (int b = 0; b < nb; ++b) {
      step2(16 * b + ro);
      step2(16 * b + ro + 4);
    }
    if (mt_n & 1) tail(16 * nb);
  }
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) d[t][e] = acc[0][t][e] + acc[1][t][e];
}

// Row of accumulator tile q held by lane row g.  The M index is free as
// well: row tiles are taken in pairs over 16 rows, lane g holding rows
// 16 q' + 2 g (tile 2 q') and 16 q' + 2 g + 1 (tile 2 q' + 1), so one LDS.128
// feeds two DMMAs; an odd last tile keeps rows 8 q + g.
__device__ __forceinline__ int b2_row(int q, int g, int mt_n) {
  return (q | 1) < mt_n ? 16 * (q >> 1) + 2 * g + (q & 1) : 8 * q + g;
}

// acc (rows b2_row(q, g), problems 2 tig + e) += A_J X_J, K = (tile, parity)
// pairs: k-step (t, e) covers coordinates 8 t + 2 tig + e, whose x values are
// this lane's xn[t][e] (problem g).  st = stage ; so[t][e] = slot * sa.
template <int NQ>
__device__ __forceinline__ void b2_gemm2_n(const double* __restrict__ st, int g, const int (&so)[2][2],
                                           const double (&xn)[2][2], double (&acc)[B2_MT][2]) {
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const double* aj = st + so[t][e];
      const double b = xn[t][e];
#pragma unroll
      for (int p = 0; p < NQ / 2; ++p) {
        const double2 v = b2_ld2(aj + 16 * p + 2 * g);
        dmma(acc[2 * p][0], acc[2 * p][1], v.x, b);
        dmma(acc[2 * p + 1][0], acc[2 * p + 1][1], v.y, b);
      }
      if constexpr (NQ & 1) dmma(acc[NQ - 1][0], acc[NQ - 1][1], aj[8 * (NQ - 1) + g], b);
    }
}
template <int MTC>
__device__ __forceinline__ void b2_gemm2(const double* __restrict__ st, int g, const int (&so)[2][2],
                                         const double (&xn)[2][2], double (&acc)[B2_MT][2], int mt_n) {
  if constexpr (MTC > 0) {
    b2_gemm2_n<MTC>(st, g, so, xn, acc);
    return;
  }
#define B2_CASE(N) \
  case N: b2_gemm2_n<N>(st, g, so, xn, acc); break;
  switch (mt_n) {  // warp-uniform
    B2_CASE(26) B2_CASE(25) B2_CASE(24) B2_CASE(23) B2_CASE(22) B2_CASE(21) B2_CASE(20) B2_CASE(19) B2_CASE(18)
    B2_CASE(17) B2_CASE(16) B2_CASE(15) B2_CASE(14) B2_CASE(13) B2_CASE(12) B2_CASE(11) B2_CASE(10) B2_CASE(9)
    B2_CASE(8) B2_CASE(7) B2_CASE(6) B2_CASE(5) B2_CASE(4) B2_CASE(3) B2_CASE(2) B2_CASE(1)
    default: break;
  }
#undef B2_CASE
}

// warp's R_y tile [8][sa] = R + beta (R - R_prev) (rows >= m zero); Rp may be
// null (beta = 0: the plain residual)
__device__ __forceinline__ void b2_load_ry(const BatchArgs& a, int sa, double* rw0, const double* R, const double* Rp,
                                           int64_t kw, double beta_g, int lane) {
  __syncwarp();
  for (int pp = 0; pp < 8; ++pp) {
    const double bt = Rp ? __shfl_sync(0xffffffffu, beta_g, pp << 2) : 0.0;
    const double* r = R + (kw + pp) * a.ldy;
    for (int i = lane; i < sa; i += 32) {
      double v = 0.0;
      if (i < a.m) {
        v = __ldcg(r + i);
        if (bt != 0.0) v = add_rn(v, mul_rn(bt, sub_rn(v, __ldcg(Rp + (kw + pp) * a.ldy + i))));
      }
      rw0[pp * sa + i] = v;
    }
  }
  __syncwarp();
}

// per-problem sums held in the GEMM2 layout (problems 2 tig + e, partial over
// g) -> the value of problem g in every lane of row g
__device__ __forceinline__ double b2_sum_to_g(double (&sq)[2], int g) {
#pragma unroll
  for (int e = 0; e < 2; ++e)
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) sq[e] += __shfl_xor_sync(0xffffffffu, sq[e], o);
  const double v0 = __shfl_sync(0xffffffffu, sq[0], g >> 1);
  const double v1 = __shfl_sync(0xffffffffu, sq[1], g >> 1);
  return (g & 1) ? v1 : v0;
}

// r = acc - y for this warp's octet into Rw, returns ||r||^2 of problem g
__device__ __forceinline__ double b2_store_r(const BatchArgs& a, const double (&acc)[B2_MT][2], double* Rw, int64_t kw,
                                             int mt_n, int g, int tig) {
  double sq[2] = {0.0, 0.0};
#pragma unroll
  for (int q = 0; q < B2_MT; ++q) {
    const int i = b2_row(q, g, mt_n);
    if (q < mt_n && i < a.m) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t o = (kw + 2 * tig + e) * a.ldy + i;
        const double r = acc[q][e] - a.Y[o];
        Rw[o] = r;
        sq[e] += r * r;
      }
    }
  }
  return b2_sum_to_g(sq, g);
}

// MTC > 0: the row-tile count ceil(m / 8) at compile time (column stride
// 8 MTC + 4, both products fully unrolled); MTC = 0: any m <= 208 at run time
template <int MTC, bool PIPE = true>
__global__ void __launch_bounds__(B2_NT, 1) k_batched_round2(const BatchArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ int dirty_epoch, sweep_epoch;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int sa = MTC ? 8 * MTC + 4 : a.sa2;
  B2Ring rg;
  double* rys;
  {
    double* p = reinterpret_cast<double*>(smem_raw);
    rg.sa = sa;
    rg.sstride = BT_CH * sa;
    rg.stage = p;
    p += (size_t)B2_NST * rg.sstride;
    rys = p;
    p += (size_t)BT_TILE * sa;
    rg.full = reinterpret_cast<uint64_t*>(p);
    rg.cnt = reinterpret_cast<int*>(rg.full + B2_NST);
    rg.it = 0;
  }
  const uint64_t pol = policy_evict_last();
  if (tid == 0) {
    for (int s = 0; s < B2_NST; ++s) {
      mbar_init(&rg.full[s], 1);
      rg.cnt[s] = 0;
    }
    dirty_epoch = 0;
    sweep_epoch = 0;
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (warp == 0)
    for (int q = 0; q < B2_NST; ++q) b2_issue(a, rg, q, lane, pol);

  double* rw0 = rys + (size_t)warp * 8 * sa;           // this warp's residual tile
  const double* rw = rw0 + g * sa;                     // GEMM1 A-fragment base (problem g's residual)
  const int sa8 = 8 * sa;
  const int mt_n = MTC ? MTC : (a.m + 7) / 8;
  const int bo = b2_slot(g) * sa;                      // GEMM1 B-fragment base in a stage (coordinate g's column)
  const int no = sa - 2;                               // row of ||a_j|| in a column slot; a_j't one further
  int so[2][2];                                        // GEMM2 A-fragment offsets
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) so[t][e] = b2_slot(8 * t + 2 * tig + e) * sa;
  int epoch = 0;
  long long dbg_wait = 0, dbg_nlong = 0;
  const long long dbg_t0 = clock64();

  // Work units of this launch: (round, tile) pairs in round-major order, unit
  // u -> round u / ntl of the launch, tile tile0 + u % ntl; CTA b takes units
  // b, b + grid, ...  One round per launch (nrl = 1) is the plain tile loop.
  // With several rounds per launch the CTAs that finish a round's last wave
  // early go on with the next round's first tiles instead of idling (1,563
  // tiles on 148 SMs leave the 11th wave 56% full): a tile's round r + 1 only
  // needs ITS round r, which another CTA finished ~10 waves earlier; each
  // octet publishes its completed rounds in a flag the next round's warp
  // acquires (everything an octet owns is written and later read by the warp
  // of the same index, so the flags are per octet and no CTA barrier is
  // involved), and every load of state another CTA may have written bypasses
  // L1 (ld.global.cg).
  const int ntl = a.tile1 - a.tile0;
  for (int u = blockIdx.x; u < a.nrl * ntl; u += gridDim.x) {
    ++epoch;
    const int rl = u / ntl;
    const int tile = a.tile0 + (u - rl * ntl);
    const int oct = tile * B2_NW + warp;
    if (rl > 0) {
      if (lane == 0)
        while ((int)ld_acquire_gpu_u32(a.oct_round + oct) < a.round0 + rl) {
        }
      __syncwarp();
    }
    const int64_t kw = (int64_t)tile * BT_TILE + warp * 8;   // first problem of the octet
    const int64_t kg = kw + g;                               // the problem of this lane's coordinate pairs
    int par = a.par ^ ((rl * a.passes) & 1);
    double mom = __ldcg(a.mom + kg), P = __ldcg(a.P + kg);
    // ---------------- FISTA steps ----------------
    for (int pass = 0; pass < a.passes; ++pass) {
      const double* X = a.X[par];
      double* Xp = a.X[1 - par];  // read as x_prev, then overwritten by x+
      const double* R = a.R[par];
      double* Rp = a.R[1 - par];
      const double tn = (1.0 + sqrt(1.0 + 4.0 * mom * mom)) / 2.0;
      const double bt = (mom - 1.0) / tn;
      b2_load_ry(a, sa, rw0, R, Rp, kw, bt, lane);
      double acc[B2_MT][2];
#pragma unroll
      for (int q = 0; q < B2_MT; ++q) acc[q][0] = acc[q][1] = 0.0;
      double gdot = 0.0, gsc = 0.0;
      // this lane's slice of the octet's rows of X: problem g, coordinates 8 t + 2 tig + {0, 1} of each chunk
      const double* xg = X + kg * a.ldx + 2 * tig;
      double* xpg = Xp + kg * a.ldx + 2 * tig;
      const uint32_t* mkg = a.mask + kg * a.nw;
      double2 xc[2], xpc[2];
      uint32_t mw;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        xc[t] = __ldcg(reinterpret_cast<const double2*>(xg + 8 * t));
        xpc[t] = __ldcg(reinterpret_cast<const double2*>(xpg + 8 * t));
      }
      mw = __ldcg(mkg);
      // Software pipeline: iteration c runs GEMM1 of chunk c + 1, the update
      // of chunk c and GEMM2 of chunk c as ONE straight block, so the update's
      // fp64 chain and the fragment loads issue between DMMAs of the same
      // warp (a warp alone keeps the DMMA pipe fed; its scheduler partner
      // does not have to be in the right phase).  The last iteration's
      // GEMM1 runs on the next sweep's first chunk and is discarded (the
      // ring cycles through the same chunks for every sweep).
      // (PIPE = false, the A/B control: GEMM1, update and GEMM2 of the same
      // chunk in sequence.)
      const double* st = nullptr;
      double d[2][2];
      if constexpr (PIPE) {
        st = b2_acquire(a, rg);
        b2_gemm1<MTC>(rw, st + bo, sa8, mt_n, tig, d);
      }
      int pend_old = 0, pend_q = -1;
      for (int c = 0; c < a.nch; ++c) {
        const int j0 = c * BT_CH;
        const long long tw0 = a.dbg ? clock64() : 0;
        const double* stn = b2_acquire_at(rg, rg.it + (PIPE ? 1 : 0));
        if (a.dbg) {
          const long long dt = clock64() - tw0;
          dbg_wait += dt;
          dbg_nlong += dt > 200;
        }
        if (pend_q >= 0) b2_release_end(a, rg, pend_old, pend_q, lane, pol);
        double dn[2][2];
        b2_gemm1<MTC>(rw, stn + bo, sa8, mt_n, tig, dn);
        if constexpr (!PIPE) {
          st = stn;
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            d[t][0] = dn[t][0];
            d[t][1] = dn[t][1];
          }
        }
        // the FISTA update of this lane's four coordinates of problem g
        double xn[2][2];
        {
          const uint32_t mb = mw >> (j0 & 31);
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const double nr[2] = {st[so[t][0] + no], st[so[t][1] + no]};
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const bool act = (mb >> (8 * t + 2 * tig + e)) & 1u;
              const double x = e ? xc[t].y : xc[t].x, xp = e ? xpc[t].y : xpc[t].x;
              double yv = x;
              if (bt != 0.0) yv = add_rn(x, mul_rn(bt, sub_rn(x, xp)));
              double v = 0.0;
              if (act) {
                v = sub_rn(yv, mul_rn(a.eta, d[t][e]));
                v = v < 0.0 ? 0.0 : v;
              }
              const double dx = v - x;
              gdot += d[t][e] * dx;
              gsc += nr[e] * fabs(dx);
              xn[t][e] = v;
            }
            // x+ into the x_prev slot (this chunk's x_prev is already in registers)
            *reinterpret_cast<double2*>(xpg + j0 + 8 * t) = make_double2(xn[t][0], xn[t][1]);
          }
        }
        // next chunk's x, x_prev and mask word: in flight during GEMM2 and the next GEMM1
        if (c + 1 < a.nch) {
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            xc[t] = __ldcg(reinterpret_cast<const double2*>(xg + j0 + BT_CH + 8 * t));
            xpc[t] = __ldcg(reinterpret_cast<const double2*>(xpg + j0 + BT_CH + 8 * t));
          }
          mw = __ldcg(mkg + ((j0 + BT_CH) >> 5));
        }
        b2_gemm2<MTC>(st, g, so, xn, acc, mt_n);
        pend_q = rg.it;
        pend_old = b2_release_begin(rg, lane);
        st = stn;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          d[t][0] = dn[t][0];
          d[t][1] = dn[t][1];
        }
      }
      b2_release_end(a, rg, pend_old, pend_q, lane, pol);
      // r+ = A x+ - y into the r_prev slot, objective, restart test
      const double sqg = b2_store_r(a, acc, Rp, kw, mt_n, g, tig);
#pragma unroll
      for (int o = 1; o < 4; o <<= 1) {
        gdot += __shfl_xor_sync(0xffffffffu, gdot, o);
        gsc += __shfl_xor_sync(0xffffffffu, gsc, o);
      }
      const double Pn = 0.5 * sqg;
      const double s_f = a.rs_f * fmax(1.0, fabs(P));
      const double s_g = a.rs_g * sqrt(2.0 * P) * gsc;
      mom = (Pn > P + s_f || gdot > s_g) ? 1.0 : tn;
      P = Pn;
      par ^= 1;
    }
    // ---------------- dual point, gap, sphere test at x ----------------
    {
      double* X = a.X[par];
      double* Xq = a.X[1 - par];
      const double* R = a.R[par];
      b2_load_ry(a, sa, rw0, R, nullptr, kw, 0.0, lane);
      // sweep 1: epsilon_k = max_j (v_jk)+ / |a_j't|, v = -A'r
      double emax = 0.0, vmin = 0.0;
      for (int c = 0; c < a.nch; ++c) {
        const int j0 = c * BT_CH;
        const double* st = b2_acquire(a, rg);
        double d[2][2];
        b2_gemm1<MTC>(rw, st + bo, sa8, mt_n, tig, d);
        double at[2][2];
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int e = 0; e < 2; ++e) at[t][e] = st[so[t][e] + no + 1];
        b2_release(a, rg, lane, pol);
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            emax = fmax(emax, fmax(-d[t][e], 0.0) * (1.0 / fabs(at[t][e])));
            vmin = fmin(vmin, -d[t][e]);
          }
      }
#pragma unroll
      for (int o = 1; o < 4; o <<= 1) {
        emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
        vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
      }
      const double eps = emax;  // of problem g
      // dual objective per problem: theta = -r + eps t (t = -1)
      double thr = 0.0;         // radius + slack of problem g
      double sm_conv = 0.0, sm_max = 0.0, sm_gap = 0.0, sm_pres = 0.0;
      for (int pb = 0; pb < 8; ++pb) {
        const double ep = __shfl_sync(0xffffffffu, eps, pb << 2);
        const double Pp = __shfl_sync(0xffffffffu, P, pb << 2);
        double s1 = 0.0, s2 = 0.0;
        for (int i = lane; i < a.m; i += 32) {
          double th = -rw0[pb * sa + i];
          if (ep > 0.0) th = add_rn(th, mul_rn(ep, -1.0));
          s1 += th * a.Y[(kw + pb) * a.ldy + i];
          s2 += th * th;
        }
        s1 = warp_sum<double>(s1);
        s2 = warp_sum<double>(s2);
        const double D = s1 - 0.5 * s2;
        const double gap = fmax(Pp - D, 0.0);
        if (kw + pb < a.K_user) {
          sm_conv += gap < a.gap_tol ? 1.0 : 0.0;
          sm_max = fmax(sm_max, gap);
          sm_gap += gap;
        }
        if (lane == 0) {
          const int64_t k = kw + pb;
          double* stt = a.stats;
          stt[k] = Pp;
          stt[a.K + k] = D;
          stt[2 * a.K + k] = gap;
          stt[3 * a.K + k] = ep;
        }
        if (g == pb) thr = sqrt(2.0 * gap) + a.slack_scale * fmax(1.0, sqrt(s2));
      }
      // sweep 2: v = -g + eps a't ; screen v < -(radius + slack) ||a_j||.
      // Sweep 1 already bounds the test of a whole problem: every statistic
      // v_j + eps a_j't + thr ||a_j|| is at least
      //     min_j v_j - eps max_j |a_j't| + thr min_j ||a_j||,
      // so when that is positive (with a margin far above the round-off of
      // the per-coordinate expression) no coordinate of the problem can be
      // screened, and when it holds for all 64 problems of the tile the
      // per-coordinate sweep -- a full A'R product -- is skipped.  Exact: a
      // skipped sweep would have screened nothing.
      bool need2 = false;
      if (a.screening) {
        const double lo = vmin - eps * a.att_max + thr * a.nrm_min;
        const bool clear = a.bound_skip && lo > 1e-9 * (fabs(vmin) + eps * a.att_max + thr * a.nrm_min);
        if (!clear) atomicMax(&sweep_epoch, epoch);
        __syncthreads();
        need2 = sweep_epoch == epoch;
        if (need2 && tid == 0 && a.sweeps2) atomicAdd(a.sweeps2, 1ull);
      }
      if (need2) {
        const uint32_t* mkg = a.mask + kg * a.nw;
        for (int c = 0; c < a.nch; ++c) {
          const int j0 = c * BT_CH;
          const double* st = b2_acquire(a, rg);
          double d[2][2];
          b2_gemm1<MTC>(rw, st + bo, sa8, mt_n, tig, d);
          double at[2][2], nr[2][2];
#pragma unroll
          for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              nr[t][e] = st[so[t][e] + no];
              at[t][e] = st[so[t][e] + no + 1];
            }
          b2_release(a, rg, lane, pol);
          const uint32_t mb = __ldcg(mkg + (j0 >> 5)) >> (j0 & 31);
#pragma unroll
          for (int t = 0; t < 2; ++t) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int jj = 8 * t + 2 * tig + e;
              const bool act = (mb >> jj) & 1u;
              const double v = add_rn(-d[t][e], mul_rn(eps, at[t][e]));
              if (act && v < -thr * nr[t][e]) {
                const int j = j0 + jj;
                atomicAnd(&a.mask[kg * a.nw + (j >> 5)], ~(1u << (j & 31)));
                X[kg * a.ldx + j] = 0.0;
                Xq[kg * a.ldx + j] = 0.0;
                atomicMax(&dirty_epoch, epoch);
              }
            }
          }
        }
      }
      // any problem of the tile screened something -> the whole tile refreshes
      // (as the oracle does for the whole batch); second barrier: nobody
      // raises the next tile's epoch before everyone has read this one
      __syncthreads();
      const bool dirty = dirty_epoch == epoch;
      __syncthreads();
      if (dirty) {
        // refresh r = A x - y and r_prev = A x_prev - y (screened x snapped to 0)
        for (int which = 0; which < 2; ++which) {
          const double* Xw = (which ? Xq : X) + kg * a.ldx + 2 * tig;
          double* Rw = a.R[which ? 1 - par : par];
          double acc[B2_MT][2];
#pragma unroll
          for (int q = 0; q < B2_MT; ++q) acc[q][0] = acc[q][1] = 0.0;
          for (int c = 0; c < a.nch; ++c) {
            double xn[2][2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              const double2 v = __ldcg(reinterpret_cast<const double2*>(Xw + c * BT_CH + 8 * t));
              xn[t][0] = v.x;
              xn[t][1] = v.y;
            }
            const double* st = b2_acquire(a, rg);
            b2_gemm2<MTC>(st, g, so, xn, acc, mt_n);
            b2_release(a, rg, lane, pol);
          }
          const double sqg = b2_store_r(a, acc, Rw, kw, mt_n, g, tig);
          if (which == 0) P = 0.5 * sqg;
        }
      }
      // preserved counts
      for (int pb = 0; pb < 8; ++pb) {
        int cnt = 0;
        for (int w = lane; w < a.nw; w += 32) cnt += __popc(__ldcg(a.mask + (kw + pb) * a.nw + w));
        cnt = warp_sum<int>(cnt);
        if (kw + pb < a.K_user) sm_pres += cnt;
        if (lane == 0) a.stats[4 * a.K + kw + pb] = cnt;
      }
      if (tig == 0) {
        a.mom[kg] = mom;
        a.P[kg] = P;
      }
      // this octet's share of the round summary {converged, max gap, sum gap,
      // sum preserved} (problems past K_user are padding), then its flag
      if (lane == 0) {
        double* o = a.osum + ((size_t)((a.round0 + rl) % a.osum_rounds) * (a.K / 8) + oct) * 4;
        o[0] = sm_conv;
        o[1] = sm_max;
        o[2] = sm_gap;
        o[3] = sm_pres;
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        st_release_gpu_u32(a.oct_round + oct, (unsigned)(a.round0 + rl + 1));
      }
    }
  }
  if (a.dbg && lane == 0) {
    unsigned long long* o = a.dbg + (size_t)(blockIdx.x * B2_NW + warp) * 4;
    o[0] = (unsigned long long)dbg_wait;
    o[1] = (unsigned long long)dbg_nlong;
    o[2] = (unsigned long long)(clock64() - dbg_t0);
    o[3] = (unsigned long long)rg.it;
  }
  // the ring always runs NST chunks ahead: wait for the copies still in flight
  for (int q = 0; q < B2_NST; ++q) {
    const int s = (rg.it + q) % B2_NST;
    mbar_wait(&rg.full[s], (uint32_t)(((rg.it + q) / B2_NST) & 1));
  }
}

// Round summary from the per-octet partials, fixed order (one block):
// out = {converged problems, max gap, sum gap, sum preserved}
__global__ void k_b2_summary(const double* __restrict__ osum, int noct, double* __restrict__ out) {
  __shared__ double sh[4][32];
  double c = 0.0, mx = 0.0, sg = 0.0, sp = 0.0;
  for (int o = threadIdx.x; o < noct; o += blockDim.x) {
    c += osum[4 * o + 0];
    mx = fmax(mx, osum[4 * o + 1]);
    sg += osum[4 * o + 2];
    sp += osum[4 * o + 3];
  }
  c = warp_sum<double>(c);
  sg = warp_sum<double>(sg);
  sp = warp_sum<double>(sp);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sh[0][warp] = c;
    sh[1][warp] = mx;
    sh[2][warp] = sg;
    sh[3][warp] = sp;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a0 += sh[0][w];
      a1 = fmax(a1, sh[1][w]);
      a2 += sh[2][w];
      a3 += sh[3][w];
    }
    out[0] = a0;
    out[1] = a1;
    out[2] = a2;
    out[3] = a3;
  }
}

// The dictionary as the ring wants it: chunk c is one contiguous block
// [16 slots][sa]; slot b2_slot(cc) holds column 16 c + cc (rows >= m zero),
// with ||a_j|| and a_j't in the slot's last two rows (never read by the
// products: they stop at row m8 <= sa - 4).  Columns past n: zero, norm 0,
// a_j't = 1 (never active, never the dual scaling's maximiser).
__global__ void k_b2_pack(const double* __restrict__ A, int64_t lda, int m, int n, const double* __restrict__ nrm,
                          const double* __restrict__ att, double* __restrict__ Ap, int sa, int nch) {
  const int64_t tot = (int64_t)nch * BT_CH * sa;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < tot; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = q / sa;
    const int row = (int)(q - col * sa);
    const int c = (int)(col / BT_CH), p = (int)(col % BT_CH);
    int cc = 0;
    for (int u = 0; u < BT_CH; ++u)
      if (b2_slot(u) == p) cc = u;
    const int64_t j = (int64_t)c * BT_CH + cc;
    double v = 0.0;
    if (row < m)
      v = j < n ? A[j * lda + row] : 0.0;
    else if (row == sa - 2)
      v = j < n ? nrm[j] : 0.0;
    else if (row == sa - 1)
      v = j < n ? att[j] : 1.0;
    Ap[q] = v;
  }
}

}  // namespace bx
