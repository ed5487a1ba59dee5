// bx_cd.cuh -- cyclic coordinate descent (reference solvers.py:119-137) on one
// thread-block cluster.
//
// The reference sweeps the preserved columns in original-index order; for each
// column k: step = a_k'r / ||a_k||^2, x_k' = clip(x_k - step, l_k, u_k),
// r += (x_k' - x_k) a_k when the move is nonzero.  Sequential in k, so the GPU
// version is "block-exact": the columns are cut into blocks J of B <= 32
// consecutive preserved columns and, per block,
//    d_J   = A_J' r                   (parallel dots, split over the cluster)
//    for i in J (in order):  c_i = d_i + sum_{l<i, l in J} G_il delta_l
//                            step = c_i / ||a_i||^2 ; x_i' = clip(...) ; delta_i
//    r    += A_J delta_J              (parallel axpy)
// with the Gram blocks G_JJ = A_J'A_J precomputed (k_gram).  In exact
// arithmetic this is the reference's sweep step for step; only the rounding
// of a_i'r differs (a block dot + Gram corrections instead of a fresh dot).
//
// Layout: a cluster of NC CTAs splits the m rows; each CTA keeps its rows of r
// in registers and its rows of A_J in shared memory (double buffered,
// prefetched with cp.async while the previous block's update runs).  The B
// partial dots of every CTA are combined through distributed shared memory in
// rank order (deterministic), then every CTA runs the (tiny) sequential update
// redundantly, so one cluster barrier per block is the only synchronisation.
#pragma once
#include <cooperative_groups.h>

#include "bx_kernels.cuh"

namespace bx {

namespace cg = cooperative_groups;

constexpr int CD_NT = 256;   // threads per CTA
constexpr int CD_B = 32;     // columns per block (one warp lane each)
constexpr int CD_RMAX = 4;   // rows per thread held in registers (m <= NC*CD_NT*CD_RMAX)

template <typename T>
struct CdArgs {
  const T* A;        // compacted preserved columns, column stride ld
  int64_t ld;
  int64_t m;
  int64_t k;         // preserved columns
  double* x;         // preserved iterate, read in even passes
  double* x2;        // written in even passes, read in odd (ping-pong: every
                     // CTA reads x_j while rank 0 publishes the new value)
  const double* lo;
  const double* hi;
  const double* nrm; // ||a_j||  (sq = nrm^2, as solvers.py:60)
  const double* gram;  // [nblocks][B][B] Gram blocks (fp64)
  double* r;         // residual (in/out, m)
  DevScalars* sc;
  int passes;
  int rows_per_cta;  // multiple of 2
};

// cp.async 16-byte global->shared copy (LDGSTS)
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// per-column state of a block (x of the pass, lo, hi, ||a_j||): thread
// f * CD_B + c loads field f of column c through L2 when the block is
// prefetched and parks it in shared memory after the current block's axpy,
// so the sequential update never waits on global memory.  x of pass p was
// written by rank 0 in pass p - 1, several cluster barriers earlier.
constexpr int CD_ST = 4;
// field 3 is stashed as 1 / ||a_j||^2 (col_norms ** 2, solvers.py:60), so the
// division is off the sequential update's critical path; zero-padded
// columns past k stash 1 (never used)
__device__ __forceinline__ double cd_isq(double nj) { return nj == 0.0 ? 1.0 : 1.0 / (nj * nj); }
template <typename T>
__device__ __forceinline__ double cd_state_load(const CdArgs<T>& a, int64_t blk, int pass) {
  const int f = threadIdx.x / CD_B, c = threadIdx.x % CD_B;
  const int64_t j = blk * CD_B + c;
  if (f >= CD_ST || j >= a.k) return 0.0;
  const double* src = f == 0 ? ((pass & 1) ? a.x2 : a.x) : (f == 1 ? a.lo : (f == 2 ? a.hi : a.nrm));
  return __ldcg(src + j);
}

template <typename T>
__device__ __forceinline__ void cd_prefetch(const CdArgs<T>& a, T* dst, double* gdst, int64_t blk, int64_t row0,
                                            int nrows) {
  // the block's 32 x 32 Gram matrix (fp64) rides along
  for (int q = threadIdx.x; q < CD_B * CD_B / 2; q += CD_NT) cp_async16(gdst + 2 * q, a.gram + blk * CD_B * CD_B + 2 * q);
  const int64_t c0 = blk * CD_B;
  const int nc = (int)min((int64_t)CD_B, a.k - c0);
  // dst[c * rows_pad + i] = A[row0 + i, 32*blk + c]; (column, vector) of
  // piece q advanced incrementally (no integer division per piece)
  constexpr int V = 16 / sizeof(T);
  const int nvec = (nrows + V - 1) / V;  // rows_per_cta is a multiple of V
  if (nvec > 0) {
    const int rows_pad = a.rows_per_cta;
    const int dc = CD_NT / nvec, dv = CD_NT - dc * nvec;
    int c = threadIdx.x / nvec, v = threadIdx.x - c * nvec;
    const T* src = a.A + c0 * a.ld + row0;
    while (c < nc) {
      cp_async16(dst + (int64_t)c * rows_pad + v * V, src + c * a.ld + v * V);
      c += dc;
      v += dv;
      if (v >= nvec) {
        v -= nvec;
        ++c;
      }
    }
  }
  cp_async_commit();
}

template <typename T>
__global__ void __launch_bounds__(CD_NT, 1) k_cd(const CdArgs<T> a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int NC = (int)cluster.num_blocks();
  extern __shared__ __align__(1024) unsigned char smem[];
  const int rows_pad = a.rows_per_cta;
  T* abuf0 = reinterpret_cast<T*>(smem);
  T* abuf1 = abuf0 + CD_B * rows_pad;
  double* part = reinterpret_cast<double*>(abuf1 + CD_B * rows_pad);  // [2][CD_B] partial dots
  double* gbuf = part + 2 * CD_B;                                       // [2][CD_B][CD_B] Gram blocks
  double* delta = gbuf + 2 * CD_B * CD_B;                               // [CD_B]
  double* allpart = delta + CD_B;                                        // [2][NC][CD_B] pushed partial dots
  double* cst = allpart + 2 * 16 * CD_B;                                 // [2][CD_ST][CD_B] column state
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t row0 = (int64_t)rank * rows_pad;
  const int nrows = (int)max((int64_t)0, min((int64_t)rows_pad, a.m - row0));

  // residual rows in registers: thread owns rows tid + q*CD_NT
  double rr[CD_RMAX];
#pragma unroll
  for (int q = 0; q < CD_RMAX; ++q) {
    const int i = tid + q * CD_NT;
    rr[q] = (i < nrows) ? a.r[row0 + i] : 0.0;
  }
  const int64_t nblk = (a.k + CD_B - 1) / CD_B;
  int64_t it = 0;  // global block counter (selects buffers)
  double pfv = 0.0;  // per-column state of the prefetched block (threads < CD_ST * CD_B)
  if (nblk > 0) {
    cd_prefetch(a, abuf0, gbuf, 0, row0, nrows);
    if (tid < CD_ST * CD_B) {
      const double v = cd_state_load(a, 0, 0);
      cst[tid] = tid >= 3 * CD_B ? cd_isq(v) : v;
    }
  }
  for (int pass = 0; pass < a.passes; ++pass) {
    for (int64_t blk = 0; blk < nblk; ++blk, ++it) {
      T* cur = (it & 1) ? abuf1 : abuf0;
      T* nxt = (it & 1) ? abuf0 : abuf1;
      const int64_t c0 = blk * CD_B;
      const int nc = (int)min((int64_t)CD_B, a.k - c0);
      cp_async_wait_all();
      const double* gcur = gbuf + (it & 1) * CD_B * CD_B;
      __syncthreads();
      // prefetch the next block while this one is processed
      {
        int64_t nb = blk + 1, np = pass;
        if (nb == nblk) {
          nb = 0;
          ++np;
        }
        if (np < a.passes) {
          cd_prefetch(a, nxt, gbuf + ((it + 1) & 1) * CD_B * CD_B, nb, row0, nrows);
          pfv = cd_state_load(a, nb, (int)np);
        }
      }
      // partial dots: every thread multiplies its register rows with the block's
      // columns; a butterfly transpose-reduction leaves column c's warp sum in
      // lane c (31 shuffles instead of 32 x 5)
      double* mypart = part + (it & 1) * CD_B;
      {
        double pd[CD_B];
#pragma unroll
        for (int c = 0; c < CD_B; ++c) pd[c] = 0.0;
#pragma unroll
        for (int q = 0; q < CD_RMAX; ++q) {
          const int i = tid + q * CD_NT;
          if (i < nrows) {
            const double rv = rr[q];
#pragma unroll
            for (int c = 0; c < CD_B; ++c)
              if (c < nc) pd[c] += static_cast<double>(cur[(int64_t)c * rows_pad + i]) * rv;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const bool upper = (lane & o) != 0;
#pragma unroll
          for (int q = 0; q < o; ++q) {
            const double send = upper ? pd[q] : pd[q + o];
            const double keep = upper ? pd[q + o] : pd[q];
            pd[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
        __shared__ double wpart[CD_NT / 32][CD_B];
        wpart[warp][lane] = pd[0];
        __syncthreads();
        // push this CTA's partials into every CTA's slot [rank] (remote
        // stores, made visible by the cluster barrier): the combine below
        // then reads local shared memory only
        double* slot = allpart + (it & 1) * 16 * CD_B + rank * CD_B;
        if (tid < CD_B) {
          double s = 0.0;
          for (int w = 0; w < CD_NT / 32; ++w) s += wpart[w][tid];
          mypart[tid] = s;
          for (int q = 0; q < NC; ++q) cluster.map_shared_rank(slot, q)[tid] = s;
        }
      }
      cluster.sync();  // every CTA's partial dots are visible
      // combine partial dots of all CTAs in rank order, then the sequential
      // block update on warp 0 (lane = column), redundantly in every CTA
      if (warp == 0) {
        double cdot = 0.0;
        if (lane < nc) {
          const double* ap = allpart + (it & 1) * 16 * CD_B + lane;
          for (int q = 0; q < NC; ++q) cdot += ap[q * CD_B];
        }
        const int64_t j = c0 + lane;
        double* xout = (pass & 1) ? a.x : a.x2;
        const double* cs = cst + (it & 1) * CD_ST * CD_B;
        double xj = 0.0, loj = 0.0, hij = 0.0;
        double sq = 1.0;
        if (lane < nc) {
          xj = cs[lane];
          loj = cs[CD_B + lane];
          hij = cs[2 * CD_B + lane];
          sq = cs[3 * CD_B + lane];  // 1 / ||a_j||^2, stashed with the column state
        }
        // Gram row of this lane's coordinate in registers; the chain per
        // coordinate is then multiply, clip, subtract, one shuffle and one FMA
        double grow[CD_B];
#pragma unroll
        for (int i = 0; i < CD_B; ++i) grow[i] = gcur[lane * CD_B + i];
        const double isq = sq;
        double dl = 0.0;
#pragma unroll
        for (int i = 0; i < CD_B; ++i) {
          if (i < nc) {
            // every lane evaluates its tentative coordinate step (no
            // divergence); only lane i's -- whose dot now carries the
            // corrections of all earlier coordinates -- is broadcast and kept
            // x - (a.r)/||a||^2 as one fused multiply-add (solvers.py:131-132)
            double nv = fma(-cdot, isq, xj);
            nv = nv < loj ? loj : nv;
            nv = nv > hij ? hij : nv;
            const double dt = nv - xj;                                 // solvers.py:133
            const double di = __shfl_sync(0xffffffffu, dt, i);
            const bool me = lane == i;
            xj = (me && dt != 0.0) ? nv : xj;
            dl = me ? dt : dl;
            cdot = fma(grow[i], di, cdot);  // lanes <= i are finished; di == 0 leaves cdot unchanged
          }
        }
        delta[lane] = dl;
        if (lane < nc && rank == 0) xout[j] = xj;
        // one block per pass: the next block's x is this block's output,
        // which every CTA has just computed redundantly
        if (nblk == 1) cst[((it + 1) & 1) * CD_ST * CD_B + lane] = xj;
      }
      __syncthreads();
      // r += A_J delta_J on this CTA's rows
#pragma unroll
      for (int q = 0; q < CD_RMAX; ++q) {
        const int i = tid + q * CD_NT;
        if (i < nrows) {
          double acc = rr[q];
          for (int c = 0; c < nc; ++c) {
            const double dc = delta[c];
            if (dc != 0.0) acc += static_cast<double>(cur[(int64_t)c * rows_pad + i]) * dc;
          }
          rr[q] = acc;
        }
      }
      // the next block's column state (its buffer was last read by warp 0
      // two blocks ago)
      if (tid < CD_ST * CD_B && (nblk > 1 || tid >= CD_B))
        cst[((it + 1) & 1) * CD_ST * CD_B + tid] = tid >= 3 * CD_B ? cd_isq(pfv) : pfv;
      __syncthreads();
    }
  }
  // write back the residual rows and the objective 0.5 ||r||^2
  double sq = 0.0;
#pragma unroll
  for (int q = 0; q < CD_RMAX; ++q) {
    const int i = tid + q * CD_NT;
    if (i < nrows) {
      a.r[row0 + i] = rr[q];
      sq += rr[q] * rr[q];
    }
  }
  sq = warp_sum<double>(sq);
  __shared__ double wsq[CD_NT / 32];
  if (lane == 0) wsq[warp] = sq;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < CD_NT / 32; ++w) s += wsq[w];
    part[0] = s;
  }
  cluster.sync();
  if (rank == 0 && tid == 0) {
    double tot = 0.0;
    for (int q = 0; q < NC; ++q) tot += *cluster.map_shared_rank(part, q);
    a.sc->P = 0.5 * tot;
  }
  cluster.sync();  // keep smem alive until rank 0 has read it
}

// Gram blocks G_JJ = A_J' A_J for consecutive blocks of CD_B preserved columns
template <typename T>
__global__ void __launch_bounds__(256) k_gram(const T* __restrict__ A, int64_t ld, int64_t m, int64_t k,
                                              double* __restrict__ gram) {
  __shared__ T tile[CD_B][129];  // 128-row chunk of the block's columns (+1 pad)
  const int64_t blk = blockIdx.x;
  const int64_t c0 = blk * CD_B;
  const int nc = (int)min((int64_t)CD_B, k - c0);
  // thread -> 4 (i, l) pairs of the 32x32 block
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t r0 = 0; r0 < m; r0 += 128) {
    const int nr = (int)min((int64_t)128, m - r0);
    __syncthreads();
    for (int q = threadIdx.x; q < CD_B * 128; q += 256) {
      const int c = q / 128, i = q % 128;
      tile[c][i] = (c < nc && i < nr) ? A[(c0 + c) * ld + r0 + i] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = threadIdx.x * 4 + u;
      const int i = p / CD_B, l = p % CD_B;
      double s = 0.0;
      for (int rr = 0; rr < nr; ++rr) s += static_cast<double>(tile[i][rr]) * static_cast<double>(tile[l][rr]);
      acc[u] += s;
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int p = threadIdx.x * 4 + u;
    gram[blk * CD_B * CD_B + p] = acc[u];
  }
}

}  // namespace bx
