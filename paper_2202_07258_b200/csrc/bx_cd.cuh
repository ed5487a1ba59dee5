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
  const double* gram;  // [nblocks][2][B][B]: G_JJ = A_J'A_J and X_J = A_next(J)'A_J (fp64)
  double* r;         // residual (in/out, m)
  DevScalars* sc;
  int passes;
  int rows_per_cta;  // multiple of 2
  int slots;         // shared-memory block slots (the kernel's NS): 3, or 2 for large m
  unsigned long long* dbg;  // BX_CD_DEBUG: per-phase clock sums of rank 0's warp 0 (null otherwise)
};

// cp.async 16-byte global->shared copy (LDGSTS)
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// per-column state of a block (x of the pass, lo, hi, ||a_j||): thread
// f * CD_B + c loads field f of column c through L2 one block ahead and parks
// it in shared memory at the end of the current block, so the sequential
// update never waits on global memory.  x of pass p was written by rank 0 in
// pass p - 1, several cluster barriers earlier.
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

// rows of a CTA are owned by warps 1..7 (warp 0 runs the sequential update):
// thread t >= 32 owns rows (t - 32) + q * CD_RT
constexpr int CD_RT = CD_NT - 32;

// Block `blk` of this CTA's rows (32 columns) plus its Gram pair into a slot:
// one cp.async.bulk per column and one for the 16 KB Gram pair, completing on
// the slot's mbarrier.  (The per-thread cp.async version cost every thread
// ~1,600 clocks of address arithmetic and issue per block, on the critical
// path of the sequential update and of the row warps alike.)  A bulk copy
// takes uniform operands, so a warp issues its lanes' copies one after the
// other (~40 clocks each): the columns are dealt round robin to the NW warps
// that call this (part = 0 .. NW-1; part 0 also arms the barrier and copies
// the Gram pair) -- issued by one warp, the 33 copies held that warp, and
// with it the row warps' named barrier, for ~1,600 clocks per block.
template <typename T>
__device__ __forceinline__ void cd_prefetch(const CdArgs<T>& a, T* dst, double* gdst, int64_t blk, int64_t row0,
                                            int nrows, uint64_t* bar, uint64_t pol, int part, int NW) {
  const int lane = threadIdx.x & 31;
  constexpr int V = 16 / sizeof(T);
  const int64_t c0 = blk * CD_B;
  const int nc = (int)min((int64_t)CD_B, a.k - c0);
  const uint32_t colbytes = (uint32_t)(((nrows + V - 1) / V) * 16);  // rows_per_cta is a multiple of V
  const uint32_t gbytes = 2 * CD_B * CD_B * 8;
  fence_proxy_async_smem();  // the slot's previous readers (generic proxy) come first
  if (part == 0) {
    // the tx-count may run negative until this arrives: completions of the
    // other warps' copies can come first
    if (lane == 0) {
      mbar_expect_tx(bar, gbytes + (uint32_t)nc * colbytes);
      bulk_g2s(gdst, a.gram + blk * 2 * CD_B * CD_B, gbytes, bar, pol);
    }
  }
  const int c = part + NW * lane;
  if (c < nc && colbytes > 0)
    bulk_g2s(dst + (int64_t)c * a.rows_per_cta, a.A + (c0 + c) * a.ld + row0, colbytes, bar, pol);
  // a last, partial block: its unused column slots read as zero columns, so
  // the dots and the axpy need no per-column guard (a guard turns each of
  // their 32 columns into a branch plus a dependent load: ~100 clocks each)
  if (c >= nc && c < CD_B)
    for (int i = 0; i < a.rows_per_cta; ++i) dst[(int64_t)c * a.rows_per_cta + i] = T(0);
}

__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// Software-pipelined block-exact CD: while warp 0 runs block J's sequential
// update, warps 1..7 compute block J+1's partial dots against the residual
// that still lacks block J's move, and push them to every CTA of the
// cluster; warp 0 then adds the missing term with the cross-Gram block
//     d_{J+1} = A_{J+1}'(r + A_J delta_J) = A_{J+1}'r + X_J delta_J,
// (exact arithmetic identity) before r += A_J delta_J.  Three shared-memory
// slots: block J (axpy), J+1 (dots), J+2 (in flight).
// RQ: row slots per row thread actually held (rows_per_cta <= RQ * CD_RT): 1
// for m <= 224 rows per CTA.  The loop body is straight-line code that every
// warp runs once per block, so its size is paid in instruction fetches: the
// fourfold unrolling for the 4-slot envelope cost ~10 clocks per instruction
// in the row warps' dots and axpy.
template <typename T, int NS, int RQ>
__global__ void __launch_bounds__(CD_NT, 1) k_cd(const CdArgs<T> a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int NC = (int)cluster.num_blocks();
  extern __shared__ __align__(1024) unsigned char smem[];
  const int rows_pad = a.rows_per_cta;
  T* abuf = reinterpret_cast<T*>(smem);                                      // [3][CD_B][rows_pad]
  double* gbuf = reinterpret_cast<double*>(abuf + NS * CD_B * rows_pad);    // [NS][2][CD_B][CD_B]
  double* part = gbuf + NS * 2 * CD_B * CD_B;                               // [2] scratch
  double* delta = part + 2;                                                 // [2][CD_B] steps of block it in delta[it & 1]
  double* allpart = delta + 2 * CD_B;                                           // [2][16][CD_B] pushed partial dots
  double* cst = allpart + 2 * 16 * CD_B;                                    // [3][CD_ST][CD_B] column state
  __shared__ double wpart[CD_NT / 32][CD_B];
  __shared__ uint64_t fullb[3];  // per slot: the block's bulk copies have landed
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NRW = CD_NT / 32 - 1;  // row warps (1 .. NRW); they share the issue of the block copies
  // Three slots: the axpy of block it runs at the start of iteration it + 1 in
  // the row warps, overlapped with warp 0's sequential update of block it + 1
  // (it was ~2,300 clocks per block with warp 0 idle); the slot it frees then
  // takes block it + 3.  Two slots (tall m): the axpy stays in its iteration.
  constexpr bool DEFER = NS == 3;
  const uint64_t pol = policy_evict_last();  // A and the Gram blocks are re-read every sweep: keep them in L2
  if (tid == 0) {
    for (int q = 0; q < 3; ++q) mbar_init(&fullb[q], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // block b lands in slot b % NS; its barrier phase is (b / NS) & 1
  auto wait_block = [&](int64_t b) { mbar_wait(&fullb[(int)b % NS], (uint32_t)(((int)b / NS) & 1)); };
  const int64_t row0 = (int64_t)rank * rows_pad;
  const int nrows = (int)max((int64_t)0, min((int64_t)rows_pad, a.m - row0));
  const int rt = tid - 32;  // row thread index (warps 1..7)

  // residual rows in registers (warps 1..7)
  double rr[RQ];
#pragma unroll
  for (int q = 0; q < RQ; ++q) {
    const int i = rt + q * CD_RT;
    rr[q] = (rt >= 0 && i < nrows) ? a.r[row0 + i] : 0.0;
  }
  // rank slots past the cluster size are never pushed to: they read as zeros
  // in combine() (nobody else writes them, so no ordering with the pushes)
  for (int q = NC * CD_B + tid; q < 16 * CD_B; q += CD_NT) {
    allpart[q] = 0.0;
    allpart[16 * CD_B + q] = 0.0;
  }
  const int64_t nblk = (a.k + CD_B - 1) / CD_B;
  const int64_t total = nblk * a.passes;  // blocks over all passes, in order
  // slot of a block (constant divisors: no integer division sequence)
  auto sidx = [&](int64_t it) { return (int)it % NS; };
  auto slot_a = [&](int64_t it) { return abuf + sidx(it) * CD_B * rows_pad; };
  auto slot_g = [&](int64_t it) { return gbuf + sidx(it) * 2 * CD_B * CD_B; };
  // 32-bit block / pass of a global block index (nblk <= 2^26 columns / 32)
  const int nb32 = (int)nblk;
  auto blk_of = [&](int64_t it) { return (int64_t)((int)it % nb32); };
  auto pass_of = [&](int64_t it) { return (int)it / nb32; };

  // partial dots of block `it` over this CTA's rows -> pushed into slot
  // parity(it) of every CTA (warps 1..7; named barrier 1 among them)
  long long trw[6] = {0, 0, 0, 0, 0, 0};
  const bool timed_r = a.dbg && rank == 0 && tid == 32;
  auto dots_push = [&](int64_t it) {
    const long long r0 = timed_r ? clock64() : 0;
    const T* cur = slot_a(it);
    double pd[CD_B];
#pragma unroll
    for (int c = 0; c < CD_B; ++c) pd[c] = 0.0;
#pragma unroll
    for (int q = 0; q < RQ; ++q) {
      const int i = rt + q * CD_RT;
      if (i < nrows) {
        const double rv = rr[q];
        const T* colp = cur + i;
#pragma unroll
        for (int c = 0; c < CD_B; ++c) pd[c] += static_cast<double>(colp[c * rows_pad]) * rv;
      }
    }
    const long long r1 = timed_r ? clock64() : 0;
    // butterfly transpose-reduction: column c's warp sum lands in lane c
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
    wpart[warp][lane] = pd[0];
    const long long r2 = timed_r ? clock64() : 0;
    asm volatile("bar.sync 1, %0;" ::"r"(CD_RT) : "memory");
    const long long r3 = timed_r ? clock64() : 0;
    if (warp == 1) {
      double s = 0.0;
      for (int w = 1; w < CD_NT / 32; ++w) s += wpart[w][lane];
      double* slot = allpart + (it & 1) * 16 * CD_B + rank * CD_B;
      for (int q = 0; q < NC; ++q) cluster.map_shared_rank(slot, q)[lane] = s;
    }
    if (timed_r) {
      const long long r4 = clock64();
      trw[0] += r1 - r0;  // partial dots (FMAs)
      trw[1] += r2 - r1;  // butterfly
      trw[2] += r3 - r2;  // named barrier
      trw[3] += r4 - r3;  // combine + remote stores
    }
  };
  // r += A_b delta_b on this CTA's rows (row warps)
  auto axpy = [&](int64_t b) {
    const T* cur = slot_a(b);
    const double* dl_b = delta + (b & 1) * CD_B;
#pragma unroll
    for (int q = 0; q < RQ; ++q) {
      const int i = rt + q * CD_RT;
      if (i < nrows) {
        // four independent chains over the block's columns (c mod 4),
        // combined in a fixed order; a zero step adds an exact zero
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const T* colp = cur + i;
#pragma unroll
        for (int c = 0; c < CD_B; ++c) acc[c & 3] += static_cast<double>(colp[c * rows_pad]) * dl_b[c];
        rr[q] += (acc[0] + acc[1]) + (acc[2] + acc[3]);
      }
    }
  };
  // warp 0: combine the pushed partials of block `it` in rank order
  auto combine = [&](int64_t it) {
    // all 16 rank slots (slots past NC hold zeros), four chains (rank mod 4)
    // combined in a fixed order
    const double* ap = allpart + (it & 1) * 16 * CD_B + lane;
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < 16; ++q) s4[q & 3] += ap[q * CD_B];
    return (s4[0] + s4[1]) + (s4[2] + s4[3]);
  };

  double pfv = 0.0;   // column state of the block after next (threads < CD_ST * CD_B)
  double cdot = 0.0;  // warp 0: the current block's dot, lane = column
  if (total > 0) {
    // prologue: blocks 0 and 1 in flight, block 0's column state, block 0's dots
    if (warp > 0) {
      cd_prefetch(a, slot_a(0), slot_g(0), blk_of(0), row0, nrows, &fullb[0], pol, warp - 1, NRW);
      if (total > 1) cd_prefetch(a, slot_a(1), slot_g(1), blk_of(1), row0, nrows, &fullb[1 % NS], pol, warp - 1, NRW);
    }
    if (tid < CD_ST * CD_B) {
      const double v = cd_state_load(a, blk_of(0), pass_of(0));
      cst[tid] = tid >= 3 * CD_B ? cd_isq(v) : v;
      if (total > 1) {
        const double w = cd_state_load(a, blk_of(1), pass_of(1));
        cst[CD_ST * CD_B + tid] = tid >= 3 * CD_B ? cd_isq(w) : w;
      }
    }
    wait_block(0);
    __syncthreads();
    if (warp == 0) {
      cluster_arrive_relaxed();
    } else {
      dots_push(0);
      cluster_arrive_release();
    }
    cluster_wait();
    if (warp == 0) cdot = combine(0);
  }
  long long tph[6] = {0, 0, 0, 0, 0, 0};
  long long tph7 = 0;
  long long tch[3] = {0, 0, 0};
  const bool timed = a.dbg && rank == 0 && tid == 0;
  // (block, pass) of iteration it and of it + 2, advanced incrementally (an
  // integer division per use was ~300 clocks of warp 0's path per block)
  int blk_c = 0, pass_c = 0;
  int blk_2 = (int)blk_of(2), pass_2 = pass_of(2);
  for (int64_t it = 0; it < total; ++it) {
    const long long tq0 = timed ? clock64() : 0;
    const int64_t blk = blk_c;
    const int pass = pass_c;
    const int64_t c0 = blk * CD_B;
    const int nc = (int)min((int64_t)CD_B, a.k - c0);
    const bool has_next = it + 1 < total;
    // block it+1's data (issued one iteration ago) must have landed
    if (has_next) wait_block(it + 1);
    __syncthreads();
    const long long tq1 = timed ? clock64() : 0;
    if (it + 2 < total) {
      // three slots: block it+2 goes into the slot block it-1 freed; two
      // slots: it must wait for block it's axpy (end of this iteration)
      pfv = cd_state_load(a, blk_2, pass_2);
    }
    const long long tq1a = timed ? clock64() : 0;
    if (warp == 0) {
      cluster_arrive_relaxed();  // warp 0 publishes nothing this phase
      const long long tc0 = timed ? clock64() : 0;
      // ---- sequential block update (lane = column), redundantly per CTA ----
      const int64_t j = c0 + lane;
      double* xout = (pass & 1) ? a.x : a.x2;
      const double* cs = cst + (it % 3) * CD_ST * CD_B;
      // lane = column: each lane keeps its own dot current.  Straight-line,
      // no guard for the columns past nc of a last, partial block: their
      // state is (x, lo, hi, 1/||a||^2) = (0, 0, 0, 1) and their dots and
      // Gram entries are zero, so their step is an exact zero.  (Measured in
      // isolation, scripts/probes/cdchain2_probe.cu: 105 clocks per step this
      // way, 172 as a rolled loop -- its counter lives in the uniform
      // datapath -- and 190 with a per-step branch on nc.)
      double xj = 0.0, loj = 0.0, hij = 0.0, isq = 1.0;
      if (lane < nc) {
        xj = cs[lane];
        loj = cs[CD_B + lane];
        hij = cs[2 * CD_B + lane];
        isq = cs[3 * CD_B + lane];  // 1 / ||a_j||^2
      }
      // G[.][lane]: the block Gram matrix is bitwise symmetric (k_gram), and
      // reading row i across the lanes is bank-conflict free (G[lane][i] is a
      // 32-way conflict: a 256-byte lane stride)
      const double* gcol = slot_g(it) + lane;
      double dl = 0.0;
      const long long tc1 = timed ? clock64() : 0;
#pragma unroll
      for (int i = 0; i < CD_B; ++i) {
        // every lane evaluates its tentative coordinate step (no
        // divergence); only lane i's -- whose dot now carries the
        // corrections of all earlier coordinates -- is broadcast and kept
        double nv = fma(-cdot, isq, xj);  // x - (a.r)/||a||^2 (solvers.py:131-132)
        nv = nv < loj ? loj : nv;
        nv = nv > hij ? hij : nv;
        const double dt = nv - xj;  // solvers.py:133
        const double di = __shfl_sync(0xffffffffu, dt, i);
        const bool me = lane == i;
        xj = (me && dt != 0.0) ? nv : xj;
        dl = me ? dt : dl;
        cdot = fma(gcol[i * CD_B], di, cdot);  // lanes <= i are finished; di == 0 leaves cdot unchanged
      }
      if (timed) {
        const long long tc2 = clock64();
        tch[1] += tc1 - tc0;   // state / first Gram entry from shared memory
        tch[2] += tc2 - tc1;   // the 32 dependent steps
      }
      delta[(it & 1) * CD_B + lane] = dl;
      if (lane < nc && rank == 0) xout[j] = xj;
      // short passes (<= 3 blocks): the x this block produces is read again
      // within the state look-ahead; every CTA computed it redundantly, so
      // it goes straight into the slot of block it + nblk
      if (nblk <= 3 && it + nblk < total) cst[((it + nblk) % 3) * CD_ST * CD_B + lane] = xj;
    } else {
      // ---- block it+1's partial dots against r without delta_it ----
      if constexpr (DEFER) {
        if (it > 0) axpy(it - 1);
      }
      if (has_next) dots_push(it + 1);
      const long long r5 = timed_r ? clock64() : 0;
      cluster_arrive_release();
      if (timed_r) trw[4] += clock64() - r5;  // arrive.release
      if constexpr (DEFER) {
        // Block it+2 goes into the slot block it-1's axpy has just left (the
        // named barrier of dots_push came after every row warp's axpy; the
        // last block has no dots: its own barrier).  Issued between the
        // cluster barrier's arrive and wait: the other CTAs do not wait for
        // it, and the copy still has the rest of the iteration to land.
        if (!has_next) asm volatile("bar.sync 1, %0;" ::"r"(CD_RT) : "memory");
        if (it + 2 < total)
          cd_prefetch(a, slot_a(it + 2), slot_g(it + 2), blk_2, row0, nrows, &fullb[(int)(it + 2) % NS], pol,
                      warp - 1, NRW);
      }
    }
    const long long tq2 = timed ? clock64() : 0;
    cluster_wait();
    const long long tq3 = timed ? clock64() : 0;
    if (warp == 0 && has_next) {
      // d_{it+1} = pushed partial dots + X_it delta_it (rank order, then the
      // cross-Gram term in column order)
      __syncwarp();  // delta[] of every lane
      const long long tk0 = timed ? clock64() : 0;
      double d = combine(it + 1);
      if (timed) {
        asm volatile("" ::"d"(d));
        tch[0] += clock64() - tk0;  // (debug: reuses the cluster-arrive slot) combine only
      }
      const double* xg = slot_g(it) + CD_B * CD_B + lane;  // X stored transposed: [l][next-block column]
      // four independent chains (l mod 4), combined in a fixed order
      double corr[4] = {0.0, 0.0, 0.0, 0.0};
      const double* dl_it = delta + (it & 1) * CD_B;
#pragma unroll
      for (int l = 0; l < CD_B; ++l) corr[l & 3] = fma(xg[l * CD_B], dl_it[l], corr[l & 3]);
      cdot = d + ((corr[0] + corr[1]) + (corr[2] + corr[3]));
    }
    const long long tq4 = timed ? clock64() : 0;
    if constexpr (!DEFER) __syncthreads();  // delta visible to the row warps
    const long long tq5 = timed ? clock64() : 0;
    // r += A_J delta_J on this CTA's rows (two slots: here; three slots: by
    // the row warps at the start of the next iteration, beside warp 0's
    // sequential update)
    if constexpr (!DEFER)
      if (warp > 0) axpy(it);
    // park block it+2's column state (its slot last held block it-1).  x of
    // a later pass comes from global memory only when rank 0 wrote it at
    // least two iterations ago (ordered by the cluster barriers since);
    // otherwise warp 0 has written it above
    if (it + 2 < total && tid < CD_ST * CD_B && (tid >= CD_B || nblk >= 4 || pass_2 == 0))
      cst[((it + 2) % 3) * CD_ST * CD_B + tid] = tid >= 3 * CD_B ? cd_isq(pfv) : pfv;
    if (NS == 2 && it + 2 < total) {  // (compile-time NS)
      __syncthreads();  // block it's slot is free
      if (warp > 0)
        cd_prefetch(a, slot_a(it + 2), slot_g(it + 2), blk_2, row0, nrows, &fullb[(int)(it + 2) % NS], pol,
                    warp - 1, NRW);
    }
    if (++blk_c == nb32) {
      blk_c = 0;
      ++pass_c;
    }
    if (++blk_2 == nb32) {
      blk_2 = 0;
      ++pass_2;
    }
    __syncthreads();
    if (timed) {
      const long long tq6 = clock64();
      tph[0] += tq1 - tq0;  // block data landed + CTA barrier
      tph[1] += tq2 - tq1;  // warp 0: prefetch issue + sequential block update
      tph7 += tq1a - tq1;   // of which: prefetch / state-load issue
      tph[2] += tq3 - tq2;  // cluster barrier wait (the row warps' dots, pushes, release)
      tph[3] += tq4 - tq3;  // combine + cross-Gram correction
      tph[4] += tq5 - tq4;  // CTA barrier
      tph[5] += tq6 - tq5;  // axpy phase (warp 0 waits for the row warps)
    }
  }
  if (timed)
    for (int q = 0; q < 6; ++q) atomicAdd(a.dbg + q, (unsigned long long)tph[q]);
  if (timed) atomicAdd(a.dbg + 6, (unsigned long long)total);
  if (timed) atomicAdd(a.dbg + 7, (unsigned long long)tph7);
  if (timed)
    for (int q = 0; q < 3; ++q) atomicAdd(a.dbg + 13 + q, (unsigned long long)tch[q]);
  if (timed_r)
    for (int q = 0; q < 5; ++q) atomicAdd(a.dbg + 8 + q, (unsigned long long)trw[q]);
  if constexpr (DEFER)
    if (total > 0 && warp > 0) axpy(total - 1);  // (the loop's closing barrier made its steps visible)
  // write back the residual rows and the objective 0.5 ||r||^2
  double sq = 0.0;
#pragma unroll
  for (int q = 0; q < RQ; ++q) {
    const int i = rt + q * CD_RT;
    if (rt >= 0 && i < nrows) {
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

// Gram blocks for consecutive blocks of CD_B preserved columns:
// [blk][0] = G_JJ = A_J'A_J and [blk][1] = X_J' = (A_next'A_J)' with next = J+1
// (block 0 after the last: the next pass starts over)
template <typename T>
__global__ void __launch_bounds__(256) k_gram(const T* __restrict__ A, int64_t ld, int64_t m, int64_t k,
                                              double* __restrict__ gram) {
  __shared__ T tile[2][CD_B][65];  // 64-row chunk of the block's / next block's columns (+1 pad)
  const int64_t nblk = (k + CD_B - 1) / CD_B;
  const int64_t blk = blockIdx.x;
  const int64_t nb = (blk + 1) % nblk;
  const int64_t c0 = blk * CD_B, c1 = nb * CD_B;
  const int nc = (int)min((int64_t)CD_B, k - c0);
  const int nc1 = (int)min((int64_t)CD_B, k - c1);
  // thread -> 4 (i, l) pairs of each 32x32 block
  double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
  for (int64_t r0 = 0; r0 < m; r0 += 64) {
    const int nr = (int)min((int64_t)64, m - r0);
    __syncthreads();
    for (int q = threadIdx.x; q < CD_B * 64; q += 256) {
      const int c = q / 64, i = q % 64;
      tile[0][c][i] = (c < nc && i < nr) ? A[(c0 + c) * ld + r0 + i] : T(0);
      tile[1][c][i] = (c < nc1 && i < nr) ? A[(c1 + c) * ld + r0 + i] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = threadIdx.x * 4 + u;
      const int i = p / CD_B, l = p % CD_B;
      double s = 0.0, sx = 0.0;
      for (int rr = 0; rr < nr; ++rr) {
        const double al = static_cast<double>(tile[0][l][rr]);
        s += static_cast<double>(tile[0][i][rr]) * al;
        sx += static_cast<double>(tile[1][i][rr]) * al;
      }
      acc[0][u] += s;
      acc[1][u] += sx;
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int p = threadIdx.x * 4 + u;
    gram[blk * 2 * CD_B * CD_B + p] = acc[0][u];
    // the cross-Gram block transposed ([l][i]): the correction reads column
    // i = lane for every l, conflict free
    gram[blk * 2 * CD_B * CD_B + CD_B * CD_B + (p % CD_B) * CD_B + p / CD_B] = acc[1][u];
  }
}

}  // namespace bx
