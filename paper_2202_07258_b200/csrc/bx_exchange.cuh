// bx_exchange.cuh -- the column-sharded step's reduction fused with the
// cross-GPU exchange over peer memory.
//
// After a sharded PG / FISTA pass every rank holds G per-CTA partial rows of
// its A_g x_g.  The NCCL schedule (bx_core.cu run_reduce) is four launches and
// two collectives: local reduce -> allreduce(m) -> allreduce(scalars) ->
// finalise.  k_xreduce does all of it in ONE kernel per rank:
//   1. each CTA sums the G partial rows of its row block (fixed order),
//   2. stores the block straight into every peer's receive buffer
//      (st.global through CUDA-IPC-mapped peer pointers: NVLink / NVSwitch),
//      CTA 0 also the pass's scalar partials (restart test, power norm),
//   3. publishes a per-(rank, CTA) flag on each peer (st.release.sys),
//   4. waits for the same row block from every peer (ld.acquire.sys),
//   5. sums the peers' blocks in rank order + the offset (z - y): the new
//      residual -- bit-identical on every rank -- and folds the objective /
//      StepSizeTooLarge / restart test exactly like k_reduce.
// The receive buffer is double-buffered by call parity and flags carry the
// call's epoch (monotonic, compared with >=), so a rank that runs ahead can
// never overwrite data a slower peer is still summing.  Every rank launches
// the same co-resident grid (cooperative launch), so the cross-GPU waits
// cannot deadlock on unscheduled CTAs.
//
// Single-GPU test transport (bx_group): one cooperative launch of
// nranks x nb CTAs emulates all ranks over their own buffers
// (k_xreduce_group), the pattern the B200 notes prescribe for testing a
// multi-rank protocol with fewer GPUs than ranks.
#pragma once
#include "bx_kernels.cuh"

namespace bx {

constexpr int kXPeers = 8;   // one NVSwitch node
constexpr int kXExtra = 8;   // scalar slots after the m rows of each payload
constexpr int XT = 256;      // block size
constexpr int XCH = 64;      // rows per chunk of the local reduction
constexpr int XG = XT / XCH; // thread groups splitting the partial rows

// rows of the reduction owned by one CTA: a multiple of the chunk
__host__ __device__ inline int64_t xrows_per_cta(int64_t m, int nb) {
  const int64_t per = (m + nb - 1) / nb;
  return (per + XCH - 1) / XCH * XCH;
}

struct XArgs {
  const void* part;   // [G][ldp] partial rows of this rank (storage type T)
  int64_t ldp;
  int G;
  int64_t m, mp;      // rows, padded rows (payload stride = mp + kXExtra)
  const double* off;  // offset added after the sum (NULL: none)
  double* out;        // the reduced vector (replicated on every rank)
  double* save;       // speculative step: out's previous contents (NULL: none)
  uint64_t timeout_ns;  // bound of every peer wait (%globaltimer); DE_PEER_TIMEOUT beyond it
  DevScalars* sc;
  double* bpart;      // [nb] per-CTA ||out||^2 partials
  const double* wpart;  // [Gw][stride] pass scalar partials (NULL: none)
  int Gw, stride;
  int mode, counter;
  int rank, nranks, nb;
  unsigned epoch;
  double* recv[kXPeers];    // peer q's receive buffer base (2 parities)
  unsigned* flag[kXPeers];  // peer q's flag array base [kXPeers][nb]
  double* my_recv;
  unsigned* my_flag;
};

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// epochs are monotonic (mod 2^32): "reached" survives a peer running ahead
__device__ __forceinline__ bool reached(unsigned v, unsigned epoch) { return (int)(v - epoch) >= 0; }
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Bounded wait for a peer's flag: a peer that errored, exited or took the
// NCCL schedule never publishes, so after timeout_ns the wait gives up and
// raises DE_PEER_TIMEOUT (the host turns it into an error on every rank that
// tripped, instead of a kernel that never returns).  Returns false on timeout.
__device__ __forceinline__ bool wait_flag(const unsigned* p, unsigned epoch, uint64_t t0, uint64_t timeout_ns,
                                          DevScalars* sc) {
  unsigned spins = 0;
  while (!reached(ld_acquire_sys(p), epoch)) {
    if ((++spins & 1023u) == 0 && globaltimer_ns() - t0 > timeout_ns) {
      atomicCAS(&sc->err, 0, DE_PEER_TIMEOUT);
      return false;
    }
  }
  return true;
}

template <typename T>
__device__ void xreduce_body(const XArgs& a, int cta) {
  __shared__ double sh[XT / 32];
  __shared__ double ex[kXExtra];
  __shared__ bool last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m = a.m;
  const int64_t pay = a.mp + kXExtra;
  const int par = (int)(a.epoch & 1u);
  const int64_t per = xrows_per_cta(m, a.nb);
  const int64_t r0 = cta * per < m ? cta * per : m;
  const int64_t r1 = r0 + per < m ? r0 + per : m;
  const T* part = static_cast<const T*>(a.part);
  // 1-2. local sums of this row block (XG thread groups split the G partial
  // rows, combined in group order: fixed), stored into every peer's buffer
  {
    __shared__ double gs[XG][XCH];
    const int g = tid / XCH, c = tid % XCH;
    for (int64_t base = r0; base < r1; base += XCH) {
      const int64_t i = base + c;
      double s = 0.0;
      if (i < r1)
        for (int b = g; b < a.G; b += XG) s += static_cast<double>(__ldcg(part + (int64_t)b * a.ldp + i));
      gs[g][c] = s;
      __syncthreads();
      if (tid < XCH && i < r1) {
        double t = gs[0][c];
#pragma unroll
        for (int h = 1; h < XG; ++h) t += gs[h][c];
        for (int q = 0; q < a.nranks; ++q) a.recv[q][((int64_t)par * kXPeers + a.rank) * pay + i] = t;
      }
      __syncthreads();
    }
  }
  if (cta == 0 && warp == 0 && a.wpart) {
    for (int e = 0; e < a.stride; ++e) {
      double v = 0.0;
      for (int b = lane; b < a.Gw; b += 32) v += __ldcg(&a.wpart[b * a.stride + e]);
      v = warp_sum<double>(v);
      if (lane == 0)
        for (int q = 0; q < a.nranks; ++q) a.recv[q][((int64_t)par * kXPeers + a.rank) * pay + a.mp + e] = v;
    }
  }
  __threadfence_system();
  __syncthreads();
  // 3. publish this block on every peer
  if (tid < a.nranks) st_release_sys(&a.flag[tid][a.rank * a.nb + cta], a.epoch);
  // 4. wait for the same block (and the scalar slots of CTA 0) from every peer
  if (tid < a.nranks) {
    const uint64_t t0 = globaltimer_ns();
    if (wait_flag(&a.my_flag[tid * a.nb + cta], a.epoch, t0, a.timeout_ns, a.sc) && a.wpart && cta != 0)
      wait_flag(&a.my_flag[tid * a.nb], a.epoch, t0, a.timeout_ns, a.sc);
  }
  __threadfence();
  __syncthreads();
  const double* rb = a.my_recv + (int64_t)par * kXPeers * pay;
  if (tid < kXExtra) {
    double v = 0.0;
    if (a.wpart && tid < a.stride)
      for (int q = 0; q < a.nranks; ++q) v += __ldcv(rb + q * pay + a.mp + tid);
    ex[tid] = v;
  }
  __syncthreads();
  const int base = a.mode & ~R_SPEC;
  const double s_div = (base == R_POWER) ? sqrt(ex[0]) : 1.0;
  // 5. the replicated result: peers summed in rank order (+ offset)
  double sq = 0.0;
  for (int64_t i = r0 + tid; i < r1; i += XT) {
    double s = __ldcv(rb + i);
    for (int q = 1; q < a.nranks; ++q) s += __ldcv(rb + q * pay + i);
    if (a.off) s = add_rn(s, a.off[i]);
    if (base == R_POWER) s = s / s_div;
    if (a.save) a.save[i] = a.out[i];
    a.out[i] = s;
    sq += s * s;
  }
  if (base == R_PLAIN) return;
  sq = warp_sum<double>(sq);
  if (lane == 0) sh[warp] = sq;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < XT / 32; ++w) t += sh[w];
    a.bpart[cta] = t;
    __threadfence();
    const unsigned prev = atomicAdd(&a.sc->counters[a.counter], 1u);
    last = (prev == (unsigned)a.nb - 1);
  }
  __syncthreads();
  if (!last || warp != 0) return;
  __threadfence();
  double total = 0.0;
  for (int b = lane; b < a.nb; b += 32) total += __ldcg(&a.bpart[b]);
  total = warp_sum<double>(total);
  if (lane != 0) return;
  finalize_objective<T>(a.sc, a.mode, 0.5 * total, base == R_POWER ? s_div : 0.0, ex[0], ex[1]);
  a.sc->counters[a.counter] = 0u;
}

// one rank (production: peers are other GPUs)
template <typename T>
__global__ void __launch_bounds__(XT) k_xreduce(const XArgs a) {
  xreduce_body<T>(a, blockIdx.x);
}

// every rank of an in-process group in one cooperative launch (one GPU)
template <typename T>
__global__ void __launch_bounds__(XT) k_xreduce_group(const XArgs* __restrict__ all, int nb) {
  const XArgs a = all[blockIdx.x / nb];
  xreduce_body<T>(a, blockIdx.x % nb);
}

}  // namespace bx
