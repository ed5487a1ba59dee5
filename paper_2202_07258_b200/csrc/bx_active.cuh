// bx_active.cuh -- the active-set primal update (bounded-variable
// Lawson-Hanson), reference solvers.py:140-204 (ActiveSetState :38-45).
//
// One outer iteration frees the bound coordinate whose multiplier most
// violates optimality, then repeatedly solves the least-squares problem on the
// passive columns and backs off along the segment to the first bound hit.
// The reference refactors the passive Gram matrix from scratch every inner
// iteration (scipy cho_factor, O(m p^2 + p^3)).  Here the Cholesky factor
// R (A_P'A_P = R'R) is kept on the device across iterations and updated:
//   * a column entering the passive set appends one column to R: one forward
//     substitution against A_P'a_j (k_as_dots + k_as_append), O(m p + p^2);
//   * a column leaving it deletes that column of R and re-triangularises the
//     Hessenberg remainder with Givens rotations (k_as_solve), O(p^2).
// Each inner iteration is then O(m k) (the fixed-column residual, one
// streamed pass) + O(p^2) (two triangular solves) instead of O(m p^2 + p^3).
//
// Factor layout (workspace, ld = pcap = min(m, n)): R is upper triangular
// in LOGICAL order; logical column j lives in physical column cslot[j] (so a
// deletion shifts an index list, not the matrix), rows are logical.
// plist[j] = preserved position of logical column j.  The passive mask itself
// travels with the per-column state through compaction (bx_core.cu).
#pragma once
#include "bx_kernels.cuh"

namespace bx {

constexpr int AS_NT = 512;

enum AsStatus : int { AS_DONE = 0, AS_CONTINUE = 1, AS_SINGULAR = 2 };

struct AsState {
  int32_t p;       // passive columns held in the factor
  int32_t jstar;   // entering preserved position of this outer iteration (-1: KKT optimal)
  int32_t status;  // AsStatus of the last kernel
  int32_t nhit;    // columns that left the passive set in the last inner iteration
  double d2;       // pivot of the last append (singularity diagnostics)
  double rnorm;    // ||r|| of the selection (tolerance scale)
};

// sum over the block, the same value (same order) in every thread
__device__ __forceinline__ double as_block_sum(double v, double* sh) {
  v = warp_sum<double>(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
  __syncthreads();
  return t;
}

__device__ __forceinline__ double& Rat(double* R, int64_t ld, const int32_t* cslot, int i, int j) {
  return R[(int64_t)i + (int64_t)cslot[j] * ld];
}

// reset: empty factor, identity slot map
__global__ void k_as_reset(int pcap, int32_t* cslot, AsState* as) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < pcap; i += gridDim.x * blockDim.x) cslot[i] = i;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    as->p = 0;
    as->jstar = -1;
    as->status = AS_DONE;
    as->nhit = 0;
  }
}

// Selection (solvers.py:166-177): w = -g, tol_j = 1e-10 ||a_j|| max(||r||, 1);
// violation of a bound coordinate at its lower bound with w > tol, or at a
// finite upper bound with w < -tol; the first index of the largest violation
// enters the passive set.
__global__ void __launch_bounds__(AS_NT) k_as_select(int64_t k, int64_t m, const double* __restrict__ x,
                                                     const double* __restrict__ lo, const double* __restrict__ hi,
                                                     const double* __restrict__ g, const double* __restrict__ nrm,
                                                     double* __restrict__ pmask, const double* __restrict__ r,
                                                     int32_t* __restrict__ plist, AsState* as) {
  __shared__ double sh[AS_NT / 32];
  __shared__ double sv[AS_NT / 32];
  __shared__ int64_t si[AS_NT / 32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += AS_NT) s += r[i] * r[i];
  const double rn = sqrt(as_block_sum(s, sh));
  const double scale = fmax(rn, 1.0);
  double best = 0.0;
  int64_t bi = INT64_MAX;
  for (int64_t j = threadIdx.x; j < k; j += AS_NT) {
    if (pmask[j] != 0.0) continue;
    const double w = -g[j];
    const double tol = 1e-10 * nrm[j] * scale;
    double v = 0.0;
    if (x[j] <= lo[j] && w > tol) v = w;
    if (!isinf(hi[j]) && x[j] >= hi[j] && w < -tol) v = fmax(v, -w);
    if (v > best) {  // ascending j per thread: first index on ties
      best = v;
      bi = j;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_down_sync(0xffffffffu, best, o);
    const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sv[warp] = best;
    si[warp] = bi;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int w = 1; w < AS_NT / 32; ++w)
    if (sv[w] > best || (sv[w] == best && si[w] < bi)) {
      best = sv[w];
      bi = si[w];
    }
  as->rnorm = rn;
  if (best > 0.0) {
    as->jstar = (int32_t)bi;
    pmask[bi] = 1.0;
    plist[as->p] = (int32_t)bi;
  } else {
    as->jstar = -1;
  }
  as->status = AS_DONE;
}

// a_j as an fp64 m-vector (j = jfix, or the selected column)
template <typename T>
__global__ void k_as_colcopy(const T* __restrict__ A, int64_t ld, const int32_t* __restrict__ colmap, int64_t m,
                             double* __restrict__ out, int32_t* __restrict__ plist, AsState* as, int32_t jfix) {
  const int32_t j = jfix >= 0 ? jfix : as->jstar;
  if (j < 0) return;
  const int64_t col = colmap ? colmap[j] : j;
  const T* a = A + col * ld;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<double>(a[i]);
  if (jfix >= 0 && blockIdx.x == 0 && threadIdx.x == 0) plist[as->p] = jfix;
}

// out[i] = a_{plist[i]} . vec for i < npl (one warp per column)
template <typename T>
__global__ void __launch_bounds__(256) k_as_dots(const T* __restrict__ A, int64_t ld,
                                                 const int32_t* __restrict__ colmap,
                                                 const int32_t* __restrict__ plist, int npl,
                                                 const double* __restrict__ vec, int64_t m,
                                                 double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= npl) return;
  const int32_t j = plist[i];
  const int64_t col = colmap ? colmap[j] : j;
  const T* a = A + col * ld;
  double s = 0.0;
  for (int64_t r = lane; r < m; r += 32) s += static_cast<double>(a[r]) * vec[r];
  s = warp_sum<double>(s);
  if (lane == 0) out[i] = s;
}

// Append the column whose A_P'a_j (first p entries) and a_j'a_j (entry p) are
// in c: R'w = c[0:p) by forward substitution, pivot d = c[p] - w'w.  A
// non-positive (or NaN) pivot is LAPACK potrf's failure condition, i.e. the
// reference's SingularSubproblem (solvers.py:144-147).
__global__ void __launch_bounds__(AS_NT) k_as_append(double* __restrict__ R, int64_t ld, int pcap,
                                                     const int32_t* __restrict__ cslot, AsState* as,
                                                     const double* __restrict__ c) {
  __shared__ double sh[AS_NT / 32];
  if (as->status == AS_SINGULAR) return;
  const int p = as->p;
  if (p >= pcap) {  // more passive columns than rows: A_P'A_P is rank deficient
    if (threadIdx.x == 0) {
      as->status = AS_SINGULAR;
      as->d2 = 0.0;
    }
    return;
  }
  double* w = R + (int64_t)cslot[p] * ld;
  for (int i = 0; i < p; ++i) {
    const double* ri = R + (int64_t)cslot[i] * ld;
    double s = 0.0;
    for (int l = threadIdx.x; l < i; l += AS_NT) s += ri[l] * w[l];
    s = as_block_sum(s, sh);
    if (threadIdx.x == 0) w[i] = (c[i] - s) / ri[i];
    __syncthreads();
  }
  double q = 0.0;
  for (int l = threadIdx.x; l < p; l += AS_NT) q += w[l] * w[l];
  q = as_block_sum(q, sh);
  if (threadIdx.x == 0) {
    const double d2 = c[p] - q;
    as->d2 = d2;
    if (!(d2 > 0.0)) {
      as->status = AS_SINGULAR;
    } else {
      w[p] = sqrt(d2);
      as->p = p + 1;
      as->status = AS_CONTINUE;
    }
  }
}

// shift list[q+1..p) one place left (all threads; staged through registers)
__device__ void as_shift_left(int32_t* list, int q, int p) {
  constexpr int CH = 8;
  for (int base = q; base < p - 1; base += AS_NT * CH) {
    int32_t v[CH];
#pragma unroll
    for (int e = 0; e < CH; ++e) {
      const int i = base + e * AS_NT + threadIdx.x;
      v[e] = (i < p - 1) ? list[i + 1] : 0;
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < CH; ++e) {
      const int i = base + e * AS_NT + threadIdx.x;
      if (i < p - 1) list[i] = v[e];
    }
    __syncthreads();
  }
}

// One inner iteration (solvers.py:180-201): s = (R'R)^-1 b; if s is within
// the bounds, x_P = s and the outer iteration ends (AS_DONE); otherwise step
// x_P toward s to the first bound hit, snap the hit coordinates to their
// bound, drop them from the passive set and from the factor (AS_CONTINUE).
__global__ void __launch_bounds__(AS_NT) k_as_solve(double* __restrict__ R, int64_t ld, int32_t* __restrict__ cslot,
                                                    int32_t* __restrict__ plist, AsState* as,
                                                    const double* __restrict__ b, double* __restrict__ s,
                                                    double* __restrict__ frac, int32_t* __restrict__ hitf,
                                                    double* __restrict__ x, const double* __restrict__ lo,
                                                    const double* __restrict__ hi, double* __restrict__ pmask) {
  __shared__ double sh[AS_NT / 32];
  __shared__ double rot[2];
  if (as->status == AS_SINGULAR) return;  // the append before this iteration failed
  int p = as->p;
  // forward substitution R'z = b (column i of R is row i of R': contiguous)
  for (int i = 0; i < p; ++i) {
    const double* ri = R + (int64_t)cslot[i] * ld;
    double t = 0.0;
    for (int l = threadIdx.x; l < i; l += AS_NT) t += ri[l] * s[l];
    t = as_block_sum(t, sh);
    if (threadIdx.x == 0) s[i] = (b[i] - t) / ri[i];
    __syncthreads();
  }
  // back substitution R s = z, column-oriented (column i contiguous)
  for (int i = p - 1; i >= 0; --i) {
    const double* ri = R + (int64_t)cslot[i] * ld;
    const double si = s[i] / ri[i];
    __syncthreads();
    if (threadIdx.x == 0) s[i] = si;
    for (int l = threadIdx.x; l < i; l += AS_NT) s[l] -= ri[l] * si;
    __syncthreads();
  }
  // bound check
  int out = 0;
  for (int i = threadIdx.x; i < p; i += AS_NT) {
    const int32_t j = plist[i];
    out |= (s[i] < lo[j]) || (s[i] > hi[j]);
  }
  if (!__syncthreads_or(out)) {
    for (int i = threadIdx.x; i < p; i += AS_NT) x[plist[i]] = s[i];
    if (threadIdx.x == 0) {
      as->status = AS_DONE;
      as->nhit = 0;
    }
    return;
  }
  // step length to the first bound hit: min over the segment fractions
  // (NaN propagates like np.min; the clamp keeps a NaN like Python's max/min)
  double mn = INFINITY;
  int nan_seen = 0;
  for (int i = threadIdx.x; i < p; i += AS_NT) {
    const int32_t j = plist[i];
    const double xp = x[j], si = s[i];
    double f = INFINITY;
    if (si < lo[j])
      f = (lo[j] - xp) / (si - xp);
    else if (si > hi[j])
      f = (hi[j] - xp) / (si - xp);
    frac[i] = f;
    if (isnan(f))
      nan_seen = 1;
    else
      mn = fmin(mn, f);
  }
  for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mn;
  nan_seen = __syncthreads_or(nan_seen);
  double alpha = sh[0];
  for (int w = 1; w < AS_NT / 32; ++w) alpha = fmin(alpha, sh[w]);
  if (nan_seen) alpha = NAN;
  if (!isnan(alpha)) alpha = fmin(fmax(alpha, 0.0), 1.0);
  int nh = 0;
  for (int i = threadIdx.x; i < p; i += AS_NT) {
    const int32_t j = plist[i];
    const double xp = x[j], si = s[i];
    const bool below = si < lo[j], above = si > hi[j];
    double xn = xp + alpha * (si - xp);
    const bool hit = frac[i] <= alpha + 1e-12;
    if (hit && below) xn = lo[j];
    if (hit && above) xn = hi[j];
    x[j] = xn;
    hitf[i] = hit ? 1 : 0;
    if (hit) {
      pmask[j] = 0.0;
      ++nh;
    }
  }
  nh = __syncthreads_count(nh);
  // delete the hit columns from the factor, highest logical index first
  for (int q = p - 1; q >= 0; --q) {
    if (!hitf[q]) continue;  // uniform: every thread reads the same flag
    const int32_t freed = cslot[q];
    as_shift_left(cslot, q, p);
    as_shift_left(plist, q, p);
    if (threadIdx.x == 0) cslot[p - 1] = freed;
    __syncthreads();
    // columns q..p-2 now have one sub-diagonal entry: Givens rotations on
    // rows (l, l+1) restore the triangle; row p-1 becomes zero and is dropped
    for (int l = q; l < p - 1; ++l) {
      if (threadIdx.x == 0) {
        const double a = Rat(R, ld, cslot, l, l), bb = Rat(R, ld, cslot, l + 1, l);
        const double h = hypot(a, bb);
        rot[0] = h > 0.0 ? a / h : 1.0;
        rot[1] = h > 0.0 ? bb / h : 0.0;
        Rat(R, ld, cslot, l, l) = h;
        Rat(R, ld, cslot, l + 1, l) = 0.0;
      }
      __syncthreads();
      const double cr = rot[0], sr = rot[1];
      for (int jj = l + 1 + threadIdx.x; jj < p - 1; jj += AS_NT) {
        double& t1 = Rat(R, ld, cslot, l, jj);
        double& t2 = Rat(R, ld, cslot, l + 1, jj);
        const double u1 = t1, u2 = t2;
        t1 = cr * u1 + sr * u2;
        t2 = -sr * u1 + cr * u2;
      }
      __syncthreads();
    }
    --p;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < p; ++i)
      if (!(Rat(R, ld, cslot, i, i) > 0.0)) as->status = AS_SINGULAR;
    if (as->status != AS_SINGULAR) as->status = AS_CONTINUE;
    as->p = p;
    as->nhit = nh;
  }
}

// coefficients of the fixed columns' contribution: -x_j off the passive set
__global__ void k_as_coef(int64_t k, const double* __restrict__ x, const double* __restrict__ pmask,
                          double* __restrict__ coef) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x)
    coef[j] = pmask[j] != 0.0 ? 0.0 : -x[j];
}

}  // namespace bx
