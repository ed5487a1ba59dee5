// The in-kernel form of the CD block update loop (k_cd, bx_cd.cuh) in
// isolation: one warp per SM, Gram row and state in shared memory.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, int blocks, int nc, double s) {
  __shared__ double g[32 * 32];
  __shared__ double cs[4 * 32];
  const int lane = threadIdx.x & 31;
  for (int q = lane; q < 1024; q += 32) g[q] = 1e-3 * (q % 37) + s * 1e-9;
  for (int q = lane; q < 128; q += 32) cs[q] = q < 32 ? 0.5 : (q < 64 ? 0.0 : (q < 96 ? 1.0 : 1.0 + s * 1e-9));
  __syncwarp();
  double cdot = 0.3 + lane * 1e-3, acc = 0.0;
  for (int b = 0; b < blocks; ++b) {
    double xj = cs[lane], loj = cs[32 + lane], hij = cs[64 + lane], isq = cs[96 + lane];
    const double* grow = g + lane * 32;
    double dl = 0.0, gnext = grow[0];
    if (MODE == 0) {
#pragma unroll 1
      for (int i = 0; i < nc; ++i) {
        const double gi = gnext;
        gnext = grow[(i + 1) & 31];
        double nv = fma(-cdot, isq, xj);
        nv = nv < loj ? loj : nv;
        nv = nv > hij ? hij : nv;
        const double dt = nv - xj;
        const double di = __shfl_sync(0xffffffffu, dt, i);
        const bool me = lane == i;
        xj = (me && dt != 0.0) ? nv : xj;
        dl = me ? dt : dl;
        cdot = fma(gi, di, cdot);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const double gi = grow[i];
        double nv = fma(-cdot, isq, xj);
        nv = nv < loj ? loj : nv;
        nv = nv > hij ? hij : nv;
        const double dt = nv - xj;
        const double di = __shfl_sync(0xffffffffu, dt, i);
        const bool me = lane == i;
        if (MODE == 1) xj = (me && dt != 0.0) ? nv : xj;
        dl = me ? dt : dl;
        cdot = fma(gi, di, cdot);
      }
    }
    acc += dl + xj;
  }
  out[blockIdx.x * 32 + lane] = cdot + acc;
}
template <int MODE>
void run(const char* name) {
  double* out; cudaMalloc(&out, 148 * 32 * 8);
  const int blocks = 4000;
  k<MODE><<<148, 32>>>(out, 10, 32, 1.0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<148, 32>>>(out, blocks, 32, 1.0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%-52s %6.1f clk per step\n", name, ms * 1e-3 * 1.965e9 / blocks / 32);
  cudaFree(out);
}
int main() {
  run<0>("rolled loop as in k_cd");
  run<1>("unrolled, with the x_j select");
  run<2>("unrolled, without the x_j select");
  return 0;
}
