// Latency of the coordinate-descent block update's dependency chain on
// sm_100a, one warp per SM: which link costs what?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cdchain_probe cdchain_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, int iters, double s) {
  if (threadIdx.x >= 32) {  // other warps of the CTA wait at a barrier, as in k_cd
    __syncthreads();
    return;
  }
  const int lane = threadIdx.x & 31;
  double c = 0.3 + lane * 1e-3, x = 0.5, lo = 0.0, hi = 1.0, isq = 1.0 + s * 1e-9, g = 1e-3 * lane + s * 1e-9;
  for (int it = 0; it < iters; ++it) {
    double nv = fma(-c, isq, x);
    if (MODE == 0 || MODE == 2) {
      nv = nv < lo ? lo : nv;
      nv = nv > hi ? hi : nv;
    } else if (MODE == 1 || MODE == 3) {
      nv = fmin(fmax(nv, lo), hi);
    }
    const double dt = nv - x;
    double di = dt;
    if (MODE == 0 || MODE == 1 || MODE == 4) di = __shfl_sync(0xffffffffu, dt, it & 31);
    c = fma(g, di, c);
  }
  out[blockIdx.x * 32 + threadIdx.x] = c;
  __syncthreads();
}
template <int MODE, int NTH = 32>
void run(const char* name) {
  double* out; cudaMalloc(&out, 148 * 32 * 8);
  const int iters = 200000;
  k<MODE><<<148, NTH>>>(out, 10, 1.0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<148, NTH>>>(out, iters, 1.0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%-44s %6.1f clk per step (at 1.965 GHz)\n", name, ms * 1e-3 * 1.965e9 / iters);
  cudaFree(out);
}
int main() {
  run<0>("fma, compare-select clip, sub, shfl, fma");
  run<1>("fma, fmin/fmax clip, sub, shfl, fma");
  run<2>("fma, compare-select clip, sub, fma (no shfl)");
  run<3>("fma, fmin/fmax clip, sub, fma (no shfl)");
  run<4>("fma, sub, shfl, fma (no clip)");
  run<5>("fma, sub, fma (no clip, no shfl)");
  run<0, 256>("full chain, 8 warps per CTA (7 at a barrier)");
  run<0, 1024>("full chain, 32 warps per CTA (31 at a barrier)");
  return 0;
}
