// Vector fp64 (DFMA) issue rate and dependent latency on sm_100a, per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dfma_probe dfma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, int iters, double s) {
  double c[CH];
  for (int i = 0; i < CH; ++i) c[i] = threadIdx.x * 1e-3 + i;
  const double a = 1.0 + s * 1e-9, b = s * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i] = fma(c[i], a, b);
  }
  double t = 0;
  for (int i = 0; i < CH; ++i) t += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int CH>
void run(int warps) {
  double* out; cudaMalloc(&out, 148 * 1024 * 8);
  const int iters = 20000;
  k<CH><<<148, warps * 32>>>(out, 10, 1.0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<CH><<<148, warps * 32>>>(out, iters, 1.0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double n = (double)warps * iters * CH;  // warp-level DFMAs per SM
  printf("warps/SM %2d chains %2d: %6.2f TFLOP/s, %.2f clk per warp-DFMA per SM sub-partition (at 1.965 GHz), %.1f clk per dependent DFMA\n",
         warps, CH, 148.0 * n * 64 / ms / 1e9, ms * 1e-3 * 1.965e9 / (n / 4.0), ms * 1e-3 * 1.965e9 / iters);
  cudaFree(out);
}
int main() {
  run<1>(1); run<8>(1); run<16>(1); run<8>(4); run<8>(16); run<1>(4); run<2>(4); run<4>(4);
  return 0;
}
