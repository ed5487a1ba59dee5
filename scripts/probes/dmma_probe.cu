// DMMA throughput by MMA shape on sm_100a: which fp64 mma.sync shape reaches
// the fp64 tensor peak?  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__device__ __forceinline__ void mma(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  if constexpr (SHAPE == 0) {  // m8n8k4: 512 flops
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a[0]), "d"(b[0]));
  } else if constexpr (SHAPE == 1) {  // m16n8k4: 1024 flops
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
  } else if constexpr (SHAPE == 2) {  // m16n8k8: 2048 flops
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  } else {  // m16n8k16: 4096 flops
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
}

template <int SHAPE, int CH>
__global__ void k(double* out, int iters, double seed) {
  double c[CH][4], a[8], b[4];
  for (int i = 0; i < CH; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  for (int j = 0; j < 8; ++j) a[j] = seed + threadIdx.x * 1e-3 + j;
  for (int j = 0; j < 4; ++j) b[j] = seed * 0.5 + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) mma<SHAPE>(c[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < CH; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int SHAPE, int CH>
void run(int warps, const char* name, double flops_per) {
  double* out;
  cudaMalloc(&out, 148 * 1024 * 8);
  const int iters = 20000;
  k<SHAPE, CH><<<148, warps * 32>>>(out, 100, 1.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<SHAPE, CH><<<148, warps * 32>>>(out, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double n = 148.0 * warps * iters * CH;
  printf("%-10s warps/SM %2d chains %2d: %7.2f TFLOP/s  (%.3f mma/ns/SM)\n", name, warps, CH, n * flops_per / ms / 1e9,
         n / 148 / (ms * 1e6));
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 16}) {
    if (w == 4) { run<0, 8>(4, "m8n8k4", 512); run<1, 8>(4, "m16n8k4", 1024); run<2, 8>(4, "m16n8k8", 2048); run<3, 8>(4, "m16n8k16", 4096); }
    if (w == 8) { run<0, 8>(8, "m8n8k4", 512); run<1, 8>(8, "m16n8k4", 1024); run<2, 8>(8, "m16n8k8", 2048); run<3, 8>(8, "m16n8k16", 4096); }
    if (w == 16) { run<0, 8>(16, "m8n8k4", 512); run<1, 8>(16, "m16n8k4", 1024); run<2, 8>(16, "m16n8k8", 2048); run<3, 8>(16, "m16n8k16", 4096); }
  }
  run<0, 1>(8, "m8n8k4", 512); run<0, 2>(8, "m8n8k4", 512); run<0, 4>(8, "m8n8k4", 512);
  run<3, 1>(8, "m16n8k16", 4096); run<3, 2>(8, "m16n8k16", 4096);
  return 0;
}
