// Which ingredient of the batched kernel's inner loops keeps DMMA below the
// register-operand rate (dmma_probe.cu: 37 TFLOP/s)?  Runs the kernel's own
// GEMM1 / GEMM2 device functions on fake shared-memory operands.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I../../paper_2202_07258_b200/csrc -o dmma_feed_probe dmma_feed_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "bx_batched2.cuh"
using namespace bx;

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(double* out, int iters, int sa) {
  extern __shared__ __align__(128) unsigned char raw[];
  double* sm = reinterpret_cast<double*>(raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, tig = lane & 3;
  for (int q = tid; q < (64 + 16 * 4) * sa; q += 256) sm[q] = 1e-3 * (q % 97);
  __syncthreads();
  double* stage = sm;
  double* rys = sm + 4 * 16 * sa;
  const double* rw = rys + warp * 8 * sa + g * sa + tig;
  const int bo = b2_slot(g) * sa + tig;
  int so[2][2];
  for (int t = 0; t < 2; ++t) for (int e = 0; e < 2; ++e) so[t][e] = b2_slot(8 * t + 2 * tig + e) * sa;
  double acc[B2_MT][2];
  for (int q = 0; q < B2_MT; ++q) acc[q][0] = acc[q][1] = 0.0;
  double s = 0.0;
  double xn[2][2] = {{1.0, 2.0}, {3.0, 4.0}};
  for (int it = 0; it < iters; ++it) {
    const double* st = stage + (it & 3) * 16 * sa;
    if (MODE & 1) {
      double d[2][2];
      b2_gemm1<25>(rw - tig, st + bo - tig, 8 * sa, 25, tig, d);
      if (MODE & 4) { xn[0][0] = d[0][0]; xn[0][1] = d[0][1]; xn[1][0] = d[1][0]; xn[1][1] = d[1][1]; }
      else s += d[0][0] + d[0][1] + d[1][0] + d[1][1];
    }
    if (MODE & 2) b2_gemm2_n<25>(st, g, so, xn, acc);
  }
  for (int q = 0; q < B2_MT; ++q) s += acc[q][0] + acc[q][1];
  out[blockIdx.x * 256 + tid] = s;
}

template <int MODE>
void run(const char* name, double dmma_per_iter) {
  double* out;
  cudaMalloc(&out, 148 * 256 * 8);
  const int sa = 204, iters = 4000;
  const size_t smem = (size_t)(64 + 64) * sa * 8;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<MODE><<<148, 256, smem>>>(out, 10, sa);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<148, 256, smem>>>(out, iters, sa);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double n = 148.0 * 8 * iters * dmma_per_iter;
  printf("%-28s %7.2f TFLOP/s  err=%s\n", name, n * 512 / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  run<1>("gemm1 only (1.5 LDS/DMMA)", 100);
  run<2>("gemm2 only (1 LDS/DMMA)", 100);
  run<3>("gemm1 + gemm2 independent", 200);
  run<7>("gemm1 -> gemm2 dependent", 200);
  return 0;
}
