// Timing harness for k_batched_round2 on synthetic buffers (values do not
// matter for timing): ablation studies with -DB2_ABL_* macros.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I../../paper_2202_07258_b200/csrc -I../../include -o b2_harness b2_harness.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "bx_batched2.cuh"
using namespace bx;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
int main(int argc, char** argv) {
  const int m = 200, n = 5000, K = 148 * 64; const int passes = argc > 2 ? atoi(argv[2]) : 10;
  const int m8 = 200, sa = m8 + 4, nch = (n + 15) / 16, npad = nch * 16;
  BatchArgs a{};
  a.m = m; a.n = n; a.K = K; a.sa = 212; a.sa2 = sa; a.nch = nch; a.ldy = m8; a.ldx = npad; a.nw = (n + 31) / 32;
  a.eta = 1e-3; a.passes = passes; a.par = 0; a.tile0 = 0; a.tile1 = K / 64; a.nrl = 1; a.round0 = 0; a.K_user = K; a.gap_tol = 1e-6; a.osum_rounds = 1; a.att_max = 14.0; a.nrm_min = 1.0; a.bound_skip = 0; a.sweeps2 = nullptr; a.screening = 1; a.rs_f = a.rs_g = a.slack_scale = 1e-12; a.dbg = nullptr;
  std::vector<double> hA((size_t)npad * sa);
  for (size_t i = 0; i < hA.size(); ++i) hA[i] = ((i * 2654435761u) % 1000) * 1e-3;
  double *Ap, *Y, *X0, *X1, *R0, *R1, *nrm, *att, *mom, *P, *stats; uint32_t* mask;
  CK(cudaMalloc(&Ap, hA.size() * 8)); CK(cudaMemcpy(Ap, hA.data(), hA.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&Y, (size_t)K * m8 * 8)); CK(cudaMemset(Y, 0, (size_t)K * m8 * 8));
  CK(cudaMalloc(&X0, (size_t)K * npad * 8)); CK(cudaMemset(X0, 0, (size_t)K * npad * 8));
  CK(cudaMalloc(&X1, (size_t)K * npad * 8)); CK(cudaMemset(X1, 0, (size_t)K * npad * 8));
  CK(cudaMalloc(&R0, (size_t)K * m8 * 8)); CK(cudaMemset(R0, 0, (size_t)K * m8 * 8));
  CK(cudaMalloc(&R1, (size_t)K * m8 * 8)); CK(cudaMemset(R1, 0, (size_t)K * m8 * 8));
  CK(cudaMalloc(&mask, (size_t)K * a.nw * 4)); CK(cudaMemset(mask, 0xff, (size_t)K * a.nw * 4));
  CK(cudaMalloc(&nrm, npad * 8)); CK(cudaMalloc(&att, npad * 8));
  unsigned* octr; double* osum;
  CK(cudaMalloc(&octr, K / 8 * 4)); CK(cudaMemset(octr, 0, K / 8 * 4)); CK(cudaMalloc(&osum, (size_t)K / 8 * 4 * 8));
  a.oct_round = octr; a.osum = osum;
  CK(cudaMalloc(&mom, K * 8)); CK(cudaMalloc(&P, K * 8)); CK(cudaMalloc(&stats, 5 * (size_t)K * 8));
  std::vector<double> ones(K > npad ? K : npad, 1.0);
  CK(cudaMemcpy(nrm, ones.data(), npad * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(att, ones.data(), npad * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(mom, ones.data(), K * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(P, ones.data(), K * 8, cudaMemcpyHostToDevice));
  a.Ap = Ap; a.A = Ap; a.lda = sa; a.Y = Y; a.X[0] = X0; a.X[1] = X1; a.R[0] = R0; a.R[1] = R1; a.mask = mask;
  a.nrm = nrm; a.att = att; a.mom = mom; a.P = P; a.stats = stats;
  const size_t smem = ((size_t)(B2_NST * BT_CH + BT_TILE) * sa) * 8 + B2_NST * 12 + 16;
  CK(cudaFuncSetAttribute(k_batched_round2<25, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k_batched_round2<25, true><<<148, B2_NT, smem>>>(a);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = (4.0 * passes + 4.0) * m * n * (double)K;
  printf("%s: %.3f ms per round, %.2f TFLOP/s (algorithmic)\n", argc > 1 ? argv[1] : "base", best, flops / best / 1e9);
  return 0;
}
