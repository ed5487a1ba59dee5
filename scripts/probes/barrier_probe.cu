// Probe: co-resident cluster capacity on this GPU and the latency of a
// grid-wide barrier (monotonic counter, release-reduction + acquire polling)
// vs a cluster barrier, in a persistent cooperative launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_probe barrier_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void gbar(unsigned* bar, unsigned& n) {
  __syncthreads();
  ++n;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    const unsigned t = n * gridDim.x;
    while (ld_acq(bar) < t) {
    }
  }
  __syncthreads();
}

__global__ void k_grid(unsigned* bar, int iters, long long* out) {
  unsigned n = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) gbar(bar, n);
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}

__global__ void k_cluster(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = t1 - t0;
}

int main() {
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, 0);
  printf("%s: %d SMs, clock %d kHz\n", pr.name, pr.multiProcessorCount, pr.clockRate);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(cs * 64, 1, 1);
    lc.blockDim = dim3(512, 1, 1);
    lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    int ncl = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, k_cluster, &lc);
    printf("cluster %2d: max active clusters %d (%d CTAs) %s\n", cs, ncl, ncl * cs, cudaGetErrorString(e));
  }
  unsigned* bar;
  long long* out;
  cudaMalloc(&bar, 4);
  cudaMalloc(&out, 16);
  const int iters = 20000;
  for (int G : {148, 144, 128, 74, 37}) {
    cudaMemset(bar, 0, 4);
    void* args[] = {&bar, (void*)&iters, &out};
    int it = iters;
    args[1] = &it;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t e = cudaLaunchCooperativeKernel((void*)k_grid, dim3(G), dim3(512), args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("grid barrier G=%3d: %.3f us per barrier (%s)\n", G, 1e3 * ms / iters, cudaGetErrorString(e));
  }
  for (int cs : {2, 4, 8, 16}) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(cs * (144 / cs / 1), 1, 1);
    if (cs == 16) lc.gridDim = dim3(128, 1, 1);
    lc.blockDim = dim3(512, 1, 1);
    lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 2;
    int it = iters;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t e = cudaLaunchKernelEx(&lc, k_cluster, it, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("cluster barrier cs=%2d grid=%d (cooperative+cluster launch): %.3f us per barrier (%s)\n", cs,
           lc.gridDim.x, 1e3 * ms / iters, cudaGetErrorString(e));
  }
  return 0;
}
