// Microbenchmark: cost of one level of a cluster-synchronous BFS step.
// Modes: 0 barrier only; 1 barrier + one global atomicMin per thread (distinct
// addresses); 2 barrier + atomicMin by 1/8 of the threads; 3 warp-0 DSMEM
// reads of 16 counters + __syncthreads + barrier.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__device__ __forceinline__ void cbar() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cbar_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__global__ void k(int mode, int iters, int* buf, long long* out) {
  __shared__ int cnt[4];
  cg::cluster_group cl = cg::this_cluster();
  if (threadIdx.x < 4) cnt[threadIdx.x] = threadIdx.x;
  cbar();
  long long t0 = clock64();
  int acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (mode == 1) acc += atomicMin(&buf[(blockIdx.x * blockDim.x + threadIdx.x) * 8], i);
    if (mode == 2 && (threadIdx.x & 7) == 0) acc += atomicMin(&buf[(blockIdx.x * blockDim.x + threadIdx.x) * 8], i);
    if (mode == 3 && threadIdx.x < 32) {
      int v = 0;
      if (threadIdx.x < gridDim.x) v = *reinterpret_cast<volatile int*>(cl.map_shared_rank(&cnt[i & 3], threadIdx.x));
      acc += v;
    }
    if (mode == 3) __syncthreads();
    if (mode == 4) { cbar_relaxed(); continue; }
    if (mode == 5) { if (threadIdx.x == 0) acc += atomicMin(&buf[blockIdx.x * 64], i); }
    cbar();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 12345) buf[0] = acc;
}
int main() {
  int* buf; long long* out;
  cudaMalloc(&buf, 64 << 20); cudaMemset(buf, 0x7f, 64 << 20);
  cudaMallocManaged(&out, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {16, 8, 2}) for (int th : {1024, 512, 256}) for (int mode = 0; mode < 6; ++mode) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs); cfg.blockDim = dim3(th); cfg.attrs = at; cfg.numAttrs = 1;
    const int iters = 2000;
    cudaLaunchKernelEx(&cfg, k, mode, iters, buf, out);
    cudaLaunchKernelEx(&cfg, k, mode, iters, buf, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("cluster %2d threads %4d mode %d: %7.1f cycles/iter %s\n", cs, th, mode, double(out[0]) / iters,
           e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
