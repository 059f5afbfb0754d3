// Microbenchmark: cost of cluster.sync() and of one DSMEM-reading Jacobi-like
// sweep per sync, for cluster sizes 1..16 and 1024/512/256 threads per CTA.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, unsigned long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) cl.sync();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
}

__global__ void k_sweep(int iters, int remote_every, unsigned long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double x[2][1024];
  const int r = cl.block_rank(), n = cl.num_blocks();
  x[0][threadIdx.x] = 1.0 + threadIdx.x;
  x[1][threadIdx.x] = 0.0;
  cl.sync();
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  int cur = 0;
  for (int i = 0; i < iters; ++i) {
    const double* src = x[cur];
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      int j = (threadIdx.x * 7 + k * 131) & 1023;
      int owner = (remote_every && (threadIdx.x % remote_every) == 0 && k == 0) ? (r + 1) % n : r;
      double v = owner == r ? src[j] : *cl.map_shared_rank(src + j, owner);
      acc = fma(0.1, v, acc);
    }
    x[cur ^ 1][threadIdx.x] = acc / 3.0;
    cl.sync();
    cur ^= 1;
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int iters = 2000;
  for (int threads : {1024, 512, 256}) {
    for (int cl : {1, 2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(cl); cfg.blockDim = dim3(threads); cfg.attrs = at; cfg.numAttrs = 1;
      cudaFuncSetAttribute(k_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_sweep, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      unsigned long long h = 0, h2 = 0, h3 = 0;
      cudaLaunchKernelEx(&cfg, k_sync, iters, d); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      cudaLaunchKernelEx(&cfg, k_sweep, iters, 0, d); cudaMemcpy(&h2, d, 8, cudaMemcpyDeviceToHost);
      cudaLaunchKernelEx(&cfg, k_sweep, iters, 8, d); cudaMemcpy(&h3, d, 8, cudaMemcpyDeviceToHost);
      cudaError_t e = cudaGetLastError();
      printf("threads %4d CL %2d: sync %.3f us  sweep(local) %.3f us  sweep(1/8 remote) %.3f us %s\n",
             threads, cl, h / 1e3 / iters, h2 / 1e3 / iters, h3 / 1e3 / iters, e ? cudaGetErrorString(e) : "");
    }
  }
  return 0;
}
