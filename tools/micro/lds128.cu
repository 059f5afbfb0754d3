// Microbenchmark: shared-memory cycles per warp-wide LDS.128 for the address
// patterns the convolution's consumers could use (one CTA per SM, 8 warps,
// 8 independent loads in flight per warp).  Prints cycles per LDS per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o lds128 lds128.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 lds(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}

__global__ void __launch_bounds__(256, 1) k(int pattern, int iters, long long* cyc, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) ((double*)sm)[i] = 1.0 + i;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned base = (unsigned)__cvta_generic_to_shared(sm) + warp * 4096;
  unsigned off;
  switch (pattern) {
    case 0: off = lane * 16; break;                      // 32 distinct consecutive (512 B)
    case 1: off = 0; break;                              // all lanes one address
    case 2: off = (lane & 7) * 16; break;                // 8 distinct, every quarter-warp covers all 8
    case 3: off = (lane >> 2) * 16; break;               // 8 distinct in 128 B, 2 per quarter-warp
    case 4: off = ((lane * 5 + 3) & 7) * 16; break;      // 8 distinct in 128 B, scrambled
    case 5: off = lane < 16 ? lane * 16 : 2048; break;   // half the lanes consecutive, half one far address
    case 6: off = ((lane * 7 + 1) & 15) * 16; break;     // 16 distinct in 256 B, scrambled
    case 7: off = (lane >> 1) * 16; break;               // 16 distinct in 256 B, pairs
    case 8: off = (lane & 7) * 16 + (lane >> 3) * 512; break;  // 4 groups of 128 B in different rows (4 cols x 8 times)
    case 9: off = (lane & 3) * 16 + (lane >> 2) * 512 + (lane >> 2) * 16; break;  // 8 rows, 4 consecutive each
    case 10: off = ((lane * 3) & 31) * 48; break;        // 48-byte stride (scattered)
    default: off = (lane & 15) * 16 + (lane >> 4) * 1024; break;  // 2 groups of 256 B
  }
  double2 acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = make_double2(0, 0);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      double2 v = lds(base + off + ((it + q) & 3) * 16 * 0);
      acc[q].x += v.x;
      acc[q].y += v.y;
    }
  }
  long long t1 = clock64();
  __syncthreads();
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += acc[q].x + acc[q].y;
  if (s == 12345.678) sink[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  long long* d;
  double* sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 4000;
  for (int p = 0; p <= 11; ++p) {
    k<<<148, 256, 65536>>>(p, iters, d, sink);
    long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    // 8 warps x 8 loads per iteration per SM
    printf("pattern %2d: %.2f cycles per warp LDS.128 (SM-wide)\n", p, (double)h / (iters * 64.0));
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
