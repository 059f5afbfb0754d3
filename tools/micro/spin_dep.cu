// Microbenchmark / repro: a kernel on stream A spins until a kernel on stream B
// (launched later, from another host thread) raises a flag.  Variants: dynamic
// shared memory of the spinner, priority of stream B, a memset before the flag kernel.
#include <cstdio>
#include <thread>
#include <chrono>
#include <cuda_runtime.h>
__global__ void spin(const int* ready, int* out) {
  extern __shared__ unsigned char sm[];
  if (threadIdx.x == 0) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      int v;
      asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ready) : "memory");
      if (v >= 1) { out[blockIdx.x] = 1; break; }
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 1000000000ull) { out[blockIdx.x] = -1; break; }
      __nanosleep(500);
    }
  }
  __syncthreads();
}
__global__ void raise(int* ready) { asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(ready), "r"(1) : "memory"); }
__global__ void work(double* p, int n) { for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = 1.0; }
int main() {
  int *ready, *out; double* buf;
  cudaMalloc(&ready, 4); cudaMalloc(&out, 4 * 148); cudaMalloc(&buf, 8 << 20);
  cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
  int lo, hi; cudaDeviceGetStreamPriorityRange(&lo, &hi);
  {  // warm-up: load every kernel before anything spins (lazy module loading)
    cudaMemset(ready, 0, 4);
    work<<<1, 32>>>(buf, 32); raise<<<1, 1>>>(ready); spin<<<1, 32>>>(ready, out); cudaMemsetAsync(buf, 0, 64, 0);
    printf("warm-up: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  }
  for (int variant = 0; variant < 8; ++variant) {
    const size_t smem = (variant & 1) ? 224 * 1024 : 0;
    const int prio = (variant & 2) ? hi : lo;
    const bool memset_first = variant & 4;
    cudaStream_t a, b;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithPriority(&b, cudaStreamNonBlocking, prio);
    cudaMemset(ready, 0, 4); cudaMemset(out, 0, 4 * 148);
    spin<<<132, 544, smem, a>>>(ready, out);
    std::thread t([&] {
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
      if (memset_first) cudaMemsetAsync(buf, 0, 8 << 20, b);
      work<<<64, 256, 0, b>>>(buf, 1 << 20);
      raise<<<1, 1, 0, b>>>(ready);
    });
    t.join();
    cudaDeviceSynchronize();
    int h[148]; cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    int ok = 0, to = 0; for (int i = 0; i < 132; ++i) { ok += h[i] == 1; to += h[i] == -1; }
    printf("variant %d (smem %zu KB, prio %s, memset %d): %d CTAs released, %d timed out, %s\n", variant, smem >> 10,
           prio == hi ? "high" : "low", (int)memset_first, ok, to, cudaGetErrorString(cudaGetLastError()));
    cudaStreamDestroy(a); cudaStreamDestroy(b);
  }
  return 0;
}
