// diag.cu -- device measurements the benchmark reports beside its own numbers.
//
// tdw_fp64_peak: FP64 FMA throughput of this GPU at its current clocks, the
// denominator of the coefficient kernel's (K1) roofline (the FP64
// peak is not in MEASURED_PEAKS.json).  Every thread runs 8 independent DFMA
// chains; the grid covers every SM several times over.  No reference
// counterpart (the reference has no device path).
#include <cuda_runtime.h>

#include "tdw.h"
#include "tdw_impl.cuh"

namespace tdw {

__global__ void __launch_bounds__(256) fp64_fma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = (double)(threadIdx.x + k) * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keeps the chains live
}

}  // namespace tdw

extern "C" int tdw_fp64_peak(tdw_ctx* ctx, double* tflops) {
  if (!ctx || !tflops) return TDW_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  double* d = nullptr;
  TDW_CUDA(ctx, cudaMalloc(&d, sizeof(double)));
  const int blocks = ctx->num_sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  TDW_CUDA(ctx, cudaEventCreate(&e0));
  TDW_CUDA(ctx, cudaEventCreate(&e1));
  tdw::fp64_fma_kernel<<<blocks, threads, 0, st>>>(d, iters, 0.999999, 1e-9);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    TDW_CUDA(ctx, cudaEventRecord(e0, st));
    tdw::fp64_fma_kernel<<<blocks, threads, 0, st>>>(d, iters, 0.999999, 1e-9);
    TDW_CUDA(ctx, cudaEventRecord(e1, st));
    TDW_CUDA(ctx, cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  TDW_CUDA(ctx, cudaGetLastError());
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  const double flop = 2.0 * 8.0 * (double)iters * (double)blocks * threads;
  *tflops = flop / (best * 1e-3) / 1e12;
  return TDW_OK;
}
