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

// ---------------------------------------------------------------------------
// Device-side boundary data: the Greville samples of the
// incident Gaussian plane pulse u_in(x, t) = exp(-((t - z - t0) / sig)^2) at the
// centroids, written straight into the known-data buffers -- no host sampling,
// no H2D copy.  which = 0: Dirichlet datum u = -u_in; 1: Neumann datum
// q = -du_in/dn = -(n_z 2 a / sig) exp(-a^2).  Same expression as
// scenarios.PlanePulseData (values agree to the last bits of exp).
namespace tdw {
__global__ void plane_pulse_kernel(double* out, int nbeta, int ns, const double* __restrict__ zc,
                                   const double* __restrict__ nz, double dt, double off, double t0,
                                   double sig, int which) {
  const long long n = (long long)nbeta * ns;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int beta = (int)(e / ns), j = (int)(e % ns);
    const double t = (double)beta * dt + off;
    const double a = (t - zc[j] - t0) / sig;
    const double ex = exp(-a * a);
    out[e] = which == 0 ? -ex : -(nz[j] * 2.0 * a / sig * ex);
  }
}
}  // namespace tdw

extern "C" int tdw_known_plane_pulse(tdw_problem* pb, int which, const double* zc, const double* nz,
                                     double t0, double sig) {
  if (!pb || which < 0 || which > 1 || !zc || (which == 1 && !nz) || !(sig > 0.0)) return TDW_ERR_INVALID_ARG;
  tdw_ctx* ctx = pb->ctx;
  cudaSetDevice(ctx->device);
  const int ns = pb->ns, nb = pb->nt - 1;
  const size_t n = (size_t)nb * ns;
  double** dst = which == 0 ? &pb->d_uk : &pb->d_qk;
  if (!*dst) TDW_CUDA(ctx, cudaMalloc(dst, sizeof(double) * n));
  double *dz = nullptr, *dn = nullptr;
  TDW_CUDA(ctx, cudaMalloc(&dz, sizeof(double) * ns));
  TDW_CUDA(ctx, cudaMemcpyAsync(dz, zc, sizeof(double) * ns, cudaMemcpyHostToDevice, ctx->stream));
  if (nz) {
    TDW_CUDA(ctx, cudaMalloc(&dn, sizeof(double) * ns));
    TDW_CUDA(ctx, cudaMemcpyAsync(dn, nz, sizeof(double) * ns, cudaMemcpyHostToDevice, ctx->stream));
  }
  const double off = 0.5 * (pb->d + 1) * pb->dt;  // Greville abscissae (marching.py:264-266)
  tdw::plane_pulse_kernel<<<4 * ctx->num_sms, 256, 0, ctx->stream>>>(*dst, nb, ns, dz, dn, pb->dt, off, t0,
                                                                      sig, which);
  TDW_CUDA(ctx, cudaGetLastError());
  TDW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  cudaFree(dz);
  if (dn) cudaFree(dn);
  return TDW_OK;
}
