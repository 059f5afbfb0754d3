// coeff_table.cu -- K1 as a table: one (point, triangle, s) triple per thread.
// C-ABI image of elemint.retarded_coeff_table (elemint.py:89-186); also the
// kernel behind the "(i,j,gamma) layer-potential evals/s" metric.
#include <cuda_runtime.h>

#include "coeff.cuh"
#include "tdw_impl.cuh"

namespace tdw {

template <int D, bool BM>
__global__ void __launch_bounds__(128) coeff_table_kernel(int64_t n, const double* __restrict__ P,
                                                          const double* __restrict__ A,
                                                          const double* __restrict__ B,
                                                          const double* __restrict__ C,
                                                          const double* __restrict__ ez,
                                                          const double* __restrict__ s,
                                                          const double* __restrict__ nx, double K,
                                                          double* __restrict__ out0,
                                                          double* __restrict__ out1) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    double p[3], a[3], b[3], c[3], e[3], q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      p[k] = P[3 * t + k];
      a[k] = A[3 * t + k];
      b[k] = B[3 * t + k];
      c[k] = C[3 * t + k];
      e[k] = ez[3 * t + k];
      q[k] = BM ? nx[3 * t + k] : 0.0;
    }
    PairGeom g;
    pair_geom<BM>(p, a, b, c, e, q, g);
    double o0, o1;
    coeff_eval<D, BM>(g, s[t], K, o0, o1);
    out0[t] = o0;
    out1[t] = o1;
  }
}

static int launch_table(tdw_ctx* ctx, int64_t n, const double* P, const double* A,
                        const double* B, const double* C, const double* ez, const double* s,
                        int d, double c, double dt, int kind, const double* nx, double* o0,
                        double* o1) {
  if (n <= 0) return TDW_OK;
  const double K = kfactor(d, c, dt);
  const int threads = 128;
  int64_t want = (n + threads - 1) / threads;
  int blocks = (int)(want < 148LL * 64 ? want : 148LL * 64);
#define TDW_L(DD, BB)                                                                  \
  coeff_table_kernel<DD, BB><<<blocks, threads, 0, ctx->stream>>>(n, P, A, B, C, ez, s, \
                                                                  nx, K, o0, o1)
  if (kind == TDW_KIND_UW) {
    if (d == 1) TDW_L(1, false);
    if (d == 2) TDW_L(2, false);
    if (d == 3) TDW_L(3, false);
  } else {
    if (d == 1) TDW_L(1, true);
    if (d == 2) TDW_L(2, true);
    if (d == 3) TDW_L(3, true);
  }
#undef TDW_L
  TDW_CUDA(ctx, cudaGetLastError());
  return TDW_OK;
}

static int check_args(tdw_ctx* ctx, int d, int kind, const double* nx) {
  if (d < 1 || d > 3)
    return tdw_fail(ctx, TDW_ERR_UNSUPPORTED_ORDER,
                    "basis order d=" + std::to_string(d) +
                        " not supported by the closed forms (d in 1..3)");
  if (kind != TDW_KIND_UW && kind != TDW_KIND_BM)
    return tdw_fail(ctx, TDW_ERR_INVALID_ARG, "unknown coefficient kind");
  if (kind == TDW_KIND_BM && nx == nullptr)
    return tdw_fail(ctx, TDW_ERR_INVALID_ARG, "bm coefficients need the collocation normal nx");
  return TDW_OK;
}

}  // namespace tdw

extern "C" int tdw_coeff_table_device(tdw_ctx* ctx, int64_t n, const double* P, const double* A,
                                      const double* B, const double* C, const double* ez,
                                      const double* s, int d, double c, double dt, int kind,
                                      const double* nx, double* out0, double* out1, float* ms) {
  if (!ctx) return TDW_ERR_INVALID_ARG;
  int rc = tdw::check_args(ctx, d, kind, nx);
  if (rc) return rc;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ms) {
    TDW_CUDA(ctx, cudaEventCreate(&e0));
    TDW_CUDA(ctx, cudaEventCreate(&e1));
    TDW_CUDA(ctx, cudaEventRecord(e0, ctx->stream));
  }
  rc = tdw::launch_table(ctx, n, P, A, B, C, ez, s, d, c, dt, kind, nx, out0, out1);
  if (rc) return rc;
  if (ms) {
    TDW_CUDA(ctx, cudaEventRecord(e1, ctx->stream));
    TDW_CUDA(ctx, cudaEventSynchronize(e1));
    TDW_CUDA(ctx, cudaEventElapsedTime(ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return TDW_OK;
}

extern "C" int tdw_coeff_table(tdw_ctx* ctx, int64_t n, const double* P, const double* A,
                               const double* B, const double* C, const double* ez,
                               const double* s, int d, double c, double dt, int kind,
                               const double* nx, double* out0, double* out1) {
  if (!ctx) return TDW_ERR_INVALID_ARG;
  int rc = tdw::check_args(ctx, d, kind, nx);
  if (rc) return rc;
  if (n <= 0) return TDW_OK;
  const size_t v3 = sizeof(double) * 3 * (size_t)n, v1 = sizeof(double) * (size_t)n;
  const int narr = kind == TDW_KIND_BM ? 6 : 5;
  char* buf = nullptr;
  size_t total = narr * v3 + 3 * v1;
  TDW_CUDA(ctx, cudaMallocAsync((void**)&buf, total, ctx->stream));
  double* dP = (double*)buf;
  double* dA = (double*)(buf + v3);
  double* dB = (double*)(buf + 2 * v3);
  double* dC = (double*)(buf + 3 * v3);
  double* dE = (double*)(buf + 4 * v3);
  double* dN = kind == TDW_KIND_BM ? (double*)(buf + 5 * v3) : nullptr;
  double* dS = (double*)(buf + narr * v3);
  double* d0 = (double*)(buf + narr * v3 + v1);
  double* d1 = (double*)(buf + narr * v3 + 2 * v1);
  cudaStream_t st = ctx->stream;
  TDW_CUDA(ctx, cudaMemcpyAsync(dP, P, v3, cudaMemcpyHostToDevice, st));
  TDW_CUDA(ctx, cudaMemcpyAsync(dA, A, v3, cudaMemcpyHostToDevice, st));
  TDW_CUDA(ctx, cudaMemcpyAsync(dB, B, v3, cudaMemcpyHostToDevice, st));
  TDW_CUDA(ctx, cudaMemcpyAsync(dC, C, v3, cudaMemcpyHostToDevice, st));
  TDW_CUDA(ctx, cudaMemcpyAsync(dE, ez, v3, cudaMemcpyHostToDevice, st));
  if (dN) TDW_CUDA(ctx, cudaMemcpyAsync(dN, nx, v3, cudaMemcpyHostToDevice, st));
  TDW_CUDA(ctx, cudaMemcpyAsync(dS, s, v1, cudaMemcpyHostToDevice, st));
  rc = tdw::launch_table(ctx, n, dP, dA, dB, dC, dE, dS, d, c, dt, kind, dN, d0, d1);
  if (rc) return rc;
  TDW_CUDA(ctx, cudaMemcpyAsync(out0, d0, v1, cudaMemcpyDeviceToHost, st));
  TDW_CUDA(ctx, cudaMemcpyAsync(out1, d1, v1, cudaMemcpyDeviceToHost, st));
  TDW_CUDA(ctx, cudaFreeAsync(buf, st));
  TDW_CUDA(ctx, cudaStreamSynchronize(st));
  return TDW_OK;
}
