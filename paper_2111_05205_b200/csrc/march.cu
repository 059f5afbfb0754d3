// march.cu -- the marching-on-in-time loop on the device.
//
// Replaces the time loop of marching.march (marching.py:315-338):
//   K2 conv_kernel    b_i = sum_j sum_{gamma in band(i,j)} V_U q^{alpha-gamma} - V_W u^{alpha-gamma}
//                     (the reference's lag loop of CSR SpMVs over tau/sigma, :318-327,
//                     rewritten in kappa-combined form; the current step's KNOWN data
//                     enters through the gamma = 1 band entries, as the tilde sums do)
//   K3/K4 solve_kernel  b = sum of partials, Jacobi sweeps on A x = b (lu.solve, :330),
//                     residual test (:331-333), promotion of x into u/q (finalize_step,
//                     :239-242), blow-up detector (:336-338), next step's known data.
// History: hist[j][pad + beta] = (q_j^beta, u_j^beta) (element-major, time contiguous,
// zero padded for beta < 0), so a band reads consecutive slots of one element.
#include <cuda_runtime.h>
#include <nccl.h>

#include <climits>
#include <cstdio>

#include "tdw_impl.cuh"

namespace tdw {

#define FULLMASK 0xffffffffu

struct ConvArgs {
  const uint32_t* __restrict__ hdr;
  const unsigned long long* __restrict__ segoff;
  const double2* __restrict__ coef;
  const int2* __restrict__ unit;
  const double2* __restrict__ hist;
  double* __restrict__ bpart;
  const int* __restrict__ flags;
  int hstride, pad, ns, row_lo, rows_loc, ntiles, tiles_per_split, alpha;
};

// One CTA = one I-block of 32 rows (8 warps x 4 rows) x one split of the
// J-tiles.  Per J-tile the CTA stages the history slice of the tile's 32
// elements over the unit's lag range in shared memory, then every warp
// streams its rows' segments (coalesced 16 B per lane per k).
__global__ void __launch_bounds__(256, 2) conv_kernel(ConvArgs a) {
  extern __shared__ double2 hs[];
  if (a.flags[0] != 0) return;
  const int iblk = blockIdx.x, split = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = split * a.tiles_per_split;
  const int t1 = min(a.ntiles, t0 + a.tiles_per_split);
  double acc[TDW_ROWS_PER_WARP];
#pragma unroll
  for (int r = 0; r < TDW_ROWS_PER_WARP; ++r) acc[r] = 0.0;
  const int rbase = iblk * TDW_TI + warp * TDW_ROWS_PER_WARP;  // local row of acc[0]

  for (int t = t0; t < t1; ++t) {
    const int2 u = a.unit[iblk * a.ntiles + t];
    if (u.y < u.x) continue;  // uniform across the CTA
    const int W = u.y - u.x + 1;
    const int nstage = TDW_TJ * W;
    const int jbase = t * TDW_TJ;
    const int bq = a.pad + a.alpha - u.x;  // slot of gamma = gmin
    __syncthreads();
    for (int q = threadIdx.x; q < nstage; q += blockDim.x) {
      const int jl = q / W, w = q - jl * W;
      const int j = jbase + jl;
      hs[q] = j < a.ns ? a.hist[(size_t)j * a.hstride + (bq - w)] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < TDW_ROWS_PER_WARP; ++r) {
      const long long seg = (long long)(rbase + r) * a.ntiles + t;
      const uint32_t h = a.hdr[seg * TDW_TJ + lane];
      const int len = hdr_len(h);
      const int lmax = __shfl_sync(FULLMASK, len, 0);
      if (lmax == 0) continue;
      const double2* cp = a.coef + a.segoff[seg] + lane;
      const double2* hp = hs + hdr_jl(h) * W + (hdr_glo(h) - u.x);
      double s = 0.0;
      int off = 0;
      for (int k = 0; k < lmax; ++k) {
        const unsigned m = __ballot_sync(FULLMASK, len > k);
        if (len > k) {
          const double2 cv = __ldcs(cp + off);
          const double2 hv = hp[k];
          s = fma(cv.x, hv.x, s);
          s = fma(-cv.y, hv.y, s);
        }
        off += __popc(m);
      }
      acc[r] += s;
    }
  }
#pragma unroll
  for (int r = 0; r < TDW_ROWS_PER_WARP; ++r) {
    double v = acc[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
    if (lane == 0) a.bpart[(size_t)split * a.rows_loc + rbase + r] = v;
  }
}

// sum of the split partials of the own rows into b (multi-GPU path, before the all-gather)
__global__ void reduce_parts_kernel(const double* __restrict__ bpart, int nsplit, int rows_loc,
                                    double* __restrict__ bown, const int* flags) {
  if (flags[0] != 0) return;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows_loc; r += gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int s = 0; s < nsplit; ++s) v += bpart[(size_t)s * rows_loc + r];
    bown[r] = v;
  }
}

struct SolveArgs {
  const double* bpart;  // nsplit > 0: sum partials here (single GPU); else read b
  double* b;
  double* x;            // [2][ns]
  const int* __restrict__ acol;
  const double* __restrict__ aval;
  const double* __restrict__ adiag;
  int ell_w, iters;
  const double* __restrict__ phi;
  const int* __restrict__ perm;
  const double* __restrict__ uk;
  const double* __restrict__ qk;
  double2* hist;
  int hstride, pad;
  double* red;          // [3][gridDim]
  unsigned* bar;        // {count, generation}
  int* flags;           // {status, n_steps, err_step, -}
  double* rhs;          // optional (nt-1, ns) original order
  double threshold;
  int ns, nsplit, rows_loc, alpha, nt;
};

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    const unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ double block_reduce_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh[k];
  return t;  // valid in thread 0
}

__device__ __forceinline__ double block_reduce_max(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULLMASK, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t = fmax(t, sh[k]);
  return t;
}

// Cooperative (all CTAs co-resident) per-step solve + history update.
__global__ void __launch_bounds__(256) solve_kernel(SolveArgs a) {
  __shared__ double sh[32];
  if (*(volatile int*)&a.flags[0] != 0) return;  // every CTA sees the same flag
  const int nth = gridDim.x * blockDim.x;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int beta0 = a.alpha - 1;
  double* x0 = a.x;
  double* x1 = a.x + a.ns;
  // right-hand side (+ first Jacobi iterate)
  for (int i = tid; i < a.ns; i += nth) {
    double bi;
    if (a.nsplit > 0) {
      bi = 0.0;
      for (int s = 0; s < a.nsplit; ++s) bi += a.bpart[(size_t)s * a.rows_loc + i];
      a.b[i] = bi;
    } else {
      bi = __ldcg(a.b + i);
    }
    x0[i] = bi / a.adiag[i];
    if (a.rhs) a.rhs[(size_t)beta0 * a.ns + a.perm[i]] = bi;
  }
  grid_barrier(a.bar, gridDim.x);
  // Jacobi sweeps (strictly diagonally dominant A, bound < 0.9 checked at assembly)
  for (int it = 0; it < a.iters; ++it) {
    const double* xin = (it & 1) ? x1 : x0;
    double* xout = (it & 1) ? x0 : x1;
    for (int i = tid; i < a.ns; i += nth) {
      double acc = __ldcg(a.b + i);
      for (int k = 0; k < a.ell_w; ++k) {
        const int j = a.acol[(size_t)k * a.ns + i];
        if (j != i) acc -= a.aval[(size_t)k * a.ns + i] * __ldcg(xin + j);
      }
      xout[i] = acc / a.adiag[i];
    }
    grid_barrier(a.bar, gridDim.x);
  }
  const double* xf = (a.iters & 1) ? x1 : x0;
  // residual and blow-up reductions
  double r2 = 0.0, b2 = 0.0, xm = 0.0;
  for (int i = tid; i < a.ns; i += nth) {
    const double bi = __ldcg(a.b + i);
    double acc = -bi;
    for (int k = 0; k < a.ell_w; ++k)
      acc += a.aval[(size_t)k * a.ns + i] * __ldcg(xf + a.acol[(size_t)k * a.ns + i]);
    r2 += acc * acc;
    b2 += bi * bi;
    xm = fmax(xm, fabs(__ldcg(xf + i)));
  }
  r2 = block_reduce_sum(r2, sh);
  b2 = block_reduce_sum(b2, sh);
  xm = block_reduce_max(xm, sh);
  if (threadIdx.x == 0) {
    a.red[blockIdx.x] = r2;
    a.red[gridDim.x + blockIdx.x] = b2;
    a.red[2 * gridDim.x + blockIdx.x] = xm;
  }
  grid_barrier(a.bar, gridDim.x);
  __shared__ int s_bad;
  __shared__ double s_xmax;
  if (threadIdx.x == 0) {
    double R = 0.0, B = 0.0, X = 0.0;
    for (int k = 0; k < (int)gridDim.x; ++k) {
      R += __ldcg(a.red + k);
      B += __ldcg(a.red + gridDim.x + k);
      X = fmax(X, __ldcg(a.red + 2 * gridDim.x + k));
    }
    s_bad = sqrt(R) > 1e-10 * fmax(sqrt(B), 1e-300);
    s_xmax = X;
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) {
      a.flags[2] = a.alpha;
      atomicExch(&a.flags[0], 2);  // residual failure: the reference raises here
    }
    return;
  }
  // finalize_step: promote x into u/q by phi, then the next step's known part
  for (int j = tid; j < a.ns; j += nth) {
    const int o = a.perm[j];
    const double xj = __ldcg(xf + j);
    const double ph = a.phi[j];
    const size_t kb = (size_t)beta0 * a.ns + o;
    const double qv = ph == 1.0 ? a.qk[kb] : xj;
    const double uv = ph == 1.0 ? xj : a.uk[kb];
    a.hist[(size_t)j * a.hstride + a.pad + beta0] = make_double2(qv, uv);
    if (beta0 + 1 < a.nt - 1 && !(s_xmax > a.threshold)) {
      const size_t kn = (size_t)(beta0 + 1) * a.ns + o;
      a.hist[(size_t)j * a.hstride + a.pad + beta0 + 1] =
          make_double2(ph * a.qk[kn], (1.0 - ph) * a.uk[kn]);
    }
  }
  if (tid == 0) {
    a.flags[1] = a.alpha;
    if (s_xmax > a.threshold) atomicExch(&a.flags[0], 1);  // "unstable"
  }
}

// hist[j][pad + 0] = known part of step beta = 0 (the loop writes the later ones)
__global__ void init_hist_kernel(double2* hist, int hstride, int pad, int ns, int nt,
                                 const double* phi, const int* perm, const double* uk,
                                 const double* qk) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ns; j += gridDim.x * blockDim.x) {
    double2* h = hist + (size_t)j * hstride;
    for (int s = 0; s < hstride; ++s) h[s] = make_double2(0.0, 0.0);
    const int o = perm[j];
    const double ph = phi[j];
    h[pad] = make_double2(ph * qk[o], (1.0 - ph) * uk[o]);
  }
}

// (nt-1, ns) outputs in the original element order; kappa sums as stock_sums
// (marching.py:205-214); rows at and after n_steps stay zero.
__global__ void outputs_kernel(const double2* hist, int hstride, int pad, int ns, int nt, int d,
                               const int* perm, const int* flags, double* u, double* q,
                               double* tau, double* sig) {
  const int nsteps = flags[1];
  double w[5] = {0, 0, 0, 0, 0};
  if (d == 1) { w[0] = 1.0; w[1] = -2.0; w[2] = 1.0; }
  if (d == 2) { w[0] = 0.5; w[1] = -1.5; w[2] = 1.5; w[3] = -0.5; }
  if (d == 3) { w[0] = 1.0 / 6.0; w[1] = -(2.0 / 3.0); w[2] = 1.0; w[3] = -(2.0 / 3.0); w[4] = 1.0 / 6.0; }
  const long long n = (long long)(nt - 1) * ns;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int beta = (int)(e / ns), j = (int)(e % ns);
    const size_t o = (size_t)beta * ns + perm[j];
    if (beta >= nsteps) {
      if (u) u[o] = 0.0;
      if (q) q[o] = 0.0;
      if (tau) tau[o] = 0.0;
      if (sig) sig[o] = 0.0;
      continue;
    }
    const double2* h = hist + (size_t)j * hstride + pad;
    if (q) q[o] = h[beta].x;
    if (u) u[o] = h[beta].y;
    if (tau || sig) {
      double ta = 0.0, sa = 0.0;
      const int kmax = min(d + 1, beta);
      for (int k = 0; k <= kmax; ++k) {
        ta += w[k] * h[beta - k].x;
        sa += w[k] * h[beta - k].y;
      }
      if (tau) tau[o] = ta;
      if (sig) sig[o] = sa;
    }
  }
}

}  // namespace tdw

using namespace tdw;

static int launch_solve(tdw_problem* pb, SolveArgs& s) {
  void* args[] = {&s};
  TDW_CUDA(pb->ctx, cudaLaunchCooperativeKernel((const void*)solve_kernel, pb->solve_grid, 256,
                                                args, 0, pb->ctx->stream));
  return TDW_OK;
}

int tdw_march_loop(tdw_problem* pb, double threshold, bool want_rhs, bool time_kernels,
                   tdw_timing* timing) {
  tdw_ctx* ctx = pb->ctx;
  cudaStream_t st = ctx->stream;
  if (!pb->assembled) return tdw_fail(ctx, TDW_ERR_STATE, "tdw_march before tdw_assemble");
  if (!pb->known_loaded) return tdw_fail(ctx, TDW_ERR_STATE, "known boundary data not uploaded");
  if (want_rhs) {
    if (!pb->d_rhs)
      TDW_CUDA(ctx, cudaMalloc(&pb->d_rhs, sizeof(double) * (size_t)(pb->nt - 1) * pb->ns));
    TDW_CUDA(ctx, cudaMemsetAsync(pb->d_rhs, 0, sizeof(double) * (size_t)(pb->nt - 1) * pb->ns, st));
  }
  TDW_CUDA(ctx, cudaMemsetAsync(pb->d_flags, 0, sizeof(int) * 4, st));
  TDW_CUDA(ctx, cudaMemsetAsync(pb->d_bar, 0, sizeof(unsigned) * 2, st));
  init_hist_kernel<<<(pb->ns + 255) / 256, 256, 0, st>>>(pb->d_hist, pb->hstride, pb->pad, pb->ns,
                                                         pb->nt, pb->d_phi, pb->d_perm, pb->d_uk,
                                                         pb->d_qk);
  TDW_CUDA(ctx, cudaGetLastError());

  ConvArgs c{};
  c.hdr = pb->d_hdr;
  c.segoff = pb->d_segoff;
  c.coef = pb->d_coef;
  c.unit = pb->d_unit;
  c.hist = pb->d_hist;
  c.bpart = pb->d_bpart;
  c.flags = pb->d_flags;
  c.hstride = pb->hstride;
  c.pad = pb->pad;
  c.ns = pb->ns;
  c.row_lo = pb->row_lo;
  c.rows_loc = pb->rows_per_rank;
  c.ntiles = pb->ntiles;
  c.tiles_per_split = (pb->ntiles + pb->nsplit - 1) / pb->nsplit;
  const size_t smem = sizeof(double2) * TDW_TJ * pb->wmax;
  TDW_CUDA(ctx, cudaFuncSetAttribute(conv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  dim3 cgrid(pb->n_iblk, pb->nsplit);

  SolveArgs s{};
  const bool multi = pb->nranks > 1;
  s.bpart = pb->d_bpart;
  s.b = pb->d_b;
  s.x = pb->d_x;
  s.acol = pb->d_acol;
  s.aval = pb->d_aval;
  s.adiag = pb->d_adiag;
  s.ell_w = pb->ell_w;
  s.iters = pb->jac_iters;
  s.phi = pb->d_phi;
  s.perm = pb->d_perm;
  s.uk = pb->d_uk;
  s.qk = pb->d_qk;
  s.hist = pb->d_hist;
  s.hstride = pb->hstride;
  s.pad = pb->pad;
  s.red = pb->d_red;
  s.bar = pb->d_bar;
  s.flags = pb->d_flags;
  s.rhs = want_rhs ? pb->d_rhs : nullptr;
  s.threshold = threshold;
  s.ns = pb->ns;
  s.nsplit = multi ? 0 : pb->nsplit;
  s.rows_loc = pb->rows_per_rank;
  s.nt = pb->nt;

  cudaEvent_t ev_all0, ev_all1;
  TDW_CUDA(ctx, cudaEventCreate(&ev_all0));
  TDW_CUDA(ctx, cudaEventCreate(&ev_all1));
  std::vector<cudaEvent_t> evs;
  if (time_kernels) {
    evs.resize(6 * (size_t)(pb->nt - 1));
    for (auto& e : evs) TDW_CUDA(ctx, cudaEventCreate(&e));
  }
  TDW_CUDA(ctx, cudaEventRecord(ev_all0, st));
  for (int alpha = 1; alpha < pb->nt; ++alpha) {
    c.alpha = alpha;
    s.alpha = alpha;
    cudaEvent_t* E = time_kernels ? &evs[6 * (size_t)(alpha - 1)] : nullptr;
    if (E) cudaEventRecord(E[0], st);
    conv_kernel<<<cgrid, 256, smem, st>>>(c);
    if (E) cudaEventRecord(E[1], st);
    if (multi) {
      reduce_parts_kernel<<<(pb->rows_per_rank + 255) / 256, 256, 0, st>>>(
          pb->d_bpart, pb->nsplit, pb->rows_per_rank, pb->d_b + pb->row_lo, pb->d_flags);
      if (E) cudaEventRecord(E[2], st);
      ncclResult_t nr = ncclAllGather(pb->d_b + pb->row_lo, pb->d_b, (size_t)pb->rows_per_rank,
                                      ncclDouble, ctx->comm, st);
      if (nr != ncclSuccess)
        return tdw_fail(ctx, TDW_ERR_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(nr));
      if (E) cudaEventRecord(E[3], st);
    }
    if (E) cudaEventRecord(E[4], st);
    int rc = launch_solve(pb, s);
    if (rc) return rc;
    if (E) cudaEventRecord(E[5], st);
  }
  TDW_CUDA(ctx, cudaGetLastError());
  TDW_CUDA(ctx, cudaEventRecord(ev_all1, st));
  TDW_CUDA(ctx, cudaEventSynchronize(ev_all1));
  if (timing) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev_all0, ev_all1);
    timing->total_ms += ms;
    timing->steps += pb->nt - 1;
    if (time_kernels) {
      for (int k = 0; k < pb->nt - 1; ++k) {
        cudaEvent_t* E = &evs[6 * (size_t)k];
        float a = 0.f;
        cudaEventElapsedTime(&a, E[0], E[1]);
        timing->conv_ms += a;
        timing->conv_launches += 1;
        cudaEventElapsedTime(&a, E[4], E[5]);
        timing->solve_ms += a;
        if (multi) {
          cudaEventElapsedTime(&a, E[2], E[3]);
          timing->comm_ms += a;
        }
      }
    }
  }
  for (auto& e : evs) cudaEventDestroy(e);
  cudaEventDestroy(ev_all0);
  cudaEventDestroy(ev_all1);
  int hflags[4];
  TDW_CUDA(ctx, cudaMemcpy(hflags, pb->d_flags, sizeof(hflags), cudaMemcpyDeviceToHost));
  if (hflags[0] == 2) {
    char msg[128];
    snprintf(msg, sizeof(msg), "step %d: solve residual too large", hflags[2]);
    return tdw_fail(ctx, TDW_ERR_RESIDUAL, msg);
  }
  return TDW_OK;
}

int tdw_outputs(tdw_problem* pb, double* u, double* q, double* tau, double* sigma) {
  tdw_ctx* ctx = pb->ctx;
  cudaStream_t st = ctx->stream;
  const size_t n = (size_t)(pb->nt - 1) * pb->ns;
  double* buf = nullptr;
  TDW_CUDA(ctx, cudaMallocAsync((void**)&buf, sizeof(double) * 4 * n, st));
  outputs_kernel<<<1024, 256, 0, st>>>(pb->d_hist, pb->hstride, pb->pad, pb->ns, pb->nt, pb->d,
                                        pb->d_perm, pb->d_flags, buf, buf + n, buf + 2 * n,
                                        buf + 3 * n);
  TDW_CUDA(ctx, cudaGetLastError());
  double* outs[4] = {u, q, tau, sigma};
  for (int k = 0; k < 4; ++k)
    if (outs[k])
      TDW_CUDA(ctx, cudaMemcpyAsync(outs[k], buf + k * n, sizeof(double) * n,
                                    cudaMemcpyDeviceToHost, st));
  TDW_CUDA(ctx, cudaFreeAsync(buf, st));
  TDW_CUDA(ctx, cudaStreamSynchronize(st));
  return TDW_OK;
}
