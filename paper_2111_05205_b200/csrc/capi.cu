// capi.cu -- C ABI of libtdw: context, problem lifetime, march drivers, NCCL.
// See include/tdw.h for the reference interface each entry point replaces.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include "coeff.cuh"
#include "tdw_impl.cuh"

int tdw_fail(tdw_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

namespace {

// max squared distance between used vertices (mesh.py:85-96), on the device
__global__ void diameter_kernel(const double* __restrict__ v, const int* __restrict__ used, int nu,
                                unsigned long long* out) {
  double best = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)nu * nu;
       e += (long long)gridDim.x * blockDim.x) {
    const int a = used[e / nu], b = used[e % nu];
    const double dx = v[3 * a] - v[3 * b], dy = v[3 * a + 1] - v[3 * b + 1],
                 dz = v[3 * a + 2] - v[3 * b + 2];
    best = fmax(best, dx * dx + dy * dy + dz * dz);
  }
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(best));
}

}  // namespace

extern "C" {

int tdw_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int tdw_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes <= 0) return TDW_ERR_INVALID_ARG;
  *out = nullptr;
  // mapped: the streamed march reads the known-data samples in place
  return cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable | cudaHostAllocMapped) == cudaSuccess
             ? TDW_OK : TDW_ERR_CUDA;
}

int tdw_host_free(void* p) {
  if (!p) return TDW_OK;
  return cudaFreeHost(p) == cudaSuccess ? TDW_OK : TDW_ERR_CUDA;
}

int tdw_init(int device, tdw_ctx** out) {
  if (!out) return TDW_ERR_INVALID_ARG;
  *out = nullptr;
  tdw_ctx* ctx = new tdw_ctx();
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  // the library stream (solves, near terms) at the highest priority: when an SM
  // frees up, a pending solve cluster is placed before more convolution or
  // near-term blocks (the time loop's critical path runs on this stream)
  int prio_lo = 0, prio_hi = 0;
  if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  const char* pe = getenv("TDW_PRIO");  // experiments: 0 = default priority
  if (e == cudaSuccess)
    e = cudaStreamCreateWithPriority(&ctx->stream, cudaStreamNonBlocking, (pe && atoi(pe) == 0) ? prio_lo : prio_hi);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) {
    delete ctx;
    return TDW_ERR_CUDA;
  }
  *out = ctx;
  return TDW_OK;
}

int tdw_finalize(tdw_ctx* ctx) {
  if (!ctx) return TDW_OK;
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return TDW_OK;
}

const char* tdw_last_error(const tdw_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int tdw_nccl_unique_id(char out[128]) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return TDW_ERR_NCCL;
  memcpy(out, id.internal, 128);
  return TDW_OK;
}

int tdw_comm_init(tdw_ctx* ctx, const char id[128], int nranks, int rank) {
  if (!ctx || nranks < 1 || rank < 0 || rank >= nranks) return TDW_ERR_INVALID_ARG;
  if (ctx->comm) return tdw_fail(ctx, TDW_ERR_STATE, "tdw_comm_init: communicator already set");
  // nranks == 1 also creates a (one-rank) communicator: the march then takes the
  // exchange path, all-gather included, which lets a single GPU exercise it
  ncclUniqueId uid;
  memcpy(uid.internal, id, 128);
  cudaSetDevice(ctx->device);
  ncclResult_t r = ncclCommInitRank(&ctx->comm, nranks, uid, rank);
  if (r != ncclSuccess) return tdw_fail(ctx, TDW_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  ctx->nranks = nranks;
  ctx->rank = rank;
  return TDW_OK;
}

int tdw_problem_create(tdw_ctx* ctx, const tdw_problem_desc* dsc, tdw_problem** out) {
  return tdw_problem_create_impl(ctx, dsc, out, false);
}

int tdw_problem_create_shard(tdw_ctx* ctx, const tdw_problem_desc* dsc, tdw_problem** out) {
  return tdw_problem_create_impl(ctx, dsc, out, true);
}

int tdw_march_emulated(tdw_problem** pbs, int n, double threshold) {
  if (!pbs || n < 1) return TDW_ERR_INVALID_ARG;
  for (int r = 0; r < n; ++r)
    if (!pbs[r] || pbs[r]->nranks != n || pbs[r]->rank != r || pbs[r]->ctx != pbs[0]->ctx)
      return TDW_ERR_INVALID_ARG;
  cudaSetDevice(pbs[0]->ctx->device);
  return tdw_march_emulated_impl(pbs, n, threshold);
}

}  // extern "C"

int tdw_problem_create_impl(tdw_ctx* ctx, const tdw_problem_desc* dsc, tdw_problem** out,
                            bool shard_only) {
  if (!ctx || !dsc || !out) return TDW_ERR_INVALID_ARG;
  *out = nullptr;
  if (dsc->d < 1 || dsc->d > 3)
    return tdw_fail(ctx, TDW_ERR_UNSUPPORTED_ORDER, "basis order must be 1..3");
  if (dsc->bie != TDW_BIE_OBIE && dsc->bie != TDW_BIE_BMBIE)
    return tdw_fail(ctx, TDW_ERR_INVALID_ARG, "unknown integral equation");
  if (dsc->nt < 2) return tdw_fail(ctx, TDW_ERR_INVALID_ARG, "need at least two time steps");
  if (dsc->ns < 1 || dsc->nv < 3 || !dsc->vertices || !dsc->triangles || !dsc->phi)
    return tdw_fail(ctx, TDW_ERR_INVALID_ARG, "empty mesh");
  if (!(dsc->dt > 0.0) || !(dsc->c > 0.0))
    return tdw_fail(ctx, TDW_ERR_INVALID_ARG, "c and dt must be positive");
  const int nranks = std::max(1, dsc->nranks), rank = dsc->rank;
  if (rank < 0 || rank >= nranks) return tdw_fail(ctx, TDW_ERR_INVALID_ARG, "rank out of range");
  if (!shard_only && (nranks != ctx->nranks || rank != ctx->rank))
    return tdw_fail(ctx, TDW_ERR_INVALID_ARG, "nranks/rank differ from tdw_comm_init");
  cudaSetDevice(ctx->device);
  tdw_problem* pb = new tdw_problem();
  pb->ctx = ctx;
  const int ns = dsc->ns, nv = dsc->nv;
  pb->ns = ns;
  pb->nv = nv;
  pb->bie = dsc->bie;
  pb->d = dsc->d;
  pb->nt = dsc->nt;
  pb->window = dsc->window ? 1 : 0;
  if (dsc->mode < TDW_MODE_AUTO || dsc->mode > TDW_MODE_ON_THE_FLY) {
    delete pb;
    return tdw_fail(ctx, TDW_ERR_INVALID_ARG, "unknown coefficient mode");
  }
  pb->mode = dsc->mode;
  {
    // temporal blocking: one convolution pass computes kb consecutive steps
    // default 4; 5 / 6 as a pass (~ ns^2 / ranks band entries) outweighs the solves
    // (~ ns).  Measured: config 0 (320 el.) best at 4, config 1 even, config 2
    // (5120) 15.5k steps/s at 5 (14.7k at 6, 13.5k at 4), config 3 (20480) 911 at 6
    // (811 at 5, 737 at 4)
    // (a function of the whole problem, not of the rank count: kb and the split
    // lags decide how each b_i is grouped into sums, so any rank count gives the
    // single-GPU densities bit for bit)
    const char* e = getenv("TDW_KB");
    const double pass_size = (double)dsc->ns * (double)dsc->ns;
    const int kb_default = pass_size >= 1e8 ? 6 : (pass_size >= 1e7 ? 5 : 4);
    pb->kb = std::max(1, std::min(TDW_KB_MAX, e ? atoi(e) : kb_default));
    // a pass waits for the solve overlap+1 steps back and runs beside the last
    // `overlap` solves; the split lags reach kb + overlap
    const char* o = getenv("TDW_OVERLAP");
    pb->overlap = std::max(1, std::min(pb->kb, o ? atoi(o) : pb->kb));
    pb->nsl = pb->kb + pb->overlap - 1;
    pb->bring = pb->kb + pb->overlap;
  }
  pb->c = dsc->c;
  pb->dt = dsc->dt;
  pb->K = tdw::kfactor(pb->d, pb->c, pb->dt);
  pb->nranks = nranks;
  pb->rank = rank;

  // mesh-derived quantities exactly as mesh.py:42-75 (host, O(ns))
  std::vector<double> rec((size_t)ns * TDW_ELEM_STRIDE);
  std::vector<double> cen((size_t)ns * 3);
  for (int e = 0; e < ns; ++e) {
    const int64_t* t = dsc->triangles + 3 * (size_t)e;
    for (int k = 0; k < 3; ++k)
      if (t[k] < 0 || t[k] >= nv) {
        delete pb;
        return tdw_fail(ctx, TDW_ERR_INVALID_ARG, "triangle index out of range");
      }
    const double* a = dsc->vertices + 3 * t[0];
    const double* b = dsc->vertices + 3 * t[1];
    const double* cc = dsc->vertices + 3 * t[2];
    double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
    double w[3] = {cc[0] - a[0], cc[1] - a[1], cc[2] - a[2]};
    double cr[3] = {u[1] * w[2] - u[2] * w[1], u[2] * w[0] - u[0] * w[2], u[0] * w[1] - u[1] * w[0]};
    double nn = std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
    if (!(nn > 0.0)) {
      delete pb;
      return tdw_fail(ctx, TDW_ERR_INVALID_ARG, "degenerate triangle");
    }
    double* r = &rec[(size_t)e * TDW_ELEM_STRIDE];
    double rad = 0.0;
    for (int k = 0; k < 3; ++k) {
      r[k] = a[k];
      r[3 + k] = b[k];
      r[6 + k] = cc[k];
      r[9 + k] = cr[k] / nn;
      r[12 + k] = (a[k] + b[k] + cc[k]) / 3.0;
      cen[3 * e + k] = r[12 + k];
    }
    const double* vv[3] = {a, b, cc};
    for (int q = 0; q < 3; ++q) {
      double dx = vv[q][0] - r[12], dy = vv[q][1] - r[13], dz = vv[q][2] - r[14];
      rad = std::max(rad, std::sqrt(dx * dx + dy * dy + dz * dz));
    }
    r[15] = rad;
  }
  // Element order: recursive coordinate bisection of the centroids into blocks
  // of 32 (median split along the longest extent, split sizes multiples of 32),
  // so every 32-row I-block and 32-column J-tile is a compact surface patch.
  pb->perm.resize(ns);
  std::iota(pb->perm.begin(), pb->perm.end(), 0);
  {
    struct Span { int lo, hi; };
    std::vector<Span> todo{{0, ns}};
    while (!todo.empty()) {
      Span sp = todo.back();
      todo.pop_back();
      const int n = sp.hi - sp.lo;
      if (n <= TDW_TI) continue;
      double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
      for (int k = sp.lo; k < sp.hi; ++k)
        for (int a = 0; a < 3; ++a) {
          lo[a] = std::min(lo[a], cen[3 * (size_t)pb->perm[k] + a]);
          hi[a] = std::max(hi[a], cen[3 * (size_t)pb->perm[k] + a]);
        }
      int ax = 0;
      for (int a = 1; a < 3; ++a)
        if (hi[a] - lo[a] > hi[ax] - lo[ax]) ax = a;
      int nl = ((n / 2 + TDW_TI / 2) / TDW_TI) * TDW_TI;
      nl = std::max(TDW_TI, std::min(nl, n - 1));
      auto first = pb->perm.begin() + sp.lo;
      std::nth_element(first, first + nl, pb->perm.begin() + sp.hi, [&](int x, int y) {
        const double cx = cen[3 * (size_t)x + ax], cy = cen[3 * (size_t)y + ax];
        return cx < cy || (cx == cy && x < y);
      });
      todo.push_back({sp.lo, sp.lo + nl});
      todo.push_back({sp.lo + nl, sp.hi});
    }
  }
  std::vector<double> prec((size_t)ns * TDW_ELEM_STRIDE), pphi(ns);
  for (int k = 0; k < ns; ++k) {
    memcpy(&prec[(size_t)k * TDW_ELEM_STRIDE], &rec[(size_t)pb->perm[k] * TDW_ELEM_STRIDE],
           sizeof(double) * TDW_ELEM_STRIDE);
    pphi[k] = dsc->phi[pb->perm[k]];
  }
  // rows per rank: whole I-blocks
  const int nblk = (ns + TDW_TI - 1) / TDW_TI;
  const int blk_per_rank = (nblk + nranks - 1) / nranks;
  pb->rows_per_rank = blk_per_rank * TDW_TI;
  pb->n_iblk = blk_per_rank;
  pb->row_lo = rank * pb->rows_per_rank;  // may exceed ns on a rank without rows
  pb->row_hi = std::min(ns, (rank + 1) * pb->rows_per_rank);
  pb->b_off = rank * pb->rows_per_rank;
  pb->ntiles = (ns + TDW_TJ - 1) / TDW_TJ;

  auto fail_cuda = [&](cudaError_t e, const char* what) {
    std::string m = std::string(what) + ": " + cudaGetErrorString(e);
    tdw_problem_destroy(pb);
    return tdw_fail(ctx, TDW_ERR_CUDA, m);
  };
  cudaError_t e;
#define TDW_TRY(call)                              \
  do {                                             \
    e = (call);                                    \
    if (e != cudaSuccess) return fail_cuda(e, #call); \
  } while (0)
  TDW_TRY(cudaMalloc(&pb->d_elem, sizeof(double) * prec.size()));
  TDW_TRY(cudaMemcpy(pb->d_elem, prec.data(), sizeof(double) * prec.size(), cudaMemcpyHostToDevice));
  TDW_TRY(cudaMalloc(&pb->d_phi, sizeof(double) * ns));
  TDW_TRY(cudaMemcpy(pb->d_phi, pphi.data(), sizeof(double) * ns, cudaMemcpyHostToDevice));
  TDW_TRY(cudaMalloc(&pb->d_perm, sizeof(int) * ns));
  TDW_TRY(cudaMemcpy(pb->d_perm, pb->perm.data(), sizeof(int) * ns, cudaMemcpyHostToDevice));
  TDW_TRY(cudaMalloc(&pb->d_flags, sizeof(int) * 4));
  TDW_TRY(cudaMemset(pb->d_flags, 0, sizeof(int) * 4));

  // gamma* = ceil(diam / (c dt)) + d + 1 (marching.py:67-69), diameter over used vertices
  {
    std::vector<char> used(nv, 0);
    for (size_t k = 0; k < 3 * (size_t)ns; ++k) used[dsc->triangles[k]] = 1;
    std::vector<int> ul;
    for (int k = 0; k < nv; ++k)
      if (used[k]) ul.push_back(k);
    double* dv = nullptr;
    int* du = nullptr;
    unsigned long long* dm = nullptr;
    TDW_TRY(cudaMalloc(&dv, sizeof(double) * 3 * nv));
    TDW_TRY(cudaMalloc(&du, sizeof(int) * ul.size()));
    TDW_TRY(cudaMalloc(&dm, sizeof(unsigned long long)));
    TDW_TRY(cudaMemcpy(dv, dsc->vertices, sizeof(double) * 3 * nv, cudaMemcpyHostToDevice));
    TDW_TRY(cudaMemcpy(du, ul.data(), sizeof(int) * ul.size(), cudaMemcpyHostToDevice));
    TDW_TRY(cudaMemset(dm, 0, sizeof(unsigned long long)));
    diameter_kernel<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(dv, du, (int)ul.size(), dm);
    TDW_TRY(cudaGetLastError());
    unsigned long long bits = 0;
    TDW_TRY(cudaStreamSynchronize(ctx->stream));
    TDW_TRY(cudaMemcpy(&bits, dm, sizeof(bits), cudaMemcpyDeviceToHost));
    cudaFree(dv);
    cudaFree(du);
    cudaFree(dm);
    double d2;
    memcpy(&d2, &bits, sizeof(d2));
    const double diam = std::sqrt(d2);
    pb->gstar = (int)std::ceil(diam / (pb->c * pb->dt)) + pb->d + 1;
  }
  pb->n_lags = pb->window ? std::min(pb->gstar, pb->nt - 1) : pb->nt - 1;
  // kappa-combined lags reach gamma = g + kappa <= gamma* with the window (marching.py:216-225)
  pb->cap = pb->window ? std::min(pb->gstar, pb->nt - 1) : pb->nt - 1;
  pb->pad = pb->cap + 1;
  // + TDW_KB_MAX zero rows at the end: the last convolution pass of a loop computes
  // kb steps even when fewer remain, and its history slices reach past step nt-2
  // (the extra steps are discarded, but their rows must be readable)
  pb->hstride = pb->pad + pb->nt - 1 + TDW_KB_MAX;
  pb->hcols = pb->ntiles * TDW_TJ;

  // step buffers
  pb->nsplit = 1;
  {
    // enough CTAs to fill the machine: (I-blocks x splits) >= 2 waves of 2 CTAs/SM
    const int want = 4 * ctx->num_sms;
    while (pb->n_iblk * pb->nsplit < want && pb->nsplit * 2 <= pb->ntiles) pb->nsplit *= 2;
  }
  TDW_TRY(cudaMalloc(&pb->d_bpart, sizeof(double) * (size_t)pb->nsplit * pb->rows_per_rank));
  TDW_TRY(cudaMemset(pb->d_bpart, 0, sizeof(double) * (size_t)pb->nsplit * pb->rows_per_rank));
  pb->bstride = (size_t)nranks * pb->rows_per_rank;
  // b ring: step s in slot s % (2 kb) (a pass writes kb slots while the
  // previous pass's last step is being solved)
  TDW_TRY(cudaMalloc(&pb->d_b, sizeof(double) * 2 * TDW_KB_MAX * pb->bstride));
  TDW_TRY(cudaMemset(pb->d_b, 0, sizeof(double) * 2 * TDW_KB_MAX * pb->bstride));
  TDW_TRY(cudaMalloc(&pb->d_x, sizeof(double) * 2 * (size_t)ns));
  TDW_TRY(cudaMalloc(&pb->d_hist, sizeof(double2) * (size_t)pb->hcols * pb->hstride));
  TDW_TRY(cudaMalloc(&pb->d_bar, sizeof(unsigned) * 2));
  {
    const int occ = 2;  // solve_kernel: 256 threads, tiny smem; 2 per SM are always co-resident
    const int rows_per_block = 256;
    int g = (ns + rows_per_block - 1) / rows_per_block;
    pb->solve_grid = std::max(1, std::min(g, occ * ctx->num_sms));
  }
  TDW_TRY(cudaMalloc(&pb->d_red, sizeof(double) * 3 * pb->solve_grid));
#undef TDW_TRY
  *out = pb;
  return TDW_OK;
}

extern "C" {

int tdw_assemble(tdw_problem* pb) {
  if (!pb) return TDW_ERR_INVALID_ARG;
  if (pb->assembled) return TDW_OK;
  cudaSetDevice(pb->ctx->device);
  return tdw_assemble_impl(pb);
}

int tdw_problem_info(const tdw_problem* pb, tdw_info* out) {
  if (!pb || !out) return TDW_ERR_INVALID_ARG;
  memset(out, 0, sizeof(*out));
  out->gamma_star = pb->gstar;
  out->n_lags = pb->n_lags;
  out->row_lo = pb->row_lo;
  out->row_hi = pb->row_hi;
  out->n_band = pb->n_band;
  out->n_pairs = pb->n_pairs;
  out->n_evals = pb->n_evals;
  out->store_bytes = pb->store_bytes;
  out->step_nnz = pb->step_nnz;
  out->jacobi_iters = pb->jac_iters;
  out->jacobi_bound = pb->jac_bound;
  out->t_assemble_ms = pb->t_assemble_ms;
  out->t_fill_ms = pb->t_fill_ms;
  out->max_unit_bytes = (int64_t)pb->max_unit_bytes;
  out->max_lag_span = pb->wmax;
  out->conv_grid = pb->conv_grid;
  out->fmm_m2l_pairs = tdw_fmm_m2l_pairs(pb);
  out->conv_splits = pb->conv_S;
  out->solve_cluster = pb->sp_cl;
  out->n_units = pb->n_units;
  out->units_hdr32 = pb->units_hdr32;
  out->steps_per_pass = pb->kb;
  out->pass_overlap = pb->overlap;
  out->solve_halo = pb->sp_halo;
  out->near_width = pb->near_w;
  out->conv_rpw = pb->conv_rpw;
  out->coeff_mode = pb->assembled ? (pb->otf ? TDW_MODE_ON_THE_FLY : TDW_MODE_STORED_BAND) : pb->mode;
  return TDW_OK;
}

int tdw_upload_known(tdw_problem* pb, const double* u_known, const double* q_known) {
  if (!pb) return TDW_ERR_INVALID_ARG;
  tdw_ctx* ctx = pb->ctx;
  cudaSetDevice(ctx->device);
  const size_t n = (size_t)(pb->nt - 1) * pb->ns;
  if (!pb->d_uk) TDW_CUDA(ctx, cudaMalloc(&pb->d_uk, sizeof(double) * n));
  if (!pb->d_qk) TDW_CUDA(ctx, cudaMalloc(&pb->d_qk, sizeof(double) * n));
  // NULL = no data callable (the reference's zero samples, marching.py:268-275)
  if (u_known)
    TDW_CUDA(ctx, cudaMemcpyAsync(pb->d_uk, u_known, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  else
    TDW_CUDA(ctx, cudaMemsetAsync(pb->d_uk, 0, sizeof(double) * n, ctx->stream));
  if (q_known)
    TDW_CUDA(ctx, cudaMemcpyAsync(pb->d_qk, q_known, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  else
    TDW_CUDA(ctx, cudaMemsetAsync(pb->d_qk, 0, sizeof(double) * n, ctx->stream));
  pb->known_loaded = true;
  return TDW_OK;
}

int tdw_download(tdw_problem* pb, double* u, double* q, double* tau, double* sigma,
                 int32_t* n_steps, int32_t* status) {
  if (!pb) return TDW_ERR_INVALID_ARG;
  cudaSetDevice(pb->ctx->device);
  int rc = tdw_outputs(pb, u, q, tau, sigma);
  if (rc) return rc;
  int hflags[4];
  TDW_CUDA(pb->ctx, cudaMemcpy(hflags, pb->d_flags, sizeof(hflags), cudaMemcpyDeviceToHost));
  if (n_steps) *n_steps = hflags[1];
  if (status) *status = hflags[0] == 1 ? 1 : 0;
  return TDW_OK;
}

int tdw_upload_known_rows(tdw_problem* pb, int which, int beta0, int nbeta, const double* src) {
  if (!pb || which < 0 || which > 1 || beta0 < 0 || nbeta < 0 || beta0 + nbeta > pb->nt - 1)
    return TDW_ERR_INVALID_ARG;
  tdw_ctx* ctx = pb->ctx;
  cudaSetDevice(ctx->device);
  const size_t n = (size_t)(pb->nt - 1) * pb->ns;
  double** dst = which == 0 ? &pb->d_uk : &pb->d_qk;
  if (!*dst) TDW_CUDA(ctx, cudaMalloc(dst, sizeof(double) * n));
  const size_t off = (size_t)beta0 * pb->ns, cnt = (size_t)nbeta * pb->ns;
  if (src)
    TDW_CUDA(ctx, cudaMemcpyAsync(*dst + off, src, sizeof(double) * cnt, cudaMemcpyHostToDevice, ctx->stream));
  else
    TDW_CUDA(ctx, cudaMemsetAsync(*dst + off, 0, sizeof(double) * cnt, ctx->stream));
  return TDW_OK;
}

int tdw_march_device_known(tdw_problem* pb, double threshold, double* u, double* q, double* tau,
                           double* sigma, double* rhs_trace, int32_t* n_steps, int32_t* status) {
  if (!pb || !pb->d_uk || !pb->d_qk) return TDW_ERR_INVALID_ARG;
  pb->known_loaded = true;
  pb->known_preloaded_call = true;
  return tdw_march(pb, nullptr, nullptr, threshold, u, q, tau, sigma, rhs_trace, n_steps, status);
}

// Streamed march: launch the loop now, the host fills the page-locked sample
// buffers (u_host / q_host from tdw_host_alloc, NULL = that datum is zero) chunk by
// chunk and publishes the number of complete chunks of `chunk` steps in *flag
// (page-locked int, -1 aborts); then tdw_march_stream_finish.
int tdw_march_stream_begin(tdw_problem* pb, double threshold, int want_rhs, const double* u_host,
                           const double* q_host, int chunk, int32_t* flag) {
  if (!pb || !flag || chunk < 1) return TDW_ERR_INVALID_ARG;
  tdw_ctx* ctx = pb->ctx;
  cudaSetDevice(ctx->device);
  if (pb->stream_in_flight) return tdw_fail(ctx, TDW_ERR_STATE, "a streamed march is already in flight");
  if (pb->fmm) return tdw_fail(ctx, TDW_ERR_STATE, "streamed march: direct path only");
  const size_t n = (size_t)(pb->nt - 1) * pb->ns;
  if (!pb->d_uk) TDW_CUDA(ctx, cudaMalloc(&pb->d_uk, sizeof(double) * n));
  if (!pb->d_qk) TDW_CUDA(ctx, cudaMalloc(&pb->d_qk, sizeof(double) * n));
  pb->h_uk_host = u_host;
  pb->h_qk_host = q_host;
  pb->h_flag_host = (const volatile int*)flag;
  pb->stream_chunk = chunk;
  if (!pb->assembled) {
    int rc = tdw_assemble_impl(pb);
    if (rc) return rc;
  }
  pb->known_loaded = true;
  return tdw_march_stream_launch(pb, threshold, want_rhs != 0);
}

// Destinations of the NEXT streamed march's outputs: page-locked (nt-1, ns) arrays
// (tdw_host_alloc; NULL = not wanted).  The loop then writes each chunk's rows as
// soon as its last step is solved, and tdw_march_stream_finish -- called with the
// same pointers -- has nothing left to copy.
int tdw_march_stream_outputs(tdw_problem* pb, double* u, double* q, double* tau, double* sigma) {
  if (!pb) return TDW_ERR_INVALID_ARG;
  tdw_ctx* ctx = pb->ctx;
  cudaSetDevice(ctx->device);
  if (pb->stream_in_flight) return tdw_fail(ctx, TDW_ERR_STATE, "a streamed march is already in flight");
  double* outs[4] = {u, q, tau, sigma};
  for (int k = 0; k < 4; ++k) {
    if (!outs[k]) continue;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, outs[k]) != cudaSuccess || at.type != cudaMemoryTypeHost) {
      cudaGetLastError();
      return tdw_fail(ctx, TDW_ERR_INVALID_ARG, "tdw_march_stream_outputs: the arrays must be page-locked (tdw_host_alloc)");
    }
  }
  for (int k = 0; k < 4; ++k) pb->out_host[k] = outs[k];
  pb->out_registered = true;
  return TDW_OK;
}

int tdw_march_stream_finish(tdw_problem* pb, double* u, double* q, double* tau, double* sigma,
                            double* rhs_trace, int32_t* n_steps, int32_t* status) {
  if (!pb) return TDW_ERR_INVALID_ARG;
  cudaSetDevice(pb->ctx->device);
  int rc = tdw_march_stream_wait(pb);
  const bool streamed = pb->out_streamed;
  pb->out_streamed = false;
  if (rc) return rc;
  if (rhs_trace)
    TDW_CUDA(pb->ctx, cudaMemcpy(rhs_trace, pb->d_rhs, sizeof(double) * (size_t)(pb->nt - 1) * pb->ns,
                                 cudaMemcpyDeviceToHost));
  // arrays the loop has written already (same pointers as registered) need no copy
  double* outs[4] = {u, q, tau, sigma};
  if (streamed)
    for (int k = 0; k < 4; ++k)
      if (outs[k] && outs[k] == pb->out_host[k]) outs[k] = nullptr;
  return tdw_download(pb, outs[0], outs[1], outs[2], outs[3], n_steps, status);
}

int tdw_march(tdw_problem* pb, const double* u_known, const double* q_known, double threshold,
              double* u, double* q, double* tau, double* sigma, double* rhs_trace,
              int32_t* n_steps, int32_t* status) {
  if (!pb) return TDW_ERR_INVALID_ARG;
  cudaSetDevice(pb->ctx->device);
  static const bool trace = getenv("TDW_TRACE_MARCH") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto t0 = now();
  // tdw_march_device_known: the rows are on the device already (both pointers NULL
  // with known_loaded set by that entry point)
  const bool preloaded = !u_known && !q_known && pb->known_loaded && pb->d_uk && pb->d_qk &&
                         pb->known_preloaded_call;
  int rc = preloaded ? TDW_OK : tdw_upload_known(pb, u_known, q_known);
  pb->known_preloaded_call = false;
  if (rc) return rc;
  if (trace) {
    cudaStreamSynchronize(pb->ctx->stream);
    fprintf(stderr, "tdw_march: upload %.2f ms\n",
            std::chrono::duration<double, std::milli>(now() - t0).count());
  }
  if (!pb->assembled) {
    rc = tdw_assemble_impl(pb);
    if (rc) return rc;
  }
  cudaStreamSynchronize(pb->ctx->stream);
  auto t1 = now();
  rc = tdw_march_loop(pb, threshold, rhs_trace != nullptr, false, nullptr);
  if (rc) return rc;
  auto t2 = now();
  if (rhs_trace) {
    TDW_CUDA(pb->ctx, cudaMemcpy(rhs_trace, pb->d_rhs, sizeof(double) * (size_t)(pb->nt - 1) * pb->ns,
                                 cudaMemcpyDeviceToHost));
  }
  rc = tdw_download(pb, u, q, tau, sigma, n_steps, status);
  auto t3 = now();
  if (trace) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    fprintf(stderr, "tdw_march: upload+assemble %.2f ms, loop %.2f ms, download %.2f ms\n", ms(t0, t1),
            ms(t1, t2), ms(t2, t3));
  }
  return rc;
}

int tdw_march_resident(tdw_problem* pb, double threshold, int n_repeat, int time_kernels,
                       tdw_timing* timing) {
  if (!pb || n_repeat < 1) return TDW_ERR_INVALID_ARG;
  cudaSetDevice(pb->ctx->device);
  static const bool trace = getenv("TDW_TRACE_SOLVE") != nullptr;
  if (trace && !pb->d_trace) {
    TDW_CUDA(pb->ctx, cudaMalloc(&pb->d_trace, sizeof(unsigned long long) * 16 * pb->nt));
    TDW_CUDA(pb->ctx, cudaMemset(pb->d_trace, 0, sizeof(unsigned long long) * 16 * pb->nt));
    if (pb->graph_exec) { cudaGraphExecDestroy(pb->graph_exec); pb->graph_exec = nullptr; }
  }
  if (timing) memset(timing, 0, sizeof(*timing));
  for (int r = 0; r < n_repeat; ++r) {
    int rc = tdw_march_loop(pb, threshold, false, time_kernels != 0, timing);
    if (rc) return rc;
  }
  if (trace) {
    std::vector<unsigned long long> h((size_t)16 * pb->nt);
    TDW_CUDA(pb->ctx, cudaMemcpy(h.data(), pb->d_trace, sizeof(unsigned long long) * h.size(),
                                 cudaMemcpyDeviceToHost));
    double acc[9] = {0};
    int n = 0;
    double sw = 0;
    for (int a = 2; a < pb->nt; ++a) {
      const unsigned long long* t = &h[(size_t)16 * a];
      if (!t[0] || !t[8]) continue;
      for (int k = 1; k <= 8; ++k) acc[k] += (double)(t[k] - t[k - 1]);
      sw += (double)t[15];
      ++n;
    }
    if (n)
      fprintf(stderr, "solve phases (us, mean of %d steps): load %.2f sync %.2f sweeps(%.1f) %.2f resid %.2f "
              "sync %.2f near %.2f sync %.2f final %.2f\n", n, acc[1] / n / 1e3, acc[2] / n / 1e3, sw / n,
              acc[3] / n / 1e3, acc[4] / n / 1e3, acc[5] / n / 1e3, acc[6] / n / 1e3, acc[7] / n / 1e3,
              acc[8] / n / 1e3);
    // timeline of the last loop: solve, near step, gaps, convolution passes
    double tl[5] = {0}, cv = 0.0;
    int m = 0, mc = 0;
    for (int a = 8; a + 1 < pb->nt; ++a) {
      const unsigned long long* t = &h[(size_t)16 * a];
      const unsigned long long* u = &h[(size_t)16 * (a + 1)];
      if (!t[0] || !t[8] || !t[9] || !t[10] || !u[0] || u[0] < t[0]) continue;
      tl[0] += (double)(t[8] - t[0]);
      tl[1] += (double)t[9] - (double)t[8];
      tl[2] += (double)(t[10] - t[9]);
      tl[3] += (double)u[0] - (double)t[10];
      tl[4] += (double)(u[0] - t[0]);
      ++m;
      if (t[11] && t[12] > t[11] && (a - 1) % pb->kb == 0) {
        cv += (double)(t[12] - t[11]);
        ++mc;
      }
    }
    if (getenv("TDW_TRACE_RAW")) {  // raw per-step stamps (us from step 40's solve start)
      const double t00 = (double)h[(size_t)16 * 40];
      for (int a = 40; a < std::min(pb->nt, 64); ++a) {
        const unsigned long long* t = &h[(size_t)16 * a];
        auto us = [&](unsigned long long v) { return v ? ((double)v - t00) / 1e3 : -1.0; };
        fprintf(stderr, "step %3d solve [%8.2f %8.2f] near [%8.2f %8.2f] conv [%8.2f %8.2f]\n", a, us(t[0]),
                us(t[8]), us(t[9]), us(t[10]), us(t[11]), us(t[12]));
      }
    }
    if (m)
      fprintf(stderr, "timeline (us, mean of %d steps): solve %.2f | gap %.2f | near %.2f | gap to next solve %.2f "
              "| step period %.2f; conv pass %.2f (%d passes)\n", m, tl[0] / m / 1e3, tl[1] / m / 1e3,
              tl[2] / m / 1e3, tl[3] / m / 1e3, tl[4] / m / 1e3, mc ? cv / mc / 1e3 : 0.0, mc);
  }
  return TDW_OK;
}

int tdw_step_matrix(tdw_problem* pb, int64_t* nnz, int64_t* rows, int64_t* cols, double* vals) {
  if (!pb || !nnz || (rows && (!cols || !vals))) return TDW_ERR_INVALID_ARG;
  cudaSetDevice(pb->ctx->device);
  return tdw_step_matrix_impl(pb, nnz, rows, cols, vals);
}

int tdw_step_solve(tdw_problem* pb, const double* b, double* x, double* stats) {
  if (!pb || !b || !x) return TDW_ERR_INVALID_ARG;
  cudaSetDevice(pb->ctx->device);
  return tdw_step_solve_impl(pb, b, x, stats);
}

int tdw_restrict_pairs(tdw_problem* pb, int64_t n, const int64_t* ii, const int64_t* jj) {
  if (!pb || n < 0 || (n > 0 && (!ii || !jj))) return TDW_ERR_INVALID_ARG;
  tdw_ctx* ctx = pb->ctx;
  if (pb->assembled) return tdw_fail(ctx, TDW_ERR_STATE, "tdw_restrict_pairs after tdw_assemble");
  if (pb->fmm) return tdw_fail(ctx, TDW_ERR_STATE, "tdw_restrict_pairs on an FMM problem");
  cudaSetDevice(ctx->device);
  const int ns = pb->ns;
  std::vector<int> inv(ns);
  for (int k = 0; k < ns; ++k) inv[pb->perm[k]] = k;
  std::vector<std::vector<int>> rows(ns);
  for (int64_t p = 0; p < n; ++p) {
    if (ii[p] < 0 || ii[p] >= ns || jj[p] < 0 || jj[p] >= ns)
      return tdw_fail(ctx, TDW_ERR_INVALID_ARG, "pairs: element index out of range");
    rows[inv[ii[p]]].push_back(inv[jj[p]]);
  }
  std::vector<int> ptr(ns + 1, 0), col;
  col.reserve((size_t)n);
  for (int i = 0; i < ns; ++i) {
    std::sort(rows[i].begin(), rows[i].end());
    rows[i].erase(std::unique(rows[i].begin(), rows[i].end()), rows[i].end());
    col.insert(col.end(), rows[i].begin(), rows[i].end());
    ptr[i + 1] = (int)col.size();
  }
  cudaFree(pb->d_pair_ptr);
  cudaFree(pb->d_pair_col);
  pb->d_pair_ptr = pb->d_pair_col = nullptr;
  TDW_CUDA(ctx, cudaMalloc(&pb->d_pair_ptr, sizeof(int) * (ns + 1)));
  TDW_CUDA(ctx, cudaMalloc(&pb->d_pair_col, sizeof(int) * std::max<size_t>(1, col.size())));
  TDW_CUDA(ctx, cudaMemcpy(pb->d_pair_ptr, ptr.data(), sizeof(int) * (ns + 1), cudaMemcpyHostToDevice));
  if (!col.empty())
    TDW_CUDA(ctx, cudaMemcpy(pb->d_pair_col, col.data(), sizeof(int) * col.size(), cudaMemcpyHostToDevice));
  return TDW_OK;
}

int tdw_fmm_time_m2l(tdw_problem* pb, int n, double* flops, float* ms) {
  if (!pb) return TDW_ERR_INVALID_ARG;
  cudaSetDevice(pb->ctx->device);
  return tdw_fmm_time_m2l_impl(pb, n, flops, ms);
}

int tdw_time_conv(tdw_problem* pb, int n, float* ms) {
  if (!pb || n < 1 || !ms) return TDW_ERR_INVALID_ARG;
  if (!pb->assembled) return tdw_fail(pb->ctx, TDW_ERR_STATE, "tdw_time_conv before tdw_assemble");
  cudaSetDevice(pb->ctx->device);
  return tdw_time_conv_impl(pb, n, ms);
}

int tdw_set_graph(tdw_problem* pb, int enable) {
  if (!pb) return TDW_ERR_INVALID_ARG;
  pb->use_graph = enable != 0;
  return TDW_OK;
}

int tdw_problem_destroy(tdw_problem* pb) {
  if (!pb) return TDW_OK;
  cudaSetDevice(pb->ctx->device);
  // a streamed march nobody finished: stop waiting for its data, let the loop
  // drain, and only then free what its kernels use
  pb->stream_cancel = true;
  if (pb->stream_thread.joinable()) pb->stream_thread.join();
  if (pb->chunk_thread.joinable()) pb->chunk_thread.join();
  if (pb->stream_in_flight) cudaDeviceSynchronize();
  void* ptrs[] = {pb->d_perm, pb->d_elem, pb->d_phi, pb->d_units, pb->d_unit_off, pb->d_sched, pb->d_sched_off,
                  pb->d_sched_item, pb->d_leafc, pb->d_pair_ptr, pb->d_pair_col, pb->d_kw, pb->d_otf_evals,
                  pb->d_unit, pb->d_acol, pb->d_aval, pb->d_adiag, pb->d_hist, pb->d_uk,
                  pb->d_qk, pb->d_bpart, pb->d_b, pb->d_x, pb->d_red, pb->d_bar, pb->d_flags,
                  pb->d_rhs, pb->d_sp_rowptr, pb->d_sp_nnzoff, pb->d_sp_col, pb->d_sp_val,
                  pb->d_ncol, pb->d_nval, pb->d_ncol_packed, pb->d_h_ncomp, pb->d_h_gi, pb->d_h_layer, pb->d_h_nz, pb->d_h_col,
                  pb->d_h_ngat, pb->d_h_gdst, pb->d_h_gsrc, pb->d_h_val, pb->d_ncnt, pb->d_n3_ptr, pb->d_n3_ent, pb->d_bnear, pb->d_out, pb->d_trace, pb->d_n2_ptr, pb->d_n2_col, pb->d_n2_val};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (pb->graph_exec) cudaGraphExecDestroy(pb->graph_exec);
  if (pb->fmm) tdw_fmm_free(pb->fmm);
  for (auto& e : pb->ev_solve) cudaEventDestroy(e);
  for (auto& e : pb->ev_conv) cudaEventDestroy(e);
  for (auto& e : pb->ev_near) cudaEventDestroy(e);
  if (pb->ev_fork) cudaEventDestroy(pb->ev_fork);
  if (pb->side) cudaStreamDestroy(pb->side);
  if (pb->side_near) cudaStreamDestroy(pb->side_near);
  if (pb->graph_exec_s) cudaGraphExecDestroy(pb->graph_exec_s);
  if (pb->ev_begin) cudaEventDestroy(pb->ev_begin);
  if (pb->d_ready) cudaFree(pb->d_ready);
  if (pb->ev_stream_end) cudaEventDestroy(pb->ev_stream_end);
  if (pb->side_data) cudaStreamDestroy(pb->side_data);
  if (pb->side_out) cudaStreamDestroy(pb->side_out);
  if (pb->ev_out) cudaEventDestroy(pb->ev_out);
  if (pb->d_outdesc) cudaFree(pb->d_outdesc);
  if (pb->d_iperm) cudaFree(pb->d_iperm);
  delete pb;
  return TDW_OK;
}

}  // extern "C"
