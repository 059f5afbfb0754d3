// fmm.cu -- interpolation space-time FMM on the device (configs 3-4).
//
// Restates the corrected fast solver (reference pkg/src/tdwavebem/fmm.py:165-531
// with the SURVEY.md 8(c) corrections; CPU restatement oracle/fmm_oracle.py):
//   near field   the banded store restricted to adjacent leaf cells, window gamma_near
//                (fmm.py:213-235, 446-457) -- assemble.cu / conv_kernel
//   extra lists  same-interval pairs of marginal interaction pairs, raw lag form
//                (fmm.py:223-234, 459-470)                           -- extra_*_kernel
//   L2P          leaf locals at the observation time (fmm.py:474-495) -- l2p_kernel
//   P2M          the step's source into its interval's leaf moment (fmm.py:509-521) -- p2m_kernel
//   tick         M2L (near-future lags + derivative operators + Algorithm-1
//                recurrence, fmm.py:329-368) -- m2l_kernel; M2M up while the
//                time-half bit is 1, L2L down into inherit slots (fmm.py:371-419)
//                -- m2m_kernel / l2l_kernel
// Interpolation orders ps = pt = 4 (BASELINE), mu <= 8.  The operator data is
// built on the host (paper_2111_05205_b200/fmm_plan.py) and handed over by
// tdw_fmm_setup; the per-step control flow (which ticks run before which step)
// is a fixed schedule, so the loop is a plain sequence of launches.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "coeff.cuh"
#include "tdw_impl.cuh"

#define FULLMASK 0xffffffffu
constexpr int FPS = 4;               // spatial nodes per dimension
constexpr int FPT = 4;               // temporal nodes
constexpr int FN3 = FPS * FPS * FPS; // 64
constexpr int FND = FN3 * FPT;       // 256
constexpr int FKR = (2 * FPS - 1) * (2 * FPS - 1) * (2 * FPS - 1);  // 343 Toeplitz rows
constexpr int FMU_MAX = 8;

struct FmmLevel {
  int L = 0, ncell = 0, noff = 0;
  double interval = 0.0;
  int* parent = nullptr;       // [ncell] index in level L-1
  int* octant = nullptr;       // [ncell] bits x | y<<1 | z<<2
  int* child_ptr = nullptr;    // [ncell+1] children at level L+1 (ascending)
  int* child_idx = nullptr;
  long long* obs_ptr = nullptr;  // [ncell+1]
  int* il_src = nullptr;
  int* il_off = nullptr;
  unsigned* dark = nullptr;    // [noff] bit l-1 set: lag l dark
  double* K0 = nullptr;        // [noff][343][ntau0]
  double* Kp = nullptr;        // [d][noff][343][ntaup]
  double *own = nullptr, *inherit = nullptr, *deriv = nullptr, *aux = nullptr, *acc = nullptr,
         *mom = nullptr;
  // GEMM form of M2L: pairs grouped by offset, stacked dense operators per offset
  std::vector<long long> grp;  // [noff+1] pair range of each offset group
  int* g_obs = nullptr;        // [nil] observer of each grouped pair
  int* g_src = nullptr;        // [nil] source
  double* Kop = nullptr;       // [noff][K = 256][M = nops*256] column-major operator stacks
  double* X = nullptr;         // [nil][256] gathered source moments
  double* tmp = nullptr;       // [d][ncell][256]
  long long nil = 0, max_grp = 0;
  // one scatter per level tick: the GEMM outputs of all offset groups side by side,
  // and per target cell its pairs in group order (the per-group scatters' order)
  int* t_ptr = nullptr;        // [ncell+1]
  int* t_pair = nullptr;       // [nil] column of Yall
  int* t_cells = nullptr;      // [n_tcell] target cells with pairs
  int n_tcell = 0;
  // own M2L kernel (m2l_dmma_kernel): work items (offset, first pair, pairs) and
  // the dark-lag bits of each grouped pair's offset (the scatter skips those rows)
  int4* items = nullptr;
  int n_items = 0;
  double m2l_flops = 0.0;      // FLOPs of one M2L launch (non-dark operators only)
  unsigned* g_dark = nullptr;  // [nil]
  // the level's GEMMs as one grouped call (one group per nonempty offset)
  std::vector<int> gm, gn, gk, glda, gldb, gldc, gsize;
  std::vector<double> galpha, gbeta;
  std::vector<cublasOperation_t> gop;
  const double** gA = nullptr;  // device pointer arrays
  const double** gB = nullptr;
  double** gC = nullptr;
};

struct FmmExtra {
  int lags = 0;
  long long npair = 0;
  int* row_ptr = nullptr;      // [ns+1] internal rows
  int* col = nullptr;          // [npair] internal columns
  int* row_of = nullptr;       // [npair]
  double *U = nullptr, *W = nullptr;  // [npair][lags]
  std::vector<long long> gmax; // per step
};

struct FmmState {
  int mu = 8, leaf = 0, ntau0 = 0, ntaup = 0, n_leaf_cells = 0, nops = 0;
  cublasHandle_t blas = nullptr;
  double* Y = nullptr;         // [max group][nops*256] GEMM output
  std::vector<FmmLevel> lev;   // index = level (entries < 2 unused)
  int* elem_cell = nullptr;    // [ns] internal order
  int* cell_ptr = nullptr;     // [ncell+1] leaf cell -> internal elements
  int* cell_elems = nullptr;
  double *p2m_tau = nullptr, *p2m_sig = nullptr, *l2p_val = nullptr, *l2p_bm = nullptr;
  double t_space[2][FPS][FPS], t_time[2][FPT][FPT];
  std::vector<FmmExtra> extra;
  std::vector<long long> ticks_before, k_obs;
  int r0 = 0, r1 = 0;          // this shard's rows (internal order)
  long long m2l_pairs = 0;     // M2L interaction pairs this shard evaluates (all levels)
  std::vector<double> wt, dwt, wts;  // [nt][FPT]
};

namespace {

struct Tr {  // transfer matrices by value (kernel argument)
  double s[2][FPS][FPS], t[2][FPT][FPT];
};

__device__ __forceinline__ void bw(int d, double* w) {
  if (d == 1) { w[0] = 1.0; w[1] = -2.0; w[2] = 1.0; }
  if (d == 2) { w[0] = 0.5; w[1] = -1.5; w[2] = 1.5; w[3] = -0.5; }
  if (d == 3) { w[0] = 1.0 / 6.0; w[1] = -(2.0 / 3.0); w[2] = 1.0; w[3] = -(2.0 / 3.0); w[4] = 1.0 / 6.0; }
}

// tau_j^beta / sigma_j^beta (stock sums, marching.py:205-214) from the history;
// slot beta holds the known part until step beta+1 is solved (tilde sums).
__device__ __forceinline__ double2 stock(const double2* __restrict__ hist, int hcols, int pad,
                                         int j, int beta, int d, const double* w) {
  double t = 0.0, s = 0.0;
  const int kmax = min(d + 1, beta);
  const double2* h = hist + (size_t)(pad + beta) * hcols + j;
  for (int k = 0; k <= kmax; ++k) {
    const double2 v = h[-(ptrdiff_t)k * hcols];
    t += w[k] * v.x;
    s += w[k] * v.y;
  }
  return make_double2(t, s);
}

// ---------------------------------------------------------------- extra lists
template <int D, bool BM>
__global__ void extra_coeff_kernel(const double* __restrict__ elem, const int* __restrict__ row_of,
                                   const int* __restrict__ col, long long npair, int lags, double c,
                                   double dt, double K, double* U, double* W) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < npair;
       p += (long long)gridDim.x * blockDim.x) {
    const int i = row_of[p], j = col[p];
    const double* pi = elem + (size_t)i * TDW_ELEM_STRIDE;
    const double* pj = elem + (size_t)j * TDW_ELEM_STRIDE;
    double ci[3] = {pi[12], pi[13], pi[14]}, nx[3] = {-pi[9], -pi[10], -pi[11]};
    // reference arrival (marching.py:108-110): U = 0 before it
    double dx = ci[0] - pj[12], dy = ci[1] - pj[13], dz = ci[2] - pj[14];
    double dist = fmax(sqrt(dx * dx + dy * dy + dz * dz) - pj[15], 0.0);
    int arr = max((int)ceil(dist / (c * dt)) - 1, 1);
    tdw::PairGeom g;
    tdw::pair_geom<BM>(ci, pj, pj + 3, pj + 6, pj + 9, nx, g);
    for (int q = 1; q <= lags; ++q) {
      double u = 0.0, w = 0.0;
      if (q >= arr) tdw::coeff_eval<D, BM>(g, (double)q * c * dt, K, u, w);
      U[p * lags + q - 1] = u;
      W[p * lags + q - 1] = w;
    }
  }
}

// one warp per row, lanes over the row's pairs (each lane runs its pair's lags),
// fixed-order warp reduction: deterministic
__global__ void extra_apply_kernel(const int* __restrict__ row_ptr, const int* __restrict__ col,
                                   const double* __restrict__ U, const double* __restrict__ W,
                                   int lags, int gmax, const double2* __restrict__ hist, int hcols,
                                   int pad, int alpha, int d, int r0, int r1, double* b,
                                   const int* flags) {
  if (flags[0] != 0) return;
  double w[5] = {0, 0, 0, 0, 0};
  bw(d, w);
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = r0 + (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < r1; i += nw) {
    const int p0 = __ldg(row_ptr + i), p1 = __ldg(row_ptr + i + 1);
    if (p0 == p1) continue;  // warp-uniform
    double acc = 0.0;
    for (int p = p0 + lane; p < p1; p += 32) {
      const int j = __ldg(col + p);
      const double* up = U + (size_t)p * lags;
      const double* wp = W + (size_t)p * lags;
      for (int g = 1; g <= gmax; ++g) {
        const double2 ts = stock(hist, hcols, pad, j, alpha - g, d, w);
        acc += __ldg(up + g - 1) * ts.x - __ldg(wp + g - 1) * ts.y;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULLMASK, acc, o);
    if (lane == 0) b[i] += acc;
  }
}

// ---------------------------------------------------------------- L2P / P2M
struct StepW {
  double wt[FPT], dwt[FPT], wts[FPT];
};

__global__ void l2p_kernel(const int* __restrict__ elem_cell, const double* __restrict__ own,
                           const double* __restrict__ inherit, int ko_own, int ko_inh, int ncell,
                           const double* __restrict__ lval, const double* __restrict__ lbm, StepW sw,
                           int r0, int r1, double* b, const int* flags) {
  if (flags[0] != 0) return;
  for (int j = r0 + blockIdx.x * blockDim.x + threadIdx.x; j < r1; j += gridDim.x * blockDim.x) {
    const int cell = elem_cell[j];
    const double* lo = own + ((size_t)ko_own * ncell + cell) * FND;
    const double* li = inherit + ((size_t)ko_inh * ncell + cell) * FND;
    double acc = 0.0;
    for (int a = 0; a < FN3; ++a) {
      double v = 0.0, dv = 0.0;
#pragma unroll
      for (int m = 0; m < FPT; ++m) {
        const double L = lo[a * FPT + m] + li[a * FPT + m];
        v += L * sw.wt[m];
        dv += L * sw.dwt[m];
      }
      if (lbm) acc += lbm[(size_t)j * FN3 + a] * v - lval[(size_t)j * FN3 + a] * dv;
      else acc += lval[(size_t)j * FN3 + a] * v;
    }
    b[j] += acc;
  }
}

__global__ void p2m_kernel(const int* __restrict__ cell_ptr, const int* __restrict__ cell_elems,
                           const double* __restrict__ ptau, const double* __restrict__ psig,
                           const double2* __restrict__ hist, int hcols, int pad, int beta0, int d,
                           StepW sw, double* acc, const int* flags) {
  if (flags[0] != 0) return;
  double w[5] = {0, 0, 0, 0, 0};
  bw(d, w);
  const int cell = blockIdx.x, s = threadIdx.x;  // 64 threads: spatial node
  double spat = 0.0;
  for (int q = cell_ptr[cell]; q < cell_ptr[cell + 1]; ++q) {
    const int e = cell_elems[q];
    const double2 ts = stock(hist, hcols, pad, e, beta0, d, w);
    spat += ptau[(size_t)e * FN3 + s] * ts.x - psig[(size_t)e * FN3 + s] * ts.y;
  }
  double* A = acc + (size_t)cell * FND + s * FPT;
#pragma unroll
  for (int t = 0; t < FPT; ++t) A[t] += spat * sw.wts[t];
}

// ---------------------------------------------------------------- recurrence coefficients
__device__ __forceinline__ double cmp_coeff_dev(int p, int m, int k) {
  // comb(p, m) ((k-1)^(p-m) - 2 k^(p-m) + (k+1)^(p-m)) (-1)^m   (fmm.py:44-49)
  double binom = 1.0;
  for (int q = 0; q < m; ++q) binom = binom * (p - q) / (q + 1);
  const int e = p - m;
  double km = 1.0, k0 = 1.0, kp = 1.0;
  for (int q = 0; q < e; ++q) { km *= (k - 1); k0 *= k; kp *= (k + 1); }
  return binom * (km - 2.0 * k0 + kp) * ((m & 1) ? -1.0 : 1.0);
}

// ---------------------------------------------------------------- M2L as GEMM
// Stacked dense operators of one offset: rows op*256 + ((a1*4+a2)*4+a3)*4+m,
// columns ((b1*4+b2)*4+b3)*4+n (the reference's dense_m2l_matrix layout,
// fmm.py:134-162); ops 0..mu = lags 1..mu+1 (toff = l (pt-1)), mu+1.. = p = 1..d.
__global__ void build_kop_kernel(const double* __restrict__ K0, const double* __restrict__ Kp,
                                 int noff, int ntau0, int ntaup, int mu, int d, double* Kop) {
  const int nops = mu + 1 + d, M = nops * FND;
  const long long total = (long long)noff * FND * M;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int off = (int)(e / ((long long)FND * M));
    const long long rem = e % ((long long)FND * M);
    const int col = (int)(rem / M), rowf = (int)(rem % M);
    const int op = rowf / FND, row = rowf % FND;
    const int a1 = row >> 6, a2 = (row >> 4) & 3, a3 = (row >> 2) & 3, m = row & 3;
    const int b1 = col >> 6, b2 = (col >> 4) & 3, b3 = (col >> 2) & 3, n = col & 3;
    const int kr = ((a1 - b1 + FPS - 1) * (2 * FPS - 1) + (a2 - b2 + FPS - 1)) * (2 * FPS - 1) +
                   (a3 - b3 + FPS - 1);
    double v;
    if (op <= mu) {
      const int l = op + 1;
      v = K0[((size_t)off * FKR + kr) * ntau0 + (m - n + l * (FPT - 1))];
    } else {
      const int p = op - mu - 1;
      v = Kp[(((size_t)p * noff + off) * FKR + kr) * ntaup + (m - n + FPT - 1)];
    }
    Kop[e] = v;
  }
}

// all offset groups of a level at once: block (target cell with pairs, operator),
// thread = node; adds the cell's GEMM columns in group order onto own / tmp, the
// same additions in the same order as one scatter per group
// (g_dark != null: rows of a pair's dark lags were not computed -- skipped, as the
// reference skips dark lags, fmm.py:343-346)
// tau_rows: Y in m2l_dmma_kernel's layout (64 NT shared near-future rows (a, tau),
// then the derivative operators); 0: one 256-row block per operator (cuBLAS path)
__global__ void scatter_all_kernel(const int* __restrict__ t_cells, const int* __restrict__ t_ptr,
                                   const int* __restrict__ t_pair, const unsigned* __restrict__ g_dark,
                                   const double* __restrict__ Y, int nops, int mu, int k, int ncell,
                                   double* own, double* tmp, int tau_rows) {
  const int ring = mu + 3;
  const int d = nops - mu - 1, NT = (mu + 1) * (FPT - 1) + 1;
  const long long M = tau_rows ? 64LL * NT + (long long)d * FND : (long long)nops * FND;
  const int cell = t_cells[blockIdx.x], op = blockIdx.y, idx = threadIdx.x;
  double* dst = op <= mu ? own + ((size_t)((k + op + 1) % ring) * ncell + cell) * FND + idx
                         : tmp + ((size_t)(op - mu - 1) * ncell + cell) * FND + idx;
  // this thread's row of operator op: lag op+1's (a, m) is the shared row (a, tau =
  // m + 3 (op + 1)), stored at a NT + tau - 3
  const long long yr = !tau_rows ? (long long)op * FND + idx
                                 : (op <= mu ? (long long)(idx >> 2) * NT + (FPT - 1) * op + (idx & 3)
                                             : 64LL * NT + (long long)(op - mu - 1) * FND + idx);
  double acc = *dst;
  for (int q = t_ptr[cell]; q < t_ptr[cell + 1]; ++q) {
    const int pq = t_pair[q];
    if (g_dark && op <= mu && ((__ldg(g_dark + pq) >> op) & 1u)) continue;
    acc += __ldg(Y + (long long)pq * M + yr);
  }
  *dst = acc;
}
// The level's M2L outputs (m2l_dmma_kernel layout) summed into the target cells,
// coalesced: thread = one row j of Y (consecutive threads read consecutive rows),
// looping over the cell's pairs in group order.  A shared near-future row (a, tau)
// feeds lag tau/3's row m = tau%3 and, when tau%3 == 0, lag tau/3 - 1's row m = 3:
// each destination has exactly one owner thread, and every destination receives
// its additions in the same order as one scatter per operator would (bit-identical).
__global__ void scatter_tau_kernel(const int* __restrict__ t_cells, const int* __restrict__ t_ptr,
                                   const int* __restrict__ t_pair, const unsigned* __restrict__ g_dark,
                                   const double* __restrict__ Y, int d, int mu, int k, int ncell, double* own,
                                   double* tmp) {
  const int ring = mu + 3, NT = (mu + 1) * (FPT - 1) + 1;
  const long long M = 64LL * NT + (long long)d * FND;
  const int cell = t_cells[blockIdx.x];
  const int j = blockIdx.y * blockDim.x + threadIdx.x;
  if (j >= M) return;
  const int q0 = t_ptr[cell], q1 = t_ptr[cell + 1];
  if (j >= 64 * NT) {  // derivative operators
    const int p = (j - 64 * NT) / FND, idx = (j - 64 * NT) % FND;
    double* dst = tmp + ((size_t)p * ncell + cell) * FND + idx;
    double acc = *dst;
    for (int q = q0; q < q1; ++q) acc += __ldg(Y + (long long)t_pair[q] * M + j);
    *dst = acc;
    return;
  }
  const int a = j / NT, tau = (FPT - 1) + j % NT;
  const int l1 = min(mu + 1, tau / (FPT - 1));       // lag with row m1 = tau - 3 l1 in 0..2 (or 3 at the top)
  const int m1 = tau - (FPT - 1) * l1;
  const bool two = m1 == 0 && l1 >= 2;               // also lag l1 - 1, row m = 3
  double* d1 = own + ((size_t)((k + l1) % ring) * ncell + cell) * FND + a * FPT + m1;
  double* d2 = two ? own + ((size_t)((k + l1 - 1) % ring) * ncell + cell) * FND + a * FPT + (FPT - 1) : nullptr;
  double acc1 = *d1, acc2 = two ? *d2 : 0.0;
  for (int q = q0; q < q1; ++q) {
    const int pq = t_pair[q];
    const unsigned dk = __ldg(g_dark + pq);
    const double y = __ldg(Y + (long long)pq * M + j);
    if (!((dk >> (l1 - 1)) & 1u)) acc1 += y;
    if (two && !((dk >> (l1 - 2)) & 1u)) acc2 += y;
  }
  *d1 = acc1;
  if (two) *d2 = acc2;
}

__global__ void gather_kernel(const int* __restrict__ g_src, long long nil,
                              const double* __restrict__ mom, double* X) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nil * FND;
       e += (long long)gridDim.x * blockDim.x)
    X[e] = mom[(size_t)g_src[e / FND] * FND + (e % FND)];
}


// ------------------------------------------------------------- M2L contraction
// The level tick's M2L (fmm.py:52-69 _toeplitz_apply, :329-368 _do_m2l) in the
// GEMM form, on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64).  One CTA =
// one work item (offset o, up to M2L_NC interaction pairs of that offset):
//   Y[pair][op*256 + a*4 + m] = sum_{b,n} Kx_op[a-b][m-n+toff_op] * mom[src][b*4 + n]
// for every non-dark operator op (lags 1..mu+1 from K0, derivative orders p =
// 1..d from Kp).  The operator is never materialised: the offset's Toeplitz
// tensors (343 spatial differences x 31 / 7 time differences, ~123 KB for
// d = 2) are staged in shared memory once per item and every A fragment is read
// from them directly (address = row part - column part, both precomputed); the
// pairs' source moments are gathered into shared memory (column stride 260
// doubles: conflict-free B fragments).  Each warp owns 32-row blocks (4 m8 x 4 n8
// DMMA tiles, 16 accumulators) of the stacked operator rows; the epilogue writes
// the pair-major output Y that scatter_all_kernel sums per target cell in
// group order (deterministic, as with the library GEMM it replaces).
constexpr int M2L_NC = 32;            // pairs (columns) per work item
constexpr int M2L_BLD = FND + 4;      // shared-memory column stride of the gathered moments
constexpr int M2L_WARPS = 8;

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// shared-memory tables, each padded to an even number of doubles (16-byte aligned)
__host__ __device__ constexpr int m2l_even(int n) { return (n + 1) & ~1; }
__host__ __device__ constexpr size_t m2l_smem_bytes(int d, int ntau0, int ntaup) {
  return sizeof(double) * ((size_t)m2l_even(FKR * ntau0) + (size_t)d * m2l_even(FKR * ntaup) +
                           (size_t)M2L_NC * M2L_BLD);
}

// S(x) = 49 x1 + 7 x2 + x3 of spatial node x = (x1 << 4) | (x2 << 2) | x3: the
// Toeplitz row of (a, b) is S(a) - S(b) + 171
__device__ __forceinline__ int m2l_S(int x) { return 49 * (x >> 4) + 7 * ((x >> 2) & 3) + (x & 3); }

template <int D>
__global__ void __launch_bounds__(M2L_WARPS * 32, 1)
m2l_dmma_kernel(const int4* __restrict__ items, const double* __restrict__ K0, const double* __restrict__ Kp,
                const int* __restrict__ g_src, const unsigned* __restrict__ dark, const double* __restrict__ mom,
                int noff, int ntau0, int ntaup, int mu, double* __restrict__ Y) {
  extern __shared__ __align__(16) double m2l_sm[];
  const int4 it = items[blockIdx.x];  // (offset, first grouped pair, pairs)
  const int o = it.x, p0 = it.y, np = it.z;
  const int tp_stride = m2l_even(FKR * ntaup);
  double* T0 = m2l_sm;                                   // [343][ntau0]
  double* Tp = T0 + m2l_even(FKR * ntau0);               // [D][343][ntaup] (stride tp_stride)
  double* Bs = Tp + (size_t)D * tp_stride;               // [M2L_NC][M2L_BLD], 16-byte aligned
  const int tid = threadIdx.x, nthr = M2L_WARPS * 32;
  {
    const double* src0 = K0 + (size_t)o * FKR * ntau0;
    for (int e = tid; e < FKR * ntau0; e += nthr) T0[e] = __ldg(src0 + e);
    for (int p = 0; p < D; ++p) {
      const double* srcp = Kp + ((size_t)p * noff + o) * FKR * ntaup;
      for (int e = tid; e < FKR * ntaup; e += nthr) Tp[p * tp_stride + e] = __ldg(srcp + e);
    }
    // gathered source moments, two doubles per thread and step (zero columns past np)
    for (int e = tid; e < M2L_NC * (FND / 2); e += nthr) {
      const int j = e / (FND / 2), k2 = e % (FND / 2);
      double2 v = make_double2(0.0, 0.0);
      if (j < np) v = __ldg(reinterpret_cast<const double2*>(mom + (size_t)g_src[p0 + j] * FND) + k2);
      *reinterpret_cast<double2*>(Bs + j * M2L_BLD + 2 * k2) = v;
    }
  }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5;
  // Rows of the contraction: the near-future lags l = 1..mu+1 read the time
  // differences m - n + l (pt - 1) of K0, and lag l's row m = pt-1 is lag l+1's
  // row m = 0: the (mu+1) pt rows per spatial node have only NT = (mu+1)(pt-1)+1
  // distinct time offsets tau = m + l (pt-1).  Each is computed once: rows
  // (a, tau) for a in 0..63, tau in pt-1 .. (mu+2)(pt-1) (64 NT rows; the
  // scatter reads both lags from the shared row -- the same products, 18% fewer
  // FLOPs at mu = 8), then the d derivative operators (a, m) (256 rows each).
  const int NT = (mu + 1) * (FPT - 1) + 1;
  const int nnear = 2 * NT;                  // 32-row blocks of the near-future rows (64 NT / 32)
  const int lr = lane >> 2, lc = lane & 3;  // fragment row / column of this lane
  const int nblk = nnear + D * (FND / 32);
  const long long M = 64LL * NT + (long long)D * FND;
  for (int blk = warp; blk < nblk; blk += M2L_WARPS) {
    const bool nearf = blk < nnear;
    const int r0 = nearf ? blk * 32 : (blk - nnear) % 8 * 32;
    const double* Tb = nearf ? T0 : Tp + (size_t)((blk - nnear) / 8) * tp_stride;
    const int ld = nearf ? ntau0 : ntaup;
    // row part of the A address per m8 tile: (S(a) + 171) * ld + time offset
    int rowp[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int row = r0 + 8 * t + lr;
      rowp[t] = nearf ? (m2l_S(row / NT) + 171) * ld + (FPT - 1) + row % NT
                      : (m2l_S(row >> 2) + 171) * ld + (row & 3) + (FPT - 1);
    }
    double acc[4][4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
    const double* Bl = Bs + lr * M2L_BLD + lc;  // B[k = lc][col = lr] of n8 tile 0
#pragma unroll 4
    for (int b = 0; b < FN3; ++b) {               // k-step: spatial source node b, n = 0..3
      const int colp = m2l_S(b) * ld + lc;
      double af[4], bf[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) af[t] = Tb[rowp[t] - colp];
#pragma unroll
      for (int u = 0; u < 4; ++u) bf[u] = Bl[u * 8 * M2L_BLD + b * FPT];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma884(acc[t][u][0], acc[t][u][1], af[t], bf[u]);
    }
    // epilogue: C[row lr][col 2 lc + i] of tile (t, u) -> Y[pair][block row]
    const long long yrow = nearf ? (long long)r0 : 64LL * NT + (long long)(blk - nnear) * 32;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int col = u * 8 + 2 * lc + i;
        if (col >= np) continue;
        double* yc = Y + (long long)(p0 + col) * M + yrow + lr;
#pragma unroll
        for (int t = 0; t < 4; ++t) yc[8 * t] = acc[t][u][i];
      }
  }
}

// distant-future recurrence, elementwise (fmm.py:355-367)
template <int D>
__global__ void recurrence_kernel(double* own, double* deriv, double* aux, const double* tmp,
                                  int ncell, int mu, int k, double T) {
  const int ring = mu + 3;
  const size_t cs = (size_t)ncell * FND;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < cs; e += (size_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int p = 1; p <= D; ++p) {
      double upd = tmp[(size_t)(p - 1) * cs + e];
#pragma unroll
      for (int mm = 0; mm <= p - 2; ++mm)
        upd = upd + cmp_coeff_dev(p, mm, k) * aux[(size_t)((p - 2) * (p - 1) / 2 + mm) * cs + e];
      deriv[(size_t)(p - 1) * cs + e] += upd;
    }
    double v = own[(size_t)((k + mu + 1) % ring) * cs + e];
    double Tq = 1.0;
#pragma unroll
    for (int p = 1; p <= D; ++p) {
      Tq *= T;
      v += deriv[(size_t)(p - 1) * cs + e] * Tq;
    }
    own[(size_t)((k + mu + 2) % ring) * cs + e] = v;
#pragma unroll
    for (int p = 2; p <= D; ++p)
#pragma unroll
      for (int mm = 0; mm <= p - 2; ++mm) {
        double km = 1.0;
        for (int q = 0; q < mm; ++q) km *= (double)k;
        aux[(size_t)((p - 2) * (p - 1) / 2 + mm) * cs + e] += tmp[(size_t)(p - 1) * cs + e] * km;
      }
  }
}

// ---------------------------------------------------------------- M2M / L2L
// index order of a 256-vector: ((a1*4 + a2)*4 + a3)*4 + m
__device__ __forceinline__ void mode_product(double* X, double* Y, const double (*T)[FPS],
                                             int mode, bool transpose, int e) {
  // e = output element index; Y[e] = sum_k T'[out_k][k] X[e with index(mode) = k]
  int idx[4] = {e >> 6, (e >> 4) & 3, (e >> 2) & 3, e & 3};
  const int o = idx[mode];
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    idx[mode] = k;
    const int src = ((idx[0] * 4 + idx[1]) * 4 + idx[2]) * 4 + idx[3];
    s += (transpose ? T[k][o] : T[o][k]) * X[src];
  }
  Y[e] = s;
}

__global__ void __launch_bounds__(FND) m2m_kernel(const int* __restrict__ child_ptr,
                                                  const int* __restrict__ child_idx,
                                                  const int* __restrict__ octant,
                                                  const double* __restrict__ mom_child, int half,
                                                  Tr tr, double* acc_parent) {
  const int P = blockIdx.x, e = threadIdx.x;
  __shared__ double X[FND], Y[FND];
  double sum = 0.0;
  for (int q = child_ptr[P]; q < child_ptr[P + 1]; ++q) {
    const int c = child_idx[q];
    const double v = mom_child[(size_t)c * FND + e];
    __syncthreads();
    X[e] = v;
    if (!__syncthreads_or(v != 0.0)) continue;
    const int oc = octant[c];
    mode_product(X, Y, tr.s[oc & 1], 0, false, e);
    __syncthreads();
    mode_product(Y, X, tr.s[(oc >> 1) & 1], 1, false, e);
    __syncthreads();
    mode_product(X, Y, tr.s[(oc >> 2) & 1], 2, false, e);
    __syncthreads();
    mode_product(Y, X, tr.t[half], 3, false, e);
    __syncthreads();
    sum += X[e];
  }
  acc_parent[(size_t)P * FND + e] += sum;
}

__global__ void __launch_bounds__(FND) l2l_kernel(const int* __restrict__ parent,
                                                  const int* __restrict__ octant,
                                                  const double* __restrict__ own_p,
                                                  const double* __restrict__ inh_p, Tr tr,
                                                  double* inh_c0, double* inh_c1) {
  const int c = blockIdx.x, e = threadIdx.x;
  const int P = parent[c];
  __shared__ double X[FND], Y[FND], Z[FND];
  const double tot = own_p[(size_t)P * FND + e] + inh_p[(size_t)P * FND + e];
  Z[e] = tot;
  const bool nz = __syncthreads_or(tot != 0.0);
  const int oc = octant[c];
  for (int half = 0; half < 2; ++half) {
    double* out = half ? inh_c1 : inh_c0;
    if (!nz) {
      out[(size_t)c * FND + e] = 0.0;
      continue;
    }
    __syncthreads();
    mode_product(Z, X, tr.s[oc & 1], 0, true, e);
    __syncthreads();
    mode_product(X, Y, tr.s[(oc >> 1) & 1], 1, true, e);
    __syncthreads();
    mode_product(Y, X, tr.s[(oc >> 2) & 1], 2, true, e);
    __syncthreads();
    mode_product(X, Y, tr.t[half], 3, true, e);
    __syncthreads();
    out[(size_t)c * FND + e] = Y[e];
  }
}

template <typename T>
int up(tdw_ctx* ctx, T** dst, const T* src, size_t n) {
  TDW_CUDA(ctx, cudaMalloc(dst, sizeof(T) * std::max<size_t>(n, 1)));
  if (n) TDW_CUDA(ctx, cudaMemcpy(*dst, src, sizeof(T) * n, cudaMemcpyHostToDevice));
  return TDW_OK;
}

}  // namespace

// ------------------------------------------------------------------ setup
extern "C" int tdw_fmm_setup(tdw_problem* pb, const tdw_fmm_desc* fd) {
  if (!pb || !fd) return TDW_ERR_INVALID_ARG;
  tdw_ctx* ctx = pb->ctx;
  cudaSetDevice(ctx->device);
  if (pb->assembled) return tdw_fail(ctx, TDW_ERR_STATE, "tdw_fmm_setup must precede tdw_assemble");
  if (fd->ps != FPS || fd->pt != FPT || fd->mu < 1 || fd->mu > FMU_MAX)
    return tdw_fail(ctx, TDW_ERR_LIMIT, "FMM supports ps = pt = 4 and mu <= 8");
  const int ns = pb->ns, nt = pb->nt, d = pb->d;
  FmmState* F = new FmmState();
  pb->fmm = F;
  F->mu = fd->mu;
  F->leaf = fd->leaf;
  F->ntau0 = (fd->mu + 2) * (FPT - 1) + 1;
  F->ntaup = 2 * (FPT - 1) + 1;
  F->n_leaf_cells = fd->n_leaf_cells;
  std::vector<int> inv(ns);
  for (int k = 0; k < ns; ++k) inv[pb->perm[k]] = k;
  // near-field filter, window and history padding
  std::vector<int> leafc(ns), ecell(ns);
  for (int k = 0; k < ns; ++k) {
    const int o = pb->perm[k];
    leafc[k] = (int)(fd->leaf_coords[3 * o] | (fd->leaf_coords[3 * o + 1] << 10) |
                     (fd->leaf_coords[3 * o + 2] << 20));
    ecell[k] = (int)fd->elem_cell[o];
  }
  int rc = up(ctx, &pb->d_leafc, leafc.data(), ns);
  if (rc) return rc;
  pb->split_lag2 = 0;
  pb->mode = TDW_MODE_STORED_BAND;  // the near field is always a store
  pb->kb = 1;  // the FMM loop is sequential: one step per convolution pass
  pb->overlap = 1;
  pb->nsl = 1;
  pb->bring = 2;
  pb->skip_empty_units = true;
  pb->cap = std::min(fd->gamma_near, nt - 1);
  pb->n_lags = pb->cap;
  int maxlag = pb->cap;
  for (int x = 0; x < fd->n_extra; ++x) maxlag = std::max(maxlag, fd->extra_lags[x]);
  pb->pad = maxlag + d + 2;
  pb->hstride = pb->pad + nt - 1;
  pb->hcols = pb->ntiles * TDW_TJ;
  cudaFree(pb->d_hist);
  TDW_CUDA(ctx, cudaMalloc(&pb->d_hist, sizeof(double2) * (size_t)pb->hcols * pb->hstride));
  // leaf element data, internal order
  if ((rc = up(ctx, &F->elem_cell, ecell.data(), ns))) return rc;
  {
    std::vector<int> cptr(F->n_leaf_cells + 1, 0), celems;
    std::vector<std::vector<int>> lists(F->n_leaf_cells);
    for (int k = 0; k < ns; ++k) lists[ecell[k]].push_back(k);
    for (int c = 0; c < F->n_leaf_cells; ++c) {
      cptr[c + 1] = cptr[c] + (int)lists[c].size();
      for (int k : lists[c]) celems.push_back(k);
    }
    if ((rc = up(ctx, &F->cell_ptr, cptr.data(), cptr.size()))) return rc;
    if ((rc = up(ctx, &F->cell_elems, celems.data(), celems.size()))) return rc;
  }
  auto rows = [&](const double* src, double** dst) -> int {
    if (!src) return TDW_OK;
    std::vector<double> v((size_t)ns * FN3);
    for (int k = 0; k < ns; ++k)
      std::copy(src + (size_t)pb->perm[k] * FN3, src + (size_t)(pb->perm[k] + 1) * FN3, &v[(size_t)k * FN3]);
    return up(ctx, dst, v.data(), v.size());
  };
  if ((rc = rows(fd->p2m_tau, &F->p2m_tau))) return rc;
  if ((rc = rows(fd->p2m_sig, &F->p2m_sig))) return rc;
  if ((rc = rows(fd->l2p_val, &F->l2p_val))) return rc;
  if (pb->bie == TDW_BIE_BMBIE && (rc = rows(fd->l2p_bm, &F->l2p_bm))) return rc;
  for (int h = 0; h < 2; ++h)
    for (int i = 0; i < FPS; ++i)
      for (int j = 0; j < FPS; ++j) {
        F->t_space[h][i][j] = fd->t_space[(h * FPS + i) * FPS + j];
        F->t_time[h][i][j] = fd->t_time[(h * FPT + i) * FPT + j];
      }
  // Target-cell sharding: a rank owns the leaf cells of its rows
  // (internal order [row_lo, row_hi): RCB blocks, compact patches) and their
  // ancestors.  It runs M2L only into owned observation cells; P2M, M2M, L2L
  // and the recurrence stay whole-tree (cheap) so every owned cell sees the
  // same moments and locals as on one GPU.  Cells straddling two ranks' rows are
  // owned by both (computed twice).
  std::vector<std::vector<char>> owned(F->leaf + 1);
  F->r0 = pb->row_lo;
  F->r1 = pb->row_hi;
  if (F->leaf >= 2) {
    owned[F->leaf].assign(fd->lev_ncell[F->leaf - 2], pb->nranks == 1 ? 1 : 0);
    for (int k = pb->row_lo; k < pb->row_hi; ++k) owned[F->leaf][ecell[k]] = 1;
    long long oc2 = 0;
    std::vector<long long> lev_off(F->leaf + 1, 0);
    for (int li = 0; li < fd->n_levels; ++li) {
      lev_off[2 + li] = oc2;
      oc2 += fd->lev_ncell[li];
    }
    for (int L = F->leaf; L > 2; --L) {
      owned[L - 1].assign(fd->lev_ncell[L - 3], pb->nranks == 1 ? 1 : 0);
      for (int c = 0; c < fd->lev_ncell[L - 2]; ++c)
        if (owned[L][c]) owned[L - 1][(int)fd->lev_parent[lev_off[L] + c]] = 1;
    }
  }
  // levels
  F->lev.resize(F->leaf + 1);
  long long oc = 0, oo = 0, oil = 0, optr = 0, ok0 = 0, okp = 0;
  std::vector<std::vector<int>> parents(F->leaf + 1), octs(F->leaf + 1);
  for (int li = 0; li < fd->n_levels; ++li) {
    const int L = 2 + li;
    FmmLevel& V = F->lev[L];
    V.L = L;
    V.ncell = fd->lev_ncell[li];
    V.noff = fd->lev_noff[li];
    V.interval = fd->lev_interval[li];
    std::vector<int> par(V.ncell), octv(V.ncell);
    for (int c = 0; c < V.ncell; ++c) {
      par[c] = (int)fd->lev_parent[oc + c];
      octv[c] = (int)(fd->lev_octant[3 * (oc + c)] | (fd->lev_octant[3 * (oc + c) + 1] << 1) |
                      (fd->lev_octant[3 * (oc + c) + 2] << 2));
    }
    parents[L] = par;
    octs[L] = octv;
    if ((rc = up(ctx, &V.parent, par.data(), par.size()))) return rc;
    if ((rc = up(ctx, &V.octant, octv.data(), octv.size()))) return rc;
    const long long nil = fd->lev_nil[li];
    std::vector<long long> optr_v(fd->lev_obs_ptr + optr, fd->lev_obs_ptr + optr + V.ncell + 1);
    std::vector<int> src(nil), off(nil);
    for (long long q = 0; q < nil; ++q) {
      src[q] = (int)fd->lev_il_src[oil + q];
      off[q] = (int)fd->lev_il_off[oil + q];
    }
    if ((rc = up(ctx, &V.obs_ptr, optr_v.data(), optr_v.size()))) return rc;
    if ((rc = up(ctx, &V.il_src, src.data(), src.size()))) return rc;
    if ((rc = up(ctx, &V.il_off, off.data(), off.size()))) return rc;
    std::vector<unsigned> dark(V.noff, 0);
    for (int o = 0; o < V.noff; ++o)
      for (int l = 1; l <= F->mu + 1; ++l)
        if (fd->lev_dark[(oo + o) * (F->mu + 1) + l - 1]) dark[o] |= 1u << (l - 1);
    if ((rc = up(ctx, &V.dark, dark.data(), dark.size()))) return rc;
    if ((rc = up(ctx, &V.K0, fd->lev_K0 + ok0, (size_t)V.noff * FKR * F->ntau0))) return rc;
    if ((rc = up(ctx, &V.Kp, fd->lev_Kp + okp, (size_t)d * V.noff * FKR * F->ntaup))) return rc;
    {
      // interaction pairs grouped by offset (stable: by observer within a group)
      // (a shard keeps the pairs whose observation cell it owns)
      std::vector<long long> grp(V.noff + 1, 0);
      std::vector<int> obs_of(nil);
      for (int c = 0; c < V.ncell; ++c)
        for (long long q = optr_v[c]; q < optr_v[c + 1]; ++q) obs_of[q] = c;
      long long nkeep = 0;
      for (long long q = 0; q < nil; ++q)
        if (owned[L][obs_of[q]]) {
          grp[off[q] + 1]++;
          ++nkeep;
        }
      std::vector<int> gobs(nkeep), gsrc(nkeep);
      for (int o = 0; o < V.noff; ++o) grp[o + 1] += grp[o];
      std::vector<long long> fillp(grp.begin(), grp.end() - 1);
      for (long long q = 0; q < nil; ++q) {
        if (!owned[L][obs_of[q]]) continue;
        const long long t = fillp[off[q]]++;
        gobs[t] = obs_of[q];
        gsrc[t] = src[q];
      }
      V.grp = grp;
      V.nil = nkeep;
      F->m2l_pairs += nkeep;
      {
        std::vector<int> tptr(V.ncell + 1, 0), tpair(nkeep), tcells;
        for (long long q = 0; q < nkeep; ++q) tptr[gobs[q] + 1]++;
        for (int c = 0; c < V.ncell; ++c) {
          if (tptr[c + 1] > 0) tcells.push_back(c);
          tptr[c + 1] += tptr[c];
        }
        std::vector<int> fill(tptr.begin(), tptr.end() - 1);
        for (long long q = 0; q < nkeep; ++q) tpair[fill[gobs[q]]++] = (int)q;  // ascending = group order
        V.n_tcell = (int)tcells.size();
        if ((rc = up(ctx, &V.t_ptr, tptr.data(), tptr.size()))) return rc;
        if ((rc = up(ctx, &V.t_pair, tpair.data(), std::max<size_t>(1, tpair.size())))) return rc;
        if ((rc = up(ctx, &V.t_cells, tcells.data(), std::max<size_t>(1, tcells.size())))) return rc;
      }
      for (int o = 0; o < V.noff; ++o) V.max_grp = std::max(V.max_grp, grp[o + 1] - grp[o]);
      {
        std::vector<int4> items;
        std::vector<unsigned> gd(std::max<long long>(1, nkeep), 0u);
        for (int o = 0; o < V.noff; ++o) {
          for (long long q = grp[o]; q < grp[o + 1]; ++q) gd[q] = dark[o];
          for (long long q = grp[o]; q < grp[o + 1]; q += M2L_NC)
            items.push_back(make_int4(o, (int)q, (int)std::min<long long>(M2L_NC, grp[o + 1] - q), 0));
        }
        V.n_items = (int)items.size();
        // executed FLOPs: 64 NT shared near-future rows + d * 256 derivative rows per pair
        const double rows = 64.0 * ((F->mu + 1) * (FPT - 1) + 1) + (double)d * FND;
        V.m2l_flops = 2.0 * FND * rows * (double)nkeep;
        if ((rc = up(ctx, &V.items, items.data(), std::max<size_t>(1, items.size())))) return rc;
        if ((rc = up(ctx, &V.g_dark, gd.data(), gd.size()))) return rc;
      }
      if ((rc = up(ctx, &V.g_obs, gobs.data(), gobs.size()))) return rc;
      if ((rc = up(ctx, &V.g_src, gsrc.data(), gsrc.size()))) return rc;
      const int nops = F->mu + 1 + d;
      F->nops = nops;
      {
        const int smem = (int)m2l_smem_bytes(d, F->ntau0, F->ntaup);
        cudaError_t ea = d == 1 ? cudaFuncSetAttribute(m2l_dmma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)
                       : d == 2 ? cudaFuncSetAttribute(m2l_dmma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)
                                : cudaFuncSetAttribute(m2l_dmma_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        TDW_CUDA(ctx, ea);
      }
      const size_t kop = (size_t)V.noff * FND * nops * FND;
      TDW_CUDA(ctx, cudaMalloc(&V.Kop, sizeof(double) * std::max<size_t>(1, kop)));
      if (V.noff)
        build_kop_kernel<<<4096, 256, 0, ctx->stream>>>(V.K0, V.Kp, V.noff, F->ntau0, F->ntaup, F->mu,
                                                         d, V.Kop);
      TDW_CUDA(ctx, cudaGetLastError());
      TDW_CUDA(ctx, cudaMalloc(&V.X, sizeof(double) * std::max<long long>(1, V.nil) * FND));
      TDW_CUDA(ctx, cudaMalloc(&V.tmp, sizeof(double) * d * (size_t)V.ncell * FND));
    }
    oc += V.ncell;
    oo += V.noff;
    oil += nil;
    optr += V.ncell + 1;
    ok0 += (long long)V.noff * FKR * F->ntau0;
    okp += (long long)d * V.noff * FKR * F->ntaup;
    const size_t cs = (size_t)V.ncell * FND;
    const int naux = d * (d - 1) / 2;
    TDW_CUDA(ctx, cudaMalloc(&V.own, sizeof(double) * (F->mu + 3) * cs));
    TDW_CUDA(ctx, cudaMalloc(&V.inherit, sizeof(double) * 4 * cs));
    TDW_CUDA(ctx, cudaMalloc(&V.deriv, sizeof(double) * d * cs));
    TDW_CUDA(ctx, cudaMalloc(&V.aux, sizeof(double) * std::max(1, naux) * cs));
    TDW_CUDA(ctx, cudaMalloc(&V.acc, sizeof(double) * cs));
    TDW_CUDA(ctx, cudaMalloc(&V.mom, sizeof(double) * cs));
  }
  // children lists (level L cells of each level L-1 parent, ascending)
  for (int L = 3; L <= F->leaf; ++L) {
    FmmLevel& P = F->lev[L - 1];
    std::vector<int> cptr(P.ncell + 1, 0), cidx;
    std::vector<std::vector<int>> ch(P.ncell);
    for (int c = 0; c < F->lev[L].ncell; ++c) ch[parents[L][c]].push_back(c);
    for (int p = 0; p < P.ncell; ++p) {
      cptr[p + 1] = cptr[p] + (int)ch[p].size();
      for (int c : ch[p]) cidx.push_back(c);
    }
    if ((rc = up(ctx, &P.child_ptr, cptr.data(), cptr.size()))) return rc;
    if ((rc = up(ctx, &P.child_idx, cidx.data(), cidx.size()))) return rc;
  }
  // extra lists: rows/cols in internal order, coefficient tables on the device
  long long oe = 0;
  for (int x = 0; x < fd->n_extra; ++x) {
    FmmExtra E;
    E.lags = fd->extra_lags[x];
    E.npair = fd->extra_npair[x];
    std::vector<std::pair<int, int>> pr;  // this shard's rows only
    pr.reserve(fd->extra_npair[x]);
    for (long long p = 0; p < fd->extra_npair[x]; ++p) {
      const int i = inv[fd->extra_i[oe + p]];
      if (i >= pb->row_lo && i < pb->row_hi) pr.push_back({i, inv[fd->extra_j[oe + p]]});
    }
    E.npair = (long long)pr.size();
    std::stable_sort(pr.begin(), pr.end(), [](auto& u, auto& v) { return u.first < v.first; });
    std::vector<int> rp(ns + 1, 0), col(E.npair), rof(E.npair);
    for (long long p = 0; p < E.npair; ++p) {
      rp[pr[p].first + 1]++;
      col[p] = pr[p].second;
      rof[p] = pr[p].first;
    }
    for (int i = 0; i < ns; ++i) rp[i + 1] += rp[i];
    if ((rc = up(ctx, &E.row_ptr, rp.data(), rp.size()))) return rc;
    if ((rc = up(ctx, &E.col, col.data(), col.size()))) return rc;
    if ((rc = up(ctx, &E.row_of, rof.data(), rof.size()))) return rc;
    TDW_CUDA(ctx, cudaMalloc(&E.U, sizeof(double) * std::max<long long>(1, E.npair * E.lags)));
    TDW_CUDA(ctx, cudaMalloc(&E.W, sizeof(double) * std::max<long long>(1, E.npair * E.lags)));
    if (E.npair) {
      const bool bm = pb->bie == TDW_BIE_BMBIE;
      const int blocks = (int)std::min<long long>((E.npair + 127) / 128, 4096);
#define TDW_X(DD, BB)                                                                            \
  extra_coeff_kernel<DD, BB><<<blocks, 128, 0, ctx->stream>>>(pb->d_elem, E.row_of, E.col, E.npair, \
                                                               E.lags, pb->c, pb->dt, pb->K, E.U, E.W)
      if (d == 1) { if (bm) TDW_X(1, true); else TDW_X(1, false); }
      if (d == 2) { if (bm) TDW_X(2, true); else TDW_X(2, false); }
      if (d == 3) { if (bm) TDW_X(3, true); else TDW_X(3, false); }
#undef TDW_X
      TDW_CUDA(ctx, cudaGetLastError());
    }
    E.gmax.assign(fd->extra_gmax + (size_t)x * nt, fd->extra_gmax + (size_t)(x + 1) * nt);
    oe += fd->extra_npair[x];
    F->extra.push_back(std::move(E));
  }
  {
    long long mg = 1;
    for (int L = 2; L <= F->leaf; ++L) mg = std::max(mg, F->lev[L].nil);  // all groups of a level
    TDW_CUDA(ctx, cudaMalloc(&F->Y, sizeof(double) * (size_t)mg * std::max(1, F->nops) * FND));
    // grouped-GEMM descriptors per level (pointers into Kop, X, Y are fixed)
    const int M = F->nops * FND;
    for (int L = 2; L <= F->leaf; ++L) {
      FmmLevel& V = F->lev[L];
      std::vector<const double*> A, B;
      std::vector<double*> Cp;
      for (int o = 0; o < V.noff; ++o) {
        const long long p0 = V.grp[o], np = V.grp[o + 1] - V.grp[o];
        if (np == 0) continue;
        A.push_back(V.Kop + (size_t)o * FND * M);
        B.push_back(V.X + (size_t)p0 * FND);
        Cp.push_back(F->Y + (size_t)p0 * M);
        V.gm.push_back(M);
        V.gn.push_back((int)np);
        V.gk.push_back(FND);
        V.glda.push_back(M);
        V.gldb.push_back(FND);
        V.gldc.push_back(M);
        V.gsize.push_back(1);
        V.galpha.push_back(1.0);
        V.gbeta.push_back(0.0);
        V.gop.push_back(CUBLAS_OP_N);
      }
      if (!A.empty()) {
        TDW_CUDA(ctx, cudaMalloc(&V.gA, sizeof(double*) * A.size()));
        TDW_CUDA(ctx, cudaMalloc(&V.gB, sizeof(double*) * B.size()));
        TDW_CUDA(ctx, cudaMalloc(&V.gC, sizeof(double*) * Cp.size()));
        TDW_CUDA(ctx, cudaMemcpy(V.gA, A.data(), sizeof(double*) * A.size(), cudaMemcpyHostToDevice));
        TDW_CUDA(ctx, cudaMemcpy(V.gB, B.data(), sizeof(double*) * B.size(), cudaMemcpyHostToDevice));
        TDW_CUDA(ctx, cudaMemcpy(V.gC, Cp.data(), sizeof(double*) * Cp.size(), cudaMemcpyHostToDevice));
      }
    }
    if (cublasCreate(&F->blas) != CUBLAS_STATUS_SUCCESS)
      return tdw_fail(ctx, TDW_ERR_CUDA, "cublasCreate failed");
    cublasSetMathMode(F->blas, CUBLAS_DEFAULT_MATH);
  }
  F->ticks_before.assign(fd->ticks_before, fd->ticks_before + nt);
  F->k_obs.assign(fd->k_obs, fd->k_obs + nt);
  F->wt.assign(fd->wt, fd->wt + (size_t)nt * FPT);
  F->dwt.assign(fd->dwt, fd->dwt + (size_t)nt * FPT);
  F->wts.assign(fd->wts, fd->wts + (size_t)nt * FPT);
  TDW_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return TDW_OK;
}

// ------------------------------------------------------------------ loop
namespace {

Tr make_tr(const FmmState* F) {
  Tr t;
  for (int h = 0; h < 2; ++h)
    for (int i = 0; i < FPS; ++i)
      for (int j = 0; j < FPS; ++j) {
        t.s[h][i][j] = F->t_space[h][i][j];
        t.t[h][i][j] = F->t_time[h][i][j];
      }
  return t;
}

int snapshot(tdw_ctx* ctx, FmmLevel& V, cudaStream_t st) {
  const size_t cs = (size_t)V.ncell * FND * sizeof(double);
  TDW_CUDA(ctx, cudaMemcpyAsync(V.mom, V.acc, cs, cudaMemcpyDeviceToDevice, st));
  TDW_CUDA(ctx, cudaMemsetAsync(V.acc, 0, cs, st));
  return TDW_OK;
}

void m2l_launch(int d, const FmmLevel& V, const FmmState* F, size_t smem, cudaStream_t st) {
  auto go = [&](auto kern) {
    kern<<<V.n_items, M2L_WARPS * 32, smem, st>>>(V.items, V.K0, V.Kp, V.g_src, V.dark, V.mom, V.noff,
                                                  F->ntau0, F->ntaup, F->mu, F->Y);
  };
  if (d == 1) go(m2l_dmma_kernel<1>);
  if (d == 2) go(m2l_dmma_kernel<2>);
  if (d == 3) go(m2l_dmma_kernel<3>);
}

int launch_m2l(tdw_problem* pb, FmmLevel& V, int k, cudaStream_t st) {
  FmmState* F = pb->fmm;
  tdw_ctx* ctx = pb->ctx;
  const int d = pb->d, nops = F->nops, M = nops * FND;
  TDW_CUDA(ctx, cudaMemsetAsync(V.tmp, 0, sizeof(double) * d * (size_t)V.ncell * FND, st));
  static const bool use_blas = getenv("TDW_M2L") && strcmp(getenv("TDW_M2L"), "cublas") == 0;
  if (V.nil > 0 && !use_blas) {
    // own DMMA contraction straight from the Toeplitz tensors and the moments
    const size_t smem = m2l_smem_bytes(d, F->ntau0, F->ntaup);
    m2l_launch(d, V, F, smem, st);
    TDW_CUDA(ctx, cudaGetLastError());
    if (V.n_tcell > 0)
    {
      const int NT = (F->mu + 1) * (FPT - 1) + 1;
      const int rows = 64 * NT + d * FND;
      scatter_tau_kernel<<<dim3(V.n_tcell, (rows + 255) / 256), 256, 0, st>>>(V.t_cells, V.t_ptr, V.t_pair, V.g_dark,
                                                                            F->Y, d, F->mu, k, V.ncell, V.own, V.tmp);
    }
    TDW_CUDA(ctx, cudaGetLastError());
  } else if (V.nil > 0) {
    gather_kernel<<<(int)std::min<long long>(4096, (V.nil * FND + 255) / 256), 256, 0, st>>>(
        V.g_src, V.nil, V.mom, V.X);
    TDW_CUDA(ctx, cudaGetLastError());
    if (cublasSetStream(F->blas, st) != CUBLAS_STATUS_SUCCESS)
      return tdw_fail(ctx, TDW_ERR_CUDA, "cublasSetStream failed");
    const double one = 1.0, zero = 0.0;
    static const bool grouped = !(getenv("TDW_GROUPED_GEMM") && atoi(getenv("TDW_GROUPED_GEMM")) == 0);
    if (grouped && V.gA) {
      cublasStatus_t bs = cublasDgemmGroupedBatched(
          F->blas, V.gop.data(), V.gop.data(), V.gm.data(), V.gn.data(), V.gk.data(), V.galpha.data(), V.gA,
          V.glda.data(), V.gB, V.gldb.data(), V.gbeta.data(), V.gC, V.gldc.data(), (int)V.gm.size(),
          V.gsize.data());
      if (bs != CUBLAS_STATUS_SUCCESS) return tdw_fail(ctx, TDW_ERR_CUDA, "cublasDgemmGroupedBatched failed");
    }
    for (int o = 0; o < (grouped && V.gA ? 0 : V.noff); ++o) {
      const long long p0 = V.grp[o], np = V.grp[o + 1] - V.grp[o];
      if (np == 0) continue;
      // Y (M x np) = Kop_o (M x 256) * X (256 x np), column-major
      cublasStatus_t bs = cublasDgemm(F->blas, CUBLAS_OP_N, CUBLAS_OP_N, M, (int)np, FND, &one,
                                      V.Kop + (size_t)o * FND * M, M, V.X + (size_t)p0 * FND, FND,
                                      &zero, F->Y + (size_t)p0 * M, M);
      if (bs != CUBLAS_STATUS_SUCCESS) return tdw_fail(ctx, TDW_ERR_CUDA, "cublasDgemm failed");
    }
    if (V.n_tcell > 0)
      scatter_all_kernel<<<dim3(V.n_tcell, nops), FND, 0, st>>>(V.t_cells, V.t_ptr, V.t_pair, nullptr, F->Y,
                                                                 nops, F->mu, k, V.ncell, V.own, V.tmp, 0);
    TDW_CUDA(ctx, cudaGetLastError());
  }
  const size_t cs = (size_t)V.ncell * FND;
  const int blocks = (int)std::min<size_t>(4096, (cs + 255) / 256);
  const double T = pb->c * V.interval;
  if (d == 1) recurrence_kernel<1><<<blocks, 256, 0, st>>>(V.own, V.deriv, V.aux, V.tmp, V.ncell, F->mu, k, T);
  if (d == 2) recurrence_kernel<2><<<blocks, 256, 0, st>>>(V.own, V.deriv, V.aux, V.tmp, V.ncell, F->mu, k, T);
  if (d == 3) recurrence_kernel<3><<<blocks, 256, 0, st>>>(V.own, V.deriv, V.aux, V.tmp, V.ncell, F->mu, k, T);
  TDW_CUDA(ctx, cudaGetLastError());
  return TDW_OK;
}

// fmm.py:371-419
int tick(tdw_problem* pb, int k_leaf, cudaStream_t st) {
  FmmState* F = pb->fmm;
  tdw_ctx* ctx = pb->ctx;
  const int leaf = F->leaf;
  if (leaf < 2) return TDW_OK;
  const Tr tr = make_tr(F);
  std::vector<int> completed{leaf};
  int rc = snapshot(ctx, F->lev[leaf], st);
  if (!rc) rc = launch_m2l(pb, F->lev[leaf], k_leaf, st);
  if (rc) return rc;
  int cur_k = k_leaf, L = leaf;
  while (L - 1 >= 2) {
    const int half = cur_k & 1;
    FmmLevel& P = F->lev[L - 1];
    m2m_kernel<<<P.ncell, FND, 0, st>>>(P.child_ptr, P.child_idx, F->lev[L].octant, F->lev[L].mom,
                                         half, tr, P.acc);
    TDW_CUDA(ctx, cudaGetLastError());
    if (half == 0) break;
    cur_k >>= 1;
    L -= 1;
    completed.push_back(L);
    if ((rc = snapshot(ctx, F->lev[L], st))) return rc;
    if ((rc = launch_m2l(pb, F->lev[L], cur_k, st))) return rc;
  }
  std::sort(completed.begin(), completed.end());
  const int ring = F->mu + 3;
  for (int Lc : completed) {
    if (Lc + 1 > leaf) continue;
    const int kl = k_leaf >> (leaf - Lc);
    FmmLevel& P = F->lev[Lc];
    FmmLevel& C = F->lev[Lc + 1];
    const size_t csp = (size_t)P.ncell * FND, csc = (size_t)C.ncell * FND;
    const int k0 = 2 * (kl + 1), k1 = 2 * (kl + 1) + 1;
    l2l_kernel<<<C.ncell, FND, 0, st>>>(C.parent, C.octant, P.own + ((kl + 1) % ring) * csp,
                                         P.inherit + ((kl + 1) % 4) * csp, tr,
                                         C.inherit + (k0 % 4) * csc, C.inherit + (k1 % 4) * csc);
    TDW_CUDA(ctx, cudaGetLastError());
  }
  return TDW_OK;
}

}  // namespace

// launched from march.cu's helpers
int launch_conv_fmm(tdw_problem* pb, void* plan, int alpha, cudaStream_t s);
int launch_solve_fmm(tdw_problem* pb, void* plan, int alpha, cudaStream_t s);
int make_plan_fmm(tdw_problem* pb, void** plan, double threshold, bool want_rhs);
void free_plan_fmm(void* plan);
int begin_loop_fmm(tdw_problem* pb, cudaStream_t st);

namespace {

// Per-step pieces of the FMM loop, shared by the single-GPU / NCCL loop and the
// one-GPU emulation of R shards (tdw_fmm_march_emulated).
struct FmmRun {
  void* plan = nullptr;
  long long last_tick = -1;
};

int fmm_begin(tdw_problem* pb, FmmRun& R, double threshold, bool want_rhs, cudaStream_t st) {
  tdw_ctx* ctx = pb->ctx;
  FmmState* F = pb->fmm;
  if (want_rhs) {
    if (!pb->d_rhs)
      TDW_CUDA(ctx, cudaMalloc(&pb->d_rhs, sizeof(double) * (size_t)(pb->nt - 1) * pb->ns));
    TDW_CUDA(ctx, cudaMemsetAsync(pb->d_rhs, 0, sizeof(double) * (size_t)(pb->nt - 1) * pb->ns, st));
  }
  int rc = make_plan_fmm(pb, &R.plan, threshold, want_rhs);
  if (rc) return rc;
  if ((rc = begin_loop_fmm(pb, st))) return rc;
  for (int L = 2; L <= F->leaf; ++L) {
    FmmLevel& V = F->lev[L];
    const size_t cs = (size_t)V.ncell * FND * sizeof(double);
    TDW_CUDA(ctx, cudaMemsetAsync(V.own, 0, cs * (F->mu + 3), st));
    TDW_CUDA(ctx, cudaMemsetAsync(V.inherit, 0, cs * 4, st));
    TDW_CUDA(ctx, cudaMemsetAsync(V.deriv, 0, cs * pb->d, st));
    TDW_CUDA(ctx, cudaMemsetAsync(V.aux, 0, cs * std::max(1, pb->d * (pb->d - 1) / 2), st));
    TDW_CUDA(ctx, cudaMemsetAsync(V.acc, 0, cs, st));
  }
  R.last_tick = -1;
  return TDW_OK;
}

StepW step_weights(const FmmState* F, int alpha) {
  StepW sw;
  for (int m = 0; m < FPT; ++m) {
    sw.wt[m] = F->wt[(size_t)alpha * FPT + m];
    sw.dwt[m] = F->dwt[(size_t)alpha * FPT + m];
    sw.wts[m] = F->wts[(size_t)alpha * FPT + m];
  }
  return sw;
}

// far-field ticks due before step alpha, then this shard's rows of b: near field
// (banded store), extra lists, L2P
int fmm_step_rhs(tdw_problem* pb, FmmRun& R, int alpha, cudaStream_t st) {
  tdw_ctx* ctx = pb->ctx;
  FmmState* F = pb->fmm;
  int rc;
  while (R.last_tick < F->ticks_before[alpha]) {
    if ((rc = tick(pb, (int)(R.last_tick + 1), st))) return rc;
    ++R.last_tick;
  }
  double* b = pb->d_b + (alpha & 1) * pb->bstride;
  if ((rc = launch_conv_fmm(pb, R.plan, alpha, st))) return rc;  // near field -> b (own rows)
  const int nrow = F->r1 - F->r0;
  const int rblocks = std::max(1, (nrow + 127) / 128);
  for (auto& E : F->extra) {
    const int g = (int)E.gmax[alpha];
    if (g <= 0 || E.npair == 0) continue;
    extra_apply_kernel<<<std::max(1, (nrow + 3) / 4), 128, 0, st>>>(E.row_ptr, E.col, E.U, E.W, E.lags, g, pb->d_hist,
                                                 pb->hcols, pb->pad, alpha, pb->d, F->r0, F->r1, b,
                                                 pb->d_flags);
  }
  FmmLevel* LV = F->leaf >= 2 ? &F->lev[F->leaf] : nullptr;
  if (LV) {
    const int ring = F->mu + 3;
    const long long ko = F->k_obs[alpha];
    l2p_kernel<<<rblocks, 128, 0, st>>>(F->elem_cell, LV->own, LV->inherit, (int)(ko % ring), (int)(ko % 4),
                                         LV->ncell, F->l2p_val,
                                         pb->bie == TDW_BIE_BMBIE ? F->l2p_bm : nullptr, step_weights(F, alpha),
                                         F->r0, F->r1, b, pb->d_flags);
  }
  TDW_CUDA(ctx, cudaGetLastError());
  return TDW_OK;
}

// the (redundant) lag-1 solve on the full b, then the step's sources into the leaf moments
int fmm_step_solve(tdw_problem* pb, FmmRun& R, int alpha, cudaStream_t st) {
  tdw_ctx* ctx = pb->ctx;
  FmmState* F = pb->fmm;
  int rc = launch_solve_fmm(pb, R.plan, alpha, st);
  if (rc) return rc;
  FmmLevel* LV = F->leaf >= 2 ? &F->lev[F->leaf] : nullptr;
  if (LV)
    p2m_kernel<<<LV->ncell, FN3, 0, st>>>(F->cell_ptr, F->cell_elems, F->p2m_tau, F->p2m_sig, pb->d_hist,
                                           pb->hcols, pb->pad, alpha - 1, pb->d, step_weights(F, alpha),
                                           LV->acc, pb->d_flags);
  TDW_CUDA(ctx, cudaGetLastError());
  return TDW_OK;
}

int fmm_check(tdw_problem* pb) {
  int hflags[4];
  TDW_CUDA(pb->ctx, cudaMemcpy(hflags, pb->d_flags, sizeof(hflags), cudaMemcpyDeviceToHost));
  if (hflags[0] == 2) return tdw_fail(pb->ctx, TDW_ERR_RESIDUAL, "FMM step: solve residual too large");
  return TDW_OK;
}

}  // namespace

int tdw_fmm_loop(tdw_problem* pb, double threshold, bool want_rhs, tdw_timing* timing) {
  tdw_ctx* ctx = pb->ctx;
  cudaStream_t st = ctx->stream;
  // the exchange runs whenever the context has a communicator (a one-rank
  // communicator exercises it on one GPU, as the direct loop does)
  const bool multi = ctx->comm != nullptr;
  if (pb->nranks > 1 && !ctx->comm)
    return tdw_fail(ctx, TDW_ERR_STATE, "sharded FMM problem without a communicator (tdw_comm_init)");
  FmmRun R;
  cudaEvent_t e0, e1;
  TDW_CUDA(ctx, cudaEventCreate(&e0));
  TDW_CUDA(ctx, cudaEventCreate(&e1));
  TDW_CUDA(ctx, cudaEventRecord(e0, st));
  int rc = fmm_begin(pb, R, threshold, want_rhs, st);
  for (int alpha = 1; rc == TDW_OK && alpha < pb->nt; ++alpha) {
    rc = fmm_step_rhs(pb, R, alpha, st);
    if (rc == TDW_OK && multi) {  // every rank's block of b, in place (NVLink)
      double* b = pb->d_b + (alpha & 1) * pb->bstride;
      ncclResult_t nr = ncclAllGather(b + pb->b_off, b, (size_t)pb->rows_per_rank, ncclDouble, ctx->comm, st);
      if (nr != ncclSuccess) rc = tdw_fail(ctx, TDW_ERR_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(nr));
    }
    if (rc == TDW_OK) rc = fmm_step_solve(pb, R, alpha, st);
  }
  TDW_CUDA(ctx, cudaEventRecord(e1, st));
  TDW_CUDA(ctx, cudaEventSynchronize(e1));
  if (timing && rc == TDW_OK) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    timing->total_ms += ms;
    timing->steps += pb->nt - 1;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (R.plan) free_plan_fmm(R.plan);
  if (rc) return rc;
  return fmm_check(pb);
}

// R shards of one FMM problem on ONE device, in lockstep: per step every shard
// forms its rows of b, the all-gather is replaced by device copies of the row
// blocks, every shard solves redundantly (the multi-GPU data flow, testable on
// one GPU).
int tdw_fmm_march_emulated(tdw_problem** pbs, int n, double threshold) {
  tdw_ctx* ctx = pbs[0]->ctx;
  cudaStream_t st = ctx->stream;
  std::vector<FmmRun> R(n);
  int rc = TDW_OK;
  for (int r = 0; r < n && rc == TDW_OK; ++r) {
    if (!pbs[r]->fmm || !pbs[r]->assembled || !pbs[r]->known_loaded)
      return tdw_fail(ctx, TDW_ERR_STATE, "emulated FMM march: shard not set up, assembled or without data");
    rc = fmm_begin(pbs[r], R[r], threshold, false, st);
  }
  const size_t rpr = (size_t)pbs[0]->rows_per_rank;
  for (int alpha = 1; rc == TDW_OK && alpha < pbs[0]->nt; ++alpha) {
    for (int r = 0; r < n && rc == TDW_OK; ++r) rc = fmm_step_rhs(pbs[r], R[r], alpha, st);
    const size_t slot = (size_t)(alpha & 1);
    for (int r = 0; r < n && rc == TDW_OK; ++r)
      for (int q = 0; q < n; ++q)
        if (q != r)
          TDW_CUDA(ctx, cudaMemcpyAsync(pbs[q]->d_b + slot * pbs[q]->bstride + pbs[r]->b_off,
                                        pbs[r]->d_b + slot * pbs[r]->bstride + pbs[r]->b_off,
                                        sizeof(double) * rpr, cudaMemcpyDeviceToDevice, st));
    for (int r = 0; r < n && rc == TDW_OK; ++r) rc = fmm_step_solve(pbs[r], R[r], alpha, st);
  }
  TDW_CUDA(ctx, cudaStreamSynchronize(st));
  for (int r = 0; r < n; ++r)
    if (R[r].plan) free_plan_fmm(R[r].plan);
  if (rc) return rc;
  for (int r = 0; r < n; ++r)
    if ((rc = fmm_check(pbs[r]))) return rc;
  return TDW_OK;
}

long long tdw_fmm_m2l_pairs(const tdw_problem* pb) { return pb->fmm ? pb->fmm->m2l_pairs : 0; }

// Average device time of the leaf level's M2L contraction (m2l_dmma_kernel, the
// FMM's dominant kernel) over n back-to-back launches on the current moments,
// and its FLOPs per launch (2 x 256 x 256 per pair and non-dark operator).
int tdw_fmm_time_m2l_impl(tdw_problem* pb, int n, double* flops, float* ms) {
  FmmState* F = pb->fmm;
  tdw_ctx* ctx = pb->ctx;
  if (!F) return tdw_fail(ctx, TDW_ERR_STATE, "tdw_fmm_time_m2l: not an FMM problem");
  FmmLevel& V = F->lev[F->leaf];
  if (flops) *flops = V.m2l_flops;
  if (ms) *ms = 0.0f;
  if (V.n_items == 0 || n < 1) return TDW_OK;
  const size_t smem = m2l_smem_bytes(pb->d, F->ntau0, F->ntaup);
  cudaStream_t st = ctx->stream;
  m2l_launch(pb->d, V, F, smem, st);  // warm-up
  cudaEvent_t e0, e1;
  TDW_CUDA(ctx, cudaEventCreate(&e0));
  TDW_CUDA(ctx, cudaEventCreate(&e1));
  TDW_CUDA(ctx, cudaEventRecord(e0, st));
  for (int k = 0; k < n; ++k) m2l_launch(pb->d, V, F, smem, st);
  TDW_CUDA(ctx, cudaEventRecord(e1, st));
  TDW_CUDA(ctx, cudaEventSynchronize(e1));
  float t = 0.0f;
  TDW_CUDA(ctx, cudaEventElapsedTime(&t, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (ms) *ms = t / n;
  return TDW_OK;
}

void tdw_fmm_free(FmmState* F) {
  if (!F) return;
  for (auto& V : F->lev) {
    void* p[] = {V.items, V.g_dark, V.parent, V.octant, V.child_ptr, V.child_idx, V.obs_ptr, V.il_src, V.il_off, V.dark,
                 V.K0, V.Kp, V.own, V.inherit, V.deriv, V.aux, V.acc, V.mom, V.g_obs, V.g_src,
                 V.Kop, V.X, V.tmp, V.t_ptr, V.t_pair, V.t_cells, (void*)V.gA, (void*)V.gB, (void*)V.gC};
    for (void* q : p)
      if (q) cudaFree(q);
  }
  for (auto& E : F->extra) {
    void* p[] = {E.row_ptr, E.col, E.row_of, E.U, E.W};
    for (void* q : p)
      if (q) cudaFree(q);
  }
  if (F->blas) cublasDestroy(F->blas);
  void* p[] = {F->elem_cell, F->cell_ptr, F->cell_elems, F->p2m_tau, F->p2m_sig, F->l2p_val, F->l2p_bm,
               F->Y};
  for (void* q : p)
    if (q) cudaFree(q);
  delete F;
}
