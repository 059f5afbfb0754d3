// tdw_impl.cuh -- internal state of libtdw (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <string>
#include <thread>
#include <vector>

#include "../../include/tdw.h"

// Tile geometry of the banded store.
#define TDW_TJ 32        // columns per J-tile == pairs per segment == one warp
#define TDW_TI 32        // rows per I-block (one conv CTA)
#define TDW_ELL_MAX 64   // max nnz per row of the lag-1 step matrix
#define TDW_KB_MAX 6     // time steps per convolution pass (temporal blocking)
#define TDW_NEAR_MAX 384 // max pairs per row in the near structure (bands reaching a split lag)
#define TDW_NSL_MAX (2 * TDW_KB_MAX - 1)  // max split lags
#define TDW_ELEM_STRIDE 16  // doubles per element record: v0 v1 v2 n c rad
// Unit layout (one (I-block, J-tile) unit = one contiguous byte range of the store):
//   [0, 128)        uint32 seg_rel[32]  entry offset of row r's segment in the unit
//   [128, 136)      int2 (gmin, gmax)   lag range of the unit (history slice)
//   [136, 140)      uint32              unit bytes
//   [140, 144)      uint32              coef offset: 2304 (16-bit headers) or 4352 (32-bit)
//   [256, coef)     hdr[32][32]         pair headers, lane = column: 32-bit ones row-major;
//                                       16-bit ones with the four rows of a consumer
//                                       warp side by side per lane (hdr16_index)
//   [coef, ...)     double2 coef[]      (V_U, V_W) entries, jagged k-major per segment:
//                                       the k-th entries of the lanes with band > k,
//                                       in lane order
// A unit whose bands are all <= 31 lags long and whose lag range spans <= 64
// lags (every unit of the benchmark configurations) carries 16-bit headers;
// any other unit falls back to 32-bit headers.
#define TDW_UNIT_LAG_OFF 128
#define TDW_UNIT_HDR_OFF 256
#define TDW_UNIT_COEF_OFF16 2304
#define TDW_UNIT_COEF_OFF 4352
#define TDW_EMPTY_UNIT 0xffffffffu
// assembly scratch: per segment, entry count | longest band << 48
#define TDW_SEG_LMAX_SHIFT 48
#define TDW_SEG_COUNT_MASK ((1ull << 48) - 1)

struct tdw_ctx {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
};

// header word of one (row, column) pair inside a segment:
//   bits 0..7 column within the J-tile, 8..15 band length, 16..31 first lag
__host__ __device__ inline uint32_t hdr_pack(int jl, int len, int glo) {
  return (uint32_t)jl | ((uint32_t)len << 8) | ((uint32_t)glo << 16);
}
__host__ __device__ inline int hdr_jl(uint32_t h) { return (int)(h & 0xffu); }
__host__ __device__ inline int hdr_len(uint32_t h) { return (int)((h >> 8) & 0xffu); }
__host__ __device__ inline int hdr_glo(uint32_t h) { return (int)(h >> 16); }
// 16-bit header: bits 0..4 column, 5..9 band length, 10..15 rel = unit gmax - first lag
__host__ __device__ inline uint16_t hdr16_pack(int jl, int len, int rel) {
  return (uint16_t)(jl | (len << 5) | (rel << 10));
}
// position of the 16-bit header of (row, lane): rows 4w..4w+3 of a lane are one 8-byte word
__host__ __device__ inline int hdr16_index(int row, int lane) { return (row >> 2) * 128 + lane * 4 + (row & 3); }
// (column, length, rel) of pair idx = row * 32 + lane of a unit, either header width
__device__ __forceinline__ void unit_hdr(const unsigned char* ub, unsigned coef_off, int gmax,
                                         int idx, int& jl, int& len, int& rel) {
  if (coef_off == TDW_UNIT_COEF_OFF16) {
    const unsigned h = ((const uint16_t*)(ub + TDW_UNIT_HDR_OFF))[hdr16_index(idx >> 5, idx & 31)];
    jl = (int)(h & 31u);
    len = (int)((h >> 5) & 31u);
    rel = (int)(h >> 10);
  } else {
    const uint32_t h = ((const uint32_t*)(ub + TDW_UNIT_HDR_OFF))[idx];
    jl = hdr_jl(h);
    len = hdr_len(h);
    rel = gmax - hdr_glo(h);
  }
}

struct tdw_problem {
  tdw_ctx* ctx = nullptr;
  // parameters
  int ns = 0, nv = 0, bie = 0, d = 1, nt = 2, window = 1;
  double c = 1.0, dt = 1.0, K = 0.0;
  int gstar = 0, n_lags = 0, cap = 0;
  int nranks = 1, rank = 0;
  // rows (internal order); rank r owns [row_lo, row_hi); rows_per_rank multiple of TDW_TI
  int rows_per_rank = 0, row_lo = 0, row_hi = 0, n_iblk = 0, ntiles = 0;
  int b_off = 0;                   // rank * rows_per_rank: this rank's block of the gathered b
  // ordering: internal index -> original element index
  std::vector<int> perm;
  int* d_perm = nullptr;
  double* d_elem = nullptr;  // ns * TDW_ELEM_STRIDE
  double* d_phi = nullptr;   // internal order
  // FMM near-field mode: pair filter (adjacent leaf cells), no lag-2 split
  int* d_leafc = nullptr;    // packed leaf-cell coords per element (internal order) or null
  int* d_pair_ptr = nullptr; // pairs= restriction (internal order): [ns+1] row pointers or null
  int* d_pair_col = nullptr; //   sorted columns of each row
  int gamma_max = 0;         // lags the store was asked to cover (0: all it needs)
  int mode = 0;              // TDW_MODE_* requested
  bool otf = false;          // coefficients recomputed by every pass (no banded store)
  int otf_tg = 8;            // J-tiles per on-the-fly partial
  unsigned long long* d_otf_evals = nullptr;  // closed-form evaluations of the on-the-fly passes
  int split_lag2 = 1;        // lags 2..nsl+1 of the store keep the known density only
  int kb = 1;                // time steps per convolution pass (1..TDW_KB_MAX)
  int conv_rpw = 2;          // rows per consumer warp of conv_kernel (2 or 4)
  int overlap = 1;           // solves a convolution pass overlaps (1..kb)
  int nsl = 1;               // split lags: kb + overlap - 1
  int bring = 2;             // b ring slots: kb + overlap
  bool skip_empty_units = false;
  struct FmmState* fmm = nullptr;
  // banded store
  bool assembled = false;
  unsigned char* d_units = nullptr;        // unit-major store (see unit layout above)
  unsigned long long* d_unit_off = nullptr; // [n_iblk * ntiles + 1] byte offsets
  int2* d_unit = nullptr;          // [n_iblk * ntiles] lag range (gmin, gmax)
  int wmax = 0;                    // max unit lag span
  int wbox = 0;                    // history box width (lags) of the widest TMA copy, >= wmax
  int hbox_n = 1, hbox_rows[4] = {1, 1, 1, 1};  // TMA box heights (rows = lag span + kb - 1), ascending
  size_t max_unit_bytes = 0;
  // conv schedule: persistent CTAs over items (I-block, tile split)
  int conv_grid = 0, conv_S = 1, conv_nstages = 2;
  bool conv_reserve = false;  // convolution CTAs leave the cluster solver's SMs free
  int conv_reserve_model = -1;  // the solver setup's step-time model decision (-1: none)
  size_t conv_stage_bytes = 0;
  unsigned* d_sched = nullptr;     // unit ids in CTA processing order (or TDW_EMPTY_UNIT)
  unsigned* d_sched_item = nullptr; // work item (I-block * S + split) of each entry
  unsigned* d_sched_off = nullptr; // [conv_grid + 1]
  int64_t n_band = 0, n_pairs = 0, n_evals = 0, store_bytes = 0;
  int64_t n_units = 0, units_hdr32 = 0;  // non-empty units; those with 32-bit headers
  // lag-1 step matrix, all rows, ELL
  int ell_w = 0, step_nnz = 0;
  int* d_acol = nullptr;
  double* d_aval = nullptr;
  double* d_adiag = nullptr;
  int jac_iters = 0;
  double cheb_rho = 0.0;           // Chebyshev bound of the halo solver's sweeps (0: Jacobi)
  bool solver_krylov = false;      // BiCGSTAB solve (Jacobi bound >= 0.9 or TDW_SOLVER=krylov)
  double* d_kw = nullptr;          // [9][ns] Krylov / standalone-solve workspace
  // near structure: pairs whose band reaches a split lag g in 2..nsl+1, all rows,
  // ELL columns [TDW_NEAR_MAX][ns], values [nsl][TDW_NEAR_MAX][ns] (lag g = 2 + index)
  int near_w = 0;
  int64_t n_near = 0, n_near_evals = 0;
  int* d_ncol = nullptr;
  double* d_nval = nullptr;
  int* d_ncol_packed = nullptr;    // ncol in the cluster solver's (owner << 24 | local) form
  int* d_ncnt = nullptr;           // near pairs per row
  // near_step_kernel's form: CSR of the nonzero near values per (split lag, row)
  int* d_n3_ptr = nullptr;         // [nsl][ns + 1]
  double2* d_n3_ent = nullptr;     // (value, column | sign bit where phi_j = 1)
  double* d_bnear = nullptr;       // [nsl][nsl+1][ns]: N_g x^(beta-1) after solve(beta), for step beta-1+g
  // pipelined loop: side stream for the far convolution, per-step events
  cudaStream_t side = nullptr;
  cudaStream_t side_near = nullptr;  // near terms of lags >= 3 (off the solve's critical path)
  bool near_split = false;
  bool known_preloaded_call = false;  // tdw_march_device_known in progress
  // lag-2 near terms inside the halo solve (its tail, x from DSMEM): CSR over the
  // rows, columns packed (owner CTA << 24) | owner-local row
  bool near_in_solve = false;
  int near_tail = 0;                 // split lags 2..near_tail+1 formed in the solve's tail
  int* d_n2_ptr = nullptr;
  int* d_n2_col = nullptr;
  double* d_n2_val = nullptr;
  std::vector<cudaEvent_t> ev_solve, ev_conv, ev_near;
  cudaEvent_t ev_fork = nullptr;
  cudaGraphExec_t graph_exec = nullptr;  // cached loop graph
  double graph_thr = 0.0;
  bool graph_rhs = false;
  double jac_bound = 0.0;
  // history and step buffers
  int pad = 0, hstride = 0;
  int hcols = 0;                   // history row length: ntiles * 32 elements (zero padded)
  double2* d_hist = nullptr;       // [hstride][hcols] (q, u) per step per element, time-major
  double* d_uk = nullptr;          // (nt-1, ns) original order
  double* d_qk = nullptr;
  bool known_loaded = false;
  int nsplit = 1;                  // == conv_S once assembled
  double* d_bpart = nullptr;       // [2][nsplit][rows_per_rank] (step parity)
  double* d_b = nullptr;           // [2][bstride] (step parity), bstride = nranks * rows_per_rank
  size_t bstride = 0;
  double* d_x = nullptr;           // [2][ns]
  double* d_red = nullptr;         // reduction scratch [3][grid]
  unsigned* d_bar = nullptr;       // grid barrier {count, generation}
  int* d_flags = nullptr;          // {status, n_steps, err_step, ell_overflow}
  double* d_rhs = nullptr;         // (nt-1, ns) original order, optional
  double* d_out = nullptr;
  unsigned long long* d_trace = nullptr;  // [nt][16] solve phase timestamps (TDW_TRACE_SOLVE)         // [4][(nt-1) ns] u, q, tau, sigma staging for the download
  int solve_grid = 0;
  // cluster solver (csrc/march.cu solve_cluster_kernel); sp_cl == 0 -> grid-barrier fallback
  int sp_cl = 0, sp_R = 0;
  int sp_reg = 0;                  // >0: register-resident solver with that many off-diagonal slots
  size_t sp_smem = 0;
  int* d_sp_rowptr = nullptr;
  long long* d_sp_nnzoff = nullptr;
  int* d_sp_col = nullptr;
  double* d_sp_val = nullptr;
  // halo (communication-avoiding) variant of the register solver
  int sp_halo = 0, sp_hT = 0, sp_hE = 0, sp_hG = 0;
  size_t sp_hsmem = 0;
  int *d_h_ncomp = nullptr, *d_h_gi = nullptr, *d_h_layer = nullptr, *d_h_nz = nullptr;
  int *d_h_col = nullptr, *d_h_ngat = nullptr, *d_h_gdst = nullptr, *d_h_gsrc = nullptr;
  double* d_h_val = nullptr;
  bool use_graph = true;
  // streamed march (tdw_march_stream_begin/finish): the host samples the known
  // data chunk by chunk into page-locked buffers while the loop runs.  A host
  // thread (the chunk server) watches the caller's chunk counter, copies every
  // published chunk to the device on the data stream and raises *d_ready; a
  // convolution pass waits (at kernel entry, on its own SMs) until the chunk of
  // the last step it reads has arrived.  No kernel of the loop itself waits on the
  // host, and no waiting kernel sits on an SM the solve cluster needs.
  bool streaming = false;
  bool stream_direct = false;       // this streamed march is launched kernel by kernel (no graph)
  const double* h_uk_host = nullptr;  // the caller's page-locked u samples (or null: zeros)
  const double* h_qk_host = nullptr;
  const volatile int* h_flag_host = nullptr;  // the caller's "chunks complete" counter (-1: abort)
  int stream_chunk = 16;            // steps per chunk
  int* d_ready = nullptr;           // chunks of known data on the device (this march)
  int need_ready = 0;               // chunks the pass being launched needs (0: not streamed)
  cudaStream_t side_data = nullptr;
  cudaEvent_t ev_begin = nullptr;   // history initialised: the chunk copies may start
  cudaGraphExec_t graph_exec_s = nullptr;  // cached streamed-loop graph
  double graph_thr_s = 0.0;
  bool graph_rhs_s = false;
  int loop_calls_s = 0;
  int stream_key_c = 0;             // what the cached streamed graph baked in: the chunk size
  bool stream_in_flight = false;
  std::thread stream_thread;        // enqueues the streamed loop while the caller samples
  std::thread chunk_thread;         // the chunk server
  int stream_rc = 0;                // their results
  int chunk_rc = 0;
  volatile bool stream_cancel = false;  // tdw_problem_destroy with a streamed march still waiting for its data
  cudaEvent_t ev_stream_end = nullptr;
  // streamed outputs (tdw_march_stream_outputs): after the last solve of each chunk
  // a side stream writes the chunk's rows of u, q, tau, sigma straight into the
  // caller's page-locked arrays (mapped), so the device-to-host traffic overlaps
  // the loop.  The destinations reach the kernels through d_outdesc (rewritten
  // before every launch), so the cached graph does not depend on them.
  double* out_host[4] = {nullptr, nullptr, nullptr, nullptr};  // registered for the next streamed march
  bool out_registered = false;
  bool out_streamed = false;       // the march in flight (or just finished) wrote them
  bool stream_key_out = false;     // the cached streamed graph contains the output kernels
  double** d_outdesc = nullptr;    // device: the four mapped destinations
  int* d_iperm = nullptr;          // original element index -> internal index
  cudaStream_t side_out = nullptr;
  cudaEvent_t ev_out = nullptr;
  int loop_calls = 0;               // time loops run on this problem (the first one is not captured)
  double t_assemble_ms = 0.0, t_fill_ms = 0.0;
};

// error helpers -----------------------------------------------------------
int tdw_fail(tdw_ctx* ctx, int code, const std::string& msg);
#define TDW_CUDA(ctx, call)                                                        \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess)                                                         \
      return tdw_fail((ctx), TDW_ERR_CUDA,                                         \
                      std::string(#call) + ": " + cudaGetErrorString(_e));         \
  } while (0)

// entry points implemented in the .cu files
int tdw_assemble_impl(tdw_problem* pb);
int tdw_march_loop(tdw_problem* pb, double threshold, bool want_rhs, bool time_kernels,
                   tdw_timing* timing);
int tdw_march_stream_launch(tdw_problem* pb, double threshold, bool want_rhs);
int tdw_march_stream_wait(tdw_problem* pb);
int tdw_outputs(tdw_problem* pb, double* u, double* q, double* tau, double* sigma);
int tdw_time_conv_impl(tdw_problem* pb, int n, float* ms_out);
int tdw_setup_cluster_solver(tdw_problem* pb);
int tdw_fmm_loop(tdw_problem* pb, double threshold, bool want_rhs, tdw_timing* timing);
int tdw_fmm_march_emulated(tdw_problem** pbs, int n, double threshold);
long long tdw_fmm_m2l_pairs(const tdw_problem* pb);
int tdw_fmm_time_m2l_impl(tdw_problem* pb, int n, double* flops, float* ms);
int tdw_step_solve_impl(tdw_problem* pb, const double* b, double* x, double* stats);
int launch_otf_conv(tdw_problem* pb, int alpha, int nb, cudaStream_t st);
int tdw_step_matrix_impl(tdw_problem* pb, int64_t* nnz, int64_t* rows, int64_t* cols, double* vals);
void tdw_fmm_free(struct FmmState* F);
int tdw_march_emulated_impl(tdw_problem** pbs, int n, double threshold);
int tdw_problem_create_impl(tdw_ctx* ctx, const tdw_problem_desc* dsc, tdw_problem** out, bool shard_only);
