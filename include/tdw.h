/*
 * tdw.h -- C ABI of libtdw (B200-native MOT hot path of the time-domain BEM,
 * arXiv 2111.05205).  Plain C: pointers, sizes and POD structs only.
 *
 * Every entry point replaces one reference interface (paths relative to
 * /root/reference/pkg/src/tdwavebem/):
 *
 *   tdw_coeff_table     <- elemint.retarded_coeff_table          elemint.py:89-186
 *   tdw_problem_create  <- marching.ProblemSpec (+mesh_stats,     marching.py:33-69,
 *                          compute_gamma_star)                    mesh.py:85-107
 *   tdw_assemble        <- marching.build_retarded_matrices       marching.py:132-181
 *   tdw_restrict_pairs  <- its pairs= argument (near-field subsets) marching.py:132-133, 149
 *   tdw_step_matrix, tdw_step_solve <- build_step_matrix (A, lu)    marching.py:279-289, 330
 *                          + build_step_matrix                    marching.py:279-289
 *   tdw_march           <- marching.march (+greville inputs,      marching.py:292-338
 *                          TimeHistory outputs)                   marching.py:184-276
 *   tdw_march_stream_begin / _finish (/ _outputs)
 *                       <- marching.march with the Greville sampling  marching.py:258-338
 *                          and the history copies overlapped with the loop (chunks)
 *   tdw_upload_known_rows + tdw_march_device_known
 *                       <- marching.march, pipelined form           marching.py:292-338
 *                          (known rows copied as they are sampled)
 *   tdw_tree_build (+ _info/_level/_near/_extra/_destroy)
 *                       <- fmm_tree.build_tree (device-side tree)  fmm_tree.py:73-231
 *   tdw_fmm_setup       <- fmm.fast_march's operator setup          fmm.py:165-531 (corrected,
 *                          (then tdw_assemble / tdw_march)          SURVEY 8(c)), fmm.py:534-544
 *   tdw_march_resident  <- same time loop, inputs/outputs resident on the device (benchmark form)
 *   tdw_nccl_unique_id / tdw_comm_init  <- (none in the reference; row-sharded multi-GPU)
 *   tdw_known_plane_pulse <- (none: device-side boundary data)
 *   tdw_fp64_peak, tdw_host_alloc / tdw_host_free, tdw_time_conv, tdw_fmm_time_m2l, tdw_set_graph,
 *   tdw_problem_create_shard / tdw_march_emulated  <- (none: diagnostics, pinned
 *                          memory, one-GPU emulation of the sharded paths)
 *
 * Host buffers are C-contiguous float64 / int64; the library copies in and out
 * and owns all device memory behind the opaque handles.  A ctx is bound to one
 * CUDA device and is not re-entrant.
 */
#ifndef TDW_H
#define TDW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes (mapped to the reference's exceptions by the Python shim) */
#define TDW_OK 0
#define TDW_ERR_INVALID_ARG 1       /* ValueError   (elemint.py:109-113, 154-155) */
#define TDW_ERR_UNSUPPORTED_ORDER 2 /* ValueError   (elemint.py:109-110) */
#define TDW_ERR_SINGULAR 3          /* RuntimeError (marching.py:284-288) */
#define TDW_ERR_RESIDUAL 4          /* RuntimeError (marching.py:331-333) */
#define TDW_ERR_CUDA 5
#define TDW_ERR_NCCL 6
#define TDW_ERR_STATE 7             /* call order (e.g. march before assemble) */
#define TDW_ERR_LIMIT 8             /* a structural limit of the banded store was exceeded */

typedef struct tdw_ctx tdw_ctx;
typedef struct tdw_problem tdw_problem;

/* kind: 0 = "uw" (U, W), 1 = "bm" (Burton-Miller Ubar, Wbar) */
#define TDW_KIND_UW 0
#define TDW_KIND_BM 1
/* coefficient mode: AUTO = the banded store when it fits in device
 * memory, else on the fly; STORED_BAND = always the store (HBM-bound pass);
 * ON_THE_FLY = every convolution pass re-evaluates the closed forms (FP64-bound) */
#define TDW_MODE_AUTO 0
#define TDW_MODE_STORED_BAND 1
#define TDW_MODE_ON_THE_FLY 2
/* bie: 0 = "obie", 1 = "bmbie" */
#define TDW_BIE_OBIE 0
#define TDW_BIE_BMBIE 1

typedef struct {
  int32_t ns;                /* elements (= collocation points)                 */
  int32_t nv;                /* vertices                                         */
  const double* vertices;    /* (nv, 3)                                          */
  const int64_t* triangles;  /* (ns, 3)                                          */
  const double* phi;         /* (ns,) 1 = u unknown (q given), 0 = q unknown     */
  int32_t bie;               /* TDW_BIE_*                                        */
  int32_t d;                 /* B-spline order, 1..3                             */
  double c, dt;
  int32_t nt;                /* time steps; the loop solves nt-1 of them         */
  int32_t window;            /* 1 = sliding window at gamma* (reference default) */
  int32_t nranks, rank;      /* row sharding; 1, 0 for a single GPU              */
  int32_t mode;              /* TDW_MODE_*: coefficients stored or recomputed     */
} tdw_problem_desc;

typedef struct {
  int32_t gamma_star;        /* compute_gamma_star (marching.py:67-69)           */
  int32_t n_lags;            /* min(gamma*, nt-1) (window) or nt-1               */
  int32_t row_lo, row_hi;    /* rows owned by this rank (internal order)         */
  int64_t n_band;            /* stored (i,j,gamma) entries of the banded store   */
  int64_t n_pairs;           /* (i,j) pairs with a non-empty band                */
  int64_t n_evals;           /* closed-form (i,j,gamma) evaluations in assembly  */
  int64_t store_bytes;       /* device bytes of the banded store (coef+headers)  */
  int32_t step_nnz;          /* nnz of the lag-1 step matrix                     */
  int32_t jacobi_iters;      /* fixed Jacobi sweeps per step                     */
  double jacobi_bound;       /* max_i sum_{j!=i} |A_ij| / |A_ii|                 */
  double t_assemble_ms;      /* device time of tdw_assemble                      */
  double t_fill_ms;          /* device time of the coefficient fill kernel       */
  int64_t max_unit_bytes;    /* largest (row block, column tile) unit of the store */
  int32_t max_lag_span;      /* largest history slice (lags) of a unit           */
  int32_t conv_grid;         /* persistent CTAs of the convolution kernel        */
  int32_t conv_splits;       /* column-tile splits per row block                 */
  int32_t solve_cluster;     /* CTAs of the cluster solver (0 = grid fallback)   */
  int64_t n_units;           /* (row block, column tile) units with band entries */
  int64_t units_hdr32;       /* of those, units stored with 32-bit pair headers  */
  int32_t steps_per_pass;    /* time steps computed per convolution pass (kb)    */
  int32_t near_width;        /* widest row of the near structure                 */
  int32_t pass_overlap;      /* solves a convolution pass runs beside            */
  int32_t solve_halo;        /* halo depth of the communication-avoiding solver (0: none) */
  int64_t fmm_m2l_pairs;     /* FMM: M2L interaction pairs this rank evaluates (0: direct) */
  int32_t conv_rpw;          /* rows per consumer warp of the convolution CTA (2 or 4) */
  int32_t coeff_mode;        /* TDW_MODE_* the problem runs in                    */
} tdw_info;

typedef struct {
  double total_ms;           /* device time of the whole timed loop              */
  double conv_ms;            /* summed device time of the history-convolution kernel */
  double solve_ms;           /* 1 if the loop ran as a CUDA graph, else 0         */
  double comm_ms;            /* summed device time of the NCCL all-gather        */
  int32_t conv_launches;
  int32_t steps;
} tdw_timing;

int tdw_init(int device, tdw_ctx** out);
int tdw_finalize(tdw_ctx* ctx);
const char* tdw_last_error(const tdw_ctx* ctx);
int tdw_device_count(void);

/* elemint.retarded_coeff_table: n triples, host arrays. nx may be NULL for kind 0. */
int tdw_coeff_table(tdw_ctx* ctx, int64_t n, const double* P, const double* A, const double* B,
                    const double* C, const double* ez, const double* s, int d, double c, double dt,
                    int kind, const double* nx, double* out0, double* out1);

/* Same, DEVICE pointers, on the ctx stream; *ms = kernel time (may be NULL). */
int tdw_coeff_table_device(tdw_ctx* ctx, int64_t n, const double* P, const double* A,
                           const double* B, const double* C, const double* ez, const double* s,
                           int d, double c, double dt, int kind, const double* nx, double* out0,
                           double* out1, float* ms);

int tdw_problem_create(tdw_ctx* ctx, const tdw_problem_desc* desc, tdw_problem** out);
int tdw_assemble(tdw_problem* pb);

/* build_retarded_matrices(spec, gamma_max, pairs=(ii, jj)) (marching.py:132-181):
 * restrict the store (and the lag-1 step matrix built from it) to the listed
 * (row, column) element pairs, caller's element order.  Call between
 * tdw_problem_create and tdw_assemble; repeated pairs count once. */
int tdw_restrict_pairs(tdw_problem* pb, int64_t n, const int64_t* ii, const int64_t* jj);

/* build_step_matrix(spec, mats) (marching.py:279-289): the assembled lag-1 step
 * matrix A = w0 (W1 phi - U1 (1 - phi)) as COO in the caller's element order
 * (rows == NULL: only *nnz), and its solve lu.solve(b) (marching.py:330) on the
 * device (BiCGSTAB with a diagonal preconditioner); stats (nullable) =
 * (||A x - b||, ||b||, iterations). */
int tdw_step_matrix(tdw_problem* pb, int64_t* nnz, int64_t* rows, int64_t* cols, double* vals);
int tdw_step_solve(tdw_problem* pb, const double* b, double* x, double* stats);
int tdw_problem_info(const tdw_problem* pb, tdw_info* out);

/* FP64 FMA throughput of the ctx's GPU (TFLOP/s, FMA = 2 FLOP): the denominator
 * of the coefficient kernel's roofline.  Diagnostics; no reference counterpart. */
int tdw_fp64_peak(tdw_ctx* ctx, double* tflops);

/* Pinned (page-locked) host memory for the march's host buffers: copies from and
 * to it run at full PCIe/C2C rate.  No reference counterpart (numpy arrays). */
int tdw_host_alloc(int64_t bytes, void** out);
int tdw_host_free(void* p);

/* Full march with host buffers.  u_known/q_known: (nt-1, ns) Greville samples
 * (marching.py:258-276); NULL = that data callable is None (zero samples).  Outputs (nt-1, ns): u, q, tau, sigma; rhs_trace may be NULL.
 * status: 0 stable, 1 unstable (blow-up detector, marching.py:336-338). */
int tdw_march(tdw_problem* pb, const double* u_known, const double* q_known, double threshold,
              double* u, double* q, double* tau, double* sigma, double* rhs_trace,
              int32_t* n_steps, int32_t* status);

/* Pipelined form of tdw_march: the caller uploads the known rows [beta0, beta0 +
 * nbeta) of u (which = 0) or q (1) as it produces them (src NULL = zeros), on the
 * library stream, then runs the march on them.  Same outputs and errors as
 * tdw_march; lets the host's Greville sampling overlap the copies. */
int tdw_upload_known_rows(tdw_problem* pb, int which, int beta0, int nbeta, const double* src);
int tdw_march_device_known(tdw_problem* pb, double threshold, double* u, double* q, double* tau,
                           double* sigma, double* rhs_trace, int32_t* n_steps, int32_t* status);

/* Streamed form of tdw_march (marching.py:292-338 with the Greville sampling of
 * :258-276 overlapped): the loop is launched at once; the caller samples the known
 * data into page-locked buffers from tdw_host_alloc (u_host / q_host; NULL = that
 * callable is None, zeros), step by step, and after every `chunk` steps stores the
 * number of complete chunks in *flag (a page-locked int32; -1 aborts the loop, e.g.
 * when a data callable raised).  A host thread of the library copies each chunk
 * to the device as soon as it is published (the pass that needs it waits for it on
 * the device); tdw_march_stream_finish waits and returns the outputs and errors of
 * tdw_march.  Direct path only (not FMM problems). */
int tdw_march_stream_begin(tdw_problem* pb, double threshold, int want_rhs, const double* u_host,
                           const double* q_host, int chunk, int32_t* flag);
int tdw_march_stream_finish(tdw_problem* pb, double* u, double* q, double* tau, double* sigma,
                            double* rhs_trace, int32_t* n_steps, int32_t* status);
/* Optional, before tdw_march_stream_begin: the (nt-1, ns) TimeHistory arrays
 * (marching.py:184-203) the NEXT streamed march will return, in page-locked memory
 * from tdw_host_alloc (NULL = not wanted).  The loop then writes each chunk's rows
 * of u, q, tau, sigma into them as soon as the chunk's last step is solved, so the
 * device-to-host traffic overlaps the loop; tdw_march_stream_finish, given the same
 * pointers, copies nothing.  Arrays that are not page-locked: TDW_ERR_INVALID_ARG. */
int tdw_march_stream_outputs(tdw_problem* pb, double* u, double* q, double* tau, double* sigma);

/* Device-side boundary data (no reference counterpart): the
 * Greville samples of the incident Gaussian plane pulse exp(-((t - z - t0)/sig)^2)
 * at the centroids (zc, nz: (ns,) centroid z and normal z, caller's element
 * order) computed on the device into the u (which = 0, -u_in) or q (1,
 * -du_in/dn) known data.  Follow with tdw_upload_known_rows(.., NULL) for a
 * None callable and tdw_march_device_known. */
int tdw_known_plane_pulse(tdw_problem* pb, int which, const double* zc, const double* nz, double t0,
                          double sig);

/* Benchmark form: known data already uploaded (tdw_upload_known), the time loop
 * runs n_repeat times on device-resident data; timings from CUDA events. */
int tdw_upload_known(tdw_problem* pb, const double* u_known, const double* q_known);
int tdw_march_resident(tdw_problem* pb, double threshold, int n_repeat, int time_kernels,
                       tdw_timing* timing);
int tdw_download(tdw_problem* pb, double* u, double* q, double* tau, double* sigma,
                 int32_t* n_steps, int32_t* status);

/* Average device time of one history-convolution launch (kernel K2) over n
 * back-to-back launches at a fixed step; inputs resident.  For the roofline. */
int tdw_time_conv(tdw_problem* pb, int n, float* ms);

/* FMM: average device time of the leaf level's M2L contraction (the fast
 * solver's dominant kernel) over n launches, and its FLOPs per launch (2 x 256 x
 * 256 per interaction pair and non-dark operator).  For the roofline. */
int tdw_fmm_time_m2l(tdw_problem* pb, int n, double* flops, float* ms);

/* 0 = launch the time loop kernel by kernel, 1 = capture it in a CUDA graph (default). */
int tdw_set_graph(tdw_problem* pb, int enable);

int tdw_problem_destroy(tdw_problem* pb);

/* Interpolation space-time FMM (configs 3-4; reference fmm.py fast_march, corrected).
 * Operator data from the host planner (paper_2111_05205_b200/fmm_plan.py); per-
 * element arrays in the caller's element order, per-level arrays concatenated
 * over levels 2..leaf.  Call after tdw_problem_create and before tdw_assemble;
 * tdw_march then runs the fast solver (near field = banded store of adjacent
 * leaf cells with window gamma_near). */
typedef struct {
  int32_t ps, pt, mu, leaf;          /* ps = pt = 4, mu <= 8 supported                  */
  int32_t gamma_near;
  int32_t n_leaf_cells;
  const int64_t* leaf_coords;        /* (ns, 3) leaf-cell coordinates of each element   */
  const int64_t* elem_cell;          /* (ns,) leaf cell index                           */
  const double* p2m_tau;             /* (ns, ps^3) P2M rows (value)                     */
  const double* p2m_sig;             /* (ns, ps^3) P2M rows (normal derivative)         */
  const double* l2p_val;             /* (ns, ps^3) L2P rows                             */
  const double* l2p_bm;              /* (ns, ps^3) Burton-Miller L2P rows or NULL       */
  const double* t_space;             /* (2, ps, ps) child->parent re-anchoring          */
  const double* t_time;              /* (2, pt, pt)                                     */
  int32_t n_levels;                  /* leaf - 1                                        */
  const int32_t* lev_ncell;
  const double* lev_interval;
  const int64_t* lev_parent;         /* concat(ncell): parent in level L-1 (-1 at L=2)  */
  const int64_t* lev_octant;         /* concat(ncell, 3)                                */
  const int32_t* lev_noff;
  const uint8_t* lev_dark;           /* concat(noff, mu+1)                              */
  const double* lev_K0;              /* concat(noff, (2ps-1)^3, (mu+2)(pt-1)+1)         */
  const double* lev_Kp;              /* concat over levels of (d, noff, (2ps-1)^3, 2pt-1) */
  const int64_t* lev_nil;
  const int64_t* lev_obs_ptr;        /* concat(ncell+1): interaction pairs by observer  */
  const int64_t* lev_il_src;
  const int64_t* lev_il_off;         /* offset index within the level                   */
  int32_t n_extra;
  const int32_t* extra_lags;
  const int64_t* extra_npair;
  const int64_t* extra_i;            /* concat(npair), caller's element order           */
  const int64_t* extra_j;
  const int64_t* ticks_before;       /* (nt,) last leaf tick to run before step alpha   */
  const int64_t* k_obs;              /* (nt,) observation interval of step alpha        */
  const double* wt;                  /* (nt, pt) L2P time weights                       */
  const double* dwt;                 /* (nt, pt) their time derivative / c              */
  const double* wts;                 /* (nt, pt) P2M time weights of step alpha's source */
  const int64_t* extra_gmax;         /* (n_extra, nt) same-interval lag limit           */
} tdw_fmm_desc;

int tdw_fmm_setup(tdw_problem* pb, const tdw_fmm_desc* desc);

/* fmm_tree.build_tree (fmm_tree.py:73-231) on the device, bit-exact: octree over
 * the centroids (ns, 3) with leaf capacity Z, interaction lists, near pairs of
 * adjacent leaf cells, the mu-interval causality check (TDW_ERR_INVALID_ARG with
 * the reference's message) and the marginal element pairs (corrected = 1: SURVEY
 * 8(c) correction 7).  rho = max element radius.  Results are read back with
 * tdw_tree_info / _level / _near / _extra (int64, caller's element order). */
typedef struct tdw_tree tdw_tree;
int tdw_tree_build(tdw_ctx* ctx, int ns, const double* centroids, double rho, double c, double dt,
                   int leaf_capacity, int mu, int max_depth, int corrected, tdw_tree** out);
int tdw_tree_info(const tdw_tree* t, int* leaf, double* centre3, double* root_half, int64_t* cells,
                  int64_t* nil, int64_t* n_near, int* n_extra);
int tdw_tree_level(const tdw_tree* t, int level, int64_t* coords, int64_t* parent, int64_t* elem_cell,
                   int64_t* il_obs, int64_t* il_src, int64_t* il_off);
int tdw_tree_near(const tdw_tree* t, int64_t* ii, int64_t* jj);
int tdw_tree_extra(const tdw_tree* t, int k, int* level, int64_t* n, int64_t* ii, int64_t* jj);
int tdw_tree_destroy(tdw_tree* t);

/* Test harness of the row-sharded path on ONE device: create the shard of rank
 * desc->rank of desc->nranks without a communicator, then run all shards in one
 * process with the per-step all-gather emulated by device copies.  Every shard
 * must be assembled and have its known data uploaded; outputs via tdw_download.
 * FMM shards (tdw_fmm_setup on a shard) own the target leaf cells of their rows
 * and evaluate M2L only into those cells and their ancestors. */
int tdw_problem_create_shard(tdw_ctx* ctx, const tdw_problem_desc* desc, tdw_problem** out);
int tdw_march_emulated(tdw_problem** shards, int n, double threshold);

/* Multi-GPU (one process per GPU): rank 0 makes the id, the host broadcasts it
 * (torch.distributed), every rank calls tdw_comm_init before tdw_problem_create.
 * nranks == 1 also creates a one-rank communicator, so the exchange path
 * (all-gather inside the captured loop) can be exercised on a single GPU. */
int tdw_nccl_unique_id(char out[128]);
int tdw_comm_init(tdw_ctx* ctx, const char id[128], int nranks, int rank);

#ifdef __cplusplus
}
#endif
#endif /* TDW_H */
