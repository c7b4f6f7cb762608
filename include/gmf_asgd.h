/*
 * gmf_asgd.h -- C ABI of the B200-native aSGD hot path for penalized
 * generalized matrix factorization (arXiv 2412.20509).
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/gmfkit):
 *
 *   Level 1 (backend seam, gmfkit/kernels):
 *     gmf_mean_of_eta      <- kernels/_ref.py:21-32  mean_of_eta(lcode, eta)
 *                             kernels/__init__.py:57-60 block_mean
 *     gmf_derivs_from_mu   <- kernels/_core.pyx:58-111 derivs_from_mu(fcode, lcode,
 *                             y, mu, w, phi, alpha) -> (dotd, ddotd)
 *                             kernels/_ref.py:65-88 (same contract)
 *     gmf_deviance_from_mu <- kernels/_ref.py:91-108 deviance_from_mu(fcode, y, mu,
 *                             w, alpha) -> float; kernels/__init__.py:80-90
 *     gmf_score_pairs      <- metrics.py:35-55 rel_log_rmse / rel_deviance sums
 *
 *   Level 2 (fit engine behind optim.fit_asgd, optim.py:383-489):
 *     gmf_create/gmf_destroy  own the device workspace of one fit (optim.py:409-414)
 *     gmf_reset               t = 0, EMA zero, initial trace entry (optim.py:404-417)
 *     gmf_minibatch_grad      gradients.py:116-132 minibatch_gradients -> GradientPair
 *     gmf_step_local          one aSGD step, rank-local half: tracked objective
 *                             (optim.py:283-290) + fused block gradient
 *                             (optim.py:427-448, gradients.py:102-113)
 *     gmf_step_apply          tracker (optim.py:301-338), EMA + adaptive update
 *                             (optim.py:450-462), NB shape update (optim.py:469-473)
 *     gmf_run                 n x (local + apply), captured in a CUDA graph
 *     gmf_status/gmf_read_*   FitReport fields (optim.py:109-127)
 *     gmf_objective_full      model.py:268-276 penalized_objective (deviance part)
 *     gmf_loglik_full         select.py:81-96 information_criteria: deviance and the
 *                             NB dispersion constant (select.py:57-78) in one pass
 *     gmf_entries_eval        select.py:141-145 _mu_at at held-out entries, fused
 *                             with metrics.py:35-55 (cv_rank_select scoring,
 *                             select.py:201-213)
 *   Initialization (initialization.py:143-169 init_ols_svd, 62-82 randomized_svd):
 *     gmf_csr_spmm            S P for the log-transformed counts' sparse part
 *                             (S' Q through the CSC); the residual's low-rank
 *                             part is applied by the host (no n x m residual)
 *     gmf_init_moments        _nb_shape_moment sums (initialization.py:93-100)
 *   File formats (io.py:104-109 read_matrix_market, densifying):
 *     gmf_mm_header/gmf_mm_read_csr  coordinate MatrixMarket -> CSR counts (host)
 *   Level 3 (identify.project_constraints (A)+(B1), identify.py:59-110):
 *     gmf_cross_rows          Z = A' B over rows (Gram / cross products), fp64
 *     gmf_rows_affine         Y <- beta Y + A M, row-local apply of a small matrix
 *
 * Conventions: plain pointers and sizes; device pointers unless stated; a
 * `stream` argument is a cudaStream_t passed as void* (NULL = legacy default
 * stream); every entry point returns GMF_OK (0) or a negative code, never
 * throws; gmf_last_error() describes the last failure on the calling thread.
 * A handle is single-writer; distinct handles are independent (re-entrant).
 */
#ifndef GMF_ASGD_H
#define GMF_ASGD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GMF_OK 0
#define GMF_ERR_CONFIG (-1)      /* gmfkit ConfigError  (exceptions.py:12)  */
#define GMF_ERR_DOMAIN (-2)      /* gmfkit DomainError  (exceptions.py:8)   */
#define GMF_ERR_CUDA (-3)        /* CUDA runtime failure                    */
#define GMF_ERR_UNSUPPORTED (-4) /* valid for gmfkit, not built here        */
#define GMF_ERR_STATE (-5)       /* call order / handle misuse              */

enum gmf_dtype { GMF_F32 = 0, GMF_F64 = 1 };

/* codes match gmfkit/kernels/_ref.py:15-16 */
enum gmf_family {
  GMF_GAUSSIAN = 0, GMF_GAMMA = 1, GMF_INV_GAUSSIAN = 2,
  GMF_POISSON = 3, GMF_BERNOULLI = 4, GMF_NEG_BINOMIAL = 5
};
enum gmf_link {
  GMF_IDENTITY = 0, GMF_LOG = 1, GMF_LOGIT = 2, GMF_INVERSE = 3, GMF_INVERSE_SQUARED = 4
};

/* Y formats: dense int32 n x m; CSR with int32 columns and counts; packed CSR
 * with one uint32 per nonzero, (count << 16) | column, for m <= 65536 and
 * counts <= 65535 (half the bytes of CSR_I32; csr_val unused) */
enum gmf_yfmt { GMF_Y_DENSE_I32 = 0, GMF_Y_CSR_I32 = 1, GMF_Y_CSR_PACK32 = 2 };
/* K1 (fused minibatch gradient) implementation: AUTO = tensor cores
 * (tcgen05, bf16-split operands) when eligible -- fp32, no prior weights,
 * q+d <= 16, p+d <= 16 -- else CUDA cores; TENSOR fails if ineligible. */
enum gmf_k1_impl { GMF_K1_AUTO = 0, GMF_K1_CUDA_CORES = 1, GMF_K1_TENSOR = 2 };

/* ---------------------------------------------------------------- level 1 */

/* mu = g^{-1}(eta), n entries of `dtype`. */
int gmf_mean_of_eta(int lcode, int dtype, const void* eta, void* mu, int64_t n,
                    void* stream);

/* dotd = -w (y - mu) / (phi nu g'), ddotd = w / (phi nu g'^2) (Fisher form).
 * w may be NULL (all ones).  Never raises on non-finite values. */
int gmf_derivs_from_mu(int fcode, int lcode, int dtype, const void* y, const void* mu,
                       const void* w, int64_t n, double phi, double alpha,
                       void* dotd, void* ddotd, void* stream);

/* *dev_sum (device double) = sum_k w_k D(y_k, mu_k), fixed-order reduction.
 * `work` is device scratch of gmf_reduce_work_bytes(n) bytes. */
int64_t gmf_reduce_work_bytes(int64_t n);
int gmf_deviance_from_mu(int fcode, int dtype, const void* y, const void* mu,
                         const void* w, int64_t n, double alpha, double* dev_sum,
                         void* work, void* stream);

/* sums4 (device, 4 doubles) = [sum D(y, mu), sum D(y, ybar), sum log^2((1+y)/(1+mu)),
 * sum log^2((1+y)/(1+ybar))] over n pairs (unit weights), fixed-order reduction;
 * `work` is device scratch of gmf_score_work_bytes() bytes. */
int64_t gmf_score_work_bytes(void);
int gmf_score_pairs(int fcode, int dtype, const void* y, const void* mu, int64_t n, double ybar,
                    double alpha, double* sums4, void* work, void* stream);

/* ---------------------------------------------------------------- level 2 */

typedef struct gmf_handle gmf_handle;

typedef struct gmf_desc {
  int64_t n;            /* rows held by this rank (block-major order)          */
  int64_t m;            /* columns                                             */
  int32_t p, q, d;      /* row design X (n x p), column design Z (m x q), rank;
                           p+q+d <= 64 (fp64: <= 32)                           */
  int32_t dtype;        /* GMF_F32 | GMF_F64: parameters and block arithmetic  */
  int32_t family, link; /* fused count paths: (POISSON|NEG_BINOMIAL, LOG); any
                           other pair -- and any fit that estimates phi --
                           runs in general mode (GMF_DESC_REAL_RESPONSE)       */
  int32_t y_format;     /* gmf_yfmt                                            */
  int32_t has_offset;   /* per-row offset in eta (BASELINE extension)          */
  int32_t has_weights;  /* dense n x m prior weights (dense Y only)            */
  int32_t world_size;   /* ranks sharing every row block (1 = single GPU)      */
  int32_t rank;
  int32_t device;       /* CUDA device ordinal                                 */
  int32_t flags;        /* GMF_DESC_* bits                                     */
} gmf_desc;

/* gmf_desc.flags: theta_row, x, offset, csr_col and csr_val may be read up to
   16 bytes past their end (the warp-specialized tensor-core K1 stages row
   ranges with TMA bulk copies of their 16-byte aligned superset; without
   the flag the handle uses the older tensor-core K1) */
#define GMF_DESC_TAIL_PADDED 1
/* general mode (families.py:267-441 with any link of :98-210, and the Pearson
   dispersion of optim.py:175-202): the response is real-valued and lives in
   gmf_buffers.y_work (n x m, compute dtype, fully observed; y_dense unused);
   K1 runs on the CUDA cores with the family and link chosen at run time,
   p+q+d <= 32 */
#define GMF_DESC_REAL_RESPONSE 2
/* general mode with unobserved entries: y_work marks a hole by the least
   significant mantissa bit of its imputed mean (seeded with g^{-1}(eta0),
   refilled on the device every nafill_every steps; optim.py:368-374,
   430-436); the caller clears that bit in the observed values (<= 1 ulp) */
#define GMF_DESC_REAL_HOLES 8
/* evaluation-only handle: holds a state for gmf_entries_eval (mu at listed
   entries, held-out scores; select.py:141-145) under ANY family / link, with
   an empty response; the fit, gradient and deviance calls return GMF_ERR_STATE */
#define GMF_DESC_EVAL_ONLY 4

typedef struct gmf_config {   /* SgdConfig (optim.py:61-106) + penalty (model.py:193-226) */
  double rate_k0, rate_k1, rate_tau;
  double smooth_a1, smooth_a2;
  double damping, tol;
  double lam_b, lam_gamma, lam_u, lam_v;
  double nb_floor, nb_ceiling;   /* optim.py:57-58 */
  double phi;                    /* fixed dispersion (Poisson / NB under "auto") */
  double eval_scale;             /* total / cap of the tracked sample (optim.py:271) */
  int64_t max_epochs;
  int32_t est_alpha;             /* NB shape estimated (optim.py:156-168) */
  int32_t snapshot_stride;       /* 4 (optim.py:309) */
  int32_t k1_impl;               /* enum gmf_k1_impl (no reference counterpart) */
  int32_t nafill_every;          /* imputation period of unobserved entries (optim.py:432) */
  int32_t est_phi;               /* Pearson dispersion update each step (optim.py:465-468);
                                    general mode only                                      */
  int32_t reserved0;
  double inv_resid_dof;          /* 1 / (nm - pm - qn - d(n+m) - 1), global n (optim.py:171-172) */
} gmf_config;

typedef struct gmf_buffers {  /* caller-owned device memory; rows block-major */
  const int32_t* y_dense;     /* n x m                          (DENSE_I32) */
  const int64_t* csr_ptr;     /* n + 1                          (CSR_I32)   */
  const int32_t* csr_col;     /* nnz, sorted within a row (PACK32: packed)  */
  const int32_t* csr_val;     /* nnz                                        */
  const void* weights;        /* n x m or NULL                              */
  const void* x;              /* n x p                                      */
  const void* z;              /* m x q                                      */
  const void* offset;         /* n or NULL                                  */
  void* theta_row;            /* n x (q+d): [gamma | u]                     */
  void* theta_col;            /* m x (p+d): [b | v]                         */
  void* gbar_row;             /* n x (q+d)  EMA of gradients               */
  void* hbar_row;
  void* gbar_col;             /* m x (p+d)                                  */
  void* hbar_col;
  void* snap_row;             /* n x (q+d) divergence snapshot              */
  void* snap_col;             /* m x (p+d)                                  */
  const int64_t* row_block_ptr;   /* R + 1 offsets of the local row blocks  */
  const double* row_block_scale;  /* R: n_global / |I_r global| (s_col)     */
  int64_t n_row_blocks;           /* R                                      */
  const int32_t* col_idx;         /* m: column blocks concatenated          */
  const int64_t* col_block_ptr;   /* S + 1                                  */
  const int32_t* col_pos;         /* m: position of column j in its block   */
  const int32_t* col_block_of;    /* m: block of column j                   */
  int64_t n_col_blocks;           /* S                                      */
  const int32_t* block_seq;       /* max_steps row-block draws (host RNG)   */
  int64_t max_steps;              /* max_epochs * S                         */
  const int64_t* eval_row;        /* E local tracked-objective entries      */
  const int32_t* eval_col;
  int64_t n_eval;
  /* responses with unobserved entries (dense only; NULL when fully observed):
     n x m working response in the compute dtype -- observed counts as >= 0
     values, an unobserved entry as -(its current imputed mean), seeded by
     the caller with -g^{-1}(eta0) (optim.py:368-374) and refilled by the
     gradient kernel every nafill_every steps (optim.py:430-436); the
     tracked objective, the deviance and the information criteria skip it */
  void* y_work;
} gmf_buffers;

typedef struct gmf_status {
  int64_t t;              /* steps applied                                    */
  int64_t trace_len;      /* objective_trace entries (epochs_run + 1)         */
  int64_t snapshot_trace_len;
  double nb_shape;
  double phi;
  double last_objective;
  int32_t converged;
  int32_t diverged;       /* non-finite objective after an epoch              */
  int32_t diverged_init;  /* non-finite at the initial state                  */
  int32_t stopped;        /* converged | diverged | max_epochs reached        */
} gmf_status;

int gmf_create(const gmf_desc* desc, const gmf_config* cfg, const gmf_buffers* bufs,
               gmf_handle** out);
int gmf_destroy(gmf_handle* h);

/* Start a fit: t = 0, EMA zeroed, trace cleared, dirty marks reset,
 * per-block row-norm sums recomputed. */
int gmf_reset(gmf_handle* h, double nb_shape, void* stream);

/* Standalone fused block gradient (no state change).  Outputs in dtype:
 * g_row/h_row (|I_r| x (q+d)), g_col/h_col (|J_s| x (p+d)); nb_sums (device,
 * 2 doubles, may be NULL) = (sum w mu^2, sum w((y-mu)^2 - mu)).
 * nb_shape is the NB alpha used for the block (ignored for Poisson). */
int gmf_minibatch_grad(gmf_handle* h, int64_t row_block, int64_t col_block, double nb_shape,
                       void* g_row, void* h_row, void* g_col, void* h_col,
                       double* nb_sums, void* stream);

/* One aSGD step split at the cross-rank exchange.  After gmf_step_local the
 * rank record (gmf_record_ptr, gmf_record_bytes) holds this rank's column-side
 * partials, NB sums and objective partials.  gmf_step_apply takes the records
 * of all ranks concatenated in rank order (`gathered`; NULL when world_size
 * is 1).  Both are no-ops once the fit has stopped. */
int gmf_step_local(gmf_handle* h, void* stream);
int gmf_step_apply(gmf_handle* h, const void* gathered, void* stream);
void* gmf_record_ptr(gmf_handle* h);
int64_t gmf_record_bytes(gmf_handle* h);
/* device-to-device copy of this rank's record into `dst` (record_bytes) */
int gmf_record_copy(gmf_handle* h, void* dst, void* stream);

/* Single-rank convenience: n_steps x (local + apply), replayed from a CUDA
 * graph captured on first use (chunk of `graph_steps` steps). */
int gmf_run(gmf_handle* h, int64_t n_steps, void* stream);

int gmf_status_read(gmf_handle* h, gmf_status* out, void* stream);   /* syncs stream */
/* Divergence snapshot bookkeeping (copy-on-write): ver[r] (R entries, host)
 * and the current snapshot period; the snapshot's rows of block r are
 * snap_row if ver[r] == period, else the live theta_row. */
int gmf_snapshot_blocks(gmf_handle* h, int64_t* ver, int64_t* period, void* stream);
/* Asynchronous D2H of the raw status word (gmf_status_raw_bytes() bytes) into
 * host memory (pinned for true asynchrony); decode later on the host. */
int64_t gmf_status_raw_bytes(void);
int gmf_status_copy_async(gmf_handle* h, void* host_dst, void* stream);
int gmf_status_decode(const void* raw, gmf_status* out);
/* Profiling hook: average device time (CUDA events on `stream`) of `iters`
 * launches of the fused gradient kernel K1 alone on row block `row_block`,
 * column block 0, at the current state (no state change). */
int gmf_time_grad(gmf_handle* h, int64_t row_block, int32_t iters, double* avg_ms, void* stream);
/* Profiling hook: phase timers of the persistent kernel (globaltimer ns):
 * out[0..5] = CTA 0's {objective partials, K1 tiles, barrier 1, phase 2,
 * barrier 2, steps}, out[6..10] phase-2 sub-timers, out[16 + 16 c + i] the
 * last profiled step's stamps of CTA c (i: start, K1 start, K1 end, after
 * barrier 1, phase-2 end) and out[16 + 16 c + 8 + i], i < 8, CTA c's summed
 * SM clocks of the tensor-core K1 sub-phases.  `out` holds gmf_profile_len(h)
 * doubles; reads (if out) and resets the counters, then enables/disables. */
int64_t gmf_profile_len(gmf_handle* h);
/* launch geometry: {persistent CTAs, its row splits, column tiles, tile
 * width, per-step-kernel row splits, feature bucket, K1 smem bytes, max |I|} */
int gmf_geometry(gmf_handle* h, int64_t* out8);
/* Streaming run (single rank, persistent kernel): ONE launch of n_steps
 * steps in which step t (global index) waits, before its gradient, until the
 * device counter at gmf_stream_ready_ptr(h) reaches t + 1 -- the caller
 * uploads step t's row block (Y rows of the drawn block, in place) on another
 * stream and then copies the value t + 1 into the counter.  After every step
 * the status word (gmf_status_raw_bytes() bytes, decode with
 * gmf_status_decode) is written to host_status[step of this launch]: mapped
 * pinned host memory, or NULL.  A block that does not arrive within 10 s
 * aborts the run (gmf_status_read reports it).  gmf_reset zeroes the counter. */
void* gmf_stream_ready_ptr(gmf_handle* h);
int gmf_run_stream(gmf_handle* h, int64_t n_steps, void* host_status, void* stream);
/* enqueue "counter = value" on `stream` (H2D copy from handle-owned pinned
 * memory), i.e. step value - 1's block is complete on that stream */
int gmf_stream_signal(gmf_handle* h, int64_t value, void* stream);
/* K1 implementation the handle runs (GMF_K1_CUDA_CORES or GMF_K1_TENSOR) */
int gmf_k1_impl(gmf_handle* h);
/* K1 kernel generation the handle runs: 0 CUDA cores, 1 tensor cores (one
   32-row chunk per step of a 256-thread CTA), 2 tensor cores, warp-specialized
   tcgen05 pipeline (one 320-thread CTA per SM; chosen when a unit is at least
   512 rows deep, GMF_TC_VERSION=1|2 forces one) */
int gmf_k1_version(gmf_handle* h);
/* number of kernels this handle has launched so far (graph nodes counted) */
int64_t gmf_launch_count(gmf_handle* h);
int gmf_profile(gmf_handle* h, int enable, double* out, void* stream);
/* host copies of the first n trace entries (objective, nb shape) */
int gmf_trace_read(gmf_handle* h, double* obj, double* nb, int64_t n, void* stream);
/* the dispersion at the same trace points (FitReport.phi_trace, optim.py:326) */
int gmf_trace_phi_read(gmf_handle* h, double* phi, int64_t n, void* stream);

/* Deviance half of penalized_objective over ALL local entries at the current
 * state: *dev_sum (device double) = sum_ij w_ij D(y_ij, mu_ij). */
int gmf_objective_full(gmf_handle* h, double* dev_sum, void* stream);

/* Same pass plus the NB dispersion constant: out2 (device, 2 doubles) =
 * [sum_ij w D(y, mu), -2 sum_ij w (sat_ij + y log y)] at the handle's nb shape
 * (second entry 0 for Poisson).  AIC/BIC follow on the host (select.py:81-96). */
int gmf_loglik_full(gmf_handle* h, double* out2, void* stream);

/* mu = exp(eta) at n listed entries (rows: the handle's local row numbers,
 * int64; cols: int32; device arrays).  mu_out (device, n doubles) may be NULL;
 * with y (device, n doubles) and sums4 (device, 4 doubles) non-NULL the
 * entries are scored as gmf_score_pairs does, against the constant ybar. */
int gmf_entries_eval(gmf_handle* h, const int64_t* rows, const int32_t* cols, const double* y,
                     int64_t n, double ybar, double* mu_out, double* sums4, void* stream);

/* ---------------------------------------------------------------- level 3 */

/* out (host or device, a x b doubles, row-major) = A' B where A is rows x a
 * (row stride lda, column offset a0) and B is rows x b (ldb, b0); dtype
 * elements, fp64 accumulation, fixed-order reduction.  `work` is device
 * scratch of gmf_cross_work_bytes(a, b) bytes. */
int64_t gmf_cross_work_bytes(int32_t a, int32_t b);
int gmf_cross_rows(int dtype, int64_t rows, const void* A, int64_t lda, int32_t a0, int32_t a,
                   const void* B, int64_t ldb, int32_t b0, int32_t b, double* out_device,
                   void* work, void* stream);

/* Y[:, y0:y0+c] <- beta * Y[:, y0:y0+c] + A[:, a0:a0+a] @ M   (M: a x c doubles,
 * device, row-major); row-local, so Y may alias A. */
int gmf_rows_affine(int dtype, int64_t rows, void* Y, int64_t ldy, int32_t y0, int32_t c,
                    double beta, const void* A, int64_t lda, int32_t a0, int32_t a,
                    const double* M, void* stream);

/* ------------------------------------------------------- initialization */

/* out (nrows x r doubles, row-major) = S P with s_k = log(val_k + eps) - log(eps)
 * at the stored entries of a CSR (ptr int64, col/val int32; pass a CSC to get
 * S' Q); P is (ncols x r) row-major doubles.  Rows longer than 2048 nonzeros
 * are split into segments whose partials are summed in fixed order in `work`
 * (gmf_spmm_work_bytes bytes; may be NULL when that is 0). */
int64_t gmf_spmm_work_bytes(int64_t nrows, int64_t max_row_nnz, int32_t r);
int gmf_csr_spmm(int64_t nrows, const int64_t* ptr, const int32_t* col, const int32_t* val,
                 int64_t max_row_nnz, double eps, const double* P, int32_t r, double* out,
                 void* work, void* stream);

/* out2 (device) = [sum mu0^2, sum ((y - mu0)^2 - mu0)] over all n x m entries,
 * mu0 = exp(clip(x_i b_j + gamma_i z_j, eta_lo, eta_hi)); fp64, fixed order. */
int64_t gmf_moments_work_bytes(void);
int gmf_init_moments(int64_t n, int64_t m, const int64_t* ptr, const int32_t* col,
                     const int32_t* val, const double* x, const double* b, int32_t p,
                     const double* gamma, const double* z, int32_t q, double eta_lo,
                     double eta_hi, double* out2, void* work, void* stream);

/* --------------------------------------------------------- file formats */

/* Coordinate MatrixMarket -> CSR (host memory, caller-owned).  gmf_mm_header
 * gives n, m and an upper bound on the stored entries; gmf_mm_read_csr fills
 * indptr (n+1 int64), indices / counts (cap int32 each; rows column-sorted,
 * duplicates summed, zeros dropped) and *nnz_out.  integer / real (integral)
 * / pattern fields, general / symmetric. */
int gmf_mm_header(const char* path, int64_t* n, int64_t* m, int64_t* max_nnz);
int gmf_mm_read_csr(const char* path, int64_t cap, int64_t* indptr, int32_t* indices,
                    int32_t* counts, int64_t* nnz_out);

const char* gmf_last_error(void);
const char* gmf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GMF_ASGD_H */
