/*
 * sas.h — C ABI of the B200-native SubApSnap online phase (libsas.so).
 *
 * This is the drop-in boundary for the reference's online hot path
 * (/root/reference/pkg/src/subapsnap/online.py).  Every entry point below names
 * the reference interface it replaces.  Plain C types only: host or device
 * pointers, sizes and a cudaStream_t passed as void*.  No torch types.
 *
 *   reference (Python)                               C ABI
 *   -----------------------------------------------  ---------------------------
 *   online.precompute_online      online.py:68-102   sas_plan_create
 *   online.solve_online/solve_batch online.py:105-134, 208-225
 *                                                    sas_solve (device buffers)
 *                                                    sas_solve_host (host buffers)
 *   linalg.solve_ls               linalg.py:89-113   (inside sas_solve)
 *   online.estimate_residual      online.py:137-153  (scalar; host shim)
 *   OnlineSolution.lift           online.py:50-54    sas_lift
 *   cli verification residual     cli.py:344-351     sas_residual
 *   (plan is a frozen dataclass)  online.py:26-37    sas_plan_destroy
 *
 * Error convention (mirrors subapsnap.errors): functions return SAS_OK or an
 * error code, sas_last_error() gives the message of the last failure on the
 * calling thread.  Per-parameter numerical outcomes go to status[]:
 *   SAS_ST_OK, SAS_ST_RANK_DEFICIENT (linalg.py:107-112, RankDeficiencyError),
 *   SAS_ST_NONFINITE (linalg.py:36-37, ValueError "non-finite entries").
 *
 * Threading (the reference's solve_online is pure and may be called from many
 * threads): every call on a plan may come from any host
 * thread; calls on one plan serialise on the plan, and device work that uses
 * the plan's scratch buffers is ordered across the callers' streams (a call
 * on a different stream than the previous one waits for it on the device).
 * Independent plans run concurrently.
 */
#ifndef SAS_H_
#define SAS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes */
#define SAS_OK 0
#define SAS_ERR_ARG 1
#define SAS_ERR_CUDA 2
#define SAS_ERR_NCCL 3
#define SAS_ERR_NUMERICAL 4

/* per-parameter status */
#define SAS_ST_OK 0
#define SAS_ST_RANK_DEFICIENT 1
#define SAS_ST_NONFINITE 2

/* element types of X, blocks, coefficients */
#define SAS_F64 0
#define SAS_C128 1

/* operator kinds (how S*A(p)*X is assembled on the device) */
#define SAS_OP_AFFINE 0   /* M = sum_k f_k(p) B_k, B_k = S A_k X (online.py:81-85, 108-112) */
#define SAS_OP_STENCIL 1  /* edge-form FD rows with log-affine coefficients, see sas_desc */
#define SAS_OP_GAUSS 2    /* Gaussian kernel rows exp(-|x_i-x_j|^2/(2p^2)) + ridge*I */

/* affine coefficient kinds (systems.py:76-100, parse_coefficient systems.py:549-570) */
#define SAS_COEF_CONST 0  /* f = scale                 (const_term)  */
#define SAS_COEF_LINEAR 1 /* f = scale * p[0]          (linear_term) */
#define SAS_COEF_EXP 2    /* f = scale * exp(rate*p[0]) ("c*exp(a*p)") */
#define SAS_COEF_TABLE 3  /* f given per parameter by the caller (opaque callables) */

/* flags for sas_plan_create */
#define SAS_FLAG_INPUT_DEVICE 1u /* X pointer is a device pointer on the plan's device */

typedef struct sas_plan sas_plan;

typedef struct sas_desc {
  int32_t op_kind;       /* SAS_OP_* */
  int32_t dtype;         /* SAS_F64 or SAS_C128: arithmetic of M, X, coefficients */
  int32_t param_dim;     /* d_p: scalars per parameter value */
  int32_t param_complex; /* 1: params are (re,im) pairs; 0: real doubles */

  /* SAS_OP_AFFINE: K terms; blocks are K x s x r row-major in `dtype` (host),
     exactly the reference plan.blocks (unweighted, duplicates expanded). */
  int32_t n_terms;
  const int32_t* term_kind;  /* K */
  const double* term_scale;  /* K x 2 (re, im) */
  const double* term_rate;   /* K x 2 (re, im), SAS_COEF_EXP only; may be NULL */
  const void* blocks;        /* K*s*r */

  /* SAS_OP_STENCIL: row i of A(p) (for selected node S_i) is
       A(p)_{i,S_i}   =  sum_e c_e(p),     A(p)_{i,nbr_e} = -c_e(p) (nbr_e >= 0)
       c_e(p)         =  exp(sum_k p_k * phi[i][e][k]) / edge_div
     (edge-midpoint FD as in systems.py:306-334).  nbr_e = -1 marks a Dirichlet
     boundary edge (contributes to the diagonal only). */
  int32_t n_edges;           /* E per row (4 in 2-D, 6 in 3-D) */
  const int64_t* edge_nbr;   /* s x E */
  const double* edge_phi;    /* s x E x d_p */
  double edge_div;           /* h*h */

  /* SAS_OP_GAUSS: rows of K_p + ridge*I, K_p(i,j) = exp(-D_ij * inv(p)),
     D_ij = sum_k (x_ik - x_jk)^2 (sequential sum, no FMA), inv = 1/(2 p p). */
  const double* points;      /* n x point_dim (host) */
  int32_t point_dim;
  double ridge;
} sas_desc;

/* Build a plan on CUDA device `device` (replaces online.precompute_online).
 *   X       n x r row-major (basis.basis), dtype per desc->dtype; host unless
 *           SAS_FLAG_INPUT_DEVICE.
 *   S       s selected row indices (selector.indices, repeats allowed).
 *   w       s weights or NULL (selector.weights).
 *   t       s values of b(p)[S] (p-independent right-hand side), dtype.
 *   proj    r values of c^H X (plan.output_projection) or NULL, dtype.
 * All host arrays are copied; the plan owns its device memory. */
int sas_plan_create(const sas_desc* desc, const void* X, int64_t n, int32_t r,
                    const int64_t* S, const double* w, int32_t s, const void* t,
                    const void* proj, int32_t device, uint32_t flags,
                    sas_plan** out);

/* Solve P parameter values (replaces solve_batch/solve_online).
 * Device pointers on the plan's device; `stream` is a cudaStream_t.
 *   params      P x d_p (x2 if param_complex)
 *   coef_table  P x K x 2 doubles, only for SAS_COEF_TABLE terms, else NULL
 *   rhs_table   P x s values of b(p)[S] in dtype, or NULL to use the plan's t
 *   coef        out, P x r (dtype)             OnlineSolution.coefficients
 *   sampled_res out, P doubles                  OnlineSolution.sampled_residual
 *   out_val     out, P x 2 doubles or NULL      OnlineSolution.output_value
 *   status      out, P int32 (SAS_ST_*)
 *   bad_col     out, P int32 or NULL: column of min |R_ii| when rank-deficient
 * Returns SAS_OK once the work is enqueued (status is filled asynchronously). */
int sas_solve(sas_plan* plan, const void* params, int64_t P,
              const double* coef_table, const void* rhs_table, void* coef,
              double* sampled_res, double* out_val, int32_t* status,
              int32_t* bad_col, void* stream);

/* Same contract with HOST buffers: copies params in, results out, synchronizes.
 * The reference-facing entry point (what a ctypes/cgo binding would call). */
int sas_solve_host(sas_plan* plan, const void* params, int64_t P,
                   const double* coef_table, const void* rhs_table, void* coef,
                   double* sampled_res, double* out_val, int32_t* status,
                   int32_t* bad_col);

/* x = X c for P coefficient vectors (OnlineSolution.lift, online.py:50-54).
 * coef: P x r device (dtype); x: P x n device (dtype). Needs the full X on the
 * device (kept by every plan). */
int sas_lift(sas_plan* plan, const void* coef, int64_t P, void* x, void* stream);

/* Full relative residual ||A(p) x - b(p)|| / max(||b(p)||, 1e-300) of x = X c
 * (cli.py:344-351); needs the full operator (sas_plan_set_operator).
 *   params      P x d_p (x2 if param_complex), device
 *   coef        P x r (dtype), device
 *   coef_table  P x K x 2 doubles (SAS_COEF_TABLE terms) or NULL, device
 *   b_table     P x n (dtype) right-hand sides b(p), or NULL for the plan's
 *               constant b (stencil plans: NULL only), device
 *   relres      out, P doubles, device
 *   floor_est   out, P doubles or NULL: the rounding floor
 *               100 eps || |A(p)| |x| || / ||b(p)|| below
 *               which a relative residual is noise, device
 * Stencil plans never materialise A(p) (edge coefficients re-evaluated per
 * parameter); affine plans run the K CSR terms; Gaussian plans re-evaluate
 * kernel rows (n^2 exps per parameter: meant for small subsets). */
int sas_residual(sas_plan* plan, const void* params, const void* coef, int64_t P,
                 const double* coef_table, const void* b_table, double* relres,
                 double* floor_est, void* stream);

/* Full operator for sas_residual (CSR per affine term, or the full stencil
 * description, or nothing for SAS_OP_GAUSS which re-evaluates kernel rows).
 *   affine:  K CSR matrices n x n (row_ptr n+1, col int64, val dtype), b (n)
 *   stencil: nbr n x E (int64), phi n x E x d_p, b (n)
 * Host pointers. */
int sas_plan_set_operator(sas_plan* plan, const int64_t* const* row_ptr,
                          const int64_t* const* col, const void* const* val,
                          const int64_t* nbr_full, const double* phi_full,
                          const void* b_full);

/* Metadata */
int sas_plan_info(const sas_plan* plan, int64_t* n, int32_t* r, int32_t* s,
                  int32_t* dtype, int32_t* op_kind, int32_t* device);

/* Number of kernels the last sas_solve enqueued (for launch accounting). */
int32_t sas_last_launch_count(const sas_plan* plan);

/* Per-launch timing.  With timing enabled, every kernel a call enqueues is
 * bracketed by CUDA events on the launching stream; sas_stage_times
 * synchronizes on them and returns, for the last sas_solve, the launch count
 * and per-launch milliseconds with their stage ids (SAS_STAGE_*). */
#define SAS_STAGE_LSQ 1        /* K4 batched least squares (+ fused assembly) */
#define SAS_STAGE_GAUSS_ROWS 2 /* K3 Gaussian kernel-row contraction */
#define SAS_STAGE_STENCIL_ROWS 3 /* K2 stencil-row assembly as its own launch (compact-WY path) */
int sas_plan_set_timing(sas_plan* plan, int32_t enable);
int32_t sas_stage_times(sas_plan* plan, float* ms, int32_t* stage, int32_t cap);

/* R factor of a tall m x w matrix (w <= 64) by TSQR (block Householder QRs,
 * then the stacked R blocks): the QR of the full least squares
 * online.solve_apsnap (online.py:156-165 -> linalg.solve_ls, linalg.py:89-113)
 * and of the leverage selector's range basis (subsample.py:144-159).
 *   A  m x w row-major, device, dtype SAS_F64 / SAS_C128
 *   R  w x w row-major, device, upper triangular (np.linalg.qr's R up to
 *      the signs of its rows)
 * Stream-ordered; scratch comes from the stream-ordered allocator. */
int sas_tsqr_r(const void* A, int64_t m, int32_t w, int32_t dtype, void* R, int32_t device, void* stream);

/* Leverage-score row selection, dense part (replaces subsample._range_basis +
 * leverage_scores, subsample.py:84-94, 144-159, for tall targets): Q = A C and
 * scores_i = ||Q_i||^2.  The caller builds C from sas_tsqr_r's R factor (SVD of
 * the small R on the host, then C <- C R2^-1 from the R factor of Q until Q is
 * orthonormal to rounding: offline.leverage_scores_gpu).
 *   A       m x w row-major, device, dtype SAS_F64 / SAS_C128
 *   C       w x k row-major, HOST (k <= w <= 64)
 *   Q       m x k row-major, device, or NULL
 *   scores  m doubles, device, or NULL
 * Stream-ordered; fixed summation order. */
int sas_range_rows(const void* A, int64_t m, int32_t w, const void* C, int32_t k, int32_t dtype, void* Q,
                   double* scores, int32_t device, void* stream);

/* Offline snapshot solve of a stencil system (replaces full_solve,
 * systems.py:187-222, for configs 3 and 5): Jacobi-preconditioned CG on
 *   (A v)_i = dg_i v_i - sum_e ct[i][e] v_{nbr[i][e]}   (nbr = -1: Dirichlet edge)
 * with fused kernels (q = A p with the direction update, then the vector
 * updates with their dot products).  Stops at ||r|| <= tol ||b|| or
 * ||r|| <= 1e-12 (a_norm ||x|| + ||b||), checked every check_every iterations.
 * All arrays device (n, n x E); outputs: iterations, the TRUE residual
 * ||b - A x|| and ||x|| (the caller applies the reference's residual guard). */
int sas_cg_stencil(int64_t n, int32_t E, const double* dg, const double* ct, const int64_t* nbr,
                   const double* b, double* x, double tol, double a_norm, int32_t maxiter,
                   int32_t check_every, int32_t device, void* stream, int32_t* iters_out,
                   double* rnorm_out, double* xnorm_out);

void sas_plan_destroy(sas_plan* plan);
const char* sas_last_error(void);
const char* sas_version(void);

/* Offline snapshot solve of a large affine system (replaces full_solve,
 * systems.py:187-222, for config 4): Jacobi-preconditioned BiCGSTAB on the
 * CSR matrix A(p) = sum_k f_k(p) A_k with fused kernels (k_bicg.cuh: direction
 * update, SpMV with its dot products, vector updates; device-side fixed-order
 * reductions).  Stops at ||r|| <= tol ||b|| or ||r|| <= 1e-12 (a_norm ||x|| +
 * ||b||), checked every check_every iterations.
 *   rowptr (n + 1), colind (nnz)  int32, device;  val (nnz), diag, b, x (n)  dtype, device
 * Outputs: iterations, the TRUE residual ||b - A x|| and ||x|| (the caller
 * applies the reference's residual guard). */
int sas_bicgstab_csr(int64_t n, const int32_t* rowptr, const int32_t* colind, const void* val, const void* diag,
                     const void* b, void* x, int32_t dtype, double tol, double a_norm, int32_t maxiter,
                     int32_t check_every, int32_t device, void* stream, int32_t* iters_out, double* rnorm_out,
                     double* xnorm_out);

#ifdef __cplusplus
}
#endif

#endif /* SAS_H_ */
