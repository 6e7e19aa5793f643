/*
 * bsb200.h — C ABI of the B200-native hot path behind the blockstat API.
 *
 * The reference (`/root/reference/pkg/src/blockstat`, pure Python + numpy) has no
 * native boundary: every local flop is a numpy call inside solvers.py /
 * distlinalg.py / distarray.py.  This header is the boundary a maintainer
 * binds (ctypes) to replace those calls.  Each entry point
 * cites the reference function(s) it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Device pointers point into the local
 *    block of a DistArray: the block of an R x C matrix is column-major, i.e.
 *    element (i, j) lives at [j * R + i] (distarray.py:82, order="F").
 *  - `dtype` codes follow the reference's wire codes (comm.py:68-72):
 *    0 = float32, 1 = float64, 2 = int64; 3 = int8 is new (genotype storage).
 *  - `op` codes follow ReduceOp's declaration order (comm.py:54-58).
 *  - Every call is asynchronous on `stream` (a cudaStream_t) and returns a
 *    status; nothing synchronizes the host.  Scalars that the reference returns
 *    to Python land in small device buffers (`double*` "_dev" arguments).
 *  - `work` is caller-owned device scratch of `work_bytes`; the matching
 *    *_workspace() query returns the bytes a call needs.  A workspace also holds
 *    the call's completion counters: zero it once before first use and keep one
 *    per stream.
 *  - The library never allocates device memory and keeps no global state
 *    besides a thread-local error string and the cached SM count.
 */
#ifndef BSB200_H
#define BSB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define BS_OK 0
#define BS_EINVAL 1   /* bad argument (maps to ValueError / ShapeError)       */
#define BS_ECUDA 2    /* CUDA launch/runtime failure                           */
#define BS_EWORK 3    /* workspace too small                                   */
#define BS_ENUMERIC 4 /* nonfinite risk weights (NumericError, solvers.py:388-389) */
#define BS_ENCCL 5    /* NCCL missing or failed                                  */
#define BS_EDEGEN 6   /* coincident embedding points (DegenerateConfigError)     */

/* dtype codes (comm.py:68-72; int8 added) */
#define BS_F32 0
#define BS_F64 1
#define BS_I64 2
#define BS_I8 3
#define BS_U2 4  /* 2-bit packed genotypes (X only; see bs_genotype_pack) */
#define BS_U2T 5 /* the packed transpose of a BS_U2 block (bs_cox_xbeta only; see bs_genotype_transpose_packed) */

/* ReduceOp codes (comm.py:54-58) */
#define BS_SUM 0
#define BS_PROD 1
#define BS_MAX 2
#define BS_MIN 3

/* element transforms applied before a reduction (distarray.py:340) */
#define BS_T_NONE 0
#define BS_T_ABS 1
#define BS_T_SQUARE 2

/* NMF algorithms (solvers.py:144, 165) */
#define BS_NMF_MU 0
#define BS_NMF_APG 1

/* device status flags written by the Cox and MDS kernels */
#define BS_FLAG_CLAMPED 1    /* exp argument clamped: RuntimeWarning, solvers.py:383-385 */
#define BS_FLAG_NONFINITE 2  /* nonfinite risk weights: NumericError, solvers.py:388-389 */
#define BS_FLAG_DEGENERATE 4 /* coincident points: DegenerateConfigError, solvers.py:291-295 */

/* ---- library ----------------------------------------------------------- */
const char* bs_last_error(void);
int bs_abi_version(void);
int bs_num_sms(void);
/* Kernels launched by this library so far in the process (all threads). */
int64_t bs_launch_count(void);
/* Adds n to bs_launch_count: the kernels a CUDA graph replay launched (their capture counted them
 * once; replays do not pass through the counting host code). */
void bs_note_replayed_launches(int64_t n);

/* ---- L1: distributed-array primitives (distarray.py) -------------------- */

/* rand_fill / _draw "uniform01" (distarray.py:170-208): writes elements
 * [first, first+count) of Generator(Philox(key)).random(N, dtype) — the numpy
 * stream, bit for bit (Philox4x64-10; f64 = (u64>>11)*2^-53, f32 = two u32
 * halves per word, low half first, (u32>>8)*2^-24).  dtype: BS_F32 / BS_F64. */
int bs_philox_uniform(void* out, int dtype, int64_t count, int64_t first,
                      uint64_t key0, uint64_t key1, void* stream);

/* Counter-based standard normals for synthetic inputs (a documented GPU normal;
 * numpy's ziggurat stream has data-dependent consumption): element e of the global stream is
 * Box-Muller on Philox4x64-10 block (e/2 + 1, 1, 0, 0) under (key0, key1), so the matrix does not
 * depend on the rank count.  Writes elements [first, first + count) to out (float32 / float64). */
int bs_philox_normal(void* out, int dtype, int64_t count, int64_t first,
                     uint64_t key0, uint64_t key1, void* stream);

/* Counter-based genotype matrix (the C5 input; no reference
 * equivalent -- the reference's rand_fill is float-only, distarray.py:176-177):
 * X[i, j] = [u1 < maf[j - lo]] + [u2 < maf[j - lo]] for the local columns j in
 * [lo, lo + n_loc), with u1, u2 elements 2e and 2e+1 (e = j*m + i) of
 * Generator(Philox(key)).random(., float64).  Rank-count independent. */
int bs_genotype_fill(int8_t* X, const double* maf, int64_t m, int64_t lo, int64_t n_loc,
                     uint64_t key0, uint64_t key1, void* stream);

/* 2-bit packed genotypes (BS_U2): column j of the local block takes
 * bs_genotype_packed_bytes(m) = ceil(m/64)*16 bytes at offset j * that; genotype i is
 * bits 2(i%4)..+1 of byte i/4.  Accepted as X by bs_cox_xbeta / bs_cox_grad_step with
 * float32 arithmetic (dtype BS_F32).  pack / unpack convert from / to int8 blocks;
 * fill_packed writes the bs_genotype_fill matrix directly packed. */
int64_t bs_genotype_packed_bytes(int64_t m);
int bs_genotype_pack(const int8_t* X, int64_t m, int64_t n_loc, void* P, void* stream);
int bs_genotype_unpack(const void* P, int64_t m, int64_t n_loc, int8_t* X, void* stream);
int bs_genotype_fill_packed(void* P, const double* maf, int64_t m, int64_t lo, int64_t n_loc,
                            uint64_t key0, uint64_t key1, void* stream);
/* Q = the packed (n_loc x m) transpose of the packed (m x n_loc) block P: row i of X takes
 * bs_genotype_packed_bytes(n_loc) bytes at offset i * that, genotype j in bits 2(j%4)..+1 of
 * byte j/4.  Passed as X with xdtype BS_U2T, bs_cox_xbeta (dtype BS_F32) computes X beta on
 * the tensor cores (kind::mxf4) from Q with the same pass as the packed gradient (an addition:
 * the layout trades the memory of a second copy for a K-major operand). */
int bs_genotype_transpose_packed(const void* P, int64_t m, int64_t n_loc, void* Q, void* stream);

/* reduce_all local fold (distarray.py:335-348): out_dev[0] = op over
 * transform(x[0..count)) in float64.  Empty input gives the neutral element. */
int64_t bs_reduce_workspace(int64_t count);
int bs_reduce(const void* x, int dtype, int64_t count, int op, int transform,
              double* out_dev, void* work, int64_t work_bytes, void* stream);

/* Communicator._fold (comm.py:93-99): dst = srcs[0] op srcs[1] op ... in
 * ascending rank order, no reassociation.  Used by the in-process backend. */
int bs_fold(void* dst, const void* const* srcs, int nsrc, int64_t count,
            int dtype, int op, void* stream);

/* diag_get owned entries (distlinalg.py:97-99): out[k] = M[lo + k, k]. */
int bs_diag_get(const void* M, int dtype, int64_t rows, int64_t lo,
                int64_t n_loc, void* out, void* stream);

/* scn d local product (distlinalg.py:265-268): G (r x r, float64) =
 * A_loc A_loc^T for the column-split r x ncols block A_loc. */
int64_t bs_gram_workspace(int r, int64_t ncols);
int bs_gram(const void* A, int dtype, int r, int64_t ncols, double* G,
            void* work, int64_t work_bytes, void* stream);

/* pairwise_euclidean (distlinalg.py:442-468), the MDS input builder:
 * Y[i, lo + k] = ||x_i - x_{lo+k}||_2 for the owned columns k < n_loc of the
 * n x n target; x is the gathered d x n point matrix (points = columns).
 * Direct-difference formula, zero diagonal. */
int bs_pairwise_euclidean(const void* x, int dtype, int64_t d, int64_t n,
                          int64_t lo, int64_t n_loc, void* Y, void* stream);

/* ---- NMF (solvers.py:73-185) ------------------------------------------- */

/* _nmf_check + ||X||^2 (solvers.py:139-141; objective constant):
 * out_dev = {min(X), sum(X^2)} over the local block, float64. */
int bs_nmf_scan(const void* X, int dtype, int64_t count, double* out_dev,
                void* work, int64_t work_bytes, void* stream);

/* Per-call pass over X (the reference's _nmf_check, solvers.py:139-141, which
 * runs at the start of every nmf_multiplicative / nmf_apg call):
 *   stats_dev = {min(X), sum(X^2), nonfinite?, scales_ready?}  (float64)
 * For float32 X (m % 4 == 0) it also writes, into xscale (bs_nmf_xscale_bytes),
 * the power-of-two block scales the integer tensor-core GEMMs use: one per
 * (row, 512 columns) for scn b and one per (column, 512 rows) for scn a. */
int64_t bs_nmf_xscale_bytes(int64_t m, int64_t n_loc);
int64_t bs_nmf_prepare_workspace(int64_t m, int64_t n_loc);
int bs_nmf_prepare(const void* X, int dtype, int64_t m, int64_t n_loc,
                   double* stats_dev, void* xscale, void* work,
                   int64_t work_bytes, void* stream);

/* How many hot-path passes ran on each kernel path since the last reset (process-wide):
 * out8 = {NMF GEMM on integer digit-slice tcgen05, NMF GEMM on 3xTF32 tcgen05,
 *         NMF GEMM on float32 CUDA cores, NMF GEMM in float64 (DMMA / CUDA cores),
 *         MDS pass on tcgen05 (mds_tc.cu), MDS pass on CUDA cores,
 *         packed-genotype Cox pass (gradient or X.beta) on tcgen05 kind::mxf4 (genotype_tc.cu), 0}. */
int bs_gemm_path_counts(int64_t* out8, int reset);
/* Adds delta8 to those counts (CUDA graph replays of captured solver iterations). */
void bs_add_gemm_path_counts(const int64_t* delta8);

/* scn b local GEMM (distlinalg.py:246-252): P (r x m, column-major, float32
 * or float64 like X) = W_loc X_loc^T summed over the rank's n_loc columns.
 * The caller reduce-scatters P across ranks (distlinalg.py:251-252).
 * xscale (nullable): scales from bs_nmf_prepare; float32 with r <= 64 then runs
 * the exact-accumulation integer digit-slice kernel (nmf_i8.cu). */
int64_t bs_nmf_wxt_workspace(int dtype, int64_t m, int64_t n_loc, int r);
int bs_nmf_wxt(const void* X, const void* W, int dtype, int64_t m,
               int64_t n_loc, int r, void* P, const void* xscale, void* work,
               int64_t work_bytes, void* stream);

/* scn b fused with _nmf_check (solvers.py:139-141, 147): the same X pass also
 * yields stats_dev = {min, sum X^2} (float64; with padded tcgen05 tiles the min
 * is min(min X, 0), enough for the nonnegativity check).  The solver uses it for
 * the first iteration of every call instead of a separate bs_nmf_scan pass. */
int64_t bs_nmf_wxt_scan_workspace(int dtype, int64_t m, int64_t n_loc, int r);
int bs_nmf_wxt_scan(const void* X, const void* W, int dtype, int64_t m,
                    int64_t n_loc, int r, void* P, double* stats_dev,
                    void* work, int64_t work_bytes, void* stream);

/* Vt half-step, fused (solvers.py:151-156 MU, 172-178 APG):
 *   WWtVt = WWt Vt_loc (scn j), sigma = 1/(2 sum WWt^2 + eps) (APG),
 *   Vt <- Vt*WXt/(WWtVt+eps) | max(0, Vt - sigma (WWtVt - WXt)),
 *   VtV = Vt_new Vt_new^T over the local columns (scn d local part, float64).
 * WXt: r x m_loc reduced block.  Vt_copy (nullable) receives a copy of the
 * new block (the caller's all-gather source). */
int64_t bs_nmf_vt_step_workspace(int r, int64_t m_loc);
int bs_nmf_vt_step(int algo, void* Vt, const void* WXt, const double* WWt,
                   int dtype, int r, int64_t m_loc, double eps, double* VtV,
                   void* Vt_copy, void* work, int64_t work_bytes, void* stream);

/* W half-step, fused (solvers.py:155-159 MU, 177-182 APG) with the next
 * iteration's scn d and the objective's cross term:
 *   VtX = Vt_full X_loc (scn a, distlinalg.py:239-243), VtVW = VtV W (scn j),
 *   tau = 1/(2 sum VtV^2 + eps) (APG), W <- update,
 *   red[0 .. r*r) = W_new W_new^T (local), red[r*r] = <VtX, W_new> (local).
 * Vt_full: r x m gathered factor. */
int64_t bs_nmf_w_step_workspace(int dtype, int64_t m, int64_t n_loc, int r);
int bs_nmf_w_step(int algo, const void* X, const void* Vt_full, void* W,
                  const double* VtV, int dtype, int64_t m, int64_t n_loc,
                  int r, double eps, double* red, const void* xscale,
                  void* work, int64_t work_bytes, void* stream);

/* nmf_objective after an update via the Gram identity
 * ||X - V^T W||^2 = ||X||^2 - 2 <VtX, W> + <VtV, WWt> (solvers.py:124-136):
 * out_dev[0] = xsq[0] - 2 red[r*r] + sum(VtV .* red[0..r*r)).
 * direct_flag (nullable) is set to 1 when kappa < 0, or when kappa > 0 and the value
 * is within the cancellation regime (xsq / obj > kappa, or obj <= 0); 0 otherwise. */
int bs_nmf_objective(const double* xsq, const double* red, const double* VtV,
                     int r, double* out_dev, int* direct_flag, double kappa,
                     void* stream);

/* Cancellation guard: direct_flag (set by bs_nmf_objective when ||X||^2 / obj
 * > kappa) selects the direct residual: out_dev[0] = direct_dev[0] if *flag. */
int bs_nmf_objective_select(const int* direct_flag, const double* direct_dev,
                            double* out_dev, void* stream);

/* nmf_objective standalone (solvers.py:124-136), direct residual:
 * out_dev[0] = sum over the local block of (X - Vt_full^T W_loc)^2.
 * flag_dev (nullable): when it points to 0 the pass is skipped and out_dev[0] = 0. */
int64_t bs_nmf_residual_workspace(int64_t m, int64_t n_loc);
int bs_nmf_residual(const void* X, const void* Vt_full, const void* W,
                    int dtype, int64_t m, int64_t n_loc, int r, double* out_dev,
                    const int* flag_dev, void* work, int64_t work_bytes,
                    void* stream);

/* ---- MDS (solvers.py:188-305) ------------------------------------------ */

/* One fused pass over the rank's columns [lo, lo+n_loc) of Y (n x n), replacing
 * _embedding_distances + the stress/zero-pair fold + Z + reduce_into + scn a
 * (solvers.py:237-247, 279-301).  theta_full: q x n gathered embedding.
 *   red[0] = sum (Y - D)^2,  red[1] = #zero off-diagonal distances  (local)
 *   zsum[j] = sum_i Z_ij,  T[:, j] = theta (W - Z)[:, j]   (mode 0 only)
 * mode 0 = full MM pass, 1 = stress only (mds_stress, solvers.py:250-266).
 * perturb != 0 substitutes 1e-10 for zero off-diagonal distances. */
int64_t bs_mds_pass_workspace(int dtype, int64_t n, int64_t n_loc, int q);
int bs_mds_pass(const void* Y, const void* theta_full, int dtype, int64_t n,
                int64_t lo, int64_t n_loc, int q, int perturb, int mode,
                double* red, void* zsum, void* T, void* work,
                int64_t work_bytes, void* stream);

/* theta update (solvers.py:291-304): if red[1] > 0 and !perturb, sets
 * BS_FLAG_DEGENERATE in *flags and leaves theta untouched; otherwise
 * theta <- (theta (zsum + wsum) + T) / (2 wsum).  A set flag on entry also
 * skips the update (an earlier iteration already failed). */
int bs_mds_update(void* theta_loc, const void* zsum, const void* T, int dtype,
                  int q, int64_t n_loc, double wsum, const double* red,
                  int perturb, int* flags, void* stream);

/* ---- l1-Cox (solvers.py:308-450) ---------------------------------------- */

/* scn m local GEMV (distlinalg.py:334-337): out (m, float64) = X_loc beta_loc.
 * xdtype: BS_F32 / BS_F64 / BS_I8 (widened in-register); beta: `dtype`. */
int64_t bs_cox_xbeta_workspace(int xdtype, int64_t m, int64_t n_loc);
int bs_cox_xbeta(const void* X, int xdtype, const void* beta, int dtype,
                 int64_t m, int64_t n_loc, double* out, void* work,
                 int64_t work_bytes, void* stream);

/* _risk_weights + the log partial likelihood (solvers.py:376-398) on the
 * reduced linear predictor xb (float64, m):
 *   Xbeta = xb, w = exp(min(xb, clamp)), W = cumsum(w) (forward),
 *   loglik_dev[0] = sum delta (xb - log W[cuts]).
 * Sets BS_FLAG_CLAMPED / BS_FLAG_NONFINITE in *flags.  Outputs in `dtype`.
 * A set BS_FLAG_NONFINITE on entry makes the call a no-op.  With a zeroed
 * workspace of bs_cox_risk_workspace(m) bytes (nonzero for long m) the scans run
 * on many CTAs with results bitwise equal to the single-CTA scan; without one
 * (NULL, 0) the single-CTA kernel runs. */
int64_t bs_cox_risk_workspace(int64_t m);
int bs_cox_risk(const double* xb, const void* delta, const int64_t* cuts,
                int dtype, int64_t m, double clamp, void* Xbeta, void* w,
                void* W, double* loglik_dev, int* flags, void* work,
                int64_t work_bytes, void* stream);

/* pi_delta over the owned range [lo, hi) (solvers.py:401-419), without the
 * allreduce: pd_i = w_i sum_{j in [lo,hi), cuts_j >= i} delta_j / W[cuts_j].
 * cuts == NULL means cuts = arange(m).  dmpd (nullable, float64) receives
 * delta - pd (solvers.py:446). */
int64_t bs_cox_pi_delta_workspace(int64_t m);
int bs_cox_pi_delta(const void* w, const void* W, const void* delta,
                    const int64_t* cuts, int dtype, int64_t m, int64_t lo,
                    int64_t hi, void* pd, double* dmpd, const int* flags,
                    void* work, int64_t work_bytes, void* stream);

/* scn p local GEMV + prox (distlinalg.py:355-358, solvers.py:447-449):
 * grad = X_loc^T dmpd; if do_step: beta <- S_lam(beta + sigma grad);
 * l1_dev[0] = sum |beta| after the call (local, float64). */
int64_t bs_cox_grad_workspace(int xdtype, int64_t m, int64_t n_loc);
int bs_cox_grad_step(const void* X, int xdtype, const double* dmpd, int dtype,
                     int64_t m, int64_t n_loc, void* grad, void* beta,
                     double sigma, double lam, int do_step, double* l1_dev,
                     const int* flags, void* work, int64_t work_bytes,
                     void* stream);

/* Fused iteration pass (solvers.py:443-449 then :436 of the next iteration):
 * grad = X_loc^T dmpd, beta <- S_lam(beta + sigma grad), xb_out[0:m] = X_loc beta
 * (local partial, float64) and xb_out[m] = sum |beta| (local) -- the effects of
 * bs_cox_grad_step(do_step = 1) followed by bs_cox_xbeta, with X streamed once
 * (cooperative persistent kernel, column waves held in shared memory).
 * allow_fused = 0 (or an unsupported shape) runs those two entry points instead;
 * pass 0 when other kernels may share the device concurrently. */
int64_t bs_cox_grad_xbeta_workspace(int xdtype, int64_t m, int64_t n_loc);
int bs_cox_grad_xbeta(const void* X, int xdtype, const double* dmpd, int dtype,
                      int64_t m, int64_t n_loc, void* grad, void* beta,
                      double sigma, double lam, double* xb_out, const int* flags,
                      int allow_fused, void* work, int64_t work_bytes, void* stream);

/* trace entry (solvers.py:438-441): out_dev[0] = -loglik + lam * l1. */
int bs_cox_objective(const double* loglik_dev, const double* l1_dev, double lam,
                     double* out_dev, void* stream);

/* ---- solver-level runtime (SURVEY.md 8(b) build proposal) ------------------
 * A per-rank context owns a stream and, for size > 1, an NCCL communicator
 * (libnccl.so.2 is loaded at run time).  Rank 0 calls bs_nccl_unique_id and ships
 * the 128 bytes to the other ranks out of band (the Python layer uses its
 * communicator); every rank then calls bs_ctx_create with the same id.  States own
 * their workspaces; the caller owns X, delta, cuts, beta and grad (device memory,
 * column split as in cox_init, solvers.py:337-373).  Every call that communicates is
 * collective: all ranks issue it in the same order. */
typedef struct bs_ctx* bs_ctx_t;
typedef struct bs_cox* bs_cox_t;
int bs_nccl_unique_id(void* out128);
int bs_ctx_create(int rank, int size, int device, const void* nccl_unique_id,
                  void* stream, bs_ctx_t* out);
int bs_ctx_destroy(bs_ctx_t ctx);

/* CoxState (solvers.py:313-373) with sigma given; float32 X with float32
 * arithmetic runs the fused one-stream pass, as cox_fit does by default. */
int bs_cox_state_create(bs_ctx_t ctx, const void* X, int xdtype, int dtype,
                        int64_t m, int64_t n_loc, const void* delta,
                        const int64_t* cuts, double lam, double sigma,
                        void* beta, void* grad, bs_cox_t* out);
int bs_cox_state_destroy(bs_cox_t state);

/* cox_fit (solvers.py:422-450): iters proximal-gradient steps.  trace_out (host,
 * >= ceil(iters / trace_every) doubles) receives the objective of the iterate
 * entering every trace_every-th step; monitor_window > 0 applies the
 * ConvergenceMonitor rule (solvers.py:54-70) with monitor_tol, which may stop
 * before stepping.  *iters_run = iterations completed (the first nonfinite one
 * on BS_ENUMERIC), *flags_out = BS_FLAG_* seen (CLAMPED means warn). */
int bs_cox_run(bs_cox_t state, int iters, int trace_every, int monitor_window,
               double monitor_tol, double* trace_out, int* ntrace_out,
               int* iters_run, int* flags_out);

/* NmfState (solvers.py:73-121) over the caller's X, Vt (r x m_loc, the rank's
 * partition_of(m) block) and W (r x n_loc); the state owns WXt, the gathered Vt
 * and the workspaces.  bs_nmf_run = nmf_multiplicative / nmf_apg (solvers.py:
 * 144-185; algo BS_NMF_MU / BS_NMF_APG): trace_out receives the objective after
 * every trace_every-th update; BS_EINVAL if X has a negative entry
 * (solvers.py:139-141). */
typedef struct bs_nmf* bs_nmf_t;
int bs_nmf_state_create(bs_ctx_t ctx, const void* X, int dtype, int64_t m,
                        int64_t n_loc, int r, double eps, void* Vt, void* W,
                        bs_nmf_t* out);
int bs_nmf_state_destroy(bs_nmf_t state);
int bs_nmf_run(bs_nmf_t state, int algo, int iters, int trace_every,
               double* trace_out, int* ntrace_out);

/* MdsState (solvers.py:193-234) over the caller's Y (n x n_loc) and theta
 * (q x n_loc); bs_mds_run = mds_fit (solvers.py:269-305): trace_out receives the
 * stress of the iterate entering every trace_every-th update; BS_EDEGEN when a
 * zero off-diagonal distance appears without perturb (traces up to that
 * iteration are returned). */
typedef struct bs_mds* bs_mds_t;
int bs_mds_state_create(bs_ctx_t ctx, const void* Y, int dtype, int64_t n,
                        int64_t n_loc, int q, int perturb, void* theta,
                        bs_mds_t* out);
int bs_mds_state_destroy(bs_mds_t state);
int bs_mds_run(bs_mds_t state, int iters, int trace_every, double* trace_out,
               int* ntrace_out);

#ifdef __cplusplus
}
#endif
#endif /* BSB200_H */
