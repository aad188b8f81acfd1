/*
 * fctn_b200.h — C ABI of the B200-native PAM sweep for trace-regularized
 * FCTN tensor completion (arXiv 2510.22506).
 *
 * The reference (`fctnlr` 0.1.0, pure Python/numpy) has no FFI layer; its
 * drop-in boundary is the Python solver API `fctnlr.solver.run(obs, cfg)`
 * (solver.py:277).  These entry points are what that API's inner loop binds
 * to (the ctypes binding lives in paper_2510_22506_b200/_native.py; see
 * INTEGRATION.md for the stub a reference maintainer would add).  Every
 * pointer is a plain host pointer; no torch types cross the boundary.
 *
 * Layout conventions (reference tensor.py:1-12): first-index-fastest.
 *  - X, mask: order-N tensor, F-order, `dims` extents.
 *  - factor k: its mode-k unfolding A_(k), an I_k x s_k column-major matrix
 *    (rows mode k, columns the other slots ascending, first fastest) —
 *    `mode_unfold(f.factor(k), k)` (solver.py:325, tensor.py:130-139).
 *  - rank table: strict upper triangle, row-major (network.py:41-85).
 *
 * Status codes: 0 ok; 1 usage/shape error (-> ValueError); 2 numerical
 * failure (-> NumericalFailure, sylvester.py:39-40,109-113, solver.py:304,357);
 * 3 CUDA/runtime error.  `fctn_last_error` gives the message.
 *
 * Determinism: fixed reduction orders, no floating-point atomics; identical
 * inputs give identical bits (test_acceptance.py:407-443 contract).
 * A context owns all its device memory and one CUDA stream; not thread-safe.
 */
#ifndef FCTN_B200_H
#define FCTN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fctn_ctx fctn_ctx;

#define FCTN_F64 0
#define FCTN_F32 1

#define FCTN_ALG_PLAIN 0       /* algorithm="fctnlr"  (solver.py:322-324, 343) */
#define FCTN_ALG_ACCEL 1       /* algorithm="afctnlr" (solver.py:318-320, 337-341) */

#define FCTN_SIGN_PD 0         /* laplacian_sign="positive-definite" (laplacian.py:22) */
#define FCTN_SIGN_PRINTED 1    /* laplacian_sign="as-printed" */

/* Sweep statistics written by fctn_sweep (indices into `out`). */
#define FCTN_ST_OBJECTIVE 0    /* objective after the sweep (solver.py:356) */
#define FCTN_ST_DIFF_SQ 1      /* ||X_new - X_old||^2 (solver.py:346) */
#define FCTN_ST_BASE_SQ 2      /* ||X_old||^2 (solver.py:347) */
#define FCTN_ST_DATA_SQ 3      /* ||X_new - C||^2 (solver.py:220) */
#define FCTN_ST_XNEW_SQ 4      /* ||X_new||^2 (solver.py:382) */
#define FCTN_ST_PENALTY 5      /* sum_k lam_k/2 tr(A^T L A) (solver.py:221-223) */
#define FCTN_ST_STEP_FAC 6     /* sum_k ||A_new - A_prev||^2 (solver.py:332) */
#define FCTN_ST_FNORM_MAX 7    /* max_k ||A_k||_F (solver.py:383-385) */
#define FCTN_ST_DEVICE_MS 8    /* CUDA-event time of the sweep */
#define FCTN_ST_COUNT 16

/* Trace counters written by fctn_sweep / fctn_plan_sweeps (indices). */
#define FCTN_CT_FLOPS 0        /* reference FLOP meter total for the sweep (tensor.py:32-72) */
#define FCTN_CT_MK 1           /* "mk" label */
#define FCTN_CT_COMPOSE 2      /* "compose" label */
#define FCTN_CT_HITS 3         /* reuse-cache hits (network.py:398-407) */
#define FCTN_CT_LAUNCHES 4     /* kernels launched by the library in the sweep */
#define FCTN_CT_COUNT 8

/* Create a context on `device`.  Replaces the setup of solver.py:278-300:
 * rank table (network.py:68-77), Laplacian spectra (laplacian.py:46-47), the
 * reuse cache with its fp64 byte budget (network.py:377-417; solver.py:127).
 * `lam`, `delta`: n values each.  `n_ranks`/`rank`: sharding along mode 0
 * (slab [slab_lo, slab_hi) of I_0 held by this rank; pass 0,1,0,dims[0] for
 * a single GPU). */
int fctn_create(int device, int dtype, int n, const int64_t* dims, const int64_t* rank_tri,
                const double* lam, const double* delta, int lap_sign, double rho, int algorithm,
                int64_t cache_budget, fctn_ctx** out);

/* Host -> device: the observed tensor (values zero off the mask; solver.py:79,297)
 * in the context dtype (double* for FCTN_F64, float* for FCTN_F32) and the
 * mask (one byte per entry, 0/1).  Sets X := values. */
int fctn_upload(fctn_ctx* ctx, const void* x_F, const uint8_t* mask_F);

/* fctn_upload for float64 host data whatever the context dtype (the FP32
 * variant converts on the device); mask one byte per entry. */
int fctn_upload_f64(fctn_ctx* ctx, const double* x_F, const uint8_t* mask_F);

/* Replace every factor (mode-k unfoldings, float64) and their version stamps
 * (network.py:193-200; growth re-layout solver.py:365-367 resets the cache). */
int fctn_set_factors(fctn_ctx* ctx, const double* const* a_unf, const int64_t* versions,
                     int reset_cache);

/* Change the rank table (rank growth, solver.py:361-368); factors must be set
 * afterwards with fctn_set_factors. */
int fctn_set_rank(fctn_ctx* ctx, const int64_t* rank_tri);

/* Device -> host. */
int fctn_get_factors(fctn_ctx* ctx, double* const* a_unf);
int fctn_get_x(fctn_ctx* ctx, void* x_F);  /* context dtype, like fctn_upload */
int fctn_get_x_f64(fctn_ctx* ctx, double* x_F);  /* float64 whatever the context dtype */

/* Closed contexts leave their large device blocks (>= 1 MB) in a process-level
 * cache so the next context of the same extents skips cudaMalloc / cudaFree
 * (the reference has no counterpart: numpy arrays are freed by the garbage
 * collector, solver.py:277-399 allocates per call).  FCTN_DEVCACHE_GB bounds
 * the idle bytes (default 16, 0 disables); this returns them to the driver. */
int fctn_trim_cache(void);

/* f(X, {A_k}) of solver.py:209-224 for the context's current X and factors
 * (full composition; used for the initial objective solver.py:302 and the
 * rank-growth continuity test solver.py:416).  Adds the compose FLOPs of the
 * reference's chain `compose` (network.py:271-278) to counters[FCTN_CT_*]
 * when counters != NULL. */
int fctn_objective(fctn_ctx* ctx, double* out_objective, int64_t* counters);

/* One PAM sweep (solver.py:307-359): N factor updates in `order` (merge of
 * all factors but k with device-resident reuse cache, network.py:426-498;
 * streaming products and exact subproblem solve, sylvester.py:51-116;
 * optional extrapolation, solver.py:240-243,330-331), then compose from the
 * last partial (network.py:313-332) fused with the P_Omega blend
 * (solver.py:227-237) and the reductions.  `extrap`=0 disables extrapolation.
 * `stats`: FCTN_ST_COUNT doubles; `counters`: FCTN_CT_COUNT int64. */
int fctn_sweep(fctn_ctx* ctx, const int32_t* order, int extrap, double alpha, double beta,
               double* stats, int64_t* counters);

/* Shape-only replay (no device needed): the reference FLOP meter and cache
 * hit counters for `n_sweeps` sweeps with the given visiting orders
 * (n_sweeps x n int32), fixed rank.  `counters`: n_sweeps x FCTN_CT_COUNT. */
int fctn_plan_sweeps(int n, const int64_t* dims, const int64_t* rank_tri, int algorithm,
                     int64_t cache_budget, int n_sweeps, const int32_t* orders, int64_t* counters);

/* Multi-GPU (one process per GPU, X and the mask sharded along mode 0,
 * SURVEY.md 8e): an NCCL unique id (128 bytes) made on rank 0 and shared by
 * the caller, then the communicator.  Must be called after fctn_create and
 * before fctn_upload; the slab is the standard partition
 * [rank*I0/nranks, (rank+1)*I0/nranks) and fctn_upload / fctn_get_x then move
 * this rank's slab (extents (hi-lo, I1, ...)).  Factors stay replicated.  Per
 * factor update k != 0 the slab's partial Y_k is all-reduced, for k == 0 the
 * slab's rows of Y_0 are all-gathered; per sweep the four sums are
 * all-reduced.  The Gram of M_k needs no exchange (factor Grams are global). */
int fctn_nccl_unique_id(uint8_t* id128);
int fctn_set_comm(fctn_ctx* ctx, const uint8_t* id128, int rank, int nranks, int64_t slab_lo,
                  int64_t slab_hi);

/* The same sharding with host-side collectives (used by the tests to run
 * ranks that share one GPU, exchanging through gloo): allreduce sums n
 * doubles in place; allgather writes nranks*n doubles, rank order. Return 0
 * on success. */
typedef int (*fctn_host_allreduce_fn)(void* user, double* buf, int64_t n);
typedef int (*fctn_host_allgather_fn)(void* user, const double* send, double* recv, int64_t n);
int fctn_set_comm_host(fctn_ctx* ctx, fctn_host_allreduce_fn allreduce, fctn_host_allgather_fn allgather,
                       void* user, int rank, int nranks, int64_t slab_lo, int64_t slab_hi);

/* Per-rank timing model and tests only: the same sharding with device-side
 * loop-back collectives (all-reduce = this rank's own part, all-gather =
 * nranks copies of the local block).  The results are not the global ones;
 * every kernel has the shape it has on a real nranks-GPU run and the sweep is
 * captured and replayed as a CUDA graph exactly as with NCCL, so one GPU can
 * time what a rank does between its collectives. */
int fctn_set_comm_loopback(fctn_ctx* ctx, int rank, int nranks, int64_t slab_lo, int64_t slab_hi);

/* Kernel self-test (tests only): Y = X_(k) M^T for a mode-k view X of
 * extents [P, I, Q] (first fastest) and a p-fastest M (p = P*Q, S rows),
 * through the K2 path the context would use (tcgen05 TF32 when use_tc and
 * dtype is FCTN_F32 and TMA can describe the view, else SIMT).  Host
 * buffers; Y is I x S column-major float64. */
int fctn_selftest_stream(int device, int dtype, int use_tc, int64_t I, int64_t P, int64_t Q, int64_t S,
                         const void* x, const void* m, double* y);

/* Kernel self-test (tests only): the per-frequency solves of K3,
 * (G + mu_w I) a_w = F_w for w < H1 (Re and Im right-hand sides, F stored
 * [w + H1 s]), in place; `reps` timed launches, best ms returned. */
int fctn_selftest_chol(int device, int64_t S, int64_t H1, const double* G, const double* mu, double* Fr, double* Fi,
                       int reps, double* ms_per_launch);
/* Self-test of the eigendecomposition of the factor subproblem
 * (sylvester.py:51-61 `eig_gram`): G (s x s, symmetric PSD, column-major)
 * = V diag(phi) V^T.  V in: the warm-start basis (identity for a cold start),
 * out: the eigenvectors; phi: eigenvalues clamped at 0; `sweeps`: Jacobi
 * sweeps used; best ms over `reps` launches. */
int fctn_selftest_eigh(int device, int64_t S, const double* G, double* V, double* phi, int reps, double* ms_per_launch,
                       int* sweeps);

/* Reconstruction quality (metrics.py:33-105).  The
 * first two modes are the image plane, every trailing-mode combination is a
 * slice (metrics.py:19-23).  `out` (FCTN_Q_COUNT doubles): mean over slices
 * of PSNR with the 100 dB zero-error cap (metrics.py:33-44); mean over slices
 * of the single-window structural index (metrics.py:47-66); the squared
 * norms behind rel_err (metrics.py:66-92) over all entries and over the mask
 * complement, and the complement's size.  The caller forms rel_err =
 * sqrt(ERR_SQ/REF_SQ) and applies the reference's errors (zero denominator
 * -> ValueError; empty complement -> nan).  Status 1 for n < 2 or peak <= 0
 * (metrics.py:20-21,35-36,50-51). */
#define FCTN_Q_PSNR 0
#define FCTN_Q_SSIM 1
#define FCTN_Q_ERR_SQ 2       /* ||est - truth||^2 */
#define FCTN_Q_REF_SQ 3       /* ||truth||^2 */
#define FCTN_Q_OFF_ERR_SQ 4   /* ||(est - truth) off the mask||^2 */
#define FCTN_Q_OFF_REF_SQ 5   /* ||truth off the mask||^2 */
#define FCTN_Q_OFF_COUNT 6    /* entries off the mask */
#define FCTN_Q_COUNT 8

/* Host tensors est / truth (same shape, `dtype`), optional mask (NULL: no
 * off-mask terms; one byte per entry, nonzero = observed).  Replaces
 * metrics.quality_report + rel_err(mask=) (metrics.py:66-105; cli.py:207-219). */
int fctn_quality(int device, int dtype, int n, const int64_t* dims, const void* est_F, const void* truth_F,
                 const uint8_t* mask_F, double peak, double* out);

/* The same for the context's resident X (no download): truth is a host
 * tensor in `truth_dtype` (this rank's slab when sharded; the per-slice sums
 * are all-reduced over ranks); mask_mode 1 uses the observation mask, 0 none. */
int fctn_quality_ctx(fctn_ctx* ctx, const void* truth_F, int truth_dtype, int mask_mode, double peak, double* out);

/* Sync the context stream. */
int fctn_sync(fctn_ctx* ctx);

/* Device timer on the context stream: op 0 records the start event, op 1
 * records the stop event, synchronises and writes the elapsed ms. */
int fctn_timer(fctn_ctx* ctx, int op, double* ms);

/* Per-kernel-class profiling with CUDA events on the launching stream.
 * Classes: FCTN_K_* below.  When on, every launch group is bracketed by
 * events; fctn_get_profile returns accumulated ms, launch counts and the
 * algorithmic bytes per class since the last reset. */
#define FCTN_K_MERGE 0    /* K1 contraction (partials, M_k) */
#define FCTN_K_STREAM_Y 1 /* K2 X_(k) M_k^T */
#define FCTN_K_GRAM 2     /* K2 M_k M_k^T */
#define FCTN_K_REDUCE 3   /* split-K reductions */
#define FCTN_K_SOLVE 4    /* K3 per-frequency Cholesky solves */
#define FCTN_K_COMPOSE 5  /* K4 compose + blend + reductions */
#define FCTN_K_DFT 6      /* K3 forward / inverse DFT along mode k (+ factor write, stats) */
#define FCTN_K_FGRAM 7    /* K3 factor Gram E_k = A_(k)^T A_(k) + stats fold */
#define FCTN_K_ZPASS 8    /* N=3 schedule: Z_0 = X x_0 A_(0) (tensor-core pass over X) */
#define FCTN_K_YSMALL 9   /* N=3 schedule: Y_k = Z_0 (*) A_(l) (small contraction) */
#define FCTN_K_MBUILD 10  /* M_k built outside the reference chain (compose operand) */
#define FCTN_K_EIGH 11    /* K3 eigendecomposition of G_k (side stream, overlaps the Y_k pass) */
#define FCTN_K_COUNT 12
int fctn_set_profiling(fctn_ctx* ctx, int on);
int fctn_get_profile(fctn_ctx* ctx, double* ms, int64_t* launches, double* bytes);

const char* fctn_last_error(fctn_ctx* ctx);
const char* fctn_version(void);
void fctn_destroy(fctn_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* FCTN_B200_H */
