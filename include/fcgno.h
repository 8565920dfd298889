/*
 * fcgno.h — C ABI of the B200-native batched FCG-NO solver (libfcgno.so).
 *
 * The library solves B independent systems A_b u_b = f_b, the 5-point finite-difference
 * discretisation of -div(k grad u) = f on (0,1)^2 with u = 0 on the boundary
 * (§2.1 Eq. 1-2), by Flexible Conjugate Gradients FCG(m) (PAPER.md:96-112,
 * Algorithm 1) preconditioned at every iteration by a spectral neural operator (SNO, Fourier
 * basis; §2.4.2 and PAPER.md:530 App. A) or by the identity.
 *
 * Conventions shared by every call
 *   - Grid: n interior nodes per dimension, h = 1/(n+1); a system is stored row-major as
 *     [n][n] with row index i <-> x2 and column index j <-> x1; a batch is [B][n][n],
 *     contiguous, system-major (element (b,i,j) at offset (b*n+i)*n+j).  fp64 throughout
 *     unless stated.
 *   - Pointers are DEVICE pointers unless marked [host].  The caller (e.g. PyTorch) owns
 *     all device memory: inputs, outputs, packed weights and workspaces.  The library never
 *     allocates device memory; it owns only the small host-side fcgno_problem descriptor.
 *   - `stream` is a cudaStream_t passed as void*.  Calls enqueue work on it.  Calls that
 *     must report data-dependent errors synchronise it (documented per call).
 *   - Return value: FCGNO_OK (0) or an fcgno_error code; fcgno_last_error() returns a
 *     thread-local message for the last non-OK return.  The library never aborts.
 *   - Numerical failures of one system (breakdown, non-finite preconditioner output) are
 *     reported per system in status[] and never abort the batch.
 *   - Workspaces must be 256-byte aligned and at least the size the *_workspace_bytes
 *     query returns, else FCGNO_EWORKSPACE.
 */
#ifndef FCGNO_H
#define FCGNO_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FCGNO_API __attribute__((visibility("default")))
#else
#define FCGNO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define FCGNO_ABI_VERSION 9
#define FCGNO_K_MODES 20   /* modes per dimension, "number of orthogonal polynomials is 20" */
#define FCGNO_LAYERS 4     /* PAPER.md:530 "Number of SNO layers is 4" */
#define FCGNO_MMAX 64      /* largest truncation parameter m accepted by fcgno_fcg_solve */
#define FCGNO_NO_NMAX 512  /* largest grid n accepted by the NO kernels */

typedef enum {
  FCGNO_OK = 0,
  FCGNO_EINVAL = 1,       /* bad shape, option or NULL pointer */
  FCGNO_ENONPOS_K = 2,    /* some k <= 0 or non-finite (SPEC.md:71 NonPositiveCoefficient) */
  FCGNO_ECUDA = 3,        /* a CUDA runtime error; message in fcgno_last_error() */
  FCGNO_EWORKSPACE = 4,   /* workspace too small or misaligned */
  FCGNO_EUNSUPPORTED = 5  /* e.g. NO with n < 20 or n > FCGNO_NO_NMAX, or no sm_100 device */
} fcgno_error;

/* Per-system solve status (int32 array [B] written by fcgno_fcg_solve). */
typedef enum {
  FCGNO_SYS_RUNNING = 0,
  FCGNO_SYS_CONVERGED = 1,  /* ||r_i||/||r_0|| <= tol at i = iters */
  FCGNO_SYS_MAXIT = 2,      /* iters == maxit without convergence */
  FCGNO_SYS_BREAKDOWN = 3,  /* (p_i, s_i) <= 0 or non-finite */
  FCGNO_SYS_NONFINITE = 4   /* preconditioner output non-finite */
} fcgno_sys_status;

typedef enum { FCGNO_FP32 = 0, FCGNO_FP64 = 1 } fcgno_precision;
typedef enum { FCGNO_SCHEDULE_PAPER = 0, FCGNO_SCHEDULE_SLIDING = 1 } fcgno_schedule;

typedef struct {
  int32_t n;      /* interior nodes per dimension, n >= 2 */
  int32_t batch;  /* number of independent systems B >= 1 */
} fcgno_grid;

/* Spectral neural operator: 2 input channels [r/||r||, k], width w, 4 Fourier
 * layers with FCGNO_K_MODES^2 modes {-10..9}^2, GELU after layers 1-3, 1 output channel.
 * Canonical fp64 weight blob (the layout fcgno_no_pack reads, [host]):
 *   E[w][2], bE[w],
 *   for l = 1..4: W_l[w_out][w_in], b_l[w], R_l[w_in][w_out][20][20][2 (re,im)],
 *   D[w], bD                                  total 3w + 4(w^2 + w + 800 w^2) + w + 1 doubles. */
/* SNO basis: FCGNO_BASIS_FOURIER, the paper's (App. A): the truncated 2-D
 * DFT on the modes {-10..9}^2 (R7-R8); FCGNO_BASIS_CHEBYSHEV: 20 Chebyshev polynomials per
 * dimension, T_k at the Gauss-Chebyshev nodes, i.e. the DCT-II pair (analysis D^-1 S^T, synthesis S) on
 * the index grid, with real mode-diagonal mixing (the blob's real parts of R; R25). */
typedef enum { FCGNO_BASIS_FOURIER = 0, FCGNO_BASIS_CHEBYSHEV = 1 } fcgno_basis;

typedef struct {
  int32_t width;      /* w >= 1 (32 / 48 / 85 in the paper's Table 5) */
  int32_t precision;  /* FCGNO_FP32 (production) or FCGNO_FP64 (trajectory-parity mode) */
  int32_t use_gelu;   /* 1; 0 = test-only linear mode */
  int32_t basis;      /* fcgno_basis */
} fcgno_no_desc;

typedef struct {
  int32_t m;            /* truncation parameter m_max, 1 <= m <= FCGNO_MMAX */
  int32_t maxit;        /* iteration cap >= 0 */
  double tol;           /* stop at the first i with ||r_i||/||r_0|| <= tol */
  int32_t schedule;     /* FCGNO_SCHEDULE_PAPER: m_i = min(i, max(1, i mod (m+1)));
                           FCGNO_SCHEDULE_SLIDING: m_i = min(i, m) */
  int32_t check_every;  /* iterations per replay of the captured loop body (0 = default 16): the
                           solve is one CUDA graph whose WHILE node replays the body while a system
                           is running (a condition kernel ends every body); work on converged
                           systems stops immediately regardless, this only bounds idle tail
                           launches.  With profiling or batch lanes the body is replayed from a
                           host loop that polls the running count per replay instead. */
  int32_t profile_mask; /* bit c set: time the launches of kernel class c (fcgno_prof_class) in the
                           first unrolled iteration of every graph chunk (one sampled iteration
                           per check_every) with CUDA events recorded inside the solve's graphs;
                           0 = no instrumentation */
  int32_t vec_fp32;     /* 0: r, w and the (p_k, s_k) ring in fp64 (default).  1: stored in fp32
                           (BASELINE configs[2] "fp32 or fp64 FCG variants"; R21): every
                           vector operation is computed in fp64 from the stored values and rounded
                           once when stored; u, the inner products (correctly rounded) and the
                           scalars stay fp64. */
} fcgno_solve_opts;

/* Kernel classes for in-graph CUDA-event profiling (diagnostics; bench.py). */
typedef enum {
  FCGNO_PROF_NO_LAYER = 0,   /* k_no_layer / k_tc_layer: SNO layers 1-3 (the dominant kernel) */
  FCGNO_PROF_NO_MIX = 1,     /* k_mix: mode-diagonal channel mixing (layers 2-4) */
  FCGNO_PROF_NO_OUT = 2,     /* k_no_out: layer 4 + projection + window dots */
  FCGNO_PROF_NO_INPUT = 3,   /* k_dft_rows + k_lift_mix: DFT of r/||r|| and layer-1 mixing */
  FCGNO_PROF_WINDOW = 4,     /* k_window_dots (identity / classical preconditioners, and the NO for wide batches) */
  FCGNO_PROF_PFORM = 5,      /* unused since ABI 2 (p is formed inside k_pform_stencil) */
  FCGNO_PROF_STENCIL = 6,    /* k_pform_stencil: lazy u += alpha p, p = w - sum beta p, s = A p, (p,s), (p,r); one launch
                                per iteration */
  FCGNO_PROF_UPDATE = 7,     /* k_update: r update, (r,r), convergence bookkeeping (u is updated lazily) */
  FCGNO_PROF_FINALIZE = 8,   /* unused since ABI 2 (folded into k_update) */
  FCGNO_PROF_NO_YDIR = 9,    /* k_yan + k_ysyn: y-direction DFTs of the tensor-core NO path */
  FCGNO_PROF_NCLASS = 10
} fcgno_prof_class;

typedef struct fcgno_problem fcgno_problem;

/* ---------------------------------------------------------------------------------------
 * assemble(k) — PAPER.md:78-82 (Eq. 2).  Validates k (> 0 and finite, else FCGNO_ENONPOS_K),
 * precomputes the DFT twiddle tables for n and the NO mode coefficients DFT_M(k) of every
 * system.  The stencil itself is matrix-free: face coefficients are harmonic means
 * H(a,b) = (2ab)/(a+b) of nodal k (BASELINE north_star), recomputed on chip.
 *   k   [B][n][n] fp64 device; must stay alive and unchanged while the problem is used.
 *   ws  device workspace of fcgno_problem_workspace_bytes(g) bytes; owned by the problem
 *       until fcgno_problem_destroy.
 * Synchronises `stream` once (to report FCGNO_ENONPOS_K).  *out receives a host handle. */
FCGNO_API size_t fcgno_problem_workspace_bytes(fcgno_grid g);
FCGNO_API int fcgno_assemble(fcgno_grid g, const double* k, void* ws, size_t ws_bytes, void* stream,
                   fcgno_problem** out);
FCGNO_API void fcgno_problem_destroy(fcgno_problem* p);

/* apply_A — y = A x for every system ("s_i <- A p_i").
 *   x, y [B][n][n] fp64 device, y != x.  Canonical op order (R5): d=(kW+kE)+(kS+kN);
 *   t=d*x; t-=kW*xW; t-=kE*xE; t-=kS*xS; t-=kN*xN; y=t*(n+1)^2, no fused multiply-add. */
FCGNO_API int fcgno_apply_A(const fcgno_problem* p, const double* x, double* y, void* stream);

/* Batched inner products out[b] = (x_b, y_b), correctly rounded in all but astronomically
 * rare ties (exact products, double-double accumulation; R6).
 *   x, y [B][n][n] fp64; out [B] fp64 device; ws of fcgno_dot_workspace_bytes(g) bytes. */
FCGNO_API size_t fcgno_dot_workspace_bytes(fcgno_grid g);
FCGNO_API int fcgno_batched_dot(const fcgno_problem* p, const double* x, const double* y, double* out,
                      void* ws, size_t ws_bytes, void* stream);

/* NO weights: fold and convert the canonical fp64 blob [host] into the device layout the
 * kernels read (lift folded into layer 1, layer 4 folded into the projection).
 * `packed` is caller-owned device memory of fcgno_no_packed_bytes(d) bytes.  Synchronises
 * `stream` before returning (the host staging buffer is then released). */
FCGNO_API size_t fcgno_no_packed_bytes(fcgno_no_desc d);
FCGNO_API int fcgno_no_pack(fcgno_no_desc d, const double* weights_host, void* packed, void* stream);

/* 1 when fcgno_apply_NO / fcgno_fcg_solve run the NO operator layers of grid g on the tcgen05 tensor
 * cores (fp32 NO, supported n and w, an sm_100 device present), 0 for the FFMA kernels.  Diagnostics. */
FCGNO_API int fcgno_no_uses_tensor_cores(fcgno_grid g, fcgno_no_desc d);

/* apply_NO(weights, r, k) — w_b = ||r_b|| * NO([r_b/||r_b||, k_b]) for every system, w_b = 0
 * when r_b = 0 ("w_i <- B(r_i)").
 *   r, w [B][n][n] fp64 device (w != r); requires 20 <= n <= FCGNO_NO_NMAX.
 *   ws of fcgno_apply_no_workspace_bytes(g, d) bytes. */
FCGNO_API size_t fcgno_apply_no_workspace_bytes(fcgno_grid g, fcgno_no_desc d);
FCGNO_API int fcgno_apply_NO(const fcgno_problem* p, fcgno_no_desc d, const void* packed, const double* r,
                   double* w, void* ws, size_t ws_bytes, void* stream);

/* fcg_solve(k, f, m, tol, maxit) — Algorithm 1 on every system, with
 * w_i = NO(r_i) (d_or_null != NULL) or w_i = r_i (identity preconditioner, d_or_null == NULL).
 *   f        [B][n][n] fp64 device right-hand sides.
 *   u        [B][n][n] fp64 device: in = initial guess u0, out = final iterate.
 *   iters    [B] int32 device: first i with ||r_i||/||r_0|| <= tol (0 if r_0 = 0), else the
 *            iteration at which the system stopped (maxit, or i of a breakdown).
 *   status   [B] int32 device: fcgno_sys_status.
 *   history  [B][maxit+1] fp64 device or NULL: history[b][i] = ||r_i||/||r_0|| for
 *            i <= iters[b] (entries beyond are left untouched).
 *   ws       fcgno_solve_workspace_bytes(g, d_or_null, o) bytes.
 * Converged systems are frozen (no further writes).  The iteration loop runs on the device (a
 * CUDA-graph WHILE node on an on-device "systems running" counter); instantiated graphs are reused
 * by later solves with identical arguments.  Identity solves of small systems (n^2 <= 1024, fp64
 * vectors, ring fitting shared memory) run as one persistent kernel, one CTA per system, with the same
 * arithmetic.  Synchronises `stream` before returning (iteration count, final lazy x update). */
FCGNO_API size_t fcgno_solve_workspace_bytes(fcgno_grid g, const fcgno_no_desc* d_or_null, fcgno_solve_opts o);
FCGNO_API int fcgno_fcg_solve(const fcgno_problem* p, const fcgno_no_desc* d_or_null, const void* packed,
                    const double* f, double* u, fcgno_solve_opts o, int32_t* iters,
                    int32_t* status, double* history, void* ws, size_t ws_bytes, void* stream);

/* fcg_solve with Theorem-1 diagnostics (Theorem 1, Eq. final_loss; SURVEY
 * §8(f) NEXT-2): as fcgno_fcg_solve, and at every iteration i < iters[b] of a running system, after
 * w_i = B(r_i), with e_i = u_star - u_i (u_i the iterate; u_star a caller-supplied reference solution,
 * e.g. a tight FCG(I) solve, so that e_i approximates A^{-1} r_i):
 *   eps  [B][maxit] device or NULL: eps[b][i]   = ||w_i - e_i||_A / ||e_i||_A  (direct form)
 *   err_a[B][maxit] device or NULL: err_a[b][i] = ||e_i||_A
 * (at least one of them non-NULL).  Adds a state kernel, two stencil applications, two correctly
 * rounded inner products and a scalar kernel per iteration.  profile_mask must be 0.
 *   u_star   [B][n][n] fp64 device.  ws: fcgno_solve_diag_workspace_bytes(g, d_or_null, o) bytes. */
FCGNO_API size_t fcgno_solve_diag_workspace_bytes(fcgno_grid g, const fcgno_no_desc* d_or_null, fcgno_solve_opts o);
FCGNO_API int fcgno_fcg_solve_diag(const fcgno_problem* p, const fcgno_no_desc* d_or_null, const void* packed,
                         const double* f, double* u, fcgno_solve_opts o, int32_t* iters, int32_t* status,
                         double* history, const double* u_star, double* eps, double* err_a, void* ws,
                         size_t ws_bytes, void* stream);

/* Notay ratio of one preconditioner application (PAPER.md Eq. final_loss), per system:
 *   eps[b] = || c B(r_b) - e_b ||_A / || e_b ||_A,   ||v||_A = sqrt((v, A v)),
 * B the NO (d_or_null != NULL) or the identity, e = A^{-1} r supplied by the caller, c = 1, or with
 * optimal_scale != 0 the minimiser c* = (B(r), A e) / (B(r), A B(r)) (FCG's iterates do not depend on
 * the scale of B).  Direct form: d = c B(r) - e is formed first, then ||d||_A and ||e||_A, each from
 * one stencil application and one correctly rounded inner product (R6), in the order of
 * oracle/notay.py.
 *   r, e [B][n][n] fp64 device; eps [B] fp64 device; ws: fcgno_notay_workspace_bytes(g, d_or_null). */
FCGNO_API size_t fcgno_notay_workspace_bytes(fcgno_grid g, const fcgno_no_desc* d_or_null);
FCGNO_API int fcgno_notay_ratio(const fcgno_problem* p, const fcgno_no_desc* d_or_null, const void* packed,
                      const double* r, const double* e, int optimal_scale, double* eps, void* ws,
                      size_t ws_bytes, void* stream);

/* Classical stationary preconditioners of the paper's comparison (§3.3.1): k sweeps
 * from x^0 = 0 with b = r of
 *   FCGNO_PRECOND_JACOBI   Jacobi, Eq. 15: x <- x + D(A)^{-1} (r - A x)
 *   FCGNO_PRECOND_SGS_RB   symmetric Gauss-Seidel, x <- x + L(A)^{-1} (r - A x), x <- x + U(A)^{-1} (r - A x),
 *                          with L, U the triangular parts of A in red-black node order (colour (i + j) mod 2,
 *                          red first; R22): each triangular solve is two colour half sweeps
 * every update x_e <- x_e + (r_e - (A x)_e) / a_ee in the canonical stencil order (R23), fp64.
 *   sweeps 1..64.  fcgno_apply_stationary: w = B(r) for every system (r, w [B][n][n] fp64 device,
 *   w != r; ws of fcgno_stationary_workspace_bytes(g) bytes).  fcgno_fcg_solve_stationary:
 *   Algorithm 1 with w_i = B(r_i); arguments as fcgno_fcg_solve. */
typedef enum { FCGNO_PRECOND_JACOBI = 1, FCGNO_PRECOND_SGS_RB = 2 } fcgno_precond_kind;
FCGNO_API size_t fcgno_stationary_workspace_bytes(fcgno_grid g);
FCGNO_API int fcgno_apply_stationary(const fcgno_problem* p, int kind, int sweeps, const double* r, double* w, void* ws,
                           size_t ws_bytes, void* stream);
FCGNO_API size_t fcgno_solve_stationary_workspace_bytes(fcgno_grid g, fcgno_solve_opts o);
FCGNO_API int fcgno_fcg_solve_stationary(const fcgno_problem* p, int kind, int sweeps, const double* f, double* u,
                               fcgno_solve_opts o, int32_t* iters, int32_t* status, double* history, void* ws,
                               size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------
 * Training the SNO on the GPU (§2.5, §3.1-3.2,
 * Table 6).  The scheme of Fig. 3: FCG with B = I on the training systems
 * (fcgno_fcg_solve with maxit = i gives the CG iterate u_i), training pairs (r_i, e_i) with
 * e_i = u_exact - u_i = A^{-1} r_i (fcgno_krylov_pair), then minibatch steps of
 *   L(theta) = mean_b ||B(r_b; theta) - e_b||_A / ||e_b||_A     (Notay loss, error form)
 *              or mean_b ||B(r_b; theta) - e_b||_2 / ||e_b||_2  (L2 form)
 * with B(r) = ||r|| NO([r/||r||, k]) exactly as fcgno_apply_NO defines it (fp32 forward, fp64 loss), the
 * gradient by the chain rule through projection, the four layers and the lift (oracle/train.py), and
 * AdamW (decoupled weight decay, R26).
 * Weights are fp32 in the canonical blob order of fcgno_no_desc (E, bE, 4 x (W, b, R), D, bD);
 * fcgno_train_param_count(w) elements.  Samples: k, r, e [S][n][n] fp64 device; the minibatch is
 * samples perm[0..count-1] (int32 device; NULL = 0..count-1), whose coefficient field is
 * k[ksys[sample]] (int32 device [S]; NULL = k[sample]).  Deterministic (fixed-order reductions). */
typedef enum { FCGNO_LOSS_NOTAY = 0, FCGNO_LOSS_L2 = 1 } fcgno_loss_kind;
typedef struct {
  int32_t n;      /* grid, 20 <= n <= 256 */
  int32_t width;  /* w, 1..128 */
  int32_t batch;  /* minibatch capacity (N_batch of Table 6), batch * n <= 65535 */
  int32_t loss;   /* fcgno_loss_kind */
} fcgno_train_desc;
typedef struct {
  double lr, beta1, beta2, eps, weight_decay;   /* Table 6: lr 1e-3 (x0.5 / 50 epochs), wd 1e-2 */
} fcgno_adamw_opts;
FCGNO_API size_t fcgno_train_param_count(int32_t width);
FCGNO_API size_t fcgno_train_workspace_bytes(fcgno_train_desc d);
/* Forward + loss of `count` <= batch samples: loss[b] (fp64 device [count], or NULL) = the sample's
 * ratio; with grad != NULL also grad [P] fp32 device = d(mean_b loss_b)/d(theta) (overwritten).
 * Enqueues on `stream`, no synchronisation. */
FCGNO_API int fcgno_train_loss_grad(fcgno_train_desc d, int32_t count, const float* params, const double* k,
                                    const double* r, const double* e, const int32_t* perm, const int32_t* ksys,
                                    double* loss, float* grad, void* ws, size_t ws_bytes, void* stream);
/* AdamW step t >= 1 on `count` fp32 parameters (params, m, v updated in place; m = v = 0 before t = 1):
 * theta <- theta (1 - lr wd); m <- b1 m + (1-b1) g; v <- b2 v + (1-b2) g^2;
 * theta <- theta - lr/(1-b1^t) m / (sqrt(v)/sqrt(1-b2^t) + eps). */
FCGNO_API int fcgno_adamw_step(size_t count, float* params, const float* grad, float* m, float* v, int32_t t,
                               fcgno_adamw_opts o, void* stream);
/* One epoch: minibatches perm[s0 .. s0+batch-1] for s0 = 0, batch, ... < nsamples (the last one may be
 * smaller), each a fcgno_train_loss_grad into grad [P] followed by an AdamW step with t = ++*t_host
 * ([host] in/out).  loss [nsamples] device or NULL: loss[j] of sample perm[j] before its step. */
FCGNO_API int fcgno_train_epoch(fcgno_train_desc d, int32_t nsamples, float* params, float* grad, float* m,
                                float* v, int32_t* t_host, fcgno_adamw_opts o, const double* k, const double* r,
                                const double* e, const int32_t* perm, const int32_t* ksys, double* loss, void* ws,
                                size_t ws_bytes, void* stream);
/* Krylov training pair (Eq. 8-9) of every system of the problem:
 * r = f - A u (u the CG iterate u_i), e = e_scale (u_star - u) (u_star = u_exact, e.g. a tight FCG(I)
 * solve); fp64 [B][n][n] device, outputs must not alias inputs.  e_scale > 0 is the unit of the target
 * (R27: 1 = A^{-1} r as printed; (n+1)^2 = the error in units of the unscaled stencil
 * h^2 A, which keeps the trained output weights O(1); FCG is invariant to a positive scaling of B).
 * Bitwise the oracle's arithmetic (R5).  FCGNO_EINVAL for e_scale <= 0 or non-finite. */
FCGNO_API int fcgno_krylov_pair(const fcgno_problem* p, const double* f, const double* u_star, const double* u,
                                double e_scale, double* r, double* e, void* stream);

/* End-to-end convenience entry point with HOST buffers ([host], pageable or pinned): copies
 * k, f, u0 to the device, assembles, solves and copies u, iters, status (and history if
 * non-NULL) back.  `dev_ws` is a device workspace of fcgno_solve_host_workspace_bytes bytes;
 * `packed` as for fcgno_fcg_solve (already resident).  Synchronises `stream`. */
FCGNO_API size_t fcgno_solve_host_workspace_bytes(fcgno_grid g, const fcgno_no_desc* d_or_null,
                                        fcgno_solve_opts o);
FCGNO_API int fcgno_solve_host(fcgno_grid g, const double* k_host, const double* f_host, double* u_host,
                     const fcgno_no_desc* d_or_null, const void* packed, fcgno_solve_opts o,
                     int32_t* iters_host, int32_t* status_host, double* history_host,
                     void* dev_ws, size_t ws_bytes, void* stream);

/* Accumulated profile of kernel class `cls` since the last reset: total device milliseconds and
 * number of timed launches (host pointers).  Returns FCGNO_EINVAL for a bad class. */
FCGNO_API int fcgno_profile_get(int cls, double* total_ms, int64_t* launches);
FCGNO_API void fcgno_profile_reset(void);
FCGNO_API const char* fcgno_profile_name(int cls);

/* Diagnostics: the clock64 stamps of the tensor-core layer pipeline events of CTA 0's first 64 tiles
 * of the last layer launch selected by FCGNO_PX_TRACE=<layer 1..3> ([tile][10] uint64, host). */
FCGNO_API int fcgno_debug_px_trace(uint64_t* host, int count);

/* Number of kernel launches the library issued in this process (diagnostics, bench.py). */
FCGNO_API uint64_t fcgno_kernel_launches(void);
FCGNO_API const char* fcgno_last_error(void);
FCGNO_API int fcgno_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FCGNO_H */
