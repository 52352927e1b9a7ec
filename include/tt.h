/*
 * tt.h — C ABI of libtt, the B200 (sm_100a) hot path of arXiv 2309.03347:
 * "Tensor Networks for Solving Realistic Time-independent Boltzmann Neutron
 * Transport Equation".  Passages are cited as P:<lines> of PAPER.md and the
 * readings Z<n> of SURVEY.md §8(c).3 (restated in DESIGN.md).
 *
 * Conventions
 *   - Everything is fp64.  All `double *` arguments are DEVICE pointers; shape
 *     arrays (`n`, `m`, `rcap`, `off`) are HOST pointers; `*_dev` are device.
 *   - TT-vector core k (0-based) is [r_k, n_k, r_{k+1}] column-major (first index
 *     fastest) stored compactly at data + off[k]; its slot holds
 *     rcap[k] * n_k * rcap[k+1] doubles, so ranks may change on the device
 *     without reallocation.  r_dev[0] = r_dev[d] = 1.
 *   - TT-matrix core k is [R_k, m_k, n_k, R_{k+1}] column-major; (i, j) =
 *     (row/output, column/input) index (Z27).  A TT-matrix viewed as
 *     a TT-vector has mode m_k n_k with the row index fastest.
 *   - Full-tensor linearisation: first core fastest (Z28).
 *   - Ranks live on the device (int32).  The library never allocates device
 *     memory and never frees; scratch is the caller's `ws` of `wsb` bytes,
 *     sized by the tt_*_workspace functions.  Every call is asynchronous and
 *     stream-ordered on `s`; buffers must outlive stream completion.
 *   - The returned tt_status covers host-detectable errors (argument, shape,
 *     capacity at the declared capacities, launch failures).  Conditions found
 *     on the device (non-convergence, NaN, no fission) are written to the
 *     caller's status word (keff_report.status_dev) and are readable after a
 *     stream synchronisation.  tt_last_error() describes the last host error
 *     of the calling thread.  There is no CPU fallback: an unavailable path
 *     returns TT_ERR_NOT_IMPLEMENTED.
 *   - Reentrant for distinct `ws` buffers and streams.
 */
#ifndef TT_B200_H
#define TT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TT_OK = 0,
  TT_ERR_ARG = 1,        /* invalid argument (NULL, d < 1, r_0 != 1, bad option)       */
  TT_ERR_SHAPE = 2,      /* mode sizes disagree ("shape mismatch")                  */
  TT_ERR_CAPACITY = 3,   /* an output rank capacity or the workspace is too small         */
  TT_ERR_NOCONV = 4,     /* (device status) iteration budget exhausted; history written   */
  TT_ERR_NOFISSION = 5,  /* (device status) <F^T 1, Psi> = 0                               */
  TT_ERR_NUMERIC = 6,    /* (device status) NaN/Inf or singular local system              */
  TT_ERR_CUDA = 7,       /* a CUDA launch failed                                          */
  TT_ERR_NOT_IMPLEMENTED = 8
} tt_status;

typedef void *tt_stream; /* cudaStream_t; NULL = legacy default stream */

#define TT_MAX_D 64      /* maximum number of cores */

/* TT-vector (eqn:TT_def_element P:492-497, eqn:TT-vector P:504-512). */
typedef struct {
  int32_t d;               /* number of cores, 1 <= d <= TT_MAX_D                       */
  const int32_t *n;        /* [d] host: mode sizes                                       */
  int32_t *r_dev;          /* [d+1] device: current ranks                                */
  const int32_t *rcap;     /* [d+1] host: rank capacities (slot sizes), rcap[0]=rcap[d]=1 */
  double *data;            /* device: core storage                                       */
  const int64_t *off;      /* [d] host: element offset of core k's slot                  */
} tt_vec;

/* TT-matrix (eqn:TT-matrix-componentwise P:670-680, eqn:TT-matrix-compact P:686-691). */
typedef struct {
  int32_t d;
  const int32_t *m;        /* [d] host: row (output) mode sizes                          */
  const int32_t *n;        /* [d] host: column (input) mode sizes                        */
  int32_t *R_dev;          /* [d+1] device: current ranks                                */
  const int32_t *Rcap;     /* [d+1] host: rank capacities                                */
  double *data;
  const int64_t *off;
} tt_mat;

const char *tt_last_error(void);
const char *tt_version(void);

/* Device-side algorithmic counters (for measurement; synchronises the device):
 * out[0] flops of the contraction GEMMs (2 M N K per call), out[1] flops of the
 * exact matvec (2 n per output entry), out[2] nominal Householder QR flops
 * (geqrf + orgqr), out[3] Jacobi SVD flops (column dots + rotations),
 * out[4] number of GEMM calls.  reset != 0 zeroes them after reading. */
void tt_counters(uint64_t *out /* [5] */, int32_t reset);

/* Live timing of the fused GMRES Arnoldi-step kernel (the dominant kernel of
 * the k-eff solves; used by bench.py for its roofline line).  enable != 0:
 * every later launch of the kernel by this thread is bracketed by CUDA events
 * on its stream (host-stepped graph modes 0/1; in mode 2 the in-kernel
 * %globaltimer of CTA 0 times each launch that does work).  _read synchronises those events and returns the number of
 * launches, their summed duration (ms) and flops[3] = {local-apply GEMM flops,
 * CGS2/norm vector flops, Arnoldi steps executed} of those launches, then
 * resets (the flop counters count every fused launch since the last read). */
void tt_fused_profile(int32_t enable);
void tt_fused_profile_read(int64_t *launches, double *ms, double *flops /* [3] */);
/* Per-core breakdown of the same recorded launches (AMEn core index k): summed
 * duration ms[k], Arnoldi steps steps[k] and launches[k], arrays of TT_MAX_D.
 * Call before tt_fused_profile_read (which resets). */
void tt_fused_profile_cores(double *ms, double *steps, int64_t *launches);
/* The in-kernel timer alone: summed %globaltimer duration (ms) and number of the
 * fused launches that did work since the last read (either this call or a
 * tt_fused_profile_read that found no events); resets it.  Used to cross-check
 * the timer against CUDA events on the host-stepped path. */
void tt_fused_timer_read(double *ms, int64_t *launches);

/* CUDA-graph execution mode of the drivers (calling thread):
 *   2 (default) device-resident loops: amen_solve, amen_mv, keff_fixed_point and
 *     alpha_secant each run as ONE graph launch whose convergence loops are
 *     conditional WHILE/IF nodes decided on the device (no host round trip
 *     inside the call; one small read-back at entry detects the operator core
 *     structure).  The fused GMRES kernel is then timed by its in-kernel
 *     %globaltimer (tt_fused_profile_read), events cannot bracket it;
 *   1 fixed launch sequences replayed as graphs, loops polled by the host
 *     (one read-back per sweep / outer iteration);
 *   0 no graphs.
 * The environment sets the default (TT_NO_GRAPHS=1 -> 0, TT_NO_DEVLOOP=1 -> 1);
 * mode < 0 restores it.  A capture or instantiation failure is returned as
 * TT_ERR_CUDA, never a silent change of mode.  Graphs are cached under the exact
 * bytes of everything they depend on (operands, workspace, options, report
 * pointers); _stats returns captures, replays and cached graphs so far. */
void tt_set_graph_mode(int32_t mode);
int32_t tt_graph_mode(void);
void tt_graph_stats(int64_t *captures, int64_t *replays, int64_t *cached);

/* ---------------------------------------------------------------- a1 ---
 * tt_matvec: exact TT-matrix x TT-vector product ("explicit and
 * exact algorithm").  For every core, independently,
 *   Y_k[rho, i, rho'] = sum_j A_k[a, i, j, a'] X_k[b, j, b'],
 *   rho = a + R_k b, rho' = a' + R_{k+1} b'  (operator rank fastest).
 * Output ranks R_k r_k are written to y->r_dev.  Requires A->n == x->n,
 * y->n == A->m, y->rcap[k] >= Rcap[k] * x->rcap[k] (else TT_ERR_CAPACITY).
 * No workspace.  y must not alias A or x. */
tt_status tt_matvec(const tt_mat *A, const tt_vec *x, tt_vec *y, tt_stream s);

/* Batched form: B independent products (A[b], x[b]) -> y[b] (same d), one
 * launch over (core, instance); a (core, instance) descriptor table is staged
 * into ws (tt_matvec_batched_workspace bytes). */
size_t tt_matvec_batched_workspace(int32_t B, const tt_mat *A);
tt_status tt_matvec_batched(int32_t B, const tt_mat *A, const tt_vec *x, tt_vec *y, void *ws, size_t wsb,
                            tt_stream s);

/* ---------------------------------------------------------------- a2 ---
 * tt_add: z = alpha x + beta y by block-diagonal core concatenation (sum of
 * TT tensors is a TT tensor): first core [alpha X_1, beta Y_1], last
 * core [X_d; Y_d], middle diag(X_k, Y_k); ranks add.  alpha_dev / beta_dev are
 * device scalars (NULL = 1.0), so k^{-1} of the fixed point never leaves the
 * device.  d = 1: z = alpha x + beta y elementwise.  z must not alias x or y. */
tt_status tt_add(const tt_vec *x, const double *alpha_dev, const tt_vec *y,
                 const double *beta_dev, tt_vec *z, tt_stream s);

/* tt_scale: x <- alpha x (scales the first core), alpha read on the device. */
tt_status tt_scale(tt_vec *x, const double *alpha_dev, tt_stream s);

/* tt_copy: y <- x (ranks and cores); y capacities must hold x's ranks. */
tt_status tt_copy(const tt_vec *x, tt_vec *y, tt_stream s);

/* ---------------------------------------------------------------- a8 ---
 * tt_dot: <x, y> by a left-to-right chain contraction (the "sum F Psi"
 * reductions of eqn:TT_k_eff_fixed_points P:1409 are <F^T 1, Psi>, Z18).
 * Result written to out_dev.  Workspace: tt_dot_workspace(x, y). */
size_t tt_dot_workspace(const tt_vec *x, const tt_vec *y);
tt_status tt_dot(const tt_vec *x, const tt_vec *y, double *out_dev, void *ws, size_t wsb,
                 tt_stream s);

/* ---------------------------------------------------------------- a3 ---
 * tt_orthogonalize (rounding internals unstated in the
 * paper, reading Z21).  dir = -1: right-to-left, for k = d-1..1:
 * Householder QR of the transposed right unfolding (n_k r_{k+1}) x r_k,
 * core k <- Q^T, core k-1 <- core k-1 x_3 R^T, r_k <- min(r_k, n_k r_{k+1}).
 * dir = +1: the left-to-right mirror (QR of the left unfoldings).  In place.
 * norm_dev (may be NULL) receives ||x||_F = ||orthogonality centre||_F.
 * Workspace: tt_orthogonalize_workspace(x). */
size_t tt_orthogonalize_workspace(const tt_vec *x);
/* tt_normalize: x <- x / ||x||_F (right-to-left orthogonalisation, then the first
 * core scaled by the reciprocal of the norm, read on the device); ||x||_F is
 * written to norm_dev (device, [1]).  Workspace: tt_orthogonalize_workspace(x).
 * Used for the per-interface normalisation of reading Z25. */
tt_status tt_normalize(tt_vec *x, double *norm_dev, void *ws, size_t wsb, tt_stream s);
tt_status tt_orthogonalize(tt_vec *x, int32_t dir, double *norm_dev, void *ws, size_t wsb,
                           tt_stream s);

/* ---------------------------------------------------------------- a4 ---
 * tt_round: TT rounding ("rank reduction step"), in place:
 * right-to-left orthogonalisation, delta = eps ||x||_F / sqrt(d-1), then for
 * k = 0..d-2 the SVD of the left unfolding (r_k n_k) x r_{k+1} (Householder QR +
 * one-sided Jacobi on the triangular factor), new rank
 *   r' = min(rmax, smallest r >= 1 with sum_{i>r} sigma_i^2 <= delta^2)   (Z21),
 * core k <- U[:, :r'], core k+1 <- (Sigma V^T)[:r'] x_1 core k+1.
 * discarded_sq_dev (may be NULL) receives the d-1 discarded tail energies;
 * sv_dev (may be NULL) receives, per bond, the singular values (stride
 * sv_stride doubles, zero padded).  Workspace: tt_round_workspace(x). */
size_t tt_round_workspace(const tt_vec *x);
tt_status tt_round(tt_vec *x, double eps, int32_t rmax, double *discarded_sq_dev,
                   double *sv_dev, int32_t sv_stride, void *ws, size_t wsb, tt_stream s);

/* tt_round_batched: tt_round (same rule, Z21) of B independent TT-vectors x[0..B-1]
 * (same number of cores; shapes, ranks and capacities may differ) in place,
 * one launch per step for all instances (BASELINE.json configs[1]: B = 64 C2
 * products).  discarded_sq_dev: [B][d-1] tail energies or NULL.  Errors as
 * tt_round; TT_ERR_SHAPE if the core counts differ.  Workspace:
 * tt_round_batched_workspace(B, x). */
size_t tt_round_batched_workspace(int32_t B, const tt_vec *x);
tt_status tt_round_batched(int32_t B, tt_vec *x, double eps, int32_t rmax, double *discarded_sq_dev,
                           void *ws, size_t wsb, tt_stream s);

/* ------------------------------------------------------------ a5, a6 ---
 * Interfaces and local operator of ALS/AMEn ("fix all but one TT
 * core").  Orientation: Phi[alpha, gamma, beta] with
 * alpha = test rank, gamma = operator rank, beta = trial rank (alpha fastest).
 *
 * als_local_apply:
 *   y[a, i, a'] = sum Phi[a, g, b] A_k[g, i, j, g'] Psi[a', g', b'] x[b, j, b']
 * Phi [rA, R, rB], Ak [R, m, n, Rp], Psi [rAp, Rp, rBp], x [rB, n, rBp] -> y [rA, m, rAp].
 * Evaluated as three FP64 tensor-core (DMMA) GEMMs: x.Psi^T, A_k.(.), Phi.(.).
 * Workspace: als_workspace(...). */
size_t als_workspace(int32_t rA, int32_t R, int32_t rB, int32_t m, int32_t n, int32_t rAp,
                     int32_t Rp, int32_t rBp);
tt_status als_local_apply(int32_t rA, int32_t R, int32_t rB, int32_t m, int32_t n, int32_t rAp,
                          int32_t Rp, int32_t rBp, const double *Phi, const double *Ak,
                          const double *Psi, const double *x, double *y, void *ws, size_t wsb,
                          tt_stream s);

/* als_update_interfaces:
 *   dir = +1 (left):  Phi_k[a', g', b'] = sum Phi_{k-1}[a, g, b] Y_k[a, i, a'] A_k[g, i, j, g'] X_k[b, j, b']
 *   dir = -1 (right): Psi_k[a, g, b]    = sum Psi_{k+1}[a', g', b'] Y_k[a, i, a'] A_k[g, i, j, g'] X_k[b, j, b']
 * Y_k [rY, m, rYp], X_k [rX, n, rXp], A_k [R, m, n, Rp].  With Ak == NULL the
 * vector interface (R = Rp = 1, B_k passed as X_k with n = m):
 *   phi_k[a', b'] = sum phi_{k-1}[a, b] Y_k[a, i, a'] X_k[b, i, b'].
 * Iprev: [rY, R, rX] (left) or [rYp, Rp, rXp] (right); Inext the other.
 * Workspace: als_workspace(rY, R, rX, m, n, rYp, Rp, rXp). */
tt_status als_update_interfaces(int32_t dir, int32_t rY, int32_t R, int32_t rX, int32_t m,
                                int32_t n, int32_t rYp, int32_t Rp, int32_t rXp,
                                const double *Iprev, const double *Yk, const double *Ak,
                                const double *Xk, double *Inext, void *ws, size_t wsb,
                                tt_stream s);

/* Structured operator cores ("the angle core n=288 has an
 * n^2 R^2 stage that grows large unless the diagonal (H) ... angular structure
 * is exploited").  The angle and group factors of H are diagonal, Q_mu =
 * C_b (x) diag(mu) and H_sigma = diag(sigma) o (C_b (x) I)
 * (P:1222-1225), and sums / roundings of such cores keep every slice
 * A_k[g, :, :, g'] diagonal: D_i[g, g'] = A_k[g, i, i, g'].
 *
 * tt_core_kinds: detects, on the device, which cores of A are TT_CORE_DIAG
 * (m == n >= 4 and max|off-diagonal| <= 1e-13 max|A_k|; the rest TT_CORE_DENSE)
 * and returns the kinds (host [d]) and the off-diagonal ratios (host [d] or
 * NULL; -1 for non-square or small cores).  Synchronises the stream once.
 * ws: >= 768 bytes of device workspace.  amen_solve / amen_mv / keff run the
 * same detection internally. */
typedef enum { TT_CORE_DENSE = 0, TT_CORE_DIAG = 1 } tt_core_kind;
tt_status tt_core_kinds(const tt_mat *A, int32_t *kinds, double *offdiag_ratio, void *ws, size_t wsb, tt_stream s);

/* als_local_apply_structured / als_update_interfaces_structured: the a6 / a5
 * contractions of als_local_apply / als_update_interfaces (same arguments and
 * layouts) for a core of the given kind.  TT_CORE_DIAG reads only the
 * diagonal slices of Ak (off-diagonal entries are ignored) and replaces the
 * dense (R m) x (n R') stage by m batched R x R' products: the apply costs
 * 2 m (rB rBp rAp Rp + R Rp rB rAp + rA rAp rB R) flops instead of
 * 2 (n rB rBp rAp Rp + m n rB rAp R Rp + m rA rAp rB R).  absorb = 1 (diagonal
 * cores only; for the interface form only dir = +1) first absorbs the left
 * operator rank into the left interface, Pt_i[a, b, g'] = sum_g Phi[a, g, b]
 * D_i[g, g'], which the AMEn local solve does once per local system:
 *   y[a, i, a'] = sum_{b, g'} Pt_i[a, b, g'] sum_b' x[b, i, b'] Psi[a', g', b'],
 * 2 m (rB rBp rAp Rp + rA rB Rp rAp) flops per apply (the C4 angle core: 1.5
 * GFLOP instead of 105.7 dense).  kind = TT_CORE_DENSE, absorb = 0 is the
 * plain call.  TT_ERR_SHAPE if a diagonal core is not square.  Workspace:
 * als_workspace_structured(...). */
size_t als_workspace_structured(int32_t kind, int32_t absorb, int32_t rA, int32_t R, int32_t rB, int32_t m, int32_t n,
                                int32_t rAp, int32_t Rp, int32_t rBp);
tt_status als_local_apply_structured(int32_t kind, int32_t absorb, int32_t rA, int32_t R, int32_t rB, int32_t m,
                                     int32_t n, int32_t rAp, int32_t Rp, int32_t rBp, const double *Phi,
                                     const double *Ak, const double *Psi, const double *x, double *y, void *ws,
                                     size_t wsb, tt_stream s);
tt_status als_update_interfaces_structured(int32_t kind, int32_t absorb, int32_t dir, int32_t rY, int32_t R,
                                           int32_t rX, int32_t m, int32_t n, int32_t rYp, int32_t Rp, int32_t rXp,
                                           const double *Iprev, const double *Yk, const double *Ak,
                                           const double *Xk, double *Inext, void *ws, size_t wsb, tt_stream s);

/* ---------------------------------------------------------------- a7 ---
 * amen_solve: x ~ A^{-1} b in TT ("amen_solve";
 * reading Z20): alternating-direction sweeps, Galerkin local systems solved by
 * device GMRES(restart) built on als_local_apply, SVD truncation with
 * delta = eps ||x_k|| / sqrt(d-1) capped at rmax, residual TT z (ranks = its
 * initial ranks = kickrank) and enrichment of the solution core with the
 * residual projected on (x frames | z frames).  Stops after a sweep whose
 * maximum local residual (measured before each local solve) is <= eps, or
 * whose maximum relative change of a local solution ||x_k^new - x_k^old|| /
 * ||x_k^new|| is <= eps (the solution-change exit of TT-Toolbox amen_solve).
 * x: in initial guess, out solution (capacities >= rmax + kickrank).
 * z: in initial residual TT (random draws are inputs), workspace afterwards.
 * sweeps_dev / res_dev (may be NULL): sweeps used and final max residual.
 * Workspace: amen_workspace(A, b, x, z). */
typedef struct {
  double eps;              /* stopping tolerance on the local residual            */
  double local_tol;        /* GMRES relative tolerance (<= 0: 0.1 eps)             */
  int32_t max_sweeps;
  int32_t rmax;
  int32_t gmres_restart;   /* Krylov basis size m                                  */
  int32_t gmres_max_restarts;
  int32_t local_dense_max; /* local systems of size <= this are solved densely      */
                           /*    (Gauss-Jordan with partial pivoting; an exactly    */
                           /*    singular system is regularised with mu = 1e-12     */
                           /*    ||B||_F, reading Z35); 0 = GMRES only (default)    */
} amen_opts;
size_t amen_workspace(const tt_mat *A, const tt_vec *b, const tt_vec *x, const tt_vec *z,
                      const amen_opts *o);
tt_status amen_solve(const tt_mat *A, const tt_vec *b, tt_vec *x, tt_vec *z, const amen_opts *o,
                     int32_t *sweeps_dev, double *res_dev, void *ws, size_t wsb, tt_stream s);

/* ------------------------------------------------------------ NEXT-1 ---
 * amen_mv: y ~ A b in TT without forming the rank-R r product (P:1489-1494,
 * P:1505-1506 "amen_mv"; reading Z37): the same alternating sweeps as
 * amen_solve with the local projection y_k = (y|A|b)_{k-1} A_k (y|A|b)_{k+1} b_k
 * in place of the local solve, SVD truncation at delta = eps ||y_k|| / sqrt(d-1)
 * capped at rmax, and enrichment by the projected residual A b - y carried
 * by the residual TT z.  Stops after a sweep whose maximum relative change of
 * a local core is <= eps, or after max_sweeps.  A may be rectangular
 * (A.m = y modes, A.n = b modes).  y: in initial guess (its ranks are kept as
 * the starting frames), out the product (capacities >= rmax + z capacities).
 * z: in initial residual TT (random draws are inputs), workspace afterwards.
 * sweeps_dev (may be NULL): sweeps used.  Workspace: amen_mv_workspace. */
size_t amen_mv_workspace(const tt_mat *A, const tt_vec *b, const tt_vec *y, const tt_vec *z);
tt_status amen_mv(const tt_mat *A, const tt_vec *b, tt_vec *y, tt_vec *z, double eps, int32_t max_sweeps,
                  int32_t rmax, int32_t *sweeps_dev, void *ws, size_t wsb, tt_stream s);

/* ---------------------------------------------------------------- a9 ---
 * keff_fixed_point: eqn:TT_k_eff_fixed_points, readings
 * Z16-Z19:
 *   B = round(round(S Psi) + k^{-1} round(F Psi))  (matvec = 0) or
 *   B = amen_mv(S + k^{-1} F, Psi)                  (matvec = 1, the paper's choice);
 *   H Psi' = B (amen_solve, warm start Psi);  k' = k <f, Psi'> / <f, Psi>,
 *   f = F^T 1;  Psi <- Psi'/||Psi'||.
 * Fixed-point residual (reading Z19): res = ||H Psi - (S + F/k) Psi|| /
 * ||H Psi|| for the normalised iterate and its k, both products by amen_mv to
 * eps_round (M = H - S - k^{-1} F as one TT-matrix, ranks add; capacities of
 * psi), the norms by orthogonalisation.  tol_res > 0: evaluated every
 * iteration and required for convergence; tol_res == 0: evaluated once after
 * the last iteration (reported, not tested); tol_res < 0: never.
 * Converged (status TT_OK) when |k' - k| <= tol_k and (tol_res <= 0 or
 * res <= tol_res); TT_ERR_NOCONV after max_outer iterations (history written).
 * The inner AMEn status of each iteration (TT_OK / TT_ERR_NOCONV: the local
 * residual did not reach eps_solve within max_sweeps, the normal state of a
 * truncation-limited solve) is reported per iteration, not folded into
 * status: the outer residual is the convergence evidence.
 * k, ||Psi||, <f, Psi>, the residual and every rank stay on the device; the
 * host polls one convergence word per outer iteration.  psi: in Psi_0, out the
 * normalised eigenvector (capacities >= rmax + kickrank).  z: AMEn residual TT
 * (random initial cores are an input; its interior ranks are the kickrank).
 * Report arrays are device memory (NULL allowed except k_dev, iters_dev,
 * status_dev).  Workspace: keff_workspace(...). */
typedef struct {
  double tol_k;            /* |k' - k| stopping tolerance                          */
  double tol_res;          /* fixed-point residual tolerance (see above)           */
  double eps_round;        /* rounding / amen_mv tolerance of B and the residual    */
  double eps_solve;        /* AMEn tolerance                                       */
  int32_t max_outer;
  int32_t rmax;
  int32_t max_sweeps;
  int32_t kickrank;        /* 0: the interior rank capacity of z; > 0: must equal it */
  int32_t gmres_restart;
  int32_t gmres_max_restarts;
  int32_t local_dense_max; /* local systems of size <= this are solved densely (*/
                           /*    Z20/Z35; see amen_opts); 0 = GMRES only             */
  int32_t matvec;          /* 0: B by exact products + rounding; 1: B = amen_mv(S +  */
                           /*    k^{-1} F, Psi) to eps_round,          */
                           /*    warm-started from the previous B                    */
  int32_t mv_max_sweeps;   /* amen_mv sweep limit (B and the residual products)      */
  int32_t warm;            /* 1: continue a previous call (same operators, options   */
                           /*    and workspace): psi is that call's normalised       */
                           /*    iterate (not re-rounded), the amen_mv guess of B,   */
                           /*    the AMEn residual start cores z0 and f = F^T 1 are  */
                           /*    kept in the workspace, k0 is its k; 0: fresh start   */
} keff_opts;
typedef struct {
  double *k_dev;           /* [1] final k                                          */
  int32_t *iters_dev;      /* [1] outer iterations performed                       */
  double *k_hist_dev;      /* [hist_cap] k after each outer iteration              */
  double *res_hist_dev;    /* [hist_cap] fixed-point residual per iteration (-1    */
                           /*    where not evaluated)                              */
  int32_t hist_cap;
  int32_t *status_dev;     /* [1] TT_OK / TT_ERR_NOCONV / TT_ERR_NOFISSION / ...   */
  int32_t *sweeps_hist_dev;/* [hist_cap] AMEn sweeps per outer iteration           */
  int32_t *inner_status_hist_dev; /* [hist_cap] AMEn status per outer iteration    */
  double *res_dev;         /* [1] last evaluated residual (-1 if none)             */
} keff_report;
size_t keff_workspace(const tt_mat *H, const tt_mat *S, const tt_mat *F, const tt_vec *psi,
                      const tt_vec *z, const keff_opts *o);
tt_status keff_fixed_point(const tt_mat *H, const tt_mat *S, const tt_mat *F, tt_vec *psi,
                           tt_vec *z, double k0, const keff_opts *o, keff_report *rep, void *ws,
                           size_t wsb, tt_stream s);

/* ------------------------------------------------------------ NEXT-2 ---
 * alpha_secant: the alpha eigenvalue of [alpha V^{-1} + H] Psi = [S + F] Psi
 * (eq. OpFormAlphaNTE; TT scheme P:1416-1462).  alpha^(0) = alpha0,
 * alpha^(1) = alpha1 (the paper: 0 and 0.01); for each alpha the
 * k-eff problem [alpha V^{-1} + H] Psi = [S + F/k] Psi is solved by the
 * keff_fixed_point machinery on H_alpha = round(H + alpha V^{-1}, eps_op),
 * warm-started from the previous Psi and k; then the secant step on
 * k(alpha) - 1 (reading Z32; the printed update is dimensionally
 * inconsistent):  alpha+ = alpha + (1 - k)(alpha - alpha_prev)/(k - k_prev).
 * Stops when |k(alpha) - 1| <= tol.  alpha, k and the secant state stay on
 * the device; the host polls one flag per k-eff solve.
 * V: the velocity operator V^{-1} (same modes as H; tt_velocity_terms).
 * psi: in Psi_0, out the eigenvector at the final alpha (capacities >=
 * keff.rmax + kickrank).  z: AMEn residual TT.  Report arrays are device
 * memory; status: TT_OK, TT_ERR_NOCONV (max_alpha reached or the secant
 * stagnated, |k - k_prev| < 1e-14), or the inner k-eff solve's error.
 * Workspace: alpha_workspace(...). */
typedef struct {
  double alpha0, alpha1;   /* first two iterates                                   */
  double tol;              /* |k(alpha) - 1| stopping tolerance                    */
  double eps_op;           /* rounding tolerance of H + alpha V^{-1}               */
  int32_t max_alpha;       /* maximum number of k-eff solves                       */
  keff_opts keff;          /* inner k-eff solves                                   */
} alpha_opts;
typedef struct {
  double *alpha_dev;       /* [1] final alpha                                      */
  double *k_dev;           /* [1] k(alpha) of the last solve                       */
  int32_t *iters_dev;      /* [1] k-eff solves performed                           */
  double *alpha_hist_dev;  /* [hist_cap] alpha of each k-eff solve                 */
  double *k_hist_dev;      /* [hist_cap] its k                                     */
  int32_t *keff_iters_hist_dev; /* [hist_cap] its outer iterations                 */
  int32_t hist_cap;
  int32_t *status_dev;     /* [1]                                                  */
} alpha_report;
size_t alpha_workspace(const tt_mat *H, const tt_mat *V, const tt_mat *S, const tt_mat *F,
                       const tt_vec *psi, const tt_vec *z, const alpha_opts *o);
tt_status alpha_secant(const tt_mat *H, const tt_mat *V, const tt_mat *S, const tt_mat *F, tt_vec *psi,
                       tt_vec *z, const alpha_opts *o, alpha_report *rep, void *ws, size_t wsb,
                       tt_stream s);

/* ------------------------------------------------ operator assembly ---
 * Host-side construction of the factor matrices of the rank-1 per-octant
 * terms of H, S, F (readings Z3-Z7, Z34), written as plain
 * column-major host arrays; the caller uploads them and sums/rounds on the
 * device with tt_add / tt_round.  This is one-off setup, not a hot-path step.
 * prob_* describe the problem; op = 0 (H),
 * 1 (S), 2 (F).  Returns the number of terms; with out == NULL only counts.
 * Each term writes 5 factors in core order (x, y, z, angle, group):
 * nv*nv*3 + L*L + G*G doubles, consecutively. */
int32_t tt_transport_terms(int32_t op, int32_t nv, double extent, int32_t G, int32_t L,
                           const double *mu, const double *eta, const double *xi,
                           const double *w, int32_t nmat, const double *sigma_t,
                           const double *sigma_s, const double *nu_sigma_f, const double *chi,
                           int32_t nbox, const int32_t *box_lo, const int32_t *box_hi,
                           const int32_t *box_mat, double *out);

/* Reflective variant of configs[0] (reading Z15, not in the paper): H terms
 * restricted to each octant's interior rows plus, per octant and first inflow
 * axis a, the face equations psi_l - psi_{refl_a(l)} = 0 as rank-1 terms
 * E_x (x) E_y (x) E_z (x) (C_b - R_{a,b}) (x) I_G; S and F as for vacuum. */
int32_t tt_transport_terms_reflective(int32_t op, int32_t nv, double extent, int32_t G, int32_t L,
                                      const double *mu, const double *eta, const double *xi,
                                      const double *w, int32_t nmat, const double *sigma_t,
                                      const double *sigma_s, const double *nu_sigma_f,
                                      const double *chi, int32_t nbox, const int32_t *box_lo,
                                      const int32_t *box_hi, const int32_t *box_mat, double *out);

/* 1-D slab variant: the same construction restricted to the x
 * factor, two half-range blocks (mu < 0 then mu > 0); homogeneous material.
 * Each term writes 3 factors (x, angle, group): nv*nv + L*L + G*G doubles. */
int32_t tt_transport_terms_1d(int32_t op, int32_t nv, double extent, int32_t G, int32_t L,
                              const double *mu, const double *w, const double *sigma_t,
                              const double *sigma_s, const double *nu_sigma_f, const double *chi,
                              double *out);

/* Algorithm 1 (alg:TTtoQTT) for one factor, on the device: the
 * 2^l x 2^l column-major matrix M (device pointer) is reshaped to 2 x..x 2, its
 * row/column bits paired (i_t, j_t) LSB first (Z28) into modes of 4 (row bit
 * fastest), written as the exact index-forwarding TT of that tensor (ranks
 * 4^min(t, l-t)) into q and rounded on the device to eps (tt_round: the
 * TT-SVD with the tail rule delta = eps ||M||_F / sqrt(l-1), reading Z21).
 * q: d = l cores, modes 4, rank capacities >= 4^min(t, l-t) (caller-owned;
 * on return its device ranks are the QTT ranks and core t, viewed as
 * [r_t, 2, 2, r_{t+1}], is the QTT-matrix core).  Errors: TT_ERR_ARG (n not a
 * power of two >= 2, NULL pointers), TT_ERR_SHAPE, TT_ERR_CAPACITY.
 * Workspace: tt_qtt_matrix_dev_workspace(q). */
size_t tt_qtt_matrix_dev_workspace(const tt_vec *q);
tt_status tt_qtt_matrix_dev(int32_t n, const double *M, double eps, tt_vec *q, void *ws, size_t wsb,
                            tt_stream s);

/* Velocity operator V^{-1} of the alpha problem (the alpha term of
 * eq. Discretized_alphaNTE): per octant b the rank-1 term
 * diag(inv_v) o (C_b (x) I) o Ip_z o Ip_y o Ip_x (spatially uniform).
 * dim = 3: 8 terms of 5 factors (x, y, z, angle, group) = 3 nv^2 + L^2 + G^2
 * doubles each; reflective != 0 restricts them to each octant's interior rows
 * (Z15).  dim = 1: 2 terms of 3 factors (x, angle, group); eta, xi may be NULL.
 * inv_v: [G] 1/v per group (host).  out: NULL = count query.  Returns the
 * number of terms, -1 on invalid arguments. */
int32_t tt_velocity_terms(int32_t dim, int32_t nv, int32_t G, int32_t L, const double *mu,
                          const double *eta, const double *xi, const double *inv_v,
                          int32_t reflective, double *out);



#ifdef __cplusplus
}
#endif
#endif /* TT_B200_H */
