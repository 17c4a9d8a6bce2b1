/* kur.h — C ABI of libkur.so: the B200 hot path of Böhle, Kuehn & Thalhammer,
 * "On the reliable and efficient numerical integration of the Kuramoto model
 * and related dynamical systems on graphs" (arXiv 2102.07167).
 *
 * Citation shorthand: P:n = line n of the paper's text.
 *
 * The problem (eq. KuramotoGraph, uniform scaling M_m = M,
 * P:404-408; A need not be symmetric):
 *
 *     theta_j' = omega_j + (K/N) * sum_k A_jk sin(theta_k - theta_j)
 *
 * evaluated through LOCALISED ORDER PARAMETERS (eq.
 * KuramotoGraphApproach) on a community-permuted adjacency:
 * z_k = e^{i theta_k} once per stage, per column community b the block sum
 * S_b = sum_{k in b} z_k, per row
 *     W_j = sum_{b dense for c(j)} S_b - sum_{k in Z_j} z_k + sum_{k in NZ_j} z_k
 * (complement lists Z_j in dense blocks; non-zero lists NZ_j in
 * sparse blocks), and
 *     RHS_j = omega_j + (K/N) Im(conj(z_j) W_j)
 * inside fixed-step classical RK4 (reading R8).
 *
 * Conventions for every call:
 *  - Every function returns a kur_status; none aborts, throws or exits.
 *    On failure a message is kept in a thread-local buffer (kur_last_error).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  All device work is stream-ordered on it; only
 *    kur_graph_build, kur_graph_destroy, kur_check and kur_graph_permutation
 *    block the host.
 *  - Device vectors (theta, omega, dtheta, r_trace, r_psi, local) are
 *    caller-owned device pointers on the handle's device, fp64, in INTERNAL
 *    (community-contiguous) order, covering this rank's rows
 *    [row_begin, row_end) of kur_graph_info.  kur_permute converts between the
 *    user order and the internal order ("permute these quantities
 *    accordingly, perform the time integration, and reorder the solution").
 *  - A handle is not thread-safe; calls on one handle must be serialised.
 *  - With world > 1, kur_rhs, kur_step and kur_order_parameter are
 *    collectives: every rank calls them in the same order.
 */
#ifndef KUR_H_
#define KUR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KUR_OK = 0,
  KUR_ERR_INVALID_ARG = 1,     /* bad scalar (h <= 0, non-finite K, n < 1, threshold outside [0,1]),
                                  NULL pointer, unsorted list, bad segment kind */
  KUR_ERR_INDEX_RANGE = 2,     /* a column id outside [0, n) */
  KUR_ERR_DUPLICATE_INDEX = 3, /* a column listed twice in one segment, or a community given
                                  two segments in one row */
  KUR_ERR_PARTITION = 4,       /* a label outside [0, n_comm), or a listed column outside its
                                  segment's community */
  KUR_ERR_SIZE_MISMATCH = 5,   /* pointer-array lengths inconsistent (e.g. idx_ptr not monotone) */
  KUR_ERR_OOM = 6,             /* host or device allocation failed */
  KUR_ERR_CUDA = 7,            /* a CUDA runtime error (message in kur_last_error) */
  KUR_ERR_NCCL = 8,            /* an NCCL error, or a fused peer exchange that timed out (message in
                                  kur_last_error) */
  KUR_ERR_NONFINITE = 9,       /* a non-finite phase was produced by kur_step (see kur_check) */
  KUR_ERR_UNSUPPORTED = 10,    /* valid request this build does not support (message says why) */
  KUR_ERR_STEPSIZE = 11        /* kur_integrate_adaptive: a step of h_min was rejected, or max_trials
                                  trials did not reach t_end */
} kur_status;

/* Segment kinds of the row-segmented adjacency pattern. */
enum { KUR_ONES = 0, KUR_ZEROS = 1 };

/* Adjacency A in USER numbering, row-segmented by column community.
 * Row u owns segments seg_ptr[u] .. seg_ptr[u+1]-1; segment s covers column
 * community seg_comm[s] (strictly increasing within a row) and lists
 * idx[idx_ptr[s] .. idx_ptr[s+1]-1], user column ids inside that community,
 * strictly ascending:
 *   KUR_ONES : the listed columns are exactly the ones of row u in that community;
 *   KUR_ZEROS: the listed columns are exactly the zeros; every other member is a one.
 * A community with no segment in row u is all zeros in that row.  The
 * diagonal A_uu is "neglected": whether or not it is listed, it
 * never contributes (reading R2).  A plain CSR matrix is the special
 * case "one KUR_ONES segment per non-empty (row, community)".
 * Host arrays are only read during kur_graph_build (copied; not retained). */
typedef struct {
  int64_t n;                /* N: number of oscillators (the paper's M) */
  int32_t n_comm;           /* C: number of communities (labels 0..C-1; empty ones allowed) */
  const int32_t *community; /* [n]     community of user node u (the partition) */
  const int64_t *seg_ptr;   /* [n+1]   seg_ptr[0] = 0, non-decreasing */
  const int32_t *seg_comm;  /* [nseg]  column community of each segment */
  const uint8_t *seg_kind;  /* [nseg]  KUR_ONES or KUR_ZEROS */
  const int64_t *idx_ptr;   /* [nseg+1] idx_ptr[0] = 0, non-decreasing */
  const int32_t *idx;       /* [idx_ptr[nseg]] user column ids (may be NULL if empty) */
  double dense_threshold;   /* block (a,b) is DENSE iff zeros_ab < threshold * entries_ab, counted
                               over off-diagonal entries; < 0 selects the paper's rule
                               "precompute when ones outnumber zeros": DENSE iff
                               zeros < ones, a tie is SPARSE (reading R3).  0 forces all-sparse
                               (direct CSR); must be <= 1. */
  int32_t hot_min;          /* tuning: minimum entries of a tile in one column window for the
                               window to be staged in shared memory; <= 0 selects the default */
  int32_t flags;            /* tuning / tests, 0 = automatic: low 16 bits a forced tile size in rows
                               (a multiple of 32 in [32, 2048]); | KUR_FLAG_REMOTE_PASS or
                               | KUR_FLAG_REMOTE_INLINE forces where the remote (global-gather)
                               entries are summed: a separate pass before each stage, or inline */
  int32_t scaling;          /* KUR_SCALING_UNIFORM: M_m = N (the north_star model), or
                               KUR_SCALING_DEGREE: M_m = sum_l A_ml (a zero row gives
                               theta_m' = omega_m).  The degree counts the off-diagonal
                               ones plus A_mm, and A_mm = 1 only when m is listed in a KUR_ONES
                               segment of its own community (reading R22). */
  int32_t reserved;         /* must be 0 */
} kur_graph_desc;

enum { KUR_SCALING_UNIFORM = 0, KUR_SCALING_DEGREE = 1 };
enum { KUR_FLAG_REMOTE_PASS = 1 << 16, KUR_FLAG_REMOTE_INLINE = 2 << 16 };

/* Multi-GPU placement: contiguous ranges of whole communities per rank,
 * balanced by stored-entry count (every rank computes the same split).
 * nccl_id points at a 128-byte ncclUniqueId that rank 0 created with
 * kur_nccl_unique_id and the caller broadcast (e.g. over a torch process
 * group); each stage then all-gathers the packed [stage phases | tile partials]
 * of every rank over NCCL.  nccl_id = NULL with world > 1 builds a rank handle
 * for the single-process group calls (kur_group_*).  NULL desc = single GPU
 * (the current device). */
typedef struct {
  int32_t rank;
  int32_t world;
  int32_t device;
  const void *nccl_id;
  int32_t flags;    /* 0, or KUR_DIST_PEER_EXCHANGE: the fused RK-stage kernel stores its phases
                       and tile partials straight into every rank's receive buffer (NVLink peer
                       memory, CUDA IPC handles exchanged over NCCL at build) and signals an
                       arrival counter there; the next stage's unpack waits on its counter — no
                       separate all-gather.  Falls back to ncclAllGather when peer mapping fails
                       (kur_graph_info.peer_exchange says which).  Group handles (nccl_id NULL):
                       in-process peers. */
  int32_t reserved;
} kur_dist_desc;
enum { KUR_DIST_PEER_EXCHANGE = 1 };

typedef struct {
  int64_t n, n_comm;
  int32_t rank, world, device, rows_per_tile;
  int64_t row_begin, row_end;  /* this rank's internal rows */
  int64_t nnz;                 /* ones of A, diagonal excluded (direct-CSR entry count) */
  int64_t n_idx;               /* stored list entries (complements + non-zeros), this rank */
  int64_t n_idx_hot;           /* of which gathered from shared-memory windows (13-bit slots) */
  int64_t n_idx_remote;        /* of which gathered from global memory (32-bit) */
  int64_t n_slots_hot;         /* hot slots incl. padding */
  int64_t n_slots_remote;      /* remote slots incl. padding */
  int64_t n_dense_blocks;      /* non-empty blocks handled by precomputed sums */
  int64_t n_sparse_blocks;     /* non-empty blocks handled by direct summation */
  int64_t n_tiles, n_hot_parts;
  int64_t n_window_loads;      /* 64 KB z windows staged in shared memory per RHS (all tiles) */
  int64_t sincos_per_rhs;      /* N sin/cos pairs = the "2M" trig evaluations of P:660 */
  int64_t bytes_per_rhs;       /* algorithmic HBM bytes of one RHS */
  int64_t bytes_pool;          /* device bytes of the index pool (incl. padding) */
  double build_seconds;        /* host time of kur_graph_build */
  int32_t remote_pass;         /* 1: remote entries summed by the separate k_remote pass before each
                                  stage kernel (2 launches per RHS), 0: inline */
  int32_t peer_exchange;       /* world > 1: 1 = fused peer-store exchange active, 0 = all-gather */
} kur_graph_info_t;

typedef struct kur_graph kur_graph; /* opaque; owns all device data and workspace */

/* Builds the block plan (census, dense/sparse rule, permutation, lists) on the
 * host and uploads it.  Blocks.  See P:524-571. */
kur_status kur_graph_build(const kur_graph_desc *desc, const kur_dist_desc *dist, void *stream,
                           kur_graph **out);
kur_status kur_graph_destroy(kur_graph *g);
kur_status kur_graph_info(const kur_graph *g, kur_graph_info_t *info);

/* Host copy of the permutation: perm[i] = user id of internal node i (all n). Blocks. */
kur_status kur_graph_permutation(const kur_graph *g, int32_t *perm);

enum { KUR_USER_TO_INTERNAL = 0, KUR_INTERNAL_TO_USER = 1 };
/* Device permutation of a full-length fp64 vector (both in and out have n
 * entries; in != out).  USER_TO_INTERNAL: out[i] = in[perm[i]];
 * INTERNAL_TO_USER: out[perm[i]] = in[i]. */
kur_status kur_permute(const kur_graph *g, const double *in, double *out, int32_t dir, void *stream);

/* dtheta = G(theta): one evaluation of the right-hand side (P:443 with the
 * block-hybrid sums of P:538-570).  theta, omega, dtheta: this rank's rows. */
kur_status kur_rhs(kur_graph *g, const double *theta, const double *omega, double K, double *dtheta,
                   void *stream);

/* nsteps classical RK4 steps of size h, theta updated in place (this rank's
 * rows).  If record_every > 0 and r_trace != NULL, the order parameter
 * (r, psi) of theta_n is written to r_trace[2*(n/record_every)]
 * for every n = 0, record_every, 2*record_every, ... <= nsteps
 * (floor(nsteps/record_every)+1 pairs, replicated on every rank).
 * A non-finite phase raises a device flag reported by kur_check.
 * Host buffers: theta and/or omega may be HOST memory (pinned or pageable);
 * with world > 1 (NCCL handle) each rank passes its own shard of n_local rows.  The library then copies them into device buffers it owns, runs
 * the same kernels, and stores theta_{n+1} back into the host theta: for
 * pinned memory, when the final stage is long enough to hide the transfer
 * (kernel bytes per RHS >= 60x the bytes of theta), the last step's final
 * stage writes it through the buffer's device mapping (the device-to-host
 * transfer overlaps that stage); otherwise one copy follows the steps.  The host result is complete when the stream is
 * synchronised; it is bitwise the device-buffer result.  Same for
 * kur_step_method.  KUR_ERR_UNSUPPORTED for host buffers on a world > 1 handle
 * without NCCL (the in-process kur_group_* handles take device buffers). */
kur_status kur_step(kur_graph *g, double *theta, const double *omega, double K, double h,
                    int64_t nsteps, int32_t record_every, double *r_trace, void *stream);

/* The paper's other one-step integrators on the same RHS,
 * fixed step h, theta updated in place, r_trace / record_every / kur_check as
 * for kur_step (which equals method KUR_RK4):
 *   KUR_RK4:    classical 4-stage Runge-Kutta;
 *   KUR_EULER:  theta_{n+1} = theta_n + h G(theta_n);
 *   KUR_HEUN:   k1 = G(theta_n), k2 = G(theta_n + h k1),
 *               theta_{n+1} = theta_n + (h/2)(k1 + k2) (explicit 2nd order);
 *   KUR_IMPLICIT_MIDPOINT: theta_{n+1} = theta_n + h G((theta_n + theta_{n+1})/2)
 *               (implicit 2nd order, geometric), solved by fixed-point
 *               iteration from the Euler predictor theta_n + h G(theta_n): iterate
 *               t <- theta_n + h G((theta_n + t)/2) until max_m |t_new - t_old| <=
 *               fp_tol or fp_max_iter iterations (reading R23); the
 *               convergence test runs on the device (iterations after it are no-ops).
 * fp_tol (>= 0, finite) and fp_max_iter (>= 1) are only read for the implicit
 * midpoint rule.  Collective for world > 1.  KUR_ERR_INVALID_ARG for an
 * unknown method or bad fixed-point parameters. */
enum { KUR_RK4 = 0, KUR_EULER = 1, KUR_HEUN = 2, KUR_IMPLICIT_MIDPOINT = 3 };
kur_status kur_step_method(kur_graph *g, int32_t method, double *theta, const double *omega, double K, double h,
                           int64_t nsteps, int32_t record_every, double *r_trace, double fp_tol,
                           int32_t fp_max_iter, void *stream);

/* Variable-step classical RK4 ("a variable stepsize fourth-order explicit
 * Runge-Kutta method leads to a reliable result"; the controller is unstated,
 * DESIGN.md reading R25 follows the SPEC's step doubling).  Integrates theta
 * in place from t = 0 to t_end.  A trial step of size hs (hs = t_end - t for the
 * last step, i.e. when t + h >= t_end - 1e-12 h) computes on the device
 * y1 = one RK4 step of hs and y2 = two RK4 steps of hs/2 from theta, then
 *     err = sqrt( (1/N) sum_m ((y2_m - y1_m) / (atol + rtol |y2_m|))^2 ) / 15
 * (per-tile partial sums on the device, added on the host in tile order); the
 * step is accepted iff err <= 1 (theta = y2, t += hs), and
 *     h <- clamp(hs * clamp(safety * err^(-1/5), fac_min, fac_max), h_min, h_max)
 * (factor fac_max when err = 0).  Blocks: the controller runs on the host, one
 * stream synchronisation per trial.  For each accepted step k < cap the host
 * arrays t_out[k], h_out[k] and rpsi_out[2k..2k+1] (the order parameter of the
 * accepted state) are written when non-NULL.  Errors: KUR_ERR_INVALID_ARG (bad
 * controls), KUR_ERR_STEPSIZE, KUR_ERR_NONFINITE (non-finite error estimate).
 * Collective for world > 1 (the per-tile partials of all ranks are all-gathered
 * and added on the host in global tile order, so every rank and every world size
 * takes the same decisions); kur_group_integrate_adaptive drives in-process rank
 * handles. */
typedef struct {
  double t_end;            /* > 0 */
  double h0;               /* first trial step, > 0 */
  double h_min, h_max;     /* 0 < h_min <= h_max */
  double atol, rtol;       /* error weights atol + rtol |y2_m|; >= 0, atol + rtol > 0 */
  double safety;           /* e.g. 0.9 */
  double fac_min, fac_max; /* 0 < fac_min <= 1 <= fac_max */
  int64_t max_trials;      /* >= 1 */
} kur_adaptive_ctrl;
kur_status kur_integrate_adaptive(kur_graph *g, double *theta, const double *omega, double K,
                                  const kur_adaptive_ctrl *ctrl, int64_t cap, double *t_out, double *h_out,
                                  double *rpsi_out, int64_t *n_accepted, int64_t *n_rejected, void *stream);
kur_status kur_group_integrate_adaptive(kur_graph *const *g, int32_t world, double *const *theta,
                                        const double *const *omega, double K, const kur_adaptive_ctrl *ctrl,
                                        int64_t cap, double *t_out, double *h_out, double *rpsi_out,
                                        int64_t *n_accepted, int64_t *n_rejected, void *stream);

/* r_psi[2] = (r, psi) of the complex order parameter r e^{i psi} =
 * (1/N) sum_k e^{i theta_k} (psi = 0 when r = 0).  local (may be
 * NULL): [n_comm][2] = (r_b, psi_b) of the localised order parameters
 * S_b / n_b; empty communities give (0, 0). */
kur_status kur_order_parameter(kur_graph *g, const double *theta, double *r_psi, double *local,
                               void *stream);

/* Single-process execution of a whole world of rank handles (built with
 * world > 1 and nccl_id = NULL, ranks 0..world-1, all on one device): the
 * same kernels as the NCCL path, the all-gather done by device copies, ranks
 * run one after another on `stream`.  Used to test the sharded path and its
 * bitwise world-size invariance on one GPU.  Arrays are indexed by rank. */
kur_status kur_group_rhs(kur_graph *const *g, int32_t world, const double *const *theta,
                         const double *const *omega, double K, double *const *dtheta, void *stream);
kur_status kur_group_step(kur_graph *const *g, int32_t world, double *const *theta, const double *const *omega,
                          double K, double h, int64_t nsteps, int32_t record_every, double *const *r_trace,
                          void *stream);
kur_status kur_group_step_method(kur_graph *const *g, int32_t world, int32_t method, double *const *theta,
                                 const double *const *omega, double K, double h, int64_t nsteps,
                                 int32_t record_every, double *const *r_trace, double fp_tol, int32_t fp_max_iter,
                                 void *stream);

/* V_out[0] (device) = the potential of the model on the graph (eq.
 * ExtendedPotentialConservation; P:221-233 for the complete graph):
 *   V = -sum_m omega_m theta_m + (K/2) sum_{m,l} (A_ml / M_m) (1 - cos(theta_l - theta_m)),
 * evaluated with the same localised sums as the RHS, through the auxiliary
 * identity of P:457-466: sum_l A_ml cos(theta_l - theta_m) = Re(conj z_m W_m).
 * V is a Lyapunov function of the flow for symmetric A with uniform scaling
 * (P:212-218).  Collective for world > 1 (replicated result). */
kur_status kur_potential(kur_graph *g, const double *theta, const double *omega, double K, double *V_out,
                         void *stream);

/* Synchronises `stream`; returns KUR_ERR_NONFINITE (and clears the flag) if a
 * previous kur_step produced a non-finite phase, and KUR_ERR_NCCL if a fused
 * peer-store exchange gave up waiting for another rank's record. */
kur_status kur_check(kur_graph *g, void *stream);

/* ---- Host-only plan introspection (no device needed; tests and tooling) ----
 * kur_plan_build runs exactly the host builder of kur_graph_build (validation,
 * census, dense/sparse rule, permutation, tiles, chunked layout) for one rank
 * and keeps the result on the host.  kur_plan_export DECODES the stored
 * layout back into plain lists, so a caller can rebuild A from it:
 *   sizes[0..15] = n, n_comm, n_local, row_begin, n_entries (stored entries of
 *   this rank, padding excluded), n_dense_pairs (length of D_idx), n_tiles,
 *   rows_per_tile, nnz, world, bank conflicts found by the last export (hot
 *   quarter-warp positions whose slots share a residue mod 8; 0 by
 *   construction), hot slots, hot entries, remote slots, remote entries,
 *   window loads per RHS;
 *   perm[n]: user id of internal node i; D_ptr[n_comm+1], D_idx: dense column
 *   communities of each row community (their block sums are added);
 *   row_ptr[n_local+1], cols[n_entries] (internal column ids), neg[n_entries]
 *   (1 = complement entry, subtracted; 0 = non-zero entry, added,
 *   P:538-542) for this rank's rows; shard_row0[world+1]: row ranges of all
 *   ranks.  Errors as kur_graph_build. */
typedef struct kur_plan kur_plan;
kur_status kur_plan_build(const kur_graph_desc *desc, int32_t rank, int32_t world, int32_t sm_count,
                          kur_plan **out);
kur_status kur_plan_sizes(const kur_plan *p, int64_t *sizes /* [16] */);
kur_status kur_plan_export(const kur_plan *p, int32_t *perm, int32_t *D_ptr, int32_t *D_idx, int64_t *row_ptr,
                           int32_t *cols, int8_t *neg, int32_t *shard_row0);
kur_status kur_plan_destroy(kur_plan *p);
/* Tile and part structure of the plan (host): tiles[n_tiles][7] = {row0 (internal), nrows,
 * community, nparts, nhot, nown, nloc}: the tile's parts are its nown own-community hot windows,
 * then nhot - nown other hot windows, then at most one remote part; the first
 * nloc <= nown of them lie inside this rank's rows (phase A of the sharded stage);
 * part_window[sum nparts] = window id of each part in that order (-1 = remote), or NULL. */
kur_status kur_plan_tiles(const kur_plan *p, int32_t *tiles, int32_t *part_window);

/* Per-launch timing for measurement (bench.py): while enabled, kur_step
 * records a CUDA event pair around every kernel it launches, on `stream`.
 * kur_timing_read blocks until the last recorded event, writes out[9] =
 * {total ms of k_prologue launches, their count, total ms of k_stage (fused
 * RK stage) launches -- or of the single-launch trajectory kernels -- the RHS
 * evaluations they did, total ms of k_remote launches (remote-pass plans; one
 * per RHS evaluation), their count, the number of timed kernel launches,
 * world > 1: total ms of the phase-A k_stage launches (also in out[2]), their
 * count} and clears the record.  Enabling also clears it. */
kur_status kur_timing(kur_graph *g, int32_t enable);
kur_status kur_timing_read(kur_graph *g, double *out /* [9] */);

/* Creates a 128-byte NCCL unique id (rank 0), to be broadcast by the caller. */
kur_status kur_nccl_unique_id(void *id128);

const char *kur_status_string(kur_status s);
const char *kur_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* KUR_H_ */
