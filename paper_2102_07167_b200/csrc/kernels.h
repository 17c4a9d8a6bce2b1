// kernels.h — device-side plan + launchers (product code; used by api.cpp).
#pragma once
#include <cuda.h>  // CUtensorMap (type only; the encoder is fetched through the runtime)
#include <cuda_runtime.h>
#include <cstdint>

#include "plan.h"

namespace kur {

struct Ctrl {             // device-resident control block
  unsigned int ticket;    // last-block detection
  int nonfinite;          // set by RK stage 4 when a phase is not finite
  int record_every;       // > 0: record (r, psi) of theta_n when n % record_every == 0
  int nrec_cap;           // capacity of r_trace in pairs
  long long step;         // n of the current theta_n inside kur_step
  int fp_done;            // implicit midpoint: the fixed-point iteration of this step converged
  int xtimeout;           // fused exchange: an unpack gave up waiting for the peers' records
  int fp_pad;
  double fp_tol;          // implicit midpoint: stop when max_m |theta^{(i+1)}_m - theta^{(i)}_m| <= fp_tol
  double* r_trace;        // [nrec_cap][2]
  double rpsi[2];         // last computed (r, psi)
};

struct DevPlan {
  int64_t n;              // global N
  int64_t n_local;        // this rank's rows
  int32_t C;
  int32_t rows_per_tile;  // <= MAX_TILE_ROWS
  int32_t ntiles;         // local tiles (one CTA each)
  int32_t tile_base;      // global id of local tile 0
  int32_t row_begin;      // internal id of local row 0
  int32_t world;
  int32_t has_parts;          // any tile has stored entries (else no shared memory is needed)
  int32_t pdl;                // world 1: k_prologue / k_remote / k_stage launched as programmatic dependents
  int32_t rov;                // > 0: k_stage overlaps the k_remote pass before it (KUR_REMOTE_OVERLAP = k_remote
                              // CTAs per SM): launched as its programmatic dependent, it stages windows and
                              // gathers the hot parts while k_remote runs and waits for it only before the
                              // finalize, the first reader of Wr
  int32_t has_remote;         // any tile has remote parts summed out of line into Wr (see remote_warp)
  int32_t remote_warp;        // has_remote: 0 = the k_remote pass before each k_stage; inside k_stage, one
                              // warp of each tile sums its remote part while the others gather the hot
                              // windows: 1 = z gathered by 16-byte TMA bulk copies into a shared-memory
                              // ring, 2 = LDG gathers, 3 = TMA tile::gather4 (4 entries per request)
  int32_t cr_hot_warps;       // > 0: inline remote parts run concurrently on warps [cr_hot_warps, NWARPS)
                              // while the hot windows are gathered by the others (k_stage<..., CR = true>)
  const CUtensorMap* tmaps;   // remote_warp 3: HOST array [2] = tensor maps of zbuf[0], zbuf[1] (launcher only)
  const double2* zbuf[2];     // zA, zB (device)
  const TileDesc* tiles;      // [ntiles]
  const int32_t* order;       // [ntiles] launch order
  const PartDesc* parts;      // [n_parts]
  const uint2* chunks;        // [n_chunks] {header offset, groups}
  const uint4* pool;          // index units
  const int32_t* comm_tile0;  // [C+1] global tile ids
  const int32_t* big_comm;    // [n_big] communities of more than 64 tiles (block-reduced block sums)
  int32_t n_big;
  const int32_t* D_ptr;       // [C+1]
  const int32_t* D_idx;
  const int32_t* comm_size;   // [C]
  const int32_t* perm;        // [n] internal -> user
  int32_t rank;
  int32_t xstride;            // doubles per rank in the exchange buffer (xrows + 2 * xtiles)
  int32_t xrows;              // max rows of a shard (theta region of the exchange buffer)
  const int32_t* shard_row0;  // [world+1] internal row range of every rank
  const int32_t* shard_tile0; // [world+1] tile range of every rank
  const double* rowscale;     // [local rows] 1/M_m (degree scaling) or NULL (uniform: K/N)
  const double* potc;         // [local rows] potential constants (kur_potential)
  double2* partial;           // [ntiles_all] per-tile sums of z (global tile ids)
  double* pmax;               // [ntiles_all] per-tile max |fixed-point update| (implicit midpoint)
  double2* Wr;                // [local rows] remote-part row sums of the current stage (k_remote -> k_stage)
  double* const* peer_x;      // fused exchange: [world] every rank's receive buffer (peer memory) or NULL
  unsigned int* const* peer_flag;  // [world] every rank's arrival counter (peer memory)
  unsigned int* xticket;      // this rank's last-CTA ticket for the arrival signal
  const uint32_t* rchunks;    // [n_rchunks][2] remote pass: {chunk id, local row of the tile's row 0}
  const uint8_t* rem_lp;      // [n_rchunks] row-piece shift of each chunk's part
  int32_t n_rchunks;
  double2* S;                 // [C] block sums S_b of the last reduction
  Ctrl* ctrl;
};

// Stage epilogues (k = RHS of the stage state, theta_n = a.theta, acc = a.acc):
//   RK4:  S1 acc = k, ts = theta_n + h/2 k;  S2 acc += 2k, ts = theta_n + h/2 k;
//                     S3 acc += 2k, ts = theta_n + h k;  S4 theta = theta_n + h/6 (acc + k)
//   Euler: E1 theta = theta_n + h k
//   Heun:      H1 acc = k, ts = theta_n + h k;    H2 theta = theta_n + h/2 (acc + k)
//   implicit midpoint (reading R23), fixed point on tp = theta_{n+1}:
//                     M0 tp = theta_n + h k (Euler predictor), ts = (theta_n + tp)/2
//                     MI nv = theta_n + h k, d = |nv - tp|, tp = nv, ts = (theta_n + tp)/2;
//                        skipped entirely once ctrl->fp_done; the finish sets fp_done = (max d <= tol)
//                     then the prologue with a.commit = tp sets theta = tp (step done)
enum StageMode {
  MODE_RHS = 0, MODE_S1 = 1, MODE_S2 = 2, MODE_S3 = 3, MODE_S4 = 4, MODE_POT = 5,
  MODE_E1 = 6, MODE_H1 = 7, MODE_H2 = 8, MODE_M0 = 9, MODE_MI = 10
};
enum RecordMode { REC_NONE = 0, REC_START = 1, REC_STEP = 2 };
enum StagePhase { PHASE_FULL = 0, PHASE_A = 1, PHASE_B = 2 };

struct StageArgs {
  double* theta;          // local rows: theta (prologue/RHS) or theta_n (RK stages; S4 writes theta_{n+1})
  const double* omega;    // local rows
  double* acc;            // local rows: k1 + 2k2 + 2k3 (RK)
  double* out;            // local rows: dtheta (MODE_RHS)
  const double2* zin;     // [n (+pad)] z of the stage state (global rows)
  double2* zout;          // [n (+pad)] z of the next stage state
  const double2* Tin;     // [C] T_a = sum_{b in D(a)} S_b of the stage state
  double2* Tout;          // [C] T of the next stage state
  double KN;              // K / N
  double K;               // coupling (degree scaling and potential)
  double h;               // step
  double* v_out;          // MODE_POT: device scalar receiving V
  double* op_rpsi;        // kur_order_parameter outputs (device) or NULL
  double* op_local;
  int record;             // RecordMode
  double* xsend;          // world > 1: packed [stage theta of local rows | tile partials | tile max]
  const double* commit;   // prologue only: theta = commit (implicit midpoint step completion) or NULL
  int fp_reset;           // the finish clears ctrl->fp_done (implicit midpoint predictor M0)
  int fp_check;           // MODE_MI: tiles publish max |update|, the finish sets ctrl->fp_done
  int no_remote;          // launch_stage: the caller launched k_remote itself (per-kernel timing)
  int phase;              // PHASE_FULL, or world > 1: PHASE_A (own-community hot parts -> Wh, overlaps
                          // the previous exchange) / PHASE_B (Wh + the rest of the tile, finalize)
  double2* Wh;            // [local rows] phase-A row sums (world > 1)
  int xpar;               // fused exchange: receive half (exchange parity) this launch stores into
  double* theta_host;     // final stages (S4, E1, H2): theta_{n+1} also stored here -- the device
                          // mapping of the caller's pinned host buffer (end-to-end path: the
                          // device-to-host copy rides on the stage) -- or NULL
  // Deferred block sums (world 1, inner stages of a step): a stage launched with no_finish writes
  // its tile partials to pout and skips the last-CTA reduction; the next stage (plazy = those
  // partials) forms S_b and T_{c} of its own tile's community at its start, in finish_reduce's
  // exact summation order, instead of reading Tin.  pout NULL = dp.partial.
  double2* pout;
  const double2* plazy;
  int no_finish;
  int rov_wait;           // k_stage launched as the programmatic dependent of k_remote: wait before the finalize
  int lazy_rec;           // the previous stage (RK4 S4) deferred its step record too: the last CTA of this
                          // grid runs finish_reduce on plazy at its start (r(t), ctrl->rpsi, step counter)
};

cudaError_t launch_prologue(const DevPlan& dp, const StageArgs& a, cudaStream_t s);
// k_remote (plans with the remote pass); launch_stage runs it first unless a.no_remote
cudaError_t launch_remote(const DevPlan& dp, const double2* zin, cudaStream_t s);
cudaError_t launch_stage(int mode, const DevPlan& dp, const StageArgs& a, cudaStream_t s);
// world > 1: after the all-gather of the packed buffers (xrecv = world x xstride doubles),
// z of every non-local row from its exchanged phase, all tile partials; then the
// fixed-order block-sum reduction by one CTA.
// world == 1, tiny graphs: the whole kur_step in one single-CTA launch.
cudaError_t launch_small(const DevPlan& dp, const StageArgs& a, double2* zA, double2* zB, double2* TA, double2* TB,
                         long long nsteps, cudaStream_t s);
// expect: with the fused peer-store exchange, the arrival count that completes this exchange
// entry-free plans, world 1: the whole RK4 trajectory in one cooperative launch (one CTA per tile,
// all co-resident; pbuf [2 * ntiles] partial halves, cnt a zeroed, monotonic 64-bit arrival counter:
// q0 = publications of the previous launches, each launch publishes 1 + 4 nsteps)
bool persist_fits(const DevPlan& dp);
cudaError_t launch_persist_rk4(const DevPlan& dp, const StageArgs& a, double2* pbuf, unsigned long long* cnt,
                               long long nsteps, unsigned long long q0, cudaStream_t s);
cudaError_t launch_unpack(const DevPlan& dp, const double* xrecv, double2* zout, unsigned int expect,
                          cudaStream_t s);
cudaError_t launch_finish(const DevPlan& dp, const StageArgs& a, cudaStream_t s);
cudaError_t launch_set_ctrl(Ctrl* c, int record_every, int nrec_cap, double* r_trace, double fp_tol,
                            cudaStream_t s);
cudaError_t launch_permute(const int32_t* perm, int64_t n, const double* in, double* out, int dir,
                           cudaStream_t s);
size_t stage_smem_bytes(int rows_per_tile);
// remote warp (remote_warp == 1): RING_SLOTS groups of 32 lanes x 4 entries x 16 bytes in flight
constexpr int RING_SLOTS = 6;
constexpr size_t RING_BYTES = (size_t)RING_SLOTS * 128 * 16;
// remote warp 3 (gather4): a slot is 32 lanes x one 128-byte cell (64 bytes used)
constexpr int RING_SLOTS_G4 = 3;
static_assert((size_t)RING_SLOTS_G4 * 32 * 128 <= RING_BYTES, "gather4 ring");
// variable-step RK4: tile_ss[t] = sum over tile t's rows of ((y2 - y1) / (atol + rtol |y2|))^2
cudaError_t launch_errnorm(const DevPlan& dp, const double* y1, const double* y2, double atol, double rtol,
                           double* tile_ss, cudaStream_t s);

}  // namespace kur
