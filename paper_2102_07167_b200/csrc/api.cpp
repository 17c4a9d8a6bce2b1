// api.cpp — the C ABI of libkur.so (include/kur.h): handle ownership, device
// memory, launch orchestration, error conventions.  Product code.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <omp.h>

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "kernels.h"
#include "kur.h"
#include "plan.h"

using namespace kur;

namespace {
thread_local std::string g_last_error;

kur_status fail(kur_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
kur_status cuda_fail(cudaError_t e, const char* what) {
  return fail(KUR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define KUR_CUDA(call)                                                     \
  do {                                                                     \
    cudaError_t e_ = (call);                                               \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);                    \
  } while (0)

template <class T>
cudaError_t upload(T** dptr, const std::vector<T>& v) {
  const size_t bytes = sizeof(T) * (v.empty() ? 1 : v.size());
  cudaError_t e = cudaMalloc((void**)dptr, bytes);
  if (e != cudaSuccess) return e;
  if (!v.empty()) e = cudaMemcpy(*dptr, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice);
  return e;
}
}  // namespace

struct kur_graph {
  int device = 0;
  int64_t n = 0, n_local = 0, n_pad = 0;
  int32_t C = 0;
  kur_graph_info_t info{};
  std::vector<int32_t> perm_host;
  std::vector<int32_t> shard_tile0_host;  // [world+1] tile ranges of all ranks
  DevPlan dp{};
  // device allocations
  TileDesc* d_tiles = nullptr;
  int32_t* d_order = nullptr;
  PartDesc* d_parts = nullptr;
  uint2* d_chunks = nullptr;
  uint4* d_pool = nullptr;
  int32_t *d_comm_tile0 = nullptr, *d_D_ptr = nullptr, *d_D_idx = nullptr, *d_csize = nullptr, *d_perm = nullptr;
  double2 *zA = nullptr, *zB = nullptr, *TA = nullptr, *TB = nullptr, *S = nullptr, *partial = nullptr;
  double* acc = nullptr;
  double *theta_ws = nullptr, *omega_ws = nullptr;  // host-buffer kur_step: device copies of theta / omega
  double* host_out = nullptr;  // device mapping of the caller's pinned theta for the final stage, or NULL
  double* pmax = nullptr;
  double2* Wr = nullptr;
  uint32_t* d_rchunks = nullptr;
  uint8_t* d_rem_lp = nullptr;
  Ctrl* ctrl = nullptr;
  ncclComm_t comm = nullptr;
  int world = 1;
  int32_t *d_shard_row0 = nullptr, *d_shard_tile0 = nullptr;
  double *d_rowscale = nullptr, *d_potc = nullptr;
  double *xsend = nullptr, *xrecv = nullptr;  // world > 1: packed exchange buffers
  double2* Wh = nullptr;                      // world > 1: phase-A row sums
  CUtensorMap tmaps[2];                       // remote warp 3: z viewed as [n_pad][2] fp64 (gather4)
  cudaStream_t comm_stream = nullptr;         // NCCL: exchange + unpack + finish, overlapping phase A
  cudaEvent_t ev_b = nullptr, ev_exch = nullptr;
  bool exch_pending = false;                  // comm_stream holds an exchange the next phase B waits for
  bool remote_on_xs = true;                   // world > 1: k_remote on the exchange stream (KUR_REMOTE_SEQ: A/B)
  // fused peer-store exchange (KUR_DIST_PEER_EXCHANGE)
  bool peer_req = false, peer_on = false;
  unsigned int* d_flag = nullptr;             // this rank's arrival counter (peers increment it)
  unsigned int* d_xticket = nullptr;
  double** d_peer_x = nullptr;                // [world] device array of receive-buffer pointers
  unsigned int** d_peer_flag = nullptr;       // [world] device array of counter pointers
  std::vector<void*> ipc_opened;              // peer allocations mapped through CUDA IPC
  unsigned int xepoch = 0;                    // exchanges completed on this handle
  // optional per-launch CUDA-event timing (kur_timing)
  bool timing = false;
  std::vector<cudaEvent_t> ev;        // pool, reused
  std::vector<std::pair<int, int>> ev_kind;  // per recorded pair: (0 prologue | 1 k_stage | 2 k_remote, RHS evals)
  bool small = false;                 // whole kur_step in one single-CTA launch
  bool persist = false;               // entry-free plan: whole RK4 kur_step in one cooperative launch
  double2* pbuf = nullptr;            // persist: [2][ntiles] tile partials
  unsigned long long* gbar = nullptr; // persist: monotonic arrival counter
  unsigned long long persist_q = 0;   // persist: publications so far
  int32_t* d_big = nullptr;           // communities of > 64 tiles
  // deferred block sums (world 1): the inner stages of a step skip the last-CTA reduction, the next
  // stage forms its T from their tile partials (StageArgs::no_finish / plazy); partial and partialB
  // alternate as the destination so a stage never overwrites the partials it reads
  bool lazy_ok = false;
  double2* partialB = nullptr;
  const double2* lazy_prev = nullptr;  // partials of the previous stage if it skipped its reduction
  bool defer_rec_ok = false;           // kur_step RK4, not the last step: S4 may defer its record too
  bool lazy_rec_ok = true;             // KUR_LAZY_REC=0: every S4 reduces itself (A/B switch)
  bool rec_pending = false;            // the previous stage (S4) deferred its record to this one
  size_t ev_used = 0;
  cudaError_t mark(cudaStream_t s) {  // records the next event of the pool on s
    if (!timing) return cudaSuccess;
    if (ev_used == ev.size()) {
      cudaEvent_t e;
      cudaError_t r = cudaEventCreate(&e);
      if (r != cudaSuccess) return r;
      ev.push_back(e);
    }
    return cudaEventRecord(ev[ev_used++], s);
  }

  ~kur_graph() {
    cudaSetDevice(device);
    void* ptrs[] = {d_tiles, d_order, d_parts, d_chunks, d_pool, d_comm_tile0, d_D_ptr, d_D_idx,
                    d_csize, d_perm, zA, zB, TA, TB, S, partial, acc, ctrl, d_shard_row0, d_shard_tile0,
                    xsend, xrecv, d_rowscale, d_potc, pmax, Wr, Wh, d_rchunks, d_rem_lp, d_flag, d_xticket,
                    d_peer_x, d_peer_flag, theta_ws, omega_ws, pbuf, gbar, d_big, partialB};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    if (comm_stream) cudaStreamSynchronize(comm_stream);
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    if (comm) ncclCommDestroy(comm);
    if (ev_b) cudaEventDestroy(ev_b);
    if (ev_exch) cudaEventDestroy(ev_exch);
    if (comm_stream) cudaStreamDestroy(comm_stream);
  }
};

extern "C" {

const char* kur_status_string(kur_status s) {
  switch (s) {
    case KUR_OK: return "KUR_OK";
    case KUR_ERR_INVALID_ARG: return "KUR_ERR_INVALID_ARG";
    case KUR_ERR_INDEX_RANGE: return "KUR_ERR_INDEX_RANGE";
    case KUR_ERR_DUPLICATE_INDEX: return "KUR_ERR_DUPLICATE_INDEX";
    case KUR_ERR_PARTITION: return "KUR_ERR_PARTITION";
    case KUR_ERR_SIZE_MISMATCH: return "KUR_ERR_SIZE_MISMATCH";
    case KUR_ERR_OOM: return "KUR_ERR_OOM";
    case KUR_ERR_CUDA: return "KUR_ERR_CUDA";
    case KUR_ERR_NCCL: return "KUR_ERR_NCCL";
    case KUR_ERR_NONFINITE: return "KUR_ERR_NONFINITE";
    case KUR_ERR_UNSUPPORTED: return "KUR_ERR_UNSUPPORTED";
    case KUR_ERR_STEPSIZE: return "KUR_ERR_STEPSIZE";
  }
  return "KUR_ERR_UNKNOWN";
}

const char* kur_last_error(void) { return g_last_error.c_str(); }

kur_status kur_nccl_unique_id(void* id128) {
  if (!id128) return fail(KUR_ERR_INVALID_ARG, "id128 is NULL");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(KUR_ERR_NCCL, ncclGetErrorString(r));
  std::memcpy(id128, &id, sizeof(id));
  return KUR_OK;
}

kur_status kur_graph_build(const kur_graph_desc* desc, const kur_dist_desc* dist, void* stream,
                           kur_graph** out) {
  (void)stream;
  if (!out) return fail(KUR_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  int32_t rank = 0, world = 1;
  int device = 0;
  if (dist) {
    rank = dist->rank;
    world = dist->world;
    device = dist->device;
  } else {
    KUR_CUDA(cudaGetDevice(&device));
  }
  KUR_CUDA(cudaSetDevice(device));
  int sm = 148;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, device);
  HostPlan P;
  std::string err;
  kur_status st;
  try {
    st = build_plan(desc, rank, world, sm, P, err);
  } catch (const std::bad_alloc&) {
    return fail(KUR_ERR_OOM, "host allocation failed in kur_graph_build");
  }
  if (st != KUR_OK) return fail(st, err);

  kur_graph* g = new (std::nothrow) kur_graph();
  if (!g) return fail(KUR_ERR_OOM, "host allocation failed");
  g->device = device;
  g->n = P.n;
  g->C = P.C;
  g->n_local = P.row_end - P.row_begin;
  g->n_pad = ((P.n + 1 + WZ - 1) / WZ) * WZ + WZ;  // z[n..n_pad) stay zero (sentinels, window tails)
  g->perm_host = P.perm;
  g->shard_tile0_host = P.shard_tile0;
  auto bail = [&](cudaError_t e, const char* what) {
    delete g;
    return e == cudaErrorMemoryAllocation ? fail(KUR_ERR_OOM, std::string(what) + ": out of device memory")
                                          : cuda_fail(e, what);
  };
  cudaError_t e;
  int64_t pool_bytes = 0;
  std::vector<int32_t> csize((size_t)P.C);
  for (int32_t c = 0; c < P.C; ++c) csize[(size_t)c] = P.comm_off[(size_t)c + 1] - P.comm_off[(size_t)c];
  if ((e = upload(&g->d_tiles, P.tiles)) != cudaSuccess) return bail(e, "tiles");
  if ((e = upload(&g->d_order, P.tile_order)) != cudaSuccess) return bail(e, "order");
  if ((e = upload(&g->d_parts, P.parts)) != cudaSuccess) return bail(e, "parts");
  {
    std::vector<uint2> ch(P.chunks.size());
    for (size_t i = 0; i < ch.size(); ++i) ch[i] = make_uint2(P.chunks[i].ofs, P.chunks[i].ng);
    if ((e = upload(&g->d_chunks, ch)) != cudaSuccess) return bail(e, "chunks");
  }
  {
    const size_t bytes = sizeof(Unit) * P.pool.size();
    pool_bytes = (int64_t)bytes;
    if ((e = cudaMalloc((void**)&g->d_pool, bytes)) != cudaSuccess) return bail(e, "pool");
    if ((e = cudaMemcpy(g->d_pool, P.pool.data(), bytes, cudaMemcpyHostToDevice)) != cudaSuccess)
      return bail(e, "pool copy");
    std::vector<Unit>().swap(P.pool);
  }
  if ((e = upload(&g->d_comm_tile0, P.comm_tile0)) != cudaSuccess) return bail(e, "comm_tile0");
  if ((e = upload(&g->d_D_ptr, P.D_ptr)) != cudaSuccess) return bail(e, "D_ptr");
  if ((e = upload(&g->d_D_idx, P.D_idx)) != cudaSuccess) return bail(e, "D_idx");
  if ((e = upload(&g->d_csize, csize)) != cudaSuccess) return bail(e, "comm sizes");
  if ((e = upload(&g->d_perm, P.perm)) != cudaSuccess) return bail(e, "perm");
  if (!P.rowscale.empty() && (e = upload(&g->d_rowscale, P.rowscale)) != cudaSuccess) return bail(e, "rowscale");
  if ((e = upload(&g->d_potc, P.potc)) != cudaSuccess) return bail(e, "potc");
  const size_t zbytes = sizeof(double2) * (size_t)g->n_pad;
  if ((e = cudaMalloc((void**)&g->zA, zbytes)) != cudaSuccess) return bail(e, "zA");
  if ((e = cudaMalloc((void**)&g->zB, zbytes)) != cudaSuccess) return bail(e, "zB");
  if ((e = cudaMemset(g->zA, 0, zbytes)) != cudaSuccess) return bail(e, "zA");
  if ((e = cudaMemset(g->zB, 0, zbytes)) != cudaSuccess) return bail(e, "zB");
  const size_t cb = sizeof(double2) * (size_t)std::max<int32_t>(P.C, 1);
  if ((e = cudaMalloc((void**)&g->TA, cb)) != cudaSuccess) return bail(e, "TA");
  if ((e = cudaMalloc((void**)&g->TB, cb)) != cudaSuccess) return bail(e, "TB");
  if ((e = cudaMalloc((void**)&g->S, cb)) != cudaSuccess) return bail(e, "S");
  const int32_t ntiles_all = P.comm_tile0[(size_t)P.C];
  if ((e = cudaMalloc((void**)&g->partial, sizeof(double2) * (size_t)std::max<int32_t>(ntiles_all, 1))) != cudaSuccess)
    return bail(e, "partial");
  if ((e = cudaMalloc((void**)&g->partialB, sizeof(double2) * (size_t)std::max<int32_t>(ntiles_all, 1))) != cudaSuccess)
    return bail(e, "partialB");
  if ((e = cudaMalloc((void**)&g->pmax, sizeof(double) * (size_t)std::max<int32_t>(ntiles_all, 1))) != cudaSuccess)
    return bail(e, "pmax");
  if ((e = cudaMalloc((void**)&g->acc, sizeof(double) * (size_t)std::max<int64_t>(g->n_local, 1))) != cudaSuccess)
    return bail(e, "acc");
  if ((e = cudaMalloc((void**)&g->ctrl, sizeof(Ctrl))) != cudaSuccess) return bail(e, "ctrl");
  if ((e = cudaMemset(g->ctrl, 0, sizeof(Ctrl))) != cudaSuccess) return bail(e, "ctrl");
  if ((e = cudaMemset(g->TA, 0, cb)) != cudaSuccess) return bail(e, "TA");
  if ((e = cudaMemset(g->TB, 0, cb)) != cudaSuccess) return bail(e, "TB");
  if ((e = cudaMemset(g->S, 0, cb)) != cudaSuccess) return bail(e, "S");
  g->world = world;
  int32_t xrows = 0, xtiles = 0;
  for (int32_t r = 0; r < world; ++r) {
    xrows = std::max(xrows, P.shard_row0[(size_t)r + 1] - P.shard_row0[(size_t)r]);
    xtiles = std::max(xtiles, P.shard_tile0[(size_t)r + 1] - P.shard_tile0[(size_t)r]);
  }
  const int32_t xstride = std::max(xrows + 3 * xtiles, 1);  // [phases | per tile (sum z, max |update|)]
  if ((e = upload(&g->d_shard_row0, P.shard_row0)) != cudaSuccess) return bail(e, "shard_row0");
  if ((e = upload(&g->d_shard_tile0, P.shard_tile0)) != cudaSuccess) return bail(e, "shard_tile0");
  if (world > 1) {
    if ((e = cudaMalloc((void**)&g->xsend, sizeof(double) * (size_t)xstride)) != cudaSuccess) return bail(e, "xsend");
    const bool peer = dist && (dist->flags & KUR_DIST_PEER_EXCHANGE);  // two halves by exchange parity
    if ((e = cudaMalloc((void**)&g->xrecv, sizeof(double) * (size_t)xstride * (size_t)world * (peer ? 2 : 1))) !=
        cudaSuccess)
      return bail(e, "xrecv");
    if ((e = cudaMemset(g->xsend, 0, sizeof(double) * (size_t)xstride)) != cudaSuccess) return bail(e, "xsend");
    if ((e = cudaMalloc((void**)&g->Wh, sizeof(double2) * (size_t)std::max<int64_t>(g->n_local, 1))) != cudaSuccess)
      return bail(e, "Wh");
    g->peer_req = dist && (dist->flags & KUR_DIST_PEER_EXCHANGE);
    if (g->peer_req) {
      if ((e = cudaMalloc((void**)&g->d_flag, 256)) != cudaSuccess || (e = cudaMemset(g->d_flag, 0, 256)) != cudaSuccess ||
          (e = cudaMalloc((void**)&g->d_xticket, sizeof(unsigned int))) != cudaSuccess ||
          (e = cudaMemset(g->d_xticket, 0, sizeof(unsigned int))) != cudaSuccess ||
          (e = cudaMalloc((void**)&g->d_peer_x, sizeof(double*) * (size_t)world)) != cudaSuccess ||
          (e = cudaMalloc((void**)&g->d_peer_flag, sizeof(unsigned int*) * (size_t)world)) != cudaSuccess)
        return bail(e, "peer exchange buffers");
    }
    g->remote_on_xs = std::getenv("KUR_REMOTE_SEQ") == nullptr;
    {
      int lo = 0, hi = 0;  // the exchange stream gets the highest priority: its few CTAs jump the queue
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      if ((e = cudaStreamCreateWithPriority(&g->comm_stream, cudaStreamNonBlocking, hi)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&g->ev_b, cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&g->ev_exch, cudaEventDisableTiming)) != cudaSuccess)
        return bail(e, "exchange stream");
    }
    if (dist && dist->nccl_id) {
      ncclUniqueId id;
      std::memcpy(&id, dist->nccl_id, sizeof(id));
      ncclResult_t nr = ncclCommInitRank(&g->comm, world, id, rank);
      if (nr != ncclSuccess) {
        delete g;
        return fail(KUR_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(nr));
      }
      if (g->peer_req) {
        // map every rank's receive buffer and arrival counter into this process: CUDA IPC
        // handles all-gathered over NCCL; any failure keeps the all-gather exchange
        cudaIpcMemHandle_t mine[2];
        bool ok = cudaIpcGetMemHandle(&mine[0], g->xrecv) == cudaSuccess &&
                  cudaIpcGetMemHandle(&mine[1], g->d_flag) == cudaSuccess;
        std::vector<cudaIpcMemHandle_t> all((size_t)world * 2);
        char* dbuf = nullptr;
        const size_t hb = sizeof(mine);
        ok = ok && cudaMalloc((void**)&dbuf, hb * (size_t)(world + 1)) == cudaSuccess;
        ok = ok && cudaMemcpy(dbuf, mine, hb, cudaMemcpyHostToDevice) == cudaSuccess;
        ok = ok && ncclAllGather(dbuf, dbuf + hb, hb, ncclChar, g->comm, g->comm_stream) == ncclSuccess;
        ok = ok && cudaStreamSynchronize(g->comm_stream) == cudaSuccess;
        ok = ok && cudaMemcpy(all.data(), dbuf + hb, hb * (size_t)world, cudaMemcpyDeviceToHost) == cudaSuccess;
        if (dbuf) cudaFree(dbuf);
        std::vector<double*> px((size_t)world, nullptr);
        std::vector<unsigned int*> pf((size_t)world, nullptr);
        for (int32_t r = 0; r < world && ok; ++r) {
          if (r == rank) {
            px[(size_t)r] = g->xrecv;
            pf[(size_t)r] = g->d_flag;
            continue;
          }
          void* a = nullptr;
          void* b = nullptr;
          ok = cudaIpcOpenMemHandle(&a, all[2 * (size_t)r], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
          if (ok) g->ipc_opened.push_back(a);
          ok = ok && cudaIpcOpenMemHandle(&b, all[2 * (size_t)r + 1], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
          if (ok) g->ipc_opened.push_back(b);
          px[(size_t)r] = (double*)a;
          pf[(size_t)r] = (unsigned int*)b;
        }
        // every rank must agree, or the ranks would disagree on the exchange protocol
        int flag_ok = ok ? 1 : 0, *dflag = nullptr;
        int all_ok = 0;
        if (cudaMalloc((void**)&dflag, sizeof(int)) == cudaSuccess &&
            cudaMemcpy(dflag, &flag_ok, sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess &&
            ncclAllReduce(dflag, dflag, 1, ncclInt, ncclMin, g->comm, g->comm_stream) == ncclSuccess &&
            cudaStreamSynchronize(g->comm_stream) == cudaSuccess &&
            cudaMemcpy(&all_ok, dflag, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess) {
        }
        if (dflag) cudaFree(dflag);
        cudaGetLastError();  // clear a failed IPC call's sticky-free error state
        if (all_ok) {
          if ((e = cudaMemcpy(g->d_peer_x, px.data(), sizeof(double*) * (size_t)world, cudaMemcpyHostToDevice)) !=
                  cudaSuccess ||
              (e = cudaMemcpy(g->d_peer_flag, pf.data(), sizeof(unsigned int*) * (size_t)world,
                              cudaMemcpyHostToDevice)) != cudaSuccess)
            return bail(e, "peer pointers");
          g->peer_on = true;
        }
      }
    }
  }
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return bail(e, "build sync");

  DevPlan& dp = g->dp;
  dp.n = P.n;
  dp.C = P.C;
  dp.rows_per_tile = P.rows_per_tile;
  dp.ntiles = (int32_t)P.tiles.size();
  dp.tile_base = P.tile_begin;
  dp.row_begin = (int32_t)P.row_begin;
  dp.world = world;
  dp.rank = rank;
  dp.rowscale = g->d_rowscale;
  dp.potc = g->d_potc;
  dp.has_parts = 0;
  dp.has_remote = 0;
  for (const TileDesc& T : P.tiles) {
    if (T.nparts > 0) dp.has_parts = 1;
    if (T.nparts > T.nhot && P.split_remote) dp.has_remote = 1;
  }
  if (dp.has_remote) {  // rows without remote entries keep Wr = 0 for good
    if ((e = cudaMalloc((void**)&g->Wr, sizeof(double2) * (size_t)std::max<int64_t>(g->n_local, 1))) != cudaSuccess ||
        (e = cudaMemset(g->Wr, 0, sizeof(double2) * (size_t)std::max<int64_t>(g->n_local, 1))) != cudaSuccess)
      return bail(e, "Wr");
    if ((e = upload(&g->d_rchunks, P.rchunks)) != cudaSuccess) return bail(e, "rchunks");
    if ((e = upload(&g->d_rem_lp, P.rem_lp)) != cudaSuccess) return bail(e, "rem_lp");
  }
  // where a remote part is summed (bitwise the same in every mode): KUR_REMOTE_MODE = 0 the k_remote
  // pass, 1 one warp of the stage kernel with TMA gathers, 2 one warp with LDG gathers
  dp.remote_warp = 0;
  if (dp.has_remote) {
    const char* rm = std::getenv("KUR_REMOTE_MODE");
    if (rm && (rm[0] == '1' || rm[0] == '2' || rm[0] == '3')) dp.remote_warp = rm[0] - '0';
  }
  // inline remote parts that are a large share of the tile's LSU work (one L1 wavefront per random
  // gather against 1/8 per staged hot entry; config 3: 4.3 M remote slots against 14.3 M hot ones)
  // run concurrently with the hot windows on half the warps; small tiles only (shared Wc)
  dp.cr_hot_warps = 0;
  if (!dp.has_remote && P.n_slots_remote > 0 && P.rows_per_tile <= 512 &&
      2 * P.n_slots_remote * 8 >= P.n_slots_hot)
    dp.cr_hot_warps = NWARPS / 2;
  if (const char* cr = std::getenv("KUR_CONC_REMOTE")) dp.cr_hot_warps = std::atoi(cr);  // (A/B: 0 off, k hot warps)
  if (dp.cr_hot_warps < 0 || dp.cr_hot_warps >= NWARPS || P.rows_per_tile > MAX_TILE_ROWS) dp.cr_hot_warps = 0;
  dp.tmaps = nullptr;
  dp.zbuf[0] = g->zA;
  dp.zbuf[1] = g->zB;
  if (dp.remote_warp == 3) {  // tensor maps for tile::gather4: 16-byte rows of z, box of one row
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q) != cudaSuccess || !enc)
      return bail(cudaErrorNotSupported, "cuTensorMapEncodeTiled");
    const double2* bufs[2] = {g->zA, g->zB};
    for (int i = 0; i < 2; ++i) {
      cuuint64_t gdim[2] = {2, (cuuint64_t)g->n_pad};
      cuuint64_t gstr[1] = {sizeof(double2)};
      cuuint32_t box[2] = {2, 1}, es[2] = {1, 1};
      if (enc(&g->tmaps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)bufs[i], gdim, gstr, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return bail(cudaErrorInvalidValue, "cuTensorMapEncodeTiled (z)");
    }
    dp.tmaps = g->tmaps;
  }
  dp.n_local = g->n_local;
  // world 1, opt-in (KUR_PDL=1): programmatic dependent launches between the stage kernels.  Measured
  // (profiles/r02/notes/pdl_ab.log): no gain on configs 3/4, config 5 4.41 -> 5.17 ms per RK4 step
  // (the early-resident k_remote / k_stage CTAs of the next stage only wait), so off by default.
  dp.pdl = (world == 1 && std::getenv("KUR_PDL") != nullptr) ? 1 : 0;
  {
    // world 1: k_stage overlaps the tail of the k_remote pass (programmatic dependent launch, waiting for
    // it only before the finalize); KUR_REMOTE_OVERLAP = k_remote CTAs per SM meanwhile (default 3, the
    // pass's own occupancy; 0 = off).  Config 5 892.6 -> 897.6 RHS/s, config 3 (which then takes the
    // pass) 29.05 K -> 29.7 K (profiles/r02/notes/remote_overlap_pdl_ab.log)
    const char* ro = std::getenv("KUR_REMOTE_OVERLAP");
    dp.rov = world == 1 ? (ro ? std::max(0, std::min(3, std::atoi(ro))) : 3) : 0;
  }
  dp.Wr = g->Wr;
  dp.peer_x = g->peer_on ? g->d_peer_x : nullptr;
  dp.peer_flag = g->d_peer_flag;
  dp.xticket = g->d_xticket;
  dp.rchunks = g->d_rchunks;
  dp.rem_lp = g->d_rem_lp;
  dp.n_rchunks = (int32_t)(P.rem_lp.size());
  // tiny graphs run a whole trajectory in one CTA (launch latency dominates otherwise)
  g->small = P.small;
  {
    std::vector<int32_t> big;
    for (int32_t c = 0; c < P.C; ++c)
      if (P.comm_tile0[(size_t)c + 1] - P.comm_tile0[(size_t)c] > 64) big.push_back(c);
    if ((e = upload(&g->d_big, big)) != cudaSuccess) return bail(e, "big communities");
    dp.big_comm = g->d_big;
    dp.n_big = (int32_t)big.size();
  }
  // deferred block sums: world 1 and no block-reduced community (lazy_T_warp sums S_b sequentially);
  // KUR_LAZY_T=0 keeps the last-CTA reduction after every stage (A/B switch)
  {
    const char* lz = std::getenv("KUR_LAZY_T");
    g->lazy_ok = world == 1 && dp.n_big == 0 && !(lz && lz[0] == '0');
    const char* lr = std::getenv("KUR_LAZY_REC");
    g->lazy_rec_ok = !(lr && lr[0] == '0');
  }
  dp.shard_row0 = g->d_shard_row0;
  dp.shard_tile0 = g->d_shard_tile0;
  dp.xrows = xrows;
  dp.xstride = xstride;
  dp.tiles = g->d_tiles;
  dp.order = g->d_order;
  dp.parts = g->d_parts;
  dp.chunks = g->d_chunks;
  dp.pool = g->d_pool;
  dp.comm_tile0 = g->d_comm_tile0;
  dp.D_ptr = g->d_D_ptr;
  dp.D_idx = g->d_D_idx;
  dp.comm_size = g->d_csize;
  dp.perm = g->d_perm;
  dp.partial = g->partial;
  dp.pmax = g->pmax;
  dp.S = g->S;
  dp.ctrl = g->ctrl;
  // entry-free plans (world 1, beyond the single-CTA size): RK4 trajectories in one cooperative launch
  if (!g->small && persist_fits(dp)) {
    if ((e = cudaMalloc((void**)&g->pbuf, sizeof(double2) * 2 * (size_t)dp.ntiles)) != cudaSuccess ||
        (e = cudaMalloc((void**)&g->gbar, sizeof(unsigned long long))) != cudaSuccess ||
        (e = cudaMemset(g->gbar, 0, sizeof(unsigned long long))) != cudaSuccess)
      return bail(e, "persistent trajectory buffers");
    g->persist = std::getenv("KUR_NO_PERSIST") == nullptr;  // (A/B switch)
  }

  kur_graph_info_t& I = g->info;
  I.n = P.n;
  I.n_comm = P.C;
  I.rank = rank;
  I.world = world;
  I.device = device;
  I.rows_per_tile = P.rows_per_tile;
  I.n_window_loads = P.n_window_loads;
  I.row_begin = P.row_begin;
  I.row_end = P.row_end;
  I.nnz = P.nnz;
  I.n_idx_hot = P.n_idx_hot;
  I.n_idx_remote = P.n_idx_remote;
  I.n_idx = P.n_idx_hot + P.n_idx_remote;
  I.n_slots_hot = P.n_slots_hot;
  I.n_slots_remote = P.n_slots_remote;
  I.n_dense_blocks = P.n_dense_blocks;
  I.n_sparse_blocks = P.n_sparse_blocks;
  I.n_tiles = (int64_t)P.tiles.size();
  I.n_hot_parts = P.n_hot_parts;
  I.sincos_per_rhs = g->n_local;
  // algorithmic bytes of one fused RK stage (= one RHS evaluation), DESIGN.md §5:
  // index stream (13 bits per hot entry, 4 B per remote entry, no padding) plus per
  // local row z_in 16 + z_out 16 + omega 8 + theta_n 8 + acc 16 = 64 B.
  I.bytes_per_rhs = (13 * P.n_idx_hot + 7) / 8 + 4 * P.n_idx_remote + 64 * g->n_local;
  I.bytes_pool = pool_bytes;
  I.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  I.remote_pass = dp.has_remote;
  I.peer_exchange = g->peer_on ? 1 : 0;
  *out = g;
  return KUR_OK;
}

kur_status kur_graph_destroy(kur_graph* g) {
  if (!g) return fail(KUR_ERR_INVALID_ARG, "graph is NULL");
  delete g;
  return KUR_OK;
}

kur_status kur_graph_info(const kur_graph* g, kur_graph_info_t* info) {
  if (!g || !info) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  *info = g->info;
  return KUR_OK;
}

kur_status kur_graph_permutation(const kur_graph* g, int32_t* perm) {
  if (!g || !perm) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  std::memcpy(perm, g->perm_host.data(), sizeof(int32_t) * g->perm_host.size());
  return KUR_OK;
}

kur_status kur_permute(const kur_graph* g, const double* in, double* out, int32_t dir, void* stream) {
  if (!g || !in || !out) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  if (in == out) return fail(KUR_ERR_INVALID_ARG, "in and out must differ");
  if (dir != KUR_USER_TO_INTERNAL && dir != KUR_INTERNAL_TO_USER) return fail(KUR_ERR_INVALID_ARG, "bad dir");
  KUR_CUDA(cudaSetDevice(g->device));
  KUR_CUDA(launch_permute(g->d_perm, g->n, in, out, dir, (cudaStream_t)stream));
  return KUR_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- orchestration
// One "phase" = k_prologue or one k_stage over every rank in `gs`.  With
// world > 1 the fused kernel packs [stage theta | tile partials] into xsend;
// the packed buffers are all-gathered (NCCL across processes, or device copies
// when all ranks live in this process: kur_group_*), then k_unpack fills z of
// the remote rows and all partials and k_finish forms S_b, T_a, (r, psi) in the
// same fixed order on every rank (bitwise identical for any world size).
namespace {

struct RankIO {
  double* theta;
  const double* omega;
  double* out;      // dtheta (RHS)
  double* op_rpsi;  // order parameter outputs
  double* op_local;
  double* v_out;    // kur_potential output
};

kur_status exchange(const std::vector<kur_graph*>& gs, cudaStream_t s) {
  kur_graph* g0 = gs[0];
  if (g0->world == 1) return KUR_OK;
  if (g0->comm) {
    ncclResult_t r = ncclAllGather(g0->xsend, g0->xrecv, (size_t)g0->dp.xstride, ncclDouble, g0->comm, s);
    if (r != ncclSuccess) return fail(KUR_ERR_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(r));
    return KUR_OK;
  }
  if ((int)gs.size() != g0->world)
    return fail(KUR_ERR_UNSUPPORTED, "this handle has world > 1 without NCCL: use the kur_group_* calls");
  const size_t bytes = sizeof(double) * (size_t)g0->dp.xstride;
  for (kur_graph* dst : gs)
    for (kur_graph* src : gs)
      KUR_CUDA(cudaMemcpyAsync(dst->xrecv + (size_t)src->dp.rank * g0->dp.xstride, src->xsend, bytes,
                               cudaMemcpyDeviceToDevice, s));
  return KUR_OK;
}

enum { PH_PROLOGUE = -1 };

// mode: PH_PROLOGUE or a StageMode.  zin/zout/Tin/Tout select the ping-pong buffers.
// commit (prologue only): theta = acc first (implicit midpoint step completion).
// NVTX range per phase (a stage = one RHS evaluation), visible in nsys/ncu timelines; free without a tool
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
const char* phase_name(int mode) {
  static const char* names[] = {"kur rhs", "kur RK4 S1", "kur RK4 S2", "kur RK4 S3", "kur RK4 S4", "kur potential",
                                "kur Euler", "kur Heun H1", "kur Heun H2", "kur midpoint M0", "kur midpoint MI"};
  return mode < 0 ? "kur prologue" : (mode < 11 ? names[mode] : "kur stage");
}

kur_status run_phase(const std::vector<kur_graph*>& gs, int mode, const std::vector<RankIO>& io, double K,
                     double h, int record, bool z_from_A, cudaStream_t s, bool commit = false) {
  NvtxRange nvtx_(phase_name(mode));
  const int world = gs[0]->world;
  std::vector<StageArgs> args(gs.size());
  for (size_t r = 0; r < gs.size(); ++r) {
    kur_graph* g = gs[r];
    StageArgs& a = args[r];
    a = StageArgs{};
    a.theta = io[r].theta;
    a.omega = io[r].omega;
    a.out = io[r].out;
    a.acc = g->acc;
    a.KN = K / (double)g->n;
    a.h = h;
    a.record = record;
    a.op_rpsi = io[r].op_rpsi;
    a.op_local = io[r].op_local;
    a.K = K;
    a.v_out = mode == MODE_POT ? io[r].v_out : nullptr;
    a.xsend = world > 1 ? g->xsend : nullptr;
    a.commit = commit ? g->acc : nullptr;
    a.fp_reset = mode == MODE_M0;
    a.fp_check = mode == MODE_MI;
    if (mode == PH_PROLOGUE) {
      a.zout = g->zA;
      a.Tout = g->TA;
    } else {
      a.zin = z_from_A ? g->zA : g->zB;
      a.zout = z_from_A ? g->zB : g->zA;
      a.Tin = z_from_A ? g->TA : g->TB;
      a.Tout = z_from_A ? g->TB : g->TA;
    }
    a.Wh = g->Wh;
    a.xpar = (int)((g->xepoch + 1) & 1u);  // parity of the exchange this phase produces
    a.theta_host = (mode == MODE_S4 || mode == MODE_E1 || mode == MODE_H2) ? g->host_out : nullptr;
    // deferred block sums (world 1): RK4 S1-S3 and Heun H1 leave the reduction to the next stage,
    // which reads their partials; the destination alternates so no stage overwrites what it reads
    // RK4 S4 of a step that is not the call's last defers its reduction AND its step record: the next
    // S1's last CTA runs the reduction (finish_reduce on S4's partials: r(t), ctrl->rpsi, the step
    // counter) while the other CTAs form their T lazily
    if (mode == PH_PROLOGUE || !g->lazy_ok) {
      g->lazy_prev = nullptr;
      g->rec_pending = false;
    } else {
      const bool s4_defer = mode == MODE_S4 && record == REC_STEP && g->defer_rec_ok && !g->host_out;
      const bool defer = s4_defer || (record == REC_NONE && (mode == MODE_S1 || mode == MODE_S2 ||
                                                             mode == MODE_S3 || mode == MODE_H1));
      const bool takes = mode == MODE_S1 || mode == MODE_S2 || mode == MODE_S3 || mode == MODE_S4 ||
                         mode == MODE_H2;
      a.plazy = takes ? g->lazy_prev : nullptr;
      a.lazy_rec = (a.plazy && g->rec_pending) ? 1 : 0;
      if (defer || a.plazy) a.pout = a.plazy == g->partialB ? g->partial : g->partialB;
      a.no_finish = defer ? 1 : 0;
      g->lazy_prev = defer ? a.pout : nullptr;
      g->rec_pending = s4_defer;
    }
  }
  if (world > 1 && mode != PH_PROLOGUE) {
    // phase A: own-community hot parts (local z only) -> Wh, while the previous stage's
    // exchange may still be running on the exchange stream
    for (size_t r = 0; r < gs.size(); ++r) {
      kur_graph* g = gs[r];
      StageArgs& a = args[r];
      a.phase = PHASE_A;
      KUR_CUDA(g->mark(s));
      KUR_CUDA(launch_stage(mode, g->dp, a, s));
      KUR_CUDA(g->mark(s));
      if (g->timing) g->ev_kind.push_back({3, 0});  // phase A (world > 1)
      a.phase = PHASE_B;
    }
    // the remote pass of this stage needs the other ranks' z of the stage state, which the previous
    // exchange unpacks on the exchange stream: queue it there too, so it runs concurrently with phase A
    // (on the SMs phase A leaves free) instead of between phase A and phase B
    kur_graph* g0 = gs[0];
    if (g0->comm_stream && g0->remote_on_xs) {
      bool pre = false;
      for (size_t r = 0; r < gs.size(); ++r)
        if (gs[r]->dp.has_remote && !gs[r]->dp.remote_warp) {
          KUR_CUDA(gs[r]->mark(g0->comm_stream));
          KUR_CUDA(launch_remote(gs[r]->dp, args[r].zin, g0->comm_stream));
          KUR_CUDA(gs[r]->mark(g0->comm_stream));
          if (gs[r]->timing) gs[r]->ev_kind.push_back({2, 1});
          args[r].no_remote = 1;
          pre = true;
        }
      if (pre) {
        KUR_CUDA(cudaEventRecord(g0->ev_exch, g0->comm_stream));
        g0->exch_pending = true;
      }
    }
    for (kur_graph* g : gs)
      if (g->exch_pending) {  // phase B needs the other ranks' z, the new block sums and Wr
        KUR_CUDA(cudaStreamWaitEvent(s, g->ev_exch, 0));
        g->exch_pending = false;
      }
  }
  for (size_t r = 0; r < gs.size(); ++r) {
    kur_graph* g = gs[r];
    StageArgs& a = args[r];
    // time k_remote apart -- unless k_stage overlaps it (then one event pair spans both: an event between
    // them would serialise the programmatic dependent launch)
    if (g->timing && mode != PH_PROLOGUE && g->dp.has_remote && !g->dp.remote_warp && !a.no_remote && !g->dp.rov) {
      KUR_CUDA(g->mark(s));
      KUR_CUDA(launch_remote(g->dp, a.zin, s));
      KUR_CUDA(g->mark(s));
      g->ev_kind.push_back({2, 1});
      a.no_remote = 1;
    }
    KUR_CUDA(g->mark(s));
    if (mode == PH_PROLOGUE) KUR_CUDA(launch_prologue(g->dp, a, s));
    else KUR_CUDA(launch_stage(mode, g->dp, a, s));
    KUR_CUDA(g->mark(s));
    if (g->timing) g->ev_kind.push_back({mode == PH_PROLOGUE ? 0 : 1, mode == PH_PROLOGUE ? 0 : 1});
  }
  if (world == 1 || mode == MODE_RHS) return KUR_OK;
  kur_graph* g0 = gs[0];
  // The exchange, unpack and fixed-order finish run on the exchange stream (NCCL ranks and in-process
  // groups alike), so the next phase A overlaps them; the prologue (no phase A follows it on its own)
  // is joined at once.
  const bool async = g0->comm_stream != nullptr;
  cudaStream_t xs = async ? g0->comm_stream : s;
  if (async) {
    KUR_CUDA(cudaEventRecord(g0->ev_b, s));
    KUR_CUDA(cudaStreamWaitEvent(xs, g0->ev_b, 0));
  }
  // fused peer-store exchange: the kernels above already stored every record into every rank's
  // receive buffer and counted their arrival; k_unpack waits for the count instead of an all-gather
  if (!g0->peer_on) {
    kur_status st = exchange(gs, xs);
    if (st != KUR_OK) return st;
  }
  for (size_t r = 0; r < gs.size(); ++r) {
    kur_graph* g = gs[r];
    const unsigned int expect = g->peer_on ? (++g->xepoch) * (unsigned int)world : 0u;
    const double* xr = g->xrecv + (g->peer_on ? (size_t)(g->xepoch & 1u) * (size_t)world * g->dp.xstride : 0);
    KUR_CUDA(launch_unpack(g->dp, xr, args[r].zout, expect, xs));
    KUR_CUDA(launch_finish(g->dp, args[r], xs));
  }
  if (async) {
    KUR_CUDA(cudaEventRecord(g0->ev_exch, xs));
    if (mode == PH_PROLOGUE) KUR_CUDA(cudaStreamWaitEvent(s, g0->ev_exch, 0));
    else g0->exch_pending = true;
  }
  return KUR_OK;
}

// The caller's stream waits for an exchange still in flight (end of kur_step and friends).
kur_status join_exchange(const std::vector<kur_graph*>& gs, cudaStream_t s) {
  for (kur_graph* g : gs)
    if (g->exch_pending) {
      KUR_CUDA(cudaStreamWaitEvent(s, g->ev_exch, 0));
      g->exch_pending = false;
    }
  return KUR_OK;
}

kur_status check_group(const std::vector<kur_graph*>& gs) {
  if (gs.empty() || !gs[0]) return fail(KUR_ERR_INVALID_ARG, "graph is NULL");
  for (kur_graph* g : gs)
    if (!g || g->device != gs[0]->device || g->world != gs[0]->world)
      return fail(KUR_ERR_INVALID_ARG, "group handles must share world size and device");
  if (gs.size() > 1) {
    for (size_t r = 0; r < gs.size(); ++r)
      if (gs[r]->dp.rank != (int)r || gs[r]->comm) return fail(KUR_ERR_INVALID_ARG, "group handles must be ranks 0..world-1 without NCCL");
    // in-process fused exchange: link every rank handle to the others' receive buffers and counters
    bool want = true, linked = true;
    for (kur_graph* g : gs) {
      want = want && g->peer_req;
      linked = linked && g->peer_on;
    }
    if (want && !linked) {
      std::vector<double*> px;
      std::vector<unsigned int*> pf;
      for (kur_graph* g : gs) {
        px.push_back(g->xrecv);
        pf.push_back(g->d_flag);
      }
      KUR_CUDA(cudaSetDevice(gs[0]->device));
      for (kur_graph* g : gs) {
        KUR_CUDA(cudaMemcpy(g->d_peer_x, px.data(), sizeof(double*) * px.size(), cudaMemcpyHostToDevice));
        KUR_CUDA(cudaMemcpy(g->d_peer_flag, pf.data(), sizeof(unsigned int*) * pf.size(), cudaMemcpyHostToDevice));
        g->peer_on = true;
        g->dp.peer_x = g->d_peer_x;
        g->info.peer_exchange = 1;
      }
    }
  }
  return KUR_OK;
}

kur_status rhs_impl(const std::vector<kur_graph*>& gs, const std::vector<RankIO>& io, double K, cudaStream_t s) {
  if (!std::isfinite(K)) return fail(KUR_ERR_INVALID_ARG, "K must be finite");
  for (size_t r = 0; r < io.size(); ++r)
    if (gs[r]->n_local > 0 && (!io[r].theta || !io[r].omega || !io[r].out))
      return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  KUR_CUDA(cudaSetDevice(gs[0]->device));
  kur_status st = run_phase(gs, PH_PROLOGUE, io, K, 0.0, REC_NONE, true, s);
  if (st != KUR_OK) return st;
  return run_phase(gs, MODE_RHS, io, K, 0.0, REC_NONE, true, s);
}

kur_status step_impl(const std::vector<kur_graph*>& gs, const std::vector<RankIO>& io, double K, double h,
                     int64_t nsteps, int32_t record_every, const std::vector<double*>& r_trace, cudaStream_t s,
                     int method = KUR_RK4, double fp_tol = 0.0, int32_t fp_max_iter = 0,
                     double* host_out = nullptr) {
  if (method < KUR_RK4 || method > KUR_IMPLICIT_MIDPOINT) return fail(KUR_ERR_INVALID_ARG, "unknown method");
  if (method == KUR_IMPLICIT_MIDPOINT && (!(fp_tol >= 0.0) || !std::isfinite(fp_tol) || fp_max_iter < 1))
    return fail(KUR_ERR_INVALID_ARG, "implicit midpoint needs fp_tol >= 0 (finite) and fp_max_iter >= 1");
  if (!std::isfinite(K)) return fail(KUR_ERR_INVALID_ARG, "K must be finite");
  if (!(h > 0.0) || !std::isfinite(h)) return fail(KUR_ERR_INVALID_ARG, "h must be finite and > 0");
  if (nsteps < 0) return fail(KUR_ERR_INVALID_ARG, "nsteps must be >= 0");
  if (record_every < 0) return fail(KUR_ERR_INVALID_ARG, "record_every must be >= 0");
  for (size_t r = 0; r < io.size(); ++r)
    if (gs[r]->n_local > 0 && (!io[r].theta || !io[r].omega)) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  KUR_CUDA(cudaSetDevice(gs[0]->device));
  for (size_t r = 0; r < gs.size(); ++r) {
    const bool rec = record_every > 0 && r_trace[r];
    const int64_t cap = rec ? nsteps / record_every + 1 : 0;
    KUR_CUDA(launch_set_ctrl(gs[r]->ctrl, rec ? record_every : 0, (int)cap, rec ? r_trace[r] : nullptr, fp_tol, s));
  }
  if (gs.size() == 1 && gs[0]->small && method == KUR_RK4) {  // tiny graph: one single-CTA launch for the whole trajectory
    kur_graph* g = gs[0];
    StageArgs a{};
    a.theta = io[0].theta;
    a.omega = io[0].omega;
    a.acc = g->acc;
    a.KN = K / (double)g->n;
    a.K = K;
    a.h = h;
    KUR_CUDA(g->mark(s));
    KUR_CUDA(launch_small(g->dp, a, g->zA, g->zB, g->TA, g->TB, (long long)nsteps, s));
    KUR_CUDA(g->mark(s));
    if (g->timing) g->ev_kind.push_back({1, (int)std::min<int64_t>(4 * nsteps, INT32_MAX)});
    return KUR_OK;
  }
  NvtxRange nvtx_("kur_step");
  if (gs.size() == 1 && gs[0]->persist && method == KUR_RK4) {  // entry-free plan: one cooperative launch
    kur_graph* g = gs[0];
    StageArgs a{};
    a.theta = io[0].theta;
    a.omega = io[0].omega;
    a.KN = K / (double)g->n;
    a.K = K;
    a.h = h;
    KUR_CUDA(g->mark(s));
    KUR_CUDA(launch_persist_rk4(g->dp, a, g->pbuf, g->gbar, (long long)nsteps, g->persist_q, s));
    g->persist_q += (unsigned long long)(1 + 4 * nsteps);
    KUR_CUDA(g->mark(s));
    if (g->timing) g->ev_kind.push_back({1, (int)std::min<int64_t>(4 * nsteps, INT32_MAX)});
    if (host_out) KUR_CUDA(cudaMemcpyAsync(host_out, io[0].theta, sizeof(double) * (size_t)g->n_local,
                                           cudaMemcpyDefault, s));
    return KUR_OK;
  }
  kur_status st = run_phase(gs, PH_PROLOGUE, io, K, h, REC_START, true, s);
  if (st != KUR_OK) return st;
  // z / T ping-pong: the prologue fills A; every stage reads one buffer and writes the other
  bool from_A = true;
  auto stage = [&](int mode, int record) {
    kur_status r = run_phase(gs, mode, io, K, h, record, from_A, s);
    from_A = !from_A;
    return r;
  };
  for (int64_t n = 0; n < nsteps && st == KUR_OK; ++n) {
    if (host_out && n + 1 == nsteps) gs[0]->host_out = host_out;  // the last step's final stage stores it
    switch (method) {
      case KUR_RK4:
        for (kur_graph* g : gs) g->defer_rec_ok = n + 1 < nsteps && g->lazy_rec_ok;  // the last S4 reduces itself
        for (int m = MODE_S1; m <= MODE_S4 && st == KUR_OK; ++m) st = stage(m, m == MODE_S4 ? REC_STEP : REC_NONE);
        for (kur_graph* g : gs) g->defer_rec_ok = false;
        break;
      case KUR_EULER:
        st = stage(MODE_E1, REC_STEP);
        break;
      case KUR_HEUN:
        st = stage(MODE_H1, REC_NONE);
        if (st == KUR_OK) st = stage(MODE_H2, REC_STEP);
        break;
      default:  // implicit midpoint: predictor, fp_max_iter iterations (no-ops once converged), commit
        st = stage(MODE_M0, REC_NONE);
        for (int32_t it = 0; it < fp_max_iter && st == KUR_OK; ++it) st = stage(MODE_MI, REC_NONE);
        if (st == KUR_OK) st = run_phase(gs, PH_PROLOGUE, io, K, h, REC_STEP, true, s, /*commit=*/true);
        from_A = true;
        break;
    }
  }
  gs[0]->host_out = nullptr;
  if (st == KUR_OK) st = join_exchange(gs, s);
  return st;
}

// kur_step / kur_step_method with theta (and possibly omega) in HOST memory (one handle,
// world 1): theta is copied into the handle's device buffer, the steps run there, and
// theta_{n+1} goes back -- for pinned (page-locked, device-mapped) memory stored by the
// last step's final stage itself through the mapping, so the device-to-host transfer
// overlaps that stage; otherwise (pageable memory, the implicit midpoint commit, the
// single-CTA path) with one copy after the steps.
int mem_kind(const void* p) {  // 0 device / managed, 1 pinned host, 2 pageable host
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return 2;
  }
  if (at.type == cudaMemoryTypeHost) return at.devicePointer ? 1 : 2;
  return at.type == cudaMemoryTypeUnregistered ? 2 : 0;
}

kur_status host_step(kur_graph* g, int method, double* theta, const double* omega, double K, double h,
                     int64_t nsteps, int32_t record_every, double* r_trace, cudaStream_t s, double fp_tol,
                     int32_t fp_max_iter, bool* handled) {
  *handled = false;
  if (g->n_local == 0 || !theta || !omega) return KUR_OK;
  KUR_CUDA(cudaSetDevice(g->device));
  const int kt = mem_kind(theta), ko = mem_kind(omega);
  if (kt == 0 && ko == 0) return KUR_OK;
  *handled = true;
  // world > 1 (NCCL job): every rank passes its own shard (n_local rows) in host memory; the
  // steps are the usual collective (only handles of one process group, not kur_group_*)
  if (g->world > 1 && !g->comm) return fail(KUR_ERR_UNSUPPORTED, "host buffers with world > 1 need an NCCL handle");
  const size_t bytes = sizeof(double) * (size_t)g->n_local;
  double* th = theta;
  if (kt != 0) {
    if (!g->theta_ws && cudaMalloc(&g->theta_ws, bytes) != cudaSuccess) return fail(KUR_ERR_OOM, "theta buffer");
    th = g->theta_ws;
    KUR_CUDA(cudaMemcpyAsync(th, theta, bytes, cudaMemcpyHostToDevice, s));
  }
  const double* om = omega;
  if (ko != 0) {
    if (!g->omega_ws && cudaMalloc(&g->omega_ws, bytes) != cudaSuccess) return fail(KUR_ERR_OOM, "omega buffer");
    KUR_CUDA(cudaMemcpyAsync(g->omega_ws, omega, bytes, cudaMemcpyHostToDevice, s));
    om = g->omega_ws;
  }
  // Stores through the mapping run at ~25 GB/s against ~50 GB/s for the copy engine: they
  // pay only when the final stage outlasts the copy, i.e. when it moves >= 60x the bytes of
  // theta (~3 TB/s vs ~50 GB/s; config 5 673 -> 747 RHS/s end to end, config 2 would lose).
  const bool long_stage = g->info.bytes_per_rhs >= 60 * 8 * g->n_local;
  double* mapped = nullptr;
  if (kt == 1 && long_stage && !g->small && method != KUR_IMPLICIT_MIDPOINT && nsteps > 0) {
    cudaPointerAttributes at{};
    KUR_CUDA(cudaPointerGetAttributes(&at, theta));
    mapped = static_cast<double*>(at.devicePointer);
  }
  std::vector<kur_graph*> gs{g};
  kur_status st = step_impl(gs, {RankIO{th, om, nullptr, nullptr, nullptr}}, K, h, nsteps, record_every, {r_trace},
                            s, method, fp_tol, fp_max_iter, mapped);
  if (st != KUR_OK) return st;
  if (kt != 0 && !mapped && nsteps > 0) KUR_CUDA(cudaMemcpyAsync(theta, th, bytes, cudaMemcpyDeviceToHost, s));
  return KUR_OK;
}

}  // namespace

extern "C" {

kur_status kur_rhs(kur_graph* g, const double* theta, const double* omega, double K, double* dtheta,
                   void* stream) {
  if (!g) return fail(KUR_ERR_INVALID_ARG, "graph is NULL");
  std::vector<kur_graph*> gs{g};
  kur_status st = check_group(gs);
  if (st != KUR_OK) return st;
  return rhs_impl(gs, {RankIO{const_cast<double*>(theta), omega, dtheta, nullptr, nullptr}}, K, (cudaStream_t)stream);
}

kur_status kur_step(kur_graph* g, double* theta, const double* omega, double K, double h, int64_t nsteps,
                    int32_t record_every, double* r_trace, void* stream) {
  if (!g) return fail(KUR_ERR_INVALID_ARG, "graph is NULL");
  std::vector<kur_graph*> gs{g};
  kur_status st = check_group(gs);
  if (st != KUR_OK) return st;
  bool handled;
  st = host_step(g, KUR_RK4, theta, omega, K, h, nsteps, record_every, r_trace, (cudaStream_t)stream, 0.0, 0,
                 &handled);
  if (handled) return st;
  return step_impl(gs, {RankIO{theta, omega, nullptr, nullptr, nullptr}}, K, h, nsteps, record_every, {r_trace},
                   (cudaStream_t)stream);
}

kur_status kur_step_method(kur_graph* g, int32_t method, double* theta, const double* omega, double K, double h,
                           int64_t nsteps, int32_t record_every, double* r_trace, double fp_tol, int32_t fp_max_iter,
                           void* stream) {
  if (!g) return fail(KUR_ERR_INVALID_ARG, "graph is NULL");
  std::vector<kur_graph*> gs{g};
  kur_status st = check_group(gs);
  if (st != KUR_OK) return st;
  if (method < KUR_RK4 || method > KUR_IMPLICIT_MIDPOINT) return fail(KUR_ERR_INVALID_ARG, "unknown method");
  bool handled;
  st = host_step(g, method, theta, omega, K, h, nsteps, record_every, r_trace, (cudaStream_t)stream, fp_tol,
                 fp_max_iter, &handled);
  if (handled) return st;
  return step_impl(gs, {RankIO{theta, omega, nullptr, nullptr, nullptr}}, K, h, nsteps, record_every, {r_trace},
                   (cudaStream_t)stream, method, fp_tol, fp_max_iter);
}

}  // extern "C"

namespace {
// Variable-step RK4 over one handle (world 1), the in-process rank handles of a group, or one
// rank of an NCCL job (collective).  The error estimate's per-tile partials of all ranks are
// summed on the host in global tile order, so every rank (and every world size) takes the
// same accept / step-size decisions.
kur_status adaptive_impl(const std::vector<kur_graph*>& gs, const std::vector<RankIO>& io, double K,
                         const kur_adaptive_ctrl* c, int64_t cap, double* t_out, double* h_out, double* rpsi_out,
                         int64_t* n_accepted, int64_t* n_rejected, cudaStream_t s) {
  if (!c) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  for (size_t r = 0; r < gs.size(); ++r)
    if (gs[r]->n_local > 0 && (!io[r].theta || !io[r].omega)) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  if (!(c->t_end > 0.0) || !std::isfinite(c->t_end) || !(c->h0 > 0.0) || !(c->h_min > 0.0) ||
      !(c->h_max >= c->h_min) || !std::isfinite(c->h_max) || !(c->atol >= 0.0) || !(c->rtol >= 0.0) ||
      !(c->atol + c->rtol > 0.0) || !(c->safety > 0.0) || !(c->fac_min > 0.0) || !(c->fac_min <= 1.0) ||
      !(c->fac_max >= 1.0) || !std::isfinite(c->fac_max) || c->max_trials < 1 || cap < 0)
    return fail(KUR_ERR_INVALID_ARG, "kur_integrate_adaptive: invalid controls");
  if (!std::isfinite(K)) return fail(KUR_ERR_INVALID_ARG, "K must be finite");
  kur_graph* g0 = gs[0];
  const int world = g0->world;
  const bool nccl = g0->comm != nullptr;
  if (world > 1 && !nccl && (int)gs.size() != world)
    return fail(KUR_ERR_UNSUPPORTED, "this handle has world > 1 without NCCL: use kur_group_integrate_adaptive");
  KUR_CUDA(cudaSetDevice(g0->device));
  // per-rank trial buffers (y1, y2) and per-tile error partials, owned by this call; the NCCL
  // case all-gathers the partials padded to the largest rank's tile count
  int32_t xt = 0;
  for (int32_t r = 0; r < world; ++r)
    xt = std::max<int32_t>(xt, g0->shard_tile0_host[(size_t)r + 1] - g0->shard_tile0_host[(size_t)r]);
  xt = std::max(xt, 1);
  std::vector<double*> y1(gs.size(), nullptr), y2(gs.size(), nullptr), tss(gs.size(), nullptr);
  double* gath = nullptr;
  auto cleanup = [&]() {
    for (size_t r = 0; r < gs.size(); ++r) {
      if (y1[r]) cudaFree(y1[r]);
      if (y2[r]) cudaFree(y2[r]);
      if (tss[r]) cudaFree(tss[r]);
    }
    if (gath) cudaFree(gath);
  };
  cudaError_t e = cudaSuccess;
  for (size_t r = 0; r < gs.size() && e == cudaSuccess; ++r) {
    const size_t vb = sizeof(double) * (size_t)std::max<int64_t>(gs[r]->n_local, 1);
    if ((e = cudaMalloc((void**)&y1[r], vb)) == cudaSuccess && (e = cudaMalloc((void**)&y2[r], vb)) == cudaSuccess &&
        (e = cudaMalloc((void**)&tss[r], sizeof(double) * (size_t)xt)) == cudaSuccess)
      e = cudaMemset(tss[r], 0, sizeof(double) * (size_t)xt);
  }
  if (e == cudaSuccess && nccl) e = cudaMalloc((void**)&gath, sizeof(double) * (size_t)xt * (size_t)world);
  if (e != cudaSuccess) {
    cleanup();
    return e == cudaErrorMemoryAllocation ? fail(KUR_ERR_OOM, "kur_integrate_adaptive: out of device memory")
                                          : cuda_fail(e, "kur_integrate_adaptive");
  }
  std::vector<double> hss((size_t)xt * (size_t)world, 0.0);
  std::vector<RankIO> io1(io), io2(io);
  for (size_t r = 0; r < gs.size(); ++r) {
    io1[r].theta = y1[r];
    io2[r].theta = y2[r];
  }
  const std::vector<double*> no_trace(gs.size(), nullptr);
  double t = 0.0, h = c->h0, rpsi[2] = {0.0, 0.0};
  int64_t acc = 0, rej = 0, trials = 0;
  auto run = [&]() -> kur_status {
    while (t < c->t_end) {
      if (trials++ >= c->max_trials) return fail(KUR_ERR_STEPSIZE, "max_trials reached before t_end");
      const bool last = !(t + h < c->t_end - 1e-12 * h);  // the last step lands exactly on t_end
      const double hs = last ? c->t_end - t : h;
      for (size_t r = 0; r < gs.size(); ++r)
        KUR_CUDA(cudaMemcpyAsync(y1[r], io[r].theta, sizeof(double) * (size_t)gs[r]->n_local, cudaMemcpyDeviceToDevice, s));
      kur_status st = step_impl(gs, io1, K, hs, 1, 0, no_trace, s);
      if (st != KUR_OK) return st;
      for (size_t r = 0; r < gs.size(); ++r)
        KUR_CUDA(cudaMemcpyAsync(y2[r], io[r].theta, sizeof(double) * (size_t)gs[r]->n_local, cudaMemcpyDeviceToDevice, s));
      st = step_impl(gs, io2, K, hs / 2.0, 2, 0, no_trace, s);
      if (st != KUR_OK) return st;
      for (size_t r = 0; r < gs.size(); ++r) KUR_CUDA(launch_errnorm(gs[r]->dp, y1[r], y2[r], c->atol, c->rtol, tss[r], s));
      if (nccl) {
        ncclResult_t nr = ncclAllGather(tss[0], gath, (size_t)xt, ncclDouble, g0->comm, s);
        if (nr != ncclSuccess) return fail(KUR_ERR_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(nr));
        KUR_CUDA(cudaMemcpyAsync(hss.data(), gath, sizeof(double) * hss.size(), cudaMemcpyDeviceToHost, s));
      } else {
        for (size_t r = 0; r < gs.size(); ++r)
          KUR_CUDA(cudaMemcpyAsync(hss.data() + r * (size_t)xt, tss[r], sizeof(double) * (size_t)xt,
                                   cudaMemcpyDeviceToHost, s));
      }
      KUR_CUDA(cudaMemcpyAsync(rpsi, g0->ctrl->rpsi, sizeof(rpsi), cudaMemcpyDeviceToHost, s));  // (r, psi) of y2
      KUR_CUDA(cudaStreamSynchronize(s));
      double ss = 0.0;
      for (int32_t r = 0; r < world; ++r) {  // fixed global tile order
        const int32_t ntr = g0->shard_tile0_host[(size_t)r + 1] - g0->shard_tile0_host[(size_t)r];
        for (int32_t k = 0; k < ntr; ++k) ss += hss[(size_t)r * (size_t)xt + (size_t)k];
      }
      const double err = std::sqrt(ss / (double)g0->n) / 15.0;
      if (!std::isfinite(err)) return fail(KUR_ERR_NONFINITE, "non-finite error estimate in kur_integrate_adaptive");
      if (err <= 1.0) {
        for (size_t r = 0; r < gs.size(); ++r)
          KUR_CUDA(cudaMemcpyAsync(io[r].theta, y2[r], sizeof(double) * (size_t)gs[r]->n_local,
                                   cudaMemcpyDeviceToDevice, s));
        t = last ? c->t_end : t + hs;
        if (acc < cap) {
          if (t_out) t_out[acc] = t;
          if (h_out) h_out[acc] = hs;
          if (rpsi_out) {
            rpsi_out[2 * acc] = rpsi[0];
            rpsi_out[2 * acc + 1] = rpsi[1];
          }
        }
        ++acc;
      } else {
        ++rej;
        if (hs <= c->h_min) return fail(KUR_ERR_STEPSIZE, "a step of h_min was rejected");
      }
      double fac = err == 0.0 ? c->fac_max : c->safety * std::pow(err, -0.2);
      fac = std::min(c->fac_max, std::max(c->fac_min, fac));
      h = std::min(c->h_max, std::max(c->h_min, hs * fac));
    }
    return KUR_OK;
  };
  kur_status st = run();
  cudaStreamSynchronize(s);
  cleanup();
  if (n_accepted) *n_accepted = acc;
  if (n_rejected) *n_rejected = rej;
  return st;
}
}  // namespace

extern "C" {

kur_status kur_integrate_adaptive(kur_graph* g, double* theta, const double* omega, double K,
                                  const kur_adaptive_ctrl* c, int64_t cap, double* t_out, double* h_out,
                                  double* rpsi_out, int64_t* n_accepted, int64_t* n_rejected, void* stream) {
  if (!g) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  std::vector<kur_graph*> gs{g};
  kur_status st = check_group(gs);
  if (st != KUR_OK) return st;
  return adaptive_impl(gs, {RankIO{theta, omega, nullptr, nullptr, nullptr}}, K, c, cap, t_out, h_out, rpsi_out,
                       n_accepted, n_rejected, (cudaStream_t)stream);
}

kur_status kur_group_integrate_adaptive(kur_graph* const* g, int32_t world, double* const* theta,
                                        const double* const* omega, double K, const kur_adaptive_ctrl* c,
                                        int64_t cap, double* t_out, double* h_out, double* rpsi_out,
                                        int64_t* n_accepted, int64_t* n_rejected, void* stream) {
  if (!g || !theta || !omega || world < 1) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  std::vector<kur_graph*> gs(g, g + world);
  kur_status st = check_group(gs);
  if (st != KUR_OK) return st;
  std::vector<RankIO> io;
  for (int r = 0; r < world; ++r) io.push_back(RankIO{theta[r], omega[r], nullptr, nullptr, nullptr});
  return adaptive_impl(gs, io, K, c, cap, t_out, h_out, rpsi_out, n_accepted, n_rejected, (cudaStream_t)stream);
}

kur_status kur_order_parameter(kur_graph* g, const double* theta, double* r_psi, double* local, void* stream) {
  if (!g || !theta || !r_psi) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  std::vector<kur_graph*> gs{g};
  kur_status st = check_group(gs);
  if (st != KUR_OK) return st;
  KUR_CUDA(cudaSetDevice(g->device));
  return run_phase(gs, PH_PROLOGUE, {RankIO{const_cast<double*>(theta), nullptr, nullptr, r_psi, local}}, 0.0, 0.0,
                   REC_NONE, true, (cudaStream_t)stream);
}

kur_status kur_potential(kur_graph* g, const double* theta, const double* omega, double K, double* V_out,
                         void* stream) {
  if (!g || !V_out) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  if (g->n_local > 0 && (!theta || !omega)) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  if (!std::isfinite(K)) return fail(KUR_ERR_INVALID_ARG, "K must be finite");
  std::vector<kur_graph*> gs{g};
  kur_status st = check_group(gs);
  if (st != KUR_OK) return st;
  KUR_CUDA(cudaSetDevice(g->device));
  std::vector<RankIO> io{RankIO{const_cast<double*>(theta), omega, nullptr, nullptr, nullptr, V_out}};
  st = run_phase(gs, PH_PROLOGUE, io, K, 0.0, REC_NONE, true, (cudaStream_t)stream);
  if (st != KUR_OK) return st;
  return run_phase(gs, MODE_POT, io, K, 0.0, REC_NONE, true, (cudaStream_t)stream);
}

kur_status kur_group_rhs(kur_graph* const* g, int32_t world, const double* const* theta,
                         const double* const* omega, double K, double* const* dtheta, void* stream) {
  if (!g || !theta || !omega || !dtheta || world < 1) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  std::vector<kur_graph*> gs(g, g + world);
  kur_status st = check_group(gs);
  if (st != KUR_OK) return st;
  std::vector<RankIO> io;
  for (int r = 0; r < world; ++r) io.push_back(RankIO{const_cast<double*>(theta[r]), omega[r], dtheta[r], nullptr, nullptr});
  return rhs_impl(gs, io, K, (cudaStream_t)stream);
}

kur_status kur_group_step(kur_graph* const* g, int32_t world, double* const* theta, const double* const* omega,
                          double K, double h, int64_t nsteps, int32_t record_every, double* const* r_trace,
                          void* stream) {
  if (!g || !theta || !omega || world < 1) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  std::vector<kur_graph*> gs(g, g + world);
  kur_status st = check_group(gs);
  if (st != KUR_OK) return st;
  std::vector<RankIO> io;
  std::vector<double*> rt;
  for (int r = 0; r < world; ++r) {
    io.push_back(RankIO{theta[r], omega[r], nullptr, nullptr, nullptr});
    rt.push_back(r_trace ? r_trace[r] : nullptr);
  }
  return step_impl(gs, io, K, h, nsteps, record_every, rt, (cudaStream_t)stream);
}

kur_status kur_group_step_method(kur_graph* const* g, int32_t world, int32_t method, double* const* theta,
                                 const double* const* omega, double K, double h, int64_t nsteps, int32_t record_every,
                                 double* const* r_trace, double fp_tol, int32_t fp_max_iter, void* stream) {
  if (!g || !theta || !omega || world < 1) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  std::vector<kur_graph*> gs(g, g + world);
  kur_status st = check_group(gs);
  if (st != KUR_OK) return st;
  std::vector<RankIO> io;
  std::vector<double*> rt;
  for (int r = 0; r < world; ++r) {
    io.push_back(RankIO{theta[r], omega[r], nullptr, nullptr, nullptr});
    rt.push_back(r_trace ? r_trace[r] : nullptr);
  }
  return step_impl(gs, io, K, h, nsteps, record_every, rt, (cudaStream_t)stream, method, fp_tol, fp_max_iter);
}

kur_status kur_timing(kur_graph* g, int32_t enable) {
  if (!g) return fail(KUR_ERR_INVALID_ARG, "graph is NULL");
  g->timing = enable != 0;
  g->ev_used = 0;
  g->ev_kind.clear();
  return KUR_OK;
}

kur_status kur_timing_read(kur_graph* g, double* out) {
  if (!g || !out) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  KUR_CUDA(cudaSetDevice(g->device));
  double ms[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t cnt[4] = {0, 0, 0, 0};
  for (size_t i = 0; i < g->ev_kind.size(); ++i) {
    float t = 0.f;
    KUR_CUDA(cudaEventSynchronize(g->ev[2 * i + 1]));
    KUR_CUDA(cudaEventElapsedTime(&t, g->ev[2 * i], g->ev[2 * i + 1]));
    ms[g->ev_kind[i].first] += t;
    cnt[g->ev_kind[i].first] += g->ev_kind[i].first == 0 ? 1 : g->ev_kind[i].second;
  }
  out[0] = ms[0];
  out[1] = (double)cnt[0];
  out[2] = ms[1];
  out[3] = (double)cnt[1];
  out[4] = ms[2];
  out[5] = (double)cnt[2];
  out[6] = (double)g->ev_kind.size();
  out[7] = ms[3];  // world > 1: phase-A k_stage launches (own-community windows), included in out[2]
  out[8] = (double)cnt[3];
  out[2] += ms[3];
  g->ev_used = 0;
  g->ev_kind.clear();
  return KUR_OK;
}

kur_status kur_check(kur_graph* g, void* stream) {
  if (!g) return fail(KUR_ERR_INVALID_ARG, "graph is NULL");
  KUR_CUDA(cudaSetDevice(g->device));
  KUR_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  int xt = 0;
  KUR_CUDA(cudaMemcpy(&xt, &g->ctrl->xtimeout, sizeof(int), cudaMemcpyDeviceToHost));
  if (xt) return fail(KUR_ERR_NCCL, "fused peer exchange: timed out waiting for the other ranks' records");
  int flag = 0;
  KUR_CUDA(cudaMemcpy(&flag, &g->ctrl->nonfinite, sizeof(int), cudaMemcpyDeviceToHost));
  if (flag) {
    const int zero = 0;
    KUR_CUDA(cudaMemcpy(&g->ctrl->nonfinite, &zero, sizeof(int), cudaMemcpyHostToDevice));
    return fail(KUR_ERR_NONFINITE, "kur_step produced a non-finite phase");
  }
  return KUR_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- host-only plan introspection
struct kur_plan {
  HostPlan P;
  mutable int64_t conflicts = 0;  // quarter-warp positions with a repeated bank group (export)
};

extern "C" {

kur_status kur_plan_build(const kur_graph_desc* desc, int32_t rank, int32_t world, int32_t sm_count,
                          kur_plan** out) {
  if (!out) return fail(KUR_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  kur_plan* p = new (std::nothrow) kur_plan();
  if (!p) return fail(KUR_ERR_OOM, "host allocation failed");
  std::string err;
  kur_status st;
  try {
    st = build_plan(desc, rank, world, sm_count > 0 ? sm_count : 148, p->P, err);
  } catch (const std::bad_alloc&) {
    delete p;
    return fail(KUR_ERR_OOM, "host allocation failed in kur_plan_build");
  }
  if (st != KUR_OK) {
    delete p;
    return fail(st, err);
  }
  *out = p;
  return KUR_OK;
}

kur_status kur_plan_sizes(const kur_plan* p, int64_t* sizes) {
  if (!p || !sizes) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  const HostPlan& P = p->P;
  sizes[0] = P.n;
  sizes[1] = P.C;
  sizes[2] = P.row_end - P.row_begin;
  sizes[3] = P.row_begin;
  sizes[4] = P.n_idx_hot + P.n_idx_remote;
  sizes[5] = (int64_t)P.D_idx.size();
  sizes[6] = (int64_t)P.tiles.size();
  sizes[7] = P.rows_per_tile;
  sizes[8] = P.nnz;
  sizes[9] = P.world;
  sizes[10] = p->conflicts;
  sizes[11] = P.n_slots_hot;
  sizes[12] = P.n_idx_hot;
  sizes[13] = P.n_slots_remote;
  sizes[14] = P.n_idx_remote;
  sizes[15] = P.n_window_loads;
  return KUR_OK;
}

kur_status kur_plan_export(const kur_plan* p, int32_t* perm, int32_t* D_ptr, int32_t* D_idx, int64_t* row_ptr,
                           int32_t* cols, int8_t* neg, int32_t* shard_row0) {
  if (!p) return fail(KUR_ERR_INVALID_ARG, "NULL plan");
  const HostPlan& P = p->P;
  p->conflicts = 0;
  if (perm) std::memcpy(perm, P.perm.data(), sizeof(int32_t) * P.perm.size());
  if (D_ptr) std::memcpy(D_ptr, P.D_ptr.data(), sizeof(int32_t) * P.D_ptr.size());
  if (D_idx && !P.D_idx.empty()) std::memcpy(D_idx, P.D_idx.data(), sizeof(int32_t) * P.D_idx.size());
  if (shard_row0) std::memcpy(shard_row0, P.shard_row0.data(), sizeof(int32_t) * P.shard_row0.size());
  if (!row_ptr) return KUR_OK;
  // decode the chunked layout exactly as the kernels read it
  const int64_t nl = P.row_end - P.row_begin;
  struct E { int32_t row, col; int8_t neg; };
  std::vector<E> ents;
  // hot chunk layout (plan.h): cd.ng = (G << 1) | tail; G groups of 9 positions as 13-bit slots
  // packed in 16 bytes per lane, then (tail) 4 positions as 16-bit slots in 8 bytes per lane
  auto hot_npos = [&](const ChunkDesc& cd) -> uint32_t { return 9 * (cd.ng >> 1) + 4 * (cd.ng & 1); };
  auto hot_slot = [&](const ChunkDesc& cd, int l, uint32_t pos) -> uint32_t {
    const uint32_t G = cd.ng >> 1;
    if (pos < 9 * G) {
      const Unit& U = P.pool[(size_t)cd.ofs + HDR_UNITS + (size_t)(pos / 9) * 32 + (size_t)l];
      uint64_t lo, hi;
      std::memcpy(&lo, U.w, 8);
      std::memcpy(&hi, U.w + 2, 8);
      const int off = 13 * (int)(pos % 9);
      uint64_t v;
      if (off + 13 <= 64) v = lo >> off;
      else if (off >= 64) v = hi >> (off - 64);
      else v = (lo >> off) | (hi << (64 - off));
      return (uint32_t)(v & 0x1FFF);
    }
    const uint16_t* t16 = reinterpret_cast<const uint16_t*>(&P.pool[(size_t)cd.ofs + HDR_UNITS + (size_t)G * 32]);
    return t16[(size_t)l * 4 + (pos - 9 * G)];
  };
  for (const TileDesc& T : P.tiles) {
    for (int pi = T.part0; pi < T.part0 + T.nparts; ++pi) {
      const PartDesc& pd = P.parts[(size_t)pi];
      const bool hot = pd.window >= 0;
      if (hot != (pi < T.part0 + T.nhot)) return fail(KUR_ERR_INVALID_ARG, "plan: part order");
      std::vector<uint8_t> seen((size_t)T.nrows, 0);
      const int pcs = 1 << (pd.neg >> 8);  // row pieces per row (aligned lane groups)
      for (uint32_t c = 0; c < pd.nchunks; ++c) {
        const ChunkDesc cd = P.chunks[(size_t)pd.chunk0 + c];
        const uint16_t* hdr = reinterpret_cast<const uint16_t*>(&P.pool[(size_t)cd.ofs]);
        for (int l = 0; l < 32; ++l) {
          const uint16_t lr = hdr[l];
          if (lr != EMPTY_LANE) {
            const bool lead = (l % pcs) == 0;
            if (lr >= T.nrows || (lead && seen[lr]) || (!lead && hdr[l - l % pcs] != lr))
              return fail(KUR_ERR_INVALID_ARG, "plan: bad chunk header");
            seen[lr] = 1;
          }
          // hot: hot_npos positions; remote: cd.ng groups of 4 32-bit columns
          for (uint32_t pos = 0; pos < (hot ? hot_npos(cd) : 4 * cd.ng); ++pos) {
            {
              int64_t col;
              int8_t eneg = (int8_t)(pd.neg & 1);
              if (hot) {
                const uint32_t e = hot_slot(cd, l, pos);
                if (e >= HOT_SENT && e < HOT_SENT + 8) continue;
                if (e > HOT_SENT) return fail(KUR_ERR_INVALID_ARG, "plan: hot index out of window");
                col = (int64_t)pd.window * WZ + e;
              } else {
                const uint32_t e = P.pool[(size_t)cd.ofs + HDR_UNITS + (size_t)(pos / 4) * 32 + (size_t)l].w[pos % 4];
                if (e == (uint32_t)P.n) continue;
                col = e & 0x7FFFFFFFu;  // bit 31: complement entry (subtracted)
                eneg = (int8_t)(e >> 31);
              }
              if (lr == EMPTY_LANE) return fail(KUR_ERR_INVALID_ARG, "plan: entry in an empty lane");
              if (col < 0 || col >= P.n) return fail(KUR_ERR_INVALID_ARG, "plan: column out of range");
              ents.push_back(E{(int32_t)(T.row0 + lr - P.row_begin), (int32_t)col, eneg});
            }
          }
        }
        if (hot) {  // bank-conflict freedom: distinct slot residues per quarter-warp position
          for (uint32_t pos = 0; pos < hot_npos(cd); ++pos)
            for (int qw = 0; qw < 4; ++qw) {
              int mask = 0;
              for (int l = qw * 8; l < qw * 8 + 8; ++l) {
                const uint32_t e = hot_slot(cd, l, pos);
                if (mask >> (e & 7) & 1) p->conflicts++;  // NOLINT
                mask |= 1 << (e & 7);
              }
            }
        }
      }
    }
  }
  std::vector<int64_t> cnt((size_t)nl + 1, 0);
  for (const E& e : ents) cnt[(size_t)e.row + 1]++;
  for (int64_t i = 0; i < nl; ++i) cnt[(size_t)i + 1] += cnt[(size_t)i];
  std::memcpy(row_ptr, cnt.data(), sizeof(int64_t) * (size_t)(nl + 1));
  std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
  for (const E& e : ents) {
    const int64_t at = fill[(size_t)e.row]++;
    if (cols) cols[at] = e.col;
    if (neg) neg[at] = e.neg;
  }
  return KUR_OK;
}

kur_status kur_plan_tiles(const kur_plan* p, int32_t* tiles, int32_t* part_window) {
  if (!p || !tiles) return fail(KUR_ERR_INVALID_ARG, "NULL argument");
  const HostPlan& P = p->P;
  size_t k = 0;
  for (size_t t = 0; t < P.tiles.size(); ++t) {
    const TileDesc& T = P.tiles[t];
    const int32_t v[7] = {T.row0, T.nrows, T.comm, T.nparts, T.nhot, T.nown, T.nloc};
    std::memcpy(tiles + 7 * t, v, sizeof(v));
    if (part_window)
      for (int32_t q = 0; q < T.nparts; ++q) part_window[k++] = P.parts[(size_t)(T.part0 + q)].window;
  }
  return KUR_OK;
}

kur_status kur_plan_destroy(kur_plan* p) {
  delete p;
  return KUR_OK;
}

}  // extern "C"
