// kernels.cu — sm_100a fp64 kernels of the localised-order-parameter RHS and
// the fused integrator stages (product code).
//
// One CTA (16 warps, 512 threads) owns one community-aligned tile of up to
// 2048 rows whose row sums W_j live in shared memory (plan.h describes the
// chunked, bank-conflict-free index layout).
//
//   k_prologue  z = e^{i theta} (= (cos, sin), P:443 / "2M" trig of P:660),
//               per-tile partial sums of z; the last CTA reduces the partials
//               to the block sums S_b, T_a = sum_{b in D(a)} S_b,
//               and the order parameter r e^{i psi} = (1/N) sum_b S_b
//               (P:236-239).
//   k_remote    (remote-pass plans) the remote part of every tile — random
//               global z gathers, signed per entry — one warp per chunk, row
//               sums into Wr.
//   k_stage     W_j = T_{c(j)} - sum_{Z_j} z_k + sum_{NZ_j} z_k:
//               hot parts gather z from a 64 KB shared-memory window
//               (staged by a TMA bulk copy), the remote part inline or from
//               Wr; then k_j = omega_j + (K/N) Im(conj z_j W_j)
//               and, fused, the integrator's stage update (RK4 / Euler / Heun
//               / implicit midpoint), the next stage's z and its per-tile
//               partials; the last CTA forms the next S_b, T_a and (r, psi)
//               exactly as k_prologue does.  world > 1: phase A (own-community
//               windows) / phase B, records packed for the exchange or stored
//               straight into the peers' receive buffers.
// All reductions are fixed-shape (no floating-point atomics): bitwise
// reproducible run to run and across world sizes.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <utility>

#include "kernels.h"

namespace kur {
// Debug build only (make debug -> libkur_debug.so, tests via KUR_LIB): device-side bounds checks
// on every index the layout feeds the kernels (compute-sanitizer is not available on this pool).
#ifdef KUR_DEBUG_BOUNDS
#define KUR_ASSERT(c) do { if (!(c)) { printf("KUR_ASSERT %s:%d %s\n", __FILE__, __LINE__, #c); __trap(); } } while (0)
__device__ uint32_t g_dbg_zlen = 0xFFFFFFFFu;  // entries of the z buffers (set by the launchers)
#else
#define KUR_ASSERT(c) do {} while (0)
#endif
#ifdef KUR_PROFILE
// Tooling build only (make prof): per-tile clock64 stamps of k_stage phases.
__device__ unsigned long long* g_prof = nullptr;
constexpr int PROF_STRIDE = 192;  // [0] start, [1+3p..] window wait begin/end + part end, [25] finalize, [26] end,
                                  // [32 + 16p + w] warp w done with part p (p < 8)
#define PROF_T(i) \
  do { if (g_prof && threadIdx.x == 0) g_prof[(size_t)blockIdx.x * PROF_STRIDE + (i)] = clock64(); } while (0)
#define PROF_W(p, w) \
  do { if (g_prof && (threadIdx.x & 31) == 0 && (p) < 8) g_prof[(size_t)blockIdx.x * PROF_STRIDE + 32 + 16 * (p) + (w)] = clock64(); } while (0)
// global-timer stamps (ns, comparable across SMs): [160] CTA start, [161] tile done, [162] last CTA: finish done
__device__ __forceinline__ unsigned long long prof_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PROF_G(i) \
  do { if (g_prof && threadIdx.x == 0) g_prof[(size_t)blockIdx.x * PROF_STRIDE + (i)] = prof_gtime(); } while (0)
#else
#define PROF_T(i) do {} while (0)
#define PROF_W(p, w) do {} while (0)
#define PROF_G(i) do {} while (0)
#endif
namespace {

// Index stream: read once per RHS, never reused within it -> do not allocate
// in L1 and evict first from L2 (keeps z L2-resident for the remote gathers).
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint4 ldg_stream(const uint4* p, uint64_t pol) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ uint2 ldg_stream2(const uint2* p, uint64_t pol) {
  uint2 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
      : "=r"(r.x), "=r"(r.y)
      : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}

// One thread: TMA bulk copy of `bytes` from global to shared memory, completion on `bar`.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
  // evict-first: a window is dead once its community's tiles have staged it; z_out (stored by this
  // kernel, gathered by the next k_remote) keeps the L2.  Measured alternative (config 5,
  // profiles/r02/notes/window_policy_ab.log, r2k_ab.log): evict-normal with the tiles of a community
  // launched together re-reads windows from L2 -- k_stage DRAM reads 3.31 -> 2.90 GB per launch --
  // but the stage got 0.5 % slower (k_stage is bound by the L1/LSU pipe, not DRAM).  Compile-time:
  // a runtime switch between policies here cost k_stage 2 % (notes/window_policy_branch_cost.log).
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}

// Programmatic dependent launch (world 1 stage sequence): the next kernel of the stream is launched
// while this one runs; its CTAs wait here until the previous grid has completed and flushed, so the
// launch latency and the previous grid's tail overlap.  No-ops for a normal launch.
__device__ __forceinline__ void pdl_wait_and_release() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void warp_sum2(double& x, double& y) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    x += __shfl_xor_sync(0xffffffffu, x, o);
    y += __shfl_xor_sync(0xffffffffu, y, o);
  }
}

// Fixed-shape block reduction of (x, y) over NTHREADS threads; result valid in warp 0.
__device__ __forceinline__ void block_sum2(double& x, double& y, double2* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_sum2(x, y);
  if (lane == 0) red[warp] = make_double2(x, y);
  __syncthreads();
  if (warp == 0) {
    const double2 v = lane < NWARPS ? red[lane] : make_double2(0.0, 0.0);
    x = v.x;
    y = v.y;
#pragma unroll
    for (int o = NWARPS / 2; o > 0; o >>= 1) {
      x += __shfl_xor_sync(0xffffffffu, x, o);
      y += __shfl_xor_sync(0xffffffffu, y, o);
    }
  }
}

// Fixed-shape block maximum over NTHREADS threads; result valid in warp 0.
__device__ __forceinline__ double block_max(double d, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
  if (lane == 0) red[warp] = d;
  __syncthreads();
  if (warp == 0) {
    d = lane < NWARPS ? red[lane] : 0.0;
#pragma unroll
    for (int o = NWARPS / 2; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
  }
  return d;
}

// a4: k_j = omega_j + (K/M_j)(cos th_j Im W_j - sin th_j Re W_j), with explicit roundings:
// every kernel evaluates it through this one expression, so the per-row arithmetic is bitwise the
// same in all of them whatever the compiler would contract.
__device__ __forceinline__ double rhs_k(double om, double kn, double zx, double zy, double wx, double wy) {
  return __fma_rn(kn, __fma_rn(zx, wy, -__dmul_rn(zy, wx)), om);
}

// Sum of the 9 window-local z entries named by one 16-byte unit of 13-bit slots
// (complement or non-zero entries; the part's sign is applied by the
// caller).  Slot e sits at bits 13e..13e+12 of the 128-bit unit; each field is
// extracted directly as a byte offset (slot * 16) into the window.
__device__ __forceinline__ void hot9(const uint4 v, const double2* zs, double& x0, double& y0,
                                     double& x1, double& y1) {
  constexpr uint32_t M = 0x1FFF0u;
  const uint32_t o[9] = {(v.x << 4) & M,
                         (v.x >> 9) & M,
                         __funnelshift_r(v.x, v.y, 22) & M,
                         (v.y >> 3) & M,
                         __funnelshift_r(v.y, v.z, 16) & M,
                         (v.z << 3) & M,
                         (v.z >> 10) & M,
                         __funnelshift_r(v.z, v.w, 23) & M,
                         (v.w >> 4) & M};
  const char* zb = reinterpret_cast<const char*>(zs);
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    KUR_ASSERT((o[e] >> 4) < WZ + 8);
    const double2 a = *reinterpret_cast<const double2*>(zb + o[e]);
    if (e & 1) {
      x1 += a.x;
      y1 += a.y;
    } else {
      x0 += a.x;
      y0 += a.y;
    }
  }
}

// The 4 window-local z entries of a trailing half-group unit (8 bytes).
__device__ __forceinline__ void hot4(const uint2 v, const double2* zs, double& x0, double& y0, double& x1,
                                     double& y1) {
  const double2 a = zs[v.x & 0xFFFFu];
  const double2 b = zs[v.x >> 16];
  const double2 c = zs[v.y & 0xFFFFu];
  const double2 d = zs[v.y >> 16];
  x0 += a.x;
  y0 += a.y;
  x1 += b.x;
  y1 += b.y;
  x0 += c.x;
  y0 += c.y;
  x1 += d.x;
  y1 += d.y;
}

// COHERENT: z was written earlier by the same kernel (single-CTA trajectory
// kernel) -> read through L2 (ld.global.cg) instead of the non-coherent path.
template <bool COHERENT>
__device__ __forceinline__ double2 ldz(const double2* p) {
  return COHERENT ? __ldcg(p) : __ldg(p);
}

// Remote entry id: column in bits 0-30, bit 31 set for a complement entry (subtracted,
// P:562-570), clear for a non-zero entry (added).  Negation is exact.
template <bool COHERENT>
__device__ __forceinline__ double2 ldz_signed(const double2* __restrict__ z, uint32_t id) {
#ifdef KUR_DEBUG_BOUNDS
  KUR_ASSERT((id & 0x7FFFFFFFu) < g_dbg_zlen);
#endif
  const double2 v = ldz<COHERENT>(z + (id & 0x7FFFFFFFu));
  return (id >> 31) ? make_double2(-v.x, -v.y) : v;
}

template <bool COHERENT>
__device__ __forceinline__ void rem4(const uint4 v, const double2* __restrict__ z, double& x0,
                                     double& y0, double& x1, double& y1) {
  const double2 a = ldz_signed<COHERENT>(z, v.x);
  const double2 b = ldz_signed<COHERENT>(z, v.y);
  const double2 c = ldz_signed<COHERENT>(z, v.z);
  const double2 d = ldz_signed<COHERENT>(z, v.w);
  x0 += a.x;
  y0 += a.y;
  x1 += b.x;
  y1 += b.y;
  x0 += c.x;
  y0 += c.y;
  x1 += d.x;
  y1 += d.y;
}

// Hot part of one chunk starting at base (the chunk's first group, no lane
// offset), H = (G << 1) | tail: G full groups of 32 16-byte units (9 13-bit slots
// per lane), then one trailing group of 32 8-byte units (4 16-bit slots per
// lane) when tail is set.  Rotating software
// pipeline: the unit of group g+4 is requested before group g is gathered, so
// four 16-byte index loads per lane are always in flight and there is no serial
// tail (loads past the last group are predicated off).
__device__ __forceinline__ void run_hot(const uint4* __restrict__ base, uint32_t H, int lane, const double2* zs,
                                        uint64_t pol, double& sx, double& sy) {
  const uint32_t ng = H >> 1;
  const uint4* q = base + lane;
  const uint2 tail = (H & 1u) ? ldg_stream2(reinterpret_cast<const uint2*>(base + (size_t)ng * 32) + lane, pol)
                              : make_uint2(0, 0);
  double x0 = 0.0, y0 = 0.0, x1 = 0.0, y1 = 0.0;
  const uint4 z4 = make_uint4(0, 0, 0, 0);
  uint4 b0 = ng > 0 ? ldg_stream(q, pol) : z4;
  uint4 b1 = ng > 1 ? ldg_stream(q + 32, pol) : z4;
  uint4 b2 = ng > 2 ? ldg_stream(q + 64, pol) : z4;
  uint4 b3 = ng > 3 ? ldg_stream(q + 96, pol) : z4;
  for (uint32_t g = 0; g < ng; g += 4) {
    const uint4* qn = q + (size_t)(g + 4) * 32;
    uint4 c = b0;
    if (g + 4 < ng) b0 = ldg_stream(qn, pol);
    hot9(c, zs, x0, y0, x1, y1);
    if (g + 1 >= ng) break;
    c = b1;
    if (g + 5 < ng) b1 = ldg_stream(qn + 32, pol);
    hot9(c, zs, x0, y0, x1, y1);
    if (g + 2 >= ng) break;
    c = b2;
    if (g + 6 < ng) b2 = ldg_stream(qn + 64, pol);
    hot9(c, zs, x0, y0, x1, y1);
    if (g + 3 >= ng) break;
    c = b3;
    if (g + 7 < ng) b3 = ldg_stream(qn + 96, pol);
    hot9(c, zs, x0, y0, x1, y1);
  }
  if (H & 1u) hot4(tail, zs, x0, y0, x1, y1);
  sx = x0 + x1;
  sy = y0 + y1;
}

// Remote part of one chunk: the index units run two groups ahead of the z gathers.
template <bool COHERENT>
__device__ __forceinline__ void run_remote(const uint4* __restrict__ q, uint32_t ng,
                                           const double2* __restrict__ z, uint64_t pol, double& sx, double& sy) {
  double x0 = 0.0, y0 = 0.0, x1 = 0.0, y1 = 0.0;
  const uint4 z4 = make_uint4(0, 0, 0, 0);
  uint4 b0 = ng > 0 ? ldg_stream(q, pol) : z4;
  uint4 b1 = ng > 1 ? ldg_stream(q + 32, pol) : z4;
  for (uint32_t g = 0; g < ng; g += 2) {
    const uint4* qn = q + (size_t)(g + 2) * 32;
    uint4 c = b0;
    if (g + 2 < ng) b0 = ldg_stream(qn, pol);
    rem4<COHERENT>(c, z, x0, y0, x1, y1);
    if (g + 1 >= ng) break;
    c = b1;
    if (g + 3 < ng) b1 = ldg_stream(qn + 32, pol);
    rem4<COHERENT>(c, z, x0, y0, x1, y1);
  }
  sx = x0 + x1;
  sy = y0 + y1;
}

// k_remote's loop: as run_remote, but two groups (8 z gathers per lane) in
// flight at once; missing groups read the zero sentinel z[sent] (sent = n).
// b0, b1: the chunk's first two index units, already requested by the caller.
__device__ __forceinline__ void run_remote_deep_pre(const uint4* __restrict__ q, uint32_t ng, uint32_t sent,
                                                    const double2* __restrict__ z, uint64_t pol, uint4 b0, uint4 b1,
                                                    double& sx, double& sy) {
  double x0 = 0.0, y0 = 0.0, x1 = 0.0, y1 = 0.0;
  const uint4 s4 = make_uint4(sent, sent, sent, sent);
  for (uint32_t g = 0; g < ng; g += 2) {
    const uint4 c0 = b0, c1 = b1;
    const uint4* qn = q + (size_t)(g + 2) * 32;
    b0 = g + 2 < ng ? ldg_stream(qn, pol) : s4;
    b1 = g + 3 < ng ? ldg_stream(qn + 32, pol) : s4;
    const double2 a0 = ldz_signed<false>(z, c0.x), a1 = ldz_signed<false>(z, c0.y);
    const double2 a2 = ldz_signed<false>(z, c0.z), a3 = ldz_signed<false>(z, c0.w);
    const double2 a4 = ldz_signed<false>(z, c1.x), a5 = ldz_signed<false>(z, c1.y);
    const double2 a6 = ldz_signed<false>(z, c1.z), a7 = ldz_signed<false>(z, c1.w);
    x0 += a0.x; y0 += a0.y; x1 += a1.x; y1 += a1.y;
    x0 += a2.x; y0 += a2.y; x1 += a3.x; y1 += a3.y;
    x0 += a4.x; y0 += a4.y; x1 += a5.x; y1 += a5.y;
    x0 += a6.x; y0 += a6.y; x1 += a7.x; y1 += a7.y;
  }
  sx = x0 + x1;
  sy = y0 + y1;
}

__device__ __forceinline__ void run_remote_deep(const uint4* __restrict__ q, uint32_t ng, uint32_t sent,
                                                const double2* __restrict__ z, uint64_t pol, double& sx, double& sy) {
  const uint4 s4 = make_uint4(sent, sent, sent, sent);
  const uint4 b0 = ng > 0 ? ldg_stream(q, pol) : s4;
  const uint4 b1 = ng > 1 ? ldg_stream(q + 32, pol) : s4;
  run_remote_deep_pre(q, ng, sent, z, pol, b0, b1, sx, sy);
}

// The chunks of one part (P:562-570 complement entries subtracted, P:538-542
// non-zero entries added into the tile's row sums Ws), snake order over the
// NWARPS warps (chunks are sorted longest first); the next chunk's descriptor
// is requested before the current chunk is gathered.  Hot parts gather from the
// staged window zs, remote parts from global z.
template <bool COHERENT, bool DEEP = false>
__device__ __forceinline__ void run_part(const DevPlan& dp, const PartDesc& P, bool hot, const double2* zs,
                                         const double2* __restrict__ z, double2* Ws, uint64_t pol, int warp,
                                         int lane, uint32_t nw = NWARPS) {
    uint32_t c = warp;
    uint2 cdn = c < P.nchunks ? __ldg(dp.chunks + P.chunk0 + c) : make_uint2(0, 0);
    for (uint32_t r = 0; c < P.nchunks; ++r) {
      const uint2 cd = cdn;
      const uint32_t cnext = (r + 1) * nw + (((r + 1) & 1) ? (nw - 1 - warp) : warp);
      if (cnext < P.nchunks) cdn = __ldg(dp.chunks + P.chunk0 + cnext);
      const uint4* q = dp.pool + cd.x;
      const uint16_t row = reinterpret_cast<const uint16_t*>(q)[lane];
      double sx, sy;
      if (hot) run_hot(q + HDR_UNITS, cd.y, lane, zs, pol, sx, sy);
      else if (DEEP) run_remote_deep(q + HDR_UNITS + lane, cd.y, (uint32_t)dp.n, z, pol, sx, sy);
      else run_remote<COHERENT>(q + HDR_UNITS + lane, cd.y, z, pol, sx, sy);
      const int lp = P.neg >> 8;  // row pieces: 2^lp consecutive lanes hold one row
      for (int o = 1; o < (1 << lp); o <<= 1) {
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
      }
      if (row != EMPTY_LANE && (lane & ((1 << lp) - 1)) == 0) {
        KUR_ASSERT(row < dp.rows_per_tile);
        double2 w = Ws[row];
        if (P.neg & 1) {
          w.x -= sx;
          w.y -= sy;
        } else {
          w.x += sx;
          w.y += sy;
        }
        Ws[row] = w;
      }
      c = cnext;
    }
}

// ---- the remote part of one tile summed by ONE warp of the tile's CTA (dp.remote_warp), while
// the other warps gather the hot windows from shared memory: W_r,j = sum over the row's remote
// entries, signed per entry (P:562-570 complement entries subtracted, P:538-542 non-zero entries
// added), written to Wr[row] (global; the finalize adds it after a block barrier).  Per lane the
// arithmetic is run_remote's exactly (x0 += e0, x1 += e1, x0 += e2, x1 += e3 per 4-entry group;
// 0 + (x0 + x1)), so every remote mode gives the same bits.
__device__ __forceinline__ void wr_store(const DevPlan& dp, const TileDesc& T, uint16_t row, int lp, int lane,
                                         double sx, double sy) {
  for (int o = 1; o < (1 << lp); o <<= 1) {
    sx += __shfl_xor_sync(0xffffffffu, sx, o);
    sy += __shfl_xor_sync(0xffffffffu, sy, o);
  }
  KUR_ASSERT(row == EMPTY_LANE || (int64_t)(T.row0 - dp.row_begin) + row < dp.n_local);
  if (row != EMPTY_LANE && (lane & ((1 << lp) - 1)) == 0)
    __stcg(dp.Wr + (T.row0 - dp.row_begin) + row, make_double2(0.0 + sx, 0.0 + sy));
}

// remote_warp == 2: LDG gathers (one L1 wavefront per entry), 8 in flight per lane.
__device__ __forceinline__ void remote_warp_ldg(const DevPlan& dp, const TileDesc& T, const double2* __restrict__ z,
                                             uint64_t pol, int lane) {
  const PartDesc P = dp.parts[T.part0 + T.nhot];
  const int lp = P.neg >> 8;
  for (uint32_t c = 0; c < P.nchunks; ++c) {
    const uint2 cd = __ldg(dp.chunks + P.chunk0 + c);
    const uint4* q = dp.pool + cd.x;
    const uint16_t row = reinterpret_cast<const uint16_t*>(q)[lane];
    double sx, sy;
    run_remote_deep(q + HDR_UNITS + lane, cd.y, (uint32_t)dp.n, z, pol, sx, sy);
    wr_store(dp, T, row, lp, lane, sx, sy);
  }
}

// remote_warp == 1: the z entries are fetched by TMA bulk copies (16 bytes each, async proxy:
// no L1 wavefront per gather) into a ring of RING_SLOTS slots in shared memory; slot s holds one
// 4-entry group of every lane, entry e of lane l at [s][e][l] (conflict-free LDS.128 reads).
// The groups of all the part's chunks form one sequence, RING_SLOTS - 1 issued ahead of the one
// being summed.
__device__ __forceinline__ void remote_warp_tma(const DevPlan& dp, const TileDesc& T, const double2* __restrict__ z,
                                             double2* ring, uint64_t* rbar, uint64_t pol, int lane) {
  const PartDesc P = dp.parts[T.part0 + T.nhot];
  const int lp = P.neg >> 8;
  const uint32_t nch = P.nchunks;
  uint32_t ci = 0, gi = 0, qi = 0;  // issue cursor: chunk, group, sequence number
  uint2 cdi = nch > 0 ? __ldg(dp.chunks + P.chunk0) : make_uint2(0, 0);
  uint32_t sgn = 0;  // per slot: the 4 entries' sign bits (bit 31 of the ids)
  auto issue = [&]() {
    while (ci < nch && gi >= cdi.y) {  // next chunk with groups left
      ++ci;
      gi = 0;
      if (ci < nch) cdi = __ldg(dp.chunks + P.chunk0 + ci);
    }
    if (ci >= nch) return;
    const uint4 u = ldg_stream(dp.pool + cdi.x + HDR_UNITS + (size_t)gi * 32 + lane, pol);
    const uint32_t s = qi % RING_SLOTS;
    sgn = (sgn & ~(0xFu << (4 * s))) |
          (((u.x >> 31) | ((u.y >> 31) << 1) | ((u.z >> 31) << 2) | ((u.w >> 31) << 3)) << (4 * s));
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(rbar + s)), "r"(128 * 16)
                   : "memory");
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint32_t ids[4] = {u.x & 0x7FFFFFFFu, u.y & 0x7FFFFFFFu, u.z & 0x7FFFFFFFu, u.w & 0x7FFFFFFFu};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      KUR_ASSERT(ids[e] < g_dbg_zlen);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
              smem_addr(ring + (size_t)s * 128 + e * 32 + lane)),
          "l"(z + ids[e]), "r"(smem_addr(rbar + s))
          : "memory");
    }
    ++gi;
    ++qi;
  };
  for (int k = 0; k < RING_SLOTS - 1; ++k) issue();
  uint32_t qc = 0, phases = 0;  // sequence number being summed; mbarrier phase bit per slot
  for (uint32_t c = 0; c < nch; ++c) {
    const uint2 cd = __ldg(dp.chunks + P.chunk0 + c);
    const uint16_t row = reinterpret_cast<const uint16_t*>(dp.pool + cd.x)[lane];
    double x0 = 0.0, y0 = 0.0, x1 = 0.0, y1 = 0.0;
    for (uint32_t g = 0; g < cd.y; ++g) {
      issue();  // fills the slot summed in the previous iteration: RING_SLOTS - 1 groups stay ahead
      const uint32_t s = qc % RING_SLOTS;
      mbar_wait(rbar + s, (phases >> s) & 1u);
      phases ^= 1u << s;
      const uint32_t m = sgn >> (4 * s);
      const double2* slot = ring + (size_t)s * 128 + lane;
      double2 a0 = slot[0], a1 = slot[32], a2 = slot[64], a3 = slot[96];
      if (m & 1u) a0 = make_double2(-a0.x, -a0.y);
      if (m & 2u) a1 = make_double2(-a1.x, -a1.y);
      if (m & 4u) a2 = make_double2(-a2.x, -a2.y);
      if (m & 8u) a3 = make_double2(-a3.x, -a3.y);
      x0 += a0.x; y0 += a0.y; x1 += a1.x; y1 += a1.y;
      x0 += a2.x; y0 += a2.y; x1 += a3.x; y1 += a3.y;
      __syncwarp();  // every lane has read slot s before the next issue() overwrites it
      ++qc;
    }
    wr_store(dp, T, row, lp, lane, x0 + x1, y0 + y1);
  }
}

// remote_warp == 3: as remote_warp_tma, but each lane fetches its 4 entries with ONE TMA
// tile::gather4 (4 rows of z viewed as a [n_pad][2] fp64 tensor) into its own 128-byte cell of the
// slot; lane l rotates its coordinates by l & 3 so a quarter-warp's reads of entry e spread over 4
// bank groups (2-way conflicts: 1/4 wavefront per entry, against 1 for an LDG gather).
__device__ __forceinline__ void remote_warp_g4(const DevPlan& dp, const TileDesc& T, const CUtensorMap* tmz,
                                               double2* ring, uint64_t* rbar, uint64_t pol, int lane) {
  const PartDesc P = dp.parts[T.part0 + T.nhot];
  const int lp = P.neg >> 8;
  const uint32_t nch = P.nchunks;
  const uint32_t rot = lane & 3;
  uint32_t ci = 0, gi = 0, qi = 0;
  uint2 cdi = nch > 0 ? __ldg(dp.chunks + P.chunk0) : make_uint2(0, 0);
  uint32_t sgn = 0;
  auto issue = [&]() {
    while (ci < nch && gi >= cdi.y) {
      ++ci;
      gi = 0;
      if (ci < nch) cdi = __ldg(dp.chunks + P.chunk0 + ci);
    }
    if (ci >= nch) return;
    const uint4 u = ldg_stream(dp.pool + cdi.x + HDR_UNITS + (size_t)gi * 32 + lane, pol);
    const uint32_t s = qi % RING_SLOTS_G4;
    sgn = (sgn & ~(0xFu << (4 * s))) |
          (((u.x >> 31) | ((u.y >> 31) << 1) | ((u.z >> 31) << 2) | ((u.w >> 31) << 3)) << (4 * s));
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(rbar + s)), "r"(32 * 64)
                   : "memory");
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    auto sel = [&](uint32_t k) {  // entry k of the unit (selects, no local-memory array)
      const uint32_t v = k == 0 ? u.x : k == 1 ? u.y : k == 2 ? u.z : u.w;
      return v & 0x7FFFFFFFu;
    };
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_addr(ring + (size_t)s * 256 + lane * 8)),
        "l"(tmz), "r"(0), "r"(sel(rot)), "r"(sel((rot + 1) & 3)), "r"(sel((rot + 2) & 3)), "r"(sel((rot + 3) & 3)),
        "r"(smem_addr(rbar + s))
        : "memory");
    ++gi;
    ++qi;
  };
  for (int k = 0; k < RING_SLOTS_G4 - 1; ++k) issue();
  uint32_t qc = 0, phases = 0;
  for (uint32_t c = 0; c < nch; ++c) {
    const uint2 cd = __ldg(dp.chunks + P.chunk0 + c);
    const uint16_t row = reinterpret_cast<const uint16_t*>(dp.pool + cd.x)[lane];
    double x0 = 0.0, y0 = 0.0, x1 = 0.0, y1 = 0.0;
    for (uint32_t g = 0; g < cd.y; ++g) {
      issue();
      const uint32_t s = qc % RING_SLOTS_G4;
      mbar_wait(rbar + s, (phases >> s) & 1u);
      phases ^= 1u << s;
      const uint32_t m = sgn >> (4 * s);
      const double2* cell = ring + (size_t)s * 256 + lane * 8;  // position p holds entry (p + rot) & 3
      double2 a0 = cell[(0 - rot) & 3], a1 = cell[(1 - rot) & 3], a2 = cell[(2 - rot) & 3], a3 = cell[(3 - rot) & 3];
      if (m & 1u) a0 = make_double2(-a0.x, -a0.y);
      if (m & 2u) a1 = make_double2(-a1.x, -a1.y);
      if (m & 4u) a2 = make_double2(-a2.x, -a2.y);
      if (m & 8u) a3 = make_double2(-a3.x, -a3.y);
      x0 += a0.x; y0 += a0.y; x1 += a1.x; y1 += a1.y;
      x0 += a2.x; y0 += a2.y; x1 += a3.x; y1 += a3.y;
      __syncwarp();
      ++qc;
    }
    wr_store(dp, T, row, lp, lane, x0 + x1, y0 + y1);
  }
}

// world > 1: one double of this rank's packed exchange record [phases | per tile (sum z, max
// |update|)] at offset off — into the send buffer (all-gather), or, with the fused peer-store
// exchange, straight into every rank's receive buffer over NVLink (slot `rank` of each).
__device__ __forceinline__ void xput(const DevPlan& dp, const StageArgs& a, int off, double v) {
  if (dp.peer_x) {
    // double-buffered by exchange parity: a fast rank's next record cannot overwrite a record a
    // slow rank is still unpacking (the next-but-one exchange needs that rank's arrival first)
    const size_t base = ((size_t)a.xpar * dp.world + dp.rank) * dp.xstride;
    for (int r = 0; r < dp.world; ++r) dp.peer_x[r][base + off] = v;
  } else {
    a.xsend[off] = v;
  }
}

// Fused exchange: after every tile of this launch stored its record, the last CTA signals every
// rank's arrival counter (release at system scope: each CTA fenced its peer stores before its ticket).
__device__ __forceinline__ void peer_arrive(const DevPlan& dp) {
  __shared__ bool s_lastx;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned int t = atomicAdd(dp.xticket, 1u);
    s_lastx = (t == gridDim.x - 1);
    if (s_lastx) {
      *dp.xticket = 0;
      __threadfence_system();
      for (int r = 0; r < dp.world; ++r) atomicAdd_system(dp.peer_flag[r], 1u);
    }
  }
}

// Sequential sum (x, y) = 0 + v[t0] + v[t0+1] + ... + v[t1-1] of tile partials in global memory,
// with the loads issued 8 at a time (the additions stay in order: the same bits as a plain loop,
// without one L2 round trip per term on the critical path of the last CTA).
__device__ __forceinline__ double2 seq_sum_partials(const double2* v, int t0, int t1) {
  double x = 0.0, y = 0.0;
  int t = t0;
  for (; t + 8 <= t1; t += 8) {
    double2 b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) b[i] = __ldcg(v + t + i);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      x += b[i].x;
      y += b[i].y;
    }
  }
  for (; t < t1; ++t) {
    const double2 b = __ldcg(v + t);
    x += b.x;
    y += b.y;
  }
  return make_double2(x, y);
}

// Deferred block sums (world 1, plans without communities of > 64 tiles): T_c of community c from
// the previous stage's tile partials P, by ONE warp, in finish_reduce's exact summation order --
// S_b = 0 + P[t0] + ... + P[t1-1] (seq_sum_partials, one lane per b in D(c)), then
// T_c = 0 + S_{D[0]} + S_{D[1]} + ... -- so the bits equal the last-CTA reduction's.
// Replaces the last CTA's reduction after the inner stages of a step: every CTA forms the one T it
// needs while its first window is in flight, instead of one CTA reducing all C after all tiles.
__device__ __forceinline__ void lazy_T_warp(const DevPlan& dp, const double2* P, int c, int lane, double2* out) {
  const int d0 = dp.D_ptr[c], d1 = dp.D_ptr[c + 1];
  double tx = 0.0, ty = 0.0;
  for (int base = d0; base < d1; base += 32) {
    double2 sb = make_double2(0.0, 0.0);
    if (base + lane < d1) {
      const int b = dp.D_idx[base + lane];
      sb = seq_sum_partials(P, dp.comm_tile0[b], dp.comm_tile0[b + 1]);
    }
    const int nb = min(32, d1 - base);
    for (int i = 0; i < nb; ++i) {
      tx += __shfl_sync(0xffffffffu, sb.x, i);
      ty += __shfl_sync(0xffffffffu, sb.y, i);
    }
  }
  if (lane == 0) *out = make_double2(tx, ty);
}

// Executed by every thread of the LAST CTA of a grid: S_b from the per-tile
// partials, T_a, the order parameter and its recording.
// S_sh: shared scratch of >= C entries for the block sums (k_stage's free window buffer), or NULL:
// then dp.S in global memory (one more L2 round trip for T_a and for (r, psi) each).
__device__ void finish_reduce(const DevPlan& dp, const StageArgs& a, double2* S_sh = nullptr) {
  __shared__ double2 fred[NWARPS];
  double2* const Sd = S_sh ? S_sh : dp.S;
  const double2* const Pt = a.pout ? a.pout : dp.partial;  // this grid's tile partials
  const int tid = threadIdx.x;
  constexpr int BIG = 64;  // communities with more tiles are reduced by the whole CTA
  if (a.v_out) {  // kur_potential: V = sum of the tile partials in tile order (fixed shape)
    double x = 0.0, y = 0.0;
    const int nt = dp.comm_tile0[dp.C];
    for (int t = tid; t < nt; t += NTHREADS) x += __ldcg(Pt + t).x;
    block_sum2(x, y, fred);
    if (tid == 0) a.v_out[0] = x;
    return;
  }
  if (a.fp_reset || a.fp_check) {  // implicit midpoint: convergence of the fixed-point iteration
    double d = 0.0;
    if (a.fp_check) {
      const int nt = dp.comm_tile0[dp.C];
      for (int t = tid; t < nt; t += NTHREADS) d = fmax(d, __ldcg(dp.pmax + t));
    }
    d = block_max(d, reinterpret_cast<double*>(fred));
    if (tid == 0) dp.ctrl->fp_done = a.fp_check ? (d <= dp.ctrl->fp_tol) : 0;
    __syncthreads();
  }
  // S_b = sum of its tiles' partials: one thread per community, tiles in order
  // (the loads of a community are independent and pipeline); > BIG tiles: block reduction
  for (int c = tid; c < dp.C; c += NTHREADS) {
    const int t0 = dp.comm_tile0[c], t1 = dp.comm_tile0[c + 1];
    if (t1 - t0 > BIG) continue;
    Sd[c] = seq_sum_partials(Pt, t0, t1);
  }
  for (int i = 0; i < dp.n_big; ++i) {  // communities of > BIG tiles (uniform): fixed-shape block reduction
    const int c = dp.big_comm[i];
    const int t0 = dp.comm_tile0[c], t1 = dp.comm_tile0[c + 1];
    double x = 0.0, y = 0.0;
    for (int t = t0 + tid; t < t1; t += NTHREADS) {
      const double2 v = __ldcg(Pt + t);
      x += v.x;
      y += v.y;
    }
    block_sum2(x, y, fred);
    if (tid == 0) Sd[c] = make_double2(x, y);
    __syncthreads();
  }
  __threadfence_block();
  __syncthreads();
  auto ldS = [&](int c) { return S_sh ? S_sh[c] : __ldcg(dp.S + c); };
  for (int c = tid; c < dp.C; c += NTHREADS) {  // T_a = sum over dense column communities
    double x = 0.0, y = 0.0;
    for (int i = dp.D_ptr[c]; i < dp.D_ptr[c + 1]; ++i) {
      const double2 v = ldS(dp.D_idx[i]);
      x += v.x;
      y += v.y;
    }
    a.Tout[c] = make_double2(x, y);
    if (a.op_local) {  // localised order parameters S_b / n_b
      const double2 v = ldS(c);
      const double nb = (double)dp.comm_size[c];
      const double cx = nb > 0 ? v.x / nb : 0.0, cy = nb > 0 ? v.y / nb : 0.0;
      const double r = sqrt(cx * cx + cy * cy);
      a.op_local[2 * c] = r;
      a.op_local[2 * c + 1] = r == 0.0 ? 0.0 : atan2(cy, cx);
    }
  }
  {  // r e^{i psi} = (1/N) sum_b S_b, fixed-shape block reduction
    double x = 0.0, y = 0.0;
    for (int c = tid; c < dp.C; c += NTHREADS) {
      const double2 v = ldS(c);
      x += v.x;
      y += v.y;
    }
    block_sum2(x, y, fred);
    if (tid == 0) {
      const double cm = x / (double)dp.n, sm = y / (double)dp.n;
      const double r = sqrt(cm * cm + sm * sm);
      const double psi = r == 0.0 ? 0.0 : atan2(sm, cm);
      Ctrl* ct = dp.ctrl;
      ct->rpsi[0] = r;
      ct->rpsi[1] = psi;
      if (a.op_rpsi) {
        a.op_rpsi[0] = r;
        a.op_rpsi[1] = psi;
      }
      if (a.record != REC_NONE) {
        if (a.record == REC_START) ct->step = 0;
        else ct->step += 1;
        const long long nstep = ct->step;
        if (ct->record_every > 0 && ct->r_trace && nstep % ct->record_every == 0) {
          const long long i = nstep / ct->record_every;
          if (i < ct->nrec_cap) {
            ct->r_trace[2 * i] = r;
            ct->r_trace[2 * i + 1] = psi;
          }
        }
      }
    }
  }
}

// Writes the tile partial, then lets the last CTA of the grid finish.
// dmax: this thread's max |fixed-point update| (implicit midpoint iterations, else 0).
__device__ __forceinline__ void tile_partial_and_finish(const DevPlan& dp, const StageArgs& a, int lt,
                                                        double x, double y, double2* red, double dmax = 0.0,
                                                        double2* S_sh = nullptr) {
  __shared__ bool s_last;
  if (a.fp_check) {
    dmax = block_max(dmax, reinterpret_cast<double*>(red));
    __syncthreads();
  }
  block_sum2(x, y, red);
  if (threadIdx.x == 0) {
    (a.pout ? a.pout : dp.partial)[dp.tile_base + lt] = make_double2(x, y);
    if (a.fp_check) dp.pmax[dp.tile_base + lt] = dmax;
    if (a.xsend) {
      xput(dp, a, dp.xrows + 3 * lt, x);
      xput(dp, a, dp.xrows + 3 * lt + 1, y);
      xput(dp, a, dp.xrows + 3 * lt + 2, dmax);
    }
    s_last = false;
    if (dp.world == 1 && !a.no_finish) {  // world > 1: the reduction runs after the exchange;
      // no_finish: the next stage forms its block sums from these partials itself (lazy_T_warp)
      __threadfence();
      const unsigned int t = atomicAdd(&dp.ctrl->ticket, 1u);
      s_last = (t == gridDim.x - 1);
    }
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  finish_reduce(dp, a, S_sh);
  if (threadIdx.x == 0) dp.ctrl->ticket = 0;
  PROF_G(162);
}

// a1 for one tile: z = e^{i theta} of its rows; returns this thread's partial sums.
__device__ __forceinline__ void prologue_rows(const DevPlan& dp, const StageArgs& a, const TileDesc& T, double& x,
                                              double& y) {
  // all of this thread's phases are loaded before the first sincos (memory-level parallelism);
  // summation order of the partials unchanged (rows in increasing lr)
  constexpr int R = MAX_TILE_ROWS_NOPARTS / NTHREADS;
  const double* src = a.commit ? a.commit : a.theta;  // implicit midpoint: theta_{n+1} = the fixed point
  double th[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int lr = threadIdx.x + k * NTHREADS;
    th[k] = lr < T.nrows ? src[T.row0 + lr - dp.row_begin] : 0.0;
  }
  x = 0.0;
  y = 0.0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int lr = threadIdx.x + k * NTHREADS;
    if (lr >= T.nrows) break;
    const int row = T.row0 + lr;
    if (a.commit) {
      a.theta[row - dp.row_begin] = th[k];
      if (!isfinite(th[k])) dp.ctrl->nonfinite = 1;
    }
    double s, c;
    sincos(th[k], &s, &c);  // z = e^{i theta}
    a.zout[row] = make_double2(c, s);
    if (a.xsend) xput(dp, a, row - dp.row_begin, th[k]);
    x += c;
    y += s;
  }
}

// a3-a5 for one tile (all threads of the CTA call it; contains barriers).
// zs: [WZ + 8] window + zero sentinels, Ws: [rows_per_tile] row sums (both
// unused when the plan has no parts).  Returns the thread's partial sums of
// the next stage's z in (px, py) and whether a phase became non-finite.
template <int MODE, bool SMALL, bool RW = false, bool CR = false>
__device__ __forceinline__ bool stage_rows(const DevPlan& dp, const StageArgs& a, const TileDesc& T, double2* zs,
                                           double2* Ws, uint64_t* bar, uint32_t& phase, double& px, double& py,
                                           double& dmax, double2* ring = nullptr, uint64_t* rbar = nullptr,
                                           const CUtensorMap* tmz = nullptr, double2* s_T = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool parts = dp.has_parts;
  // the remote part of the tile was summed by k_remote into Wr (added in the finalize);
  // small plans (k_small, or kur_rhs on them) keep it inline
  const bool split = !SMALL && dp.has_remote;
  const bool addr = split && T.nparts > T.nhot && a.phase != PHASE_A;
  // world > 1: phase A sums the own-community hot parts (local z only) into Wh while the
  // previous stage's exchange is in flight; phase B continues from Wh (exact copy)
  const bool from_wh = !SMALL && a.phase == PHASE_B && T.nloc > 0;
  // concurrent inline remote part (compile-time variant CR, plans whose inline remote part is a large
  // share of the LSU work, e.g. config 3): warps [cr_hot_warps, NWARPS) sum the tile's remote part
  // into Wc (shared) while the others gather the hot windows; the finalize adds Wc once per row --
  // the k_remote pass's arithmetic (Ws + (0 + remote sum)), so every mode gives the same bits
  const bool cr = CR && !SMALL && !split && T.nparts > T.nhot && a.phase != PHASE_A;
  double2* Wc = Ws + dp.rows_per_tile;
  if (parts) {
    for (int r = tid; r < T.nrows; r += NTHREADS) {
      Ws[r] = from_wh ? __ldcg(a.Wh + (T.row0 - dp.row_begin) + r) : make_double2(0.0, 0.0);
      if (cr) Wc[r] = make_double2(0.0, 0.0);
    }
    __syncthreads();
  }
  // ---- parts: hot ones gather from the staged window, remote ones from global memory
  const uint64_t pol = evict_first_policy();
  int loaded = -1;
  if (!SMALL) PROF_T(0);
#ifdef KUR_PROFILE
  if (!SMALL && g_prof && tid == 0) {
    g_prof[(size_t)blockIdx.x * PROF_STRIDE + 27] = (unsigned long long)T.nhot;
    g_prof[(size_t)blockIdx.x * PROF_STRIDE + 28] = (unsigned long long)T.nparts;
  }
#endif
  // Canonical order (builder): own-community hot windows, other hot windows, then the
  // single remote part (inline) — or its k_remote row sum Wr added in the finalize: one
  // addition per row either way, so both modes and every world size are bitwise identical.
  const int nrem = split ? 0 : T.nparts - T.nhot;
  const int pbeg = (!SMALL && a.phase == PHASE_B) ? T.nloc : 0;
  const int pend = (!SMALL && a.phase == PHASE_A) ? T.nloc : T.nhot + nrem;
  bool pending = false;
#ifdef KUR_PROFILE
  if (!SMALL && g_prof && tid == 0) g_prof[(size_t)blockIdx.x * PROF_STRIDE + 29] = (unsigned long long)nrem;
#endif
  // remote warp: the last warp sums the tile's remote part (into Wr) while the other NWARPS - 1
  // gather the hot parts, which then synchronise on named barrier 1 instead of the block barrier
  // (a compile-time variant: the branch alone costs the default kernel ~4 % even when not taken)
  const bool rw = RW && !SMALL && addr;
  if (rw && warp == NWARPS - 1) {
    if (dp.remote_warp == 3) remote_warp_g4(dp, T, tmz, ring, rbar, pol, lane);
    else if (dp.remote_warp == 1) remote_warp_tma(dp, T, a.zin, ring, rbar, pol, lane);
    else remote_warp_ldg(dp, T, a.zin, pol, lane);
    __syncthreads();  // joins the hot warps below (Wr complete, Ws complete)
  } else if (cr && warp >= dp.cr_hot_warps) {
    run_part<false, true>(dp, dp.parts[T.part0 + T.nhot], false, zs, a.zin, Wc, pol, warp - dp.cr_hot_warps, lane,
                          NWARPS - dp.cr_hot_warps);
    __syncthreads();  // joins the hot warps below
  } else {
  const uint32_t nhw = rw ? NWARPS - 1 : (cr ? dp.cr_hot_warps : NWARPS);
  const bool named = rw || cr;  // the hot group synchronises on named barrier 1
  const int pend_h = cr ? min(pend, T.nhot) : pend;
  if (pbeg < T.nhot && pbeg < pend_h) {
    loaded = dp.parts[T.part0 + pbeg].window;
    pending = true;
    if (tid == 0) tma_load_1d(zs, a.zin + (size_t)loaded * WZ, WZ * sizeof(double2), bar);
  }
  // deferred block sums: warp 0 forms T of the tile's community while the first window is in flight
  if (!SMALL && a.plazy && warp == 0) lazy_T_warp(dp, a.plazy, T.comm, lane, s_T);
  for (int pi = pbeg; pi < pend_h; ++pi) {
    const int p = T.part0 + pi;
    const PartDesc P = dp.parts[p];
    const bool hot = P.window >= 0;
    if (!SMALL && pi < 8) PROF_T(1 + 3 * pi);
    if (hot && (P.window != loaded || pending)) {  // all reads of the previous window ended at the last barrier
      if (P.window != loaded && tid == 0) tma_load_1d(zs, a.zin + (size_t)P.window * WZ, WZ * sizeof(double2), bar);
      mbar_wait(bar, phase);
      phase ^= 1u;
      loaded = P.window;
      pending = false;
    }
    if (!SMALL && pi < 8) PROF_T(2 + 3 * pi);
    // large tiles: warm L2 with the next hot window while this part is gathered, so its TMA
    // copy hits L2 (cfg5 1.190 -> 1.183 ms; small tiles lose slightly, cfg4 0.321 -> 0.323)
    if (dp.rows_per_tile >= MAX_TILE_ROWS && tid == 0 && pi + 1 < pend_h && pi + 1 < T.nhot) {
      const int wn = dp.parts[T.part0 + pi + 1].window;
      if (wn != loaded)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.zin + (size_t)wn * WZ),
                     "r"((uint32_t)(WZ * sizeof(double2)))
                     : "memory");
    }
    run_part<SMALL, !SMALL>(dp, P, hot, zs, a.zin, Ws, pol, warp, lane, nhw);
    if (!SMALL) PROF_W(pi, warp);
    if (named) asm volatile("bar.sync 1, %0;" ::"r"(nhw * 32) : "memory");
    else __syncthreads();
    if (!SMALL && pi < 8) PROF_T(3 + 3 * pi);
  }
  if (named) __syncthreads();  // joins the remote warp(s)
  }
  if (!SMALL && a.plazy) __syncthreads();  // s_T visible (tiles without parts have no barrier above)
  if (!SMALL) PROF_T(25);
  if (!SMALL && a.phase == PHASE_A) {  // hand the own-community sums to phase B
    for (int r = tid; r < T.nrows; r += NTHREADS) a.Wh[(T.row0 - dp.row_begin) + r] = Ws[r];
    px = py = dmax = 0.0;
    return false;
  }

  // ---- finalize: k_j = omega_j + (K/N) Im(conj z_j W_j), fused RK4 stage
  if (!SMALL && a.rov_wait) asm volatile("griddepcontrol.wait;" ::: "memory");  // k_remote done: Wr complete
  const double2 Tc = (!SMALL && a.plazy) ? *s_T : __ldcg(a.Tin + T.comm);
  px = 0.0;
  py = 0.0;
  dmax = 0.0;
  bool bad = false;
  for (int lr = tid; lr < T.nrows; lr += NTHREADS) {
    const int row = T.row0 + lr;
    const int li = row - dp.row_begin;
    double2 w = parts ? Ws[lr] : make_double2(0.0, 0.0);
    if (addr) {
      const double2 r = rw ? __ldcg(dp.Wr + li) : __ldcs(dp.Wr + li);
      w.x += r.x;
      w.y += r.y;
    }
    if (cr) {
      const double2 r = Wc[lr];
      w.x += r.x;
      w.y += r.y;
    }
    const double wx = Tc.x + w.x, wy = Tc.y + w.y;
    const double2 zj = SMALL ? __ldcg(a.zin + row) : a.zin[row];
    // K/M_m: uniform K/N, or K/deg_m for the degree scaling
    const double kn = dp.rowscale ? a.K * dp.rowscale[li] : a.KN;
    if (MODE == MODE_POT) {  // -omega_m theta_m + (K/2)(1/M_m)(sum_l A_ml - Re(conj z_m W_m))
      const double sm = dp.rowscale ? dp.rowscale[li] : a.KN / a.K;
      px += -a.omega[li] * a.theta[li] + 0.5 * a.K * sm * (dp.potc[li] - (zj.x * wx + zj.y * wy));
      continue;
    }
    const double k = rhs_k(a.omega[li], kn, zj.x, zj.y, wx, wy);
    if (MODE == MODE_RHS) {
      a.out[li] = k;
    } else {
      const double thn = a.theta[li];
      double ts;
      if (MODE == MODE_S1) {
        a.acc[li] = k;
        ts = __dadd_rn(thn, __dmul_rn(a.h / 2.0, k));
      } else if (MODE == MODE_S2) {
        a.acc[li] = __dadd_rn(a.acc[li], __dmul_rn(2.0, k));
        ts = __dadd_rn(thn, __dmul_rn(a.h / 2.0, k));
      } else if (MODE == MODE_S3) {
        a.acc[li] = __dadd_rn(a.acc[li], __dmul_rn(2.0, k));
        ts = __dadd_rn(thn, __dmul_rn(a.h, k));
      } else if (MODE == MODE_S4) {  // theta_{n+1} = theta_n + (h/6)(k1 + 2k2 + 2k3 + k4)
        ts = __dadd_rn(thn, __dmul_rn(a.h / 6.0, __dadd_rn(a.acc[li], k)));
        a.theta[li] = ts;
        if (a.theta_host) a.theta_host[li] = ts;
        bad |= !isfinite(ts);
      } else if (MODE == MODE_E1) {  // explicit Euler: theta_{n+1} = theta_n + h k
        ts = __dadd_rn(thn, __dmul_rn(a.h, k));
        a.theta[li] = ts;
        if (a.theta_host) a.theta_host[li] = ts;
        bad |= !isfinite(ts);
      } else if (MODE == MODE_H1) {  // Heun: k1, stage state theta_n + h k1
        a.acc[li] = k;
        ts = __dadd_rn(thn, __dmul_rn(a.h, k));
      } else if (MODE == MODE_H2) {  // theta_{n+1} = theta_n + (h/2)(k1 + k2)
        ts = __dadd_rn(thn, __dmul_rn(a.h / 2.0, __dadd_rn(a.acc[li], k)));
        a.theta[li] = ts;
        if (a.theta_host) a.theta_host[li] = ts;
        bad |= !isfinite(ts);
      } else {  // MODE_M0 / MODE_MI: implicit midpoint fixed point on tp (kept in acc)
        const double nv = __dadd_rn(thn, __dmul_rn(a.h, k));
        if (MODE == MODE_MI) dmax = fmax(dmax, fabs(__dadd_rn(nv, -a.acc[li])));
        a.acc[li] = nv;
        ts = __dadd_rn(thn, nv) / 2.0;
        if (MODE == MODE_MI && !(fabs(nv) <= 1.79e308)) dmax = __longlong_as_double(0x7ff0000000000000ll);
      }
      double s, c;
      sincos(ts, &s, &c);
      a.zout[row] = make_double2(c, s);
      if (a.xsend) xput(dp, a, li, ts);
      px += c;
      py += s;
    }
  }
  return bad;
}

__global__ void __launch_bounds__(NTHREADS) k_prologue(const DevPlan dp, const StageArgs a) {
  __shared__ double2 red[NWARPS];
  pdl_wait_and_release();
  const int lt = dp.order[blockIdx.x];
  const TileDesc T = dp.tiles[lt];
  double x, y;
  prologue_rows(dp, a, T, x, y);
  tile_partial_and_finish(dp, a, lt, x, y, red);
  if (dp.peer_x && a.xsend) peer_arrive(dp);
}

// a3, remote half: W_r,j = sum over the row's remote entries (signed, P:562-570 /
// P:538-542) into Wr.  A warp sums one remote chunk (32 rows) at a time; all tiles'
// chunks form one flat list, longest first, which the grid's warps stride over: every
// row lies in exactly one remote chunk of its tile (one remote part per tile), so the
// row sum is written, not accumulated, and rows without remote entries keep the zero
// Wr was initialised with.  3 CTAs of 8 warps per SM (80 registers: the next chunk's
// index units are in flight with the current gathers; 4 CTAs at 64 registers: slower).
constexpr int KREM_THREADS = 256;
constexpr int KREM_CTAS_PER_SM = 3;
__global__ void __launch_bounds__(KREM_THREADS, KREM_CTAS_PER_SM) k_remote(const DevPlan dp,
                                                                           const double2* __restrict__ zin) {
  // Persistent warps striding over the chunk list.  The next chunk's header and first two
  // index units are requested before the current chunk's gathers (and its list entry /
  // descriptor two and one chunks ahead), so a warp never waits on an index load between
  // chunks; only the drain of the current gathers before its row sums remains.
  pdl_wait_and_release();
  const int lane = threadIdx.x & 31;
  const int nw = (int)gridDim.x * (KREM_THREADS / 32);
  int w = (int)blockIdx.x * (KREM_THREADS / 32) + (threadIdx.x >> 5);
  const int n = dp.n_rchunks;
  if (w >= n) return;
  const uint2* rcs = reinterpret_cast<const uint2*>(dp.rchunks);  // {chunk id, tile row base}
  const uint64_t pol = evict_first_policy();
  const uint32_t sent = (uint32_t)dp.n;
  const uint4 s4 = make_uint4(sent, sent, sent, sent);
  uint2 rc = __ldg(rcs + w);
  uint2 cd = __ldg(dp.chunks + rc.x);
  const uint4* q = dp.pool + cd.x;
  uint16_t row = reinterpret_cast<const uint16_t*>(q)[lane];
  int lp = dp.rem_lp[w];
  uint4 b0 = cd.y > 0 ? ldg_stream(q + HDR_UNITS + lane, pol) : s4;
  uint4 b1 = cd.y > 1 ? ldg_stream(q + HDR_UNITS + lane + 32, pol) : s4;
  uint2 rc1 = make_uint2(0, 0), cd1 = make_uint2(0, 0);
  if (w + nw < n) {
    rc1 = __ldg(rcs + w + nw);
    cd1 = __ldg(dp.chunks + rc1.x);
  }
  for (;;) {
    const bool more = w + nw < n;
    const uint4* q1 = dp.pool + cd1.x;
    uint16_t row1 = EMPTY_LANE;
    int lp1 = 0;
    uint4 b0n = s4, b1n = s4;
    if (more) {
      row1 = reinterpret_cast<const uint16_t*>(q1)[lane];
      lp1 = dp.rem_lp[w + nw];
      if (cd1.y > 0) b0n = ldg_stream(q1 + HDR_UNITS + lane, pol);
      if (cd1.y > 1) b1n = ldg_stream(q1 + HDR_UNITS + lane + 32, pol);
    }
    const uint2 rc2 = w + 2 * nw < n ? __ldg(rcs + w + 2 * nw) : make_uint2(0, 0);
    double sx, sy;
    run_remote_deep_pre(q + HDR_UNITS + lane, cd.y, sent, zin, pol, b0, b1, sx, sy);
    const uint2 cd2 = w + 2 * nw < n ? __ldg(dp.chunks + rc2.x) : make_uint2(0, 0);
    for (int o = 1; o < (1 << lp); o <<= 1) {
      sx += __shfl_xor_sync(0xffffffffu, sx, o);
      sy += __shfl_xor_sync(0xffffffffu, sy, o);
    }
    // 0 + s: the same single rounding-free addition the inline path does into a zeroed sum
    KUR_ASSERT(row == EMPTY_LANE || (int64_t)(rc.y + row) < dp.n_local);
    if (row != EMPTY_LANE && (lane & ((1 << lp) - 1)) == 0)
      __stcs(dp.Wr + rc.y + row, make_double2(0.0 + sx, 0.0 + sy));  // streaming: keep z in L2
    if (!more) break;
    w += nw;
    rc = rc1;
    cd = cd1;
    q = q1;
    row = row1;
    lp = lp1;
    b0 = b0n;
    b1 = b1n;
    rc1 = rc2;
    cd1 = cd2;
  }
}

template <int MODE, bool RW, bool CR>
__global__ void __launch_bounds__(NTHREADS, 2) k_stage(const DevPlan dp, const StageArgs a,
                                                       const __grid_constant__ CUtensorMap tmz) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* zs = reinterpret_cast<double2*>(smem_raw);  // [WZ + 8]: window + 8 zero sentinels
  double2* Ws = zs + (WZ + 8);                         // [rows_per_tile]: W_j of the tile
  double2* ring = Ws + dp.rows_per_tile;               // [RING_SLOTS][4][32] remote warp (TMA)
  __shared__ double2 red[NWARPS];
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t rbar[RING_SLOTS];
  __shared__ int s_nonfinite;
  __shared__ double2 s_T;  // deferred block sums: T of the tile's community
  const int tid = threadIdx.x;
  if (!a.rov_wait) pdl_wait_and_release();  // rov_wait: only Wr depends on k_remote (waited for before the finalize)
  PROF_G(160);
  // implicit midpoint: iterations after convergence are no-ops (uniform: every CTA reads the same flag)
  // (phase A never skips: it may run before the finish that sets or clears the flag, and
  // phase B, which does check it, then reads Wh)
  if (MODE == MODE_MI && a.phase != PHASE_A && *(volatile const int*)&dp.ctrl->fp_done) {
    if (dp.peer_x && a.xsend) {  // re-publish this rank's previous record (the all-gather path
      // re-sends the unchanged send buffer) into the current receive half of every rank
      const double* prev = dp.peer_x[dp.rank] + ((size_t)(1 - a.xpar) * dp.world + dp.rank) * dp.xstride;
      for (int i = blockIdx.x * NTHREADS + threadIdx.x; i < dp.xstride; i += gridDim.x * NTHREADS)
        xput(dp, a, i, prev[i]);
      peer_arrive(dp);
    }
    return;
  }
  if (a.lazy_rec && blockIdx.x == gridDim.x - 1) {  // the deferred S4 reduction + step record, by the
    StageArgs ra = a;                                 // last-launched (lightest) tile's CTA, in
    ra.pout = const_cast<double2*>(a.plazy);          // finish_reduce's order (same bits)
    ra.record = REC_STEP;
    ra.op_rpsi = ra.op_local = ra.v_out = nullptr;
    ra.fp_reset = ra.fp_check = 0;
    finish_reduce(dp, ra, nullptr);
    __syncthreads();
  }
  const int lt = dp.order[blockIdx.x];
  const TileDesc T = dp.tiles[lt];
  if (a.phase == PHASE_A && T.nloc == 0) return;  // nothing local to pre-sum (phase B starts from 0)
  if (dp.has_parts && tid < 8) zs[WZ + tid] = make_double2(0.0, 0.0);
  if (tid == 0) {
    s_nonfinite = 0;
    mbar_init(&bar, 1);
  }
  if (RW && (dp.remote_warp == 1 || dp.remote_warp == 3) && tid >= 32 && tid < 32 + RING_SLOTS)
    mbar_init(rbar + (tid - 32), 1);
  __syncthreads();
  uint32_t phase = 0;
  double px, py, dmax;
  const bool bad =
      stage_rows<MODE, false, RW, CR>(dp, a, T, zs, Ws, &bar, phase, px, py, dmax, ring, rbar, &tmz, &s_T);
  if (MODE == MODE_RHS || a.phase == PHASE_A) return;
  constexpr bool FINAL = MODE == MODE_S4 || MODE == MODE_E1 || MODE == MODE_H2;
  if (FINAL && bad) s_nonfinite = 1;
  __syncthreads();
  if (FINAL && tid == 0 && s_nonfinite) dp.ctrl->nonfinite = 1;
  PROF_T(26);
  PROF_G(161);
  // the window buffer is free now: the last CTA keeps the block sums in it (WZ >= C)
  tile_partial_and_finish(dp, a, lt, px, py, red, dmax, (dp.has_parts && dp.C <= WZ) ? zs : nullptr);
  if (dp.peer_x && a.xsend) peer_arrive(dp);
}

// ---- single-CTA trajectory kernel for tiny graphs (world == 1): the whole
// kur_step (prologue + nsteps x 4 stages, each followed by the block-sum
// reduction) in one launch, barriers instead of kernel boundaries.
template <int MODE>
__device__ __forceinline__ void small_stage(const DevPlan& dp, StageArgs a, const double2* zin, double2* zout,
                                            const double2* Tin, double2* Tout, int record, double2* zs,
                                            double2* Ws, uint64_t* bar, uint32_t& phase, double2* red,
                                            int* s_bad) {
  a.zin = zin;
  a.zout = zout;
  a.Tin = Tin;
  a.Tout = Tout;
  a.record = record;
  for (int lt = 0; lt < dp.ntiles; ++lt) {
    const TileDesc T = dp.tiles[lt];
    double px, py, dmax;
    const bool bad = stage_rows<MODE, true>(dp, a, T, zs, Ws, bar, phase, px, py, dmax);
    if (MODE == MODE_S4 && bad) *s_bad = 1;
    block_sum2(px, py, red);
    if (threadIdx.x == 0) dp.partial[lt] = make_double2(px, py);
    __syncthreads();
  }
  __threadfence_block();
  __syncthreads();
  finish_reduce(dp, a);
  __threadfence_block();
  __syncthreads();
}

__global__ void __launch_bounds__(NTHREADS, 1) k_small(const DevPlan dp, StageArgs a, double2* zA, double2* zB,
                                                       double2* TA, double2* TB, long long nsteps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* zs = reinterpret_cast<double2*>(smem_raw);
  double2* Ws = zs + (WZ + 8);
  __shared__ double2 red[NWARPS];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int s_bad;
  if (dp.has_parts && threadIdx.x < 8) zs[WZ + threadIdx.x] = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    s_bad = 0;
    mbar_init(&bar, 1);
  }
  __syncthreads();
  uint32_t phase = 0;
  // prologue: z(theta_n) and the block sums of theta_n, record n = 0
  a.zout = zA;
  a.Tout = TA;
  a.record = REC_START;
  for (int lt = 0; lt < dp.ntiles; ++lt) {
    double x, y;
    prologue_rows(dp, a, dp.tiles[lt], x, y);
    block_sum2(x, y, red);
    if (threadIdx.x == 0) dp.partial[lt] = make_double2(x, y);
    __syncthreads();
  }
  __threadfence_block();
  __syncthreads();
  finish_reduce(dp, a);
  __threadfence_block();
  __syncthreads();
  for (long long n = 0; n < nsteps; ++n) {
    small_stage<MODE_S1>(dp, a, zA, zB, TA, TB, REC_NONE, zs, Ws, &bar, phase, red, &s_bad);
    small_stage<MODE_S2>(dp, a, zB, zA, TB, TA, REC_NONE, zs, Ws, &bar, phase, red, &s_bad);
    small_stage<MODE_S3>(dp, a, zA, zB, TA, TB, REC_NONE, zs, Ws, &bar, phase, red, &s_bad);
    small_stage<MODE_S4>(dp, a, zB, zA, TB, TA, REC_STEP, zs, Ws, &bar, phase, red, &s_bad);
  }
  if (threadIdx.x == 0 && s_bad) dp.ctrl->nonfinite = 1;
}

// Tiny entry-free plans (one tile, no stored entries: the classical all-to-all model of
// P:130-255 at small N): the whole RK4 trajectory in one CTA with every row's state
// (theta_n, omega, acc, z) in registers and the block sum reduced in shared memory — no
// global round trips between stages.  W_j = T_c (P:557-561 with empty complement lists),
// T_c = S_c when the diagonal block is dense, and the arithmetic is the general path's.
__global__ void __launch_bounds__(NTHREADS, 1) k_small_dense(const DevPlan dp, StageArgs a, long long nsteps) {
  constexpr int R = MAX_TILE_ROWS / NTHREADS;
  __shared__ double2 red[NWARPS];
  __shared__ double2 sS;
  const int tid = threadIdx.x;
  const TileDesc T = dp.tiles[0];
  bool dense_self = false;
  for (int i = dp.D_ptr[T.comm]; i < dp.D_ptr[T.comm + 1]; ++i) dense_self |= dp.D_idx[i] == T.comm;
  double th[R], om[R], acc[R], zc[R], zsn[R], kn[R];
  double x = 0.0, y = 0.0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int lr = tid + k * NTHREADS;
    const bool v = lr < T.nrows;
    const int li = T.row0 + lr - dp.row_begin;
    th[k] = v ? a.theta[li] : 0.0;
    om[k] = v ? a.omega[li] : 0.0;
    kn[k] = v ? (dp.rowscale ? a.K * dp.rowscale[li] : a.KN) : 0.0;
    acc[k] = 0.0;
    sincos(th[k], &zsn[k], &zc[k]);
    if (v) {
      x += zc[k];
      y += zsn[k];
    }
  }
  Ctrl* ct = dp.ctrl;
  // block sum -> sS, order parameter (r, psi) = S_c / N, record when due
  auto reduce = [&](bool record, long long step) {
    block_sum2(x, y, red);
    if (tid == 0) {
      sS = make_double2(x, y);
      const double cm = x / (double)dp.n, sm = y / (double)dp.n;
      const double r = sqrt(cm * cm + sm * sm);
      const double psi = r == 0.0 ? 0.0 : atan2(sm, cm);
      ct->rpsi[0] = r;
      ct->rpsi[1] = psi;
      if (record && ct->record_every > 0 && ct->r_trace && step % ct->record_every == 0) {
        const long long i = step / ct->record_every;
        if (i < ct->nrec_cap) {
          ct->r_trace[2 * i] = r;
          ct->r_trace[2 * i + 1] = psi;
        }
      }
    }
    __syncthreads();
    x = y = 0.0;
  };
  reduce(true, 0);
  bool bad = false;
  double thn[R];
  for (long long n = 0; n < nsteps; ++n) {
#pragma unroll
    for (int k = 0; k < R; ++k) thn[k] = th[k];
#pragma unroll 1
    for (int st = 1; st <= 4; ++st) {
      const double2 Tc = dense_self ? sS : make_double2(0.0, 0.0);
      const double wx = Tc.x + 0.0, wy = Tc.y + 0.0;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int lr = tid + k * NTHREADS;
        if (lr >= T.nrows) break;
        const double kk = rhs_k(om[k], kn[k], zc[k], zsn[k], wx, wy);
        double ts;
        if (st == 1) {
          acc[k] = kk;
          ts = __dadd_rn(thn[k], __dmul_rn(a.h / 2.0, kk));
        } else if (st == 2) {
          acc[k] = __dadd_rn(acc[k], __dmul_rn(2.0, kk));
          ts = __dadd_rn(thn[k], __dmul_rn(a.h / 2.0, kk));
        } else if (st == 3) {
          acc[k] = __dadd_rn(acc[k], __dmul_rn(2.0, kk));
          ts = __dadd_rn(thn[k], __dmul_rn(a.h, kk));
        } else {
          ts = __dadd_rn(thn[k], __dmul_rn(a.h / 6.0, __dadd_rn(acc[k], kk)));
          th[k] = ts;
          bad |= !isfinite(ts);
        }
        sincos(ts, &zsn[k], &zc[k]);
        x += zc[k];
        y += zsn[k];
      }
      reduce(st == 4, n + 1);
    }
  }
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int lr = tid + k * NTHREADS;
    if (lr < T.nrows) a.theta[T.row0 + lr - dp.row_begin] = th[k];
  }
  if (bad) ct->nonfinite = 1;
  if (tid == 0) ct->step = nsteps;
}

// ---- persistent grid-synchronous RK4 for entry-free plans (no stored entries: complete graphs and
// graphs whose blocks are all full or empty; world 1, every tile's CTA co-resident -- cooperative
// launch).  W_j = T_{c(j)} (P:557-561 with empty lists; P:240-255 for one community), so a stage
// needs nothing but the block sums of the previous one: each CTA keeps its tile's z and omega in
// shared memory and theta_n, acc in registers for the whole trajectory, publishes its tile partial
// of z, and every CTA reduces all partials itself in finish_reduce's exact summation shapes -- the
// same bits as the general path (k_prologue + k_stage<S1..S4>), without a kernel boundary or a
// last-CTA tail per stage.  Grid synchronisation: a monotonic 64-bit arrival counter -- publication q
// is complete when it reaches q * (number of CTAs); one atomic and one spinning thread per CTA (one
// spinning thread per partial measured 16.8 against 10.3 us per stage: the acquire polls load the
// L2).  Partials are double-buffered by the parity of q: a CTA can publish q + 2 (same half) only
// after publication q + 1 completed, i.e. after every CTA finished reading publication q.
__device__ __forceinline__ void publish_and_wait(double2* pbuf, unsigned long long* cnt, int nt, int lt,
                                                 unsigned long long q, double x, double y) {
  if (threadIdx.x == 0) {  // (block_sum2's result is in thread 0)
    __stcg(pbuf + (size_t)(q & 1ull) * nt + lt, make_double2(x, y));
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(cnt) : "memory");  // orders the partial before
    const unsigned long long target = q * (unsigned long long)nt;
    unsigned long long v;
    do {  // acquire polls, no trailing fence: the kernel rereads nothing through L1, and a relaxed poll
          // + fence.acq_rel measured 8.10 against 7.81 us per stage on config 2 (profiles/r02/notes/persist_acq_poll_ab.log)
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
    } while ((long long)(v - target) < 0);  // the partials are then read through L2 (ld.global.cg)
  }
  __syncthreads();
}

// S_b of every community from the tile partials of publication q (finish_reduce's shapes: one thread
// per community summing its tiles in order, or a fixed-shape block reduction for communities of
// > 64 tiles), into shared S_sh; then T of community c_own; (r, psi) = (1/N) sum_b S_b only if
// want_rpsi.  Ends with a block barrier.
__device__ __forceinline__ void local_reduce(const DevPlan& dp, const double2* pbuf, int nt, unsigned long long q,
                                             double2* S_sh, double2* red, int c_own, double2* sT, double* s_rpsi,
                                             bool want_rpsi) {
  const double2* src = pbuf + (size_t)(q & 1ull) * nt;
  const int tid = threadIdx.x;
  constexpr int BIG = 64;
  for (int c = tid; c < dp.C; c += NTHREADS) {
    const int t0 = dp.comm_tile0[c], t1 = dp.comm_tile0[c + 1];
    if (t1 - t0 > BIG) continue;
    S_sh[c] = seq_sum_partials(src, t0, t1);
  }
  for (int i = 0; i < dp.n_big; ++i) {
    if (i > 0) __syncthreads();  // red is reused: warp 0 has read the previous iteration's
    const int c = dp.big_comm[i];
    const int t0 = dp.comm_tile0[c], t1 = dp.comm_tile0[c + 1];
    double x = 0.0, y = 0.0;
    for (int t = t0 + tid; t < t1; t += NTHREADS) {
      const double2 v = __ldcg(src + t);
      x += v.x;
      y += v.y;
    }
    block_sum2(x, y, red);  // its barrier also orders the small communities' S_sh before thread 0's reads
    if (tid == 0) S_sh[c] = make_double2(x, y);
  }
  if (dp.n_big == 0) __syncthreads();
  if (tid == 0) {  // T of this tile's community = sum over its dense column communities
    double x = 0.0, y = 0.0;
    for (int i = dp.D_ptr[c_own]; i < dp.D_ptr[c_own + 1]; ++i) {
      const double2 v = S_sh[dp.D_idx[i]];
      x += v.x;
      y += v.y;
    }
    *sT = make_double2(x, y);
  }
  if (want_rpsi) {  // uniform branch
    __syncthreads();          // thread 0's S_sh entries visible; red free
    double x = 0.0, y = 0.0;  // r e^{i psi} = (1/N) sum_b S_b
    for (int c = tid; c < dp.C; c += NTHREADS) {
      const double2 v = S_sh[c];
      x += v.x;
      y += v.y;
    }
    block_sum2(x, y, red);
    if (tid == 0) {
      const double cm = x / (double)dp.n, sm = y / (double)dp.n;
      const double r = sqrt(cm * cm + sm * sm);
      s_rpsi[0] = r;
      s_rpsi[1] = r == 0.0 ? 0.0 : atan2(sm, cm);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void record_rpsi(const DevPlan& dp, const double* rp, long long step) {
  Ctrl* ct = dp.ctrl;
  ct->rpsi[0] = rp[0];
  ct->rpsi[1] = rp[1];
  if (ct->record_every > 0 && ct->r_trace && step % ct->record_every == 0) {
    const long long i = step / ct->record_every;
    if (i < ct->nrec_cap) {
      ct->r_trace[2 * i] = rp[0];
      ct->r_trace[2 * i + 1] = rp[1];
    }
  }
}

// R = rows per thread (ceil(rows_per_tile / NTHREADS)): config 2's 3552-row tiles need 7, and every
// row slot held in registers costs two live doubles (theta_n, acc) across the whole trajectory
template <int R>
__global__ void __launch_bounds__(NTHREADS, 2) k_persist_rk4(const DevPlan dp, const StageArgs a, double2* pbuf,
                                                             unsigned long long* cnt, long long nsteps,
                                                             unsigned long long q0) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* zc = reinterpret_cast<double*>(smem_raw);  // [rows_per_tile] z of the stage state
  double* zsn = zc + dp.rows_per_tile;
  double* om = zsn + dp.rows_per_tile;                // [rows_per_tile] omega
  double2* S_sh = reinterpret_cast<double2*>(om + dp.rows_per_tile);  // [C]
  __shared__ double2 red[NWARPS];
  __shared__ double2 sT;
  __shared__ double s_rpsi[2];
  const int tid = threadIdx.x, lt = blockIdx.x;
  const TileDesc T = dp.tiles[lt];
  const int nt = gridDim.x;
  const bool rec = lt == 0 && dp.ctrl->record_every > 0;  // CTA 0 keeps (r, psi) and the record
  const int re = rec ? dp.ctrl->record_every : 0;
  const double KN = a.KN, K = a.K, h = a.h;
  const double* __restrict__ rs = dp.rowscale;
  double thn[R], acc[R];
  unsigned long long q = q0;  // publication counter (the arrival counter is monotonic across launches)
  // prologue: z(theta_n), the tile partial, S_b, T, (r, psi) of theta_0 (recorded as n = 0)
  double x = 0.0, y = 0.0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int lr = tid + k * NTHREADS;
    thn[k] = lr < T.nrows ? a.theta[T.row0 + lr - dp.row_begin] : 0.0;
    acc[k] = 0.0;
    if (lr < T.nrows) om[lr] = a.omega[T.row0 + lr - dp.row_begin];
  }
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int lr = tid + k * NTHREADS;
    if (lr >= T.nrows) break;
    double s, c;
    sincos(thn[k], &s, &c);
    zc[lr] = c;
    zsn[lr] = s;
    x += c;
    y += s;
  }
  block_sum2(x, y, red);
  publish_and_wait(pbuf, cnt, nt, lt, ++q, x, y);
  local_reduce(dp, pbuf, nt, q, S_sh, red, T.comm, &sT, s_rpsi, lt == 0);
  if (lt == 0 && tid == 0) record_rpsi(dp, s_rpsi, 0);
  bool bad = false;
  for (long long n = 0; n < nsteps; ++n) {
#pragma unroll 1
    for (int st = 1; st <= 4; ++st) {
      const double2 Tc = sT;
      const double wx = Tc.x + 0.0, wy = Tc.y + 0.0;  // W_j = T_c + (empty lists)
      const double hs = st == 4 ? h / 6.0 : (st == 3 ? h : h / 2.0);
      double px = 0.0, py = 0.0;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int lr = tid + k * NTHREADS;
        if (lr >= T.nrows) break;
        const double kn = rs ? K * rs[T.row0 + lr - dp.row_begin] : KN;
        const double kk = rhs_k(om[lr], kn, zc[lr], zsn[lr], wx, wy);
        double ts;
        if (st == 1) {
          acc[k] = kk;
          ts = __dadd_rn(thn[k], __dmul_rn(hs, kk));
        } else if (st < 4) {
          acc[k] = __dadd_rn(acc[k], __dmul_rn(2.0, kk));
          ts = __dadd_rn(thn[k], __dmul_rn(hs, kk));
        } else {  // theta_{n+1} = theta_n + (h/6)(k1 + 2k2 + 2k3 + k4)
          ts = __dadd_rn(thn[k], __dmul_rn(hs, __dadd_rn(acc[k], kk)));
          thn[k] = ts;
          bad |= !isfinite(ts);
        }
        double s, c;
        sincos(ts, &s, &c);
        zc[lr] = c;
        zsn[lr] = s;
        px += c;
        py += s;
      }
      block_sum2(px, py, red);
      publish_and_wait(pbuf, cnt, nt, lt, ++q, px, py);
      // (r, psi) only where it is recorded, or of the final state (ctrl->rpsi)
      const bool want = lt == 0 && st == 4 && ((re > 0 && (n + 1) % re == 0) || n + 1 == nsteps);
      local_reduce(dp, pbuf, nt, q, S_sh, red, T.comm, &sT, s_rpsi, want);
      if (want && tid == 0) record_rpsi(dp, s_rpsi, n + 1);
    }
  }
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int lr = tid + k * NTHREADS;
    if (lr < T.nrows) a.theta[T.row0 + lr - dp.row_begin] = thn[k];
  }
  if (bad) dp.ctrl->nonfinite = 1;
  if (lt == 0 && tid == 0) dp.ctrl->step = nsteps;
}

// world > 1: z of the non-local rows from the exchanged stage phases (the same
// sincos the owner evaluated -> bitwise identical), and every tile partial.
// Fused exchange: ONE thread waits until every rank's record of this stage has landed in xrecv
// (arrival counter, acquire at system scope); k_unpack is stream-ordered after it, so its blocks
// start on complete data instead of each spinning on the flag.
__global__ void k_wait_peers(const DevPlan dp, unsigned int expect) {
  unsigned int v;
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(dp.peer_flag[dp.rank]) : "memory");
    if ((int)(v - expect) >= 0) break;
    __nanosleep(64);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 20000000000ull) {  // 20 s: a rank is gone; fail loudly instead of hanging
      dp.ctrl->xtimeout = 1;
      break;
    }
  }
}

__global__ void k_unpack(const DevPlan dp, const double* __restrict__ xrecv, double2* __restrict__ zout) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < dp.n) {
    int r = 0;
    while (dp.shard_row0[r + 1] <= i) ++r;
    if (r != dp.rank) {
      double s, c;
      sincos(xrecv[(size_t)r * dp.xstride + (i - dp.shard_row0[r])], &s, &c);
      zout[i] = make_double2(c, s);
    }
  }
  const int64_t nt = dp.shard_tile0[dp.world];
  if (i < nt) {
    int r = 0;
    while (dp.shard_tile0[r + 1] <= i) ++r;
    const double* src = xrecv + (size_t)r * dp.xstride + dp.xrows + 3 * (i - dp.shard_tile0[r]);
    dp.partial[i] = make_double2(src[0], src[1]);
    dp.pmax[i] = src[2];
  }
}

// A rank without tiles still signals its (empty) contribution to a fused exchange.
__global__ void k_arrive(const DevPlan dp) {
  __threadfence_system();
  for (int r = 0; r < dp.world; ++r) atomicAdd_system(dp.peer_flag[r], 1u);
}

__global__ void __launch_bounds__(NTHREADS) k_finish(const DevPlan dp, const StageArgs a) {
  finish_reduce(dp, a);
}

// Variable-step RK4 (reading R25): per-tile partial of sum_m ((y2 - y1) / (atol + rtol |y2|))^2.
__global__ void __launch_bounds__(NTHREADS) k_errnorm(const DevPlan dp, const double* __restrict__ y1,
                                                      const double* __restrict__ y2, double atol, double rtol,
                                                      double* __restrict__ tile_ss) {
  __shared__ double2 red[NWARPS];
  const TileDesc T = dp.tiles[blockIdx.x];
  double ss = 0.0, dummy = 0.0;
  for (int lr = threadIdx.x; lr < T.nrows; lr += NTHREADS) {
    const int li = T.row0 + lr - dp.row_begin;
    const double b = y2[li];
    const double e = (b - y1[li]) / (atol + rtol * fabs(b));
    ss += e * e;
  }
  block_sum2(ss, dummy, red);
  if (threadIdx.x == 0) tile_ss[blockIdx.x] = ss;
}

__global__ void k_set_ctrl(Ctrl* c, int record_every, int nrec_cap, double* r_trace, double fp_tol) {
  c->fp_tol = fp_tol;
  c->record_every = record_every;
  c->nrec_cap = nrec_cap;
  c->r_trace = r_trace;
}

__global__ void k_permute(const int32_t* __restrict__ perm, int64_t n, const double* __restrict__ in,
                          double* __restrict__ out, int dir) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (dir == KUR_USER_TO_INTERNAL) out[i] = in[perm[i]];
  else out[perm[i]] = in[i];
}

// Launch with the programmatic-stream-serialization attribute (PDL) when dp.pdl (world 1, the
// kernels call pdl_wait_and_release first), else a plain launch.
template <class... P, class... A>
cudaError_t launch_maybe_pdl(bool pdl, void (*k)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

template <int MODE, bool RW, bool CR>
cudaError_t launch_stage_m(const DevPlan& dp, const StageArgs& a, cudaStream_t s) {
  static std::atomic<uint64_t> attr_set{0};  // one bit per device (the attribute is per device context)
  const size_t smem = stage_smem_bytes(MAX_TILE_ROWS) + (RW ? RING_BYTES : 0) +
                      (CR ? sizeof(double2) * (size_t)MAX_TILE_ROWS : 0);
  int dev = 0;
  cudaGetDevice(&dev);
  if (!((attr_set.load() >> (dev & 63)) & 1)) {
    cudaError_t e = cudaFuncSetAttribute(k_stage<MODE, RW, CR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(1ull << (dev & 63));
  }
  bool rov = false;
  if (dp.has_remote && !dp.remote_warp && !a.no_remote && a.phase != PHASE_A) {
    cudaError_t e = launch_remote(dp, a.zin, s);
    if (e != cudaSuccess) return e;
    rov = dp.rov > 0 && dp.world == 1 && a.phase == PHASE_FULL;
  }
  const size_t dyn = dp.has_parts ? stage_smem_bytes(dp.rows_per_tile) +
                                         ((dp.remote_warp == 1 || dp.remote_warp == 3) ? RING_BYTES : 0) +
                                         (CR ? sizeof(double2) * (size_t)dp.rows_per_tile : 0) : 0;
  CUtensorMap tm;  // remote_warp 3: the tensor map of the stage's input z (zA or zB)
  if (dp.tmaps) tm = dp.tmaps[a.zin == dp.zbuf[0] ? 0 : 1];
  else memset(&tm, 0, sizeof(tm));
  if (rov) {  // programmatic dependent of the k_remote just launched (it releases us at its start)
    StageArgs b = a;
    b.rov_wait = 1;
    return launch_maybe_pdl(true, k_stage<MODE, RW, CR>, dim3(dp.ntiles), dim3(NTHREADS), dyn, s, dp, b, tm);
  }
  return launch_maybe_pdl(dp.pdl != 0, k_stage<MODE, RW, CR>, dim3(dp.ntiles), dim3(NTHREADS), dyn, s, dp, a, tm);
}

template <int MODE>
cudaError_t launch_stage_m(const DevPlan& dp, const StageArgs& a, cudaStream_t s) {
  if (dp.remote_warp) return launch_stage_m<MODE, true, false>(dp, a, s);
  if (dp.cr_hot_warps > 0) return launch_stage_m<MODE, false, true>(dp, a, s);
  return launch_stage_m<MODE, false, false>(dp, a, s);
}

}  // namespace

#ifdef KUR_PROFILE
}  // namespace kur
extern "C" int kur_prof_attach(unsigned long long* p) {
  return (int)cudaMemcpyToSymbol(kur::g_prof, &p, sizeof(p));
}
namespace kur {
#endif

cudaError_t launch_remote(const DevPlan& dp, const double2* zin, cudaStream_t s) {
  if (!dp.has_remote || dp.remote_warp || dp.n_rchunks <= 0) return cudaSuccess;
  constexpr int wpb = KREM_THREADS / 32;
  static thread_local int dev_cached = -1, sms = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev != dev_cached) {
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    dev_cached = dev;
  }
  const long long need = (dp.n_rchunks + wpb - 1) / wpb,
                  full = (long long)(dp.rov > 0 ? dp.rov : KREM_CTAS_PER_SM) * sms;
  return launch_maybe_pdl(dp.pdl != 0, k_remote, dim3((unsigned)(need < full ? need : full)), dim3(KREM_THREADS), 0, s,
                          dp, zin);
}

size_t stage_smem_bytes(int rows_per_tile) { return sizeof(double2) * (size_t)(WZ + 8 + rows_per_tile); }

cudaError_t launch_prologue(const DevPlan& dp, const StageArgs& a, cudaStream_t s) {
  if (dp.ntiles <= 0) {
    if (dp.peer_x && a.xsend) k_arrive<<<1, 1, 0, s>>>(dp);
    return cudaGetLastError();
  }
  return launch_maybe_pdl(dp.pdl != 0, k_prologue, dim3(dp.ntiles), dim3(NTHREADS), 0, s, dp, a);
}

cudaError_t launch_stage(int mode, const DevPlan& dp, const StageArgs& a, cudaStream_t s) {
#ifdef KUR_DEBUG_BOUNDS
  {
    const uint32_t zl = (uint32_t)(dp.n + 1);  // real rows + the zero sentinel z[n]
    cudaMemcpyToSymbolAsync(g_dbg_zlen, &zl, sizeof(zl), 0, cudaMemcpyHostToDevice, s);
  }
#endif
  if (dp.ntiles <= 0) {  // no rows here; a fused exchange still counts this rank's arrival
    if (dp.peer_x && a.xsend && mode != MODE_RHS && a.phase != PHASE_A) k_arrive<<<1, 1, 0, s>>>(dp);
    return cudaGetLastError();
  }
  switch (mode) {
    case MODE_RHS: return launch_stage_m<MODE_RHS>(dp, a, s);
    case MODE_S1: return launch_stage_m<MODE_S1>(dp, a, s);
    case MODE_S2: return launch_stage_m<MODE_S2>(dp, a, s);
    case MODE_S3: return launch_stage_m<MODE_S3>(dp, a, s);
    case MODE_S4: return launch_stage_m<MODE_S4>(dp, a, s);
    case MODE_POT: return launch_stage_m<MODE_POT>(dp, a, s);
    case MODE_E1: return launch_stage_m<MODE_E1>(dp, a, s);
    case MODE_H1: return launch_stage_m<MODE_H1>(dp, a, s);
    case MODE_H2: return launch_stage_m<MODE_H2>(dp, a, s);
    case MODE_M0: return launch_stage_m<MODE_M0>(dp, a, s);
    case MODE_MI: return launch_stage_m<MODE_MI>(dp, a, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_small(const DevPlan& dp, const StageArgs& a, double2* zA, double2* zB, double2* TA, double2* TB,
                         long long nsteps, cudaStream_t s) {
  if (!dp.has_parts && dp.ntiles == 1) {  // registers + shared-memory reductions only
    k_small_dense<<<1, NTHREADS, 0, s>>>(dp, a, nsteps);
    return cudaGetLastError();
  }
  static std::atomic<uint64_t> attr_set{0};  // one bit per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!((attr_set.load() >> (dev & 63)) & 1)) {
    cudaError_t e = cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)stage_smem_bytes(MAX_TILE_ROWS));
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(1ull << (dev & 63));
  }
  k_small<<<1, NTHREADS, dp.has_parts ? stage_smem_bytes(dp.rows_per_tile) : 0, s>>>(dp, a, zA, zB, TA, TB, nsteps);
  return cudaGetLastError();
}

size_t persist_smem_bytes(const DevPlan& dp) {
  return sizeof(double) * 3 * (size_t)dp.rows_per_tile + sizeof(double2) * (size_t)std::max(dp.C, 1);
}

using PersistKernel = void (*)(const DevPlan, const StageArgs, double2*, unsigned long long*, long long,
                               unsigned long long);
// R = 1..4 rows per thread compile without spills; above that the kernel spills a few bytes either
// way and R = 8 measured faster than the exact R = 7 on config 2 (8.06 vs 8.19 us per stage,
// profiles/r02/notes/persist_r7_r8.log)
PersistKernel persist_kernel(const DevPlan& dp) {
  switch ((dp.rows_per_tile + NTHREADS - 1) / NTHREADS) {
    case 1: return k_persist_rk4<1>;
    case 2: return k_persist_rk4<2>;
    case 3: return k_persist_rk4<3>;
    case 4: return k_persist_rk4<4>;
    default: return k_persist_rk4<8>;
  }
}

bool persist_fits(const DevPlan& dp) {
  if (dp.world != 1 || dp.has_parts || dp.ntiles <= 0 || dp.rows_per_tile > MAX_TILE_ROWS_NOPARTS) return false;
  const size_t smem = persist_smem_bytes(dp);
  if (smem > 200 * 1024) return false;
  int dev = 0, sms = 0, nb = 0;
  const PersistKernel k = persist_kernel(dp);
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, NTHREADS, smem) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return (long long)nb * sms >= dp.ntiles;
}

cudaError_t launch_persist_rk4(const DevPlan& dp, const StageArgs& a, double2* pbuf, unsigned long long* cnt,
                               long long nsteps, unsigned long long q0, cudaStream_t s) {
  const size_t smem = persist_smem_bytes(dp);
  const PersistKernel k = persist_kernel(dp);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  DevPlan d = dp;
  StageArgs aa = a;
  void* args[] = {(void*)&d, (void*)&aa, (void*)&pbuf, (void*)&cnt, (void*)&nsteps, (void*)&q0};
  return cudaLaunchCooperativeKernel((const void*)k, dim3((unsigned)dp.ntiles), dim3(NTHREADS), args, smem, s);
}

cudaError_t launch_unpack(const DevPlan& dp, const double* xrecv, double2* zout, unsigned int expect,
                          cudaStream_t s) {
  const int64_t m = std::max<int64_t>(dp.n, (int64_t)1);
  const int bs = 256;
  if (dp.peer_x) k_wait_peers<<<1, 1, 0, s>>>(dp, expect);
  k_unpack<<<(unsigned)((m + bs - 1) / bs), bs, 0, s>>>(dp, xrecv, zout);
  return cudaGetLastError();
}

cudaError_t launch_finish(const DevPlan& dp, const StageArgs& a, cudaStream_t s) {
  k_finish<<<1, NTHREADS, 0, s>>>(dp, a);
  return cudaGetLastError();
}

cudaError_t launch_set_ctrl(Ctrl* c, int record_every, int nrec_cap, double* r_trace, double fp_tol,
                            cudaStream_t s) {
  k_set_ctrl<<<1, 1, 0, s>>>(c, record_every, nrec_cap, r_trace, fp_tol);
  return cudaGetLastError();
}

cudaError_t launch_errnorm(const DevPlan& dp, const double* y1, const double* y2, double atol, double rtol,
                           double* tile_ss, cudaStream_t s) {
  if (dp.ntiles <= 0) return cudaSuccess;
  k_errnorm<<<dp.ntiles, NTHREADS, 0, s>>>(dp, y1, y2, atol, rtol, tile_ss);
  return cudaGetLastError();
}

cudaError_t launch_permute(const int32_t* perm, int64_t n, const double* in, double* out, int dir,
                           cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int bs = 256;
  k_permute<<<(unsigned)((n + bs - 1) / bs), bs, 0, s>>>(perm, n, in, out, dir);
  return cudaGetLastError();
}

}  // namespace kur
