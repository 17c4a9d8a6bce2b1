// mb_lds.cu — microbenchmark (tooling, not product): the achievable rate of
// conflict-free 16-byte shared-memory gathers + fp64 accumulation on one SM,
// i.e. the ceiling of k_stage's hot loop.  Variants:
//   0: slot ids computed in registers (pure LDS.128 + DADD)
//   1: slot ids streamed from global memory as 16-bit pairs (k_stage's layout), L2-resident
//   2: as 1 with 4 independent accumulator pairs per lane
//   3: slot ids staged by per-warp TMA bulk copies (cp.async.bulk, 4-deep ring of 512-byte
//      groups, mbarrier per slot) and read back with LDS.128 (no LSU global loads)
//   5: slot ids staged per CTA in 48 KB blocks by one TMA bulk copy each, double-buffered,
//      1 CTA x 32 warps per SM (k_gather5)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_lds tools/mb_lds.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int NT = 512, WZ = 4096;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int VAR>
__global__ void __launch_bounds__(NT, 2) k_gather(const uint4* __restrict__ units, int ngroups, int reps, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  double2* zs = reinterpret_cast<double2*>(sm);
  for (int i = threadIdx.x; i < WZ; i += NT) zs[i] = make_double2(i * 1e-3, 1.0 - i * 1e-3);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double x0 = 0, y0 = 0, x1 = 0, y1 = 0, x2 = 0, y2 = 0, x3 = 0, y3 = 0;
  uint32_t h = 2654435761u * (blockIdx.x * NT + threadIdx.x + 1);
  for (int r = 0; r < reps; ++r) {
    for (int g = blockIdx.x * (NT / 32) + wid; g < ngroups; g += gridDim.x * (NT / 32)) {
      uint32_t w[4];
      if (VAR == 3) break;
      if (VAR == 0) {
        h = h * 1664525u + 1013904223u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t base = (h >> (q * 3)) & (WZ - 8);
          const uint32_t s0 = (base & ~7u) | ((lane + 2 * q) & 7), s1 = ((base ^ 0x5a8) & ~7u) | ((lane + 2 * q + 1) & 7);
          w[q] = s0 | (s1 << 16);
        }
      } else {
        const uint4 v = __ldg(units + (size_t)g * 32 + lane);
        w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 a = zs[w[q] & 0xFFFF], b = zs[w[q] >> 16];
        if (VAR == 2 && (q & 1)) { x2 += a.x; y2 += a.y; x3 += b.x; y3 += b.y; }
        else { x0 += a.x; y0 += a.y; x1 += b.x; y1 += b.y; }
      }
    }
  }
  if (VAR == 3) {
    constexpr int D = 4;
    uint4* ring = reinterpret_cast<uint4*>(sm + WZ * 16) + wid * D * 32;
    __shared__ __align__(8) uint64_t bar[NT / 32][D];
    if (lane < D) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[wid][lane])));
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    const int g0 = blockIdx.x * (NT / 32) + wid, gs = gridDim.x * (NT / 32);
    const long long per = ((long long)ngroups - g0 + gs - 1) / gs;  // groups of this warp per rep
    const long long total = per * reps;
    auto issue = [&](long long k) {
      const int g = (int)(g0 + (k % per) * gs);
      const int d = (int)(k % D);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[wid][d])), "r"(512) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(ring + d * 32)), "l"(units + (size_t)g * 32), "r"(512), "r"(sa(&bar[wid][d]))
                   : "memory");
    };
    if (lane == 0)
      for (long long k = 0; k < D && k < total; ++k) issue(k);
    uint32_t ph = 0;  // bit d = parity of slot d
    for (long long k = 0; k < total; ++k) {
      const int d = (int)(k % D);
      asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                       sa(&bar[wid][d])), "r"((ph >> d) & 1u) : "memory");
      ph ^= 1u << d;
      const uint4 v = ring[d * 32 + lane];
      __syncwarp();
      if (lane == 0 && k + D < total) issue(k + D);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 a = zs[w[q] & 0xFFFF], b = zs[w[q] >> 16];
        x0 += a.x; y0 += a.y; x1 += b.x; y1 += b.y;
      }
    }
  }
  out[blockIdx.x * NT + threadIdx.x] = x0 + x1 + x2 + x3 + 3 * (y0 + y1 + y2 + y3);
}

// variant 5: block-staged index stream (one CTA of 1024 threads per SM)
constexpr int NT5 = 1024, BLK5 = 96;  // groups per staged block (96 x 512 B = 48 KB)
__global__ void __launch_bounds__(NT5, 1) k_gather5(const uint4* __restrict__ units, int ngroups, int reps, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  double2* zs = reinterpret_cast<double2*>(sm);
  uint4* stage = reinterpret_cast<uint4*>(sm + WZ * 16);  // 2 x BLK5 x 32 units
  __shared__ __align__(8) uint64_t bar[2];
  for (int i = threadIdx.x; i < WZ; i += NT5) zs[i] = make_double2(i * 1e-3, 1.0 - i * 1e-3);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // this CTA's share: blocks b = blockIdx.x, blockIdx.x + gridDim.x, ... of BLK5 groups, per rep
  const int nblk = ngroups / BLK5;
  const int myb = (nblk - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const long long total = (long long)myb * reps;
  auto issue = [&](long long k) {
    const int b = (int)blockIdx.x + (int)(k % myb) * gridDim.x;
    const int d = (int)(k & 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[d])), "r"(BLK5 * 512) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa(stage + d * BLK5 * 32)), "l"(units + (size_t)b * BLK5 * 32), "r"(BLK5 * 512), "r"(sa(&bar[d]))
                 : "memory");
  };
  double x0 = 0, y0 = 0, x1 = 0, y1 = 0;
  if (threadIdx.x == 0) {
    if (total > 0) issue(0);
    if (total > 1) issue(1);
  }
  uint32_t ph = 0;
  for (long long k = 0; k < total; ++k) {
    const int d = (int)(k & 1);
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                     sa(&bar[d])), "r"((ph >> d) & 1u) : "memory");
    ph ^= 1u << d;
    const uint4* st = stage + d * BLK5 * 32;
    for (int g = wid; g < BLK5; g += NT5 / 32) {
      const uint4 v = st[g * 32 + lane];
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 a = zs[w[q] & 0xFFFF], b = zs[w[q] >> 16];
        x0 += a.x; y0 += a.y; x1 += b.x; y1 += b.y;
      }
    }
    __syncthreads();  // everybody done with buffer d
    if (threadIdx.x == 0 && k + 2 < total) issue(k + 2);
  }
  out[blockIdx.x * NT5 + threadIdx.x] = x0 + x1 + 3 * (y0 + y1);
}

int main(int argc, char** argv) {
  // default: 4096 groups x 512 B = 2 MB of index units (L2-resident); argv[1] groups (e.g. 4194304 = 2 GB: HBM)
  const int ngroups = argc > 1 ? atoi(argv[1]) : 4096;
  std::vector<uint32_t> hu((size_t)ngroups * 32 * 4);  // up to 2 GB
  uint32_t s = 12345;
  for (size_t i = 0; i < hu.size(); ++i) {
    const int lane = (int)((i / 4) % 32), q = (int)(i % 4);
    s = s * 1664525u + 1013904223u;
    const uint32_t b0 = (s >> 8) & (WZ - 8), b1 = (s >> 20) & (WZ - 8);
    hu[i] = (b0 | ((lane + 2 * q) & 7)) | ((b1 | ((lane + 2 * q + 1) & 7)) << 16);
  }
  uint4* du; double* dout;
  const int grid = 148 * 2, reps = argc > 2 ? atoi(argv[2]) : 20000;
  cudaMalloc(&du, hu.size() * 4);
  cudaMalloc(&dout, sizeof(double) * grid * NT);
  cudaMemcpy(du, hu.data(), hu.size() * 4, cudaMemcpyHostToDevice);
  const int smem = WZ * 16 + (NT / 32) * 4 * 512;
  cudaFuncSetAttribute(k_gather<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_gather<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_gather<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_gather<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int smem5 = WZ * 16 + 2 * BLK5 * 512;
  cudaFuncSetAttribute(k_gather5, cudaFuncAttributeMaxDynamicSharedMemorySize, smem5);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int var = 0; var < 6; ++var) {
    if (var == 4) continue;
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      if (var == 0) k_gather<0><<<grid, NT, smem>>>(du, ngroups, reps, dout);
      if (var == 1) k_gather<1><<<grid, NT, smem>>>(du, ngroups, reps, dout);
      if (var == 2) k_gather<2><<<grid, NT, smem>>>(du, ngroups, reps, dout);
      if (var == 3) k_gather<3><<<grid, NT, smem>>>(du, ngroups, reps, dout);
      if (var == 5) k_gather5<<<148, NT5, smem5>>>(du, ngroups, reps, dout);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) best = ms < best ? ms : best;
    }
    const double slots = (double)reps * (var == 5 ? (ngroups / BLK5) * BLK5 : ngroups) * 256;  // each group once per rep
    const double per_clk = slots / (best * 1e-3) / 148 / (1965e6);
    printf("var %d: %.3f ms, %.1f G slots/s, %.2f slots/clk/SM at 1965 MHz (peak 8), err=%s\n", var, best,
           slots / (best * 1e6), per_clk, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
