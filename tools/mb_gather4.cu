// mb_gather4.cu — microbenchmark (tooling, not product): random 16-byte z gathers
// through the LSU (one LDG.128 per entry, one L1 wavefront per touched line)
// versus TMA tile::gather4 into shared memory (4 entries per TMA op, read back
// with conflict-free LDS.128).  Same entries, same sums (up to order).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_gather4 tools/mb_gather4.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));     \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

constexpr int NT = 512, NW = NT / 32;

template <int KIND>
__device__ __forceinline__ double2 ldz(const double2* p) {
  double2 r;
  if (KIND == 0) return __ldg(p);
  if (KIND == 1) return __ldcg(p);
  if (KIND == 2) {
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
  }
  asm("ld.global.nc.L1::evict_first.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

// KIND 4: z via __ldg, index units as k_remote loads them (L1::no_allocate + L2 evict_first)
__device__ __forceinline__ uint4 ldg_idx(const uint4* p, int kind) {
  if (kind != 4) return __ldg(p);
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "l"(pol));
  return r;
}

template <int KIND>
__global__ void __launch_bounds__(NT, 2) k_ldg(const uint4* __restrict__ units, long long ngroups,
                                               const double2* __restrict__ z, double* out) {
  double x = 0, y = 0;
  const int lane = threadIdx.x & 31;
  const long long w = (long long)blockIdx.x * NW + (threadIdx.x >> 5), nw = (long long)gridDim.x * NW;
  for (long long g = w; g < ngroups; g += nw) {
    const uint4 u = ldg_idx(units + g * 32 + lane, KIND);
    const double2 a = ldz<KIND == 4 ? 0 : KIND>(z + u.x), b = ldz<KIND == 4 ? 0 : KIND>(z + u.y), c = ldz<KIND == 4 ? 0 : KIND>(z + u.z), d = ldz<KIND == 4 ? 0 : KIND>(z + u.w);
    x += a.x + b.x + c.x + d.x;
    y += a.y + b.y + c.y + d.y;
  }
  out[(size_t)blockIdx.x * NT + threadIdx.x] = x + 3.0 * y;
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(NT, 1) k_tma(const __grid_constant__ CUtensorMap tm, const uint4* __restrict__ units,
                                               long long ngroups, double* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[NW][2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double2* ring = reinterpret_cast<double2*>(sm) + wid * 512;  // 2 slots x 32 quads x 128 B (TMA dst 128-B aligned)
  if (lane < 2) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[wid][lane])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  const long long w = (long long)blockIdx.x * NW + wid, nw = (long long)gridDim.x * NW;
  uint32_t ph0 = 0, ph1 = 0;
  auto issue = [&](long long g, int s) {
    const uint4 u = __ldg(units + g * 32 + lane);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[wid][s])), "r"(2048)
                   : "memory");
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    void* dst = ring + s * 256 + lane * 8;  // quad (e = lane/8, m = lane%8) -> its own 128-byte slot
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sa(dst)),
        "l"(&tm), "r"(0), "r"((int)u.x), "r"((int)u.y), "r"((int)u.z), "r"((int)u.w), "r"(sa(&bar[wid][s]))
        : "memory");
  };
  double x = 0, y = 0;
  long long g0 = w;
  if (g0 < ngroups) issue(g0, 0);
  if (g0 + nw < ngroups) issue(g0 + nw, 1);
  int s = 0;
  for (long long g = g0; g < ngroups; g += nw, s ^= 1) {
    const uint32_t ph = s ? ph1 : ph0;
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            sa(&bar[wid][s])),
        "r"(ph)
        : "memory");
    if (s) ph1 ^= 1; else ph0 ^= 1;
    // quads were written as [e][lane-quad m]: entry e of lane l is at index e*32 + l
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double2 v = ring[s * 256 + (e * 8 + (lane >> 2)) * 8 + (lane & 3)];
      x += v.x;
      y += v.y;
    }
    __syncwarp();
    if (g + 2 * nw < ngroups) issue(g + 2 * nw, s);
  }
  out[(size_t)blockIdx.x * NT + threadIdx.x] = x + 3.0 * y;
}

int main(int argc, char** argv) {
  const long long n = argc > 2 ? atoll(argv[2]) : (1LL << 22), E = argc > 1 ? atoll(argv[1]) : (1LL << 26);
  const long long ngroups = E / 128;
  std::vector<double2> hz(n + 64);
  srand(1);
  for (auto& v : hz) v = make_double2(rand() / (double)RAND_MAX, rand() / (double)RAND_MAX);
  std::vector<uint32_t> idx(E);
  uint64_t s = 88172645463325252ull;
  // optional third argument: percentage of "padding" entries that all name one sentinel
  // column n (the layout's zero padding), placed in the last group of each 128-entry block
  const int pad_pct = argc > 3 ? atoi(argv[3]) : 0;
  for (size_t k = 0; k < idx.size(); ++k) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    idx[k] = (uint32_t)(s % n);
    if ((int)((k % 128) * 100 / 128) >= 100 - pad_pct) idx[k] = (uint32_t)n;
  }
  double2* dz; uint4* du; double* dout;
  CK(cudaMalloc(&dz, sizeof(double2) * (n + 64)));
  CK(cudaMalloc(&du, sizeof(uint32_t) * E));
  const int grid = 148 * 2;
  CK(cudaMalloc(&dout, sizeof(double) * grid * NT));
  CK(cudaMemcpy(dz, hz.data(), sizeof(double2) * (n + 64), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(du, idx.data(), sizeof(uint32_t) * E, cudaMemcpyHostToDevice));

  PFN_cuTensorMapEncodeTiled enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t gdim[2] = {2, (cuuint64_t)(n + 64)};
  cuuint64_t gstr[1] = {16};
  cuuint32_t box[2] = {2, 1}, es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dz, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  const int smem = NW * 512 * 16;
  CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  std::vector<double> ho(grid * NT);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  double sums[2];
  for (int which = 0; which < 6; ++which) {
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(a);
      if (which == 0) k_ldg<0><<<grid, NT>>>(du, ngroups, dz, dout);
      if (which == 1) k_tma<<<grid / 2, NT, smem>>>(tm, du, ngroups, dout);
      if (which == 2) k_ldg<1><<<grid, NT>>>(du, ngroups, dz, dout);
      if (which == 3) k_ldg<2><<<grid, NT>>>(du, ngroups, dz, dout);
      if (which == 4) k_ldg<3><<<grid, NT>>>(du, ngroups, dz, dout);
      if (which == 5) k_ldg<4><<<grid, NT>>>(du, ngroups, dz, dout);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) best = ms < best ? ms : best;
    }
    CK(cudaGetLastError());
    CK(cudaMemcpy(ho.data(), dout, sizeof(double) * grid * NT, cudaMemcpyDeviceToHost));
    if (which == 1) for (int i = grid / 2 * NT; i < grid * NT; ++i) ho[i] = 0;
    double t = 0; for (double v : ho) t += v;
    if (which < 2) sums[which] = t;
    const char* nm[6] = {"ldg.nc", "tma_gather4", "ldg.cg", "ldg.nc.L1::no_allocate", "ldg.nc.L1::evict_first",
                         "ldg.nc, index streamed (no_allocate + L2 evict_first)"};
    printf("%s: %.3f ms for %lld entries = %.2f G entries/s, sum %.10e\n", nm[which], best, E, E / (best * 1e6), t);
  }
  double ref = 0;
  for (long long i = 0; i < E; ++i) ref += hz[idx[i]].x + 3.0 * hz[idx[i]].y;
  printf("host sum %.10e  rel err ldg %.2e tma %.2e\n", ref, (sums[0] - ref) / ref, (sums[1] - ref) / ref);
  return 0;
}
