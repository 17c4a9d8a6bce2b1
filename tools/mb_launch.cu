// mb_launch.cu — microbenchmark (tooling, not product): back-to-back launch cost of an empty kernel
// as a function of thread-block clusters, dynamic shared memory and grid size (CUDA events, 2000
// launches per variant).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_launch tools/mb_launch.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>

__global__ void __launch_bounds__(512, 1) k_empty(int* out, int sync) {
  extern __shared__ unsigned char sm[];
  if (sync) cooperative_groups::this_cluster().sync();
  if (threadIdx.x == 0 && out) sm[0] = 1;
}

int main() {
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int cls[] = {1, 2, 4, 8};
  const int smems[] = {0, 64 * 1024, 190 * 1024};
  const int grids[] = {120, 240, 296};
  for (int grid : grids)
    for (int smem : smems)
      for (int cl : cls)
        for (int sync = 0; sync < (cl > 1 ? 2 : 1); ++sync) {
          cudaLaunchConfig_t cfg{};
          cfg.gridDim = dim3(grid);
          cfg.blockDim = dim3(512);
          cfg.dynamicSmemBytes = smem;
          cfg.stream = s;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = cl;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          if (grid % cl) continue;
          for (int i = 0; i < 50; ++i) cudaLaunchKernelEx(&cfg, k_empty, (int*)nullptr, sync);
          cudaEventRecord(e0, s);
          const int N = 2000;
          for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, k_empty, (int*)nullptr, sync);
          cudaEventRecord(e1, s);
          cudaError_t err = cudaEventSynchronize(e1);
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          printf("grid %3d smem %6d cluster %d sync %d: %7.2f us per launch %s\n", grid, smem, cl, sync,
                 1000.0 * ms / N, err == cudaSuccess ? "" : cudaGetErrorString(err));
        }
  return 0;
}
