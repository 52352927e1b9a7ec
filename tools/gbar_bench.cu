// Grid-barrier latency microbenchmark: a cooperative grid of G CTAs x 128 threads
// runs N barriers of (a) the fused GMRES kernel's gbar (atomic counter +
// generation word, volatile polling) and (b) cooperative_groups grid.sync().
// Usage: gbar_bench [G] [N]
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
namespace cg = cooperative_groups;

__device__ __forceinline__ void gbar(unsigned int *bar, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int *gen = bar + 1;
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// single-atomic version (the one the fused GMRES kernel uses now)
__device__ __forceinline__ void gbar1(unsigned int *bar, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int inc = blockIdx.x == 0 ? 0x80000000u - (nblocks - 1) : 1u;
    __threadfence();
    const unsigned int old = atomicAdd(bar, inc);
    volatile unsigned int *w = bar;
    while (((old ^ *w) & 0x80000000u) == 0) {
    }
    __threadfence();
  }
  __syncthreads();
}
__global__ void k_gbar1(unsigned int *bar, int n) {
  for (int i = 0; i < n; ++i) gbar1(bar, gridDim.x);
}
__global__ void k_gbar(unsigned int *bar, int n) {
  for (int i = 0; i < n; ++i) gbar(bar, gridDim.x);
}
__global__ void k_cg(int n) {
  cg::grid_group gg = cg::this_grid();
  for (int i = 0; i < n; ++i) gg.sync();
}

int main(int argc, char **argv) {
  int G = argc > 1 ? atoi(argv[1]) : 296, N = argc > 2 ? atoi(argv[2]) : 2000;
  unsigned int *bar;
  cudaMalloc(&bar, 64);
  cudaMemset(bar, 0, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int v = 0; v < 3; ++v) {
    void *a0[] = {&bar, &N};
    void *a1[] = {&N};
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      cudaMemset(bar, 0, 64);
      cudaError_t e = v == 0   ? cudaLaunchCooperativeKernel((void *)k_gbar, G, 128, a0, 0, 0)
                      : v == 1 ? cudaLaunchCooperativeKernel((void *)k_cg, G, 128, a1, 0, 0)
                               : cudaLaunchCooperativeKernel((void *)k_gbar1, G, 128, a0, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("%s G=%d: %.3f us per barrier (%s)\n", v == 0 ? "gbar (2 atomics)" : v == 1 ? "cg grid.sync" : "gbar (1 atomic)", G, 1e3 * ms / N,
                      cudaGetErrorString(e));
    }
  }
  return 0;
}
