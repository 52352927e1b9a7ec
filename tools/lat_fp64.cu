// Latency micro-benchmark (clock64 cycles per dependent op) for the QR/Jacobi
// critical path on sm_100a: fp64 sqrt, div, rcp, rsqrt, warp_sum of doubles,
// __syncthreads at 1024 threads, shared-memory load.
#include <cstdio>
#include <cuda_runtime.h>
__device__ double sink;
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__global__ void lat(long long *out, double seed, int iters) {
  __shared__ double sm[1024];
  sm[threadIdx.x] = seed + threadIdx.x;
  __syncthreads();
  double x = seed + 1.0;
  long long t0, t1;
  // sqrt
  t0 = clock64(); for (int i = 0; i < iters; ++i) x = sqrt(x + 1.0); t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  // div
  t0 = clock64(); for (int i = 0; i < iters; ++i) x = 3.0 / (x + 1.0); t1 = clock64();
  if (threadIdx.x == 0) out[1] = (t1 - t0) / iters;
  // rcp (1/x)
  t0 = clock64(); for (int i = 0; i < iters; ++i) x = __drcp_rn(x + 1.0); t1 = clock64();
  if (threadIdx.x == 0) out[2] = (t1 - t0) / iters;
  // rsqrt
  t0 = clock64(); for (int i = 0; i < iters; ++i) x = rsqrt(x + 1.0); t1 = clock64();
  if (threadIdx.x == 0) out[3] = (t1 - t0) / iters;
  // fma
  t0 = clock64(); for (int i = 0; i < iters; ++i) x = fma(x, 0.999, 1e-3); t1 = clock64();
  if (threadIdx.x == 0) out[4] = (t1 - t0) / iters;
  // warp_sum
  t0 = clock64(); for (int i = 0; i < iters; ++i) x = warp_sum(x) * 1e-3; t1 = clock64();
  if (threadIdx.x == 0) out[5] = (t1 - t0) / iters;
  // syncthreads
  t0 = clock64(); for (int i = 0; i < iters; ++i) { x += 1e-9; __syncthreads(); } t1 = clock64();
  if (threadIdx.x == 0) out[6] = (t1 - t0) / iters;
  // smem dependent load
  int idx = threadIdx.x;
  t0 = clock64(); for (int i = 0; i < iters; ++i) { idx = ((int)sm[idx] + 1) & 1023; } t1 = clock64();
  if (threadIdx.x == 0) out[7] = (t1 - t0) / iters;
  // global load of a value this thread just wrote (L1 hit?)
  t0 = clock64(); for (int i = 0; i < iters; ++i) { double *p = (double *)&out[16 + (i & 7)]; if (threadIdx.x == 0) { *p = x; x = *(volatile double *)p + 1.0; } } t1 = clock64();
  if (threadIdx.x == 0) out[8] = (t1 - t0) / iters;
  sink = x + idx;
}
int main() {
  long long *d, h[32];
  cudaMalloc(&d, 32 * sizeof(long long));
  const char *nm[] = {"sqrt", "div", "rcp_rn", "rsqrt", "dfma", "warp_sum(f64)", "syncthreads(1024)", "lds dep", "st+ld global(volatile)"};
  for (int thr : {32, 1024}) {
    lat<<<1, thr>>>(d, 1.5, 256);
    lat<<<1, thr>>>(d, 1.5, 1024);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads %d\n", thr);
    for (int i = 0; i < 9; ++i) printf("  %-24s %lld cycles\n", nm[i], h[i]);
  }
  return 0;
}
