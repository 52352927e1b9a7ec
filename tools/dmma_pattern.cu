// DMMA throughput with a GEMM-like operand pattern: TM x TN accumulators fed by
// TM distinct A and TN distinct B fragments per k-step (fragments refreshed
// from shared memory every step or kept in registers).
#include <cstdio>
#include <cuda_runtime.h>
template <int TM, int TN, bool LDS>
__global__ void k(double *out, int iters) {
  __shared__ double sm[64 * 64];
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double acc[TM][TN][2];
  for (int i = 0; i < TM; ++i) for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int lane = threadIdx.x & 31;
  double af[TM], bf[TN];
  for (int i = 0; i < TM; ++i) af[i] = sm[lane + 32 * i];
  for (int j = 0; j < TN; ++j) bf[j] = sm[1024 + lane + 32 * j];
  for (int it = 0; it < iters; ++it) {
    if (LDS) {
      const int o = (it & 7) * 128;
#pragma unroll
      for (int i = 0; i < TM; ++i) af[i] = sm[o + lane + 32 * i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bf[j] = sm[2048 + o + lane + 32 * j];
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[i][j][0]), "+d"(acc[i][j][1]) : "d"(af[i]), "d"(bf[j]));
  }
  double s = 0;
  for (int i = 0; i < TM; ++i) for (int j = 0; j < TN; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 12345.0) out[0] = s;
}
template <int TM, int TN, bool LDS>
void run(int sms, double *out, int wps) {
  int wpb = wps < 16 ? wps : 16, bps = wps / wpb;
  int iters = 4096 * 16 / (TM * TN);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<TM, TN, LDS><<<sms * bps, wpb * 32>>>(out, iters);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<TM, TN, LDS><<<sms * bps, wpb * 32>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 5.0 * sms * bps * wpb * (double)iters * TM * TN * 512.0;
  printf("TM %d TN %d lds %d warps/SM %2d: %.2f TF/s\n", TM, TN, (int)LDS, wps, fl / (ms * 1e-3) / 1e12);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out; cudaMalloc(&out, 8);
  for (int w : {4, 8, 12, 16}) {
    run<4, 4, false>(sms, out, w); run<4, 4, true>(sms, out, w);
    run<2, 2, false>(sms, out, w); run<2, 2, true>(sms, out, w);
    run<8, 4, true>(sms, out, w); run<4, 8, true>(sms, out, w);
  }
  return 0;
}
