// DMMA.8x8x4 throughput vs warps per SM and independent accumulator chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double *out, int iters) {
  double c[CH][2];
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
template <int CH>
void run(int sms, double *out) {
  for (int wps = 4; wps <= 64; wps *= 2) {  // warps per SM
    int wpb = wps < 16 ? wps : 16, bps = wps / wpb;
    int iters = 2048 * 8 / CH;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<CH><<<sms * bps, wpb * 32>>>(out, iters);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k<CH><<<sms * bps, wpb * 32>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 5.0 * sms * bps * wpb * (double)iters * CH * 512.0;
    printf("chains %2d warps/SM %2d: %.2f TF/s\n", CH, wps, fl / (ms * 1e-3) / 1e12);
  }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out; cudaMalloc(&out, 8);
  run<1>(sms, out); run<2>(sms, out); run<4>(sms, out); run<8>(sms, out); run<16>(sms, out);
  return 0;
}
