// FP64 peak microbenchmarks for B200 (K12 of SURVEY.md §2.6): DMMA
// (mma.sync.m8n8k4.f64, 8 independent accumulator chains per warp), DFMA
// (8 independent chains per thread) and an fp64 HBM copy.  Prints one JSON
// object.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks peaks_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_kernel(double *out, int iters) {
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_kernel(double *out, int iters) {
  double c[8];
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3 + i;
  const double a = 0.999999, b = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void copy_kernel(const double2 *__restrict__ a, double2 *__restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// L2-resident read bandwidth: every CTA sweeps the whole (L2-sized) buffer
__global__ void l2_read_kernel(const double2 *__restrict__ a, size_t n, int reps, double *out) {
  double2 acc = make_double2(0.0, 0.0);
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      const double2 v = __ldcg(a + i);
      acc.x += v.x;
      acc.y += v.y;
    }
  if (acc.x == 12345.0) out[0] = acc.y;
}

__global__ void fill_kernel(double2 *__restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = make_double2(1.0, 2.0);
}

template <class F>
float time_ms(F f, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  double *out;
  cudaMalloc(&out, 8);
  const int iters = 4096;
  // DMMA: sweep warps per block
  double best_dmma = 0;
  int best_w = 0;
  for (int warps = 4; warps <= 16; warps *= 2) {
    int blocks = sms * 4;
    float ms = time_ms([&] { dmma_kernel<<<blocks, warps * 32>>>(out, iters); }, 5);
    double flops = (double)blocks * warps * iters * 8 * 512.0;
    double tf = flops / (ms * 1e-3) / 1e12;
    if (tf > best_dmma) { best_dmma = tf; best_w = warps; }
  }
  double best_dfma = 0;
  for (int threads = 256; threads <= 1024; threads *= 2) {
    int blocks = sms * 4;
    float ms = time_ms([&] { dfma_kernel<<<blocks, threads>>>(out, iters); }, 5);
    double flops = (double)blocks * threads * iters * 8 * 2.0;
    double tf = flops / (ms * 1e-3) / 1e12;
    if (tf > best_dfma) best_dfma = tf;
  }
  // sustained DMMA: back to back for ~2 s
  float sus_ms = 0;
  int sus_launches = 0;
  {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (sus_launches = 0; sus_launches < 200; ++sus_launches)
      dmma_kernel<<<sms * 4, best_w * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&sus_ms, e0, e1);
  }
  double sus = (double)sms * 4 * best_w * iters * 8 * 512.0 * sus_launches / (sus_ms * 1e-3) / 1e12;
  size_t n = (size_t)1 << 27;  // 128M double2 = 2 GiB per buffer
  double2 *a, *b;
  cudaMalloc(&a, n * sizeof(double2));
  cudaMalloc(&b, n * sizeof(double2));
  cudaMemset(a, 0, n * sizeof(double2));
  float cms = time_ms([&] { copy_kernel<<<sms * 8, 512>>>(a, b, n); }, 10);
  double gbs = 2.0 * n * sizeof(double2) / (cms * 1e-3) / 1e9;
  float wms = time_ms([&] { fill_kernel<<<sms * 8, 512>>>(b, n); }, 10);
  double wgbs = 1.0 * n * sizeof(double2) / (wms * 1e-3) / 1e9;
  // L2: a 48 MB buffer read 20 times (well inside the 126 MB L2)
  const size_t nl2 = (size_t)48 * 1024 * 1024 / sizeof(double2);
  const int reps = 20;
  float lms = time_ms([&] { l2_read_kernel<<<sms * 4, 512>>>(a, nl2, reps, out); }, 5);
  double l2gbs = (double)reps * nl2 * sizeof(double2) / (lms * 1e-3) / 1e9;
  printf("{\"sms\": %d, \"l2_bytes\": %d, \"dmma_tflops_burst\": %.3f, \"dmma_tflops_sustained\": %.3f, "
         "\"dmma_best_warps_per_block\": %d, \"dfma_tflops_burst\": %.3f, \"hbm_copy_gbs\": %.1f, "
         "\"hbm_write_gbs\": %.1f, \"l2_read_gbs\": %.1f}\n",
         sms, l2, best_dmma, sus, best_w, best_dfma, gbs, wgbs, l2gbs);
  return 0;
}
