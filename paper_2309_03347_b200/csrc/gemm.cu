// FP64 tensor-core GEMM for sm_100a: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).
// tcgen05 has no f64 kind, so FP64 tensor work on Blackwell is warp-level
// DMMA.  64x64x16 CTA tile, 4 warps of 32x32, operands staged
// through double-buffered shared memory with cp.async (zero-filled edges),
// descriptor read from device memory so sizes can follow device ranks.
#include "tt_common.cuh"

namespace tt {

// algorithmic flop counter of the contraction GEMMs (2 M N K per call) and launch count
__device__ unsigned long long g_gemm_counters[2];

namespace {

constexpr int BM = 64, BN = 64, BK = 16, PAD = 4;

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct Tile {
  double a[2][BK][BM + PAD];
  double b[2][BK][BN + PAD];
};

__device__ __forceinline__ void load_tile(Tile &t, int buf, const GemmDesc &g, int m0, int n0, int k0,
                                          int tid) {
  const double *A = g.A, *B = g.B;
  // A tile: BM x BK of op(A)
  if (!g.transA) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int m = tid & 63, k = (tid >> 6) + 2 * i;
      int gm = m0 + m, gk = k0 + k;
      bool p = gm < g.M && gk < g.K;
      const double *src = p ? A + gm + (long long)gk * g.lda : A;
      cp_async8(&t.a[buf][k][m], src, p);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int k = tid & 15, m = (tid >> 4) + 8 * i;
      int gm = m0 + m, gk = k0 + k;
      bool p = gm < g.M && gk < g.K;
      const double *src = p ? A + gk + (long long)gm * g.lda : A;
      cp_async8(&t.a[buf][k][m], src, p);
    }
  }
  if (!g.transB) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int k = tid & 15, n = (tid >> 4) + 8 * i;
      int gn = n0 + n, gk = k0 + k;
      bool p = gn < g.N && gk < g.K;
      const double *src = p ? B + gk + (long long)gn * g.ldb : B;
      cp_async8(&t.b[buf][k][n], src, p);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int n = tid & 63, k = (tid >> 6) + 2 * i;
      int gn = n0 + n, gk = k0 + k;
      bool p = gn < g.N && gk < g.K;
      const double *src = p ? B + gn + (long long)gk * g.ldb : B;
      cp_async8(&t.b[buf][k][n], src, p);
    }
  }
}

// splits > 1: split-K; CTA z computes the K-slice z and writes its raw partial
// product to partial + z * pstride (column-major, ld = pld); gemm_splitk_reduce
// sums the slices and applies the epilogue (deterministic order).
__global__ void __launch_bounds__(128) gemm_dmma_kernel(const GemmDesc *__restrict__ descs, int splits,
                                                        double *__restrict__ partial, long long pld,
                                                        long long pstride) {
  __shared__ __align__(16) Tile t;
  const GemmDesc g0 = descs[splits > 1 ? 0 : blockIdx.z];
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0 && g0.M > 0 && g0.N > 0) {
    atomicAdd(&g_gemm_counters[0], 2ull * (unsigned long long)g0.M * g0.N * (g0.K > 0 ? g0.K : 0));
    atomicAdd(&g_gemm_counters[1], 1ull);
  }
  if (m0 >= g0.M || n0 >= g0.N) return;
  GemmDesc g = g0;
  int kbeg = 0;
  if (splits > 1) {
    const int kc = ((g0.K + splits - 1) / splits + BK - 1) / BK * BK;
    kbeg = blockIdx.z * kc;
    const int kend = min(g0.K, kbeg + kc);
    g.K = kend > kbeg ? kend - kbeg : 0;
    // shift the operands to the K-slice
    g.A = g0.transA ? g0.A + kbeg : g0.A + (long long)kbeg * g0.lda;
    g.B = g0.transB ? g0.B + (long long)kbeg * g0.ldb : g0.B + kbeg;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (g.K + BK - 1) / BK;
  if (nk > 0) {
    load_tile(t, 0, g, m0, n0, 0, tid);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    cp_async_wait_all();
    __syncthreads();
    if (kt + 1 < nk) {
      load_tile(t, buf ^ 1, g, m0, n0, (kt + 1) * BK, tid);
      cp_async_commit();
    }
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = t.a[buf][kk + (lane & 3)][wm + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = t.b[buf][kk + (lane & 3)][wn + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
  if (splits > 1) {
    double *P = partial + (long long)blockIdx.z * pstride;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = m0 + wm + i * 8 + (lane >> 2);
      if (r >= g.M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = n0 + wn + j * 8 + (lane & 3) * 2 + h;
          if (c < g.N) P[r + c * pld] = acc[i][j][h];
        }
    }
    return;
  }
  double alpha = g.alpha;
  if (g.alpha_dev) alpha *= *g.alpha_dev;
  const double beta = g.beta;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + wm + i * 8 + (lane >> 2);
    if (r >= g.M) continue;
    const long long roff = (long long)(r % g.dr) * g.s_r0 + (long long)(r / g.dr) * g.s_r1;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = n0 + wn + j * 8 + (lane & 3) * 2 + h;
        if (c >= g.N) continue;
        const long long addr = roff + (long long)(c % g.dc) * g.s_c0 + (long long)(c / g.dc) * g.s_c1;
        double v = alpha * acc[i][j][h];
        if (beta != 0.0) v += beta * g.C[addr];
        g.C[addr] = v;
      }
    }
  }
}

__global__ void gemm_splitk_reduce(const GemmDesc *__restrict__ descs, int splits, const double *__restrict__ partial,
                                   long long pld, long long pstride) {
  const GemmDesc g = descs[0];
  const long long total = (long long)g.M * g.N;
  double alpha = g.alpha;
  if (g.alpha_dev) alpha *= *g.alpha_dev;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e % g.M), c = (int)(e / g.M);
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += partial[z * pstride + r + c * pld];
    const long long addr = (long long)(r % g.dr) * g.s_r0 + (long long)(r / g.dr) * g.s_r1 +
                           (long long)(c % g.dc) * g.s_c0 + (long long)(c / g.dc) * g.s_c1;
    double v = alpha * s;
    if (g.beta != 0.0) v += g.beta * g.C[addr];
    g.C[addr] = v;
  }
}

struct SplitScratch {
  double *ptr = nullptr;
  size_t bytes = 0;
};
thread_local SplitScratch g_split;

}  // namespace

void set_gemm_scratch(double *ptr, size_t bytes) {
  g_split.ptr = ptr;
  g_split.bytes = ptr ? bytes : 0;
}

tt_status launch_gemm(const GemmDesc *descs_dev, int count, int Mcap, int Ncap, cudaStream_t s) {
  return launch_gemm_k(descs_dev, count, Mcap, Ncap, 0, s);
}

tt_status launch_gemm_k(const GemmDesc *descs_dev, int count, int Mcap, int Ncap, int Kcap, cudaStream_t s) {
  if (count <= 0 || Mcap <= 0 || Ncap <= 0) return TT_OK;
  const int tm = (Mcap + BM - 1) / BM, tn = (Ncap + BN - 1) / BN;
  int splits = 1;
  if (count == 1 && Kcap >= 256 && (long long)tm * tn < 148) {
    splits = 296 / (tm * tn);
    splits = splits > Kcap / 128 ? Kcap / 128 : splits;
    splits = splits > 16 ? 16 : splits;
    const size_t need = (size_t)splits * Mcap * Ncap * sizeof(double);
    if (splits < 2 || !g_split.ptr || need > g_split.bytes) splits = 1;
  }
  if (splits > 1) {
    const long long pld = Mcap, pstride = (long long)Mcap * Ncap;
    gemm_dmma_kernel<<<dim3(tm, tn, splits), 128, 0, s>>>(descs_dev, splits, g_split.ptr, pld, pstride);
    int rb = (int)((pstride + 255) / 256);
    rb = rb > 1184 ? 1184 : (rb < 1 ? 1 : rb);
    gemm_splitk_reduce<<<rb, 256, 0, s>>>(descs_dev, splits, g_split.ptr, pld, pstride);
    return check_launch("gemm_dmma splitk");
  }
  dim3 grid(tm, tn, count);
  gemm_dmma_kernel<<<grid, 128, 0, s>>>(descs_dev, 1, nullptr, 0, 0);
  return check_launch("gemm_dmma");
}

void gemm_counters(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, g_gemm_counters, sizeof(g_gemm_counters));
  if (reset) {
    unsigned long long z[2] = {0, 0};
    cudaMemcpyToSymbol(g_gemm_counters, z, sizeof(z));
  }
}

}  // namespace tt
