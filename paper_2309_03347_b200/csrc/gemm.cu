// FP64 tensor-core GEMM for sm_100a: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).
// tcgen05 has no f64 kind, so FP64 tensor work on Blackwell is warp-level
// DMMA.  Templated CTA tile (BM x BN x BK) of WARPS_M x
// WARPS_N warps, each computing a (BM/WARPS_M) x (BN/WARPS_N) block of 8x8
// DMMA tiles; operands staged through multi-stage cp.async shared-memory
// buffers (zero-filled edges); the descriptor is read from device memory so
// sizes can follow device-resident ranks; optional split-K with a
// deterministic slice reduction.
#include <cstdlib>

#include <cooperative_groups.h>
#include <string>
#include <vector>

#include "gmres.h"
#include "tt_common.cuh"

namespace tt {

// algorithmic flop counter of the contraction GEMMs (2 M N K per call) and launch count
__device__ unsigned long long g_gemm_counters[2];
// fused GMRES step kernel: [0] local-apply GEMM flops, [1] CGS2 / norm vector flops, [2] steps
__device__ unsigned long long g_gm_counters[3];
// per-tag (AMEn core index) Arnoldi steps of the fused kernel (tt_fused_profile_cores)
__device__ unsigned long long g_gm_tag_steps[TT_MAX_D];
// per-tag in-kernel duration (%globaltimer ns, CTA 0 from entry to exit) and launches that
// did work: the fused kernel's timing when it runs inside device-resident graph loops,
// where no host-recorded event can bracket an individual launch
__device__ unsigned long long g_gm_tag_ns[TT_MAX_D];
__device__ unsigned long long g_gm_tag_launches[TT_MAX_D];

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

namespace {

constexpr int PAD = 4;

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int BM, int BN, int BK, int WM_, int WN_, int STAGES>
struct Cfg {
  static constexpr int WARPS = WM_ * WN_;
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int TM = BM / WM_ / 8;  // 8x8 tiles per warp along M
  static constexpr int TN = BN / WN_ / 8;
  static constexpr int A_ELEMS = BK * (BM + PAD);
  static constexpr int B_ELEMS = BK * (BN + PAD);
  static constexpr size_t SMEM = (size_t)STAGES * (A_ELEMS + B_ELEMS) * sizeof(double);
};

// Two-level scatter index idx -> (idx % d) s0 + (idx / d) s1 walked incrementally:
// one division per thread and tile, then carries (the epilogue's per-row and
// per-column divisions were 11% of the fused GMRES kernel's stall samples).
struct ScatIdx {
  int q, rem, d;
  __device__ __forceinline__ void init(int idx, int d_) {
    d = d_ > 0 ? d_ : (1 << 30);
    q = idx / d;
    rem = idx - q * d;
  }
  __device__ __forceinline__ void advance(int step) {
    rem += step;
    while (rem >= d) { rem -= d; ++q; }
  }
  __device__ __forceinline__ long long off(long long s0, long long s1) const { return (long long)rem * s0 + (long long)q * s1; }
};

// Operand tile loader with strength-reduced addressing.  An operand tile is
// MN x BK (MN = BM rows of A or BN columns of B) staged as smem[k][MN + PAD].
// Each thread owns NI = MN BK / T elements whose (mn, k) positions inside the
// tile never change, so the global address of element i at k-tile kt is
// p + i istride + kt kstep: one pointer, advanced once per k-tile, instead of a
// 64-bit multiply, two divisions and two bound tests per element and k-tile
// (ncu source page of the round-2 fused GMRES kernel: ~50 SASS instructions per
// cp.async, as many issue slots in the load code as in the DMMA block).
//   mn-contiguous operand (A not transposed, B transposed): thread -> mn = tid % MN,
//     k = tid / MN + i (T / MN); the mn bound is one bit, the k bound per element.
//   k-contiguous operand (A transposed, B not transposed): thread -> k = tid % BK,
//     mn = tid / BK + i (T / BK); the k bound is one test, the mn bounds a bit mask.
template <int MN, int BK, int T>
struct OpLoader {
  static constexpr int NI = MN * BK / T;
  static_assert(T % MN == 0 && T % BK == 0 && NI >= 1 && NI <= 32, "tile / thread-count mismatch");
  const double *p;      // element 0 of this thread at the next k-tile to load
  const double *safe;   // any valid address (predicated-off copies read nothing)
  long long istride, kstep;
  unsigned mask;        // bit i: element i inside the mn range
  int soff;             // smem offset of element 0
  int kfirst;           // k index of element 0 inside a k-tile
  int K;
  bool kc;              // k-contiguous operand
  __device__ __forceinline__ void init(const double *base, long long ld, bool kcontig, int mn0, int MNtot, int K_,
                                       int tid) {
    kc = kcontig;
    K = K_;
    safe = base;
    if (!kc) {
      const int mn = tid % MN, kk = tid / MN;
      p = base + (mn0 + mn) + (long long)kk * ld;
      istride = (long long)(T / MN) * ld;
      kstep = (long long)BK * ld;
      soff = kk * (MN + PAD) + mn;
      kfirst = kk;
      mask = (mn0 + mn < MNtot) ? 0xffffffffu : 0u;
    } else {
      const int kk = tid % BK, mn = tid / BK;
      p = base + kk + (long long)(mn0 + mn) * ld;
      istride = (long long)(T / BK) * ld;
      kstep = BK;
      soff = kk * (MN + PAD) + mn;
      kfirst = kk;
      unsigned mk = 0;
#pragma unroll
      for (int i = 0; i < NI; ++i)
        if (mn0 + mn + i * (T / BK) < MNtot) mk |= 1u << i;
      mask = mk;
    }
  }
  // load the k-tile starting at k0 (k-tiles must be requested in increasing order)
  __device__ __forceinline__ void load(double *sbuf, int k0) {
    const double *q = p;
    if (!kc) {
      const bool mok = mask != 0;
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const bool pr = mok && (k0 + kfirst + i * (T / MN) < K);
        cp_async8(sbuf + soff + i * ((T / MN) * (MN + PAD)), pr ? q : safe, pr);
        q += istride;
      }
    } else {
      const bool kok = k0 + kfirst < K;
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const bool pr = kok && ((mask >> i) & 1u);
        cp_async8(sbuf + soff + i * (T / BK), pr ? q : safe, pr);
        q += istride;
      }
    }
    p += kstep;
  }
};

// splits > 1: split-K; CTA z computes the K-slice z and writes its raw partial
// product to partial + z * pstride (column-major, ld = pld); gemm_splitk_reduce
// sums the slices and applies the epilogue (deterministic order).

// One output tile (m0, n0) of the K-slice z (splits > 1) or of the whole K.
template <int BM, int BN, int BK, int WM_, int WN_, int STAGES>
__device__ __forceinline__ void gemm_tile(const GemmDesc &g0, int m0, int n0, int z, int splits,
                                          double *__restrict__ partial, long long pld, long long pstride,
                                          double *smem) {
  using C = Cfg<BM, BN, BK, WM_, WN_, STAGES>;
  double *sA = smem;
  double *sB = smem + STAGES * C::A_ELEMS;
  if (m0 >= g0.M || n0 >= g0.N) return;
  GemmDesc g = g0;
  if (splits > 1) {
    const int kc = ((g0.K + splits - 1) / splits + BK - 1) / BK * BK;
    const int kbeg = z * kc;
    const int kend = min(g0.K, kbeg + kc);
    g.K = kend > kbeg ? kend - kbeg : 0;
    g.A = g0.transA ? g0.A + kbeg : g0.A + (long long)kbeg * g0.lda;
    g.B = g0.transB ? g0.B + (long long)kbeg * g0.ldb : g0.B + kbeg;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp % WM_) * (BM / WM_), wn = (warp / WM_) * (BN / WN_);
  double acc[C::TM][C::TN][2];
#pragma unroll
  for (int i = 0; i < C::TM; ++i)
#pragma unroll
    for (int j = 0; j < C::TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (g.K + BK - 1) / BK;
  OpLoader<BM, BK, C::THREADS> la;
  OpLoader<BN, BK, C::THREADS> lb;
  la.init(g.A, g.lda, g.transA != 0, m0, g.M, g.K, tid);
  lb.init(g.B, g.ldb, g.transB == 0, n0, g.N, g.K, tid);
  // prologue: STAGES-1 tiles in flight
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nk) {
      la.load(sA + st * C::A_ELEMS, st * BK);
      lb.load(sB + st * C::B_ELEMS, st * BK);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {  // issue the load of tile kt + STAGES - 1 into the slot freed at kt - 1
      const int nt = kt + STAGES - 1;
      if (nt < nk) {
        const int sl = nt % STAGES;
        la.load(sA + sl * C::A_ELEMS, nt * BK);
        lb.load(sB + sl * C::B_ELEMS, nt * BK);
      }
      cp_async_commit();
    }
    const double *a = sA + (kt % STAGES) * C::A_ELEMS;
    const double *b = sB + (kt % STAGES) * C::B_ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[C::TM], bf[C::TN];
      const int kr = kk + (lane & 3);
#pragma unroll
      for (int i = 0; i < C::TM; ++i) af[i] = a[kr * (BM + PAD) + wm + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < C::TN; ++j) bf[j] = b[kr * (BN + PAD) + wn + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < C::TM; ++i)
#pragma unroll
        for (int j = 0; j < C::TN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  if (splits > 1) {
    double *P = partial + (long long)z * pstride;
#pragma unroll
    for (int i = 0; i < C::TM; ++i) {
      const int r = m0 + wm + i * 8 + (lane >> 2);
      if (r >= g.M) continue;
#pragma unroll
      for (int j = 0; j < C::TN; ++j)
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
  // scatter offsets: one div/mod per owned row and column (not per element)
  long long coff[C::TN][2];
  ScatIdx ci, ri;
  ci.init(n0 + wn + (lane & 3) * 2, g.dc);
#pragma unroll
  for (int j = 0; j < C::TN; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = n0 + wn + j * 8 + (lane & 3) * 2 + h;
      coff[j][h] = (c < g.N) ? ci.off(g.s_c0, g.s_c1) : -1;
      ci.advance(h == 0 ? 1 : 7);
    }
  ri.init(m0 + wm + (lane >> 2), g.dr);
#pragma unroll
  for (int i = 0; i < C::TM; ++i) {
    const int r = m0 + wm + i * 8 + (lane >> 2);
    const long long roff = ri.off(g.s_r0, g.s_r1);
    ri.advance(8);
    if (r >= g.M) continue;
#pragma unroll
    for (int j = 0; j < C::TN; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (coff[j][h] < 0) continue;
        const long long addr = roff + coff[j][h];
        double v = alpha * acc[i][j][h];
        if (beta != 0.0) v += beta * g.C[addr];
        g.C[addr] = v;
      }
    }
  }
}

// splits > 1: each K-slice CTA writes its raw partial tile; gemm_splitk_reduce
// sums the slices in slice order (deterministic) and applies the epilogue.
template <int BM, int BN, int BK, int WM_, int WN_, int STAGES>
#ifndef GEMM_MINB
#define GEMM_MINB 4   // 64x64 tiles: 128 registers, 4 CTAs per SM (C5 r=256 17.3 -> 18.2 TF/s in the same run; 5 measured slower)
#endif
__global__ void __launch_bounds__(32 * WM_ * WN_, (BM == 64 && BN == 64) ? GEMM_MINB : 1)
    gemm_dmma_kernel(const GemmDesc *__restrict__ descs, int splits,
                                                                   double *__restrict__ partial, long long pld,
                                                                   long long pstride) {
  extern __shared__ __align__(16) double smem[];
  // batched descriptor (count 1, no split-K): grid z = batch capacity, z = problem index
  GemmDesc g0 = descs[0];
  const bool batched = g0.batch >= 1;
  if (!batched) g0 = descs[splits > 1 ? 0 : blockIdx.z];
  if (g0.skip && *g0.skip) return;
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0 && g0.M > 0 && g0.N > 0) {
    atomicAdd(&g_gemm_counters[0], 2ull * (unsigned long long)g0.M * g0.N * (g0.K > 0 ? g0.K : 0) * gemm_nbatch(g0));
    atomicAdd(&g_gemm_counters[1], 1ull);
  }
  int z = blockIdx.z;
  if (batched) {
    if ((int)blockIdx.z >= g0.batch) return;
    g0 = gemm_batch_item(g0, blockIdx.z);
    z = 0;
  }
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  gemm_tile<BM, BN, BK, WM_, WN_, STAGES>(g0, m0, n0, z, splits, partial, pld, pstride, smem);
}

__global__ void gemm_splitk_reduce(const GemmDesc *__restrict__ descs, int splits, const double *__restrict__ partial,
                                   long long pld, long long pstride) {
  const GemmDesc g = descs[0];
  if (g.skip && *g.skip) return;
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

// ---- variants: (BM, BN, BK, warps M, warps N, stages)
template <int BM, int BN, int BK, int WM_, int WN_, int ST>
struct Variant {
  using C = Cfg<BM, BN, BK, WM_, WN_, ST>;
  static constexpr int bm = BM, bn = BN;
  static void prepare() {
    static bool done = false;
    if (!done) {
      cudaFuncSetAttribute(gemm_dmma_kernel<BM, BN, BK, WM_, WN_, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)C::SMEM);
      done = true;
    }
  }
  static void launch(dim3 grid, const GemmDesc *d, int splits, double *p, long long pld, long long ps, cudaStream_t s) {
    prepare();
    gemm_dmma_kernel<BM, BN, BK, WM_, WN_, ST><<<grid, C::THREADS, C::SMEM, s>>>(d, splits, p, pld, ps);
  }
};

// (64x64x32 3-stage, 128x64, 128x128 and 3/4-stage 64x64 variants were measured
// slower on the B200 in round 1 and removed)
using V64 = Variant<64, 64, 16, 2, 2, 2>;
using V32 = Variant<32, 32, 16, 2, 2, 2>;     // small tiles for GEMMs that fill less than a wave

int small_tiles_enabled() {
  static int v = -1;
  if (v < 0) v = std::getenv("TT_GEMM_NOSMALL") ? 0 : 1;
  return v;
}
int small_tiles_waves() {   // use 32x32 tiles below this many 64x64 tiles
  static int v = -1;
  if (v < 0) { const char *e = std::getenv("TT_GEMM_SMALL_T"); v = e ? std::atoi(e) : 296; }
  return v;
}
int small_tiles_kmax() {
  static int v = -1;
  if (v < 0) { const char *e = std::getenv("TT_GEMM_SMALL_K"); v = e ? std::atoi(e) : 256; }
  return v;
}

template <class Vt>
tt_status launch_variant(const GemmDesc *descs_dev, int count, int Mcap, int Ncap, int Kcap, cudaStream_t s,
                         int batch) {
  const int tm = (Mcap + Vt::bm - 1) / Vt::bm, tn = (Ncap + Vt::bn - 1) / Vt::bn;
  const int nb = batch >= 1 ? batch : 1;
  const int zdim = batch >= 1 ? batch : count;
  // less than one wave of 64x64 tiles and a short K (no split-K), or a thin batched
  // problem: 32x32 tiles (4x the CTAs, less padding)
  if (Vt::bm == 64 && Vt::bn == 64 && small_tiles_enabled() &&
      (((long long)tm * tn * count * nb < small_tiles_waves() && Kcap < small_tiles_kmax()) ||
       (batch >= 1 && (Mcap <= 32 || Ncap <= 32)))) {
    const int sm_ = (Mcap + 31) / 32, sn_ = (Ncap + 31) / 32;
    V32::launch(dim3(sm_, sn_, zdim), descs_dev, 1, nullptr, 0, 0, s);
    return check_launch("gemm_dmma small tiles");
  }
  if (batch >= 1) {
    Vt::launch(dim3(tm, tn, zdim), descs_dev, 1, nullptr, 0, 0, s);
    return check_launch("gemm_dmma batched");
  }
  static int tgt = -1, kmin = -1;
  if (tgt < 0) {
    const char *a = std::getenv("TT_SPLIT_TARGET"), *b = std::getenv("TT_SPLIT_KMIN");
    tgt = a ? std::atoi(a) : 296;     // aim for ~2 waves of CTAs
    kmin = b ? std::atoi(b) : 64;     // minimum K per slice (64 measured best: C5 r=128, C1)
  }
  int splits = 1;
  if (count == 1 && Kcap >= 2 * kmin && (long long)tm * tn < 148) {
    splits = tgt / (tm * tn);
    splits = splits > Kcap / kmin ? Kcap / kmin : splits;
    splits = splits > 16 ? 16 : splits;
    const size_t need = (size_t)splits * Mcap * Ncap * sizeof(double);
    if (splits < 2 || !g_split.ptr || need > g_split.bytes) splits = 1;
  }
  if (splits > 1) {
    const long long pld = Mcap, pstride = (long long)Mcap * Ncap;
    Vt::launch(dim3(tm, tn, splits), descs_dev, splits, g_split.ptr, pld, pstride, s);
    int rb = (int)((pstride + 255) / 256);
    rb = rb > 1184 ? 1184 : (rb < 1 ? 1 : rb);
    gemm_splitk_reduce<<<rb, 256, 0, s>>>(descs_dev, splits, g_split.ptr, pld, pstride);
    return check_launch("gemm_dmma splitk");
  }
  Vt::launch(dim3(tm, tn, count), descs_dev, 1, nullptr, 0, 0, s);
  return check_launch("gemm_dmma");
}

// ------------------------------------------------ fused GMRES Arnoldi steps ---
// One cooperative persistent launch runs Arnoldi steps j0..j1-1 of the device
// GMRES (gmres.cu) for the AMEn local system: per step the three chained
// local-apply GEMM stages (descriptors gapp[3(j+1)+s], DMMA tiles distributed
// over the CTAs, split-K with an in-kernel reduction when a stage has few
// tiles), then CGS2 (two dot/axpy passes), the norm, the Givens update and the
// normalisation of the new basis vector.  Every CTA owns a slice of the local
// vector; the cross-CTA sums are reduced redundantly (same order) by every
// CTA, so all CTAs take identical decisions and only grid barriers separate
// the phases (6-7 per step instead of ~8 kernel launches).
constexpr int GF_THREADS = 128;
#ifndef GF_ST
#define GF_ST 2
#endif
#ifndef GF_MAXSPLIT
#define GF_MAXSPLIT 32   // measured: 16 -> 32 = 10.68 -> 10.25 ms per large C4 fused-GMRES launch
#endif
#ifndef GF_BK
#define GF_BK 16
#endif
#ifndef GF_EFF32
#define GF_EFF32 0.8   // DMMA efficiency of a 32x32 tile relative to 64x64 in the stage-time model
#endif
#ifndef GF_FLEX
#define GF_FLEX 1      // flexible streamed tiles for the plain stage GEMMs of the persistent kernel
#endif
#ifndef GF_FLEX_FIXED
#define GF_FLEX_FIXED 1.0   // fixed cost of a tile (epilogue, bookkeeping) in k-tiles
#endif
#ifndef GF_FLEX_LDS
#define GF_FLEX_LDS 0.5     // cost of a fragment load relative to a DMMA
#endif
#ifndef GF_FLEX_KT0
#define GF_FLEX_KT0 4.0     // per-k-tile overhead of a warp (barrier, cp.async issue) in DMMA units
#endif
#ifndef GF_FLEX_RED
#define GF_FLEX_RED 0.25    // cost of one split-K slice element in the reduction pass
#endif
using GF = Cfg<64, 64, GF_BK, 2, 2, GF_ST>;   // persistent-kernel tiles
constexpr int GF_LD = GM_MAX_M + 2;
constexpr int GF_MAX_GRID = 1024;   // partial-sum buffer capacity (gmres_fused_part_doubles)
// dynamic shared memory of the fused kernel: GEMM tile buffers + the apply
// descriptors of up to GM_MAX_M steps
#ifndef GF_FS
#define GF_FS 2        // pipeline slots of the flexible streamed tiles (3 slots measured 17% slower on C4:
                       // 2 x 87 KB of shared memory per SM leave 60 KB of L1 for the operands shared by a stage's tiles)
#endif
constexpr size_t GF_FLEX_SMEM = (size_t)GF_FS * (GF::A_ELEMS + GF::B_ELEMS) * sizeof(double);
constexpr size_t GF_TILE_SMEM = GF::SMEM > GF_FLEX_SMEM ? GF::SMEM : GF_FLEX_SMEM;
constexpr size_t GM_SMEM = GF_TILE_SMEM + (size_t)3 * sizeof(GemmDesc);

// Software grid barrier with one atomic per CTA: the arrival word counts up and
// the last arriver's increment flips its top bit (CTA 0 adds 0x80000000 -
// (nblocks - 1), the others 1), so a waiter is released when the top bit
// differs from the one it saw — no reset store and no second generation atomic
// on the release path (the two-atomic version measured 2.5 us per barrier at
// 296 CTAs, tools/gbar_bench.cu).  The word must start at 0 and every barrier
// must see all nblocks CTAs.
__device__ __forceinline__ void gbar(unsigned int *bar, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int inc = blockIdx.x == 0 ? 0x80000000u - (nblocks - 1) : 1u;
    __threadfence();
    const unsigned int old = atomicAdd(bar, inc);
    volatile unsigned int *w = bar;
    unsigned int spins = 0;
    const long long t0 = clock64();
    while (((old ^ *w) & 0x80000000u) == 0) {
      if ((++spins & 1023u) == 0 && clock64() - t0 > 8000000000LL) __trap();   // never hang the device
    }
    __threadfence();
  }
  __syncthreads();
}

// The same barrier split into arrival and wait, so work that nobody else waits
// for (the Givens update of an Arnoldi step) overlaps the barrier's latency.
// The token is meaningful in thread 0 only.
__device__ __forceinline__ unsigned int gbar_arrive(unsigned int *bar, unsigned int nblocks) {
  __syncthreads();
  unsigned int old = 0;
  if (threadIdx.x == 0) {
    const unsigned int inc = blockIdx.x == 0 ? 0x80000000u - (nblocks - 1) : 1u;
    __threadfence();
    old = atomicAdd(bar, inc);
  }
  return old;
}
__device__ __forceinline__ void gbar_wait(unsigned int *bar, unsigned int old) {
  if (threadIdx.x == 0) {
    volatile unsigned int *w = bar;
    unsigned int spins = 0;
    const long long t0 = clock64();
    while (((old ^ *w) & 0x80000000u) == 0) {
      if ((++spins & 1023u) == 0 && clock64() - t0 > 8000000000LL) __trap();   // never hang the device
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct GmChunkArgs {
  GmState *st;
  const GemmDesc *gapp;
  double *V;
  long long ldv;
  double *w;
  double *part;          // [3][G][GF_LD]
  double *split;
  long long split_elems;
  unsigned int *bar;
  int j0, j1;
  int mode;              // 0 grid only, 1 cluster only, 2 device decides (both variants launched)
  int cs;                // cluster size (for the device-side choice)
  int full;              // 1: the whole restarted solve (start, cycles, updates) in this launch
  int max_restarts;
  const double *b;       // full: right-hand side
  double *x;             // full: initial guess in, solution out
  int tag;               // profiling tag (AMEn core index, < TT_MAX_D)
};

// ---- flexible streamed tiles for the persistent kernel --------------------
// The stage GEMMs of the C4 local applies have awkward sizes (ranks 132 = 128 +
// kickrank, 264, R m = 68 / 152 rows) and a short K (132 - 152): fixed 64x64
// tiles lost 20-45% of their DMMAs to padding, up to 40% of a stage to the last
// partial round of tiles over the grid, and paid the pipeline prologue and the
// scattered epilogue once per tile.  Here every warp computes a x b units of
// 8 x 8 (a, b <= 4, the same for all warps of a stage: 12 compiled shapes), the
// 4 warps are laid out 2 x 2 or 1 x 4, so a CTA tile is (WM a) x (WN b) units;
// the shape is chosen per stage by a small cost model (rounds of tiles over the
// grid x k-tiles x DMMAs and fragment loads of a warp), and a CTA streams
// through all its (tile, k-tile) pairs in ONE software pipeline: the first
// k-tile of the next output tile is in flight while the current tile's last
// k-tile is multiplied and its epilogue is stored.
struct FlexPlan {
  int a, b, wm;           // warp tile in units, warps along M (1 or 2; along N: 4 / wm)
  int tm, tn, splits, kc; // tiles per dimension, K slices, K per slice (multiple of BK)
};
struct FlexTile {
  int m0, n0, z, kbeg, klen, nk;
};
__device__ __forceinline__ FlexTile flex_tile(const GemmDesc &g, const FlexPlan &pl, int w) {
  FlexTile t;
  const int T = pl.tm * pl.tn;
  t.z = w / T;
  const int tt = w - t.z * T;
  t.m0 = (tt % pl.tm) * (8 * pl.wm * pl.a);
  t.n0 = (tt / pl.tm) * (8 * (4 / pl.wm) * pl.b);
  t.kbeg = t.z * pl.kc;
  const int kend = min(g.K, t.kbeg + pl.kc);
  t.klen = kend > t.kbeg ? kend - t.kbeg : 0;
  t.nk = max(1, (t.klen + GF_BK - 1) / GF_BK);   // an empty slice still writes its zeros
  return t;
}
__device__ inline FlexPlan flex_plan(const GemmDesc &g, int G, long long split_elems) {
  FlexPlan best;
  best.a = best.b = 4; best.wm = 2;
  best.tm = best.tn = best.splits = 1;
  best.kc = GF_BK;
  if (g.M <= 0 || g.N <= 0) return best;
  const int Um = (g.M + 7) >> 3, Un = (g.N + 7) >> 3;
  double bc = -1.0;
  for (int wm = 2; wm >= 1; --wm)
    for (int a = 2; a <= 4; ++a)
      for (int b = (wm == 1 ? 1 : 2); b <= (wm == 1 ? 2 : 4); ++b) {
        const int wn = 4 / wm;
        const int tm = (Um + wm * a - 1) / (wm * a), tn = (Un + wn * b - 1) / (wn * b);
        const long long T = (long long)tm * tn;
        int sp = 1;
        if (T * 2 <= G && g.K >= 256) {
          sp = (int)min((long long)G / T, (long long)min(g.K / 128, GF_MAXSPLIT));
          while (sp > 1 && (long long)sp * g.M * g.N > split_elems) --sp;
          if (sp < 1) sp = 1;
        }
        const int kt = ((g.K + sp - 1) / sp + GF_BK - 1) / GF_BK;
        const double rounds = (double)((T * sp + G - 1) / G);
        const double ktile = a * b + GF_FLEX_LDS * (a + b) + GF_FLEX_KT0;
        double cost = rounds * (kt + GF_FLEX_FIXED) * ktile;
        if (sp > 1) cost += (double)g.M * g.N * sp / (G * GF_THREADS) * GF_FLEX_RED;
        if (bc < 0.0 || cost < bc) {
          bc = cost;
          best.a = a; best.b = b; best.wm = wm; best.tm = tm; best.tn = tn; best.splits = sp;
        }
      }
  best.kc = ((g.K + best.splits - 1) / best.splits + GF_BK - 1) / GF_BK * GF_BK;
  return best;
}

template <int A, int B>
__device__ __forceinline__ void flex_mma(double (&acc)[4][4][2], const double *__restrict__ a,
                                         const double *__restrict__ b, int lane) {
  constexpr int LD = 64 + PAD;
#pragma unroll
  for (int kk = 0; kk < GF_BK; kk += 4) {
    const int kr = kk + (lane & 3);
    double af[A], bf[B];
#pragma unroll
    for (int i = 0; i < A; ++i) af[i] = a[kr * LD + i * 8];
#pragma unroll
    for (int j = 0; j < B; ++j) bf[j] = b[kr * LD + j * 8];
#pragma unroll
    for (int i = 0; i < A; ++i)
#pragma unroll
      for (int j = 0; j < B; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
}

// All tiles of one GEMM owned by this CTA (work items blockIdx.x, + G, ...).
__device__ __forceinline__ void flex_gemm(const GemmDesc &g, const FlexPlan &pl, double *__restrict__ split, int G,
                                          double *smem) {
  using C = Cfg<64, 64, GF_BK, 2, 2, 2>;
  double *sA = smem;
  double *sB = smem + GF_FS * C::A_ELEMS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // This CTA's items: a contiguous range of the (m-tile fastest) item order, so its
  // successive tiles share their B columns (and split-K slice): the second operand of
  // a tile is then an L1 hit instead of another L2 read (cp.async.ca; the operand
  // traffic of a stage was ~2.6 TB/s out of L2 with items dealt out round-robin).
  const int Wtot = pl.tm * pl.tn * pl.splits;
  int wl, W;                           // item being loaded, end of the range
  {
    const int q = Wtot / G, rem = Wtot - q * G, c = blockIdx.x;
    wl = c * q + min(c, rem);
    W = wl + q + (c < rem ? 1 : 0);
  }
  if (wl >= W) return;
  const int wfirst = wl;
  const int tileM = 8 * pl.wm * pl.a, tileN = 8 * (4 / pl.wm) * pl.b;
  const int wm = (warp % pl.wm) * 8 * pl.a, wn = (warp / pl.wm) * 8 * pl.b;
  const int code = pl.a * 4 + pl.b;
  OpLoader<64, GF_BK, C::THREADS> la, lb;
  FlexTile tl = flex_tile(g, pl, wl);
  int ktl = 0;
  auto init_loaders = [&](const FlexTile &t) {
    const double *A = g.transA ? g.A + t.kbeg : g.A + (long long)t.kbeg * g.lda;
    const double *B = g.transB ? g.B + (long long)t.kbeg * g.ldb : g.B + t.kbeg;
    la.init(A, g.lda, g.transA != 0, t.m0, min(g.M, t.m0 + tileM), t.klen, tid);
    lb.init(B, g.ldb, g.transB == 0, t.n0, min(g.N, t.n0 + tileN), t.klen, tid);
  };
  init_loaders(tl);
  int lslot = 0;                       // ring slot of the next load
  auto issue_next = [&]() {            // next k-tile of the item being loaded, or the first one of the next item
    if (wl < W && ktl >= tl.nk) {
      wl += 1;
      if (wl < W) {
        tl = flex_tile(g, pl, wl);
        init_loaders(tl);
        ktl = 0;
      }
    }
    if (wl < W) {
      la.load(sA + lslot * C::A_ELEMS, ktl * GF_BK);
      lb.load(sB + lslot * C::B_ELEMS, ktl * GF_BK);
      ++ktl;
      lslot = lslot + 1 == GF_FS ? 0 : lslot + 1;
    }
    cp_async_commit();
  };
#pragma unroll
  for (int d = 0; d < GF_FS - 1; ++d) issue_next();
  int wc = wfirst;                     // item being multiplied
  FlexTile tc = flex_tile(g, pl, wc);
  int ktc = 0, slot = 0;
  double alpha = g.alpha;
  if (g.alpha_dev) alpha *= *g.alpha_dev;
  const double beta = g.beta;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  while (wc < W) {
    cp_async_wait<GF_FS - 2>();
    __syncthreads();
    issue_next();
    {
      const double *a = sA + slot * C::A_ELEMS + wm + (lane >> 2);
      const double *b = sB + slot * C::B_ELEMS + wn + (lane >> 2);
      switch (code) {   // uniform over the CTA
        case 4 * 2 + 1: flex_mma<2, 1>(acc, a, b, lane); break;
        case 4 * 3 + 1: flex_mma<3, 1>(acc, a, b, lane); break;
        case 4 * 4 + 1: flex_mma<4, 1>(acc, a, b, lane); break;
        case 4 * 2 + 2: flex_mma<2, 2>(acc, a, b, lane); break;
        case 4 * 2 + 3: flex_mma<2, 3>(acc, a, b, lane); break;
        case 4 * 2 + 4: flex_mma<2, 4>(acc, a, b, lane); break;
        case 4 * 3 + 2: flex_mma<3, 2>(acc, a, b, lane); break;
        case 4 * 3 + 3: flex_mma<3, 3>(acc, a, b, lane); break;
        case 4 * 3 + 4: flex_mma<3, 4>(acc, a, b, lane); break;
        case 4 * 4 + 2: flex_mma<4, 2>(acc, a, b, lane); break;
        case 4 * 4 + 3: flex_mma<4, 3>(acc, a, b, lane); break;
        default: flex_mma<4, 4>(acc, a, b, lane); break;
      }
    }
    ++ktc;
    slot = slot + 1 == GF_FS ? 0 : slot + 1;
    if (ktc == tc.nk) {   // epilogue of this output tile (the next tile's first k-tile is in flight)
      if (pl.splits > 1) {
        double *P = split + (long long)tc.z * ((long long)g.M * g.N);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = tc.m0 + wm + i * 8 + (lane >> 2);
          if (i >= pl.a || r >= g.M) continue;
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = tc.n0 + wn + j * 8 + (lane & 3) * 2 + h;
              if (j < pl.b && c < g.N) P[r + (long long)c * g.M] = acc[i][j][h];
            }
        }
      } else {
        long long coff[4][2];
        ScatIdx ci, ri;
        ci.init(tc.n0 + wn + (lane & 3) * 2, g.dc);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = tc.n0 + wn + j * 8 + (lane & 3) * 2 + h;
            coff[j][h] = (j < pl.b && c < g.N) ? ci.off(g.s_c0, g.s_c1) : -1;
            ci.advance(h == 0 ? 1 : 7);
          }
        ri.init(tc.m0 + wm + (lane >> 2), g.dr);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = tc.m0 + wm + i * 8 + (lane >> 2);
          const long long roff = ri.off(g.s_r0, g.s_r1);
          ri.advance(8);
          if (i >= pl.a || r >= g.M) continue;
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (coff[j][h] < 0) continue;
              const long long addr = roff + coff[j][h];
              double v = alpha * acc[i][j][h];
              if (beta != 0.0) v += beta * g.C[addr];
              g.C[addr] = v;
            }
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      wc += 1;
      ktc = 0;
      if (wc < W) tc = flex_tile(g, pl, wc);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// Phase barrier: whole cooperative grid (atomics in global memory) or one
// thread-block cluster (hardware barrier.cluster with release/acquire).
template <bool CLUSTER>
__device__ __forceinline__ unsigned int phase_arrive(unsigned int *bar, unsigned int nblocks) {
  if (CLUSTER) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    return 0;
  }
  return gbar_arrive(bar, nblocks);
}
template <bool CLUSTER>
__device__ __forceinline__ void phase_wait(unsigned int *bar, unsigned int token) {
  if (CLUSTER) {
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  } else {
    gbar_wait(bar, token);
  }
}
template <bool CLUSTER>
__device__ __forceinline__ void phase_sync(unsigned int *bar, unsigned int nblocks) {
  if (CLUSTER) {
    // release/acquire at cluster scope orders the global-memory partials too
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  } else {
    gbar(bar, nblocks);
  }
}


// One GEMM as a phase of a persistent kernel: DMMA tiles distributed over the
// CTAs (split-K with an in-kernel reduction when the GEMM has few tiles), then a
// phase barrier.  Uniform control flow: every CTA reads the same descriptor.
// own_lo/own_hi >= 0: the output is the plain contiguous vector C[0 .. M N) and the
// caller goes on to work on its own slice [own_lo, own_hi) only: after a split-K
// pass each CTA reduces the slices of exactly that range and the closing grid
// barrier is dropped (the next phase reads what this CTA wrote itself).
template <bool CLUSTER>
__device__ void gemm_stage(const GemmDesc &g, double *split, long long split_elems, unsigned int *bar, int G,
                           double *smem, bool gm_count, bool check_skip = true, int own_lo = -1, int own_hi = -1,
                           const FlexPlan *plan = nullptr) {
  if (g.M <= 0 || g.N <= 0) return;
  if (check_skip && g.skip && *g.skip) return;
  const int tid = threadIdx.x;
  const int nb = gemm_nbatch(g);
  if (g.batch >= 1) {   // batched: tiles of every problem distributed over the CTAs, no split-K
    if (blockIdx.x == 0 && tid == 0) {
      const unsigned long long f = 2ull * (unsigned long long)g.M * g.N * (g.K > 0 ? g.K : 0) * nb;
      atomicAdd(&g_gemm_counters[0], f);
      atomicAdd(&g_gemm_counters[1], 1ull);
      if (gm_count) atomicAdd(&g_gm_counters[0], f);
    }
    const bool sm32 = g.M <= 32 || g.N <= 32;
    const int bm = sm32 ? 32 : 64;
    const int tm = (g.M + bm - 1) / bm, tn = (g.N + bm - 1) / bm, T = tm * tn;
    for (int t = blockIdx.x; t < T * nb; t += G) {
      const int b = t / T, tt = t - b * T;
      const GemmDesc h = gemm_batch_item(g, b);
      if (sm32) gemm_tile<32, 32, 16, 2, 2, 2>(h, (tt % tm) * 32, (tt / tm) * 32, 0, 1, nullptr, 0, 0, smem);
      else gemm_tile<64, 64, GF_BK, 2, 2, GF_ST>(h, (tt % tm) * 64, (tt / tm) * 64, 0, 1, nullptr, 0, 0, smem);
      __syncthreads();
    }
    phase_sync<CLUSTER>(bar, G);
    return;
  }
  if (blockIdx.x == 0 && tid == 0) {
    const unsigned long long f = 2ull * (unsigned long long)g.M * g.N * (g.K > 0 ? g.K : 0);
    atomicAdd(&g_gemm_counters[0], f);
    atomicAdd(&g_gemm_counters[1], 1ull);
    if (gm_count) atomicAdd(&g_gm_counters[0], f);
  }
#if GF_FLEX
  // uniform: the same model on the same descriptor in every CTA (the persistent kernel plans each stage once)
  const FlexPlan pl = plan ? *plan : flex_plan(g, G, split_elems);
  const int splits = pl.splits;
  flex_gemm(g, pl, split, G, smem);
#else
  // Tile shape per stage: 64x64 or 32x32 tiles, each with split-K when the output
  // has few tiles, whichever minimises the modelled stage time = rounds of tiles
  // over the G CTAs x padded tile work (the ranks of the C4 local systems, e.g.
  // 264 = 4 x 64 + 8 and 68 = 64 + 4 rows, waste up to half of a 64-wide tile on
  // padding; 32x32 tiles pay GF_EFF32 for their lower operand reuse).  Uniform:
  // every CTA evaluates the same model on the same descriptor.
  int bm = 64, tm = (g.M + 63) / 64, tn = (g.N + 63) / 64, splits = 1;
  {
    double best = 0.0;
    for (int v = 0; v < 2; ++v) {
      const int b = v == 0 ? 64 : 32;
      const int m_ = (g.M + b - 1) / b, n_ = (g.N + b - 1) / b, T_ = m_ * n_;
      int sp = 1;
      if (T_ * 2 <= G && g.K >= 256) {
        sp = min(G / T_, min(g.K / 128, GF_MAXSPLIT));
        while (sp > 1 && (long long)sp * g.M * g.N > split_elems) --sp;
      }
      const int kt = ((g.K + sp - 1) / sp + 15) / 16;
      const double rounds = (double)((T_ * sp + G - 1) / G);
      double cost = rounds * (double)b * b * kt * (v == 0 ? 1.0 : 1.0 / GF_EFF32);
      if (sp > 1) cost += (double)g.M * g.N * sp / (G * GF_THREADS) * 8.0;   // slice reduction (+ a barrier)
      if (v == 0 || cost < best) { best = cost; bm = b; tm = m_; tn = n_; splits = sp; }
    }
  }
  const int T = tm * tn;
  if (bm == 32) {
    for (int t = blockIdx.x; t < T * splits; t += G) {
      const int z = t / T, tt = t - z * T;
      gemm_tile<32, 32, 16, 2, 2, 2>(g, (tt % tm) * 32, (tt / tm) * 32, z, splits, split, g.M,
                                     (long long)g.M * g.N, smem);
      __syncthreads();
    }
  } else {
    for (int t = blockIdx.x; t < T * splits; t += G) {
      const int z = t / T, tt = t - z * T;
      gemm_tile<64, 64, GF_BK, 2, 2, GF_ST>(g, (tt % tm) * 64, (tt / tm) * 64, z, splits, split, g.M,
                                        (long long)g.M * g.N, smem);
      __syncthreads();
    }
  }
#endif
  phase_sync<CLUSTER>(bar, G);
  if (splits > 1) {
    const long long total = (long long)g.M * g.N, ps = total;
    double alpha = g.alpha;
    if (g.alpha_dev) alpha *= *g.alpha_dev;
    if (own_lo >= 0 && g.s_r0 == 1 && g.s_c0 == g.M && g.dr >= g.M && g.dc >= g.N) {
      for (int e = own_lo + tid; e < own_hi; e += GF_THREADS) {
        double sum = 0.0;
        for (int z = 0; z < splits; ++z) sum += split[z * ps + e];
        double v = alpha * sum;
        if (g.beta != 0.0) v += g.beta * g.C[e];
        g.C[e] = v;
      }
      __syncthreads();
      return;
    }
    for (long long e = (long long)blockIdx.x * GF_THREADS + tid; e < total; e += (long long)G * GF_THREADS) {
      const int r = (int)(e % g.M), c = (int)(e / g.M);
      double sum = 0.0;
      for (int z = 0; z < splits; ++z) sum += split[z * ps + e];
      const long long addr = (long long)(r % g.dr) * g.s_r0 + (long long)(r / g.dr) * g.s_r1 +
                             (long long)(c % g.dc) * g.s_c0 + (long long)(c / g.dc) * g.s_c1;
      double v = alpha * sum;
      if (g.beta != 0.0) v += g.beta * g.C[addr];
      g.C[addr] = v;
    }
    phase_sync<CLUSTER>(bar, G);
  }
}

// out[i] = sum_{e in [lo, hi)} V_i[e] w[e] for i < n: each warp takes groups of
// 8 vectors and keeps 8 accumulators per lane; two elements per lane and trip,
// so 16 basis loads are in flight before the first FMA (a CTA's slice of a QTT
// core's local vector is ~120 elements: the phase is pure L2 latency).
__device__ __forceinline__ void slice_dots(const double *V, long long ldv, const double *w, int lo, int hi, int n,
                                           double *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NWp = GF_THREADS / 32;
  for (int i0 = warp * 8; i0 < n; i0 += NWp * 8) {
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    const double *Vg = V + (long long)i0 * ldv;
    for (int e = lo + lane; e < hi; e += 64) {
      const int e2 = e + 32;
      const bool p2 = e2 < hi;
      const double w0 = w[e], w1 = p2 ? w[e2] : 0.0;
      double v0[8], v1[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const bool pq = i0 + q < n;
        v0[q] = pq ? Vg[(long long)q * ldv + e] : 0.0;
        v1[q] = (pq && p2) ? Vg[(long long)q * ldv + e2] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = fma(v1[q], w1, fma(v0[q], w0, acc[q]));
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double s = warp_sum(acc[q]);
      if (lane == 0 && i0 + q < n) out[i0 + q] = s;
    }
  }
}
// x - sum_{i < nv} h[i] V_i[e]: the Gram-Schmidt update of one element, basis
// loads in batches of 8 (independent loads; a plain loop paid one L2 round trip
// per basis vector: ~19 us per Arnoldi step at j ~ 40).
__device__ __forceinline__ double gs_update(const double *V, long long ldv, const double *h, int nv, int e,
                                            double x) {
  for (int i0 = 0; i0 < nv; i0 += 8) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = (i0 + q < nv) ? V[(long long)(i0 + q) * ldv + e] : 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (i0 + q < nv) x = fma(-h[i0 + q], v[q], x);
  }
  return x;
}
// Two-level cross-CTA sum, first level: the CTAs form groups of GF_GRP; each CTA
// publishes its partial row and takes a ticket of its group's counter; the last
// arriver sums the group's rows in CTA order (the same bits whoever is last) into
// the group's row of gpart.  After the grid barrier every CTA sums the ~19 group
// rows instead of all 296 CTA rows: each CTA reading every other CTA's row was
// 29 MB of L2 reads per reduction (4.3 us, twice per Arnoldi step).  The counters
// only ever grow by the group size per reduction, and a grid barrier separates
// successive reductions, so "ticket + 1 divisible by the group size" marks the last.
constexpr int GF_GRP = 16;
__device__ __forceinline__ void group_reduce(const double *part, double *gpart, unsigned int *cnt, int G, int n,
                                             int *s_last) {
  const int grp = blockIdx.x / GF_GRP, c0 = grp * GF_GRP;
  const int gsize = min(GF_GRP, G - c0);
  __syncthreads();   // this CTA's row is complete
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int t = atomicAdd(cnt + grp, 1u);
    const int last = ((t + 1u) % (unsigned int)gsize) == 0u;
    if (last) __threadfence();
    *s_last = last;
  }
  __syncthreads();
  if (*s_last) {
    for (int i = threadIdx.x; i < n; i += GF_THREADS) {
      double v[GF_GRP];
#pragma unroll
      for (int c = 0; c < GF_GRP; ++c) v[c] = c < gsize ? __ldcg(part + (size_t)(c0 + c) * GF_LD + i) : 0.0;
      double sacc = 0.0;
#pragma unroll
      for (int c = 0; c < GF_GRP; ++c) sacc += v[c];
      gpart[(size_t)grp * GF_LD + i] = sacc;
    }
  }
}

__device__ __forceinline__ void cross_cta_sum(const double *part, int G, int n, double *out) {
  // out[i] = sum_c part[c * GF_LD + i] for i < n
  // lanes over the CTAs (fixed order: the same bits in every CTA), each warp a group
  // of 8 entries, four CTAs per lane and trip so 32 loads are in flight (one entry
  // at a time paid one L2 round trip per entry; a single thread summing G values
  // from shared memory cost 4 us for the norm alone)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i0 = warp * 8; i0 < n; i0 += (GF_THREADS / 32) * 8) {
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    for (int c0 = lane; c0 < G; c0 += 128) {
      double v[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + 32 * u;
        const double *pc = part + (size_t)c * GF_LD + i0;
#pragma unroll
        for (int q = 0; q < 8; ++q) v[u][q] = (c < G && i0 + q < n) ? pc[q] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] += v[u][q];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double s = warp_sum(acc[q]);
      if (lane == 0 && i0 + q < n) out[i0 + q] = s;
    }
  }
  __syncthreads();
}

template <bool CLUSTER>
#ifndef GF_MINB
#define GF_MINB 3   // 168 registers, 3 CTAs per SM (444 CTAs): C4 fused time -4% against 2 per SM after the
                    // round-2 loader and tile work (the GEMM stages hide more latency; the barrier-bound
                    // core 8 loses 8%); 4 per SM (128 registers) is 20% slower; round 2 began at 1 -> 254
                    // registers, 2 per SM
#endif
__global__ void __launch_bounds__(GF_THREADS, GF_MINB) gm_chunk_kernel(GmChunkArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double h1s[GF_LD], h2s[GF_LD], css[GF_LD], sns[GF_LD];
  __shared__ double red[GF_THREADS / 32 + 4];
  const int G = gridDim.x;
  GmState *st = a.st;
  if (st->converged || st->stop) return;   // uniform: written by earlier launches
  const int N = st->N, m = st->m;
  if (a.mode == 2) {  // both variants launched: the device-resident sizes choose one (uniform)
    int tiles = 0;
    for (int q = 0; q < 3; ++q) {
      const GemmDesc &g = a.gapp[3 * (a.j0 + 1) + q];
      const int t = ((g.M + 63) / 64) * ((g.N + 63) / 64) * gemm_nbatch(g);
      tiles = t > tiles ? t : tiles;
    }
    const bool small = tiles <= 2 * a.cs && N <= 16384;
    if (small != CLUSTER) return;
  }
  const unsigned long long t_entry = (blockIdx.x == 0 && threadIdx.x == 0) ? globaltimer_ns() : 0ull;
  const double tol = st->tol;
  double bnorm = st->bnorm;
  const int per = (N + G - 1) / G;
  const int lo = min(N, (int)blockIdx.x * per), hi = min(N, lo + per);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = GF_THREADS / 32;
  double *part1 = a.part, *part2 = a.part + (size_t)G * GF_LD, *part3 = a.part + 2 * (size_t)G * GF_LD;
  // two-level sums on the big grid: group rows behind the three CTA-row tables
  double *gpart1 = a.part + 3 * (size_t)G * GF_LD, *gpart2 = gpart1 + (size_t)GM_GROUPS_MAX * GF_LD;
  unsigned int *gcnt = a.bar + 2;
  const bool two_level = !CLUSTER && G >= 4 * GF_GRP;
  const int NG = (G + GF_GRP - 1) / GF_GRP;
  __shared__ int s_last;
  double *w = a.w;
#ifdef GM_PHASE_TIMING
  long long ph[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long nre = 0;
  long long tcl = clock64();
#define GM_PH(i) do { const long long t_ = clock64(); ph[i] += t_ - tcl; tcl = t_; } while (0)
#else
#define GM_PH(i) do { } while (0)
#endif
  // The three apply descriptors of the CURRENT step live in shared memory; the
  // next step's are fetched into registers before the barrier that opens the
  // step and stored after it (the barrier wait hides the L2 latency).  Staging
  // the descriptors of all <= 41 steps took 18 KB of shared memory per CTA; the
  // kernel's operands shared by all tiles of a stage (x, A_k) live in L1, and
  // the shared-memory carve-out of 2 CTAs per SM decides its size.
  // full: descriptor set 0 = apply to x, set j + 1 = apply to basis vector j.
  const int jend = a.full ? m : min(a.j1, m);
  GemmDesc *sdesc = reinterpret_cast<GemmDesc *>(smem + GF_TILE_SMEM / sizeof(double));
  constexpr int DW = 3 * (int)sizeof(GemmDesc) / (int)sizeof(long long);
  static_assert(DW <= GF_THREADS && sizeof(GemmDesc) % sizeof(long long) == 0, "descriptor staging");
  auto desc_fetch = [&](int set) -> long long {
    return threadIdx.x < DW ? reinterpret_cast<const long long *>(a.gapp + 3 * set)[threadIdx.x] : 0ll;
  };
  auto desc_store = [&](long long v) {
    __syncthreads();
    if (threadIdx.x < DW) reinterpret_cast<long long *>(sdesc)[threadIdx.x] = v;
    __syncthreads();
  };
  desc_store(desc_fetch(a.full ? 0 : a.j0 + 1));
  // tile plans of the three apply stages (the same shapes at every step of this launch)
  __shared__ FlexPlan plans[3];
  if (threadIdx.x < 3) plans[threadIdx.x] = flex_plan(sdesc[threadIdx.x], G, a.split_elems);
  __syncthreads();
  __shared__ double ys[GF_LD];
  int nsteps = 0;
  const int ncycles = a.full ? a.max_restarts : 1;
  for (int cyc = 0; cyc < ncycles; ++cyc) {
  int jfirst = a.j0;
  if (a.full) {
    // ---- cycle start: r = b - A x, beta = ||r||, V_0 = r / beta (gm_start_kernel's work)
    if (cyc > 0) desc_store(desc_fetch(0));
    for (int sidx = 0; sidx < 3; ++sidx)
      gemm_stage<CLUSTER>(sdesc[sidx], a.split, a.split_elems, a.bar, G, smem, true, false, sidx == 2 ? lo : -1, hi,
                          &plans[sidx]);
    double pb = 0.0, pr = 0.0;
    for (int e = lo + tid; e < hi; e += GF_THREADS) {
      const double r = a.b[e] - w[e];
      a.V[e] = r;
      pb = fma(a.b[e], a.b[e], pb);
      pr = fma(r, r, pr);
    }
    pb = warp_sum(pb);
    pr = warp_sum(pr);
    if (lane == 0) { red[warp] = pb; h1s[warp] = pr; }
    __syncthreads();
    if (tid == 0) {
      double tb = 0.0, tr = 0.0;
      for (int q = 0; q < NW; ++q) { tb += red[q]; tr += h1s[q]; }
      part1[(size_t)blockIdx.x * GF_LD] = tb;
      part1[(size_t)blockIdx.x * GF_LD + 1] = tr;
    }
    phase_sync<CLUSTER>(a.bar, G);
    cross_cta_sum(part1, G, 2, h2s);
    const double bn = sqrt(h2s[0]), beta = sqrt(h2s[1]);
    if (cyc == 0) bnorm = bn;
    const double rel = bn > 0.0 ? beta / bn : 0.0;
    const bool done = (rel <= tol) || (beta == 0.0);
    if (blockIdx.x == 0 && tid == 0) {
      if (cyc == 0) { st->bnorm = bn; st->res0 = rel; }
      st->beta = beta;
      st->j = 0;
      st->jdone = 0;
      st->g[0] = beta;
      st->res = rel;
      if (done) { st->converged = 1; st->stop = 1; }
    }
    if (done) break;
    const double inv = 1.0 / beta;
    for (int e = lo + tid; e < hi; e += GF_THREADS) a.V[e] *= inv;
    phase_sync<CLUSTER>(a.bar, G);   // V_0 and g[0] complete
    jfirst = 0;
  }
  bool nan_stop = false;
  int jlast = jfirst - 1;
  for (int j = jfirst; j < jend; ++j) {
    // (V[:, j] is complete: the previous step ended with a barrier; its descriptors were
    // stored there too)
    if (j == jfirst) desc_store(desc_fetch(j + 1));
    GM_PH(0);
    ++nsteps;
    jlast = j;
    // ---- w = A V[:, j] (three chained GEMM stages; the kernel itself stops on the stop word)
    for (int sidx = 0; sidx < 3; ++sidx) {
      gemm_stage<CLUSTER>(sdesc[sidx], a.split, a.split_elems, a.bar, G, smem, true, false,
                          sidx == 2 ? lo : -1, hi, &plans[sidx]);
#ifdef GM_PHASE_TIMING
      if (sidx < 2) GM_PH(5 + sidx);
#endif
    }
    GM_PH(1);
    // ---- CGS pass 1: slice dots, plus |w|^2 for the reorthogonalisation test
    double *my1 = part1 + (size_t)blockIdx.x * GF_LD;
    slice_dots(a.V, a.ldv, w, lo, hi, j + 1, my1);
    {
      double w2 = 0.0;
      for (int e = lo + tid; e < hi; e += GF_THREADS) w2 = fma(w[e], w[e], w2);
      w2 = warp_sum(w2);
      if (lane == 0) red[warp] = w2;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int q = 0; q < NW; ++q) t += red[q];
        my1[j + 1] = t;
      }
    }
    if (two_level) group_reduce(part1, gpart1, gcnt, G, j + 2, &s_last);
    phase_sync<CLUSTER>(a.bar, G);
    GM_PH(2);
    // fixed order: identical in every CTA
    if (two_level) cross_cta_sum(gpart1, NG, j + 2, h1s);
    else cross_cta_sum(part1, G, j + 2, h1s);
    GM_PH(7);
    // w' = w - V h1 on the own slice, with |w'|^2 accumulated on the way
    double n1 = 0.0;
    for (int e = lo + tid; e < hi; e += GF_THREADS) {
      const double x = gs_update(a.V, a.ldv, h1s, j + 1, e, w[e]);
      w[e] = x;
      n1 = fma(x, x, n1);
    }
    n1 = warp_sum(n1);
    if (lane == 0) red[warp] = n1;
    GM_PH(8);
    // DGKS test (Daniel, Gragg, Kaufman & Stewart 1976): a second Gram-Schmidt
    // pass only when the projection removed more than half of |w|^2
    // (|w'|^2 = |w|^2 - sum h^2 < |w|^2 / 2); the decision is made on values
    // that are identical in every CTA, so it is uniform over the grid
    bool reorth;
    {
      double hh = 0.0;
      for (int i = 0; i <= j; ++i) hh = fma(h1s[i], h1s[i], hh);
      reorth = !(h1s[j + 1] - hh > 0.5 * h1s[j + 1]);
    }
    // rotations and g[j] of earlier steps, read before CTA 0 rewrites them in this step
    for (int i = tid; i < j; i += GF_THREADS) { css[i] = st->cs[i]; sns[i] = st->sn[i]; }
    const double gj = st->g[j];
    __syncthreads();
    double n1cta = 0.0;
    for (int q = 0; q < NW; ++q) n1cta += red[q];   // this CTA's share of |w'|^2 (same value in every thread)
    // With the second pass, |w''|^2 = |w' - V h2|^2 = |w'|^2 - |h2|^2 (V orthonormal), and
    // h2 is a rounding-level correction (|h2| << |w'|), so the subtraction loses nothing:
    // |w'|^2 rides along with the pass-2 dots in ONE reduction and the separate norm
    // reduction + barrier are dropped; the update w'' and the normalisation are then one
    // pass over the slice.  Guard: if |h2|^2 > |w'|^2 / 100 (never seen; near-breakdown)
    // the norm is reduced explicitly as in the single-pass case.
    bool fused_norm = false;
    double hn2 = 0.0;
    if (reorth) {
      // ---- pass 2 on the updated slice
      double *my2 = part2 + (size_t)blockIdx.x * GF_LD;
      slice_dots(a.V, a.ldv, w, lo, hi, j + 1, my2);
      if (tid == 0) my2[j + 1] = n1cta;
      if (two_level) group_reduce(part2, gpart2, gcnt, G, j + 2, &s_last);
      phase_sync<CLUSTER>(a.bar, G);
      if (two_level) cross_cta_sum(gpart2, NG, j + 2, h2s);
      else cross_cta_sum(part2, G, j + 2, h2s);
      double hh2 = 0.0;
      for (int i = 0; i <= j; ++i) hh2 = fma(h2s[i], h2s[i], hh2);
      const double n1tot = h2s[j + 1];
      fused_norm = hh2 <= 0.01 * n1tot;
      hn2 = n1tot - hh2;
#ifdef GM_PHASE_TIMING
      ++nre;
#endif
      GM_PH(9);
    } else {
      for (int i = tid; i <= j; i += GF_THREADS) h2s[i] = 0.0;
      __syncthreads();
    }
    if (!fused_norm) {
      double nrm = n1cta;
      if (reorth) {   // rare: explicit second update and norm
        nrm = 0.0;
        for (int e = lo + tid; e < hi; e += GF_THREADS) {
          const double x = gs_update(a.V, a.ldv, h2s, j + 1, e, w[e]);
          w[e] = x;
          nrm = fma(x, x, nrm);
        }
        nrm = warp_sum(nrm);
        __syncthreads();
        if (lane == 0) red[warp] = nrm;
        __syncthreads();
        nrm = 0.0;
        for (int q = 0; q < NW; ++q) nrm += red[q];
      }
      if (tid == 0) part3[(size_t)blockIdx.x * GF_LD] = nrm;
      GM_PH(10);
      phase_sync<CLUSTER>(a.bar, G);
      GM_PH(3);
      __syncthreads();
      cross_cta_sum(part3, G, 1, red + 2);
      hn2 = red[2];
    }
    // ---- norm, normalisation, then the barrier that publishes V[:, j+1] with the
    //      Givens update (identical in every CTA, nobody waits for it) between the
    //      barrier's arrival and its wait
    const double hn = hn2 < 0.0 ? 0.0 : sqrt(hn2);   // (a NaN stays a NaN: the Givens step reports it)
    if (hn > 0.0) {
      const double inv = 1.0 / hn;
      double *vn = a.V + (long long)(j + 1) * a.ldv;
      if (fused_norm) {   // w'' = w' - V h2 and its normalisation in one pass
        for (int e = lo + tid; e < hi; e += GF_THREADS) vn[e] = gs_update(a.V, a.ldv, h2s, j + 1, e, w[e]) * inv;
      } else {
        for (int e = lo + tid; e < hi; e += GF_THREADS) vn[e] = w[e] * inv;
      }
    }
    const long long dnext = j + 1 < jend ? desc_fetch(j + 2) : 0ll;
    const unsigned int token = phase_arrive<CLUSTER>(a.bar, G);
    // H column j: h1 + h2, then the earlier rotations
    if (tid == 0) {
      double col_j = 0.0, col_j1 = hn;
      double *H = st->H;
      // rotate entries 0..j (sequential; j <= GM_MAX_M)
      double prev = h1s[0] + h2s[0];
      for (int i = 0; i < j; ++i) {
        const double b = h1s[i + 1] + h2s[i + 1];
        const double ra = css[i] * prev + sns[i] * b;
        const double rb = -sns[i] * prev + css[i] * b;
        if (blockIdx.x == 0) H[i + (m + 1) * j] = ra;
        prev = rb;
      }
      col_j = prev;
      const double den = hypot(col_j, col_j1);
      const double c = den > 0.0 ? col_j / den : 1.0, sn = den > 0.0 ? col_j1 / den : 0.0;
      const double gnew = -sn * gj;
      const double rel = bnorm > 0.0 ? fabs(gnew) / bnorm : 0.0;
      int stop = 0;
      if (rel <= tol || hn == 0.0 || j + 1 >= m) stop = 1;
      if (!(rel == rel)) stop = 2;
      if (blockIdx.x == 0) {
        H[j + (m + 1) * j] = den;
        H[j + 1 + (m + 1) * j] = 0.0;
        st->cs[j] = c;
        st->sn[j] = sn;
        st->g[j + 1] = gnew;
        st->g[j] = c * gj;
        st->jdone = j + 1;
        st->res = rel;
        if (stop == 2) st->nan = 1;
        st->stop = stop ? 1 : 0;
        atomicAdd(&g_gm_counters[1], (unsigned long long)N * ((reorth ? 8ull : 4ull) * (j + 1) + 5ull));
        atomicAdd(&g_gm_counters[2], 1ull);
        atomicAdd(&g_gm_tag_steps[a.tag], 1ull);
      }
      red[0] = stop ? 1.0 : 0.0;
      red[3] = (stop == 2) ? 1.0 : 0.0;
    }
    __syncthreads();   // red[] of the Givens step (the cluster barrier's wait does not order it)
    phase_wait<CLUSTER>(a.bar, token);
    const bool stop = red[0] != 0.0;
    GM_PH(4);
    if (red[3] != 0.0) nan_stop = true;
    if (stop) break;
    if (j + 1 < jend) desc_store(dnext);
  }
  if (!a.full) break;
  // ---- cycle end: x += V y with H y = g (gm_update_kernel's work), restart test
  phase_sync<CLUSTER>(a.bar, G);   // H, g, res written by CTA 0 are visible
  const int jd = jlast + 1;
  if (tid == 0) {
    const double *H = st->H;
    for (int i = jd - 1; i >= 0; --i) {
      double sacc = st->g[i];
      for (int k = i + 1; k < jd; ++k) sacc -= H[i + (m + 1) * k] * ys[k];
      ys[i] = sacc / H[i + (m + 1) * i];
    }
  }
  __syncthreads();
  for (int e = lo + tid; e < hi; e += GF_THREADS) {
    double sacc = a.x[e];
    for (int i = 0; i < jd; ++i) sacc = fma(ys[i], a.V[(long long)i * a.ldv + e], sacc);
    a.x[e] = sacc;
  }
  const bool conv = st->res <= tol;   // written by CTA 0 before the barrier above
  if (blockIdx.x == 0 && tid == 0) {
    st->cycle += 1;
    st->converged = conv ? 1 : 0;
    st->stop = (conv || nan_stop || cyc + 1 >= ncycles) ? 1 : 0;
  }
  if (conv || nan_stop) break;
  phase_sync<CLUSTER>(a.bar, G);   // x complete before the next cycle's A x
  }   // cycles
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    atomicAdd(&g_gm_tag_ns[a.tag], globaltimer_ns() - t_entry);
    atomicAdd(&g_gm_tag_launches[a.tag], 1ull);
  }
#ifdef GM_PHASE_TIMING
  if (blockIdx.x == 0 && threadIdx.x == 0 && nsteps > 0)
    printf("GMPH %d %d %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld\n", (int)CLUSTER, nsteps, ph[0], ph[1],
           ph[2], ph[3], ph[4], ph[5], ph[6], ph[7], ph[8], ph[9], ph[10], nre);
#endif
}

}  // namespace

void set_gemm_scratch(double *ptr, size_t bytes) {
  g_split.ptr = ptr;
  g_split.bytes = ptr ? bytes : 0;
}

tt_status launch_gemm(const GemmDesc *descs_dev, int count, int Mcap, int Ncap, cudaStream_t s) {
  return launch_gemm_k(descs_dev, count, Mcap, Ncap, 0, s);
}

tt_status launch_gemm_k(const GemmDesc *descs_dev, int count, int Mcap, int Ncap, int Kcap, cudaStream_t s,
                        int batch) {
  if (count <= 0 || Mcap <= 0 || Ncap <= 0 || batch < 0) return TT_OK;
  return launch_variant<V64>(descs_dev, count, Mcap, Ncap, Kcap, s, batch);
}

void gemm_counters(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, g_gemm_counters, sizeof(g_gemm_counters));
  if (reset) {
    unsigned long long z[2] = {0, 0};
    cudaMemcpyToSymbol(g_gemm_counters, z, sizeof(z));
  }
}

}  // namespace tt

namespace tt {

size_t gmres_fused_part_doubles(int G) { return (size_t)(3 * G + 2 * GM_GROUPS_MAX) * GF_LD; }

int gmres_fused_grid() {
  static int G = 0;
  if (!G) {
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(gm_chunk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GM_SMEM);
    cudaFuncSetAttribute(gm_chunk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GM_SMEM);
    cudaFuncSetAttribute(gm_chunk_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gm_chunk_kernel<false>, GF_THREADS, GM_SMEM);
    const char *e = std::getenv("TT_GF_GRID");
    // two CTAs per SM when they fit (more bytes in flight for the CGS2 phases of
    // large local systems; measured +4% on C4)
    // all SMs equally loaded: the same number of CTAs (up to 3) on each of the 148 SMs
    G = (occ >= 1) ? (e ? std::atoi(e) : (occ >= 3 ? 3 : occ) * sms) : -1;
    if (G > occ * sms || G > GF_MAX_GRID) G = occ * sms < GF_MAX_GRID ? occ * sms : GF_MAX_GRID;
  }
  return G;
}

// live timing of the fused kernel (tt_fused_profile): events around every launch
struct FusedProfile {
  bool on = false;
  std::vector<cudaEvent_t> ev;   // pairs
  std::vector<int> tags;         // tag of each pair
  size_t used = 0;
  int tag = 0;
};
thread_local FusedProfile g_fp;

void fused_profile(int enable) {
  g_fp.on = enable != 0;
  g_fp.used = 0;
}
void fused_profile_tag(int tag) { g_fp.tag = tag < 0 ? 0 : (tag >= TT_MAX_D ? TT_MAX_D - 1 : tag); }

// per-tag sums of the recorded launches (does not reset; fused_profile_read does)
void fused_profile_cores(double *ms, double *steps, long long *launches) {
  for (int t = 0; t < TT_MAX_D; ++t) { ms[t] = 0.0; launches[t] = 0; }
  for (size_t i = 0; i + 1 < g_fp.used; i += 2) {
    cudaEventSynchronize(g_fp.ev[i + 1]);
    float e = 0.f;
    cudaEventElapsedTime(&e, g_fp.ev[i], g_fp.ev[i + 1]);
    ms[g_fp.tags[i / 2]] += e;
    launches[g_fp.tags[i / 2]] += 1;
  }
  unsigned long long c[TT_MAX_D];
  cudaMemcpyFromSymbol(c, g_gm_tag_steps, sizeof(c));
  for (int t = 0; t < TT_MAX_D; ++t) steps[t] = (double)c[t];
  if (g_fp.used == 0) {   // no events (device-resident loops): the in-kernel timer
    unsigned long long ns[TT_MAX_D], nl[TT_MAX_D];
    cudaMemcpyFromSymbol(ns, g_gm_tag_ns, sizeof(ns));
    cudaMemcpyFromSymbol(nl, g_gm_tag_launches, sizeof(nl));
    for (int t = 0; t < TT_MAX_D; ++t) { ms[t] = 1e-6 * (double)ns[t]; launches[t] = (long long)nl[t]; }
  }
}

// in-kernel timer totals since the last read (ms, launches that did work); resets them
void fused_timer_read(double *ms, long long *launches) {
  unsigned long long ns[TT_MAX_D], nl[TT_MAX_D];
  cudaMemcpyFromSymbol(ns, g_gm_tag_ns, sizeof(ns));
  cudaMemcpyFromSymbol(nl, g_gm_tag_launches, sizeof(nl));
  double t = 0.0;
  long long l = 0;
  for (int i = 0; i < TT_MAX_D; ++i) { t += 1e-6 * (double)ns[i]; l += (long long)nl[i]; }
  const unsigned long long z[TT_MAX_D] = {};
  cudaMemcpyToSymbol(g_gm_tag_ns, z, sizeof(z));
  cudaMemcpyToSymbol(g_gm_tag_launches, z, sizeof(z));
  if (ms) *ms = t;
  if (launches) *launches = l;
}

void fused_profile_read(long long *launches, double *ms, double *flops) {
  double t = 0.0;
  for (size_t i = 0; i + 1 < g_fp.used; i += 2) {
    cudaEventSynchronize(g_fp.ev[i + 1]);
    float e = 0.f;
    cudaEventElapsedTime(&e, g_fp.ev[i], g_fp.ev[i + 1]);
    t += e;
  }
  const bool events = g_fp.used > 0;
  double tk = 0.0;
  long long lk = 0;
  if (!events) fused_timer_read(&tk, &lk);   // (with events the timer totals stay for tt_fused_timer_read)
  unsigned long long c[3] = {0, 0, 0};
  cudaMemcpyFromSymbol(c, g_gm_counters, sizeof(c));
  const unsigned long long z[3] = {0, 0, 0};
  cudaMemcpyToSymbol(g_gm_counters, z, sizeof(z));
  const unsigned long long zt[TT_MAX_D] = {};
  cudaMemcpyToSymbol(g_gm_tag_steps, zt, sizeof(zt));
  // events when they were recorded (host-stepped loops), else the in-kernel timer
  if (launches) *launches = events ? (long long)(g_fp.used / 2) : lk;
  if (ms) *ms = events ? t : tk;
  if (flops) { flops[0] = (double)c[0]; flops[1] = (double)c[1]; flops[2] = (double)c[2]; }
  g_fp.used = 0;
}

// Dependent GEMM chain: one cluster launch when every GEMM is small at its
// capacity shape (<= 2 tiles per CTA of the cluster), else one launch per GEMM.
tt_status launch_gemm_seq(const GemmDesc *descs_dev, int count, const int *Mcap, const int *Ncap, const int *Kcap,
                          cudaStream_t s, const int *Bcap) {
  if (count <= 0) return TT_OK;
  for (int i = 0; i < count; ++i)
    TT_TRY(launch_gemm_k(descs_dev + i, 1, Mcap[i], Ncap[i], Kcap[i], s, Bcap ? Bcap[i] : 0));
  return TT_OK;
}

int gmres_cluster_size() {
  static int cs = 0;
  if (!cs) {
    const char *e = std::getenv("TT_GF_CLUSTER");
    cs = e ? std::atoi(e) : 8;
    cs = cs >= 16 ? 16 : (cs >= 8 ? 8 : (cs >= 4 ? 4 : 2));
  }
  return cs;
}

tt_status launch_gmres_chunk(GmState *st, const GemmDesc *gapp, double *V, long long ldv, double *w, double *part,
                             double *split, long long split_elems, unsigned int *bar, int j0, int j1,
                             cudaStream_t s, int cluster, int decide, int full, int max_restarts, const double *b,
                             double *x) {
  const int G = cluster ? gmres_cluster_size() : gmres_fused_grid();
  if (G <= 0) return fail(TT_ERR_CUDA, "gmres: fused step kernel cannot be co-resident");
  GmChunkArgs a;
  a.mode = decide ? 2 : cluster;
  a.cs = gmres_cluster_size();
  a.full = full;
  a.max_restarts = max_restarts;
  a.b = b;
  a.x = x;
  a.st = st; a.gapp = gapp; a.V = V; a.ldv = ldv; a.w = w; a.part = part; a.split = split;
  a.split_elems = split_elems; a.bar = bar; a.j0 = j0; a.j1 = j1;
  a.tag = g_fp.tag;
  void *args[] = {(void *)&a};
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (g_fp.on && !stream_capturing(s)) {   // (inside a captured graph: the in-kernel timer only)
    while (g_fp.ev.size() < g_fp.used + 2) {
      cudaEvent_t ev;
      cudaEventCreate(&ev);
      g_fp.ev.push_back(ev);
    }
    e0 = g_fp.ev[g_fp.used];
    e1 = g_fp.ev[g_fp.used + 1];
    if (g_fp.tags.size() < g_fp.used / 2 + 1) g_fp.tags.resize(g_fp.used / 2 + 1);
    g_fp.tags[g_fp.used / 2] = g_fp.tag;
    g_fp.used += 2;
    cudaEventRecord(e0, s);
  }
  cudaError_t e;
  if (cluster) {   // one thread-block cluster: hardware cluster barriers between the phases
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(GF_THREADS);
    cfg.dynamicSmemBytes = GM_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, gm_chunk_kernel<true>, a);
  } else {
    e = cudaLaunchCooperativeKernel((const void *)gm_chunk_kernel<false>, dim3(G), dim3(GF_THREADS), args, GM_SMEM,
                                    s);
  }
  if (e1) cudaEventRecord(e1, s);
  if (e != cudaSuccess) return fail(TT_ERR_CUDA, std::string("gm_chunk: ") + cudaGetErrorString(e));
  return TT_OK;
}

}  // namespace tt
