// Elementwise / structural TT operations: exact matvec (a1), add / scale (a2),
// copy, dot (a8), plus the meta plumbing and error state of the C ABI.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "tt_common.cuh"

namespace tt {

// ------------------------------------------------------------- errors ---
static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }
const char *last_error_cstr() { return g_last_error.c_str(); }
tt_status fail(tt_status st, const std::string &msg) {
  g_last_error = msg;
  return st;
}
tt_status check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return TT_OK;
}

// Small device -> host read of a convergence word: a pinned per-thread staging
// buffer and an event polled by the calling thread (the drivers' sweep and
// outer-iteration tests; measured: a pageable copy + stream synchronise left
// the GPU idle ~80 us per test).
tt_status read_back(void *dst, const void *src_dev, size_t bytes, cudaStream_t s) {
  struct Stage {
    void *buf = nullptr;
    cudaEvent_t ev = nullptr;
  };
  static thread_local Stage st;
  if (bytes > 256) return fail(TT_ERR_ARG, "read_back: at most 256 bytes");
  if (!st.buf) {
    if (cudaMallocHost(&st.buf, 256) != cudaSuccess) return check_launch("read_back: cudaMallocHost");
    if (cudaEventCreateWithFlags(&st.ev, cudaEventDisableTiming) != cudaSuccess) return check_launch("read_back: event");
  }
  cudaMemcpyAsync(st.buf, src_dev, bytes, cudaMemcpyDeviceToHost, s);
  cudaEventRecord(st.ev, s);
  cudaError_t e;
  while ((e = cudaEventQuery(st.ev)) == cudaErrorNotReady) {
  }
  if (e != cudaSuccess) return fail(TT_ERR_CUDA, std::string("read_back: ") + cudaGetErrorString(e));
  std::memcpy(dst, st.buf, bytes);
  return TT_OK;
}

// --------------------------------------------------------------- metas ---
tt_status make_vec_meta(const tt_vec *x, VecMeta &m) {
  if (!x || !x->n || !x->rcap || !x->off || !x->r_dev || !x->data)
    return fail(TT_ERR_ARG, "tt_vec has a NULL field");
  if (x->d < 1 || x->d > TT_MAX_D) return fail(TT_ERR_ARG, "tt_vec: d out of range");
  if (x->rcap[0] != 1 || x->rcap[x->d] != 1) return fail(TT_ERR_ARG, "tt_vec: rcap[0], rcap[d] must be 1");
  std::memset(&m, 0, sizeof(m));
  m.d = x->d;
  for (int k = 0; k < x->d; ++k) {
    if (x->n[k] < 1) return fail(TT_ERR_ARG, "tt_vec: mode size < 1");
    m.n[k] = x->n[k];
    m.off[k] = x->off[k];
  }
  for (int k = 0; k <= x->d; ++k) {
    if (x->rcap[k] < 1) return fail(TT_ERR_ARG, "tt_vec: rank capacity < 1");
    m.rcap[k] = x->rcap[k];
  }
  m.data = x->data;
  m.r = x->r_dev;
  return TT_OK;
}

tt_status make_mat_meta(const tt_mat *A, MatMeta &m) {
  if (!A || !A->m || !A->n || !A->Rcap || !A->off || !A->R_dev || !A->data)
    return fail(TT_ERR_ARG, "tt_mat has a NULL field");
  if (A->d < 1 || A->d > TT_MAX_D) return fail(TT_ERR_ARG, "tt_mat: d out of range");
  if (A->Rcap[0] != 1 || A->Rcap[A->d] != 1) return fail(TT_ERR_ARG, "tt_mat: Rcap[0], Rcap[d] must be 1");
  std::memset(&m, 0, sizeof(m));
  m.d = A->d;
  for (int k = 0; k < A->d; ++k) {
    if (A->m[k] < 1 || A->n[k] < 1) return fail(TT_ERR_ARG, "tt_mat: mode size < 1");
    m.m[k] = A->m[k];
    m.n[k] = A->n[k];
    m.off[k] = A->off[k];
  }
  for (int k = 0; k <= A->d; ++k) m.Rcap[k] = A->Rcap[k];
  m.data = A->data;
  m.R = A->R_dev;
  return TT_OK;
}

VecMeta mat_as_vec(const MatMeta &A) {
  VecMeta v;
  std::memset(&v, 0, sizeof(v));
  v.d = A.d;
  for (int k = 0; k < A.d; ++k) {
    v.n[k] = A.m[k] * A.n[k];
    v.off[k] = A.off[k];
  }
  for (int k = 0; k <= A.d; ++k) v.rcap[k] = A.Rcap[k];
  v.data = A.data;
  v.r = A.R;
  return v;
}

// ------------------------------------------------------ core structure ---
// grid (blocks, d): max|A_k| and max|off-diagonal| as float bit patterns (non-negative
// floats order like their unsigned bits) via atomicMax; zeroed by the caller
__global__ void core_offdiag_max_kernel(const MatMeta A, unsigned int *mx) {
  const int k = blockIdx.y;
  const int m = A.m[k], n = A.n[k];
  if (m != n || m < 4) return;
  const int R0 = A.R[k], R1 = A.R[k + 1];
  const double *c = A.data + A.off[k];
  const long long tot = (long long)R0 * m * n * R1;
  double amax = 0.0, omax = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const long long t = e / R0;
    const int i = (int)(t % m), j = (int)((t / m) % n);
    const double v = fabs(c[e]);
    amax = v > amax ? v : amax;
    if (i != j) omax = v > omax ? v : omax;
  }
  for (int o = 16; o > 0; o >>= 1) {
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    omax = fmax(omax, __shfl_xor_sync(0xffffffffu, omax, o));
  }
  if ((threadIdx.x & 31) == 0) {
    // round up so that a tiny nonzero never becomes 0
    atomicMax(mx + 2 * k, __float_as_uint(__double2float_ru(amax)));
    atomicMax(mx + 2 * k + 1, __float_as_uint(__double2float_ru(omax)));
  }
}

__global__ void core_offdiag_ratio_kernel(const MatMeta A, const unsigned int *mx, float *out) {
  const int k = threadIdx.x;
  if (k >= A.d) return;
  if (A.m[k] != A.n[k] || A.m[k] < 4) { out[k] = -1.f; return; }
  const float a = __uint_as_float(mx[2 * k]), b = __uint_as_float(mx[2 * k + 1]);
  out[k] = a > 0.f ? b / a : 0.f;
}

tt_status detect_core_kinds(MatMeta &A, float *scratch_dev, cudaStream_t s, double *ratio_out) {
  // scratch: [d] ratios, then 2 d max words
  unsigned int *mx = reinterpret_cast<unsigned int *>(scratch_dev + TT_MAX_D);
  cudaMemsetAsync(mx, 0, 2 * sizeof(unsigned int) * A.d, s);
  core_offdiag_max_kernel<<<dim3(64, A.d), 256, 0, s>>>(A, mx);
  core_offdiag_ratio_kernel<<<1, TT_MAX_D, 0, s>>>(A, mx, scratch_dev);
  TT_TRY(check_launch("detect_core_kinds"));
  float r[TT_MAX_D];
  TT_TRY(read_back(r, scratch_dev, sizeof(float) * A.d, s));
  for (int k = 0; k < A.d; ++k) {
    A.kind[k] = (r[k] >= 0.f && r[k] <= (float)KIND_DIAG_TOL) ? 1 : 0;
    if (ratio_out) ratio_out[k] = r[k];
  }
  A.kinds_set = 1;
  return TT_OK;
}

int max_slot(const VecMeta &x) {
  long long mx = 0;
  for (int k = 0; k < x.d; ++k) {
    long long s = (long long)x.rcap[k] * x.n[k] * x.rcap[k + 1];
    if (s > mx) mx = s;
  }
  return (int)mx;
}
int max_rank(const VecMeta &x) {
  int mx = 1;
  for (int k = 0; k <= x.d; ++k) mx = x.rcap[k] > mx ? x.rcap[k] : mx;
  return mx;
}

// algorithmic flops of the exact matvec (2 n per output entry)
__device__ unsigned long long g_matvec_flops;
void matvec_counters(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, g_matvec_flops, sizeof(unsigned long long));
  if (reset) {
    unsigned long long z = 0;
    cudaMemcpyToSymbol(g_matvec_flops, &z, sizeof(z));
  }
}

// -------------------------------------------------------------- matvec ---
// Y_k[rho, i, rho'] = sum_j A_k[a, i, j, a'] X_k[b, j, b'], rho = a + R b.
// One launch over all cores: blockIdx.y = core, grid-stride over output entries
// (consecutive threads write consecutive rho: coalesced stores, which are the
// HBM traffic that bounds this kernel for QTT 2x2 cores).
__device__ void matvec_core_cols(const double *__restrict__ A, const double *__restrict__ X,
                                 double *__restrict__ Y, int R0, int R1, int r0, int r1, int m, int n, double *sm,
                                 int smcap);

__global__ void __launch_bounds__(256) matvec_kernel(const MatMeta A, const VecMeta x, const VecMeta y, int smcap) {
  extern __shared__ double dsm_mv[];
  const int k = blockIdx.y;
  const int R0 = A.R[k], R1 = A.R[k + 1], r0 = x.r[k], r1 = x.r[k + 1];
  const int m = A.m[k], n = A.n[k];
  matvec_core_cols(A.data + A.off[k], x.data + x.off[k], y.data + y.off[k], R0, R1, r0, r1, m, n, dsm_mv, smcap);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    y.r[k] = R0 * r0;
    if (k == A.d - 1) y.r[k + 1] = R1 * r1;
    atomicAdd(&g_matvec_flops, 2ull * (unsigned long long)R0 * r0 * m * R1 * r1 * n);
  }
}

tt_status matvec_meta(const MatMeta &A, const VecMeta &x, const VecMeta &y, cudaStream_t s) {
  if (A.d != x.d || A.d != y.d) return fail(TT_ERR_SHAPE, "tt_matvec: number of cores differ");
  long long mx = 0;
  for (int k = 0; k < A.d; ++k) {
    if (A.n[k] != x.n[k]) return fail(TT_ERR_SHAPE, "tt_matvec: shape mismatch (A.n != x.n)");
    if (A.m[k] != y.n[k]) return fail(TT_ERR_SHAPE, "tt_matvec: shape mismatch (A.m != y.n)");
    long long c = (long long)A.Rcap[k] * x.rcap[k] * A.m[k] * A.Rcap[k + 1] * x.rcap[k + 1];
    if (c > (1LL << 31) - 1) return fail(TT_ERR_CAPACITY, "tt_matvec: core too large");
    mx = c > mx ? c : mx;
  }
  for (int k = 0; k <= A.d; ++k)
    if ((long long)y.rcap[k] < (long long)A.Rcap[k] * x.rcap[k])
      return fail(TT_ERR_CAPACITY, "tt_matvec: y rank capacity < R*r");
  int bx = 2368 / A.d;  // columns of each core spread over bx CTAs (~16 CTAs per SM in total)
  bx = bx < 1 ? 1 : (bx > 512 ? 512 : bx);
  (void)mx;
  long long acap = 1;  // operator core staged in shared memory (host-known capacity)
  for (int k = 0; k < A.d; ++k) {
    const long long c = (long long)A.Rcap[k] * A.m[k] * A.n[k] * A.Rcap[k + 1];
    acap = c > acap ? c : acap;
  }
  const int smcap = acap <= 6144 ? (int)acap : 0;
  matvec_kernel<<<dim3(bx, A.d), 256, (size_t)smcap * sizeof(double), s>>>(A, x, y, smcap);
  return check_launch("tt_matvec");
}

// ------------------------------------------------------- batched matvec ---
// One launch over (core, instance): blockIdx.y = core, blockIdx.z = instance,
// per-pair pointers and sizes from a descriptor table in the workspace.
struct MvPair {
  const double *A;
  const double *X;
  double *Y;
  const int *R;   // operator ranks (device), index k, k+1
  const int *r;   // vector ranks (device)
  int *ry;        // output ranks (device)
  int m, n, k, last;
  int blk0;       // work estimate at the capacity ranks (host sort key)
};

// One CTA per output column rho' = a' + R1 b' (grid-strided): the slices
// A[:, :, :, a'] (R0 m n) and X[:, :, b'] (r0 n) are staged in shared memory and
// the contiguous column Y[:, :, rho'] (P m entries) is streamed out with
// coalesced stores — one small division per entry, no per-entry index algebra.

template <int MC, int NC>   // MC = NC = 2: QTT 2x2 cores (compile-time modes); 0: runtime modes
__device__ __forceinline__ void matvec_cols_t(const double *__restrict__ A, const double *__restrict__ X,
                                              double *__restrict__ Y, int R0, int R1, int r0, int r1, int m_,
                                              int n_, double *sm, int smcap, int cta, int ncta) {
  const int m = MC ? MC : m_, n = NC ? NC : n_;
  const int P = R0 * r0;
  const int na = R0 * m * n * R1;                         // the whole operator core
  const double *As = A;
  if (na <= smcap) {
    for (int e = threadIdx.x; e < na; e += blockDim.x) sm[e] = A[e];
    __syncthreads();
    As = sm;
  }
  // one thread per (rho, b'): its X[b, :, b'] values are loaded once and reused
  // for every a' in [0, R1) and i in [0, m) (R1 m independent coalesced stores per item)
  const int items = P * r1;
  const int per_col = P * m;
  for (int e = cta * blockDim.x + threadIdx.x; e < items; e += ncta * blockDim.x) {
    const int b1 = e / P, rho = e - b1 * P;
    const int b = rho / R0, a = rho - b * R0;
    const double *Xr = X + b + r0 * n * b1;
    double *Yr = Y + rho + (size_t)per_col * R1 * b1;
    const double *Ar = As + a;
    if (NC == 2 && MC == 2) {
      const double x0 = __ldg(Xr), x1 = __ldg(Xr + r0);
#pragma unroll 2
      for (int a1 = 0; a1 < R1; ++a1) {
        const double *Aa = Ar + 4 * R0 * a1;
        const double y0 = fma(Aa[0], x0, Aa[2 * R0] * x1);
        const double y1 = fma(Aa[R0], x0, Aa[3 * R0] * x1);
        double *Ya = Yr + 2 * P * a1;
        __stcs(Ya, y0);
        __stcs(Ya + P, y1);
      }
    } else {
      for (int a1 = 0; a1 < R1; ++a1) {
        const double *Aa = Ar + R0 * m * n * a1;
        double *Ya = Yr + (size_t)per_col * a1;
        for (int i = 0; i < m; ++i) {
          double s = 0.0;
          for (int j = 0; j < n; ++j) s = fma(Aa[R0 * (i + m * j)], Xr[r0 * j], s);
          Ya[P * i] = s;
        }
      }
    }
  }
}

__device__ void matvec_core_cols(const double *__restrict__ A, const double *__restrict__ X,
                                 double *__restrict__ Y, int R0, int R1, int r0, int r1, int m, int n, double *sm,
                                 int smcap) {
  if (m == 2 && n == 2) matvec_cols_t<2, 2>(A, X, Y, R0, R1, r0, r1, m, n, sm, smcap, blockIdx.x, gridDim.x);
  else matvec_cols_t<0, 0>(A, X, Y, R0, R1, r0, r1, m, n, sm, smcap, blockIdx.x, gridDim.x);
}

// Grid (bx, pairs): blockIdx.x = CTA within the pair, (y, z) = pair index in
// the instance-major descriptor table.
template <int MC, int NC, int MINB>
__global__ void __launch_bounds__(256, MINB) matvec_batched_kernel(const MvPair *__restrict__ pairs, int np,
                                                                   int smcap) {
  extern __shared__ double sm[];
  const int pi = blockIdx.z * gridDim.y + blockIdx.y;
  if (pi >= np) return;
  const MvPair *pp = pairs + pi;
  const int cta = blockIdx.x, ncta = gridDim.x;
  const int k = pp->k;
  const int *R = pp->R, *r = pp->r;
  const int R0 = R[k], R1 = R[k + 1], r0 = r[k], r1 = r[k + 1];
  matvec_cols_t<MC, NC>(pp->A, pp->X, pp->Y, R0, R1, r0, r1, pp->m, pp->n, sm, smcap, cta, ncta);
  if (cta == 0 && threadIdx.x == 0) {
    pp->ry[k] = R0 * r0;
    if (pp->last) pp->ry[k + 1] = R1 * r1;
    atomicAdd(&g_matvec_flops, 2ull * (unsigned long long)R0 * r0 * pp->m * R1 * r1 * pp->n);
  }
}

size_t matvec_batched_ws(int B, int d) { return (size_t)B * d * sizeof(MvPair); }

tt_status matvec_batched_meta(int B, const MatMeta *A, const VecMeta *x, const VecMeta *y, void *ws, size_t wsb,
                              cudaStream_t s) {
  if (B <= 0) return TT_OK;
  const int d = A[0].d;
  const size_t need = (size_t)B * d * sizeof(MvPair);
  if (!ws || wsb < need) return fail(TT_ERR_CAPACITY, "tt_matvec_batched: workspace too small");
  // pageable staging: cudaMemcpyAsync returns once the source has been consumed
  std::vector<MvPair> host((size_t)B * d);
  long long mx = 0;
  for (int b = 0; b < B; ++b) {
    if (A[b].d != d || x[b].d != d || y[b].d != d) return fail(TT_ERR_SHAPE, "tt_matvec_batched: d differs");
    for (int k = 0; k < d; ++k) {
      if (A[b].n[k] != x[b].n[k] || A[b].m[k] != y[b].n[k]) return fail(TT_ERR_SHAPE, "tt_matvec_batched: shape mismatch");
      if ((long long)y[b].rcap[k] < (long long)A[b].Rcap[k] * x[b].rcap[k])
        return fail(TT_ERR_CAPACITY, "tt_matvec_batched: y rank capacity < R*r");
      long long c = (long long)A[b].Rcap[k] * x[b].rcap[k] * A[b].m[k] * A[b].Rcap[k + 1] * x[b].rcap[k + 1];
      mx = c > mx ? c : mx;
      MvPair &p = host[(size_t)b * d + k];
      p.A = A[b].data + A[b].off[k];
      p.X = x[b].data + x[b].off[k];
      p.Y = y[b].data + y[b].off[k];
      p.R = A[b].R;
      p.r = x[b].r;
      p.ry = y[b].r;
      p.m = A[b].m[k];
      p.n = A[b].n[k];
      p.k = k;
      p.last = (k == d - 1);
      p.blk0 = (int)std::min<long long>((long long)A[b].Rcap[k] * x[b].rcap[k] * x[b].rcap[k + 1] *
                                            A[b].Rcap[k + 1] * A[b].m[k], 1LL << 30);   // work (sort key)
    }
  }
  // (kept in instance-major order: concurrent CTAs then write neighbouring
  //  cores of one instance, which measured faster than a largest-first order)
  // pinned staging so the table upload is a true async copy (the previous upload
  // from this staging buffer must have completed before it is refilled)
  static thread_local MvPair *stage = nullptr;
  static thread_local size_t stage_cap = 0;
  static thread_local cudaEvent_t stage_done = nullptr;
  if (stage_done) cudaEventSynchronize(stage_done);
  else cudaEventCreateWithFlags(&stage_done, cudaEventDisableTiming);
  if (stage_cap < host.size()) {
    if (stage) cudaFreeHost(stage);
    if (cudaHostAlloc((void **)&stage, host.size() * sizeof(MvPair), cudaHostAllocDefault) != cudaSuccess) {
      stage = nullptr;
      stage_cap = 0;
      return fail(TT_ERR_CUDA, "tt_matvec_batched: pinned staging allocation failed");
    }
    stage_cap = host.size();
  }
  std::memcpy(stage, host.data(), need);
  cudaMemcpyAsync(ws, stage, need, cudaMemcpyHostToDevice, s);
  cudaEventRecord(stage_done, s);
  bool qtt = true;
  for (const MvPair &p : host) qtt = qtt && p.m == 2 && p.n == 2;
  (void)mx;
  long long acap = 1;
  for (int b = 0; b < B; ++b)
    for (int k = 0; k < d; ++k) {
      const long long c = (long long)A[b].Rcap[k] * A[b].m[k] * A[b].n[k] * A[b].Rcap[k + 1];
      acap = c > acap ? c : acap;
    }
  const int smcap = acap <= 6144 ? (int)acap : 0;
  const int np = B * d;
  const char *ev = getenv("TT_MV_MINB");
  const int minb = ev ? atoi(ev) : 5;
  const char *eb = getenv("TT_MV_BX");
  int bx = eb ? atoi(eb) : 4;
  bx = bx < 1 ? 1 : (bx > 256 ? 256 : bx);
  const int gy = np < 65535 ? np : 65535;
  const dim3 grid(bx, gy, (np + gy - 1) / gy);
  const size_t shb = (size_t)smcap * sizeof(double);
  if (!qtt) matvec_batched_kernel<0, 0, 1><<<grid, 256, shb, s>>>((const MvPair *)ws, np, smcap);
  else if (minb >= 6) matvec_batched_kernel<2, 2, 6><<<grid, 256, shb, s>>>((const MvPair *)ws, np, smcap);
  else if (minb == 5) matvec_batched_kernel<2, 2, 5><<<grid, 256, shb, s>>>((const MvPair *)ws, np, smcap);
  else matvec_batched_kernel<2, 2, 4><<<grid, 256, shb, s>>>((const MvPair *)ws, np, smcap);
  return check_launch("tt_matvec_batched");
}

// ----------------------------------------------------------------- add ---
// z = alpha x + beta y, block-diagonal concatenation.
__global__ void add_kernel(const VecMeta x, const double *alpha, const VecMeta y, const double *beta,
                           const VecMeta z) {
  const int k = blockIdx.y, d = x.d;
  const int n = x.n[k];
  const int rx0 = x.r[k], rx1 = x.r[k + 1], ry0 = y.r[k], ry1 = y.r[k + 1];
  const double *Xk = x.data + x.off[k];
  const double *Yk = y.data + y.off[k];
  double *Zk = z.data + z.off[k];
  const double al = (k == 0 && alpha) ? *alpha : 1.0;
  const double be = (k == 0 && beta) ? *beta : 1.0;
  if (d == 1) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
      Zk[e] = al * Xk[e] + be * Yk[e];
    if (blockIdx.x == 0 && threadIdx.x == 0) { z.r[0] = 1; z.r[1] = 1; }
    return;
  }
  const int rz0 = (k == 0) ? 1 : rx0 + ry0;
  const int rz1 = (k == d - 1) ? 1 : rx1 + ry1;
  const int total = rz0 * n * rz1;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int p = e % rz0, t = e / rz0, i = t % n, q = t / n;
    double v = 0.0;
    if (k == 0) {
      v = (q < rx1) ? al * Xk[i + n * q] : be * Yk[i + n * (q - rx1)];
    } else if (k == d - 1) {
      v = (p < rx0) ? Xk[p + rx0 * i] : Yk[(p - rx0) + ry0 * i];
    } else {
      if (p < rx0 && q < rx1) v = Xk[p + rx0 * (i + n * q)];
      else if (p >= rx0 && q >= rx1) v = Yk[(p - rx0) + ry0 * (i + n * (q - rx1))];
    }
    Zk[e] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    z.r[k] = rz0;
    if (k == d - 1) z.r[k + 1] = 1;
  }
}

tt_status add_meta(const VecMeta &x, const double *alpha, const VecMeta &y, const double *beta,
                   const VecMeta &z, cudaStream_t s) {
  if (x.d != y.d || x.d != z.d) return fail(TT_ERR_SHAPE, "tt_add: number of cores differ");
  long long mx = 0;
  for (int k = 0; k < x.d; ++k) {
    if (x.n[k] != y.n[k] || x.n[k] != z.n[k]) return fail(TT_ERR_SHAPE, "tt_add: shape mismatch");
    long long c = (long long)z.rcap[k] * z.n[k] * z.rcap[k + 1];
    mx = c > mx ? c : mx;
  }
  for (int k = 1; k < x.d; ++k)
    if (z.rcap[k] < x.rcap[k] + y.rcap[k]) return fail(TT_ERR_CAPACITY, "tt_add: z rank capacity < rx+ry");
  // (keff sizes B with exactly these capacities)
  int bx = (int)((mx + 255) / 256);
  bx = bx > 1024 ? 1024 : (bx < 1 ? 1 : bx);
  add_kernel<<<dim3(bx, x.d), 256, 0, s>>>(x, alpha, y, beta, z);
  return check_launch("tt_add");
}

// --------------------------------------------------------------- scale ---
__global__ void scale_kernel(const VecMeta x, const double *alpha, double ah, int invert) {
  const int n = x.n[0] * x.r[1];
  double a = alpha ? *alpha : ah;
  if (invert) a = 1.0 / a;
  double *X0 = x.data + x.off[0];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) X0[e] *= a;
}
tt_status scale_meta(const VecMeta &x, const double *alpha_dev, double alpha_host, int invert,
                     cudaStream_t s) {
  int cap = x.n[0] * x.rcap[1];
  int bx = (cap + 255) / 256;
  bx = bx > 256 ? 256 : bx;
  scale_kernel<<<bx, 256, 0, s>>>(x, alpha_dev, alpha_host, invert);
  return check_launch("tt_scale");
}

// ---------------------------------------------------------------- copy ---
__global__ void copy_kernel(const VecMeta x, const VecMeta y) {
  const int k = blockIdx.y;
  const int total = x.r[k] * x.n[k] * x.r[k + 1];
  const double *X = x.data + x.off[k];
  double *Y = y.data + y.off[k];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) Y[e] = X[e];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    y.r[k] = x.r[k];
    if (k == x.d - 1) y.r[k + 1] = x.r[k + 1];
  }
}
tt_status copy_meta(const VecMeta &x, const VecMeta &y, cudaStream_t s) {
  if (x.d != y.d) return fail(TT_ERR_SHAPE, "tt_copy: number of cores differ");
  for (int k = 0; k < x.d; ++k)
    if (x.n[k] != y.n[k]) return fail(TT_ERR_SHAPE, "tt_copy: shape mismatch");
  for (int k = 0; k <= x.d; ++k)
    if (y.rcap[k] < x.rcap[k]) return fail(TT_ERR_CAPACITY, "tt_copy: capacity");
  int bx = (max_slot(x) + 255) / 256;
  bx = bx > 1024 ? 1024 : (bx < 1 ? 1 : bx);
  copy_kernel<<<dim3(bx, x.d), 256, 0, s>>>(x, y);
  return check_launch("tt_copy");
}

// ----------------------------------------------------------------- dot ---
// <x, y> by the left-to-right chain W_k = sum_i X_k(i)^T W_{k-1} Y_k(i), one CTA.
__global__ void __launch_bounds__(512) dot_kernel(const VecMeta x, const VecMeta y, double *W, double *Z,
                                                  double *out) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) W[0] = 1.0;
  __syncthreads();
  for (int k = 0; k < x.d; ++k) {
    const int n = x.n[k];
    const int rx0 = x.r[k], rx1 = x.r[k + 1], ry0 = y.r[k], ry1 = y.r[k + 1];
    const double *X = x.data + x.off[k];
    const double *Y = y.data + y.off[k];
    // Z[a, i, b'] = sum_b W[a, b] Y[b, i, b']
    const int nz = rx0 * n * ry1;
    for (int e = tid; e < nz; e += nt) {
      const int a = e % rx0, t = e / rx0, i = t % n, b1 = t / n;
      double s = 0.0;
      for (int b = 0; b < ry0; ++b) s = fma(W[a + rx0 * b], Y[b + ry0 * (i + n * b1)], s);
      Z[e] = s;
    }
    __syncthreads();
    // W'[a', b'] = sum_{a, i} X[a, i, a'] Z[a, i, b']
    const int nw = rx1 * ry1;
    const int kk = rx0 * n;
    for (int e = tid; e < nw; e += nt) {
      const int a1 = e % rx1, b1 = e / rx1;
      double s = 0.0;
      for (int q = 0; q < kk; ++q) s = fma(X[q + kk * a1], Z[q + kk * b1], s);
      W[e] = s;
    }
    __syncthreads();
  }
  if (tid == 0) *out = W[0];
}

tt_status dot_meta(const VecMeta &x, const VecMeta &y, double *out, Arena &ar, cudaStream_t s) {
  if (x.d != y.d) return fail(TT_ERR_SHAPE, "tt_dot: number of cores differ");
  long long wmax = 1, zmax = 1;
  for (int k = 0; k < x.d; ++k) {
    if (x.n[k] != y.n[k]) return fail(TT_ERR_SHAPE, "tt_dot: shape mismatch");
    long long w = (long long)x.rcap[k + 1] * y.rcap[k + 1];
    long long z = (long long)x.rcap[k] * x.n[k] * y.rcap[k + 1];
    wmax = w > wmax ? w : wmax;
    zmax = z > zmax ? z : zmax;
  }
  double *W = ar.take<double>(wmax);
  double *Z = ar.take<double>(zmax);
  if (!ar.base) return TT_OK;
  if (!ar.ok()) return fail(TT_ERR_CAPACITY, "tt_dot: workspace too small");
  dot_kernel<<<1, 512, 0, s>>>(x, y, W, Z, out);
  return check_launch("tt_dot");
}

// ---------------------------------------------------------------- copy ---
__global__ void copy_desc_kernel(const CopyDesc *descs) {
  const CopyDesc g = descs[blockIdx.y];
  const long long total = (long long)g.rows * g.cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e % g.rows), c = (int)(e / g.rows);
    g.dst[r * g.ds_r + c * g.ds_c] = g.src[r * g.ss_r + c * g.ss_c];
  }
}
tt_status launch_copy(const CopyDesc *descs_dev, int count, long long cap, cudaStream_t s) {
  if (count <= 0) return TT_OK;
  int bx = (int)((cap + 255) / 256);
  bx = bx > 1024 ? 1024 : (bx < 1 ? 1 : bx);
  copy_desc_kernel<<<dim3(bx, count), 256, 0, s>>>(descs_dev);
  return check_launch("copy");
}

}  // namespace tt
