// tt_orthogonalize (a3) and tt_round (a4): host-ordered chains of kernels whose
// sizes follow the device-resident ranks.  Each step launches a one-thread
// "plan" kernel that reads the current ranks and writes the descriptors of
// the step's QR / SVD / GEMM / copy kernels into the workspace; nothing is
// read back to the host, so the whole sweep is graph-capturable.
#include <algorithm>
#include <cmath>
#include <vector>

#include "tt_common.cuh"

namespace tt {

namespace {

struct StepWS {
  double *A, *Q, *R, *tau, *T, *U, *V, *S, *J, *QU, *tmp;
  QRDesc *qd;
  SVDDesc *sd;
  GemmDesc *gd;   // [2]: slot s at gd[s * bs]
  CopyDesc *cd;   // [2]: slot s at cd[s * bs]
  int bs;         // batch stride of the descriptor slots (1 unbatched, B in tt_round_batched)
  int *iv;        // [8] step integers (wide flag, sizes)
  double *norm;   // [1]
  unsigned int *bar;  // [4] grid barrier of the block Jacobi
  long long Acap, slot;
  char *qrws;         // TSQR scratch of the tall unfoldings
  size_t qrwsb;
};

struct Caps {
  long long slot;  // max core slot (elements)
  int rmax;        // max rank capacity
  int mq, pq;      // max QR rows / cols
};

// capacity shapes of the QR problems of orthogonalisation / truncation step k
struct QCap { int m, n; };
QCap qcap_rl(const VecMeta &x, int k) { return {x.n[k] * x.rcap[k + 1], x.rcap[k]}; }
QCap qcap_lr(const VecMeta &x, int k) { return {x.rcap[k] * x.n[k], x.rcap[k + 1]}; }
QCap qcap_trunc(const VecMeta &x, int k) {
  const int a = x.rcap[k] * x.n[k], b = x.rcap[k + 1];
  return {a > b ? a : b, a < b ? a : b};
}
size_t qr_ws_max(const VecMeta &x) {
  size_t b = 0;
  for (int k = 0; k < x.d; ++k) {
    QCap c[3] = {qcap_rl(x, k), qcap_lr(x, k), qcap_trunc(x, k)};
    for (auto &q : c) {
      const size_t v = qr_tall_ws_bytes(q.m, q.n);
      b = v > b ? v : b;
    }
  }
  return b;
}

Caps caps_of(const VecMeta &x) {
  Caps c;
  c.slot = max_slot(x);
  c.rmax = max_rank(x);
  c.mq = 1;
  c.pq = 1;
  for (int k = 0; k < x.d; ++k) {
    int a = x.n[k] * x.rcap[k + 1], b = x.rcap[k] * x.n[k];
    c.mq = a > c.mq ? a : c.mq;
    c.mq = b > c.mq ? b : c.mq;
  }
  c.pq = c.rmax;
  return c;
}

StepWS carve(const VecMeta &x, Arena &ar) {
  Caps c = caps_of(x);
  StepWS w;
  const long long pc = c.rmax;
  w.slot = c.slot;
  w.Acap = c.slot;
  w.A = ar.take<double>(c.slot);
  w.Q = ar.take<double>(c.slot);
  w.R = ar.take<double>(pc * pc);
  w.tau = ar.take<double>(pc);
  w.T = ar.take<double>(32 * 32 * (pc / 32 + 1));
  w.U = ar.take<double>(pc * pc);
  w.V = ar.take<double>(pc * pc);
  w.S = ar.take<double>(pc);
  w.J = ar.take<double>(2 * pc * pc);
  w.QU = ar.take<double>(c.slot);
  w.tmp = ar.take<double>(c.slot);
  w.qd = ar.take<QRDesc>(1);
  w.sd = ar.take<SVDDesc>(1);
  w.gd = ar.take<GemmDesc>(2);
  w.cd = ar.take<CopyDesc>(2);
  w.bs = 1;
  w.iv = ar.take<int>(8);
  w.norm = ar.take<double>(1);
  w.bar = ar.take<unsigned int>(4);
  w.qrwsb = qr_ws_max(x);
  w.qrws = ar.take<char>(w.qrwsb);
  return w;
}

__device__ GemmDesc gemm_desc(int M, int N, int K, const double *A, long long lda, int tA, const double *B,
                              long long ldb, int tB, double *C, long long ldc) {
  GemmDesc g;
  g.M = M; g.N = N; g.K = K;
  g.transA = tA; g.transB = tB;
  g.A = A; g.lda = lda;
  g.B = B; g.ldb = ldb;
  gemm_plain_c(g, C, ldc);
  g.alpha = 1.0; g.beta = 0.0; g.alpha_dev = nullptr; g.skip = nullptr;
  g.batch = 0; g.bsA = g.bsB = g.bsC = 0;
  return g;
}

__device__ CopyDesc copy_desc(int rows, int cols, const double *src, long long ssr, long long ssc, double *dst,
                              long long dsr, long long dsc) {
  CopyDesc c;
  c.rows = rows; c.cols = cols;
  c.src = src; c.ss_r = ssr; c.ss_c = ssc;
  c.dst = dst; c.ds_r = dsr; c.ds_c = dsc;
  return c;
}

// ---- right-to-left orthogonalisation step at core k (k >= 1)
__device__ __forceinline__ void plan_orth_rl_d(const VecMeta &x, int k, const StepWS &w) {
  const int r0 = x.r[k], n = x.n[k], r1 = x.r[k + 1];
  const int rp = x.r[k - 1], np = x.n[k - 1];
  const int m = n * r1, p = r0, q = min(m, p);
  double *core = x.data + x.off[k];
  double *prev = x.data + x.off[k - 1];
  QRDesc &d = *w.qd;
  d.m = m; d.n = p;
  d.src = core; d.src_rs = r0; d.src_cs = 1;          // M^T(row=(i,b), col=a) = core[a + r0 row]
  d.A = w.A; d.lda = m;
  d.Q = core; d.q_rs = q; d.q_cs = 1;                 // new core [q, n, r1] = Q^T
  d.R = w.R; d.ldr = q;
  d.tau = w.tau; d.T = w.T;
  d.rt = 0;
  w.gd[0] = gemm_desc(rp * np, q, p, prev, (long long)rp * np, 0, w.R, q, 1, w.tmp, (long long)rp * np);
  w.cd[0] = copy_desc(rp * np, q, w.tmp, 1, (long long)rp * np, prev, 1, (long long)rp * np);
  x.r[k] = q;
}

// ---- left-to-right orthogonalisation step at core k (k <= d-2)
__device__ __forceinline__ void plan_orth_lr_d(const VecMeta &x, int k, const StepWS &w) {
  const int r0 = x.r[k], n = x.n[k], r1 = x.r[k + 1];
  const int n2 = x.n[k + 1], r2 = x.r[k + 2];
  const int m = r0 * n, p = r1, q = min(m, p);
  double *core = x.data + x.off[k];
  double *next = x.data + x.off[k + 1];
  QRDesc &d = *w.qd;
  d.m = m; d.n = p;
  d.src = core; d.src_rs = 1; d.src_cs = m;
  d.A = w.A; d.lda = m;
  d.Q = core; d.q_rs = 1; d.q_cs = m;                 // new core [r0, n, q] = Q
  d.R = w.R; d.ldr = q;
  d.tau = w.tau; d.T = w.T;
  d.rt = 0;
  w.gd[0] = gemm_desc(q, n2 * r2, p, w.R, q, 0, next, p, 0, w.tmp, q);
  w.cd[0] = copy_desc(q, n2 * r2, w.tmp, 1, q, next, 1, q);
  x.r[k + 1] = q;
}

__device__ __forceinline__ void core_norm_d(const VecMeta &x, int k, double *out, double *out2) {
  __shared__ double red[32];
  const int total = x.r[k] * x.n[k] * x.r[k + 1];
  const double *c = x.data + x.off[k];
  double s = 0.0;
  for (int e = threadIdx.x; e < total; e += blockDim.x) s = fma(c[e], c[e], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    t = sqrt(t);
    if (out) *out = t;
    if (out2) *out2 = t;
  }
}

// ---- truncation step at core k (k <= d-2): SVD of the left unfolding
__device__ __forceinline__ void plan_trunc_d(const VecMeta &x, int k, const StepWS &w) {
  const int r0 = x.r[k], n = x.n[k], r1 = x.r[k + 1];
  const int m0 = r0 * n, p0 = r1;
  const int wide = m0 < p0;
  const int p = wide ? m0 : p0;
  double *core = x.data + x.off[k];
  QRDesc &d = *w.qd;
  if (!wide) {
    d.m = m0; d.n = p0;
    d.src = core; d.src_rs = 1; d.src_cs = m0;
    d.Q = w.Q; d.q_rs = 1; d.q_cs = m0;
  } else {
    d.m = p0; d.n = m0;
    d.src = core; d.src_rs = m0; d.src_cs = 1;
    d.Q = w.Q; d.q_rs = 1; d.q_cs = p0;
  }
  d.A = w.A; d.lda = d.m;
  d.R = w.R; d.ldr = p;
  d.tau = w.tau; d.T = w.T;
  // one-sided Jacobi on R^T (= V_R S U_R^T): converges in far fewer sweeps than on R
  // when the spectrum decays (preconditioning by the QR); U and V swap roles
  d.rt = 1;
  SVDDesc &s = *w.sd;
  s.m = p; s.p = p;
  s.W = w.R; s.ldw = p;
  s.U = w.V; s.ldu = p;
  s.V = w.U; s.ldv = p;
  s.sigma = w.S;
  s.work = w.J;
  s.sweeps_out = nullptr;
  w.iv[0] = wide; w.iv[1] = p; w.iv[2] = m0; w.iv[3] = p0;
}

__device__ __forceinline__ void trunc_d(const VecMeta &x, int k, const StepWS &w, double eps, int rmax,
                                        double *disc, double *sv, int sv_stride) {
  __shared__ int s_r;
  const int wide = w.iv[0], p = w.iv[1], m0 = w.iv[2], p0 = w.iv[3];
  const int tid = threadIdx.x;
  if (tid == 0) {
    const double delta = (x.d > 1) ? eps * (*w.norm) / sqrt((double)(x.d - 1)) : 0.0;
    const double d2 = delta * delta;
    // reading Z21: smallest r >= 1 with sum_{i>r} s_i^2 <= delta^2, then min(r, rmax)
    double tail = 0.0;
    int r = p;
    for (int i = p - 1; i >= 1; --i) {
      const double t2 = tail + w.S[i] * w.S[i];
      if (t2 <= d2) {
        tail = t2;
        r = i;
      } else {
        break;
      }
    }
    r = r < 1 ? 1 : r;
    r = r > rmax ? rmax : r;
    double disc_v = 0.0;
    for (int i = r; i < p; ++i) disc_v += w.S[i] * w.S[i];
    if (disc) disc[k] = disc_v;
    s_r = r;
    x.r[k + 1] = r;
  }
  if (sv)
    for (int i = tid; i < sv_stride; i += blockDim.x) sv[(long long)k * sv_stride + i] = i < p ? w.S[i] : 0.0;
  __syncthreads();
  const int r = s_r;
  // fold Sigma into V (not wide) or U (wide)
  double *Mx = wide ? w.U : w.V;
  for (int e = tid; e < p * r; e += blockDim.x) {
    const int row = e % p, c = e / p;
    Mx[row + (long long)c * p] *= w.S[c];
  }
  if (tid == 0) {
    const int n2 = x.n[k + 1], r2 = x.r[k + 2];
    double *core = x.data + x.off[k];
    double *next = x.data + x.off[k + 1];
    if (!wide) {
      w.gd[0] = gemm_desc(m0, r, p, w.Q, m0, 0, w.U, p, 0, core, m0);
      w.gd[w.bs] = gemm_desc(r, n2 * r2, p0, w.V, p, 1, next, p0, 0, w.tmp, r);
      w.cd[0] = copy_desc(0, 0, nullptr, 0, 0, nullptr, 0, 0);
    } else {
      w.gd[0] = gemm_desc(p0, r, m0, w.Q, p0, 0, w.U, m0, 0, w.QU, p0);
      w.cd[0] = copy_desc(m0, r, w.V, 1, p, core, 1, m0);
      w.gd[w.bs] = gemm_desc(r, n2 * r2, p0, w.QU, p0, 1, next, p0, 0, w.tmp, r);
    }
    w.cd[w.bs] = copy_desc(r, n2 * r2, w.tmp, 1, r, next, 1, r);
  }
}

// single-instance kernels and their batched forms (instance = blockIdx.x)
__global__ void plan_orth_rl(const VecMeta x, int k, StepWS w) { plan_orth_rl_d(x, k, w); }
__global__ void plan_orth_lr(const VecMeta x, int k, StepWS w) { plan_orth_lr_d(x, k, w); }
__global__ void plan_trunc(const VecMeta x, int k, StepWS w) { plan_trunc_d(x, k, w); }
__global__ void core_norm_kernel(const VecMeta x, int k, double *out, double *out2) { core_norm_d(x, k, out, out2); }
__global__ void trunc_kernel(const VecMeta x, int k, StepWS w, double eps, int rmax, double *disc, double *sv,
                             int sv_stride) {
  trunc_d(x, k, w, eps, rmax, disc, sv, sv_stride);
}
__global__ void plan_orth_rl_b(const VecMeta *xs, int k, const StepWS *ws) {
  if (k < xs[blockIdx.x].d) plan_orth_rl_d(xs[blockIdx.x], k, ws[blockIdx.x]);
}
__global__ void plan_trunc_b(const VecMeta *xs, int k, const StepWS *ws) {
  plan_trunc_d(xs[blockIdx.x], k, ws[blockIdx.x]);
}
__global__ void core_norm_b(const VecMeta *xs, const StepWS *ws) {
  core_norm_d(xs[blockIdx.x], 0, nullptr, ws[blockIdx.x].norm);
}
__global__ void trunc_b(const VecMeta *xs, int k, const StepWS *ws, double eps, int rmax, double *disc, int dstride) {
  trunc_d(xs[blockIdx.x], k, ws[blockIdx.x], eps, rmax, disc ? disc + (long long)blockIdx.x * dstride : nullptr,
          nullptr, 0);
}

}  // namespace

// --------------------------------------------------------------- drivers ---
tt_status orth_meta(const VecMeta &x, int dir, double *norm_dev, Arena &ar, cudaStream_t s) {
  StepWS w = carve(x, ar);
  if (!ar.base) return TT_OK;
  if (!ar.ok()) return fail(TT_ERR_CAPACITY, "tt_orthogonalize: workspace too small");
  const Caps c = caps_of(x);
  const int d = x.d;
  if (dir < 0) {
    for (int k = d - 1; k >= 1; --k) {
      plan_orth_rl<<<1, 1, 0, s>>>(x, k, w);
      const QCap qc = qcap_rl(x, k);
      TT_TRY(launch_qr_tall(w.qd, qc.m, qc.n, w.qrws, w.qrwsb, s));
      TT_TRY(launch_gemm(w.gd, 1, x.rcap[k - 1] * x.n[k - 1], x.rcap[k], s));
      TT_TRY(launch_copy(w.cd, 1, (long long)x.rcap[k - 1] * x.n[k - 1] * x.rcap[k], s));
    }
    core_norm_kernel<<<1, 256, 0, s>>>(x, 0, norm_dev, w.norm);
  } else {
    for (int k = 0; k <= d - 2; ++k) {
      plan_orth_lr<<<1, 1, 0, s>>>(x, k, w);
      const QCap qc = qcap_lr(x, k);
      TT_TRY(launch_qr_tall(w.qd, qc.m, qc.n, w.qrws, w.qrwsb, s));
      TT_TRY(launch_gemm(w.gd, 1, x.rcap[k + 1], x.n[k + 1] * x.rcap[k + 2], s));
      TT_TRY(launch_copy(w.cd, 1, (long long)x.rcap[k + 1] * x.n[k + 1] * x.rcap[k + 2], s));
    }
    core_norm_kernel<<<1, 256, 0, s>>>(x, d - 1, norm_dev, w.norm);
  }
  (void)c;
  return check_launch("tt_orthogonalize");
}

tt_status round_meta(const VecMeta &x, double eps, int rmax, double *disc, double *sv, int sv_stride,
                     Arena &ar, cudaStream_t s) {
  if (eps < 0.0 || !(eps == eps)) return fail(TT_ERR_ARG, "tt_round: eps must be >= 0");
  if (rmax < 1) return fail(TT_ERR_ARG, "tt_round: rmax must be >= 1");
  const size_t mark = ar.used;
  StepWS w = carve(x, ar);
  if (!ar.base) return TT_OK;
  if (!ar.ok()) return fail(TT_ERR_CAPACITY, "tt_round: workspace too small");
  ar.used = mark;  // orth_meta re-carves the same layout
  TT_TRY(orth_meta(x, -1, nullptr, ar, s));
  set_jacobi_sync(w.bar);
  const Caps c = caps_of(x);
  const int d = x.d;
  for (int k = 0; k <= d - 2; ++k) {
    const int m0cap = x.rcap[k] * x.n[k], p0cap = x.rcap[k + 1];
    const int pcap = m0cap < p0cap ? m0cap : p0cap;
    plan_trunc<<<1, 1, 0, s>>>(x, k, w);
    const QCap qc = qcap_trunc(x, k);
    TT_TRY(launch_qr_tall(w.qd, qc.m, qc.n, w.qrws, w.qrwsb, s));
    TT_TRY(launch_jacobi(w.sd, 1, pcap, pcap, s));
    trunc_kernel<<<1, 256, 0, s>>>(x, k, w, eps, rmax, disc, sv, sv_stride);
    const int mx = m0cap > p0cap ? m0cap : p0cap;
    TT_TRY(launch_gemm(w.gd, 1, mx, x.rcap[k + 1], s));
    TT_TRY(launch_copy(w.cd, 1, (long long)m0cap * x.rcap[k + 1], s));
    TT_TRY(launch_gemm(w.gd + 1, 1, x.rcap[k + 1], x.n[k + 1] * x.rcap[k + 2], s));
    TT_TRY(launch_copy(w.cd + 1, 1, (long long)x.rcap[k + 1] * x.n[k + 1] * x.rcap[k + 2], s));
  }
  (void)c;
  return check_launch("tt_round");
}

// ----------------------------------------------------- batched rounding ---
// B independent TT-vectors of the same number of cores rounded together: every
// orthogonalisation / truncation step is one plan launch over the B instances
// (grid B), one QR launch with B descriptors (one CTA per instance), one
// Jacobi launch with B descriptors, and batched GEMM / copy launches (grid z =
// instance) — 4 + 8 launches per core instead of B times that, and the B
// latency-bound QR / SVD chains run side by side on the SMs.
tt_status round_batched_meta(int B, const VecMeta *xs, double eps, int rmax, double *disc, int dstride, Arena &ar,
                             cudaStream_t s) {
  if (B < 1) return fail(TT_ERR_ARG, "tt_round_batched: B must be >= 1");
  if (eps < 0.0 || !(eps == eps)) return fail(TT_ERR_ARG, "tt_round_batched: eps must be >= 0");
  if (rmax < 1) return fail(TT_ERR_ARG, "tt_round_batched: rmax must be >= 1");
  const int d = xs[0].d;
  for (int b = 1; b < B; ++b)
    if (xs[b].d != d) return fail(TT_ERR_SHAPE, "tt_round_batched: instances must have the same number of cores");
  std::vector<StepWS> w(B);
  for (int b = 0; b < B; ++b) w[b] = carve(xs[b], ar);
  QRDesc *qd = ar.take<QRDesc>(B);
  SVDDesc *sd = ar.take<SVDDesc>(B);
  GemmDesc *gd = ar.take<GemmDesc>(2 * B);
  CopyDesc *cd = ar.take<CopyDesc>(2 * B);
  VecMeta *xd = ar.take<VecMeta>(B);
  StepWS *wd = ar.take<StepWS>(B);
  if (!ar.base) return TT_OK;
  if (!ar.ok()) return fail(TT_ERR_CAPACITY, "tt_round_batched: workspace too small");
  for (int b = 0; b < B; ++b) {
    w[b].qd = qd + b;
    w[b].sd = sd + b;
    w[b].gd = gd + b;
    w[b].cd = cd + b;
    w[b].bs = B;
  }
  // pageable source: cudaMemcpyAsync returns once the host arrays have been consumed
  if (cudaMemcpyAsync(xd, xs, sizeof(VecMeta) * B, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(wd, w.data(), sizeof(StepWS) * B, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return fail(TT_ERR_CUDA, "tt_round_batched: descriptor upload");
  auto cap_max = [&](auto f) {
    long long v = 0;
    for (int b = 0; b < B; ++b) v = std::max<long long>(v, f(xs[b]));
    return v;
  };
  // right-to-left orthogonalisation
  for (int k = d - 1; k >= 1; --k) {
    plan_orth_rl_b<<<B, 1, 0, s>>>(xd, k, wd);
    TT_TRY(launch_qr(qd, B, s));
    const int Mc = (int)cap_max([&](const VecMeta &x) { return (long long)x.rcap[k - 1] * x.n[k - 1]; });
    const int Nc = (int)cap_max([&](const VecMeta &x) { return (long long)x.rcap[k]; });
    TT_TRY(launch_gemm(gd, B, Mc, Nc, s));
    TT_TRY(launch_copy(cd, B, cap_max([&](const VecMeta &x) {
      return (long long)x.rcap[k - 1] * x.n[k - 1] * x.rcap[k]; }), s));
  }
  core_norm_b<<<B, 256, 0, s>>>(xd, wd);
  // left-to-right truncation
  for (int k = 0; k <= d - 2; ++k) {
    const int m0c = (int)cap_max([&](const VecMeta &x) { return (long long)x.rcap[k] * x.n[k]; });
    const int p0c = (int)cap_max([&](const VecMeta &x) { return (long long)x.rcap[k + 1]; });
    const int pcap = (int)cap_max([&](const VecMeta &x) {
      const long long a = (long long)x.rcap[k] * x.n[k], c = x.rcap[k + 1];
      return a < c ? a : c; });
    plan_trunc_b<<<B, 1, 0, s>>>(xd, k, wd);
    TT_TRY(launch_qr(qd, B, s));
    TT_TRY(launch_jacobi(sd, B, pcap, pcap, s));
    trunc_b<<<B, 256, 0, s>>>(xd, k, wd, eps, rmax, disc, dstride);
    TT_TRY(launch_gemm(gd, B, m0c > p0c ? m0c : p0c, p0c, s));
    TT_TRY(launch_copy(cd, B, (long long)m0c * p0c, s));
    const int n2r2 = (int)cap_max([&](const VecMeta &x) { return (long long)x.n[k + 1] * x.rcap[k + 2]; });
    TT_TRY(launch_gemm(gd + B, B, p0c, n2r2, s));
    TT_TRY(launch_copy(cd + B, B, (long long)p0c * n2r2, s));
  }
  return check_launch("tt_round_batched");
}

}  // namespace tt
