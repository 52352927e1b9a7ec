// als_local_apply (a6) and als_update_interfaces (a5) with host-side sizes:
// three DMMA GEMMs per call; descriptors staged into the workspace by a tiny
// by-value kernel (graph-capturable, no host->device memcpy).
#include "als.h"

namespace tt {

namespace {
struct Desc3 {
  GemmDesc g[3];
};
struct Desc4 {
  GemmDesc g[4];
};
__global__ void set_descs4_kernel(Desc4 in, GemmDesc *out, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) out[i] = in.g[i];
}
// Dc[g + R (g' + Rp i)] = Ak[g, i, i, g'] (host sizes)
__global__ void diag_extract_raw_kernel(const double *Ak, int R, int Rp, int m, double *Dc) {
  const long long tot = (long long)R * Rp * m;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(e % R);
    const long long t = e / R;
    const int gp = (int)(t % Rp), i = (int)(t / Rp);
    Dc[e] = Ak[g + (long long)R * i * (1 + m) + (long long)R * m * m * gp];
  }
}
__global__ void set_descs_kernel(Desc3 in, GemmDesc *out, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) out[i] = in.g[i];
}

long long prod(long long a, long long b, long long c, long long d) { return a * b * c * d; }
}  // namespace

static tt_status run3(const Desc3 &d, int count, GemmDesc *dev, const int *Mc, const int *Nc, cudaStream_t s) {
  set_descs_kernel<<<1, 32, 0, s>>>(d, dev, count);
  TT_TRY(check_launch("set_descs"));
  for (int i = 0; i < count; ++i) TT_TRY(launch_gemm_k(dev + i, 1, Mc[i], Nc[i], d.g[i].K, s, d.g[i].batch));
  return TT_OK;
}
// descriptors with host sizes: grid caps are the descriptors' own sizes
static tt_status run_descs(const GemmDesc *g, int count, GemmDesc *dev, cudaStream_t s) {
  Desc4 d;
  for (int i = 0; i < count; ++i) d.g[i] = g[i];
  set_descs4_kernel<<<1, 32, 0, s>>>(d, dev, count);
  TT_TRY(check_launch("set_descs"));
  for (int i = 0; i < count; ++i)
    if (g[i].M > 0 && g[i].N > 0) TT_TRY(launch_gemm_k(dev + i, 1, g[i].M, g[i].N, g[i].K, s, g[i].batch));
  return TT_OK;
}

size_t als_ws_bytes(long long rA, long long R, long long rB, long long m, long long n, long long rAp, long long Rp,
                    long long rBp) {
  long long t1 = prod(rB, n, rAp, Rp);
  long long t1b = prod(R, m, rB, rAp);
  long long mx = t1 > t1b ? t1 : t1b;
  // covers apply (T1, T2) and both interface directions (T1, T2 of at most the same sizes)
  long long t2 = prod(R, m, rB, rAp);
  long long t2b = prod(rB, n, rAp, Rp);
  long long mx2 = t2 > t2b ? t2 : t2b;
  size_t b = 0;
  b += ((size_t)mx * 8 + 255) & ~size_t(255);
  b += ((size_t)mx2 * 8 + 255) & ~size_t(255);
  b += ((4 * sizeof(GemmDesc)) + 255) & ~size_t(255);
  b += GEMM_SPLIT_SCRATCH;
  return b;
}

// structured forms: the dense workspace plus, for absorb, Pt [rA rB Rp m] and Dc [R Rp m]
size_t als_ws_bytes_structured(int absorb, long long rA, long long R, long long rB, long long m, long long n,
                               long long rAp, long long Rp, long long rBp) {
  size_t b = als_ws_bytes(rA, R, rB, m, n, rAp, Rp, rBp);
  if (absorb) {
    b += ((size_t)prod(rA, rB, Rp, m) * 8 + 255) & ~size_t(255);
    b += ((size_t)prod(R, Rp, m, 1) * 8 + 255) & ~size_t(255);
  }
  return b;
}

}  // namespace tt

using namespace tt;

static bool dims_ok(int a, int b, int c, int d, int e, int f, int g, int h) {
  return a > 0 && b > 0 && c > 0 && d > 0 && e > 0 && f > 0 && g > 0 && h > 0;
}

extern "C" size_t als_workspace(int32_t rA, int32_t R, int32_t rB, int32_t m, int32_t n, int32_t rAp, int32_t Rp,
                                int32_t rBp) {
  return als_ws_bytes(rA, R, rB, m, n, rAp, Rp, rBp);
}

extern "C" tt_status als_local_apply(int32_t rA, int32_t R, int32_t rB, int32_t m, int32_t n, int32_t rAp,
                                     int32_t Rp, int32_t rBp, const double *Phi, const double *Ak,
                                     const double *Psi, const double *x, double *y, void *ws, size_t wsb,
                                     tt_stream st) {
  if (!dims_ok(rA, R, rB, m, n, rAp, Rp, rBp)) return fail(TT_ERR_ARG, "als_local_apply: sizes must be >= 1");
  if (!Phi || !Ak || !Psi || !x || !y || !ws) return fail(TT_ERR_ARG, "als_local_apply: NULL pointer");
  if (wsb < als_ws_bytes(rA, R, rB, m, n, rAp, Rp, rBp)) return fail(TT_ERR_CAPACITY, "als_local_apply: workspace");
  cudaStream_t s = (cudaStream_t)st;
  Arena ar;
  ar.base = (char *)ws;
  ar.cap = wsb;
  long long t1n = (long long)rB * n * rAp * Rp, t2n = (long long)R * m * rB * rAp;
  long long mx = t1n > t2n ? t1n : t2n;
  double *T1 = ar.take<double>(mx);
  double *T2 = ar.take<double>(mx);
  GemmDesc *dev = ar.take<GemmDesc>(3);
  set_gemm_scratch(ar.take<double>(GEMM_SPLIT_SCRATCH / 8), GEMM_SPLIT_SCRATCH);
  ScratchScope scratch_scope;
  Desc3 d;
  descs_local_apply(rA, R, rB, m, n, rAp, Rp, rBp, Phi, Ak, Psi, x, y, T1, T2, d.g);
  int Mc[3] = {rB * n, R * m, rA}, Nc[3] = {rAp * Rp, rB * rAp, m * rAp};
  return run3(d, 3, dev, Mc, Nc, s);
}

extern "C" tt_status als_update_interfaces(int32_t dir, int32_t rY, int32_t R, int32_t rX, int32_t m, int32_t n,
                                           int32_t rYp, int32_t Rp, int32_t rXp, const double *Iprev,
                                           const double *Yk, const double *Ak, const double *Xk, double *Inext,
                                           void *ws, size_t wsb, tt_stream st) {
  if (!dims_ok(rY, R, rX, m, n, rYp, Rp, rXp)) return fail(TT_ERR_ARG, "als_update_interfaces: sizes must be >= 1");
  if (!Iprev || !Yk || !Xk || !Inext || !ws) return fail(TT_ERR_ARG, "als_update_interfaces: NULL pointer");
  if (dir != 1 && dir != -1) return fail(TT_ERR_ARG, "als_update_interfaces: dir must be +1 or -1");
  if (!Ak && (R != 1 || Rp != 1 || m != n))
    return fail(TT_ERR_ARG, "als_update_interfaces: vector interface needs R = Rp = 1 and m = n");
  if (wsb < als_ws_bytes(rY, R, rX, m, n, rYp, Rp, rXp))
    return fail(TT_ERR_CAPACITY, "als_update_interfaces: workspace");
  cudaStream_t s = (cudaStream_t)st;
  Arena ar;
  ar.base = (char *)ws;
  ar.cap = wsb;
  long long t1n = (long long)rX * n * rYp * Rp, t2n = (long long)R * m * rX * rYp;
  long long mx = t1n > t2n ? t1n : t2n;
  double *T1 = ar.take<double>(mx);
  double *T2 = ar.take<double>(mx);
  GemmDesc *dev = ar.take<GemmDesc>(3);
  set_gemm_scratch(ar.take<double>(GEMM_SPLIT_SCRATCH / 8), GEMM_SPLIT_SCRATCH);
  ScratchScope scratch_scope;
  Desc3 d;
  if (Ak) {
    if (dir > 0) {
      descs_iface_left(rY, R, rX, m, n, rYp, Rp, rXp, Iprev, Yk, Ak, Xk, Inext, T1, T2, d.g);
      int Mc[3] = {R * rX, rX * rYp, rYp * Rp}, Nc[3] = {m * rYp, n * Rp, rXp};
      return run3(d, 3, dev, Mc, Nc, s);
    } else {
      descs_iface_right(rY, R, rX, m, n, rYp, Rp, rXp, Iprev, Yk, Ak, Xk, Inext, T1, T2, d.g);
      int Mc[3] = {rX * n, R * m, rY}, Nc[3] = {rYp * Rp, rX * rYp, R * rX};
      return run3(d, 3, dev, Mc, Nc, s);
    }
  }
  if (dir > 0) {
    descs_iface_left_vec(rY, rX, m, rYp, rXp, Iprev, Yk, Xk, Inext, T1, d.g);
    int Mc[2] = {rX, rYp}, Nc[2] = {m * rYp, rXp};
    return run3(d, 2, dev, Mc, Nc, s);
  }
  descs_iface_right_vec(rY, rX, m, rYp, rXp, Iprev, Yk, Xk, Inext, T1, d.g);
  int Mc[2] = {rX * m, rY}, Nc[2] = {rYp, rX};
  return run3(d, 2, dev, Mc, Nc, s);
}

extern "C" tt_status tt_core_kinds(const tt_mat *A, int32_t *kinds, double *offdiag_ratio, void *ws, size_t wsb,
                                   tt_stream st) {
  MatMeta am;
  TT_TRY(make_mat_meta(A, am));
  if (!kinds) return fail(TT_ERR_ARG, "tt_core_kinds: kinds is NULL");
  if (!ws || wsb < KIND_SCRATCH_FLOATS * sizeof(float)) return fail(TT_ERR_CAPACITY, "tt_core_kinds: workspace");
  TT_TRY(detect_core_kinds(am, (float *)ws, (cudaStream_t)st, offdiag_ratio));
  for (int k = 0; k < am.d; ++k) kinds[k] = am.kind[k];
  return TT_OK;
}

extern "C" size_t als_workspace_structured(int32_t kind, int32_t absorb, int32_t rA, int32_t R, int32_t rB, int32_t m,
                                           int32_t n, int32_t rAp, int32_t Rp, int32_t rBp) {
  (void)kind;
  return als_ws_bytes_structured(absorb, rA, R, rB, m, n, rAp, Rp, rBp);
}

static tt_status check_structured(int32_t kind, int32_t absorb, int32_t m, int32_t n, int32_t R, int32_t Rp) {
  if (kind != TT_CORE_DENSE && kind != TT_CORE_DIAG) return fail(TT_ERR_ARG, "structured: unknown core kind");
  if (kind == TT_CORE_DIAG && m != n) return fail(TT_ERR_SHAPE, "structured: a diagonal core needs m == n");
  if (absorb && (kind != TT_CORE_DIAG)) return fail(TT_ERR_ARG, "structured: absorb needs a diagonal core");
  (void)R; (void)Rp;
  return TT_OK;
}

extern "C" tt_status als_local_apply_structured(int32_t kind, int32_t absorb, int32_t rA, int32_t R, int32_t rB,
                                                int32_t m, int32_t n, int32_t rAp, int32_t Rp, int32_t rBp,
                                                const double *Phi, const double *Ak, const double *Psi, const double *x,
                                                double *y, void *ws, size_t wsb, tt_stream st) {
  if (!dims_ok(rA, R, rB, m, n, rAp, Rp, rBp)) return fail(TT_ERR_ARG, "als_local_apply_structured: sizes must be >= 1");
  if (!Phi || !Ak || !Psi || !x || !y || !ws) return fail(TT_ERR_ARG, "als_local_apply_structured: NULL pointer");
  TT_TRY(check_structured(kind, absorb, m, n, R, Rp));
  if (wsb < als_ws_bytes_structured(absorb, rA, R, rB, m, n, rAp, Rp, rBp))
    return fail(TT_ERR_CAPACITY, "als_local_apply_structured: workspace");
  cudaStream_t s = (cudaStream_t)st;
  Arena ar;
  ar.base = (char *)ws;
  ar.cap = wsb;
  long long t1n = (long long)rB * n * rAp * Rp, t2n = (long long)R * m * rB * rAp;
  long long mx = t1n > t2n ? t1n : t2n;
  double *T1 = ar.take<double>(mx);
  double *T2 = ar.take<double>(mx);
  GemmDesc *dev = ar.take<GemmDesc>(4);
  set_gemm_scratch(ar.take<double>(GEMM_SPLIT_SCRATCH / 8), GEMM_SPLIT_SCRATCH);
  ScratchScope scratch_scope;
  GemmDesc g[4];
  if (!absorb) {
    descs_local_apply_k(kind, rA, R, rB, m, n, rAp, Rp, rBp, Phi, Ak, Psi, x, y, T1, T2, g);
    return run_descs(g, 3, dev, s);
  }
  double *Pt = ar.take<double>((size_t)rA * rB * Rp * m);
  double *Dc = ar.take<double>((size_t)R * Rp * m);
  diag_extract_raw_kernel<<<64, 256, 0, s>>>(Ak, R, Rp, m, Dc);
  TT_TRY(check_launch("diag_extract"));
  desc_pt_precompute(rA, R, rB, m, Rp, Phi, Dc, Pt, g);
  TT_TRY(run_descs(g, 1, dev, s));
  descs_local_apply_pt(rA, rB, m, rAp, Rp, rBp, Pt, Psi, x, y, T1, g);
  return run_descs(g, 3, dev + 1, s);
}

extern "C" tt_status als_update_interfaces_structured(int32_t kind, int32_t absorb, int32_t dir, int32_t rY, int32_t R,
                                                      int32_t rX, int32_t m, int32_t n, int32_t rYp, int32_t Rp,
                                                      int32_t rXp, const double *Iprev, const double *Yk,
                                                      const double *Ak, const double *Xk, double *Inext, void *ws,
                                                      size_t wsb, tt_stream st) {
  if (!dims_ok(rY, R, rX, m, n, rYp, Rp, rXp)) return fail(TT_ERR_ARG, "als_update_interfaces_structured: sizes");
  if (!Iprev || !Yk || !Ak || !Xk || !Inext || !ws) return fail(TT_ERR_ARG, "als_update_interfaces_structured: NULL");
  if (dir != 1 && dir != -1) return fail(TT_ERR_ARG, "als_update_interfaces_structured: dir must be +1 or -1");
  TT_TRY(check_structured(kind, absorb, m, n, R, Rp));
  if (absorb && dir != 1) return fail(TT_ERR_ARG, "als_update_interfaces_structured: absorb is a left (+1) form");
  if (wsb < als_ws_bytes_structured(absorb, rY, R, rX, m, n, rYp, Rp, rXp))
    return fail(TT_ERR_CAPACITY, "als_update_interfaces_structured: workspace");
  cudaStream_t s = (cudaStream_t)st;
  Arena ar;
  ar.base = (char *)ws;
  ar.cap = wsb;
  long long t1n = (long long)rX * n * rYp * Rp, t2n = (long long)R * m * rX * rYp;
  long long mx = t1n > t2n ? t1n : t2n;
  double *T1 = ar.take<double>(mx);
  double *T2 = ar.take<double>(mx);
  GemmDesc *dev = ar.take<GemmDesc>(4);
  set_gemm_scratch(ar.take<double>(GEMM_SPLIT_SCRATCH / 8), GEMM_SPLIT_SCRATCH);
  ScratchScope scratch_scope;
  GemmDesc g[4];
  if (!absorb) {
    if (dir > 0) descs_iface_left_k(kind, rY, R, rX, m, n, rYp, Rp, rXp, Iprev, Yk, Ak, Xk, Inext, T1, T2, g);
    else descs_iface_right_k(kind, rY, R, rX, m, n, rYp, Rp, rXp, Iprev, Yk, Ak, Xk, Inext, T1, T2, g);
    return run_descs(g, 3, dev, s);
  }
  double *Pt = ar.take<double>((size_t)rY * rX * Rp * m);
  double *Dc = ar.take<double>((size_t)R * Rp * m);
  diag_extract_raw_kernel<<<64, 256, 0, s>>>(Ak, R, Rp, m, Dc);
  TT_TRY(check_launch("diag_extract"));
  desc_pt_precompute(rY, R, rX, m, Rp, Iprev, Dc, Pt, g);
  TT_TRY(run_descs(g, 1, dev, s));
  descs_iface_left_pt(rY, rX, m, rYp, Rp, rXp, Pt, Yk, Xk, Inext, T1, g);
  return run_descs(g, 3, dev + 1, s);
}
