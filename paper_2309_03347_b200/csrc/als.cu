// als_local_apply (a6) and als_update_interfaces (a5) with host-side sizes:
// three DMMA GEMMs per call; descriptors staged into the workspace by a tiny
// by-value kernel (graph-capturable, no host->device memcpy).
#include "als.h"

namespace tt {

namespace {
struct Desc3 {
  GemmDesc g[3];
};
__global__ void set_descs_kernel(Desc3 in, GemmDesc *out, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) out[i] = in.g[i];
}

long long prod(long long a, long long b, long long c, long long d) { return a * b * c * d; }
}  // namespace

static tt_status run3(const Desc3 &d, int count, GemmDesc *dev, const int *Mc, const int *Nc, cudaStream_t s) {
  set_descs_kernel<<<1, 32, 0, s>>>(d, dev, count);
  TT_TRY(check_launch("set_descs"));
  for (int i = 0; i < count; ++i) TT_TRY(launch_gemm_k(dev + i, 1, Mc[i], Nc[i], d.g[i].K, s));
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
  b += ((3 * sizeof(GemmDesc)) + 255) & ~size_t(255);
  b += GEMM_SPLIT_SCRATCH;
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
