// extern "C" entry points of libtt (include/tt.h): argument checks, meta
// marshalling, workspace planning.  All compute is in the kernels.
#include <cstring>
#include <string>
#include <vector>

#include "tt_common.cuh"

using namespace tt;

extern "C" const char *tt_version(void) { return "libtt-b200 0.1 (sm_100a, fp64 DMMA)"; }

// tt_last_error is defined next to the error state.
namespace tt {
const char *last_error_cstr();
}
extern "C" const char *tt_last_error(void) { return tt::last_error_cstr(); }

extern "C" tt_status tt_matvec(const tt_mat *A, const tt_vec *x, tt_vec *y, tt_stream s) {
  MatMeta a;
  VecMeta xm, ym;
  TT_TRY(make_mat_meta(A, a));
  TT_TRY(make_vec_meta(x, xm));
  TT_TRY(make_vec_meta(y, ym));
  return matvec_meta(a, xm, ym, (cudaStream_t)s);
}

namespace tt {
size_t matvec_batched_ws(int B, int d);
tt_status matvec_batched_meta(int B, const MatMeta *A, const VecMeta *x, const VecMeta *y, void *ws, size_t wsb,
                              cudaStream_t s);
}

extern "C" size_t tt_matvec_batched_workspace(int32_t B, const tt_mat *A) {
  if (B <= 0 || !A) return 0;
  return matvec_batched_ws(B, A->d);
}

extern "C" tt_status tt_matvec_batched(int32_t B, const tt_mat *A, const tt_vec *x, tt_vec *y, void *ws, size_t wsb,
                                       tt_stream s) {
  if (B < 0 || (B > 0 && (!A || !x || !y))) return fail(TT_ERR_ARG, "tt_matvec_batched: bad batch");
  if (B == 0) return TT_OK;
  std::vector<MatMeta> am(B);
  std::vector<VecMeta> xm(B), ym(B);
  for (int b = 0; b < B; ++b) {
    TT_TRY(make_mat_meta(A + b, am[b]));
    TT_TRY(make_vec_meta(x + b, xm[b]));
    TT_TRY(make_vec_meta(y + b, ym[b]));
  }
  return matvec_batched_meta(B, am.data(), xm.data(), ym.data(), ws, wsb, (cudaStream_t)s);
}

extern "C" tt_status tt_add(const tt_vec *x, const double *alpha_dev, const tt_vec *y, const double *beta_dev,
                            tt_vec *z, tt_stream s) {
  VecMeta xm, ym, zm;
  TT_TRY(make_vec_meta(x, xm));
  TT_TRY(make_vec_meta(y, ym));
  TT_TRY(make_vec_meta(z, zm));
  return add_meta(xm, alpha_dev, ym, beta_dev, zm, (cudaStream_t)s);
}

extern "C" tt_status tt_scale(tt_vec *x, const double *alpha_dev, tt_stream s) {
  VecMeta xm;
  TT_TRY(make_vec_meta(x, xm));
  if (!alpha_dev) return fail(TT_ERR_ARG, "tt_scale: alpha_dev is NULL");
  return scale_meta(xm, alpha_dev, 1.0, 0, (cudaStream_t)s);
}

extern "C" tt_status tt_copy(const tt_vec *x, tt_vec *y, tt_stream s) {
  VecMeta xm, ym;
  TT_TRY(make_vec_meta(x, xm));
  TT_TRY(make_vec_meta(y, ym));
  return copy_meta(xm, ym, (cudaStream_t)s);
}

extern "C" size_t tt_dot_workspace(const tt_vec *x, const tt_vec *y) {
  VecMeta xm, ym;
  if (make_vec_meta(x, xm) != TT_OK || make_vec_meta(y, ym) != TT_OK) return 0;
  Arena ar;
  if (dot_meta(xm, ym, nullptr, ar, nullptr) != TT_OK) return 0;
  return ar.used;
}

extern "C" tt_status tt_dot(const tt_vec *x, const tt_vec *y, double *out_dev, void *ws, size_t wsb, tt_stream s) {
  VecMeta xm, ym;
  TT_TRY(make_vec_meta(x, xm));
  TT_TRY(make_vec_meta(y, ym));
  if (!out_dev || !ws) return fail(TT_ERR_ARG, "tt_dot: NULL pointer");
  Arena ar;
  ar.base = (char *)ws;
  ar.cap = wsb;
  return dot_meta(xm, ym, out_dev, ar, (cudaStream_t)s);
}

extern "C" size_t tt_orthogonalize_workspace(const tt_vec *x) {
  VecMeta xm;
  if (make_vec_meta(x, xm) != TT_OK) return 0;
  Arena ar;
  orth_meta(xm, -1, nullptr, ar, nullptr);
  return ar.used;
}

extern "C" tt_status tt_orthogonalize(tt_vec *x, int32_t dir, double *norm_dev, void *ws, size_t wsb,
                                      tt_stream s) {
  VecMeta xm;
  TT_TRY(make_vec_meta(x, xm));
  if (dir != 1 && dir != -1) return fail(TT_ERR_ARG, "tt_orthogonalize: dir must be +1 or -1");
  if (!ws) return fail(TT_ERR_ARG, "tt_orthogonalize: NULL workspace");
  Arena ar;
  ar.base = (char *)ws;
  ar.cap = wsb;
  return orth_meta(xm, dir, norm_dev, ar, (cudaStream_t)s);
}

extern "C" tt_status tt_normalize(tt_vec *x, double *norm_dev, void *ws, size_t wsb, tt_stream s) {
  VecMeta xm;
  TT_TRY(make_vec_meta(x, xm));
  if (!ws || !norm_dev) return fail(TT_ERR_ARG, "tt_normalize: NULL workspace or norm");
  Arena ar;
  ar.base = (char *)ws;
  ar.cap = wsb;
  TT_TRY(orth_meta(xm, -1, norm_dev, ar, (cudaStream_t)s));
  return scale_meta(xm, norm_dev, 1.0, 1, (cudaStream_t)s);
}

extern "C" size_t tt_round_workspace(const tt_vec *x) {
  VecMeta xm;
  if (make_vec_meta(x, xm) != TT_OK) return 0;
  Arena ar;
  round_meta(xm, 0.0, 1, nullptr, nullptr, 0, ar, nullptr);
  return ar.used;
}

extern "C" tt_status tt_round(tt_vec *x, double eps, int32_t rmax, double *discarded_sq_dev, double *sv_dev,
                              int32_t sv_stride, void *ws, size_t wsb, tt_stream s) {
  VecMeta xm;
  TT_TRY(make_vec_meta(x, xm));
  if (!ws) return fail(TT_ERR_ARG, "tt_round: NULL workspace");
  if (sv_dev && sv_stride < 1) return fail(TT_ERR_ARG, "tt_round: sv_stride must be >= 1");
  Arena ar;
  ar.base = (char *)ws;
  ar.cap = wsb;
  return round_meta(xm, eps, rmax, discarded_sq_dev, sv_dev, sv_stride, ar, (cudaStream_t)s);
}

extern "C" size_t tt_round_batched_workspace(int32_t B, const tt_vec *x) {
  if (B < 1 || !x) return 0;
  std::vector<VecMeta> xm(B);
  for (int b = 0; b < B; ++b)
    if (make_vec_meta(x + b, xm[b]) != TT_OK) return 0;
  Arena ar;
  if (round_batched_meta(B, xm.data(), 0.0, 1, nullptr, 0, ar, nullptr) != TT_OK) return 0;
  return ar.used;
}

extern "C" tt_status tt_round_batched(int32_t B, tt_vec *x, double eps, int32_t rmax, double *discarded_sq_dev,
                                      void *ws, size_t wsb, tt_stream s) {
  if (B < 1 || !x) return fail(TT_ERR_ARG, "tt_round_batched: B >= 1 instances required");
  if (!ws) return fail(TT_ERR_ARG, "tt_round_batched: NULL workspace");
  std::vector<VecMeta> xm(B);
  for (int b = 0; b < B; ++b) TT_TRY(make_vec_meta(x + b, xm[b]));
  Arena ar;
  ar.base = (char *)ws;
  ar.cap = wsb;
  return round_batched_meta(B, xm.data(), eps, rmax, discarded_sq_dev, xm[0].d - 1, ar, (cudaStream_t)s);
}

namespace tt {
void gemm_counters(unsigned long long *out, int reset);
void matvec_counters(unsigned long long *out, int reset);
void linalg_counters(unsigned long long *out, int reset);
}

namespace tt {
void fused_profile(int enable);
void fused_profile_read(long long *launches, double *ms, double *flops);
void fused_profile_cores(double *ms, double *steps, long long *launches);
void fused_timer_read(double *ms, long long *launches);
}

extern "C" void tt_fused_timer_read(double *ms, int64_t *launches) {
  long long l = 0;
  tt::fused_timer_read(ms, &l);
  if (launches) *launches = l;
}

extern "C" void tt_fused_profile(int32_t enable) { tt::fused_profile(enable); }

extern "C" void tt_set_graph_mode(int32_t mode) { tt::set_graph_mode(mode); }
extern "C" int32_t tt_graph_mode(void) { return tt::graph_mode(); }
extern "C" void tt_graph_stats(int64_t *captures, int64_t *replays, int64_t *cached) {
  long long c = 0, r = 0, n = 0;
  tt::graph_stats(&c, &r, &n);
  if (captures) *captures = c;
  if (replays) *replays = r;
  if (cached) *cached = n;
}

extern "C" void tt_fused_profile_cores(double *ms, double *steps, int64_t *launches) {
  long long l[TT_MAX_D];
  tt::fused_profile_cores(ms, steps, l);
  for (int t = 0; t < TT_MAX_D; ++t) launches[t] = l[t];
}

extern "C" void tt_fused_profile_read(int64_t *launches, double *ms, double *flops) {
  long long l = 0;
  tt::fused_profile_read(&l, ms, flops);
  if (launches) *launches = l;
}

extern "C" void tt_counters(uint64_t *out, int32_t reset) {
  unsigned long long g[2] = {0, 0}, mv = 0, la[2] = {0, 0};
  cudaDeviceSynchronize();
  tt::gemm_counters(g, reset);
  tt::matvec_counters(&mv, reset);
  tt::linalg_counters(la, reset);
  if (out) {
    out[0] = g[0];
    out[1] = mv;
    out[2] = la[0];
    out[3] = la[1];
    out[4] = g[1];
  }
}
