// Entry points whose device path is not built yet: they fail loudly (no CPU fallback).
#include "tt_common.cuh"
using namespace tt;
extern "C" size_t amen_workspace(const tt_mat *, const tt_vec *, const tt_vec *, const tt_vec *, const amen_opts *) {
  return 0;
}
extern "C" tt_status amen_solve(const tt_mat *, const tt_vec *, tt_vec *, tt_vec *, const amen_opts *, int32_t *,
                                double *, void *, size_t, tt_stream) {
  return fail(TT_ERR_NOT_IMPLEMENTED, "amen_solve: not implemented");
}
extern "C" size_t keff_workspace(const tt_mat *, const tt_mat *, const tt_mat *, const tt_vec *, const tt_vec *,
                                 const keff_opts *) {
  return 0;
}
extern "C" tt_status keff_fixed_point(const tt_mat *, const tt_mat *, const tt_mat *, tt_vec *, tt_vec *, double,
                                      const keff_opts *, keff_report *, void *, size_t, tt_stream) {
  return fail(TT_ERR_NOT_IMPLEMENTED, "keff_fixed_point: not implemented");
}
extern "C" int32_t tt_transport_terms(int32_t, int32_t, double, int32_t, int32_t, const double *, const double *,
                                      const double *, const double *, int32_t, const double *, const double *,
                                      const double *, const double *, int32_t, const int32_t *, const int32_t *,
                                      const int32_t *, double *) {
  set_error("tt_transport_terms: not implemented");
  return -1;
}
