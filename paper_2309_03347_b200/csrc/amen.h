// AMEn linear solve on the device (amen.cu), shared by the ABI and keff.
#pragma once
#include "tt_common.cuh"

namespace tt {
struct AmenOpts {
  double eps, local_tol;
  int max_sweeps, rmax, restart, max_restarts;
  int dense_max = 0;   // local systems with N <= dense_max: dense solve (a7)
};
size_t amen_ws_bytes(const MatMeta &A, const VecMeta &b, const VecMeta &x, const VecMeta &z, int restart,
                     int dense_max = 0);
tt_status amen_solve_meta(const MatMeta &A, const VecMeta &b, const VecMeta &x, const VecMeta &z, const AmenOpts &o,
                          int *sweeps_dev, double *res_dev, int *status_dev, Arena &ar, cudaStream_t s);
size_t amen_mv_ws_bytes(const MatMeta &A, const VecMeta &b, const VecMeta &y, const VecMeta &z);
tt_status amen_mv_meta(const MatMeta &A, const VecMeta &b, const VecMeta &y, const VecMeta &z, double eps,
                       int max_sweeps, int rmax, int *sweeps_dev, Arena &ar, cudaStream_t s);
}  // namespace tt
