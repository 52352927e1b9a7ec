// Device-resident restarted GMRES(m) for the AMEn local systems.
// The whole restarted solve runs in ONE persistent launch of the fused
// Arnoldi-step kernel (gemm.cu gm_chunk_kernel): local-apply DMMA GEMM stages,
// classical Gram-Schmidt with the DGKS re-orthogonalisation test, Givens
// rotations, the triangular solve and the x update, all on the device; the
// convergence flag stays in device memory.  The vector length N follows the
// device-resident TT ranks.  (The round-1 per-operation and per-cycle paths
// were measured slower and removed.)
#include <cstdlib>

#include "gmres.h"

namespace tt {

namespace {

__global__ void gm_init_kernel(GmState *st, const int *Nptr, int m, double tol, int dense_max) {
  st->N = *Nptr;
  st->m = m;
  st->tol = tol;
  // N <= dense_max: the dense local solver takes this system, the fused GMRES
  // launches return at once
  const int skip = st->N <= dense_max ? 1 : 0;
  st->converged = skip;
  st->stop = skip;
  st->cycle = 0;
  st->nan = 0;
  st->jdone = 0;
}

}  // namespace

tt_status gmres_solve(const GmresCtx &c, cudaStream_t s) {
  gm_init_kernel<<<1, 1, 0, s>>>(c.st, c.Nptr, c.m, c.tol, c.dense_max);
  TT_TRY(check_launch("gm_init"));
  if (!(c.gapp && c.part && c.bar && gmres_fused_grid() > 0))
    return fail(TT_ERR_CUDA, "gmres: the fused solve kernel is unavailable (not co-resident)");
  cudaMemsetAsync(c.bar, 0, GM_BAR_WORDS * sizeof(unsigned int), s);
  const int decide = c.cluster == 2;
  if (c.cluster != 0)
    TT_TRY(launch_gmres_chunk(c.st, c.gapp, c.V, c.ldv, c.w, c.part, c.split, c.split_elems, c.bar, 0, c.m, s, 1,
                              decide, 1, c.max_restarts, c.b, c.x));
  if (c.cluster != 1)
    TT_TRY(launch_gmres_chunk(c.st, c.gapp, c.V, c.ldv, c.w, c.part, c.split, c.split_elems, c.bar, 0, c.m, s, 0,
                              decide, 1, c.max_restarts, c.b, c.x));
  return check_launch("gmres (persistent)");
}

}  // namespace tt
