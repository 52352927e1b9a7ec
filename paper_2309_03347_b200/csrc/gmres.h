// Device GMRES state and host driver context (see gmres.cu).
#pragma once
#include "tt_common.cuh"

namespace tt {

constexpr int GM_MAX_M = 128;
// grid-barrier word (+1 spare) followed by the arrival counters of the CTA groups of the
// fused kernel's two-level cross-CTA sums; zeroed by gmres_solve
constexpr int GM_GROUPS_MAX = 64;
constexpr int GM_BAR_WORDS = 2 + GM_GROUPS_MAX;

struct GmState {
  int N, m, converged, stop, cycle, nan, j, jdone;
  double tol, beta, bnorm, res, res0;
  double g[GM_MAX_M + 1];
  double cs[GM_MAX_M];
  double sn[GM_MAX_M];
  double *H;  // (m+1) x m
};

struct GmresCtx {
  GmState *st;
  const int *Nptr;       // device: local size
  int m, max_restarts;
  double tol;
  const double *b;       // rhs (device, length N)
  double *x;             // in: initial guess, out: solution
  double *w;             // scratch vector
  double *V;             // basis, (m+1) vectors of stride ldv
  long long ldv;
  // fused Arnoldi steps (gemm.cu gm_chunk_kernel): the apply GEMM descriptors of
  // basis vector j are gapp[3(j+1) .. 3(j+1)+2]; NULL = one launch per operation
  const GemmDesc *gapp = nullptr;
  double *part = nullptr;        // gmres_fused_part_doubles(grid) doubles
  unsigned int *bar = nullptr;   // [GM_BAR_WORDS] grid barrier word + group counters (zeroed by gmres_solve)
  double *split = nullptr;       // split-K scratch
  long long split_elems = 0;
  int dense_max = 0;             // local systems with N <= dense_max go to the dense solver
  int cluster = 0;               // 0: cooperative grid; 1: one thread-block cluster (small local
                                 // systems); 2: both launched, the device-resident sizes decide
};

tt_status gmres_solve(const GmresCtx &c, cudaStream_t s);

// dense local solver (dense.cu): local systems with N <= dense_max
struct DenseArgs {
  const int *Nptr;        // device: local size N
  int dense_max, k, n;    // size threshold, core index, mode size
  const int *r, *R;       // device ranks of x and of the operator
  const double *Phi, *A, *Psi;   // left interface [r0, R0, r0], core [R0, n, n, R1], right [r1, R1, r1]
  const double *rhs;
  double *x;              // in: initial guess, out: solution
  double *M, *lbuf, *part;   // [dm x (dm+1)], [2 (dm+2)], [1024 x 4]
  unsigned int *bar;
  int *mu_count;          // device counter of mu-regularised solves (Z35)
  GmState *st;            // res0 / res / converged for the sweep bookkeeping
};
tt_status launch_dense_local(const DenseArgs &a, int dense_cap, cudaStream_t s);

size_t gmres_fused_part_doubles(int G);
int gmres_fused_grid();
tt_status launch_gmres_chunk(GmState *st, const GemmDesc *gapp, double *V, long long ldv, double *w, double *part,
                             double *split, long long split_elems, unsigned int *bar, int j0, int j1, cudaStream_t s,
                             int cluster, int decide, int full = 0, int max_restarts = 1, const double *b = nullptr,
                             double *x = nullptr);
int gmres_cluster_size();
void fused_profile_tag(int tag);   // profiling tag of later fused launches (AMEn core index)

}  // namespace tt
