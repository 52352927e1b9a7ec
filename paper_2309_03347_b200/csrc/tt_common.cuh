// Internal definitions shared by the libtt translation units (sm_100a, fp64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <functional>
#include <string>

#include "tt.h"

namespace tt {

// Host-side shape of a TT-vector / TT-matrix, passed to kernels BY VALUE (it
// is captured into CUDA graphs with the launch).  Ranks stay on the device.
struct VecMeta {
  int d;
  int n[TT_MAX_D];
  int rcap[TT_MAX_D + 1];
  long long off[TT_MAX_D];
  double *data;
  int *r;  // device ranks [d+1]
};

struct MatMeta {
  int d;
  int m[TT_MAX_D];
  int n[TT_MAX_D];
  int Rcap[TT_MAX_D + 1];
  long long off[TT_MAX_D];
  double *data;
  int *R;  // device ranks [d+1]
  int kind[TT_MAX_D];  // core structure (als.h CoreKind), set by detect_core_kinds; 0 = dense
  int kinds_set;       // 1: kind[] is valid (the drivers detect once per call, before any capture)
  int pad_;            // explicit: no padding bytes (metas are part of the CUDA-graph cache keys)
};

// Device-side structure detection of the operator cores (als.h CoreKind): a
// core with m == n >= 4 whose off-diagonal entries are all <= 1e-13 max|A_k| is
// diagonal.  scratch_dev: >= 3 TT_MAX_D floats of device workspace.  Writes
// A.kind (host) after one small read-back; the off-diagonal ratio
// max|offdiag| / max|A_k| of each core goes to ratio_out (host [d], may be NULL;
// -1 for cores that are not square or smaller than 4).
constexpr double KIND_DIAG_TOL = 1e-13;
constexpr int KIND_SCRATCH_FLOATS = 3 * TT_MAX_D;
tt_status detect_core_kinds(MatMeta &A, float *scratch_dev, cudaStream_t s, double *ratio_out = nullptr);

// ---------------------------------------------------------------- errors ---
void set_error(const std::string &msg);
tt_status fail(tt_status st, const std::string &msg);
tt_status check_launch(const char *what);
// device -> host copy of a few bytes, waited for by polling an event (<= 256 bytes)
tt_status read_back(void *dst, const void *src_dev, size_t bytes, cudaStream_t s);

#define TT_TRY(expr)                    \
  do {                                  \
    tt_status _st = (expr);             \
    if (_st != TT_OK) return _st;       \
  } while (0)

// ----------------------------------------------------------- workspace ---
// Bump allocator over the caller's workspace.  With base == nullptr it only
// counts (used by the *_workspace size queries, which run the same plan).
struct Arena {
  char *base = nullptr;
  size_t cap = 0;
  size_t used = 0;
  template <class T>
  T *take(size_t count) {
    size_t bytes = ((count * sizeof(T)) + 255) & ~size_t(255);
    T *p = base ? reinterpret_cast<T *>(base + used) : nullptr;
    used += bytes;
    return p;
  }
  bool ok() const { return base == nullptr || used <= cap; }
};

// ----------------------------------------------------------------- GEMM ---
// C[M x N] = alpha op(A)[M x K] op(B)[K x N] + beta C, fp64, column-major A, B.
// C is written through a two-level scatter: row r = r0 + dr r1 (r0 < dr),
// col c = c0 + dc c1, address = r0 s_r0 + r1 s_r1 + c0 s_c0 + c1 s_c1 — this
// lets every tensor-contraction stage write its output directly in the layout
// the next stage reads as a plain matrix.  The descriptor lives in device
// memory so that sizes can follow device-resident ranks.
struct GemmDesc {
  int M, N, K;
  int transA, transB;
  long long lda, ldb;
  const double *A;
  const double *B;
  double *C;
  int dr, dc;
  long long s_r0, s_r1, s_c0, s_c1;
  double alpha, beta;
  const double *alpha_dev;  // if non-null, alpha *= *alpha_dev
  const int *skip;          // if non-null and *skip != 0 the GEMM is a no-op (GMRES steps after convergence)
  // batch of independent GEMMs of the same shape: problem b reads A + b bsA, B + b bsB and
  // writes through the scatter at C + b bsC (structured operator cores: one small GEMM per
  // mode index i of a diagonal core).  batch = 0: a plain GEMM; batch >= 1: that many
  // problems (may follow device ranks; launchers size grid z by a host capacity).
  int batch;
  long long bsA, bsB, bsC;
};

// problem b of a batched descriptor as a plain descriptor
__host__ __device__ inline GemmDesc gemm_batch_item(const GemmDesc &g, int b) {
  GemmDesc h = g;
  h.A = g.A + (long long)b * g.bsA;
  h.B = g.B + (long long)b * g.bsB;
  h.C = g.C + (long long)b * g.bsC;
  h.batch = 0;
  return h;
}
__host__ __device__ inline int gemm_nbatch(const GemmDesc &g) { return g.batch >= 1 ? g.batch : 1; }

__host__ __device__ inline void gemm_plain_c(GemmDesc &g, double *C, long long ldc) {
  g.C = C;
  g.dr = 1 << 30;
  g.s_r0 = 1;
  g.s_r1 = 0;
  g.dc = 1 << 30;
  g.s_c0 = ldc;
  g.s_c1 = 0;
}

// Launch `count` GEMMs described at descs_dev[0..count) with a grid sized for
// Mcap x Ncap (tiles beyond the device-side M, N exit immediately).
tt_status launch_gemm(const GemmDesc *descs_dev, int count, int Mcap, int Ncap, cudaStream_t s);
// With Kcap (host upper bound of K) the launcher may split K across CTAs when the
// output has few tiles, using the scratch registered by set_gemm_scratch (the
// calling thread's current workspace slice); deterministic slice-sum reduction.
// batch: 0 for plain descriptors, else the host capacity of the descriptor's batch
// count (count must then be 1).
tt_status launch_gemm_k(const GemmDesc *descs_dev, int count, int Mcap, int Ncap, int Kcap, cudaStream_t s,
                        int batch = 0);
// CUDA-graph replay of a fixed launch sequence (graph.cu): `enqueue` launches on
// `s` (taken by reference: it points at a private capture stream while recording).
// The key is the exact bytes the sequence depends on (compared in full on a hit).
uint64_t hash_bytes(const void *p, size_t n, uint64_t h = 1469598103934665603ull);
struct GraphKey {
  uint64_t h = 1469598103934665603ull;
  std::string bytes;
  void add(const void *p, size_t n);
  template <class T> void add(const T &v) { add(&v, sizeof(T)); }
};
tt_status run_captured(const GraphKey &key, cudaStream_t &s, const std::function<tt_status()> &enqueue);
// 0 no graphs, 1 replayed sequences + host-polled loops, 2 device-resident loops
int graph_mode();
void set_graph_mode(int mode);   // -1: back to the environment default
void graph_stats(long long *captures, long long *replays, long long *cached);
bool stream_capturing(cudaStream_t s);
// true when the drivers' convergence loops are to be emitted as conditional
// graph nodes (graph mode 2 and s is being captured)
bool device_loops(cudaStream_t s);
tt_status cond_handle(cudaStream_t s, cudaGraphConditionalHandle *h);
tt_status cond_node(cudaStream_t &s, cudaGraphConditionalHandle h, int is_while,
                    const std::function<tt_status()> &body);
tt_status cond_set(cudaGraphConditionalHandle h, unsigned int v, cudaStream_t s);
tt_status cond_from_flag(cudaGraphConditionalHandle h, const int *flag_dev, cudaStream_t s);   // h = (*flag == 0)
// do { body(h) } while (h): the body must end by setting h on the device
tt_status dev_while(cudaStream_t &s, const std::function<tt_status(cudaGraphConditionalHandle)> &body);
// A dependent chain of `count` GEMMs (descriptor i consumes earlier outputs) with
// per-GEMM capacity shapes, one launch each.
tt_status launch_gemm_seq(const GemmDesc *descs_dev, int count, const int *Mcap, const int *Ncap, const int *Kcap,
                          cudaStream_t s, const int *Bcap = nullptr);
void set_gemm_scratch(double *ptr, size_t bytes);
// the split-K scratch registered by a driver is a slice of ITS workspace: cleared
// when the driver returns, so no later launch writes into a released workspace
struct ScratchScope {
  ~ScratchScope() { set_gemm_scratch(nullptr, 0); }
};
constexpr size_t GEMM_SPLIT_SCRATCH = 32ull << 20;  // bytes reserved by callers that enable split-K

// ------------------------------------------------------------- linalg ---
// Householder QR of an m x n column-major matrix (one CTA per problem,
// blocked with panel width 32, compact-WY trailing updates, explicit Q).
struct QRDesc {
  int m, n;              // device-side sizes (written by a plan kernel)
  const double *src;     // input element (r, c) = src[r*src_rs + c*src_cs]
  long long src_rs, src_cs;
  double *A;             // workspace copy (lda >= m): R above, V below the diagonal
  long long lda;
  double *Q;             // out: explicit Q, m x min(m,n); element (r,c) at Q[r*q_rs + c*q_cs]
  long long q_rs, q_cs;
  double *R;             // out: R, min(m,n) x n, column-major (ldr); may be nullptr
  long long ldr;
  int rt;                // 1: write R^T instead (element (r, c) of R at R[c + r*ldr])
  double *tau;           // workspace >= min(m,n)
  double *T;             // workspace >= 32*32 * ceil(min(m,n)/32)
};
tt_status launch_qr(const QRDesc *descs_dev, int count, cudaStream_t s);
// One QR whose capacity shape is mcap x ncap: tall shapes (mcap >= 3 ncap and
// mcap > 600) run as a multi-CTA TSQR tree (linalg.cu) in the caller's
// workspace of qr_tall_ws_bytes(mcap, ncap) bytes (0: not tall, plain QR).
size_t qr_tall_ws_bytes(int mcap, int ncap);
tt_status launch_qr_tall(const QRDesc *desc_dev, int mcap, int ncap, void *ws, size_t wsb, cudaStream_t s);

// One-sided (Hestenes) Jacobi SVD of an m x p matrix W (m >= p), one CTA.
// Outputs sorted by decreasing sigma: U (m x p, unit columns; zero columns for
// sigma = 0), V (p x p), sigma (p).  W is read only.  work >= (m + p) p doubles
// (used only when the problem does not fit in shared memory).
struct SVDDesc {
  int m, p;
  const double *W; long long ldw;
  double *U; long long ldu;
  double *V; long long ldv;
  double *sigma;
  double *work;
  int *sweeps_out;
};
// (V == NULL in a descriptor: left singular vectors and sigma only.)
tt_status launch_jacobi(const SVDDesc *descs_dev, int count, int mcap, int pcap, cudaStream_t s);
// Grid-barrier words (>= 16 bytes of the caller's workspace) for the block
// Jacobi kernel used when p is too large for one CTA's shared memory.
void set_jacobi_sync(unsigned int *bar);

// Strided 2-D copy with device-side sizes and strides.
struct CopyDesc {
  int rows, cols;
  const double *src; long long ss_r, ss_c;
  double *dst; long long ds_r, ds_c;
};
tt_status launch_copy(const CopyDesc *descs_dev, int count, long long cap_elems, cudaStream_t s);

// ----------------------------------------------------------- TT helpers ---
tt_status make_vec_meta(const tt_vec *x, VecMeta &m);
tt_status make_mat_meta(const tt_mat *A, MatMeta &m);
VecMeta mat_as_vec(const MatMeta &A);

// Internal operations on metas (used by the drivers; the ABI wraps them).
tt_status matvec_meta(const MatMeta &A, const VecMeta &x, const VecMeta &y, cudaStream_t s);
tt_status add_meta(const VecMeta &x, const double *alpha, const VecMeta &y, const double *beta,
                   const VecMeta &z, cudaStream_t s);
tt_status scale_meta(const VecMeta &x, const double *alpha_dev, double alpha_host, int invert,
                     cudaStream_t s);
tt_status copy_meta(const VecMeta &x, const VecMeta &y, cudaStream_t s);
tt_status dot_meta(const VecMeta &x, const VecMeta &y, double *out, Arena &ar, cudaStream_t s);
tt_status orth_meta(const VecMeta &x, int dir, double *norm_dev, Arena &ar, cudaStream_t s);
tt_status round_meta(const VecMeta &x, double eps, int rmax, double *disc, double *sv, int sv_stride,
                     Arena &ar, cudaStream_t s);
tt_status round_batched_meta(int B, const VecMeta *xs, double eps, int rmax, double *disc, int dstride, Arena &ar,
                             cudaStream_t s);

int max_slot(const VecMeta &x);      // max_k rcap[k] n_k rcap[k+1]
int max_rank(const VecMeta &x);

}  // namespace tt
