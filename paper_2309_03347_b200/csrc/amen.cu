// amen_solve (a7): AMEn for A x = b in TT on the device (P:1481-1486,
// P:1512-1531 "amen_solve"; reading Z20).  Alternating-direction sweeps; at
// core k:
//   rhs_k = phi^b_{k-1} b_k psi^b_{k+1};  solve (Phi_{k-1} A_k Psi_{k+1}) x_k = rhs_k
//   with device GMRES (warm start x_k); the local residual before the solve is
//   the sweep's stopping measure; SVD-truncate x_k; residual core z_k with z
//   frames on both sides; enrich x_k with the residual projected on (x frames |
//   z frames); QR; carry the rest into the neighbour; update the interface
//   families xAx, xb, zAx, zb.
// Both directions share one code path: the unfolding M is the left unfolding
// (r0 n x r1) for left-to-right and the TRANSPOSED right unfolding (n r1 x r0)
// for right-to-left, so "columns of M" are always the orthonormal side.
// Every size follows device-resident ranks: one-thread plan kernels write the
// GEMM / QR / SVD / copy descriptors; the host only enqueues launches (it polls
// the GMRES flag once per cycle and the sweep residual once per sweep).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "als.h"
#include "amen.h"
#include "gmres.h"

namespace tt {

namespace {

constexpr int NG = 48;

struct Dev {  // device-side view passed by value to the plan kernels
  VecMeta x, z, b;
  MatMeta A;
  double *AL[TT_MAX_D + 1], *AR[TT_MAX_D + 1], *BL[TT_MAX_D + 1], *BR[TT_MAX_D + 1];
  double *ZAL[TT_MAX_D + 1], *ZAR[TT_MAX_D + 1], *ZBL[TT_MAX_D + 1], *ZBR[TT_MAX_D + 1];
  double *rhs, *sol, *w, *V, *T1, *T2, *crz, *xfull, *tmp, *tmpz, *K, *xold;
  double *qA, *qQ, *qR, *tau, *qT;      // SVD-QR of M, then the enrichment QR (qA, tau, qT reused)
  double *qA2, *tau2, *qT2;             // z QR (runs in the same launch as the enrichment QR)
  double *qRe;                          // R factor of the enrichment QR
  double *U, *Vs, *S, *J, *Ue, *Ct;
  long long ldv;
  GemmDesc *gd;     // [NG]
  GemmDesc *gapp;   // [(m+1)*3] GMRES apply table
  QRDesc *qd;       // [2]
  SVDDesc *sd;      // [1]
  CopyDesc *cd;     // [8]
  int *iv;          // [16]
  double *dv;       // [8]: [0] sweep max residual, [1] eps
  int *limit;       // [d+1] per-bond truncation limit
  int m;            // GMRES restart
  const int *gskip; // GMRES stop word: apply GEMMs after convergence are no-ops
  double *Pt, *Dc;  // diagonal cores: left interface with the operator rank absorbed, compact diagonal
  float *kscr;      // core-structure detection scratch
  char *qrws;       // TSQR scratch of the tall unfoldings
  size_t qrwsb;
};

// capacity shapes of the QR problems at core k: the SVD-QR of the local solution
// (tall or transposed) and the enrichment QR of [x | z-part]
struct QCap { int m, n; };
inline QCap qcap_svd(const VecMeta &x, int k, int dir) {
  const int n = x.n[k];
  const int mm = dir > 0 ? x.rcap[k] * n : n * x.rcap[k + 1], nn = dir > 0 ? x.rcap[k + 1] : x.rcap[k];
  return {mm > nn ? mm : nn, mm < nn ? mm : nn};
}
inline QCap qcap_enrich(const VecMeta &x, int k, int dir) {
  const int n = x.n[k];
  const int mm = dir > 0 ? x.rcap[k] * n : n * x.rcap[k + 1], cols = dir > 0 ? x.rcap[k + 1] : x.rcap[k];
  return {mm, cols < mm ? cols : mm};
}
inline size_t qr_ws_amen(const VecMeta &x) {
  size_t b = 0;
  for (int k = 0; k < x.d; ++k)
    for (int dir = -1; dir <= 1; dir += 2) {
      const QCap a = qcap_svd(x, k, dir), e = qcap_enrich(x, k, dir);
      const size_t v = qr_tall_ws_bytes(a.m, a.n), u = qr_tall_ws_bytes(e.m, e.n);
      b = v > b ? v : b;
      b = u > b ? u : b;
    }
  return b;
}

// diagonal core whose left operator rank is absorbed into the left interface
// (als.h descs_local_apply_pt); decided on capacities so host and device agree
__host__ __device__ inline bool use_pt(const MatMeta &A, int k) {
  return A.kind[k] == KIND_DIAG && A.m[k] == A.n[k] && A.Rcap[k] >= A.Rcap[k + 1];
}

// Dc[g + R (g' + Rp i)] = A_k[g, i, i, g'] (device ranks)
__global__ void diag_extract_kernel(const MatMeta A, int k, double *Dc) {
  const int R0 = A.R[k], R1 = A.R[k + 1], m = A.m[k];
  const double *c = A.data + A.off[k];
  const long long tot = (long long)R0 * R1 * m;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int g = (int)(e % R0);
    const long long t = e / R0;
    const int gp = (int)(t % R1), i = (int)(t / R1);
    Dc[e] = c[g + (long long)R0 * i * (1 + m) + (long long)R0 * m * m * gp];
  }
}

__device__ GemmDesc gdd(int M, int N, int K, const double *A, long long lda, int tA, const double *B, long long ldb,
                        int tB, double *C, long long ldc) {
  GemmDesc g = gd_make(M, N, K, A, lda, tA, B, ldb, tB);
  gd_plain(g, C, ldc);
  return g;
}
__device__ CopyDesc cpy(int rows, int cols, const double *src, long long ssr, long long ssc, double *dst,
                        long long dsr, long long dsc) {
  CopyDesc c;
  c.rows = rows; c.cols = cols; c.src = src; c.ss_r = ssr; c.ss_c = ssc; c.dst = dst; c.ds_r = dsr; c.ds_c = dsc;
  return c;
}

__global__ void init_ifaces_kernel(Dev D) {
  const int d = D.x.d;
  D.AL[0][0] = 1.0; D.BL[0][0] = 1.0; D.ZAL[0][0] = 1.0; D.ZBL[0][0] = 1.0;
  D.AR[d][0] = 1.0; D.BR[d][0] = 1.0; D.ZAR[d][0] = 1.0; D.ZBR[d][0] = 1.0;
}

__global__ void set_dv_kernel(double *dv, int i, double v) { dv[i] = v; }
// device scalar store without a host round trip (a pageable host-to-device
// copy of a stack value would synchronise the stream first)
__global__ void set_i32_kernel(int *p, int v) { *p = v; }

// per-bond truncation limits min(rmax, xcap - zcap) >= 1 (room for the enrichment)
__global__ void set_limits_kernel(const VecMeta x, const VecMeta z, int rmax, int *limit) {
  for (int k = threadIdx.x; k <= x.d; k += blockDim.x) {
    int l = x.rcap[k] - z.rcap[k];
    l = l > rmax ? rmax : l;
    limit[k] = l < 1 ? 1 : l;
  }
}

// interfaces: right ones at bond k from bond k+1 and core k; left ones at bond k+1 from bond k and core k
__global__ void plan_iface(Dev D, int k, int dir) {
  const int n = D.x.n[k];
  const int r0 = D.x.r[k], r1 = D.x.r[k + 1], z0 = D.z.r[k], z1 = D.z.r[k + 1];
  const int R0 = D.A.R[k], R1 = D.A.R[k + 1], b0 = D.b.r[k], b1 = D.b.r[k + 1];
  const double *X = D.x.data + D.x.off[k], *Z = D.z.data + D.z.off[k], *Bk = D.b.data + D.b.off[k];
  const double *Ak = D.A.data + D.A.off[k];
  const int kd = D.A.kind[k];
  if (dir < 0) {
    descs_iface_right_k(kd, r0, R0, r0, n, n, r1, R1, r1, D.AR[k + 1], X, Ak, X, D.AR[k], D.T1, D.T2, D.gd + 0);
    descs_iface_right_vec(r0, b0, n, r1, b1, D.BR[k + 1], X, Bk, D.BR[k], D.T1, D.gd + 3);
    descs_iface_right_k(kd, z0, R0, r0, n, n, z1, R1, r1, D.ZAR[k + 1], Z, Ak, X, D.ZAR[k], D.T1, D.T2, D.gd + 5);
    descs_iface_right_vec(z0, b0, n, z1, b1, D.ZBR[k + 1], Z, Bk, D.ZBR[k], D.T1, D.gd + 8);
  } else {
    // (x|A|x): the Pt of this core's local solve (same AL[k] and A_k) when absorbed
    if (use_pt(D.A, k)) descs_iface_left_pt(r0, r0, n, r1, R1, r1, D.Pt, X, X, D.AL[k + 1], D.T1, D.gd + 0);
    else descs_iface_left_k(kd, r0, R0, r0, n, n, r1, R1, r1, D.AL[k], X, Ak, X, D.AL[k + 1], D.T1, D.T2, D.gd + 0);
    descs_iface_left_vec(r0, b0, n, r1, b1, D.BL[k], X, Bk, D.BL[k + 1], D.T1, D.gd + 3);
    descs_iface_left_k(kd, z0, R0, r0, n, n, z1, R1, r1, D.ZAL[k], Z, Ak, X, D.ZAL[k + 1], D.T1, D.T2, D.gd + 5);
    descs_iface_left_vec(z0, b0, n, z1, b1, D.ZBL[k], Z, Bk, D.ZBL[k + 1], D.T1, D.gd + 8);
  }
}

// local system at core k: rhs descs, GMRES apply table, copies x_k <-> sol
__global__ void plan_local(Dev D, int k) {
  const int n = D.x.n[k];
  const int r0 = D.x.r[k], r1 = D.x.r[k + 1];
  const int R0 = D.A.R[k], R1 = D.A.R[k + 1], b0 = D.b.r[k], b1 = D.b.r[k + 1];
  const double *Bk = D.b.data + D.b.off[k], *Ak = D.A.data + D.A.off[k];
  const int N = r0 * n * r1;
  D.iv[0] = N;
  descs_local_rhs(r0, b0, n, r1, b1, D.BL[k], Bk, D.BR[k + 1], D.rhs, D.T1, D.gd + 0);
  const bool pt = use_pt(D.A, k);
  if (pt) desc_pt_precompute(r0, R0, r0, n, R1, D.AL[k], D.Dc, D.Pt, D.gd + 40);
  for (int j = -1; j < D.m; ++j) {
    const double *in = (j < 0) ? D.sol : D.V + (long long)j * D.ldv;
    GemmDesc *ga = D.gapp + 3 * (j + 1);
    if (pt) descs_local_apply_pt(r0, r0, n, r1, R1, r1, D.Pt, D.AR[k + 1], in, D.w, D.T1, ga);
    else descs_local_apply_k(D.A.kind[k], r0, R0, r0, n, n, r1, R1, r1, D.AL[k], Ak, D.AR[k + 1], in, D.w, D.T1,
                             D.T2, ga);
    ga[0].skip = ga[1].skip = ga[2].skip = D.gskip;
  }
  D.cd[0] = cpy(N, 1, D.x.data + D.x.off[k], 1, N, D.sol, 1, N);
  D.cd[1] = cpy(N, 1, D.sol, 1, N, D.x.data + D.x.off[k], 1, N);
  D.cd[2] = cpy(N, 1, D.x.data + D.x.off[k], 1, N, D.xold, 1, N);
}

// relative change of the local solution (solution-change exit, reading Z20)
__global__ void track_dx_kernel(const int *Nptr, const double *sol, const double *xold, double *dv) {
  __shared__ double r1[32], r2[32];
  const int N = *Nptr;
  double a = 0.0, b = 0.0;
#pragma unroll 4
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const double sv = sol[i], d = sv - xold[i];
    a = fma(d, d, a);
    b = fma(sv, sv, b);
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) { r1[threadIdx.x >> 5] = a; r2[threadIdx.x >> 5] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ta = 0.0, tb = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { ta += r1[i]; tb += r2[i]; }
    const double dx = tb > 0.0 ? sqrt(ta / tb) : 0.0;
    if (dx > dv[2] || !(dx == dx)) dv[2] = dx;
  }
}

__global__ void track_res_kernel(const GmState *st, double *dv, int *status) {
  const double r = st->res0;
  if (r > dv[0] || !(r == r)) dv[0] = r;
  if (st->nan && status) *status = TT_ERR_NUMERIC;
}

// SVD of M (mm x nn) read from sol: dir > 0 left unfolding, dir < 0 transposed right unfolding.
__global__ void plan_svd(Dev D, int k, int dir) {
  const int n = D.x.n[k], r0 = D.x.r[k], r1 = D.x.r[k + 1];
  const int mm = dir > 0 ? r0 * n : n * r1;
  const int nn = dir > 0 ? r1 : r0;
  const long long srs = dir > 0 ? 1 : r0, scs = dir > 0 ? (long long)r0 * n : 1;  // M(row,col) in sol
  const int wide = mm < nn;
  const int p = wide ? mm : nn;
  QRDesc &q = D.qd[0];
  if (!wide) {  // QR of M
    q.m = mm; q.n = nn; q.src = D.sol; q.src_rs = srs; q.src_cs = scs;
    q.Q = D.qQ; q.q_rs = 1; q.q_cs = mm;
  } else {      // QR of M^T
    q.m = nn; q.n = mm; q.src = D.sol; q.src_rs = scs; q.src_cs = srs;
    q.Q = D.qQ; q.q_rs = 1; q.q_cs = nn;
  }
  q.A = D.qA; q.lda = q.m;
  q.R = D.qR; q.ldr = p;
  q.tau = D.tau; q.T = D.qT;
  q.rt = 1;   // Jacobi on R^T = V_R S U_R^T (fewer sweeps for decaying spectra): U, V swap
  SVDDesc &s = D.sd[0];
  s.m = p; s.p = p; s.W = D.qR; s.ldw = p; s.U = D.Vs; s.ldu = p; s.V = D.U; s.ldv = p;
  s.sigma = D.S; s.work = D.J;
#ifdef TT_DEBUG_SVD
  s.sweeps_out = D.iv + 15;
#else
  s.sweeps_out = nullptr;
#endif
  D.iv[2] = wide; D.iv[3] = p; D.iv[4] = mm; D.iv[5] = nn;
}

// Truncation (reading Z20: delta = eps ||x_k|| / sqrt(d-1), capped by the bond
// limit) and the factors of the truncated local solution:
//   Ue[:, :r] = left singular vectors of M (mm x r, ld mm)
//   Ct        = V_r Sigma_r (nn x r)   (so the carry is C = Ct^T)
//   xfull     = the truncated local solution in [r0, n, r1] layout.
__global__ void trunc_kernel(Dev D, int k, int dir) {
  __shared__ int s_r;
  const int wide = D.iv[2], p = D.iv[3], mm = D.iv[4], nn = D.iv[5];
  const int d = D.x.d, tid = threadIdx.x;
#ifdef TT_DEBUG_SVD
  if (tid == 0) printf("SVDDBG %d %d %d %d\n", mm, nn, p, D.iv[15]);
#endif
  if (tid == 0) {
    double tot = 0.0;
    for (int i = 0; i < p; ++i) tot += D.S[i] * D.S[i];
    const double delta = D.dv[1] * sqrt(tot) / sqrt((double)(d > 1 ? d - 1 : 1));
    const double d2 = delta * delta;
    double tail = 0.0;
    int r = p;
    for (int i = p - 1; i >= 1; --i) {
      const double t2 = tail + D.S[i] * D.S[i];
      if (t2 <= d2) { tail = t2; r = i; } else break;
    }
    const int lim = D.limit[dir > 0 ? k + 1 : k];
    r = r < 1 ? 1 : r;
    r = r > lim ? lim : r;
    s_r = r;
    D.iv[1] = r;
  }
  __syncthreads();
  const int r = s_r;
  // tall: L = Q U_R, R = V_R;  wide: L = V_R, R = Q U_R.  Fold Sigma into the right factor.
  double *Rfac = wide ? D.U : D.Vs;
  for (int e = tid; e < p * r; e += blockDim.x) {
    const int row = e % p, c = e / p;
    Rfac[row + (long long)c * p] *= D.S[c];
  }
  if (tid == 0) {
    if (!wide) {
      D.gd[0] = gdd(mm, r, p, D.qQ, mm, 0, D.U, p, 0, D.Ue, mm);   // Ue = Q U_R[:, :r]
      D.cd[0] = cpy(nn, r, D.Vs, 1, p, D.Ct, 1, nn);              // Ct = V_R[:, :r] S
    } else {
      D.cd[0] = cpy(mm, r, D.Vs, 1, p, D.Ue, 1, mm);              // Ue = V_R[:, :r]
      D.gd[0] = gdd(nn, r, p, D.qQ, nn, 0, D.U, p, 0, D.Ct, nn);   // Ct = Q U_R[:, :r] S
    }
    if (dir > 0) D.gd[1] = gdd(mm, nn, r, D.Ue, mm, 0, D.Ct, nn, 1, D.xfull, mm);   // [r0 n, r1] = Ue Ct^T
    else D.gd[1] = gdd(nn, mm, r, D.Ct, nn, 0, D.Ue, mm, 1, D.xfull, nn);           // [r0, n r1] = Ct Ue^T
  }
}

// QR of crz (z core) and of Ue (x core) in one launch, K = Re[:, :r] Ct^T, and
// the carry into the neighbour core (shared by amen_solve and amen_mv).
__device__ void enrich_tail(const Dev &D, int k, int dir, int n, int r, int mm, int nn, int ze, int z0, int z1,
                            GemmDesc *g) {
  QRDesc &qz = D.qd[0];
  QRDesc &qx = D.qd[1];
  double *Zk = D.z.data + D.z.off[k];
  double *Xk = D.x.data + D.x.off[k];
  int qzr;
  if (dir > 0) {
    qz.m = z0 * n; qz.n = z1; qz.src = D.crz; qz.src_rs = 1; qz.src_cs = (long long)z0 * n;
    qzr = min(z0 * n, z1);
    qz.Q = Zk; qz.q_rs = 1; qz.q_cs = (long long)z0 * n;
  } else {
    qz.m = n * z1; qz.n = z0; qz.src = D.crz; qz.src_rs = z0; qz.src_cs = 1;
    qzr = min(n * z1, z0);
    qz.Q = Zk; qz.q_rs = qzr; qz.q_cs = 1;
  }
  qz.A = D.qA2; qz.lda = qz.m; qz.R = nullptr; qz.ldr = 1; qz.tau = D.tau2; qz.T = D.qT2; qz.rt = 0;
  const int q = min(mm, r + ze);
  qx.m = mm; qx.n = r + ze; qx.src = D.Ue; qx.src_rs = 1; qx.src_cs = mm;
  qx.A = D.qA; qx.lda = mm; qx.R = D.qRe; qx.ldr = q; qx.tau = D.tau; qx.T = D.qT; qx.rt = 0;
  if (dir > 0) { qx.Q = Xk; qx.q_rs = 1; qx.q_cs = mm; }     // x_k = Q as [r0, n, q]
  else { qx.Q = Xk; qx.q_rs = q; qx.q_cs = 1; }              // x_k = Q^T as [q, n, r1]
  // ---- K = Re[:, :r] C = Re[:, :r] Ct^T  (q x nn)
  g[10] = gdd(q, nn, r, D.qRe, q, 0, D.Ct, nn, 1, D.K, q);
  // ---- neighbour update
  if (dir > 0) {
    const int n2 = D.x.n[k + 1], r2 = D.x.r[k + 2];
    double *Xn = D.x.data + D.x.off[k + 1];
    g[11] = gdd(q, n2 * r2, nn, D.K, q, 0, Xn, nn, 0, D.tmp, q);           // K x_{k+1}
    D.cd[0] = cpy(q, n2 * r2, D.tmp, 1, q, Xn, 1, q);
    // z_{k+1}: keep its first qzr rows (left rank shrinks when z0 n < z1)
    const int zn2 = D.z.n[k + 1], zz2 = D.z.r[k + 2];
    double *Zn = D.z.data + D.z.off[k + 1];
    if (qzr < z1) {
      D.cd[1] = cpy(qzr, zn2 * zz2, Zn, 1, z1, D.tmpz, 1, qzr);
      D.cd[2] = cpy(qzr, zn2 * zz2, D.tmpz, 1, qzr, Zn, 1, qzr);
    } else {
      D.cd[1] = cpy(0, 0, nullptr, 0, 0, nullptr, 0, 0);
      D.cd[2] = cpy(0, 0, nullptr, 0, 0, nullptr, 0, 0);
    }
    D.x.r[k + 1] = q;
    D.z.r[k + 1] = qzr;
  } else {
    const int rp = D.x.r[k - 1], np = D.x.n[k - 1];
    double *Xp = D.x.data + D.x.off[k - 1];
    g[11] = gdd(rp * np, q, nn, Xp, (long long)rp * np, 0, D.K, q, 1, D.tmp, (long long)rp * np);  // x_{k-1} K^T
    D.cd[0] = cpy(rp * np, q, D.tmp, 1, (long long)rp * np, Xp, 1, (long long)rp * np);
    D.cd[1] = cpy(0, 0, nullptr, 0, 0, nullptr, 0, 0);
    D.cd[2] = cpy(0, 0, nullptr, 0, 0, nullptr, 0, 0);
    D.x.r[k] = q;
    D.z.r[k] = qzr;   // z_{k-1} keeps its first qzr columns (no data movement)
  }
}

// Residual core z_k, enrichment of the solution core, neighbour update.
__global__ void plan_enrich(Dev D, int k, int dir) {
  const int d = D.x.d;
  const int n = D.x.n[k];
  const int r0 = D.x.r[k], r1 = D.x.r[k + 1], z0 = D.z.r[k], z1 = D.z.r[k + 1];
  const int R0 = D.A.R[k], R1 = D.A.R[k + 1], b0 = D.b.r[k], b1 = D.b.r[k + 1];
  const double *Bk = D.b.data + D.b.off[k], *Ak = D.A.data + D.A.off[k];
  const int r = D.iv[1], mm = D.iv[4], nn = D.iv[5];
  GemmDesc *g = D.gd;
  // ---- crz [z0, n, z1] = zb-rhs - zAx-apply(xfull)
  descs_local_rhs(z0, b0, n, z1, b1, D.ZBL[k], Bk, D.ZBR[k + 1], D.crz, D.T1, g + 0);
  const int kd = D.A.kind[k];
  descs_local_apply_k(kd, z0, R0, r0, n, n, z1, R1, r1, D.ZAL[k], Ak, D.ZAR[k + 1], D.xfull, D.crz, D.T1, D.T2, g + 2);
  g[4].alpha = -1.0; g[4].beta = 1.0;
  // ---- crs: x frames on the orthonormal side, z frames on the carry side, written as extra
  //      columns of Ue (M orientation): dir > 0: [r0, n, z1] left unfolding -> Ue[:, r:r+z1]
  //      dir < 0: [z0, n, r1] transposed right unfolding -> Ue[:, r:r+z0]
  double *Uc = D.Ue + (long long)r * mm;
  if (dir > 0) {
    descs_local_rhs(r0, b0, n, z1, b1, D.BL[k], Bk, D.ZBR[k + 1], Uc, D.T1, g + 5);
    descs_local_apply_k(kd, r0, R0, r0, n, n, z1, R1, r1, D.AL[k], Ak, D.ZAR[k + 1], D.xfull, Uc, D.T1, D.T2, g + 7);
  } else {
    descs_local_rhs(z0, b0, n, r1, b1, D.ZBL[k], Bk, D.BR[k + 1], Uc, D.T1, g + 5);
    descs_local_apply_k(kd, z0, R0, r0, n, n, r1, R1, r1, D.ZAL[k], Ak, D.AR[k + 1], D.xfull, Uc, D.T1, D.T2, g + 7);
    // output element (a, c) of the final GEMMs -> Ue[c + mm a] (transposed)
    g[6].s_r0 = mm; g[6].s_c0 = 1;
    g[9].s_r0 = mm; g[9].s_c0 = 1;
  }
  g[9].alpha = -1.0; g[9].beta = 1.0;
  const int ze = dir > 0 ? z1 : z0;  // extra columns
  enrich_tail(D, k, dir, n, r, mm, nn, ze, z0, z1, g);
  (void)d;
}

}  // namespace

static long long lmax(long long a, long long b) { return a > b ? a : b; }

namespace {
__global__ void set_gm_H(GmState *st, double *H) { st->H = H; }

// ---- device-resident sweep loops ---------------------------------
// after a sweep: count it and decide on the device whether another one runs.
// AMEn (mv = 0): stop when the max local residual dv[0] <= eps or the max
// relative solution change dv[2] <= eps (Z20); amen_mv (mv = 1): dv[2] <= eps.
__global__ void sweep_check_kernel(const double *dv, double eps, int max_sweeps, int *cnt, int mv,
                                   cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hi) {
  const bool conv = mv ? (dv[2] <= eps) : (dv[0] <= eps || dv[2] <= eps);
  const int c = *cnt + 1;
  *cnt = c;
  const unsigned int more = (!conv && c < max_sweeps) ? 1u : 0u;
  cudaGraphSetConditional(hw, more);
  cudaGraphSetConditional(hi, more);
}
// workspace-internal report of a captured solve -> the caller's pointers
__global__ void report_out_kernel(const int *sw, const double *res, const int *st, int *sweeps_dev, double *res_dev,
                                  int *status_dev) {
  if (sweeps_dev) *sweeps_dev = *sw;
  if (res_dev) *res_dev = *res;
  if (status_dev && *st != 0) *status_dev = *st;
}
// the host loop's epilogue: sweeps performed, last residual, NOCONV unless dv[0] <= eps
__global__ void sweep_post_kernel(const double *dv, double eps, const int *cnt, int *sweeps_dev, double *res_dev,
                                  int *status_dev) {
  if (sweeps_dev) *sweeps_dev = *cnt;
  if (res_dev) *res_dev = dv[0];
  if (status_dev && !(dv[0] <= eps)) *status_dev = (int)TT_ERR_NOCONV;
}
// while (more) { sweep(+1); check; if (more) { sweep(-1); check } } as a WHILE
// node with a nested IF: the directions alternate exactly as in the host loop
tt_status sweep_loop(cudaStream_t &s, const double *dv, double eps, int max_sweeps, int *cnt, int mv,
                     const std::function<tt_status(int)> &one_sweep) {
  return dev_while(s, [&](cudaGraphConditionalHandle hw) -> tt_status {
    TT_TRY(one_sweep(+1));
    cudaGraphConditionalHandle hi;
    TT_TRY(cond_handle(s, &hi));
    sweep_check_kernel<<<1, 1, 0, s>>>(dv, eps, max_sweeps, cnt, mv, hw, hi);
    TT_TRY(check_launch("sweep_check"));
    return cond_node(s, hi, 0, [&]() -> tt_status {
      TT_TRY(one_sweep(-1));
      sweep_check_kernel<<<1, 1, 0, s>>>(dv, eps, max_sweeps, cnt, mv, hw, hw);
      return check_launch("sweep_check");
    });
  });
}

// host evaluation of a descriptor chain with capacity ranks -> per-GEMM grid caps
struct CapChain {
  int M[12], N[12];
};
}  // namespace

struct AmenCtx {
  Dev D;
  int d, m;
  long long Ncap, Scap;
  int pc, zcm, nmax;
  GmState *gst;
  double *H, *h1, *h2;
  double *gpart;
  unsigned int *gbar;
  char *orth_base;
  size_t orth_cap;
  double *split;
  unsigned int *bar;
  int dcap;                      // dense local solver capacity (0: off)
  double *dM, *dl, *dpart;
  unsigned int *dbar;
  int *dmu;
};

static tt_status carve_amen(const MatMeta &A, const VecMeta &b, const VecMeta &x, const VecMeta &z, int m, Arena &ar,
                            AmenCtx &P, int dense_max = 0) {
  const int d = A.d;
  if (b.d != d || x.d != d || z.d != d) return fail(TT_ERR_SHAPE, "amen_solve: number of cores differ");
  for (int k = 0; k < d; ++k) {
    if (A.m[k] != A.n[k]) return fail(TT_ERR_SHAPE, "amen_solve: A must be square in every mode");
    if (A.n[k] != x.n[k] || A.m[k] != b.n[k] || z.n[k] != x.n[k]) return fail(TT_ERR_SHAPE, "amen_solve: shape mismatch");
  }
  if (m < 2 || m > GM_MAX_M) return fail(TT_ERR_ARG, "amen_solve: gmres_restart must be in [2, 128]");
  for (int k = 1; k < d; ++k)
    if (x.rcap[k] <= z.rcap[k])
      return fail(TT_ERR_CAPACITY, "amen_solve: x rank capacity must exceed z rank capacity (enrichment)");
  std::memset(&P, 0, sizeof(P));
  P.d = d;
  P.m = m;
  Dev &D = P.D;
  D.x = x; D.z = z; D.b = b; D.A = A;
  D.m = m;
  long long Ncap = 1, Zcap = 1, Tcap = 1, Ecap = 1, Scap = 1;
  int pc = 1, zcm = 1, nmax = 1;
  for (int k = 0; k <= d; ++k) { pc = x.rcap[k] > pc ? x.rcap[k] : pc; zcm = z.rcap[k] > zcm ? z.rcap[k] : zcm; }
  for (int k = 0; k < d; ++k) {
    const long long n = x.n[k];
    nmax = x.n[k] > nmax ? x.n[k] : nmax;
    Ncap = lmax(Ncap, (long long)x.rcap[k] * n * x.rcap[k + 1]);
    Zcap = lmax(Zcap, (long long)z.rcap[k] * n * z.rcap[k + 1]);
    long long rm = x.rcap[k];
    rm = lmax(rm, x.rcap[k + 1]); rm = lmax(rm, z.rcap[k]); rm = lmax(rm, z.rcap[k + 1]);
    rm = lmax(rm, b.rcap[k]); rm = lmax(rm, b.rcap[k + 1]);
    long long Rm = lmax(A.Rcap[k], A.Rcap[k + 1]);
    Tcap = lmax(Tcap, n * rm * rm * lmax(Rm, 1));
    Ecap = lmax(Ecap, n * lmax(x.rcap[k], x.rcap[k + 1]) * (pc + zcm));
    Scap = lmax(Scap, (long long)x.rcap[k] * n * x.rcap[k + 1]);
    Scap = lmax(Scap, (long long)z.rcap[k] * n * z.rcap[k + 1]);
  }
  P.Ncap = Ncap; P.Scap = Scap; P.pc = pc; P.zcm = zcm; P.nmax = nmax;
  // diagonal-core buffers, sized for every square core with m >= 4 (kinds are detected later)
  long long Ptcap = 1, Dccap = 1;
  for (int k = 0; k < d; ++k)
    if (A.m[k] == A.n[k] && A.m[k] >= 4) {
      Ptcap = lmax(Ptcap, (long long)A.m[k] * A.Rcap[k + 1] * x.rcap[k] * x.rcap[k]);
      Dccap = lmax(Dccap, (long long)A.m[k] * A.Rcap[k] * A.Rcap[k + 1]);
    }
  D.Pt = ar.take<double>(Ptcap);
  D.Dc = ar.take<double>(Dccap);
  D.kscr = ar.take<float>(KIND_SCRATCH_FLOATS);
  D.qrwsb = qr_ws_amen(x);
  D.qrws = ar.take<char>(D.qrwsb);
  for (int k = 0; k <= d; ++k) {
    D.AL[k] = ar.take<double>((size_t)x.rcap[k] * x.rcap[k] * A.Rcap[k]);
    D.AR[k] = ar.take<double>((size_t)x.rcap[k] * x.rcap[k] * A.Rcap[k]);
    D.BL[k] = ar.take<double>((size_t)x.rcap[k] * b.rcap[k]);
    D.BR[k] = ar.take<double>((size_t)x.rcap[k] * b.rcap[k]);
    D.ZAL[k] = ar.take<double>((size_t)z.rcap[k] * x.rcap[k] * A.Rcap[k]);
    D.ZAR[k] = ar.take<double>((size_t)z.rcap[k] * x.rcap[k] * A.Rcap[k]);
    D.ZBL[k] = ar.take<double>((size_t)z.rcap[k] * b.rcap[k]);
    D.ZBR[k] = ar.take<double>((size_t)z.rcap[k] * b.rcap[k]);
  }
  D.ldv = (Ncap + 31) / 32 * 32;
  D.rhs = ar.take<double>(Ncap);
  D.sol = ar.take<double>(Ncap);
  D.xold = ar.take<double>(Ncap);
  D.w = ar.take<double>(Ncap);
  D.V = ar.take<double>((size_t)D.ldv * (m + 1));
  D.T1 = ar.take<double>(Tcap);
  D.T2 = ar.take<double>(Tcap);
  D.crz = ar.take<double>(Zcap);
  D.xfull = ar.take<double>(Ncap);
  D.tmp = ar.take<double>(Scap);
  D.tmpz = ar.take<double>(Zcap);
  D.K = ar.take<double>(Ecap);
  D.qA = ar.take<double>(lmax(Ncap, Ecap));
  D.qQ = ar.take<double>(Ncap);
  D.qR = ar.take<double>((size_t)pc * pc);
  D.tau = ar.take<double>(pc + zcm);
  D.qT = ar.take<double>(32 * 32 * ((pc + zcm) / 32 + 2));
  D.qA2 = ar.take<double>(Zcap);
  D.tau2 = ar.take<double>(zcm + 1);
  D.qT2 = ar.take<double>(32 * 32 * (zcm / 32 + 2));
  D.qRe = ar.take<double>((size_t)(pc + zcm) * (pc + zcm));
  D.U = ar.take<double>((size_t)pc * pc);
  D.Vs = ar.take<double>((size_t)pc * pc);
  D.S = ar.take<double>(pc);
  D.J = ar.take<double>((size_t)2 * pc * pc);
  D.Ue = ar.take<double>(Ecap);
  D.Ct = ar.take<double>(Ncap);
  D.gd = ar.take<GemmDesc>(NG);
  D.gapp = ar.take<GemmDesc>((size_t)3 * (m + 1));
  D.qd = ar.take<QRDesc>(2);
  D.sd = ar.take<SVDDesc>(1);
  D.cd = ar.take<CopyDesc>(8);
  D.iv = ar.take<int>(16);
  D.dv = ar.take<double>(8);
  D.limit = ar.take<int>(TT_MAX_D + 1);
  P.gst = ar.take<GmState>(1);
  D.gskip = P.gst ? &P.gst->stop : nullptr;
  P.H = ar.take<double>((size_t)(m + 1) * m);
  P.h1 = ar.take<double>(m + 1);
  P.h2 = ar.take<double>(m + 1);
  P.gpart = ar.take<double>(gmres_fused_part_doubles(1024));
  P.gbar = ar.take<unsigned int>(GM_BAR_WORDS + 2);
  // orthogonalisation scratch (x or z)
  Arena c1, c2;
  orth_meta(x, -1, nullptr, c1, nullptr);
  orth_meta(z, -1, nullptr, c2, nullptr);
  P.orth_cap = c1.used > c2.used ? c1.used : c2.used;
  P.orth_base = ar.take<char>(P.orth_cap);
  P.split = ar.take<double>(GEMM_SPLIT_SCRATCH / 8);
  P.bar = ar.take<unsigned int>(4);
  if (dense_max < 0) return fail(TT_ERR_ARG, "amen_solve: local_dense_max must be >= 0");
  P.dcap = (int)(dense_max < Ncap ? dense_max : Ncap);
  if (P.dcap > 0) {
    P.dM = ar.take<double>((size_t)P.dcap * (P.dcap + 1));
    P.dl = ar.take<double>((size_t)2 * (P.dcap + 2));
    P.dpart = ar.take<double>((size_t)4 * 1024);
    P.dbar = ar.take<unsigned int>(4);
    P.dmu = ar.take<int>(4);
  }
  return TT_OK;
}

size_t amen_ws_bytes(const MatMeta &A, const VecMeta &b, const VecMeta &x, const VecMeta &z, int restart,
                     int dense_max) {
  Arena ar;
  AmenCtx P;
  if (carve_amen(A, b, x, z, restart, ar, P, dense_max) != TT_OK) return 0;
  return ar.used;
}


tt_status amen_solve_meta(const MatMeta &A, const VecMeta &b, const VecMeta &x, const VecMeta &z, const AmenOpts &o,
                          int *sweeps_dev, double *res_dev, int *status_dev, Arena &ar, cudaStream_t s) {
  AmenCtx P;
  const Arena ar0 = ar;
  TT_TRY(carve_amen(A, b, x, z, o.restart, ar, P, o.dense_max));
  if (!ar.base) return TT_OK;
  if (!ar.ok()) return fail(TT_ERR_CAPACITY, "amen_solve: workspace too small");
  if (!(o.eps > 0.0)) return fail(TT_ERR_ARG, "amen_solve: eps must be > 0");
  Dev &D = P.D;
  const int d = P.d, m = P.m;
  const int pc = P.pc, zcm = P.zcm, nmax = P.nmax;
  if (!D.A.kinds_set) TT_TRY(detect_core_kinds(D.A, D.kscr, s));   // one read-back, before any capture
  if (graph_mode() >= 2 && !stream_capturing(s)) {
    // the whole solve as one graph: sweep loop on the device (K11); replayed while
    // the operands, workspace and options are the same
    gmres_fused_grid();   // one-time attribute / occupancy queries outside the capture
    GraphKey key;
    key.add(D);
    const double dd[2] = {o.eps, o.local_tol};
    const int ii[5] = {o.max_sweeps, o.rmax, o.restart, o.max_restarts, o.dense_max};
    key.add(dd);
    key.add(ii);
    const MatMeta Ak = D.A;
    // the graph reports into the workspace (iv[13] sweeps, dv[6] residual, iv[12]
    // status) so it does not depend on the caller's pointers; copied out below
    TT_TRY(run_captured(key, s, [&]() -> tt_status {
      set_i32_kernel<<<1, 1, 0, s>>>(D.iv + 12, 0);
      Arena a = ar0;
      return amen_solve_meta(Ak, b, x, z, o, D.iv + 13, D.dv + 6, D.iv + 12, a, s);
    }));
    report_out_kernel<<<1, 1, 0, s>>>(D.iv + 13, D.dv + 6, D.iv + 12, sweeps_dev, res_dev, status_dev);
    return check_launch("amen_solve report");
  }
  ScratchScope scratch_scope;
  const MatMeta &Ah = D.A;   // host copy with the detected kinds
  // per-bond truncation limits: min(rmax, xcap - zcap) (room for the enrichment)
  set_limits_kernel<<<1, 64, 0, s>>>(x, z, o.rmax, D.limit);   // no host round trip
  set_gm_H<<<1, 1, 0, s>>>(P.gst, P.H);
  set_dv_kernel<<<1, 1, 0, s>>>(D.dv, 1, o.eps);
  if (P.dcap > 0) cudaMemsetAsync(P.dmu, 0, sizeof(int), s);
  set_gemm_scratch(P.split, GEMM_SPLIT_SCRATCH);
  set_jacobi_sync(P.bar);
  Arena oa;
  oa.base = P.orth_base;
  oa.cap = P.orth_cap;
  TT_TRY(orth_meta(x, -1, nullptr, oa, s));
  oa.used = 0;
  TT_TRY(orth_meta(z, -1, nullptr, oa, s));
  init_ifaces_kernel<<<1, 1, 0, s>>>(D);
  // per-GEMM grid caps: the same descriptor builders evaluated on the host with capacity ranks
  const int *xc = x.rcap, *zc = z.rcap, *bc = b.rcap, *Rc = A.Rcap;
  struct Caps12 { GemmDesc g[12]; int cnt; };
  auto launch_caps = [&](const GemmDesc *dev, const Caps12 &hc, int from, int cnt) -> tt_status {
    int Mc[12], Nc[12], Kc[12], Bc[12];
    for (int i = 0; i < cnt; ++i) {
      Mc[i] = hc.g[from + i].M; Nc[i] = hc.g[from + i].N; Kc[i] = hc.g[from + i].K; Bc[i] = hc.g[from + i].batch;
    }
    return launch_gemm_seq(dev, cnt, Mc, Nc, Kc, s, Bc);
  };
  auto iface_caps = [&](int k, int dir) {
    Caps12 c;
    const int n = x.n[k];
    const int kd = Ah.kind[k];
    if (dir < 0) {
      descs_iface_right_k(kd, xc[k], Rc[k], xc[k], n, n, xc[k + 1], Rc[k + 1], xc[k + 1], 0, 0, 0, 0, 0, 0, 0, c.g + 0);
      descs_iface_right_vec(xc[k], bc[k], n, xc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, c.g + 3);
      descs_iface_right_k(kd, zc[k], Rc[k], xc[k], n, n, zc[k + 1], Rc[k + 1], xc[k + 1], 0, 0, 0, 0, 0, 0, 0, c.g + 5);
      descs_iface_right_vec(zc[k], bc[k], n, zc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, c.g + 8);
    } else {
      if (use_pt(Ah, k)) descs_iface_left_pt(xc[k], xc[k], n, xc[k + 1], Rc[k + 1], xc[k + 1], 0, 0, 0, 0, 0, c.g + 0);
      else descs_iface_left_k(kd, xc[k], Rc[k], xc[k], n, n, xc[k + 1], Rc[k + 1], xc[k + 1], 0, 0, 0, 0, 0, 0, 0,
                              c.g + 0);
      descs_iface_left_vec(xc[k], bc[k], n, xc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, c.g + 3);
      descs_iface_left_k(kd, zc[k], Rc[k], xc[k], n, n, zc[k + 1], Rc[k + 1], xc[k + 1], 0, 0, 0, 0, 0, 0, 0, c.g + 5);
      descs_iface_left_vec(zc[k], bc[k], n, zc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, c.g + 8);
    }
    return c;
  };
  auto iface = [&](int k, int dir) -> tt_status {
    plan_iface<<<1, 1, 0, s>>>(D, k, dir);
    Caps12 c = iface_caps(k, dir);
    return launch_caps(D.gd, c, 0, 10);
  };
  for (int k = d - 1; k >= 1; --k) TT_TRY(iface(k, -1));
  const double ltol = o.local_tol > 0.0 ? o.local_tol : 0.1 * o.eps;
  Caps12 appc;
  GmresCtx gc;
  gc.st = P.gst;
  gc.Nptr = D.iv;
  gc.m = m;
  gc.max_restarts = o.max_restarts;
  gc.tol = ltol;
  gc.b = D.rhs;
  gc.x = D.sol;
  gc.w = D.w;
  gc.V = D.V;
  gc.ldv = D.ldv;
  gc.gapp = D.gapp;
  gc.part = P.gpart;
  gc.bar = P.gbar;
  gc.split = P.split;
  gc.split_elems = GEMM_SPLIT_SCRATCH / 8 - 4096;
  gc.dense_max = P.dcap;
  const bool cluster_off = std::getenv("TT_GMRES_NOCLUSTER") != nullptr;
  GraphKey base;   // D is fixed for the whole solve
  base.add(D);
  {
    const long long extra[6] = {P.Ncap, P.Scap, pc, (long long)(size_t)status_dev, P.dcap, 0x616d};
    base.add(extra);
  }
  // one sweep in direction dir: a fixed launch sequence whose sizes follow the device ranks
  auto one_sweep = [&](int dir) -> tt_status {
    set_dv_kernel<<<1, 1, 0, s>>>(D.dv, 0, 0.0);
    set_dv_kernel<<<1, 1, 0, s>>>(D.dv, 2, 0.0);
    for (int t = 0; t < d; ++t) {
      const int k = dir > 0 ? t : d - 1 - t;
      const int last = (t == d - 1);
      const int n = x.n[k];
      const bool pt = use_pt(Ah, k);
      descs_local_rhs(xc[k], bc[k], n, xc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, appc.g + 0);
      if (pt) descs_local_apply_pt(xc[k], xc[k], n, xc[k + 1], Rc[k + 1], xc[k + 1], 0, 0, 0, 0, 0, appc.g + 2);
      else descs_local_apply_k(Ah.kind[k], xc[k], Rc[k], xc[k], n, n, xc[k + 1], Rc[k + 1], xc[k + 1], 0, 0, 0, 0, 0,
                               0, 0, appc.g + 2);
      {  // small local systems: fused Arnoldi steps inside one thread-block cluster
        int tiles = 0;
        for (int q = 2; q < 5; ++q) {
          const int t = ((appc.g[q].M + 63) / 64) * ((appc.g[q].N + 63) / 64) * gemm_nbatch(appc.g[q]);
          tiles = t > tiles ? t : tiles;
        }
        const long long nloc = (long long)xc[k] * n * xc[k + 1];
        // at capacity sizes the cluster certainly applies: launch it alone; otherwise launch
        // both variants and let the device-resident sizes pick one (the other exits at once)
        gc.cluster = cluster_off ? 0 : ((tiles <= 2 * gmres_cluster_size() && nloc <= 16384) ? 1 : 2);
      }
      // fixed launch sequences before and after the GMRES solve: CUDA-graph replays
      // (recorded inline when the whole solve is being captured)
      GraphKey key1 = base, key2;
      {
        const int extra[3] = {k, dir, last};
        key1.add(extra);
        key2 = key1;
        key1.add(1);
        key2.add(2);
      }
      TT_TRY(run_captured(key1, s, [&]() -> tt_status {
        plan_local<<<1, 1, 0, s>>>(D, k);
        TT_TRY(launch_copy(D.cd, 1, P.Ncap, s));
        TT_TRY(launch_copy(D.cd + 2, 1, P.Ncap, s));
        if (pt) {   // Pt_i = Phi_{k-1} x_2 D_i, once per local system
          diag_extract_kernel<<<64, 256, 0, s>>>(D.A, k, D.Dc);
          TT_TRY(launch_gemm_k(D.gd + 40, 1, xc[k], Rc[k + 1] * n, Rc[k], s, xc[k]));
        }
        return launch_caps(D.gd, appc, 0, 2);
      }));
      fused_profile_tag(k);
      TT_TRY(gmres_solve(gc, s));
      if (P.dcap > 0) {   // N <= local_dense_max: dense solve (the GMRES launches above returned at once)
        DenseArgs da;
        da.Nptr = D.iv; da.dense_max = P.dcap; da.k = k; da.n = n;
        da.r = D.x.r; da.R = D.A.R;
        da.Phi = D.AL[k]; da.A = D.A.data + D.A.off[k]; da.Psi = D.AR[k + 1];
        da.rhs = D.rhs; da.x = D.sol;
        da.M = P.dM; da.lbuf = P.dl; da.part = P.dpart; da.bar = P.dbar; da.mu_count = P.dmu; da.st = P.gst;
        TT_TRY(launch_dense_local(da, P.dcap, s));
      }
      TT_TRY(run_captured(key2, s, [&]() -> tt_status {
      track_res_kernel<<<1, 1, 0, s>>>(P.gst, D.dv, status_dev);
      track_dx_kernel<<<1, 1024, 0, s>>>(D.iv, D.sol, D.xold, D.dv);
      if (last) {
        TT_TRY(launch_copy(D.cd + 1, 1, P.Ncap, s));
        return TT_OK;
      }
      const int pcap = dir > 0 ? (xc[k] * n < xc[k + 1] ? xc[k] * n : xc[k + 1])
                               : (n * xc[k + 1] < xc[k] ? n * xc[k + 1] : xc[k]);
      plan_svd<<<1, 1, 0, s>>>(D, k, dir);
      { const QCap qc = qcap_svd(x, k, dir); TT_TRY(launch_qr_tall(D.qd, qc.m, qc.n, D.qrws, D.qrwsb, s)); }
      TT_TRY(launch_jacobi(D.sd, 1, pcap, pcap, s));
      trunc_kernel<<<1, 256, 0, s>>>(D, k, dir);
      const int big = n * (xc[k] > xc[k + 1] ? xc[k] : xc[k + 1]);
      TT_TRY(launch_copy(D.cd, 1, P.Ncap, s));
      TT_TRY(launch_gemm(D.gd, 1, big, pc, s));
      TT_TRY(launch_gemm(D.gd + 1, 1, big, big, s));
      plan_enrich<<<1, 1, 0, s>>>(D, k, dir);
      {
        Caps12 ec;
        const int kd = Ah.kind[k];
        descs_local_rhs(zc[k], bc[k], n, zc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, ec.g + 0);
        descs_local_apply_k(kd, zc[k], Rc[k], xc[k], n, n, zc[k + 1], Rc[k + 1], xc[k + 1], 0, 0, 0, 0, 0, 0, 0,
                            ec.g + 2);
        if (dir > 0) {
          descs_local_rhs(xc[k], bc[k], n, zc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, ec.g + 5);
          descs_local_apply_k(kd, xc[k], Rc[k], xc[k], n, n, zc[k + 1], Rc[k + 1], xc[k + 1], 0, 0, 0, 0, 0, 0, 0,
                              ec.g + 7);
        } else {
          descs_local_rhs(zc[k], bc[k], n, xc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, ec.g + 5);
          descs_local_apply_k(kd, zc[k], Rc[k], xc[k], n, n, xc[k + 1], Rc[k + 1], xc[k + 1], 0, 0, 0, 0, 0, 0, 0,
                              ec.g + 7);
        }
        TT_TRY(launch_caps(D.gd, ec, 0, 10));
      }
      TT_TRY(launch_qr(D.qd, 1, s));   // z core
      { const QCap qc = qcap_enrich(x, k, dir); TT_TRY(launch_qr_tall(D.qd + 1, qc.m, qc.n, D.qrws, D.qrwsb, s)); }
      TT_TRY(launch_gemm(D.gd + 10, 1, pc, big, s));
      {
        const int nb_ = dir > 0 ? x.n[k + 1] * xc[k + 2 <= d ? k + 2 : d] : pc;
        const int mb_ = dir > 0 ? pc : x.n[k - 1] * xc[k - 1];
        TT_TRY(launch_gemm(D.gd + 11, 1, mb_, nb_, s));
      }
      TT_TRY(launch_copy(D.cd, 3, P.Scap, s));
      return iface(k, dir);
      }));
    }
    return check_launch("amen sweep");
  };
  (void)zcm; (void)nmax;
  // converged when the max local residual (before the sweep's solves) is <= eps; the
  // solution-change exit (Z20) also stops, but then reports TT_ERR_NOCONV unless the
  // residual test holds too
  if (device_loops(s)) {   // K11: the sweep loop as conditional graph nodes, decided on the device
    set_i32_kernel<<<1, 1, 0, s>>>(D.iv + 14, 0);
    TT_TRY(sweep_loop(s, D.dv, o.eps, o.max_sweeps, D.iv + 14, 0, one_sweep));
    sweep_post_kernel<<<1, 1, 0, s>>>(D.dv, o.eps, D.iv + 14, sweeps_dev, res_dev, status_dev);
    return check_launch("amen_solve");
  }
  int dir = +1, sweep = 0;
  double hres = 0.0;
  for (sweep = 0; sweep < o.max_sweeps; ++sweep) {
    TT_TRY(one_sweep(dir));
    double hv[3] = {0.0, 0.0, 0.0};
    TT_TRY(read_back(hv, D.dv, 3 * sizeof(double), s));
    TT_TRY(check_launch("amen sweep"));
    hres = hv[0];
    if (hv[0] <= o.eps || hv[2] <= o.eps) { ++sweep; break; }
    dir = -dir;
  }
  if (sweeps_dev) set_i32_kernel<<<1, 1, 0, s>>>(sweeps_dev, sweep);
  if (res_dev) cudaMemcpyAsync(res_dev, D.dv, sizeof(double), cudaMemcpyDeviceToDevice, s);
  if (status_dev && !(hres <= o.eps)) set_i32_kernel<<<1, 1, 0, s>>>(status_dev, (int)TT_ERR_NOCONV);
  return check_launch("amen_solve");
}

// =====================================================================
// amen_mv (NEXT-1): y ~ A b by ALS on ||A b - y||^2.  Reuses the
// AMEn machinery with D.x = y and the interface families
//   AL/AR = (y | A | b) [ry, R, rb],  ZAL/ZAR = (z | A | b) [rz, R, rb],
//   ZBL/ZBR = (z | y) [rz, ry];
// the local "solve" is the projection y_k = Phi^{yAb} A_k Psi^{yAb} b_k.
// =====================================================================
namespace {

__global__ void init_ifaces_mv(Dev D) {
  const int d = D.x.d;
  D.AL[0][0] = 1.0; D.ZAL[0][0] = 1.0; D.ZBL[0][0] = 1.0;
  D.AR[d][0] = 1.0; D.ZAR[d][0] = 1.0; D.ZBR[d][0] = 1.0;
}

__global__ void plan_iface_mv(Dev D, int k, int dir) {
  const int n = D.x.n[k], nb = D.b.n[k];
  const int y0 = D.x.r[k], y1 = D.x.r[k + 1], z0 = D.z.r[k], z1 = D.z.r[k + 1];
  const int R0 = D.A.R[k], R1 = D.A.R[k + 1], b0 = D.b.r[k], b1 = D.b.r[k + 1];
  const double *Y = D.x.data + D.x.off[k], *Z = D.z.data + D.z.off[k], *Bk = D.b.data + D.b.off[k];
  const double *Ak = D.A.data + D.A.off[k];
  const int kd = D.A.kind[k];
  if (dir < 0) {
    descs_iface_right_k(kd, y0, R0, b0, n, nb, y1, R1, b1, D.AR[k + 1], Y, Ak, Bk, D.AR[k], D.T1, D.T2, D.gd + 0);
    descs_iface_right_k(kd, z0, R0, b0, n, nb, z1, R1, b1, D.ZAR[k + 1], Z, Ak, Bk, D.ZAR[k], D.T1, D.T2, D.gd + 3);
    descs_iface_right_vec(z0, y0, n, z1, y1, D.ZBR[k + 1], Z, Y, D.ZBR[k], D.T1, D.gd + 6);
  } else {
    descs_iface_left_k(kd, y0, R0, b0, n, nb, y1, R1, b1, D.AL[k], Y, Ak, Bk, D.AL[k + 1], D.T1, D.T2, D.gd + 0);
    descs_iface_left_k(kd, z0, R0, b0, n, nb, z1, R1, b1, D.ZAL[k], Z, Ak, Bk, D.ZAL[k + 1], D.T1, D.T2, D.gd + 3);
    descs_iface_left_vec(z0, y0, n, z1, y1, D.ZBL[k], Z, Y, D.ZBL[k + 1], D.T1, D.gd + 6);
  }
}

// local projection into sol, copies y_k -> xold (dx) and sol -> y_k (last core)
__global__ void plan_local_mv(Dev D, int k) {
  const int n = D.x.n[k], nb = D.b.n[k];
  const int y0 = D.x.r[k], y1 = D.x.r[k + 1];
  const int R0 = D.A.R[k], R1 = D.A.R[k + 1], b0 = D.b.r[k], b1 = D.b.r[k + 1];
  const double *Bk = D.b.data + D.b.off[k], *Ak = D.A.data + D.A.off[k];
  const int N = y0 * n * y1;
  D.iv[0] = N;
  descs_local_apply_k(D.A.kind[k], y0, R0, b0, n, nb, y1, R1, b1, D.AL[k], Ak, D.AR[k + 1], Bk, D.sol, D.T1, D.T2,
                      D.gd + 0);
  D.cd[1] = cpy(N, 1, D.sol, 1, N, D.x.data + D.x.off[k], 1, N);
  D.cd[2] = cpy(N, 1, D.x.data + D.x.off[k], 1, N, D.xold, 1, N);
}

__global__ void plan_enrich_mv(Dev D, int k, int dir) {
  const int n = D.x.n[k], nb = D.b.n[k];
  const int y0 = D.x.r[k], y1 = D.x.r[k + 1], z0 = D.z.r[k], z1 = D.z.r[k + 1];
  const int R0 = D.A.R[k], R1 = D.A.R[k + 1], b0 = D.b.r[k], b1 = D.b.r[k + 1];
  const double *Bk = D.b.data + D.b.off[k], *Ak = D.A.data + D.A.off[k];
  const int r = D.iv[1], mm = D.iv[4], nn = D.iv[5];
  GemmDesc *g = D.gd;
  // crz [z0, n, z1] = (z|A|b) apply - (z|y) projection of the truncated y_k
  const int kd = D.A.kind[k];
  descs_local_apply_k(kd, z0, R0, b0, n, nb, z1, R1, b1, D.ZAL[k], Ak, D.ZAR[k + 1], Bk, D.crz, D.T1, D.T2, g + 0);
  descs_local_rhs(z0, y0, n, z1, y1, D.ZBL[k], D.xfull, D.ZBR[k + 1], D.crz, D.T1, g + 3);
  g[4].alpha = -1.0; g[4].beta = 1.0;
  double *Uc = D.Ue + (long long)r * mm;
  if (dir > 0) {
    // [y0, n, z1]: (y|A|b) left, (z|A|b) right; minus y_k x_3 (z|y)_{k+1}^T
    descs_local_apply_k(kd, y0, R0, b0, n, nb, z1, R1, b1, D.AL[k], Ak, D.ZAR[k + 1], Bk, Uc, D.T1, D.T2, g + 5);
    g[8] = gd_make(y0 * n, z1, y1, D.xfull, (long long)y0 * n, 0, D.ZBR[k + 1], z1, 1);
    gd_plain(g[8], Uc, mm);
  } else {
    // [z0, n, y1]: (z|A|b) left, (y|A|b) right; minus (z|y)_k y_k; written transposed into Ue
    descs_local_apply_k(kd, z0, R0, b0, n, nb, y1, R1, b1, D.ZAL[k], Ak, D.AR[k + 1], Bk, Uc, D.T1, D.T2, g + 5);
    g[7].s_r0 = mm; g[7].s_c0 = 1;
    g[8] = gd_make(z0, n * y1, y0, D.ZBL[k], z0, 0, D.xfull, y0, 0);
    gd_plain(g[8], Uc, 1);
    g[8].s_r0 = mm; g[8].s_c0 = 1;
  }
  g[8].alpha = -1.0; g[8].beta = 1.0;
  g[9] = gd_make(0, 0, 0, nullptr, 1, 0, nullptr, 1, 0);
  gd_plain(g[9], nullptr, 1);
  const int ze = dir > 0 ? z1 : z0;
  enrich_tail(D, k, dir, n, r, mm, nn, ze, z0, z1, g);
}

}  // namespace

struct MvCtx {
  Dev D;
  char *orth_base;
  size_t orth_cap;
  double *split;
  unsigned int *bar;
  long long Ncap, Scap;
  int pc;
};

static tt_status carve_mv(const MatMeta &A, const VecMeta &b, const VecMeta &y, const VecMeta &z, Arena &ar,
                          MvCtx &P) {
  const int d = A.d;
  if (b.d != d || y.d != d || z.d != d) return fail(TT_ERR_SHAPE, "amen_mv: number of cores differ");
  for (int k = 0; k < d; ++k)
    if (A.n[k] != b.n[k] || A.m[k] != y.n[k] || z.n[k] != y.n[k]) return fail(TT_ERR_SHAPE, "amen_mv: shape mismatch");
  for (int k = 1; k < d; ++k)
    if (y.rcap[k] <= z.rcap[k]) return fail(TT_ERR_CAPACITY, "amen_mv: y rank capacity must exceed z's");
  std::memset(&P, 0, sizeof(P));
  Dev &D = P.D;
  D.x = y; D.z = z; D.b = b; D.A = A;
  D.m = 0;
  long long Ncap = 1, Zcap = 1, Tcap = 1, Ecap = 1, Scap = 1;
  int pc = 1, zcm = 1;
  for (int k = 0; k <= d; ++k) { pc = y.rcap[k] > pc ? y.rcap[k] : pc; zcm = z.rcap[k] > zcm ? z.rcap[k] : zcm; }
  for (int k = 0; k < d; ++k) {
    const long long n = lmax(y.n[k], b.n[k]);
    Ncap = lmax(Ncap, (long long)y.rcap[k] * n * y.rcap[k + 1]);
    Zcap = lmax(Zcap, (long long)z.rcap[k] * n * z.rcap[k + 1]);
    long long rm = lmax(lmax(y.rcap[k], y.rcap[k + 1]), lmax(z.rcap[k], z.rcap[k + 1]));
    rm = lmax(rm, lmax(b.rcap[k], b.rcap[k + 1]));
    const long long Rm = lmax(A.Rcap[k], A.Rcap[k + 1]);
    Tcap = lmax(Tcap, n * rm * rm * Rm);
    Ecap = lmax(Ecap, n * lmax(y.rcap[k], y.rcap[k + 1]) * (pc + zcm));
    Scap = lmax(Scap, lmax((long long)y.rcap[k] * n * y.rcap[k + 1], (long long)z.rcap[k] * n * z.rcap[k + 1]));
  }
  P.Ncap = Ncap; P.Scap = Scap; P.pc = pc;
  D.kscr = ar.take<float>(KIND_SCRATCH_FLOATS);
  D.qrwsb = qr_ws_amen(y);
  D.qrws = ar.take<char>(D.qrwsb);
  for (int k = 0; k <= d; ++k) {
    D.AL[k] = ar.take<double>((size_t)y.rcap[k] * A.Rcap[k] * b.rcap[k]);
    D.AR[k] = ar.take<double>((size_t)y.rcap[k] * A.Rcap[k] * b.rcap[k]);
    D.ZAL[k] = ar.take<double>((size_t)z.rcap[k] * A.Rcap[k] * b.rcap[k]);
    D.ZAR[k] = ar.take<double>((size_t)z.rcap[k] * A.Rcap[k] * b.rcap[k]);
    D.ZBL[k] = ar.take<double>((size_t)z.rcap[k] * y.rcap[k]);
    D.ZBR[k] = ar.take<double>((size_t)z.rcap[k] * y.rcap[k]);
  }
  D.sol = ar.take<double>(Ncap);
  D.xold = ar.take<double>(Ncap);
  D.T1 = ar.take<double>(Tcap);
  D.T2 = ar.take<double>(Tcap);
  D.crz = ar.take<double>(Zcap);
  D.xfull = ar.take<double>(Ncap);
  D.tmp = ar.take<double>(Scap);
  D.tmpz = ar.take<double>(Zcap);
  D.K = ar.take<double>(Ecap);
  D.qA = ar.take<double>(lmax(Ncap, Ecap));
  D.qQ = ar.take<double>(Ncap);
  D.qR = ar.take<double>((size_t)pc * pc);
  D.tau = ar.take<double>(pc + zcm);
  D.qT = ar.take<double>(32 * 32 * ((pc + zcm) / 32 + 2));
  D.qA2 = ar.take<double>(Zcap);
  D.tau2 = ar.take<double>(zcm + 1);
  D.qT2 = ar.take<double>(32 * 32 * (zcm / 32 + 2));
  D.qRe = ar.take<double>((size_t)(pc + zcm) * (pc + zcm));
  D.U = ar.take<double>((size_t)pc * pc);
  D.Vs = ar.take<double>((size_t)pc * pc);
  D.S = ar.take<double>(pc);
  D.J = ar.take<double>((size_t)2 * pc * pc);
  D.Ue = ar.take<double>(Ecap);
  D.Ct = ar.take<double>(Ncap);
  D.gd = ar.take<GemmDesc>(NG);
  D.qd = ar.take<QRDesc>(2);
  D.sd = ar.take<SVDDesc>(1);
  D.cd = ar.take<CopyDesc>(8);
  D.iv = ar.take<int>(16);
  D.dv = ar.take<double>(8);
  D.limit = ar.take<int>(TT_MAX_D + 1);
  Arena c1, c2;
  orth_meta(y, -1, nullptr, c1, nullptr);
  orth_meta(z, -1, nullptr, c2, nullptr);
  P.orth_cap = c1.used > c2.used ? c1.used : c2.used;
  P.orth_base = ar.take<char>(P.orth_cap);
  P.split = ar.take<double>(GEMM_SPLIT_SCRATCH / 8);
  P.bar = ar.take<unsigned int>(4);
  return TT_OK;
}

size_t amen_mv_ws_bytes(const MatMeta &A, const VecMeta &b, const VecMeta &y, const VecMeta &z) {
  Arena ar;
  MvCtx P;
  if (carve_mv(A, b, y, z, ar, P) != TT_OK) return 0;
  return ar.used;
}

tt_status amen_mv_meta(const MatMeta &A, const VecMeta &b, const VecMeta &y, const VecMeta &z, double eps,
                       int max_sweeps, int rmax, int *sweeps_dev, Arena &ar, cudaStream_t s) {
  MvCtx P;
  const Arena ar0 = ar;
  TT_TRY(carve_mv(A, b, y, z, ar, P));
  if (!ar.base) return TT_OK;
  if (!ar.ok()) return fail(TT_ERR_CAPACITY, "amen_mv: workspace too small");
  if (!(eps > 0.0) || max_sweeps < 1 || rmax < 1) return fail(TT_ERR_ARG, "amen_mv: eps > 0, max_sweeps, rmax >= 1");
  Dev &D = P.D;
  const int d = A.d;
  if (!D.A.kinds_set) TT_TRY(detect_core_kinds(D.A, D.kscr, s));   // one read-back, before any capture
  if (graph_mode() >= 2 && !stream_capturing(s)) {   // the whole product as one graph (K11)
    GraphKey key;
    key.add(D);
    const int ii[2] = {max_sweeps, rmax};
    key.add(eps);
    key.add(ii);
    const MatMeta Ak = D.A;
    TT_TRY(run_captured(key, s, [&]() -> tt_status {
      Arena a = ar0;
      return amen_mv_meta(Ak, b, y, z, eps, max_sweeps, rmax, D.iv + 13, a, s);
    }));
    report_out_kernel<<<1, 1, 0, s>>>(D.iv + 13, nullptr, nullptr, sweeps_dev, nullptr, nullptr);
    return check_launch("amen_mv report");
  }
  ScratchScope scratch_scope;
  const MatMeta &Ah = D.A;
  set_limits_kernel<<<1, 64, 0, s>>>(y, z, rmax, D.limit);
  set_dv_kernel<<<1, 1, 0, s>>>(D.dv, 1, eps);
  set_gemm_scratch(P.split, GEMM_SPLIT_SCRATCH);
  set_jacobi_sync(P.bar);
  Arena oa;
  oa.base = P.orth_base;
  oa.cap = P.orth_cap;
  TT_TRY(orth_meta(y, -1, nullptr, oa, s));
  oa.used = 0;
  TT_TRY(orth_meta(z, -1, nullptr, oa, s));
  init_ifaces_mv<<<1, 1, 0, s>>>(D);
  const int *yc = y.rcap, *zc = z.rcap, *bc = b.rcap, *Rc = A.Rcap;
  struct Caps12 { GemmDesc g[12]; };
  auto launch_caps = [&](const GemmDesc *dev, const Caps12 &hc, int from, int cnt) -> tt_status {
    int Mc[12], Nc[12], Kc[12], Bc[12];
    for (int i = 0; i < cnt; ++i) {
      Mc[i] = hc.g[from + i].M; Nc[i] = hc.g[from + i].N; Kc[i] = hc.g[from + i].K; Bc[i] = hc.g[from + i].batch;
    }
    return launch_gemm_seq(dev, cnt, Mc, Nc, Kc, s, Bc);
  };
  auto iface = [&](int k, int dir) -> tt_status {
    plan_iface_mv<<<1, 1, 0, s>>>(D, k, dir);
    Caps12 c;
    const int n = y.n[k], nb = b.n[k];
    const int kd = Ah.kind[k];
    if (dir < 0) {
      descs_iface_right_k(kd, yc[k], Rc[k], bc[k], n, nb, yc[k + 1], Rc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, 0, 0, c.g + 0);
      descs_iface_right_k(kd, zc[k], Rc[k], bc[k], n, nb, zc[k + 1], Rc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, 0, 0, c.g + 3);
      descs_iface_right_vec(zc[k], yc[k], n, zc[k + 1], yc[k + 1], 0, 0, 0, 0, 0, c.g + 6);
    } else {
      descs_iface_left_k(kd, yc[k], Rc[k], bc[k], n, nb, yc[k + 1], Rc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, 0, 0, c.g + 0);
      descs_iface_left_k(kd, zc[k], Rc[k], bc[k], n, nb, zc[k + 1], Rc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, 0, 0, c.g + 3);
      descs_iface_left_vec(zc[k], yc[k], n, zc[k + 1], yc[k + 1], 0, 0, 0, 0, 0, c.g + 6);
    }
    return launch_caps(D.gd, c, 0, 8);
  };
  for (int k = d - 1; k >= 1; --k) TT_TRY(iface(k, -1));
  // one sweep = a fixed launch sequence (device-resident sizes): replayed as a CUDA graph
  auto one_sweep = [&](int dir) -> tt_status {
    set_dv_kernel<<<1, 1, 0, s>>>(D.dv, 2, 0.0);
    for (int t = 0; t < d; ++t) {
      const int k = dir > 0 ? t : d - 1 - t;
      const int last = (t == d - 1);
      const int n = y.n[k], nb = b.n[k];
      Caps12 lc;
      const int kd = Ah.kind[k];
      descs_local_apply_k(kd, yc[k], Rc[k], bc[k], n, nb, yc[k + 1], Rc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, 0, 0, lc.g + 0);
      plan_local_mv<<<1, 1, 0, s>>>(D, k);
      TT_TRY(launch_copy(D.cd + 2, 1, P.Ncap, s));
      TT_TRY(launch_caps(D.gd, lc, 0, 3));
      track_dx_kernel<<<1, 1024, 0, s>>>(D.iv, D.sol, D.xold, D.dv);
      if (last) {
        TT_TRY(launch_copy(D.cd + 1, 1, P.Ncap, s));
        continue;
      }
      const int pcap = dir > 0 ? (yc[k] * n < yc[k + 1] ? yc[k] * n : yc[k + 1])
                               : (n * yc[k + 1] < yc[k] ? n * yc[k + 1] : yc[k]);
      plan_svd<<<1, 1, 0, s>>>(D, k, dir);
      { const QCap qc = qcap_svd(y, k, dir); TT_TRY(launch_qr_tall(D.qd, qc.m, qc.n, D.qrws, D.qrwsb, s)); }
      TT_TRY(launch_jacobi(D.sd, 1, pcap, pcap, s));
      trunc_kernel<<<1, 256, 0, s>>>(D, k, dir);
      const int big = n * (yc[k] > yc[k + 1] ? yc[k] : yc[k + 1]);
      TT_TRY(launch_copy(D.cd, 1, P.Ncap, s));
      TT_TRY(launch_gemm(D.gd, 1, big, P.pc, s));
      TT_TRY(launch_gemm(D.gd + 1, 1, big, big, s));
      plan_enrich_mv<<<1, 1, 0, s>>>(D, k, dir);
      {
        Caps12 ec;
        descs_local_apply_k(kd, zc[k], Rc[k], bc[k], n, nb, zc[k + 1], Rc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, 0, 0,
                            ec.g + 0);
        descs_local_rhs(zc[k], yc[k], n, zc[k + 1], yc[k + 1], 0, 0, 0, 0, 0, ec.g + 3);
        if (dir > 0) {
          descs_local_apply_k(kd, yc[k], Rc[k], bc[k], n, nb, zc[k + 1], Rc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, 0, 0,
                              ec.g + 5);
          ec.g[8] = gd_make(yc[k] * n, zc[k + 1], yc[k + 1], nullptr, 1, 0, nullptr, 1, 1);
        } else {
          descs_local_apply_k(kd, zc[k], Rc[k], bc[k], n, nb, yc[k + 1], Rc[k + 1], bc[k + 1], 0, 0, 0, 0, 0, 0, 0,
                              ec.g + 5);
          ec.g[8] = gd_make(zc[k], n * yc[k + 1], yc[k], nullptr, 1, 0, nullptr, 1, 0);
        }
        TT_TRY(launch_caps(D.gd, ec, 0, 9));
      }
      TT_TRY(launch_qr(D.qd, 1, s));   // z core
      { const QCap qc = qcap_enrich(y, k, dir); TT_TRY(launch_qr_tall(D.qd + 1, qc.m, qc.n, D.qrws, D.qrwsb, s)); }
      TT_TRY(launch_gemm(D.gd + 10, 1, P.pc, big, s));
      {
        const int nb_ = dir > 0 ? y.n[k + 1] * yc[k + 2 <= d ? k + 2 : d] : P.pc;
        const int mb_ = dir > 0 ? P.pc : y.n[k - 1] * yc[k - 1];
        TT_TRY(launch_gemm(D.gd + 11, 1, mb_, nb_, s));
      }
      TT_TRY(launch_copy(D.cd, 3, P.Scap, s));
      TT_TRY(iface(k, dir));
    }
    return TT_OK;
  };
  if (device_loops(s)) {   // K11: sweep loop decided on the device
    set_i32_kernel<<<1, 1, 0, s>>>(D.iv + 14, 0);
    TT_TRY(sweep_loop(s, D.dv, eps, max_sweeps, D.iv + 14, 1, one_sweep));
    sweep_post_kernel<<<1, 1, 0, s>>>(D.dv, eps, D.iv + 14, sweeps_dev, nullptr, nullptr);
    return check_launch("amen_mv");
  }
  GraphKey base;   // D is fixed for the whole product
  base.add(D);
  {
    const long long extra[4] = {P.Ncap, P.Scap, P.pc, 0x6d76};
    base.add(extra);
  }
  int dir = +1, sweep = 0;
  for (sweep = 0; sweep < max_sweeps; ++sweep) {
    GraphKey key = base;
    key.add(dir);
    TT_TRY(run_captured(key, s, [&]() { return one_sweep(dir); }));
    double hv[3] = {0.0, 0.0, 0.0};
    TT_TRY(read_back(hv, D.dv, 3 * sizeof(double), s));
    TT_TRY(check_launch("amen_mv sweep"));
    if (hv[2] <= eps) { ++sweep; break; }
    dir = -dir;
  }
  if (sweeps_dev) set_i32_kernel<<<1, 1, 0, s>>>(sweeps_dev, sweep);
  return check_launch("amen_mv");
}

}  // namespace tt
