// Descriptor builders for the ALS / AMEn contractions.
// Every contraction is a chain of DMMA GEMMs whose epilogue writes the
// intermediate directly in the layout the next GEMM reads as a plain matrix.
// Usable on the host (ABI calls with host sizes) and on the device (AMEn plan
// kernels with device-resident ranks).
#pragma once
#include "tt_common.cuh"

namespace tt {

__host__ __device__ inline GemmDesc gd_make(int M, int N, int K, const double *A, long long lda, int tA,
                                            const double *B, long long ldb, int tB) {
  GemmDesc g;
  g.M = M; g.N = N; g.K = K;
  g.transA = tA; g.transB = tB;
  g.A = A; g.lda = lda;
  g.B = B; g.ldb = ldb;
  g.C = nullptr;
  g.dr = 1 << 30; g.dc = 1 << 30;
  g.s_r0 = 1; g.s_r1 = 0; g.s_c0 = 0; g.s_c1 = 0;
  g.alpha = 1.0; g.beta = 0.0; g.alpha_dev = nullptr; g.skip = nullptr;
  return g;
}
__host__ __device__ inline void gd_scatter(GemmDesc &g, double *C, int dr, long long sr0, long long sr1, int dc,
                                           long long sc0, long long sc1) {
  g.C = C; g.dr = dr; g.s_r0 = sr0; g.s_r1 = sr1; g.dc = dc; g.s_c0 = sc0; g.s_c1 = sc1;
}
__host__ __device__ inline void gd_plain(GemmDesc &g, double *C, long long ldc) {
  g.C = C; g.dr = 1 << 30; g.s_r0 = 1; g.s_r1 = 0; g.dc = 1 << 30; g.s_c0 = ldc; g.s_c1 = 0;
}

// y[a,i,a'] = sum Phi[a,g,b] A[g,i,j,g'] Psi[a',g',b'] x[b,j,b']
// T1 >= rB n rAp Rp, T2 >= R m rB rAp.
__host__ __device__ inline void descs_local_apply(int rA, int R, int rB, int m, int n, int rAp, int Rp, int rBp,
                                                  const double *Phi, const double *Ak, const double *Psi,
                                                  const double *x, double *y, double *T1, double *T2,
                                                  GemmDesc *g) {
  // (1) T1'[(j,g'),(b,a')] = sum_b' x[(b,j), b'] Psi[(a',g'), b']
  g[0] = gd_make(rB * n, rAp * Rp, rBp, x, (long long)rB * n, 0, Psi, (long long)rAp * Rp, 1);
  gd_scatter(g[0], T1, rB, (long long)n * Rp, 1, rAp, (long long)n * Rp * rB, n);
  // (2) T2''[g, b, i, a'] = sum_{(j,g')} A[(g,i),(j,g')] T1'[(j,g'),(b,a')]
  g[1] = gd_make(R * m, rB * rAp, n * Rp, Ak, (long long)R * m, 0, T1, (long long)n * Rp, 0);
  gd_scatter(g[1], T2, R, 1, (long long)R * rB, rB, R, (long long)R * rB * m);
  // (3) y[a,(i,a')] = sum_{(g,b)} Phi[a,(g,b)] T2''[(g,b),(i,a')]
  g[2] = gd_make(rA, m * rAp, R * rB, Phi, rA, 0, T2, (long long)R * rB, 0);
  gd_plain(g[2], y, rA);
}

// Left interface: Phi_k[a',g',b'] = sum Phi[a,g,b] Y[a,i,a'] A[g,i,j,g'] X[b,j,b']
// T1 >= R m rX rYp, T2 >= rX n rYp Rp.
__host__ __device__ inline void descs_iface_left(int rY, int R, int rX, int m, int n, int rYp, int Rp, int rXp,
                                                 const double *Phi, const double *Y, const double *Ak,
                                                 const double *X, double *out, double *T1, double *T2,
                                                 GemmDesc *g) {
  // (1) T1'[(g,i),(b,a')] = sum_a Phi[a,(g,b)] Y[a,(i,a')]
  g[0] = gd_make(R * rX, m * rYp, rY, Phi, rY, 1, Y, rY, 0);
  gd_scatter(g[0], T1, R, 1, (long long)R * m, m, R, (long long)R * m * rX);
  // (2) T2'[(b,j),(a',g')] = sum_{(g,i)} T1'[(g,i),(b,a')] A[(g,i),(j,g')]
  g[1] = gd_make(rX * rYp, n * Rp, R * m, T1, (long long)R * m, 1, Ak, (long long)R * m, 0);
  gd_scatter(g[1], T2, rX, 1, (long long)rX * n, n, rX, (long long)rX * n * rYp);
  // (3) Phi_k[(a',g'), b'] = sum_{(b,j)} T2'[(b,j),(a',g')] X[(b,j), b']
  g[2] = gd_make(rYp * Rp, rXp, rX * n, T2, (long long)rX * n, 1, X, (long long)rX * n, 0);
  gd_plain(g[2], out, (long long)rYp * Rp);
}

// Right interface: Psi_k[a,g,b] = sum Psi[a',g',b'] Y[a,i,a'] A[g,i,j,g'] X[b,j,b']
// T1 >= rX n rYp Rp, T2 >= m rYp R rX.
__host__ __device__ inline void descs_iface_right(int rY, int R, int rX, int m, int n, int rYp, int Rp, int rXp,
                                                  const double *Psi, const double *Y, const double *Ak,
                                                  const double *X, double *out, double *T1, double *T2,
                                                  GemmDesc *g) {
  // (1) T1'[(j,g'),(b,a')] = sum_b' X[(b,j), b'] Psi[(a',g'), b']
  g[0] = gd_make(rX * n, rYp * Rp, rXp, X, (long long)rX * n, 0, Psi, (long long)rYp * Rp, 1);
  gd_scatter(g[0], T1, rX, (long long)n * Rp, 1, rYp, (long long)n * Rp * rX, n);
  // (2) T2'[(i,a'),(g,b)] = sum_{(j,g')} A[(g,i),(j,g')] T1'[(j,g'),(b,a')]
  g[1] = gd_make(R * m, rX * rYp, n * Rp, Ak, (long long)R * m, 0, T1, (long long)n * Rp, 0);
  gd_scatter(g[1], T2, R, (long long)m * rYp, 1, rX, (long long)m * rYp * R, m);
  // (3) Psi_k[a,(g,b)] = sum_{(i,a')} Y[a,(i,a')] T2'[(i,a'),(g,b)]
  g[2] = gd_make(rY, R * rX, m * rYp, Y, rY, 0, T2, (long long)m * rYp, 0);
  gd_plain(g[2], out, rY);
}

// Vector left interface: phi_k[a',b'] = sum phi[a,b] Y[a,i,a'] X[b,i,b'];  T1 >= rX m rYp.
__host__ __device__ inline void descs_iface_left_vec(int rY, int rX, int m, int rYp, int rXp, const double *phi,
                                                     const double *Y, const double *X, double *out, double *T1,
                                                     GemmDesc *g) {
  g[0] = gd_make(rX, m * rYp, rY, phi, rY, 1, Y, rY, 0);
  gd_plain(g[0], T1, rX);
  g[1] = gd_make(rYp, rXp, rX * m, T1, (long long)rX * m, 1, X, (long long)rX * m, 0);
  gd_plain(g[1], out, rYp);
}

// Vector right interface: psi_k[a,b] = sum psi[a',b'] Y[a,i,a'] X[b,i,b'];  T1 >= rX m rYp.
__host__ __device__ inline void descs_iface_right_vec(int rY, int rX, int m, int rYp, int rXp, const double *psi,
                                                      const double *Y, const double *X, double *out, double *T1,
                                                      GemmDesc *g) {
  g[0] = gd_make(rX * m, rYp, rXp, X, (long long)rX * m, 0, psi, rYp, 1);
  gd_plain(g[0], T1, (long long)rX * m);
  g[1] = gd_make(rY, rX, m * rYp, Y, rY, 0, T1, rX, 1);
  gd_plain(g[1], out, rY);
}

// Local right-hand side: rhs[a,i,a'] = sum phi[a,b] B[b,i,b'] psi[a',b'];  T1 >= rB m rAp.
__host__ __device__ inline void descs_local_rhs(int rA, int rB, int m, int rAp, int rBp, const double *phi,
                                                const double *Bk, const double *psi, double *rhs, double *T1,
                                                GemmDesc *g) {
  g[0] = gd_make(rB * m, rAp, rBp, Bk, (long long)rB * m, 0, psi, rAp, 1);
  gd_plain(g[0], T1, (long long)rB * m);
  g[1] = gd_make(rA, m * rAp, rB, phi, rA, 0, T1, rB, 0);
  gd_plain(g[1], rhs, rA);
}

}  // namespace tt
