// Batched small dense linear algebra for TT rounding / AMEn on sm_100a (fp64):
//   * blocked Householder QR (LAPACK geqrf/larft/larfb/orgqr structure) with an
//     explicit Q — rank-deficient safe (tau = 0 for a zero column);
//   * one-sided Hestenes Jacobi SVD, parallel round-robin ordering, one warp
//     per column pair, data in shared memory when it fits.
// One CTA per problem; problems are batched over the grid.  Sizes come from
// descriptors in device memory (they follow device-resident TT ranks).
#include <cfloat>

#include <cooperative_groups.h>

#include "tt_common.cuh"

namespace tt {

// nominal flops: [0] Householder QR (geqrf + orgqr), [1] Jacobi rotations + column dots
__device__ unsigned long long g_linalg_flops[2];

namespace {

#ifndef QR_THREADS_DEF
#define QR_THREADS_DEF 1024   // measured: 1024 > 512 > 256 (C1 94.1 / 94.0 / 91.1 iter/s, C2 6.13 / 6.05 / 5.55;
                              // re-measured on the final round-1 code: 1024 vs 512 = C1 103.7 / 103.5, C2 6.32 / 6.24)
#endif
constexpr int QR_THREADS = QR_THREADS_DEF;
constexpr int NB = 32;
// panels of up to QR_PANEL_ROWS rows are factorised in shared memory (the
// per-column reductions and updates then never touch L2)
constexpr int QR_PANEL_ROWS = 640;
constexpr size_t QR_PANEL_SMEM = (size_t)QR_PANEL_ROWS * NB * sizeof(double);

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}


// Block reflector application on a target matrix X (element (r, c) at
// X[r*rs + c*cs]):  X[j0:m, c] -= V * (op(T) * (V^T X[j0:m, c])) for the
// columns c in [c_begin, c_end), op(T) = T^T (transT = 1, the trailing update
// of geqrf) or T (transT = 0, orgqr).  V is the unit lower trapezoidal panel:
// element (row j0 + rr, reflector l) at V[rr + l * ldv], the shared-memory
// panel copy (SM) or the working matrix in global memory (V = A + j0 + j0 lda).
// On the FP64 tensor pipe (mma.sync.m8n8k4.f64 = DMMA), one warp per chunk of 8
// target columns, no block barrier:
//   W  (32 x 8)  = V^T X_chunk       4 accumulator tiles over mr/4 k-steps
//   W' (32 x 8)  = op(T) W            8 k-steps, W moved from the accumulator
//                                     layout to B fragments by shuffles
//   X_chunk     -= V W'              row tiles of 8, X loaded as the accumulator
// (the scalar version read one shared-memory double per FMA and was bound by
// shared-memory bandwidth: 373 us for the Q of a 264 x 132 QR).
__device__ __forceinline__ void dmma_f64(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// 32 x 8 block in accumulator layout (tile i: lane t holds rows 8i + t/4, columns
// 2(t%4) + {0, 1}) -> B fragments of the 8 k-steps (lane t: row 4kk + t%4, column t/4)
__device__ __forceinline__ void acc_to_bfrag(const double (&d)[4][2], double (&b)[8], int lane) {
  const int n = lane >> 2;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const int mrow = 4 * kk + (lane & 3);
    const int src = (mrow & 7) * 4 + (n >> 1);
    const double v0 = __shfl_sync(0xffffffffu, d[kk >> 1][0], src);
    const double v1 = __shfl_sync(0xffffffffu, d[kk >> 1][1], src);
    b[kk] = (n & 1) ? v1 : v0;
  }
}

template <bool SM>
__device__ __forceinline__ void apply_block_reflector(int m, int j0, int jb, const double *__restrict__ V, int ldv,
                                                      const double (*sT)[NB + 1], int transT, double *X,
                                                      long long rs, long long cs, int c_begin, int c_end) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
  const int mr = m - j0;                  // rows j0..m-1
  const int q4 = lane & 3, g8 = lane >> 2;
  // masked V element (row rr, reflector l): unit lower trapezoid, zero outside
  auto vm = [&](int rr, int l) -> double {
    if (l >= jb || rr >= mr || rr < l) return 0.0;
    return rr == l ? 1.0 : V[rr + l * ldv];
  };
  const int nchunk = (c_end - c_begin + 7) >> 3;
  for (int ch = warp; ch < nchunk; ch += NW) {
    const int c0 = c_begin + 8 * ch;
    double *X0 = X + (long long)j0 * rs + (long long)c0 * cs;
    // ---- W = V^T X_chunk: A[m = l][k = rr] = V(rr, l), B[k = rr][n] = X(rr, c0 + n)
    double w[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i][0] = w[i][1] = 0.0;
    const bool colok = c0 + g8 < c_end;
    const double *xb = X0 + (long long)g8 * cs;
    int r0 = 0;
    for (; r0 < 32 && r0 < mr; r0 += 4) {                 // triangle rows: masked
      const int rr = r0 + q4;
      const double b = (colok && rr < mr) ? xb[(long long)rr * rs] : 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma_f64(w[i][0], w[i][1], vm(rr, 8 * i + g8), b);
    }
    if (jb == NB) {
      // full rows, all 32 reflectors stored: 8 k-steps per batch, their X loads
      // issued together (X lives in L2 / global memory)
      for (; r0 + 32 <= mr; r0 += 32) {
        double b[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) b[u] = colok ? xb[(long long)(r0 + 4 * u + q4) * rs] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double *vp = V + r0 + 4 * u + q4 + g8 * ldv;
#pragma unroll
          for (int i = 0; i < 4; ++i) dmma_f64(w[i][0], w[i][1], vp[8 * i * ldv], b[u]);
        }
      }
      for (; r0 + 4 <= mr; r0 += 4) {
        const int rr = r0 + q4;
        const double b = colok ? xb[(long long)rr * rs] : 0.0;
        const double *vp = V + rr + g8 * ldv;
#pragma unroll
        for (int i = 0; i < 4; ++i) dmma_f64(w[i][0], w[i][1], vp[8 * i * ldv], b);
      }
    }
    for (; r0 < mr; r0 += 4) {                            // ragged tail / short panel
      const int rr = r0 + q4;
      const double b = (colok && rr < mr) ? xb[(long long)rr * rs] : 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma_f64(w[i][0], w[i][1], vm(rr, 8 * i + g8), b);
    }
    // ---- W' = op(T) W: A[m][k] = op(T)(m, k) from shared memory, B = W fragments
    double bw[8];
    acc_to_bfrag(w, bw, lane);
    double wp[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) wp[i][0] = wp[i][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int k = 4 * kk + q4;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int mm = 8 * i + g8;
        const double a = transT ? sT[k][mm] : sT[mm][k];
        dmma_f64(wp[i][0], wp[i][1], a, bw[kk]);
      }
    }
    double bn[8];
    acc_to_bfrag(wp, bn, lane);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) bn[kk] = -bn[kk];
    // ---- X_chunk -= V W': row tiles of 8; C = X (lane: row t/4, columns 2(t%4) + {0,1})
    const int ca = c0 + 2 * q4, cb = ca + 1;
    const bool oka = ca < c_end, okb = cb < c_end;
    double *xa = X0 + (long long)(2 * q4) * cs, *xbb = xa + cs;
    int t0 = 0;
    if (jb == NB) {
      for (; t0 < 32 && t0 < mr; t0 += 8) {                // triangle rows: masked
        const int rr = t0 + g8;
        const bool rok = rr < mr;
        double d0 = (rok && oka) ? xa[(long long)rr * rs] : 0.0;
        double d1 = (rok && okb) ? xbb[(long long)rr * rs] : 0.0;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) dmma_f64(d0, d1, vm(rr, 4 * kk + q4), bn[kk]);
        if (rok && oka) xa[(long long)rr * rs] = d0;
        if (rok && okb) xbb[(long long)rr * rs] = d1;
      }
      for (; t0 + 32 <= mr; t0 += 32) {                   // 4 full row tiles per batch
        double d[4][2];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const long long rr = t0 + 8 * u + g8;
          d[u][0] = oka ? xa[rr * rs] : 0.0;
          d[u][1] = okb ? xbb[rr * rs] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double *vp = V + t0 + 8 * u + g8 + q4 * ldv;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) dmma_f64(d[u][0], d[u][1], vp[4 * kk * ldv], bn[kk]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const long long rr = t0 + 8 * u + g8;
          if (oka) xa[rr * rs] = d[u][0];
          if (okb) xbb[rr * rs] = d[u][1];
        }
      }
    }
    for (; t0 < mr; t0 += 8) {
      const int rr = t0 + g8;
      const bool rok = rr < mr;
      double d0 = (rok && oka) ? xa[(long long)rr * rs] : 0.0;
      double d1 = (rok && okb) ? xbb[(long long)rr * rs] : 0.0;
      if (t0 >= 32 && t0 + 8 <= mr && jb == NB) {
        const double *vp = V + rr + q4 * ldv;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) dmma_f64(d0, d1, vp[4 * kk * ldv], bn[kk]);
      } else {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) dmma_f64(d0, d1, vm(rr, 4 * kk + q4), bn[kk]);
      }
      if (rok && oka) xa[(long long)rr * rs] = d0;
      if (rok && okb) xbb[(long long)rr * rs] = d1;
    }
  }
}

// Register-resident panel for short panels (pr <= 32 MR rows, panel in shared
// memory): warp w owns panel column w and keeps it in registers (MR doubles per
// lane) for the whole panel factorisation.  Step jj: warp jj forms reflector jj
// from its registers and writes the finished column (R above the diagonal, beta,
// v below) to the panel; one block barrier; every later warp reads v_jj once
// from shared memory and updates its own registers.  The column-in-shared-memory
// version moved three columns' worth of shared-memory traffic per updated column
// and step (read v, read and write the column) and the lookahead warp's dependent
// loads queued behind it; here a step reads v once per warp and the next owner
// goes straight from its update to its reflector.
template <int MR>
__device__ __forceinline__ void qr_panel_reg(const QRDesc &g, int j0, int jb, int pr, double *sP, double *s_tau) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool own = warp < jb;
  double *mycol = sP + (size_t)warp * pr;
  double x[MR];
#pragma unroll
  for (int q = 0; q < MR; ++q) {
    const int r = lane + 32 * q;
    x[q] = (own && r < pr) ? mycol[r] : 0.0;
  }
  for (int jj = 0; jj < jb; ++jj) {
    if (warp == jj) {   // local diagonal row jj < 32: lane jj, q = 0
      double sigma = 0.0;
#pragma unroll
      for (int q = 0; q < MR; ++q)
        if (lane + 32 * q > jj) sigma = fma(x[q], x[q], sigma);
      sigma = warp_sum(sigma);
      const double alpha = __shfl_sync(0xffffffffu, x[0], jj);
      double tau = 0.0, scal = 0.0, beta = alpha;
      if (sigma > 0.0 && fma(alpha, alpha, sigma) > 1e-200) {   // tiny-column guard: reading Z41
        const double ss = fma(alpha, alpha, sigma);
        const double rs = rsqrt(ss);
        const double nrm = ss * rs, aa = fabs(alpha);
        beta = alpha >= 0.0 ? -nrm : nrm;
        tau = fma(aa, rs, 1.0);
        const double qv = __drcp_rn(aa + nrm);
        scal = alpha >= 0.0 ? qv : -qv;
      }
      if (tau != 0.0) {
#pragma unroll
        for (int q = 0; q < MR; ++q)
          if (lane + 32 * q > jj) x[q] *= scal;
      }
      if (lane == jj) x[0] = beta;
#pragma unroll
      for (int q = 0; q < MR; ++q) {
        const int r = lane + 32 * q;
        if (r < pr) mycol[r] = x[q];
      }
      if (lane == 0) {
        s_tau[jj & 1] = tau;
        g.tau[j0 + jj] = tau;
      }
    }
    __syncthreads();
    const double tau = s_tau[jj & 1];
    if (own && warp > jj && tau != 0.0) {
      const double *v = sP + (size_t)jj * pr;
      double vv[MR];
#pragma unroll
      for (int q = 0; q < MR; ++q) {
        const int r = lane + 32 * q;
        vv[q] = (r > jj && r < pr) ? v[r] : 0.0;
      }
      double d = (lane == jj) ? x[0] : 0.0;   // v_jj[jj] = 1
#pragma unroll
      for (int q = 0; q < MR; ++q) d = fma(vv[q], x[q], d);
      d = warp_sum(d) * tau;
#pragma unroll
      for (int q = 0; q < MR; ++q) x[q] = fma(-d, vv[q], x[q]);
      if (lane == jj) x[0] -= d;
    }
  }
  __syncthreads();
}

// Panel factorisation of columns j0..j0+jb-1 (rows j0..m-1) and the Gram
// entries G[l][i] = v_l^T v_i (l < i) of the T factor.  SM: the panel lives in
// shared memory (sP, leading dimension pr) — a separate instantiation so the
// accesses compile to plain shared-memory loads rather than generic ones.
template <bool SM>
__device__ __forceinline__ void qr_panel(const QRDesc &g, int m, int j0, int jb, int pr, double *A, long long lda,
                                         double *sP, double *s_tau, double (*sG)[NB + 1]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = QR_THREADS / 32;
  // panel column j of the working matrix: element i at colp[i] (global) or sP (shifted by j0)
  auto colp = [&](int j) -> double * {
    if constexpr (SM) return sP + (j - j0) * pr - j0;
    else return A + (long long)j * lda;
  };
  // ---- panel factorisation (unblocked, Householder per column) with a
  //      one-column lookahead: warp 0 owns column j+1 — it applies reflector j
  //      to it and immediately forms reflector j+1 while the other warps
  //      update the rest of the panel, so each column costs one block barrier
  //      and the reflector formation is off the critical path of the update.
  // per-lane strided loops over rows lo..m-1 with four independent chains, so the
  // shared-memory loads of one lane overlap (the column step is a latency chain)
  auto dot_rows = [&](const double *a, const double *b, int lo) -> double {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int i = lo + lane;
    for (; i + 96 < m; i += 128) {
      s0 = fma(a[i], b[i], s0);
      s1 = fma(a[i + 32], b[i + 32], s1);
      s2 = fma(a[i + 64], b[i + 64], s2);
      s3 = fma(a[i + 96], b[i + 96], s3);
    }
    for (; i < m; i += 32) s0 = fma(a[i], b[i], s0);
    return (s0 + s1) + (s2 + s3);
  };
  auto axpy_rows = [&](double *y, const double *x, double a, int lo) {
    int i = lo + lane;
    for (; i + 96 < m; i += 128) {
      const double x0 = x[i], x1 = x[i + 32], x2 = x[i + 64], x3 = x[i + 96];
      y[i] = fma(-a, x0, y[i]);
      y[i + 32] = fma(-a, x1, y[i + 32]);
      y[i + 64] = fma(-a, x2, y[i + 64]);
      y[i + 96] = fma(-a, x3, y[i + 96]);
    }
    for (; i < m; i += 32) y[i] = fma(-a, x[i], y[i]);
  };
  auto form_reflector = [&](int j, int slot) {   // warp 0 only; column j already up to date
    double *col = colp(j);
    const double sigma = warp_sum(dot_rows(col, col, j + 1));
    const double alpha = col[j];
    double tau = 0.0, scal = 0.0, beta = alpha;
    // a column whose squared norm is below 1e-200 is numerically zero: no
    // reflection (tau = 0).  Without this guard, exactly rank-deficient sparse
    // inputs (e.g. the index-forwarding TT of Alg. 1, matrices with a few
    // scattered nonzero rows) drive the trailing columns geometrically towards
    // the subnormal range, where alpha and sigma keep only a few significant
    // bits and tau no longer matches v (measured: Q orthogonality 4e-2 at 256
    // columns); LAPACK's dlarfg rescales by safmin for the same reason
    if (sigma > 0.0 && fma(alpha, alpha, sigma) > 1e-200) {
      // dlarfg with beta = -sign(alpha) ||x||: tau = (beta - alpha) / beta =
      // 1 + |alpha| / ||x||, 1 / (alpha - beta) = sign(alpha) / (|alpha| + ||x||);
      // one rsqrt and one reciprocal instead of sqrt + two divisions on the
      // per-column critical path
      const double ss = fma(alpha, alpha, sigma);
      const double rs = rsqrt(ss);
      const double nrm = ss * rs, aa = fabs(alpha);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = fma(aa, rs, 1.0);
      const double q = __drcp_rn(aa + nrm);
      scal = alpha >= 0.0 ? q : -q;
    }
    if (tau != 0.0) {
      int i = j + 1 + lane;
      for (; i + 96 < m; i += 128) {
        col[i] *= scal;
        col[i + 32] *= scal;
        col[i + 64] *= scal;
        col[i + 96] *= scal;
      }
      for (; i < m; i += 32) col[i] *= scal;
    }
    __syncwarp();
    if (lane == 0) {
      col[j] = beta;
      s_tau[slot] = tau;
      g.tau[j] = tau;
    }
    __syncwarp();
  };
  constexpr int PANEL_MR = 9;
  const bool regpanel = SM && pr <= 32 * PANEL_MR;
  if (regpanel) qr_panel_reg<PANEL_MR>(g, j0, jb, pr, sP, s_tau);
  if (!regpanel && warp == 0) form_reflector(j0, 0);
  __syncthreads();
  for (int jj = 0; jj < (regpanel ? 0 : jb); ++jj) {
    const int j = j0 + jj;
    const double *col = colp(j);
    const double tau = s_tau[jj & 1];
    if (tau != 0.0) {
      for (int c = j + 1 + warp; c < j0 + jb; c += NW) {
        double *cc = colp(c);
        // w = tau v^T cc with v = (1, col[j+1..m-1])
        const double w = warp_sum(dot_rows(col, cc, j + 1) + (lane == 0 ? cc[j] : 0.0)) * tau;
        if (lane == 0) cc[j] -= w;
        axpy_rows(cc, col, w, j + 1);
      }
    }
    if (warp == 0 && jj + 1 < jb) {
      __syncwarp();
      form_reflector(j + 1, (jj + 1) & 1);
    }
    __syncthreads();
  }
  // ---- T factor (larft, forward, columnwise): T upper triangular jb x jb
  //      G[l][i] = v_l^T v_i for l < i: the upper 8x8 tiles of V^T V on the
  //      FP64 tensor pipe (one warp per tile, rows over the k-steps)
  {
    const double *V = SM ? sP : A + j0 + (long long)j0 * lda;
    const int ldv = SM ? pr : (int)lda, mr = m - j0, q4 = lane & 3, g8 = lane >> 2;
    auto vm = [&](int rr, int l) -> double {
      if (l >= jb || rr >= mr || rr < l) return 0.0;
      return rr == l ? 1.0 : V[rr + l * ldv];
    };
    const int nt = (jb + 7) >> 3;
    for (int t = warp; t < nt * nt; t += NW) {
      const int ti = t % nt, tj = t / nt;
      if (ti > tj) continue;
      double d0 = 0.0, d1 = 0.0;
      int r0 = 0;
      for (; r0 < 32 && r0 < mr; r0 += 4) dmma_f64(d0, d1, vm(r0 + q4, 8 * ti + g8), vm(r0 + q4, 8 * tj + g8));
      if (jb == NB)
        for (; r0 + 4 <= mr; r0 += 4) {
          const double *vp = V + r0 + q4;
          dmma_f64(d0, d1, vp[(8 * ti + g8) * ldv], vp[(8 * tj + g8) * ldv]);
        }
      for (; r0 < mr; r0 += 4) dmma_f64(d0, d1, vm(r0 + q4, 8 * ti + g8), vm(r0 + q4, 8 * tj + g8));
      const int l = 8 * ti + g8, i0 = 8 * tj + 2 * q4;
      if (l < i0 && i0 < jb) sG[l][i0] = d0;
      if (l < i0 + 1 && i0 + 1 < jb) sG[l][i0 + 1] = d1;
    }
  }
}

#ifdef QR_PHASE_TIMING
#define QR_PH(i) do { if (threadIdx.x == 0) { const long long t_ = clock64(); qph[i] += t_ - qtc; qtc = t_; } } while (0)
#else
#define QR_PH(i) do { } while (0)
#endif
__global__ void __launch_bounds__(QR_THREADS) qr_kernel(const QRDesc *__restrict__ descs) {
  const QRDesc g = descs[blockIdx.x];
#ifdef QR_PHASE_TIMING
  long long qph[6] = {0, 0, 0, 0, 0, 0};
  long long qtc = clock64();
#endif
  const int m = g.m, n = g.n, kmin = min(m, n);
  if (threadIdx.x == 0) {
    // geqrf: 2 m n k - (m + n) k^2 + 2/3 k^3 ; orgqr (explicit Q, m x k): 4 m k^2 - 4/3 k^3 (LAPACK counts)
    const double M = m, N = n, K = kmin;
    double f = 2.0 * M * N * K - (M + N) * K * K + 2.0 / 3.0 * K * K * K;
    if (g.Q) f += 4.0 * M * K * K - 4.0 / 3.0 * K * K * K;
    atomicAdd(&g_linalg_flops[0], (unsigned long long)(f > 0 ? f : 0));
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ double sT[NB][NB + 1];
  __shared__ double sG[NB][NB + 1];
  __shared__ double s_tau[2];
  double *A = g.A;
  const long long lda = g.lda;
  // copy input into the working matrix
  for (long long e = tid; e < (long long)m * n; e += QR_THREADS) {
    const int r = (int)(e % m), c = (int)(e / m);
    A[r + c * lda] = g.src[r * g.src_rs + c * g.src_cs];
  }
  __syncthreads();

  extern __shared__ double sP[];   // panel copy (rows j0..m-1) when it fits
  QR_PH(0);
  for (int j0 = 0; j0 < kmin; j0 += NB) {
    const int jb = min(NB, kmin - j0);
    const int pr = m - j0;                           // panel rows
    const bool in_smem = pr <= QR_PANEL_ROWS;
    if (in_smem) {
      for (int e = tid; e < pr * jb; e += QR_THREADS) {
        const int r = e % pr, l = e / pr;
        sP[r + l * pr] = A[j0 + r + (long long)(j0 + l) * lda];
      }
      __syncthreads();
    }
    if (in_smem) qr_panel<true>(g, m, j0, jb, pr, A, lda, sP, s_tau, sG);
    else qr_panel<false>(g, m, j0, jb, pr, A, lda, sP, s_tau, sG);
    QR_PH(1);
    for (int e = tid; e < NB * (NB + 1); e += QR_THREADS) (&sT[0][0])[e] = 0.0;
    __syncthreads();
    if (warp == 0) {
      for (int i = 0; i < jb; ++i) {
        const double ti = g.tau[j0 + i];
        // T[c][i] = -tau_i * sum_{l=c}^{i-1} T[c][l] G[l][i]
        double v = 0.0;
        if (lane < i) {
          // four independent chains: the loads pipeline instead of waiting on one fma chain
          double v1 = 0.0, v2 = 0.0, v3 = 0.0;
          int l = lane;
          for (; l + 3 < i; l += 4) {
            v = fma(sT[lane][l], sG[l][i], v);
            v1 = fma(sT[lane][l + 1], sG[l + 1][i], v1);
            v2 = fma(sT[lane][l + 2], sG[l + 2][i], v2);
            v3 = fma(sT[lane][l + 3], sG[l + 3][i], v3);
          }
          for (; l < i; ++l) v = fma(sT[lane][l], sG[l][i], v);
          v = (v + v1) + (v2 + v3);
          v = -ti * v;
        }
        __syncwarp();
        if (lane < i) sT[lane][i] = v;
        if (lane == 0) sT[i][i] = ti;
        __syncwarp();
      }
    }
    __syncthreads();
    if (in_smem) {   // panel back to the working matrix (V below the diagonal, R on/above)
      for (int e = tid; e < pr * jb; e += QR_THREADS) {
        const int r = e % pr, l = e / pr;
        A[j0 + r + (long long)(j0 + l) * lda] = sP[r + l * pr];
      }
      __syncthreads();
    }
    // keep T for the Q formation
    double *Tg = g.T + (long long)(j0 / NB) * NB * NB;
    for (int e = tid; e < NB * NB; e += QR_THREADS) Tg[e] = sT[e % NB][e / NB];
    __syncthreads();
    QR_PH(2);
    // ---- trailing update: A[:, j0+jb:n] <- (I - V T V^T)^T A = A - V T^T (V^T A)
    if (j0 + jb < n)
      if (in_smem) apply_block_reflector<true>(m, j0, jb, sP, pr, sT, 1, A, 1, lda, j0 + jb, n);
      else apply_block_reflector<false>(m, j0, jb, A + j0 + (long long)j0 * lda, (int)lda, sT, 1, A, 1, lda, j0 + jb,
                                        n);
    __syncthreads();
  }
  QR_PH(3);
  // ---- R
  if (g.R) {
    for (long long e = tid; e < (long long)kmin * n; e += QR_THREADS) {
      const int r = (int)(e % kmin), c = (int)(e / kmin);
      const double v = (c >= r) ? A[r + c * lda] : 0.0;
      if (g.rt) g.R[c + r * g.ldr] = v;
      else g.R[r + c * g.ldr] = v;
    }
  }
  // ---- explicit Q = H_1 ... H_k [I; 0]  (orgqr, backward over panels)
  if (g.Q) {
    for (long long e = tid; e < (long long)m * kmin; e += QR_THREADS) {
      const int r = (int)(e % m), c = (int)(e / m);
      g.Q[r * g.q_rs + c * g.q_cs] = (r == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    const int npan = (kmin + NB - 1) / NB;
    for (int pnl = npan - 1; pnl >= 0; --pnl) {
      const int j0 = pnl * NB, jb = min(NB, kmin - j0);
      const double *Tg = g.T + (long long)pnl * NB * NB;
      for (int e = tid; e < NB * NB; e += QR_THREADS) sT[e % NB][e / NB] = Tg[e];
      const int pr = m - j0;
      const bool in_smem = pr <= QR_PANEL_ROWS;
      if (in_smem)
        for (int e = tid; e < pr * jb; e += QR_THREADS) {
          const int r = e % pr, l = e / pr;
          sP[r + l * pr] = A[j0 + r + (long long)(j0 + l) * lda];
        }
      __syncthreads();
      if (in_smem) apply_block_reflector<true>(m, j0, jb, sP, pr, sT, 0, g.Q, g.q_rs, g.q_cs, j0, kmin);
      else apply_block_reflector<false>(m, j0, jb, A + j0 + (long long)j0 * lda, (int)lda, sT, 0, g.Q, g.q_rs,
                                        g.q_cs, j0, kmin);
      __syncthreads();
    }
  }
#ifdef QR_PHASE_TIMING
  QR_PH(4);
  if (threadIdx.x == 0) printf("QRPH %d %d %d %lld %lld %lld %lld %lld\n", m, n, g.Q ? 1 : 0, qph[0], qph[1], qph[2], qph[3], qph[4]);
#endif
}

// ------------------------------------------------------------ Jacobi SVD ---
// |ga| <= tol sqrt(al be) with one square root (two when al be over/underflows);
// the FP64 sqrt/div sequences are the cost of a latency-bound Jacobi round
__device__ __forceinline__ bool jacobi_orthogonal(double al, double be, double ga, double tol) {
  const double pr = al * be;
  if (pr > 0.0 && pr < 1e300) return ga * ga <= (tol * tol) * pr;   // |ga| <= sqrt(pr) < 1e150: no overflow
  return fabs(ga) <= tol * sqrt(al) * sqrt(be);
}

__device__ void jacobi_core(int m, int p, double *W, long long ldw, double *V, long long ldv, double *s_sig,
                            int *s_pos, int *flag, int *sweeps_out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NW = blockDim.x >> 5;
  const int P2 = p + (p & 1);  // even number of players (a phantom player is skipped)
  const double tol = 4.0 * DBL_EPSILON;
  unsigned long long fl = 0;   // flop count, one atomic per warp at the end (not per rotation)
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    if (tid == 0) *flag = 0;
    __syncthreads();
    for (int rnd = 0; rnd < P2 - 1; ++rnd) {
      for (int pr = warp; pr < P2 / 2; pr += NW) {
        int a, b;
        if (pr == 0) {
          a = P2 - 1;
          b = rnd;
        } else {
          a = (rnd + pr) % (P2 - 1);
          b = (rnd - pr + (P2 - 1)) % (P2 - 1);
        }
        if (a >= p || b >= p) continue;
        if (a > b) { int t = a; a = b; b = t; }
        double *wa = W + (long long)a * ldw, *wb = W + (long long)b * ldw;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int r = lane; r < m; r += 32) {
          const double x = wa[r], y = wb[r];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (ga == 0.0 || al == 0.0 || be == 0.0) continue;
        fl += 6ull * m;
        if (jacobi_orthogonal(al, be, ga, tol)) continue;
        fl += 6ull * (m + p);
        const double zeta = (be - al) * __drcp_rn(2.0 * ga);
        const double tr = __drcp_rn(fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        const double t = zeta >= 0.0 ? tr : -tr;
        const double c = rsqrt(fma(t, t, 1.0)), s = c * t;
        for (int r = lane; r < m; r += 32) {
          const double x = wa[r], y = wb[r];
          wa[r] = c * x - s * y;
          wb[r] = s * x + c * y;
        }
        if (V) {
          double *va = V + (long long)a * ldv, *vb = V + (long long)b * ldv;
          for (int r = lane; r < p; r += 32) {
            const double x = va[r], y = vb[r];
            va[r] = c * x - s * y;
            vb[r] = s * x + c * y;
          }
        }
        if (lane == 0) *flag = 1;
      }
      __syncthreads();
    }
    if (*flag == 0) break;
    __syncthreads();
  }
  if (tid == 0 && sweeps_out) *sweeps_out = sweep + 1;
  if (lane == 0 && fl) atomicAdd(&g_linalg_flops[1], fl);
  // singular values = column norms
  for (int c = warp; c < p; c += NW) {
    const double *w = W + (long long)c * ldw;
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s = fma(w[r], w[r], s);
    s = warp_sum(s);
    if (lane == 0) s_sig[c] = sqrt(s);
  }
  __syncthreads();
  // rank sort: position of column i in decreasing order (ties by index)
  for (int i = tid; i < p; i += blockDim.x) {
    const double si = s_sig[i];
    int pos = 0;
    for (int j = 0; j < p; ++j) {
      const double sj = s_sig[j];
      pos += (sj > si) || (sj == si && j < i);
    }
    s_pos[i] = pos;
  }
  __syncthreads();
}

template <bool SMEM>
__global__ void __launch_bounds__(1024) jacobi_kernel(const SVDDesc *__restrict__ descs) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ int s_flag;
  const SVDDesc g = descs[blockIdx.x];
  const int m = g.m, p = g.p, tid = threadIdx.x;
  const bool wantv = g.V != nullptr;   // V == nullptr: left vectors and sigma only
  double *W, *V;
  long long ldw, ldv;
  double *s_sig;
  int *s_pos;
  if (SMEM) {
    W = dsm;
    ldw = m;
    V = wantv ? dsm + (long long)m * p : nullptr;
    ldv = p;
    s_sig = dsm + (long long)m * p + (wantv ? (long long)p * p : 0);
    s_pos = reinterpret_cast<int *>(s_sig + p);
  } else {
    W = g.work;
    ldw = m;
    V = wantv ? g.work + (long long)m * p : nullptr;
    ldv = p;
    s_sig = dsm;
    s_pos = reinterpret_cast<int *>(dsm + p);
  }
  for (long long e = tid; e < (long long)m * p; e += blockDim.x) {
    const int r = (int)(e % m), c = (int)(e / m);
    W[r + c * ldw] = g.W[r + c * g.ldw];
  }
  if (wantv)
    for (long long e = tid; e < (long long)p * p; e += blockDim.x) {
      const int r = (int)(e % p), c = (int)(e / p);
      V[r + c * ldv] = (r == c) ? 1.0 : 0.0;
    }
  __syncthreads();
  jacobi_core(m, p, W, ldw, V, ldv, s_sig, s_pos, &s_flag, g.sweeps_out);
  // sorted outputs
  for (long long e = tid; e < (long long)m * p; e += blockDim.x) {
    const int r = (int)(e % m), c = (int)(e / m);
    const double sc = s_sig[c];
    g.U[r + (long long)s_pos[c] * g.ldu] = sc > 0.0 ? W[r + c * ldw] / sc : 0.0;
  }
  if (wantv)
    for (long long e = tid; e < (long long)p * p; e += blockDim.x) {
      const int r = (int)(e % p), c = (int)(e / p);
      g.V[r + (long long)s_pos[c] * g.ldv] = V[r + c * ldv];
    }
  for (int c = tid; c < p; c += blockDim.x) g.sigma[s_pos[c]] = s_sig[c];
}

// ------------------------------------ cluster Jacobi (distributed shared memory) ---
// One-sided Jacobi as a systolic array (Brent & Luk 1985) over a thread-block
// cluster: every warp of the cluster owns the two columns of one pair of the
// round-robin tournament and keeps them (W part and V part) in REGISTERS; after
// its rotation it writes the two rotated columns straight into the mailboxes of
// the warps that own them in the next round (top row moves right, bottom row
// moves left: distributed shared memory when the neighbour sits in another
// CTA), one hardware cluster barrier, and every warp reads its own (local)
// mailbox.  A round is then register arithmetic + one store + one barrier + one
// local load; the first cluster version kept the columns in place in shared
// memory and read AND wrote both (mostly remote) columns of a pair every round:
// two distributed-shared-memory latencies per round, 1.78 us per round at
// p = 136 against ~1 us now.  Mailboxes are double buffered by round parity.
// Dummy columns (id < 0) pad the tournament to 2 x (active warps); column
// identity does not matter for the result (sigma, U, V are sorted at the end).
// One cluster per problem (grid = count x C).  Same rotation and convergence
// test as jacobi_core.
constexpr int JC_MAXC = 16;
constexpr int JC_R = 10;   // rows per lane held in registers: m, p <= 320 (instantiated for 5 and 10: the
                           // C4 bonds, m = p <= 136, need half the registers and instructions)
template <int JR>
__global__ void __launch_bounds__(512) jacobi_cluster_kernel(const SVDDesc *__restrict__ descs, int C) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double jsm[];
  __shared__ int s_flag;
  const int rank = (int)cl.block_rank();
  const SVDDesc g = descs[blockIdx.x / C];
  const int m = g.m, p = g.p, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NW = blockDim.x >> 5;
  const bool wantv = g.V != nullptr;
  const int pairs = (p + 1) / 2;
  int nw = (pairs + C - 1) / C;                 // active warps per CTA for this problem
  nw = nw < 1 ? 1 : (nw > NW ? NW : nw);
  const int NWT = nw * C, P2 = 2 * NWT;         // players of the tournament (>= p)
  const int cl_len = m + p;                     // a column: W part then V part
  // mailbox [parity][warp][slot 0 = top, 1 = bottom][m + p], ids alongside
  double *mb = jsm;
  int *mbid = reinterpret_cast<int *>(mb + (size_t)4 * NW * cl_len);   // [parity][warp][slot]
  double *sig = reinterpret_cast<double *>(mbid + 4 * NW + (4 * NW & 1));   // p
  int *pos = reinterpret_cast<int *>(sig + p);                           // p
  auto box = [&](int par, int w, int slot) -> double * { return mb + ((size_t)(par * NW + w) * 2 + slot) * cl_len; };
  auto boxid = [&](int par, int w, int slot) -> int * { return mbid + (par * NW + w) * 2 + slot; };
  const bool active = warp < nw;
  const int gw = rank * nw + warp;              // position of this warp's pair in the systolic row
  // columns of this warp: top = position gw, bottom = position P2 - 1 - gw
  double xa[JR], xb[JR], ya[JR], yb[JR];
  int ida = -1, idb = -1;
  if (active) {
    const int ca = gw, cb = P2 - 1 - gw;
    ida = ca < p ? ca : -1;
    idb = cb < p ? cb : -1;
#pragma unroll
    for (int q = 0; q < JR; ++q) {
      const int r = lane + 32 * q;
      xa[q] = (ida >= 0 && r < m) ? g.W[r + (long long)ca * g.ldw] : 0.0;
      xb[q] = (idb >= 0 && r < m) ? g.W[r + (long long)cb * g.ldw] : 0.0;
      ya[q] = (wantv && r == ida) ? 1.0 : 0.0;
      yb[q] = (wantv && r == idb) ? 1.0 : 0.0;
    }
  }
  // destinations of the rotation (fixed for the whole run): top -> top of gw + 1 (the last
  // warp's top turns into its own bottom, warp 0's top stays), bottom -> bottom of gw - 1
  // (warp 0's bottom becomes the top of warp 1)
  int dta = gw, dsa = 0, dtb = gw, dsb = 1;     // (warp, slot) for the top and the bottom column
  if (NWT > 1) {
    if (gw == 0) { dta = 0; dsa = 0; dtb = 1; dsb = 0; }
    else {
      if (gw == NWT - 1) { dta = gw; dsa = 1; } else { dta = gw + 1; dsa = 0; }
      dtb = gw - 1; dsb = 1;
    }
  }
  if (tid == 0) s_flag = 0;
  cl.sync();
  const double tol = 4.0 * DBL_EPSILON;
  unsigned long long fl = 0;
  int sweep = 0, par = 0;
  for (; sweep < 60; ++sweep) {
    for (int rnd = 0; rnd < P2 - 1; ++rnd) {
      if (active) {
        if (ida >= 0 && idb >= 0) {
          double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
          for (int q = 0; q < JR; ++q) {
            al = fma(xa[q], xa[q], al);
            be = fma(xb[q], xb[q], be);
            ga = fma(xa[q], xb[q], ga);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {   // three interleaved butterflies
            al += __shfl_xor_sync(0xffffffffu, al, o);
            be += __shfl_xor_sync(0xffffffffu, be, o);
            ga += __shfl_xor_sync(0xffffffffu, ga, o);
          }
          if (ga != 0.0 && al != 0.0 && be != 0.0) {
            fl += 6ull * m;
            if (!jacobi_orthogonal(al, be, ga, tol)) {
              fl += 6ull * (m + p);
              const double zeta = (be - al) * __drcp_rn(2.0 * ga);
              const double tr = __drcp_rn(fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
              const double t = zeta >= 0.0 ? tr : -tr;
              const double c = rsqrt(fma(t, t, 1.0)), sn = c * t;
#pragma unroll
              for (int q = 0; q < JR; ++q) {
                const double x = xa[q], y = xb[q];
                xa[q] = c * x - sn * y;
                xb[q] = sn * x + c * y;
                const double u = ya[q], v = yb[q];
                ya[q] = c * u - sn * v;
                yb[q] = sn * u + c * v;
              }
              if (lane == 0) s_flag = 1;
            }
          }
        }
        // send both columns to their next owners
        double *da = cl.map_shared_rank(box(par, dta % nw, dsa), dta / nw);
        double *db = cl.map_shared_rank(box(par, dtb % nw, dsb), dtb / nw);
#pragma unroll
        for (int q = 0; q < JR; ++q) {
          const int r = lane + 32 * q;
          if (r < m) { da[r] = xa[q]; db[r] = xb[q]; }
          if (wantv && r < p) { da[m + r] = ya[q]; db[m + r] = yb[q]; }
        }
        if (lane == 0) {
          *cl.map_shared_rank(boxid(par, dta % nw, dsa), dta / nw) = ida;
          *cl.map_shared_rank(boxid(par, dtb % nw, dsb), dtb / nw) = idb;
        }
      }
      cl.sync();
      if (active) {
        const double *ra = box(par, warp, 0), *rb = box(par, warp, 1);
        ida = *boxid(par, warp, 0);
        idb = *boxid(par, warp, 1);
#pragma unroll
        for (int q = 0; q < JR; ++q) {
          const int r = lane + 32 * q;
          xa[q] = r < m ? ra[r] : 0.0;
          xb[q] = r < m ? rb[r] : 0.0;
          ya[q] = (wantv && r < p) ? ra[m + r] : 0.0;
          yb[q] = (wantv && r < p) ? rb[m + r] : 0.0;
        }
      }
      par ^= 1;
    }
    // any rotation in the cluster this sweep?
    int any = 0;
    for (int q = 0; q < C; ++q) any |= *cl.map_shared_rank(&s_flag, q);
    cl.sync();
    if (tid == 0) s_flag = 0;
    if (!any) break;
    cl.sync();
  }
  if (lane == 0 && fl) atomicAdd(&g_linalg_flops[1], fl);
  if (rank == 0 && tid == 0 && g.sweeps_out) *g.sweeps_out = sweep + 1;
  // sigma of this warp's columns, pushed into every CTA's table, then the rank sort
  cl.sync();
  if (active) {
    double sa = 0.0, sb = 0.0;
#pragma unroll
    for (int q = 0; q < JR; ++q) { sa = fma(xa[q], xa[q], sa); sb = fma(xb[q], xb[q], sb); }
    sa = warp_sum(sa);
    sb = warp_sum(sb);
    if (lane < C) {
      double *rs = cl.map_shared_rank(sig, lane);
      if (ida >= 0) rs[ida] = sqrt(sa);
      if (idb >= 0) rs[idb] = sqrt(sb);
    }
  }
  cl.sync();
  for (int i = tid; i < p; i += blockDim.x) {
    const double si = sig[i];
    int ps = 0;
    for (int j = 0; j < p; ++j) {
      const double sj = sig[j];
      ps += (sj > si) || (sj == si && j < i);
    }
    pos[i] = ps;
  }
  __syncthreads();
  if (active) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int id = h == 0 ? ida : idb;
      if (id < 0) continue;
      const double sc = sig[id];
      const double inv = sc > 0.0 ? 1.0 / sc : 0.0;
      const long long cu = (long long)pos[id] * g.ldu, cv = (long long)pos[id] * g.ldv;
#pragma unroll
      for (int q = 0; q < JR; ++q) {
        const int r = lane + 32 * q;
        const double x = h == 0 ? xa[q] : xb[q];
        if (r < m) g.U[r + cu] = sc > 0.0 ? x * inv : 0.0;
        if (wantv && r < p) g.V[r + cv] = h == 0 ? ya[q] : yb[q];
      }
    }
  }
  if (rank == 0)
    for (int c = tid; c < p; c += blockDim.x) g.sigma[pos[c]] = sig[c];
}

// ------------------------------------------- block Jacobi across a grid ---
// One-sided block Jacobi for larger p: the p columns form nb blocks of JB
// columns; each round pairs blocks by a round-robin tournament and every CTA
// orthogonalises its 2 JB columns (plus the matching V columns) in shared
// memory with one inner Jacobi pass; a software grid barrier separates rounds
// (the grid is launched cooperatively, so all CTAs are co-resident).
constexpr int JB = 4;   // measured: 4 > 8 > 2 > 16 on C2 (instances/s 5.29, 5.16, 5.11, 4.20)
constexpr int BJ_THREADS = 256;

__device__ void grid_barrier(unsigned int *bar, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int *gen = bar + 1;
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      const long long t0 = clock64();
      while (*gen == g) {
        if (clock64() - t0 > 8000000000LL) __trap();   // never hang the device (~4 s)
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(BJ_THREADS) jacobi_block_kernel(const SVDDesc *__restrict__ descs, unsigned int *bar,
                                                                  int *flag) {
  extern __shared__ __align__(16) double sm[];
  const SVDDesc g = descs[0];
  const int m = g.m, p = g.p, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = BJ_THREADS / 32;
  const int nb = (p + JB - 1) / JB;
  const int NB2 = nb + (nb & 1);
  const unsigned int G = gridDim.x;
  double *W = g.work;                       // m x p, ld m
  double *V = g.work + (long long)m * p;    // p x p, ld p
  double *sW = sm;                          // m x 2JB
  double *sV = sm + (long long)m * 2 * JB;  // p x 2JB
  // LAPACK dgesvj's convergence threshold sqrt(m) eps: within-block pairs are
  // revisited nb-1 times per sweep, so a tighter threshold only adds rotations
  // of noise-level pairs (and their roundoff).
  const double tol = fmax(4.0, sqrt((double)m)) * DBL_EPSILON;
  unsigned long long fl = 0;   // flop count, one atomic per warp at the end
  // init (grid-strided)
  for (long long e = blockIdx.x * (long long)BJ_THREADS + tid; e < (long long)m * p; e += (long long)G * BJ_THREADS) {
    const int r = (int)(e % m), c = (int)(e / m);
    W[e] = g.W[r + c * g.ldw];
  }
  const bool wantv = g.V != nullptr;
  if (wantv)
    for (long long e = blockIdx.x * (long long)BJ_THREADS + tid; e < (long long)p * p; e += (long long)G * BJ_THREADS)
      V[e] = ((e % p) == (e / p)) ? 1.0 : 0.0;
  if (blockIdx.x == 0 && tid == 0) *flag = 0;
  grid_barrier(bar, G);
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    for (int rnd = 0; rnd < NB2 - 1; ++rnd) {
      for (int pr = blockIdx.x; pr < NB2 / 2; pr += G) {
        int A, B;
        if (pr == 0) { A = NB2 - 1; B = rnd; }
        else { A = (rnd + pr) % (NB2 - 1); B = (rnd - pr + (NB2 - 1)) % (NB2 - 1); }
        // gather the 2JB columns (phantom / out-of-range columns become empty)
        int col[2 * JB];
#pragma unroll
        for (int q = 0; q < JB; ++q) {
          const int ca = A * JB + q, cb = B * JB + q;
          col[q] = (A < nb && ca < p) ? ca : -1;
          col[JB + q] = (B < nb && cb < p) ? cb : -1;
        }
        for (int e = tid; e < m * 2 * JB; e += BJ_THREADS) {
          const int r = e % m, q = e / m;
          sW[e] = col[q] >= 0 ? W[r + (long long)col[q] * m] : 0.0;
        }
        if (wantv)
          for (int e = tid; e < p * 2 * JB; e += BJ_THREADS) {
            const int r = e % p, q = e / p;
            sV[e] = col[q] >= 0 ? V[r + (long long)col[q] * p] : 0.0;
          }
        __syncthreads();
        // one inner pass over all pairs of the 2JB columns (round robin, one warp per pair)
        int rotated = 0;
        for (int ir = 0; ir < 2 * JB - 1; ++ir) {
          for (int ip = warp; ip < JB; ip += NW) {
            int a, b;
            if (ip == 0) { a = 2 * JB - 1; b = ir; }
            else { a = (ir + ip) % (2 * JB - 1); b = (ir - ip + (2 * JB - 1)) % (2 * JB - 1); }
            if (col[a] < 0 || col[b] < 0) continue;
            if (col[a] > col[b]) { int t = a; a = b; b = t; }
            double *wa = sW + (long long)a * m, *wb = sW + (long long)b * m;
            double al = 0.0, be = 0.0, ga = 0.0;
            for (int r = lane; r < m; r += 32) {
              const double x = wa[r], y = wb[r];
              al = fma(x, x, al); be = fma(y, y, be); ga = fma(x, y, ga);
            }
            al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
            fl += 6ull * m;
            if (ga == 0.0 || al == 0.0 || be == 0.0) continue;
            if (jacobi_orthogonal(al, be, ga, tol)) continue;
            const double zeta = (be - al) * __drcp_rn(2.0 * ga);
            const double tr = __drcp_rn(fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
            const double t = zeta >= 0.0 ? tr : -tr;
            const double c = rsqrt(fma(t, t, 1.0)), s = c * t;
            for (int r = lane; r < m; r += 32) {
              const double x = wa[r], y = wb[r];
              wa[r] = c * x - s * y; wb[r] = s * x + c * y;
            }
            if (wantv) {
              double *va = sV + (long long)a * p, *vb = sV + (long long)b * p;
              for (int r = lane; r < p; r += 32) {
                const double x = va[r], y = vb[r];
                va[r] = c * x - s * y; vb[r] = s * x + c * y;
              }
            }
            rotated = 1;
            fl += 6ull * (m + p);
          }
          __syncthreads();
        }
        if (__syncthreads_or(rotated) && tid == 0) *flag = 1;
        for (int e = tid; e < m * 2 * JB; e += BJ_THREADS) {
          const int r = e % m, q = e / m;
          if (col[q] >= 0) W[r + (long long)col[q] * m] = sW[e];
        }
        if (wantv)
          for (int e = tid; e < p * 2 * JB; e += BJ_THREADS) {
            const int r = e % p, q = e / p;
            if (col[q] >= 0) V[r + (long long)col[q] * p] = sV[e];
          }
        __syncthreads();
      }
      grid_barrier(bar, G);
    }
    const int f = *(volatile int *)flag;
    grid_barrier(bar, G);
    if (f == 0) break;
    if (blockIdx.x == 0 && tid == 0) *flag = 0;
    grid_barrier(bar, G);
  }
  if (lane == 0 && fl) atomicAdd(&g_linalg_flops[1], fl);
  if (blockIdx.x != 0) return;
  if (tid == 0 && g.sweeps_out) *g.sweeps_out = sweep + 1;
  // sigma, sort, outputs (CTA 0)
  double *s_sig = sm;
  int *s_pos = reinterpret_cast<int *>(sm + p);
  for (int c = warp; c < p; c += NW) {
    const double *w = W + (long long)c * m;
    double s = 0.0;
    for (int r = lane; r < m; r += 32) s = fma(w[r], w[r], s);
    s = warp_sum(s);
    if (lane == 0) s_sig[c] = sqrt(s);
  }
  __syncthreads();
  for (int i = tid; i < p; i += BJ_THREADS) {
    const double si = s_sig[i];
    int pos = 0;
    for (int j = 0; j < p; ++j) {
      const double sj = s_sig[j];
      pos += (sj > si) || (sj == si && j < i);
    }
    s_pos[i] = pos;
  }
  __syncthreads();
  for (long long e = tid; e < (long long)m * p; e += BJ_THREADS) {
    const int r = (int)(e % m), c = (int)(e / m);
    const double sc = s_sig[c];
    g.U[r + (long long)s_pos[c] * g.ldu] = sc > 0.0 ? W[e] / sc : 0.0;
  }
  if (wantv)
    for (long long e = tid; e < (long long)p * p; e += BJ_THREADS) {
      const int r = (int)(e % p), c = (int)(e / p);
      g.V[r + (long long)s_pos[c] * g.ldv] = V[e];
    }
  for (int c = tid; c < p; c += BJ_THREADS) g.sigma[s_pos[c]] = s_sig[c];
}

}  // namespace

void linalg_counters(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, g_linalg_flops, sizeof(g_linalg_flops));
  if (reset) {
    unsigned long long z[2] = {0, 0};
    cudaMemcpyToSymbol(g_linalg_flops, z, sizeof(z));
  }
}

tt_status launch_qr(const QRDesc *descs_dev, int count, cudaStream_t s) {
  if (count <= 0) return TT_OK;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QR_PANEL_SMEM);
    attr = true;
  }
  qr_kernel<<<count, QR_THREADS, QR_PANEL_SMEM, s>>>(descs_dev);
  return check_launch("qr");
}

// one warp per column pair of a round: p/2 pairs -> up to 32 warps
static int svd_threads(int pcap) {
  int w = (pcap + 1) / 2;
  w = w < 2 ? 2 : (w > 32 ? 32 : w);
  return 32 * w;
}

struct BJSync {
  unsigned int *bar = nullptr;
  int *flag = nullptr;
};
static thread_local BJSync g_bj;

static size_t svd_smem_bytes(int mcap, int pcap, bool wantv) {
  return ((size_t)mcap * pcap + (wantv ? (size_t)pcap * pcap : 0) + pcap) * sizeof(double) +
         (size_t)pcap * sizeof(int) + 16;
}

// cluster Jacobi: the smallest cluster (2..16 CTAs) whose per-CTA share of W and
// V fits in shared memory; false if none does (or the launch is refused)
static bool cluster_jacobi(const SVDDesc *descs_dev, int count, int mcap, int pcap, size_t limit, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(jacobi_cluster_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)limit);
    cudaFuncSetAttribute(jacobi_cluster_kernel<5>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(jacobi_cluster_kernel<JC_R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)limit);
    cudaFuncSetAttribute(jacobi_cluster_kernel<JC_R>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  if (mcap > 32 * JC_R || pcap > 32 * JC_R) return false;
  const int pairs = (pcap + 1) / 2;
  // Cluster sizes in order of preference.  One problem (latency): the shortest modelled
  // SVD = rounds per sweep (2 C ceil(pairs / C) - 1 players: dummy columns pad the
  // tournament) x time per round, which grows with the warps per CTA (measured at
  // p = 132: 1.01 / 1.11 / 1.22 us per round at 6 / 9 / 11 warps => ~0.75 + 0.042 warps):
  // p = 132 runs on 11 CTAs x 6 warps (131 rounds, 1.05 ms) instead of 8 x 9 (143 rounds,
  // 1.27 ms).  Batched problems (throughput): the smallest power of two that fits, so as
  // many problems as possible are co-resident.
  int order[JC_MAXC + 1], no = 0;
  static int forced = -1;
  if (forced < 0) { const char *e = std::getenv("TT_JC_CLUSTER"); forced = e ? std::atoi(e) : 0; }
  if (count > 1) {
    for (int C = 2; C <= JC_MAXC; C *= 2) order[no++] = C;
  } else {
    for (int C = 2; C <= JC_MAXC; ++C) order[no++] = C;
    auto key = [&](int C) {
      const int nw = (pairs + C - 1) / C;
      return (long long)(2 * C * nw) * (18 + (nw < 2 ? 2 : nw));
    };
    for (int i = 1; i < no; ++i)
      for (int j = i; j > 0 && key(order[j]) < key(order[j - 1]); --j) {
        const int t = order[j]; order[j] = order[j - 1]; order[j - 1] = t;
      }
  }
  if (forced >= 2 && forced <= JC_MAXC) { order[0] = forced; no = 1; }
  for (int oi = 0; oi < no; ++oi) {
    const int C = order[oi];
    int warps = (pairs + C - 1) / C;
    warps = warps < 2 ? 2 : warps;
    // mailboxes [2 parities][warps][2 slots][m + p], their ids, sigma and the sort positions
    const size_t smem = (size_t)4 * warps * (mcap + pcap) * sizeof(double) + (size_t)(4 * warps + 2) * sizeof(int) +
                        (size_t)pcap * (sizeof(double) + sizeof(int)) + 16;
    if (smem > limit || warps > 16) continue;   // <= 512 threads
    const int threads = 32 * (warps < 2 ? 2 : warps);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(count * C);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const bool small = mcap <= 160 && pcap <= 160;
    if ((small ? cudaLaunchKernelEx(&cfg, jacobi_cluster_kernel<5>, descs_dev, C)
               : cudaLaunchKernelEx(&cfg, jacobi_cluster_kernel<JC_R>, descs_dev, C)) == cudaSuccess)
      return true;
    cudaGetLastError();
  }
  return false;
}

tt_status launch_jacobi(const SVDDesc *descs_dev, int count, int mcap, int pcap, cudaStream_t s) {
  if (count <= 0) return TT_OK;
  const size_t smem = svd_smem_bytes(mcap, pcap, true);
  const size_t limit = 220 * 1024;
  if (smem <= limit) {
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(jacobi_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)limit);
      attr_set = true;
    }
    jacobi_kernel<true><<<count, svd_threads(pcap), smem, s>>>(descs_dev);
  } else if (cluster_jacobi(descs_dev, count, mcap, pcap, limit, s)) {
    // one thread-block cluster per problem, columns in distributed shared memory
  } else if (count == 1 && g_bj.bar &&
             ((size_t)mcap + pcap) * 2 * JB * sizeof(double) <= limit) {
    // block Jacobi over a cooperative grid: one CTA per block pair
    const int nb = (pcap + JB - 1) / JB;
    const int G = (nb + (nb & 1)) / 2;
    size_t smb = ((size_t)mcap + pcap) * 2 * JB * sizeof(double);
    const size_t sort_b = (size_t)pcap * (sizeof(double) + sizeof(int)) + 16;
    smb = smb > sort_b ? smb : sort_b;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(jacobi_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)limit);
      attr = true;
    }
    cudaMemsetAsync(g_bj.bar, 0, 2 * sizeof(unsigned int) + sizeof(int) * 2, s);
    void *args[] = {(void *)&descs_dev, (void *)&g_bj.bar, (void *)&g_bj.flag};
    cudaError_t e = cudaLaunchCooperativeKernel((const void *)jacobi_block_kernel, dim3(G), dim3(BJ_THREADS), args,
                                                smb, s);
    if (e != cudaSuccess) return fail(TT_ERR_CUDA, std::string("jacobi_block: ") + cudaGetErrorString(e));
  } else {
    const size_t sm2 = (size_t)pcap * (sizeof(double) + sizeof(int)) + 16;
    if (sm2 > 48 * 1024) {
      cudaFuncSetAttribute(jacobi_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)limit);
    }
    jacobi_kernel<false><<<count, svd_threads(pcap), sm2, s>>>(descs_dev);
  }
  return check_launch("jacobi");
}

void set_jacobi_sync(unsigned int *bar) {
  g_bj.bar = bar;
  g_bj.flag = bar ? reinterpret_cast<int *>(bar + 2) : nullptr;
}


// ------------------------------------------------------------------ TSQR ---
// Tall QR (m >> n) as a tree of Householder QRs (communication-avoiding TSQR):
// level l splits its rows_l x n input into P_l row blocks (P_l - 1 of
// ceil(rows_l / P_l) >= 2n rows and a ragged last one that may be shorter than
// n), each factorised by its own CTA with the panel in shared memory
// (qr_kernel); the R factors are stacked into the ((P_l - 1) n + min(last, n))
// x n input of level l+1; the last (small) stack is factorised once (top).  The explicit Q
// is formed top-down: Q_l = blockdiag(Q_leaf,l,i) Q_(l+1), i.e. one batched
// DMMA GEMM per level (leaf i: mb x n times the n x n block i of Q_(l+1)),
// the level-0 product written straight into the caller's Q (strides).
// Backward stable like the single Householder QR; R (and Q) differ from it
// only by the column signs (gauge).  Sizes follow the device-resident
// descriptor; the level structure is planned on the host from capacities.
namespace {
constexpr int TSQR_MB = 600;     // leaf rows: the 32-column panels of a leaf stay in shared memory
constexpr int TSQR_MAXL = 8;

struct TsqrPlan {
  int levels = 0;
  int mb = TSQR_MB;
  int Pcap[TSQR_MAXL] = {};
  long long rows[TSQR_MAXL + 1] = {};   // capacity rows of each level's input
};

TsqrPlan tsqr_plan_caps(int mcap, int ncap) {
  TsqrPlan p;
  p.mb = TSQR_MB > 4 * ncap ? TSQR_MB : 4 * ncap;   // >= 4n: each level shrinks the rows >= 2x
  long long rows = mcap;
  p.rows[0] = rows;
  if (ncap < 1 || mcap < 3 * ncap || mcap <= p.mb) return p;
  while (rows > p.mb && p.levels < TSQR_MAXL) {
    const int P = (int)((rows + p.mb - 1) / p.mb);
    p.Pcap[p.levels] = P;
    rows = (long long)P * ncap;
    p.rows[++p.levels] = rows;
  }
  return p;
}

struct TsqrDev {
  int levels, mb, ncap;
  int Pcap[TSQR_MAXL];
  QRDesc *qd[TSQR_MAXL];           // leaves of each level
  QRDesc *qtop;
  GemmDesc *gd;                    // [2 TSQR_MAXL]: uniform leaves, last leaf
  double *A[TSQR_MAXL + 1];        // working copies (level inputs; [levels] = top)
  double *Ql[TSQR_MAXL];           // leaf Q factors
  double *S[TSQR_MAXL + 1];        // stacked R factors = input of level l (l >= 1)
  double *Qacc[TSQR_MAXL + 1];     // Q of level l's input (l >= 1)
  double *tau[TSQR_MAXL + 1], *T[TSQR_MAXL + 1];
  long long Tstride;
};

__device__ QRDesc qr_empty() {
  QRDesc q;
  q.m = 0; q.n = 0; q.src = nullptr; q.src_rs = 0; q.src_cs = 0; q.A = nullptr; q.lda = 1; q.Q = nullptr;
  q.q_rs = 0; q.q_cs = 0; q.R = nullptr; q.ldr = 1; q.rt = 0; q.tau = nullptr; q.T = nullptr;
  return q;
}
__device__ GemmDesc gemm_empty() {
  GemmDesc g;
  g.M = 0; g.N = 0; g.K = 0; g.transA = 0; g.transB = 0; g.lda = 1; g.ldb = 1; g.A = nullptr; g.B = nullptr;
  g.C = nullptr; g.dr = 1 << 30; g.dc = 1 << 30; g.s_r0 = 1; g.s_r1 = 0; g.s_c0 = 0; g.s_c1 = 0; g.alpha = 1.0;
  g.beta = 0.0; g.alpha_dev = nullptr; g.skip = nullptr; g.batch = 1; g.bsA = g.bsB = g.bsC = 0;
  return g;
}
__device__ GemmDesc gemm_q(int M, int N, int K, const double *A, long long lda, const double *B, long long ldb,
                           double *C, long long crs, long long ccs) {
  GemmDesc g = gemm_empty();
  g.M = M; g.N = N; g.K = K; g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.C = C;
  g.s_r0 = crs; g.s_c0 = ccs; g.batch = 0;
  return g;
}

__global__ void tsqr_plan_kernel(const QRDesc *__restrict__ in_p, TsqrDev D) {
  const QRDesc in = *in_p;
  const int n = in.n, m = in.m;
  for (int l = 0; l < D.levels; ++l)
    for (int i = 0; i < D.Pcap[l]; ++i) D.qd[l][i] = qr_empty();
  *D.qtop = qr_empty();
  for (int q = 0; q < 2 * D.levels; ++q) D.gd[q] = gemm_empty();
  if (m < 3 * n || m <= D.mb || n < 1) {   // not tall at the device sizes: the plain QR
    D.qd[0][0] = in;
    return;
  }
  long long rows = m;
  int P[TSQR_MAXL], mbl[TSQR_MAXL];
  long long rl[TSQR_MAXL + 1];
  rl[0] = rows;
  for (int l = 0; l < D.levels; ++l) {
    // p - 1 leaves of ceil(rows / p) rows (>= 2n) and a ragged last one (>= 1 row)
    const int p = (int)((rows + D.mb - 1) / D.mb);
    const int mb = (int)((rows + p - 1) / p);
    const long long last = rows - (long long)(p - 1) * mb;
    const int qlast = (int)(last < n ? last : n);
    P[l] = p;
    mbl[l] = mb;
    const long long nxt = (long long)(p - 1) * n + qlast;
    for (int i = 0; i < p; ++i) {
      QRDesc &q = D.qd[l][i];
      const long long r0 = (long long)i * mb;
      q.m = (int)(i < p - 1 ? mb : last);
      q.n = n;
      if (l == 0) { q.src = in.src + r0 * in.src_rs; q.src_rs = in.src_rs; q.src_cs = in.src_cs; }
      else { q.src = D.S[l] + r0; q.src_rs = 1; q.src_cs = rows; }
      q.A = D.A[l] + r0; q.lda = rows;
      q.Q = in.Q ? D.Ql[l] + r0 : nullptr; q.q_rs = 1; q.q_cs = rows;
      q.R = D.S[l + 1] + (long long)i * n; q.ldr = nxt; q.rt = 0;
      q.tau = D.tau[l] + (long long)i * D.ncap;
      q.T = D.T[l] + (long long)i * D.Tstride;
    }
    rows = nxt;
    rl[l + 1] = rows;
  }
  const int L = D.levels;
  QRDesc &t = *D.qtop;
  t.m = (int)rows; t.n = n;
  t.src = D.S[L]; t.src_rs = 1; t.src_cs = rows;
  t.A = D.A[L]; t.lda = rows;
  t.Q = in.Q ? D.Qacc[L] : nullptr; t.q_rs = 1; t.q_cs = rows;
  t.R = in.R; t.ldr = in.ldr; t.rt = in.rt;
  t.tau = D.tau[L]; t.T = D.T[L];
  if (!in.Q) return;
  for (int l = L - 1; l >= 0; --l) {
    const int p = P[l], mb = mbl[l];
    const double *Qn = D.Qacc[l + 1];
    const long long ldn = rl[l + 1];
    double *out = l == 0 ? in.Q : D.Qacc[l];
    const long long crs = l == 0 ? in.q_rs : 1, ccs = l == 0 ? in.q_cs : rl[l];
    GemmDesc &u = D.gd[2 * l];
    if (p > 1) {   // leaves 0 .. p-2: one batched GEMM (mb x n) (n x n)
      u = gemm_q(mb, n, n, D.Ql[l], rl[l], Qn, ldn, out, crs, ccs);
      u.batch = p - 1; u.bsA = mb; u.bsB = n; u.bsC = (long long)mb * crs;
    }
    const long long r0 = (long long)(p - 1) * mb, last = rl[l] - r0;
    D.gd[2 * l + 1] = gemm_q((int)last, n, (int)(last < n ? last : n), D.Ql[l] + r0, rl[l],
                             Qn + (long long)(p - 1) * n, ldn, out + r0 * crs, crs, ccs);
  }
}
}  // namespace

size_t qr_tall_ws_bytes(int mcap, int ncap) {
  const TsqrPlan p = tsqr_plan_caps(mcap, ncap);
  if (p.levels == 0) return 0;
  Arena ar;
  const long long Tstride = 32LL * 32 * ((ncap + 31) / 32 + 1);
  for (int l = 0; l < p.levels; ++l) {
    ar.take<QRDesc>(p.Pcap[l]);
    ar.take<double>(p.rows[l] * ncap);             // A
    ar.take<double>(p.rows[l] * ncap);             // Ql
    ar.take<double>((long long)p.Pcap[l] * ncap);  // tau
    ar.take<double>((long long)p.Pcap[l] * Tstride);
  }
  for (int l = 1; l <= p.levels; ++l) {
    ar.take<double>(p.rows[l] * ncap);   // S
    ar.take<double>(p.rows[l] * ncap);   // Qacc
  }
  ar.take<double>(p.rows[p.levels] * ncap);   // A top
  ar.take<double>(ncap);                      // tau top
  ar.take<double>(Tstride);                   // T top
  ar.take<QRDesc>(1);
  ar.take<GemmDesc>(2 * TSQR_MAXL);
  return ar.used;
}

tt_status launch_qr_tall(const QRDesc *desc_dev, int mcap, int ncap, void *ws, size_t wsb, cudaStream_t s) {
  const TsqrPlan p = tsqr_plan_caps(mcap, ncap);
  if (p.levels == 0 || !ws) return launch_qr(desc_dev, 1, s);
  Arena ar;
  ar.base = (char *)ws;
  ar.cap = wsb;
  TsqrDev D;
  D.levels = p.levels;
  D.mb = p.mb;
  D.ncap = ncap;
  D.Tstride = 32LL * 32 * ((ncap + 31) / 32 + 1);
  for (int l = 0; l < TSQR_MAXL; ++l) { D.Pcap[l] = p.Pcap[l]; D.qd[l] = nullptr; D.Ql[l] = nullptr; }
  for (int l = 0; l <= TSQR_MAXL; ++l) { D.A[l] = D.S[l] = D.Qacc[l] = D.tau[l] = D.T[l] = nullptr; }
  for (int l = 0; l < p.levels; ++l) {
    D.qd[l] = ar.take<QRDesc>(p.Pcap[l]);
    D.A[l] = ar.take<double>(p.rows[l] * ncap);
    D.Ql[l] = ar.take<double>(p.rows[l] * ncap);
    D.tau[l] = ar.take<double>((long long)p.Pcap[l] * ncap);
    D.T[l] = ar.take<double>((long long)p.Pcap[l] * D.Tstride);
  }
  for (int l = 1; l <= p.levels; ++l) {
    D.S[l] = ar.take<double>(p.rows[l] * ncap);
    D.Qacc[l] = ar.take<double>(p.rows[l] * ncap);
  }
  D.A[p.levels] = ar.take<double>(p.rows[p.levels] * ncap);
  D.tau[p.levels] = ar.take<double>(ncap);
  D.T[p.levels] = ar.take<double>(D.Tstride);
  D.qtop = ar.take<QRDesc>(1);
  D.gd = ar.take<GemmDesc>(2 * TSQR_MAXL);
  if (!ar.ok()) return fail(TT_ERR_CAPACITY, "qr (tall): workspace too small");
  tsqr_plan_kernel<<<1, 1, 0, s>>>(desc_dev, D);
  TT_TRY(check_launch("tsqr plan"));
  for (int l = 0; l < p.levels; ++l) TT_TRY(launch_qr(D.qd[l], p.Pcap[l], s));
  TT_TRY(launch_qr(D.qtop, 1, s));
  for (int l = p.levels - 1; l >= 0; --l) {
    if (p.Pcap[l] > 1) TT_TRY(launch_gemm_k(D.gd + 2 * l, 1, p.mb, ncap, ncap, s, p.Pcap[l] - 1));
    TT_TRY(launch_gemm_k(D.gd + 2 * l + 1, 1, (int)(p.rows[l] < p.mb ? p.rows[l] : p.mb), ncap, ncap, s));
  }
  return TT_OK;
}

}  // namespace tt
