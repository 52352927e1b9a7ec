// Elementwise / structural TT operations: exact matvec (a1), add / scale (a2),
// copy, dot (a8), plus the meta plumbing and error state of the C ABI.
#include <cstdio>
#include <cstring>
#include <string>

#include "tt_common.cuh"

namespace tt {

// ------------------------------------------------------------- errors ---
static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }
const char *last_error_cstr() { return g_last_error.c_str(); }
tt_status fail(tt_status st, const std::string &msg) {
  g_last_error = msg;
  return st;
}
tt_status check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return TT_OK;
}

// --------------------------------------------------------------- metas ---
tt_status make_vec_meta(const tt_vec *x, VecMeta &m) {
  if (!x || !x->n || !x->rcap || !x->off || !x->r_dev || !x->data)
    return fail(TT_ERR_ARG, "tt_vec has a NULL field");
  if (x->d < 1 || x->d > TT_MAX_D) return fail(TT_ERR_ARG, "tt_vec: d out of range");
  if (x->rcap[0] != 1 || x->rcap[x->d] != 1) return fail(TT_ERR_ARG, "tt_vec: rcap[0], rcap[d] must be 1");
  std::memset(&m, 0, sizeof(m));
  m.d = x->d;
  for (int k = 0; k < x->d; ++k) {
    if (x->n[k] < 1) return fail(TT_ERR_ARG, "tt_vec: mode size < 1");
    m.n[k] = x->n[k];
    m.off[k] = x->off[k];
  }
  for (int k = 0; k <= x->d; ++k) {
    if (x->rcap[k] < 1) return fail(TT_ERR_ARG, "tt_vec: rank capacity < 1");
    m.rcap[k] = x->rcap[k];
  }
  m.data = x->data;
  m.r = x->r_dev;
  return TT_OK;
}

tt_status make_mat_meta(const tt_mat *A, MatMeta &m) {
  if (!A || !A->m || !A->n || !A->Rcap || !A->off || !A->R_dev || !A->data)
    return fail(TT_ERR_ARG, "tt_mat has a NULL field");
  if (A->d < 1 || A->d > TT_MAX_D) return fail(TT_ERR_ARG, "tt_mat: d out of range");
  if (A->Rcap[0] != 1 || A->Rcap[A->d] != 1) return fail(TT_ERR_ARG, "tt_mat: Rcap[0], Rcap[d] must be 1");
  std::memset(&m, 0, sizeof(m));
  m.d = A->d;
  for (int k = 0; k < A->d; ++k) {
    if (A->m[k] < 1 || A->n[k] < 1) return fail(TT_ERR_ARG, "tt_mat: mode size < 1");
    m.m[k] = A->m[k];
    m.n[k] = A->n[k];
    m.off[k] = A->off[k];
  }
  for (int k = 0; k <= A->d; ++k) m.Rcap[k] = A->Rcap[k];
  m.data = A->data;
  m.R = A->R_dev;
  return TT_OK;
}

VecMeta mat_as_vec(const MatMeta &A) {
  VecMeta v;
  std::memset(&v, 0, sizeof(v));
  v.d = A.d;
  for (int k = 0; k < A.d; ++k) {
    v.n[k] = A.m[k] * A.n[k];
    v.off[k] = A.off[k];
  }
  for (int k = 0; k <= A.d; ++k) v.rcap[k] = A.Rcap[k];
  v.data = A.data;
  v.r = A.R;
  return v;
}

int max_slot(const VecMeta &x) {
  long long mx = 0;
  for (int k = 0; k < x.d; ++k) {
    long long s = (long long)x.rcap[k] * x.n[k] * x.rcap[k + 1];
    if (s > mx) mx = s;
  }
  return (int)mx;
}
int max_rank(const VecMeta &x) {
  int mx = 1;
  for (int k = 0; k <= x.d; ++k) mx = x.rcap[k] > mx ? x.rcap[k] : mx;
  return mx;
}

// algorithmic flops of the exact matvec (2 n per output entry)
__device__ unsigned long long g_matvec_flops;
void matvec_counters(unsigned long long *out, int reset) {
  cudaMemcpyFromSymbol(out, g_matvec_flops, sizeof(unsigned long long));
  if (reset) {
    unsigned long long z = 0;
    cudaMemcpyToSymbol(g_matvec_flops, &z, sizeof(z));
  }
}

// -------------------------------------------------------------- matvec ---
// Y_k[rho, i, rho'] = sum_j A_k[a, i, j, a'] X_k[b, j, b'], rho = a + R b.
// One launch over all cores: blockIdx.y = core, grid-stride over output entries
// (consecutive threads write consecutive rho: coalesced stores, which are the
// HBM traffic that bounds this kernel for QTT 2x2 cores).
__global__ void matvec_kernel(const MatMeta A, const VecMeta x, const VecMeta y) {
  const int k = blockIdx.y;
  const int R0 = A.R[k], R1 = A.R[k + 1], r0 = x.r[k], r1 = x.r[k + 1];
  const int m = A.m[k], n = A.n[k];
  const int P = R0 * r0, P1 = R1 * r1;
  const int total = P * m * P1;
  const double *__restrict__ Ak = A.data + A.off[k];
  const double *__restrict__ Xk = x.data + x.off[k];
  double *__restrict__ Yk = y.data + y.off[k];
  const int jsA = R0 * m;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int rho = e % P;
    const int t = e / P;
    const int i = t % m;
    const int rho1 = t / m;
    const int a = rho % R0, b = rho / R0, a1 = rho1 % R1, b1 = rho1 / R1;
    const double *Ap = Ak + a + R0 * i + (long long)jsA * n * a1;
    const double *Xp = Xk + b + (long long)r0 * n * b1;
    double s = 0.0;
    for (int j = 0; j < n; ++j) s = fma(Ap[(long long)j * jsA], Xp[(long long)j * r0], s);
    Yk[e] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    y.r[k] = P;
    if (k == A.d - 1) y.r[k + 1] = P1;
    atomicAdd(&g_matvec_flops, 2ull * (unsigned long long)total * n);
  }
}

tt_status matvec_meta(const MatMeta &A, const VecMeta &x, const VecMeta &y, cudaStream_t s) {
  if (A.d != x.d || A.d != y.d) return fail(TT_ERR_SHAPE, "tt_matvec: number of cores differ");
  long long mx = 0;
  for (int k = 0; k < A.d; ++k) {
    if (A.n[k] != x.n[k]) return fail(TT_ERR_SHAPE, "tt_matvec: shape mismatch (A.n != x.n)");
    if (A.m[k] != y.n[k]) return fail(TT_ERR_SHAPE, "tt_matvec: shape mismatch (A.m != y.n)");
    long long c = (long long)A.Rcap[k] * x.rcap[k] * A.m[k] * A.Rcap[k + 1] * x.rcap[k + 1];
    if (c > (1LL << 31) - 1) return fail(TT_ERR_CAPACITY, "tt_matvec: core too large");
    mx = c > mx ? c : mx;
  }
  for (int k = 0; k <= A.d; ++k)
    if ((long long)y.rcap[k] < (long long)A.Rcap[k] * x.rcap[k])
      return fail(TT_ERR_CAPACITY, "tt_matvec: y rank capacity < R*r");
  int bx = (int)((mx + 255) / 256);
  if (bx > 2048) bx = 2048;
  if (bx < 1) bx = 1;
  matvec_kernel<<<dim3(bx, A.d), 256, 0, s>>>(A, x, y);
  return check_launch("tt_matvec");
}

// ----------------------------------------------------------------- add ---
// z = alpha x + beta y, block-diagonal concatenation.
__global__ void add_kernel(const VecMeta x, const double *alpha, const VecMeta y, const double *beta,
                           const VecMeta z) {
  const int k = blockIdx.y, d = x.d;
  const int n = x.n[k];
  const int rx0 = x.r[k], rx1 = x.r[k + 1], ry0 = y.r[k], ry1 = y.r[k + 1];
  const double *Xk = x.data + x.off[k];
  const double *Yk = y.data + y.off[k];
  double *Zk = z.data + z.off[k];
  const double al = (k == 0 && alpha) ? *alpha : 1.0;
  const double be = (k == 0 && beta) ? *beta : 1.0;
  if (d == 1) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
      Zk[e] = al * Xk[e] + be * Yk[e];
    if (blockIdx.x == 0 && threadIdx.x == 0) { z.r[0] = 1; z.r[1] = 1; }
    return;
  }
  const int rz0 = (k == 0) ? 1 : rx0 + ry0;
  const int rz1 = (k == d - 1) ? 1 : rx1 + ry1;
  const int total = rz0 * n * rz1;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int p = e % rz0, t = e / rz0, i = t % n, q = t / n;
    double v = 0.0;
    if (k == 0) {
      v = (q < rx1) ? al * Xk[i + n * q] : be * Yk[i + n * (q - rx1)];
    } else if (k == d - 1) {
      v = (p < rx0) ? Xk[p + rx0 * i] : Yk[(p - rx0) + ry0 * i];
    } else {
      if (p < rx0 && q < rx1) v = Xk[p + rx0 * (i + n * q)];
      else if (p >= rx0 && q >= rx1) v = Yk[(p - rx0) + ry0 * (i + n * (q - rx1))];
    }
    Zk[e] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    z.r[k] = rz0;
    if (k == d - 1) z.r[k + 1] = 1;
  }
}

tt_status add_meta(const VecMeta &x, const double *alpha, const VecMeta &y, const double *beta,
                   const VecMeta &z, cudaStream_t s) {
  if (x.d != y.d || x.d != z.d) return fail(TT_ERR_SHAPE, "tt_add: number of cores differ");
  long long mx = 0;
  for (int k = 0; k < x.d; ++k) {
    if (x.n[k] != y.n[k] || x.n[k] != z.n[k]) return fail(TT_ERR_SHAPE, "tt_add: shape mismatch");
    long long c = (long long)z.rcap[k] * z.n[k] * z.rcap[k + 1];
    mx = c > mx ? c : mx;
  }
  for (int k = 1; k < x.d; ++k)
    if (z.rcap[k] < x.rcap[k] + y.rcap[k]) return fail(TT_ERR_CAPACITY, "tt_add: z rank capacity < rx+ry");
  // (keff sizes B with exactly these capacities)
  int bx = (int)((mx + 255) / 256);
  bx = bx > 1024 ? 1024 : (bx < 1 ? 1 : bx);
  add_kernel<<<dim3(bx, x.d), 256, 0, s>>>(x, alpha, y, beta, z);
  return check_launch("tt_add");
}

// --------------------------------------------------------------- scale ---
__global__ void scale_kernel(const VecMeta x, const double *alpha, double ah, int invert) {
  const int n = x.n[0] * x.r[1];
  double a = alpha ? *alpha : ah;
  if (invert) a = 1.0 / a;
  double *X0 = x.data + x.off[0];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) X0[e] *= a;
}
tt_status scale_meta(const VecMeta &x, const double *alpha_dev, double alpha_host, int invert,
                     cudaStream_t s) {
  int cap = x.n[0] * x.rcap[1];
  int bx = (cap + 255) / 256;
  bx = bx > 256 ? 256 : bx;
  scale_kernel<<<bx, 256, 0, s>>>(x, alpha_dev, alpha_host, invert);
  return check_launch("tt_scale");
}

// ---------------------------------------------------------------- copy ---
__global__ void copy_kernel(const VecMeta x, const VecMeta y) {
  const int k = blockIdx.y;
  const int total = x.r[k] * x.n[k] * x.r[k + 1];
  const double *X = x.data + x.off[k];
  double *Y = y.data + y.off[k];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) Y[e] = X[e];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    y.r[k] = x.r[k];
    if (k == x.d - 1) y.r[k + 1] = x.r[k + 1];
  }
}
tt_status copy_meta(const VecMeta &x, const VecMeta &y, cudaStream_t s) {
  if (x.d != y.d) return fail(TT_ERR_SHAPE, "tt_copy: number of cores differ");
  for (int k = 0; k < x.d; ++k)
    if (x.n[k] != y.n[k]) return fail(TT_ERR_SHAPE, "tt_copy: shape mismatch");
  for (int k = 0; k <= x.d; ++k)
    if (y.rcap[k] < x.rcap[k]) return fail(TT_ERR_CAPACITY, "tt_copy: capacity");
  int bx = (max_slot(x) + 255) / 256;
  bx = bx > 1024 ? 1024 : (bx < 1 ? 1 : bx);
  copy_kernel<<<dim3(bx, x.d), 256, 0, s>>>(x, y);
  return check_launch("tt_copy");
}

// ----------------------------------------------------------------- dot ---
// <x, y> by the left-to-right chain W_k = sum_i X_k(i)^T W_{k-1} Y_k(i), one CTA.
__global__ void __launch_bounds__(512) dot_kernel(const VecMeta x, const VecMeta y, double *W, double *Z,
                                                  double *out) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) W[0] = 1.0;
  __syncthreads();
  for (int k = 0; k < x.d; ++k) {
    const int n = x.n[k];
    const int rx0 = x.r[k], rx1 = x.r[k + 1], ry0 = y.r[k], ry1 = y.r[k + 1];
    const double *X = x.data + x.off[k];
    const double *Y = y.data + y.off[k];
    // Z[a, i, b'] = sum_b W[a, b] Y[b, i, b']
    const int nz = rx0 * n * ry1;
    for (int e = tid; e < nz; e += nt) {
      const int a = e % rx0, t = e / rx0, i = t % n, b1 = t / n;
      double s = 0.0;
      for (int b = 0; b < ry0; ++b) s = fma(W[a + rx0 * b], Y[b + ry0 * (i + n * b1)], s);
      Z[e] = s;
    }
    __syncthreads();
    // W'[a', b'] = sum_{a, i} X[a, i, a'] Z[a, i, b']
    const int nw = rx1 * ry1;
    const int kk = rx0 * n;
    for (int e = tid; e < nw; e += nt) {
      const int a1 = e % rx1, b1 = e / rx1;
      double s = 0.0;
      for (int q = 0; q < kk; ++q) s = fma(X[q + kk * a1], Z[q + kk * b1], s);
      W[e] = s;
    }
    __syncthreads();
  }
  if (tid == 0) *out = W[0];
}

tt_status dot_meta(const VecMeta &x, const VecMeta &y, double *out, Arena &ar, cudaStream_t s) {
  if (x.d != y.d) return fail(TT_ERR_SHAPE, "tt_dot: number of cores differ");
  long long wmax = 1, zmax = 1;
  for (int k = 0; k < x.d; ++k) {
    if (x.n[k] != y.n[k]) return fail(TT_ERR_SHAPE, "tt_dot: shape mismatch");
    long long w = (long long)x.rcap[k + 1] * y.rcap[k + 1];
    long long z = (long long)x.rcap[k] * x.n[k] * y.rcap[k + 1];
    wmax = w > wmax ? w : wmax;
    zmax = z > zmax ? z : zmax;
  }
  double *W = ar.take<double>(wmax);
  double *Z = ar.take<double>(zmax);
  if (!ar.base) return TT_OK;
  if (!ar.ok()) return fail(TT_ERR_CAPACITY, "tt_dot: workspace too small");
  dot_kernel<<<1, 512, 0, s>>>(x, y, W, Z, out);
  return check_launch("tt_dot");
}

// ---------------------------------------------------------------- copy ---
__global__ void copy_desc_kernel(const CopyDesc *descs) {
  const CopyDesc g = descs[blockIdx.y];
  const long long total = (long long)g.rows * g.cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e % g.rows), c = (int)(e / g.rows);
    g.dst[r * g.ds_r + c * g.ds_c] = g.src[r * g.ss_r + c * g.ss_c];
  }
}
tt_status launch_copy(const CopyDesc *descs_dev, int count, long long cap, cudaStream_t s) {
  if (count <= 0) return TT_OK;
  int bx = (int)((cap + 255) / 256);
  bx = bx > 1024 ? 1024 : (bx < 1 ? 1 : bx);
  copy_desc_kernel<<<dim3(bx, count), 256, 0, s>>>(descs_dev);
  return check_launch("copy");
}

}  // namespace tt
