// Dense local solver of the AMEn local systems ("dense if
// local size <= 2000, else GMRES", readings Z20 / Z35).  One
// cooperative launch per local system:
//   1. assemble the local matrix B[(a,i,a'), (b,j,b')] = sum_{g,g'} Phi[a,g,b]
//      A[g,i,j,g'] Psi[a',g',b'] (the same index conventions as the local apply,
//      P:1517-1519) and the right-hand side into an N x (N+1) column-major array;
//   2. the relative residual of the initial guess ||rhs - B x0|| / ||rhs|| (the
//      sweep's "local residual before the solve", as the GMRES path reports it);
//   3. Gauss-Jordan elimination with partial pivoting (the pivot is the first
//      row of maximal |entry| in the column, as LAPACK's idamax), columns owned
//      cyclically by the CTAs, one grid barrier per pivot step; the solution is
//      the last column.  An exactly zero pivot (singular local system) restarts
//      the elimination on B + mu I with mu = 1e-12 ||B||_F (reading Z35), as the
//      oracle's _local_solve does on LinAlgError.
// The local size N follows the device-resident ranks; the kernel returns at
// once (uniformly) when N > dense_max, and the GMRES path skips itself when
// N <= dense_max (gm_init_kernel).
#include <cfloat>

#include "gmres.h"

namespace tt {

namespace {

__device__ __forceinline__ void dbar(unsigned int *bar, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int inc = blockIdx.x == 0 ? 0x80000000u - (nblocks - 1) : 1u;
    __threadfence();
    const unsigned int old = atomicAdd(bar, inc);
    volatile unsigned int *w = bar;
    unsigned int spins = 0;
    const long long t0 = clock64();
    while (((old ^ *w) & 0x80000000u) == 0) {
      if ((++spins & 1023u) == 0 && clock64() - t0 > 8000000000LL) __trap();   // never hang the device
    }
    __threadfence();
  }
  __syncthreads();
}

constexpr int DT = 256;   // threads per CTA

__device__ __forceinline__ double block_sum(double v, double *red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int q = 0; q < DT / 32; ++q) t += red[q];
  return t;
}

__global__ void __launch_bounds__(DT) dense_local_kernel(DenseArgs a) {
  __shared__ double red[DT / 32];
  __shared__ double s_val[DT / 32];
  __shared__ int s_idx[DT / 32];
  const int N = *a.Nptr;
  if (N > a.dense_max || N < 1) return;   // uniform: the GMRES path handles this system
  const int G = gridDim.x, c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r0 = a.r[a.k], n = a.n, r1 = a.r[a.k + 1], R0 = a.R[a.k], R1 = a.R[a.k + 1];
  double *M = a.M;
  const long long ld = N;
  double *part = a.part;   // [G][4]
  // ---- 1. assembly (grid-stride over the N x N entries) and the rhs column
  auto assemble = [&](double mu) {
    double fro = 0.0;
    const long long NN = (long long)N * N;
    for (long long e = (long long)c * DT + tid; e < NN; e += (long long)G * DT) {
      const int row = (int)(e % N), col = (int)(e / N);
      const int ai = row % r0, ii = (row / r0) % n, ap = row / (r0 * n);
      const int bj = col % r0, jj = (col / r0) % n, bp = col / (r0 * n);
      double s = 0.0;
      for (int gp = 0; gp < R1; ++gp) {
        const double psi = a.Psi[ap + (long long)r1 * (gp + (long long)R1 * bp)];
        if (psi == 0.0) continue;
        double t = 0.0;
        for (int g = 0; g < R0; ++g)
          t = fma(a.Phi[ai + (long long)r0 * (g + (long long)R0 * bj)],
                  a.A[g + (long long)R0 * (ii + (long long)n * (jj + (long long)n * gp))], t);
        s = fma(t, psi, s);
      }
      fro = fma(s, s, fro);
      if (row == col) s += mu;
      M[row + ld * col] = s;
    }
    for (int i = c * DT + tid; i < N; i += G * DT) M[i + ld * N] = a.rhs[i];
    return fro;
  };
  const double fro = assemble(0.0);
  // ---- 2. residual of the initial guess: rows over the CTAs, columns over the threads
  double rr = 0.0, bb = 0.0;
  for (int i = c; i < N; i += G) {
    double s = 0.0;
    for (int j = tid; j < N; j += DT) s = fma(M[i + ld * j], a.x[j], s);
    s = block_sum(s, red);
    const double ri = a.rhs[i] - s;
    rr = fma(ri, ri, rr);
    bb = fma(a.rhs[i], a.rhs[i], bb);
  }
  {
    const double f = block_sum(fro, red);
    if (tid == 0) {
      part[4 * c] = rr;
      part[4 * c + 1] = bb;
      part[4 * c + 2] = f;
    }
  }
  dbar(a.bar, G);
  double trr = 0.0, tbb = 0.0, tff = 0.0;
  for (int q = 0; q < G; ++q) { trr += part[4 * q]; tbb += part[4 * q + 1]; tff += part[4 * q + 2]; }
  if (c == 0 && tid == 0) {
    a.st->res0 = tbb > 0.0 ? sqrt(trr) / sqrt(tbb) : 0.0;
    a.st->res = 0.0;
    a.st->converged = 1;
    a.st->stop = 1;
  }
  // ---- 3. Gauss-Jordan with partial pivoting; singular -> B + mu I (Z35)
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (attempt == 1) {
      dbar(a.bar, G);   // every CTA left the failed elimination
      assemble(1e-12 * sqrt(tff));
      if (c == 0 && tid == 0) atomicAdd(a.mu_count, 1);
      dbar(a.bar, G);
    }
    bool singular = false;
    for (int k = 0; k < N; ++k) {
      double *lb = a.lbuf + (size_t)(k & 1) * (N + 2);
      if (k % G == c) {   // owner of column k: pivot search, the swapped column k
        double best = -1.0;
        int bi = k;
        for (int i = k + tid; i < N; i += DT) {
          const double v = fabs(M[i + ld * k]);
          if (v > best) { best = v; bi = i; }   // first max per thread (ascending i)
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
        }
        if (lane == 0) { s_val[warp] = best; s_idx[warp] = bi; }
        __syncthreads();
        if (tid == 0) {
          double bv = s_val[0];
          int bix = s_idx[0];
          for (int q = 1; q < DT / 32; ++q)
            if (s_val[q] > bv || (s_val[q] == bv && s_idx[q] < bix)) { bv = s_val[q]; bix = s_idx[q]; }
          lb[N] = (double)bix;
          lb[N + 1] = M[bix + ld * k];
        }
        __syncthreads();
        const int p = (int)lb[N];
        for (int i = tid; i < N; i += DT) {
          const int src = (i == k) ? p : (i == p ? k : i);
          lb[i] = M[src + ld * k];
        }
      }
      dbar(a.bar, G);
      const int p = (int)lb[N];
      const double piv = lb[N + 1];
      if (piv == 0.0) { singular = true; break; }   // uniform: every CTA read the same word
      const double inv = 1.0 / piv;
      // own columns j > k (and the rhs column N): swap rows k <-> p, scale the pivot
      // row, eliminate every other row (one warp per column)
      const int first = k + 1 + ((c - (k + 1) % G) % G + G) % G;
      for (int j = first + warp * G; j <= N; j += (DT / 32) * G) {
        double *col = M + ld * j;
        const double ak = col[k], ap = col[p];
        const double t = ap * inv;
        for (int i = lane; i < N; i += 32) {
          if (i == k) col[i] = t;
          else if (i == p) col[i] = fma(-lb[i], t, ak);
          else col[i] = fma(-lb[i], t, col[i]);
        }
      }
      __syncthreads();
    }
    if (!singular) break;
  }
  // ---- solution: the last column (owned by CTA N % G)
  if (N % G == c)
    for (int i = tid; i < N; i += DT) a.x[i] = M[i + ld * N];
}

}  // namespace

tt_status launch_dense_local(const DenseArgs &a, int dense_cap, cudaStream_t s) {
  static int G = 0;
  if (!G) {
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, dense_local_kernel, DT, 0);
    G = occ >= 1 ? sms : -1;
  }
  if (G < 1) return fail(TT_ERR_CUDA, "dense local solver: kernel not co-resident");
  int g = G;
  const int colcap = dense_cap + 1;
  if (g > colcap) g = colcap;   // at least one column per CTA at the capacity size
  cudaMemsetAsync(a.bar, 0, sizeof(unsigned int), s);
  DenseArgs arg = a;
  void *args[] = {(void *)&arg};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void *)dense_local_kernel, dim3(g), dim3(DT), args, 0, s);
  if (e != cudaSuccess) return fail(TT_ERR_CUDA, std::string("dense local solver: ") + cudaGetErrorString(e));
  return TT_OK;
}

}  // namespace tt
