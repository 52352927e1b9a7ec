// Device-resident restarted GMRES(m) for the AMEn local systems:
// classical Gram-Schmidt with one re-orthogonalisation (CGS2), Givens rotations
// on the device, convergence flag in device memory.  The vector length N
// follows the device-resident TT ranks; kernels early-exit once converged so
// the host can enqueue a whole cycle without reading anything back.
#include <cstdlib>

#include "gmres.h"

namespace tt {

namespace {
constexpr int RT = 1024;  // reduction CTA size

__device__ double block_reduce_sum(double v) {
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < nw; ++i) t += red[i];
  return t;
}

// r = b - Ax (Ax already computed), beta = ||r||, bnorm = ||b||; V0 = r / beta.
__global__ void __launch_bounds__(RT) gm_start_kernel(GmState *st, const double *b, const double *Ax, double *V) {
  if (st->converged) return;
  const int N = st->N;
  double sb = 0.0, sr = 0.0;
  for (int i = threadIdx.x; i < N; i += RT) {
    const double r = b[i] - Ax[i];
    V[i] = r;
    sb = fma(b[i], b[i], sb);
    sr = fma(r, r, sr);
  }
  sb = block_reduce_sum(sb);
  sr = block_reduce_sum(sr);
  const double beta = sqrt(sr), bn = sqrt(sb);
  __shared__ int s_done;
  if (threadIdx.x == 0) {
    if (st->cycle == 0) {
      st->bnorm = bn;
      st->res0 = bn > 0.0 ? beta / bn : 0.0;  // local residual before the solve
    }
    st->beta = beta;
    st->j = 0;
    st->jdone = 0;
    st->g[0] = beta;
    const double rel = bn > 0.0 ? beta / bn : 0.0;
    st->res = rel;
    s_done = (rel <= st->tol) || (beta == 0.0);
    if (s_done) { st->converged = 1; st->stop = 1; }
  }
  __syncthreads();
  if (s_done) return;
  const double inv = 1.0 / beta;
  for (int i = threadIdx.x; i < N; i += RT) V[i] *= inv;
}

// h[i] (+)= <V_i, w> for i <= j  (grid = m+1 CTAs; CTA i handles column i)
__global__ void __launch_bounds__(256) gm_dots_kernel(GmState *st, const double *V, long long ldv, const double *w,
                                                      double *h, int j, int accumulate) {
  if (st->converged || st->stop) return;
  const int i = blockIdx.x;
  if (i > j) return;
  const int N = st->N;
  const double *vi = V + (long long)i * ldv;
  double s = 0.0;
  for (int e = threadIdx.x; e < N; e += blockDim.x) s = fma(vi[e], w[e], s);
  s = block_reduce_sum(s);
  if (threadIdx.x == 0) h[i] = accumulate ? h[i] + s : s;
}

// w -= sum_{i<=j} hsub[i] V_i  (elementwise, grid-stride)
__global__ void gm_axpy_kernel(GmState *st, const double *V, long long ldv, double *w, const double *hsub, int j) {
  if (st->converged || st->stop) return;
  const int N = st->N;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < N; e += gridDim.x * blockDim.x) {
    double s = w[e];
    for (int i = 0; i <= j; ++i) s = fma(-hsub[i], V[(long long)i * ldv + e], s);
    w[e] = s;
  }
}

// norm of w, V_{j+1} = w / ||w||, Hessenberg column, Givens update (one CTA)
__global__ void __launch_bounds__(RT) gm_finish_step_kernel(GmState *st, double *V, long long ldv, const double *w,
                                                            const double *h1, const double *h2, int j) {
  if (st->converged || st->stop) return;
  const int N = st->N;
  double s = 0.0;
  for (int e = threadIdx.x; e < N; e += RT) s = fma(w[e], w[e], s);
  s = block_reduce_sum(s);
  const double hn = sqrt(s);
  __shared__ int s_flag;
  if (threadIdx.x == 0) {
    const int m = st->m;
    double *H = st->H;  // (m+1) x m, column-major, ld = m+1
    for (int i = 0; i <= j; ++i) H[i + (m + 1) * j] = h1[i] + h2[i];
    H[j + 1 + (m + 1) * j] = hn;
    // apply previous rotations
    for (int i = 0; i < j; ++i) {
      const double a = H[i + (m + 1) * j], b = H[i + 1 + (m + 1) * j];
      H[i + (m + 1) * j] = st->cs[i] * a + st->sn[i] * b;
      H[i + 1 + (m + 1) * j] = -st->sn[i] * a + st->cs[i] * b;
    }
    const double a = H[j + (m + 1) * j], b = H[j + 1 + (m + 1) * j];
    const double den = hypot(a, b);
    const double c = den > 0.0 ? a / den : 1.0, sn = den > 0.0 ? b / den : 0.0;
    st->cs[j] = c;
    st->sn[j] = sn;
    H[j + (m + 1) * j] = den;
    H[j + 1 + (m + 1) * j] = 0.0;
    st->g[j + 1] = -sn * st->g[j];
    st->g[j] = c * st->g[j];
    st->jdone = j + 1;
    const double rel = st->bnorm > 0.0 ? fabs(st->g[j + 1]) / st->bnorm : 0.0;
    st->res = rel;
    int stop = 0;
    if (rel <= st->tol) stop = 1;
    if (hn == 0.0) stop = 1;          // happy breakdown
    if (j + 1 >= st->m) stop = 1;     // end of cycle
    if (!(rel == rel)) { stop = 1; st->nan = 1; }
    st->stop = stop;
    s_flag = (hn > 0.0);
  }
  __syncthreads();
  if (s_flag) {
    const double inv = 1.0 / hn;
    double *vn = V + (long long)(j + 1) * ldv;
    for (int e = threadIdx.x; e < N; e += RT) vn[e] = w[e] * inv;
  }
}

// y = H^{-1} g (upper triangular, jdone x jdone), x += V y; marks convergence.
__global__ void __launch_bounds__(RT) gm_update_kernel(GmState *st, const double *V, long long ldv, double *x) {
  if (st->converged) return;
  const int jd = st->jdone;
  __shared__ double y[GM_MAX_M];
  if (threadIdx.x == 0) {
    const int m = st->m;
    const double *H = st->H;
    for (int i = jd - 1; i >= 0; --i) {
      double s = st->g[i];
      for (int k = i + 1; k < jd; ++k) s -= H[i + (m + 1) * k] * y[k];
      y[i] = s / H[i + (m + 1) * i];
    }
  }
  __syncthreads();
  const int N = st->N;
  for (int e = threadIdx.x; e < N; e += RT) {
    double s = x[e];
    for (int i = 0; i < jd; ++i) s = fma(y[i], V[(long long)i * ldv + e], s);
    x[e] = s;
  }
  if (threadIdx.x == 0) {
    if (st->res <= st->tol) st->converged = 1;
    st->cycle += 1;
    st->stop = 0;
  }
}

__global__ void gm_init_kernel(GmState *st, const int *Nptr, int m, double tol) {
  st->N = *Nptr;
  st->m = m;
  st->tol = tol;
  st->converged = 0;
  st->stop = 0;
  st->cycle = 0;
  st->nan = 0;
  st->jdone = 0;
}


}  // namespace

// Lagged polling of the stop word: after every GM_CHUNK Arnoldi steps the word
// is copied to pinned host memory behind an event; the host checks the copy of
// the PREVIOUS chunk (complete while the current one runs), so the GPU never
// drains.  Steps enqueued after the stop are no-ops (every kernel and the
// apply GEMMs test the word).
constexpr int GM_CHUNK = 6;
static int gm_fchunk() {        // Arnoldi steps per fused launch (TT_GM_FCHUNK)
  static int c = 0;
  if (!c) {
    const char *e = std::getenv("TT_GM_FCHUNK");
    c = e ? std::atoi(e) : 128;   // default: one launch per GMRES cycle (measured fastest)
    c = c < 1 ? 1 : (c > 128 ? 128 : c);
  }
  return c;
}

struct PollSlots {
  int *flag = nullptr;         // pinned [2]
  cudaEvent_t ev[2] = {nullptr, nullptr};
};
thread_local PollSlots g_poll;

tt_status gmres_solve(const GmresCtx &c, cudaStream_t s) {
  // c.apply(in, out) enqueues out = A in for device vectors.
  gm_init_kernel<<<1, 1, 0, s>>>(c.st, c.Nptr, c.m, c.tol);
  TT_TRY(check_launch("gm_init"));
  if (c.poll && !g_poll.flag) {
    if (cudaHostAlloc((void **)&g_poll.flag, 2 * sizeof(int), cudaHostAllocDefault) != cudaSuccess)
      return fail(TT_ERR_CUDA, "gmres: pinned poll word allocation failed");
    cudaEventCreateWithFlags(&g_poll.ev[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&g_poll.ev[1], cudaEventDisableTiming);
  }
  const bool fused = c.gapp && c.part && c.bar && gmres_fused_grid() > 0;
  if (fused) cudaMemsetAsync(c.bar, 0, 2 * sizeof(unsigned int), s);
  static int whole = -1;   // the whole restarted solve in one persistent launch (no host polling)
  if (whole < 0) whole = std::getenv("TT_GMRES_PERCYCLE") ? 0 : 1;
  if (fused && whole) {
    const int decide = c.cluster == 2;
    if (c.cluster != 0)
      TT_TRY(launch_gmres_chunk(c.st, c.gapp, c.V, c.ldv, c.w, c.part, c.split, c.split_elems, c.bar, 0, c.m, s, 1,
                                decide, 1, c.max_restarts, c.b, c.x));
    if (c.cluster != 1)
      TT_TRY(launch_gmres_chunk(c.st, c.gapp, c.V, c.ldv, c.w, c.part, c.split, c.split_elems, c.bar, 0, c.m, s, 0,
                                decide, 1, c.max_restarts, c.b, c.x));
    return check_launch("gmres (persistent)");
  }
  for (int cyc = 0; cyc < c.max_restarts; ++cyc) {
    TT_TRY(c.apply(c.x, c.w, -1));
    gm_start_kernel<<<1, RT, 0, s>>>(c.st, c.b, c.w, c.V);
    int pending = -1;  // slot of the last enqueued poll copy
    if (fused) {
      for (int j0 = 0, q = 0; j0 < c.m; j0 += gm_fchunk(), ++q) {
        const int j1 = j0 + gm_fchunk() < c.m ? j0 + gm_fchunk() : c.m;
        const int decide = c.cluster == 2;
        if (c.cluster != 0)
          TT_TRY(launch_gmres_chunk(c.st, c.gapp, c.V, c.ldv, c.w, c.part, c.split, c.split_elems, c.bar, j0, j1,
                                    s, 1, decide));
        if (c.cluster != 1)
          TT_TRY(launch_gmres_chunk(c.st, c.gapp, c.V, c.ldv, c.w, c.part, c.split, c.split_elems, c.bar, j0, j1,
                                    s, 0, decide));
        if (c.poll) {
          // copy this chunk's stop word, then wait for the PREVIOUS chunk's copy
          // (that chunk finished while this one runs): the GPU never drains
          const int slot = q & 1, prev = slot ^ 1;
          cudaMemcpyAsync(&g_poll.flag[slot], &c.st->stop, sizeof(int), cudaMemcpyDeviceToHost, s);
          cudaEventRecord(g_poll.ev[slot], s);
          if (pending == prev) {
            cudaEventSynchronize(g_poll.ev[prev]);
            if (g_poll.flag[prev]) break;
          }
          pending = slot;
        }
      }
    }
    for (int j = 0; j < (fused ? 0 : c.m); ++j) {
      if (c.poll && j > 0 && j % GM_CHUNK == 0) {
        const int slot = (j / GM_CHUNK) & 1;
        if (pending == slot) cudaEventSynchronize(g_poll.ev[slot]);   // (never: slots alternate)
        cudaMemcpyAsync(&g_poll.flag[slot], &c.st->stop, sizeof(int), cudaMemcpyDeviceToHost, s);
        cudaEventRecord(g_poll.ev[slot], s);
        const int prev = slot ^ 1;
        if (pending == prev) {
          cudaEventSynchronize(g_poll.ev[prev]);
          if (g_poll.flag[prev]) break;
        }
        pending = slot;
      }
      TT_TRY(c.apply(c.V + (long long)j * c.ldv, c.w, j));
      gm_dots_kernel<<<j + 1, 256, 0, s>>>(c.st, c.V, c.ldv, c.w, c.h1, j, 0);
      gm_axpy_kernel<<<c.axpy_blocks, 256, 0, s>>>(c.st, c.V, c.ldv, c.w, c.h1, j);
      gm_dots_kernel<<<j + 1, 256, 0, s>>>(c.st, c.V, c.ldv, c.w, c.h2, j, 0);
      gm_axpy_kernel<<<c.axpy_blocks, 256, 0, s>>>(c.st, c.V, c.ldv, c.w, c.h2, j);
      gm_finish_step_kernel<<<1, RT, 0, s>>>(c.st, c.V, c.ldv, c.w, c.h1, c.h2, j);
    }
    gm_update_kernel<<<1, RT, 0, s>>>(c.st, c.V, c.ldv, c.x);
    TT_TRY(check_launch("gmres"));
    if (c.poll) {
      int conv = 0;
      cudaMemcpyAsync(c.host_flag, &c.st->converged, sizeof(int), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      conv = *c.host_flag;
      if (conv) break;
    }
  }
  return TT_OK;
}

}  // namespace tt
