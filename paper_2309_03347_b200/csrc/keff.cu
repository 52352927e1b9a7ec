// keff_fixed_point (a9): eqn:TT_k_eff_fixed_points, readings
// Z16-Z19.  k, <f, Psi>, ||Psi|| and all ranks stay on the device; the host
// polls one convergence word per outer iteration.
#include <cmath>
#include <cstring>

#include "amen.h"
#include "gmres.h"
#include "tt_common.cuh"

namespace tt {

namespace {

struct KeffScal {
  double k, kinv, s_old, s_new, nrm, nrm_inv, one, minus_one, dk, res, rnorm, hnorm;
  int flag, iters, status;
};

__global__ void transpose_ttm_kernel(const MatMeta F, const MatMeta FT) {
  const int k = blockIdx.y;
  const int R0 = F.R[k], R1 = F.R[k + 1], m = F.m[k], n = F.n[k];
  const int total = R0 * m * n * R1;
  const double *src = F.data + F.off[k];
  double *dst = FT.data + FT.off[k];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int a = e % R0, t = e / R0, i = t % m, t2 = t / m, j = t2 % n, b = t2 / n;
    dst[a + R0 * (j + n * (i + m * b))] = src[e];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    FT.R[k] = R0;
    if (k == F.d - 1) FT.R[k + 1] = R1;
  }
}

__global__ void ones_kernel(const VecMeta v) {
  const int k = blockIdx.x;
  double *c = v.data + v.off[k];
  for (int i = threadIdx.x; i < v.n[k]; i += blockDim.x) c[i] = 1.0;
  if (threadIdx.x == 0) {
    v.r[k] = 1;
    if (k == v.d - 1) v.r[k + 1] = 1;
  }
}

__global__ void keff_init_kernel(KeffScal *sc, double k0, const double *k0_dev, const double *nrm) {
  if (k0_dev && *k0_dev != 0.0 && *k0_dev == *k0_dev) k0 = *k0_dev;
  sc->k = k0;
  sc->kinv = 1.0 / k0;
  sc->one = 1.0;
  sc->minus_one = -1.0;
  sc->dk = 0.0;
  sc->res = -1.0;
  sc->flag = 0;
  sc->iters = 0;
  sc->status = 0;
  sc->nrm = *nrm;
  sc->nrm_inv = (*nrm > 0.0) ? 1.0 / *nrm : 1.0;
}

__global__ void set_i32_k(int *p, int v) { *p = v; }
__global__ void fill_kernel(double *p, int n, double v) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = v;
}

__global__ void keff_after_solve_kernel(KeffScal *sc) {
  // k' = k <f, Psi'> / <f, Psi>
  if (sc->s_old == 0.0 || !(sc->s_old == sc->s_old)) {
    sc->status = TT_ERR_NOFISSION;
    sc->flag = 1;
    return;
  }
  sc->nrm_inv = 0.0;  // set after the norm
}

// k' = k <f, Psi'> / <f, Psi> and the history; the convergence decision is
// keff_decide_kernel's (after the optional residual evaluation)
__global__ void keff_update_kernel(KeffScal *sc, const double *nrm, double *khist, int *shist, int *ihist,
                                   const int *sweeps, const int *inner, int hist_cap) {
  if (sc->status == TT_ERR_NOFISSION) return;
  const double knew = sc->k * sc->s_new / sc->s_old;
  const double nn = *nrm;
  sc->nrm = nn;
  sc->nrm_inv = nn > 0.0 ? 1.0 / nn : 1.0;
  sc->s_old = sc->s_new * sc->nrm_inv;
  const int it = sc->iters;
  if (khist && it < hist_cap) khist[it] = knew;
  if (shist && it < hist_cap) shist[it] = sweeps ? *sweeps : 0;
  if (ihist && it < hist_cap) ihist[it] = inner ? *inner : 0;
  sc->iters = it + 1;
  sc->dk = fabs(knew - sc->k);
  sc->k = knew;
  sc->kinv = 1.0 / knew;
  sc->res = -1.0;
  if (!(knew == knew)) sc->status = TT_ERR_NUMERIC;
}

// res = ||M Psi|| / ||H Psi|| of the iteration just finished (history slot it)
__global__ void keff_res_kernel(KeffScal *sc, double *rhist, int hist_cap, double *res_out) {
  const double r = sc->hnorm > 0.0 ? sc->rnorm / sc->hnorm : (sc->rnorm > 0.0 ? INFINITY : 0.0);
  sc->res = r;
  const int it = sc->iters - 1;
  if (rhist && it >= 0 && it < hist_cap) rhist[it] = r;
  if (res_out) *res_out = r;
}

__global__ void keff_decide_kernel(KeffScal *sc, double tol_k, double tol_res, int max_outer, double *k_out,
                                   int *iters_out, int *status_out) {
  if (sc->status == TT_ERR_NOFISSION || sc->status == TT_ERR_NUMERIC) {
    sc->flag = 1;
  } else if (sc->dk <= tol_k && (tol_res <= 0.0 || (sc->res >= 0.0 && sc->res <= tol_res))) {
    sc->status = TT_OK;
    sc->flag = 1;
  } else if (sc->iters >= max_outer) {
    sc->status = TT_ERR_NOCONV;
    sc->flag = 1;
  }
  if (k_out) *k_out = sc->k;
  if (iters_out) *iters_out = sc->iters;
  if (status_out) *status_out = sc->status;
}

constexpr int KEFF_HIST = 1024;   // iterations recorded in the histories (include/tt.h)

struct KeffWS {
  MatMeta FT, SF, M;
  VecMeta ones, f, SP, FP, B, z0, zmv, Rv, Hv, zr;
  KeffScal *sc;
  double *nrm, *dbuf, *k0buf;
  float *kscr;     // operator-kind detection scratch
  // report buffers inside the workspace: the captured graph writes these (so it
  // does not depend on the caller's report pointers) and a copy-out kernel after
  // the launch fills the caller's keff_report
  double *ok, *ores, *okh, *orh;
  int *oit, *ost, *osh, *oih;
  int *sweeps, *inner;
  char *sub;       // scratch for round / dot / orth / amen
  size_t sub_cap;
};

VecMeta vec_like(Arena &ar, int d, const int *n, const int *rcap) {
  VecMeta v;
  std::memset(&v, 0, sizeof(v));
  v.d = d;
  long long off = 0;
  for (int k = 0; k < d; ++k) {
    v.n[k] = n[k];
    v.off[k] = off;
    off += (long long)rcap[k] * n[k] * rcap[k + 1];
  }
  for (int k = 0; k <= d; ++k) v.rcap[k] = rcap[k];
  v.data = ar.take<double>(off);
  v.r = ar.take<int>(d + 1);
  return v;
}

tt_status carve_keff(const MatMeta &H, const MatMeta &S, const MatMeta &F, const VecMeta &psi, const VecMeta &z,
                     const keff_opts &o, Arena &ar, KeffWS &W) {
  const int d = H.d;
  if (S.d != d || F.d != d || psi.d != d || z.d != d) return fail(TT_ERR_SHAPE, "keff: number of cores differ");
  for (int k = 0; k < d; ++k) {
    if (H.m[k] != H.n[k] || S.m[k] != S.n[k] || F.m[k] != F.n[k]) return fail(TT_ERR_SHAPE, "keff: operators must be square");
    if (H.n[k] != psi.n[k] || S.n[k] != psi.n[k] || F.n[k] != psi.n[k]) return fail(TT_ERR_SHAPE, "keff: shape mismatch");
  }
  std::memset(&W, 0, sizeof(W));
  // F^T
  W.FT = F;
  for (int k = 0; k < d; ++k) { W.FT.m[k] = F.n[k]; W.FT.n[k] = F.m[k]; }
  long long tot = 0;
  for (int k = 0; k < d; ++k) tot += (long long)F.Rcap[k] * F.m[k] * F.n[k] * F.Rcap[k + 1];
  W.FT.data = ar.take<double>(tot);
  W.FT.R = ar.take<int>(d + 1);
  int one[TT_MAX_D + 1], cap[TT_MAX_D + 1];
  for (int k = 0; k <= d; ++k) one[k] = 1;
  W.ones = vec_like(ar, d, F.m, one);
  for (int k = 0; k <= d; ++k) cap[k] = F.Rcap[k];
  W.f = vec_like(ar, d, F.n, cap);
  const bool mv = o.matvec == 1;
  if (o.matvec != 0 && o.matvec != 1) return fail(TT_ERR_ARG, "keff: matvec must be 0 (exact) or 1 (amen_mv)");
  if (o.local_dense_max < 0) return fail(TT_ERR_ARG, "keff: local_dense_max must be >= 0");
  if (o.kickrank != 0) {
    int zc = 0;
    for (int k = 1; k < d; ++k) zc = z.rcap[k] > zc ? z.rcap[k] : zc;
    if (d > 1 && o.kickrank != zc) return fail(TT_ERR_ARG, "keff: kickrank must equal z's interior rank capacity");
  }
  // S + k^{-1} F as one TT-matrix (ranks add): the amen_mv operator of B and part of the residual
  W.SF = S;
  {
    long long off = 0;
    for (int k = 0; k <= d; ++k) W.SF.Rcap[k] = (k == 0 || k == d) ? 1 : S.Rcap[k] + F.Rcap[k];
    for (int k = 0; k < d; ++k) {
      W.SF.off[k] = off;
      off += (long long)W.SF.Rcap[k] * S.m[k] * S.n[k] * W.SF.Rcap[k + 1];
    }
    W.SF.data = ar.take<double>(off);
    W.SF.R = ar.take<int>(d + 1);
  }
  const bool res_on = o.tol_res >= 0.0;
  if (res_on) {   // residual operator M = H - (S + k^{-1} F)
    W.M = H;
    long long off = 0;
    for (int k = 0; k <= d; ++k) W.M.Rcap[k] = (k == 0 || k == d) ? 1 : H.Rcap[k] + W.SF.Rcap[k];
    for (int k = 0; k < d; ++k) {
      W.M.off[k] = off;
      off += (long long)W.M.Rcap[k] * H.m[k] * H.n[k] * W.M.Rcap[k + 1];
    }
    W.M.data = ar.take<double>(off);
    W.M.R = ar.take<int>(d + 1);
    W.Rv = vec_like(ar, d, psi.n, psi.rcap);
    W.Hv = vec_like(ar, d, psi.n, psi.rcap);
    W.zr = vec_like(ar, d, z.n, z.rcap);
  }
  if (!mv) {
    for (int k = 0; k <= d; ++k) cap[k] = S.Rcap[k] * psi.rcap[k];
    W.SP = vec_like(ar, d, S.m, cap);
    int capF[TT_MAX_D + 1];
    for (int k = 0; k <= d; ++k) capF[k] = F.Rcap[k] * psi.rcap[k];
    W.FP = vec_like(ar, d, F.m, capF);
    for (int k = 0; k <= d; ++k) cap[k] = (k == 0 || k == d) ? 1 : S.Rcap[k] * psi.rcap[k] + F.Rcap[k] * psi.rcap[k];
    W.B = vec_like(ar, d, psi.n, cap);
  } else {
    // B fitted by amen_mv in psi's capacities
    W.B = vec_like(ar, d, psi.n, psi.rcap);
    W.zmv = vec_like(ar, d, z.n, z.rcap);
  }
  W.z0 = vec_like(ar, d, z.n, z.rcap);
  W.sc = ar.take<KeffScal>(1);
  W.nrm = ar.take<double>(1);
  W.dbuf = ar.take<double>(4);
  W.k0buf = ar.take<double>(1);
  W.kscr = ar.take<float>(KIND_SCRATCH_FLOATS);
  W.ok = ar.take<double>(1);
  W.ores = ar.take<double>(1);
  W.okh = ar.take<double>(KEFF_HIST);
  W.orh = ar.take<double>(KEFF_HIST);
  W.oit = ar.take<int>(1);
  W.ost = ar.take<int>(1);
  W.osh = ar.take<int>(KEFF_HIST);
  W.oih = ar.take<int>(KEFF_HIST);
  W.sweeps = ar.take<int>(1);
  W.inner = ar.take<int>(1);
  // scratch: the max over the sub-operations
  size_t mx = 0;
  auto upd = [&](size_t v) { mx = v > mx ? v : mx; };
  if (!mv) {
    { Arena c; round_meta(W.SP, 0.0, 1, nullptr, nullptr, 0, c, nullptr); upd(c.used); }
    { Arena c; round_meta(W.FP, 0.0, 1, nullptr, nullptr, 0, c, nullptr); upd(c.used); }
    { Arena c; round_meta(W.B, 0.0, 1, nullptr, nullptr, 0, c, nullptr); upd(c.used); }
  } else {
    const size_t b = amen_mv_ws_bytes(W.SF, psi, W.B, W.zmv);
    if (b == 0) return fail(TT_ERR_CAPACITY, "keff: amen_mv operands rejected (psi capacities must exceed z's)");
    upd(b);
  }
  { Arena c; round_meta(W.f, 0.0, 1, nullptr, nullptr, 0, c, nullptr); upd(c.used); }
  { Arena c; round_meta(psi, 0.0, 1, nullptr, nullptr, 0, c, nullptr); upd(c.used); }
  { Arena c; dot_meta(W.f, psi, nullptr, c, nullptr); upd(c.used); }
  upd(amen_ws_bytes(H, W.B, psi, z, o.gmres_restart, o.local_dense_max));
  if (res_on) {
    const size_t b1 = amen_mv_ws_bytes(W.M, psi, W.Rv, W.zr), b2 = amen_mv_ws_bytes(H, psi, W.Hv, W.zr);
    if (b1 == 0 || b2 == 0) return fail(TT_ERR_CAPACITY, "keff: residual amen_mv operands rejected");
    upd(b1);
    upd(b2);
    { Arena c; orth_meta(W.Rv, -1, nullptr, c, nullptr); upd(c.used); }
  }
  W.sub_cap = mx;
  W.sub = ar.take<char>(mx);
  return TT_OK;
}

}  // namespace

size_t keff_ws_bytes(const MatMeta &H, const MatMeta &S, const MatMeta &F, const VecMeta &psi, const VecMeta &z,
                     const keff_opts &o) {
  Arena ar;
  KeffWS W;
  if (carve_keff(H, S, F, psi, z, o, ar, W) != TT_OK) return 0;
  return ar.used;
}

// kinds of the operator cores (als.h CoreKind) detected once per call, before any
// capture; the derived operators inherit them: S + F/k and H - (S + F/k) are
// block sums whose core k is diagonal iff every summand's core k is
tt_status detect_ops_kinds(MatMeta &H, MatMeta &S, MatMeta &F, float *scratch, cudaStream_t s) {
  if (!H.kinds_set) TT_TRY(detect_core_kinds(H, scratch, s));
  if (!S.kinds_set) TT_TRY(detect_core_kinds(S, scratch, s));
  if (!F.kinds_set) TT_TRY(detect_core_kinds(F, scratch, s));
  return TT_OK;
}
void derive_kinds(KeffWS &W, const MatMeta &H, const MatMeta &S, const MatMeta &F) {
  for (int k = 0; k < H.d; ++k) {
    W.SF.kind[k] = S.kind[k] && F.kind[k];
    W.M.kind[k] = H.kind[k] && W.SF.kind[k];
  }
  W.SF.kinds_set = 1;
  W.M.kinds_set = 1;
}

// The enqueue of one keff_fixed_point call; k0 is read on the device (k0_dev).
// Kinds of H, S, F must be set.  Under a capture with device loops the outer
// iteration is a conditional WHILE node (K11).
tt_status keff_body(const MatMeta &H, const MatMeta &S, const MatMeta &F, const VecMeta &psi, const VecMeta &z,
                    const double *k0_dev, const keff_opts &o, const keff_report &rep, Arena &ar, cudaStream_t s) {
  KeffWS W;
  TT_TRY(carve_keff(H, S, F, psi, z, o, ar, W));
  if (!ar.base) return TT_OK;
  if (!ar.ok()) return fail(TT_ERR_CAPACITY, "keff_fixed_point: workspace too small");
  if (!H.kinds_set || !S.kinds_set || !F.kinds_set) return fail(TT_ERR_ARG, "keff: operator kinds not detected");
  derive_kinds(W, H, S, F);
  const double k0 = 1.0;   // placeholder: keff_init_kernel takes *k0_dev
  const int d = H.d;
  auto sub = [&]() {
    Arena a;
    a.base = W.sub;
    a.cap = W.sub_cap;
    return a;
  };
  // f = round(F^T 1)   (reading Z18: built once per solve; a warm call continues a solve
  // with the same operators, so f is still in the workspace like z0 and the amen_mv guess)
  if (!o.warm) {
    transpose_ttm_kernel<<<dim3(64, d), 256, 0, s>>>(F, W.FT);
    ones_kernel<<<d, 256, 0, s>>>(W.ones);
    TT_TRY(matvec_meta(W.FT, W.ones, W.f, s));
    { Arena a = sub(); TT_TRY(round_meta(W.f, 1e-14, 1 << 30, nullptr, nullptr, 0, a, s)); }
  }
  // keep the AMEn residual TT's initial cores (the oracle restarts every solve from z0);
  // a warm call continues the previous one: z0 and the amen_mv guess of B are
  // still in the workspace and psi is already a rounded, normalised iterate
  if (!o.warm) TT_TRY(copy_meta(z, W.z0, s));
  // Psi <- round(Psi0) / ||.||   (Z16, Z17)
  if (!o.warm) { Arena a = sub(); TT_TRY(round_meta(psi, o.eps_round, o.rmax, nullptr, nullptr, 0, a, s)); }
  { Arena a = sub(); TT_TRY(orth_meta(psi, -1, W.nrm, a, s)); }
  keff_init_kernel<<<1, 1, 0, s>>>(W.sc, k0, k0_dev, W.nrm);
  TT_TRY(scale_meta(psi, &W.sc->nrm_inv, 1.0, 0, s));
  { Arena a = sub(); TT_TRY(dot_meta(W.f, psi, &W.sc->s_old, a, s)); }
  AmenOpts ao;
  ao.eps = o.eps_solve;
  ao.local_tol = 0.0;
  ao.max_sweeps = o.max_sweeps;
  ao.rmax = o.rmax;
  ao.restart = o.gmres_restart;
  ao.max_restarts = o.gmres_max_restarts;
  ao.dense_max = o.local_dense_max;
  const bool mv = o.matvec == 1;
  // fixed-point residual ||H Psi - (S + F/k) Psi|| / ||H Psi|| (Z19) of the
  // current normalised Psi and k, both products fitted by amen_mv
  auto residual = [&]() -> tt_status {
    TT_TRY(add_meta(mat_as_vec(S), nullptr, mat_as_vec(F), &W.sc->kinv, mat_as_vec(W.SF), s));
    TT_TRY(add_meta(mat_as_vec(H), nullptr, mat_as_vec(W.SF), &W.sc->minus_one, mat_as_vec(W.M), s));
    TT_TRY(copy_meta(psi, W.Rv, s));
    TT_TRY(copy_meta(W.z0, W.zr, s));
    { Arena a = sub(); TT_TRY(amen_mv_meta(W.M, psi, W.Rv, W.zr, o.eps_round, o.mv_max_sweeps, o.rmax, nullptr, a, s)); }
    { Arena a = sub(); TT_TRY(orth_meta(W.Rv, -1, &W.sc->rnorm, a, s)); }
    TT_TRY(copy_meta(psi, W.Hv, s));
    TT_TRY(copy_meta(W.z0, W.zr, s));
    { Arena a = sub(); TT_TRY(amen_mv_meta(H, psi, W.Hv, W.zr, o.eps_round, o.mv_max_sweeps, o.rmax, nullptr, a, s)); }
    { Arena a = sub(); TT_TRY(orth_meta(W.Hv, -1, &W.sc->hnorm, a, s)); }
    keff_res_kernel<<<1, 1, 0, s>>>(W.sc, rep.res_hist_dev, rep.hist_cap, rep.res_dev);
    return check_launch("keff residual");
  };
  if (rep.res_dev) cudaMemsetAsync(rep.res_dev, 0xff, sizeof(double), s);   // NaN pattern until evaluated
  if (rep.res_hist_dev && rep.hist_cap > 0) fill_kernel<<<1, 256, 0, s>>>(rep.res_hist_dev, rep.hist_cap, -1.0);
  if (mv && !o.warm) TT_TRY(copy_meta(psi, W.B, s));   // first amen_mv guess: Psi_0
  // one fixed-point iteration (Eq. 8), ending with the device decision in sc->flag
  auto iteration = [&]() -> tt_status {
    if (!mv) {
      TT_TRY(matvec_meta(S, psi, W.SP, s));
      { Arena a = sub(); TT_TRY(round_meta(W.SP, o.eps_round, o.rmax, nullptr, nullptr, 0, a, s)); }
      TT_TRY(matvec_meta(F, psi, W.FP, s));
      { Arena a = sub(); TT_TRY(round_meta(W.FP, o.eps_round, o.rmax, nullptr, nullptr, 0, a, s)); }
      TT_TRY(add_meta(W.SP, nullptr, W.FP, &W.sc->kinv, W.B, s));
      { Arena a = sub(); TT_TRY(round_meta(W.B, o.eps_round, o.rmax, nullptr, nullptr, 0, a, s)); }
    } else {
      TT_TRY(add_meta(mat_as_vec(S), nullptr, mat_as_vec(F), &W.sc->kinv, mat_as_vec(W.SF), s));
      TT_TRY(copy_meta(W.z0, W.zmv, s));
      { Arena a = sub(); TT_TRY(amen_mv_meta(W.SF, psi, W.B, W.zmv, o.eps_round, o.mv_max_sweeps, o.rmax, nullptr, a, s)); }
    }
    TT_TRY(copy_meta(W.z0, z, s));
    set_i32_k<<<1, 1, 0, s>>>(W.inner, 0);
    { Arena a = sub(); TT_TRY(amen_solve_meta(H, W.B, psi, z, ao, W.sweeps, nullptr, W.inner, a, s)); }
    { Arena a = sub(); TT_TRY(dot_meta(W.f, psi, &W.sc->s_new, a, s)); }
    keff_after_solve_kernel<<<1, 1, 0, s>>>(W.sc);
    { Arena a = sub(); TT_TRY(orth_meta(psi, -1, W.nrm, a, s)); }
    keff_update_kernel<<<1, 1, 0, s>>>(W.sc, W.nrm, rep.k_hist_dev, rep.sweeps_hist_dev, rep.inner_status_hist_dev,
                                       W.sweeps, W.inner, rep.hist_cap);
    TT_TRY(scale_meta(psi, &W.sc->nrm_inv, 1.0, 0, s));
    if (o.tol_res > 0.0) TT_TRY(residual());
    keff_decide_kernel<<<1, 1, 0, s>>>(W.sc, o.tol_k, o.tol_res, o.max_outer, rep.k_dev, rep.iters_dev, rep.status_dev);
    return check_launch("keff iteration");
  };
  if (device_loops(s)) {   // K11: do { iteration } while (!flag) as a conditional WHILE node
    TT_TRY(dev_while(s, [&](cudaGraphConditionalHandle h) -> tt_status {
      TT_TRY(iteration());
      return cond_from_flag(h, &W.sc->flag, s);
    }));
  } else {
    for (int it = 0; it < o.max_outer; ++it) {
      TT_TRY(iteration());
      int hflag = 0;
      TT_TRY(read_back(&hflag, &W.sc->flag, sizeof(int), s));
      TT_TRY(check_launch("keff iteration"));
      if (hflag) break;
    }
  }
  if (o.tol_res == 0.0) TT_TRY(residual());   // reported once for the final iterate
  return check_launch("keff_fixed_point");
}

__global__ void set_f64_kernel(double *p, double v) { *p = v; }

// internal report -> the caller's keff_report (n history entries; res_hist beyond
// them keeps the "not evaluated" mark -1)
__global__ void keff_copy_out_kernel(const keff_report in, const keff_report out, int n) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (out.k_dev) *out.k_dev = *in.k_dev;
    if (out.iters_dev) *out.iters_dev = *in.iters_dev;
    if (out.status_dev) *out.status_dev = *in.status_dev;
    if (out.res_dev) *out.res_dev = *in.res_dev;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < out.hist_cap; i += gridDim.x * blockDim.x) {
    const bool h = i < n;
    if (out.k_hist_dev && h) out.k_hist_dev[i] = in.k_hist_dev[i];
    if (out.res_hist_dev) out.res_hist_dev[i] = h ? in.res_hist_dev[i] : -1.0;
    if (out.sweeps_hist_dev && h) out.sweeps_hist_dev[i] = in.sweeps_hist_dev[i];
    if (out.inner_status_hist_dev && h) out.inner_status_hist_dev[i] = in.inner_status_hist_dev[i];
  }
}

// keff_fixed_point entry: detect the operator kinds (one read-back), store k0 on
// the device, then enqueue the call — as ONE graph launch in graph mode 2 (the
// outer loop and every sweep loop decided on the device), replayed while the
// operands, workspace and options are the same.
tt_status keff_meta(const MatMeta &H0, const MatMeta &S0, const MatMeta &F0, const VecMeta &psi, const VecMeta &z,
                    double k0, const keff_opts &o, const keff_report &rep, Arena &ar, cudaStream_t s) {
  KeffWS W;
  const Arena ar0 = ar;
  TT_TRY(carve_keff(H0, S0, F0, psi, z, o, ar, W));
  if (!ar.base) return TT_OK;
  if (!ar.ok()) return fail(TT_ERR_CAPACITY, "keff_fixed_point: workspace too small");
  if (!(k0 != 0.0)) return fail(TT_ERR_ARG, "keff_fixed_point: k0 must be nonzero");
  MatMeta H = H0, S = S0, F = F0;
  TT_TRY(detect_ops_kinds(H, S, F, W.kscr, s));
  set_f64_kernel<<<1, 1, 0, s>>>(W.k0buf, k0);
  TT_TRY(check_launch("keff k0"));
  keff_report ir;
  ir.k_dev = W.ok; ir.iters_dev = W.oit; ir.k_hist_dev = W.okh; ir.res_hist_dev = W.orh; ir.hist_cap = KEFF_HIST;
  ir.status_dev = W.ost; ir.sweeps_hist_dev = W.osh; ir.inner_status_hist_dev = W.oih; ir.res_dev = W.ores;
  auto body = [&]() -> tt_status {
    Arena a = ar0;
    return keff_body(H, S, F, psi, z, W.k0buf, o, ir, a, s);
  };
  auto copy_out = [&]() -> tt_status {
    const int n = rep.hist_cap < KEFF_HIST ? rep.hist_cap : KEFF_HIST;
    keff_copy_out_kernel<<<1, 256, 0, s>>>(ir, rep, n < 0 ? 0 : n);
    return check_launch("keff report");
  };
  if (graph_mode() < 2 || stream_capturing(s)) {
    TT_TRY(body());
    return copy_out();
  }
  gmres_fused_grid();   // one-time attribute / occupancy queries outside the capture
  GraphKey key;
  key.add(H); key.add(S); key.add(F); key.add(psi); key.add(z);
  key.add(o.tol_k); key.add(o.tol_res); key.add(o.eps_round); key.add(o.eps_solve);
  const int ii[10] = {o.max_outer, o.rmax, o.max_sweeps, o.kickrank, o.gmres_restart, o.gmres_max_restarts,
                      o.local_dense_max, o.matvec, o.mv_max_sweeps, o.warm};
  key.add(ii);
  key.add(ar0.base);
  key.add(ar0.cap);
  TT_TRY(run_captured(key, s, body));
  return copy_out();
}


// ---------------------------------------------------------------- NEXT-2 ---
// alpha_secant: eq. TT_alpha_eig_fixed_points with the secant
// reading Z32.  For each alpha: H_alpha = round(H + alpha V^{-1}) on the device
// (TT-matrices viewed as TT-vectors with modes m n), then keff_fixed_point
// warm-started from the previous Psi and k.  alpha, k and the secant state stay
// on the device; the host polls one flag per k-eff solve.
namespace {

struct AlphaState {
  double a_prev, a, k_prev, k, one;
  int flag, iters, status;
};

__global__ void alpha_init_kernel(AlphaState *st, double a0) {
  st->a_prev = 0.0; st->a = a0; st->k_prev = 0.0; st->k = 1.0; st->one = 1.0;
  st->flag = 0; st->iters = 0; st->status = 0;
}

__global__ void alpha_update_kernel(AlphaState *st, const double *k_dev, const int *kit_dev, const int *kst_dev,
                                    double a1, double tol, int max_alpha, double *ahist, double *khist, int *ithist,
                                    int hist_cap, double *a_out, double *k_out, int *iters_out, int *status_out) {
  const double k = *k_dev;
  const int it = st->iters;
  if (it < hist_cap) {
    if (ahist) ahist[it] = st->a;
    if (khist) khist[it] = k;
    if (ithist) ithist[it] = *kit_dev;
  }
  st->iters = it + 1;
  if (*kst_dev != 0) {   // the k-eff solve did not converge (or no fission / NaN): stop with its status
    st->status = *kst_dev;
    st->flag = 1;
  } else if (fabs(k - 1.0) <= tol) {
    st->k = k;
    st->flag = 1;
  } else if (st->iters >= max_alpha) {
    st->k = k;
    st->status = TT_ERR_NOCONV;
    st->flag = 1;
  } else if (it == 0) {                                // alpha^(1) = 0.01
    st->a_prev = st->a; st->k_prev = k; st->k = k;
    st->a = a1;
  } else if (fabs(k - st->k_prev) < 1e-14) {           // stagnation
    st->k = k;
    st->status = TT_ERR_NOCONV;
    st->flag = 1;
  } else {                                             // secant on k(alpha) - 1 (Z32)
    const double an = st->a + (1.0 - k) * (st->a - st->a_prev) / (k - st->k_prev);
    st->a_prev = st->a; st->k_prev = k; st->k = k;
    st->a = an;
  }
  if (st->flag) {
    // report the alpha the last k-eff solve used
    if (a_out) *a_out = st->a;
  } else if (a_out) {
    *a_out = st->a;
  }
  if (k_out) *k_out = k;
  if (iters_out) *iters_out = st->iters;
  if (status_out) *status_out = st->status;
}

constexpr int ALPHA_HIST = 256;   // alpha iterations recorded in the histories

__global__ void alpha_copy_out_kernel(const alpha_report in, const alpha_report out, int n) {
  if (threadIdx.x == 0) {
    if (out.alpha_dev) *out.alpha_dev = *in.alpha_dev;
    if (out.k_dev) *out.k_dev = *in.k_dev;
    if (out.iters_dev) *out.iters_dev = *in.iters_dev;
    if (out.status_dev) *out.status_dev = *in.status_dev;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (out.alpha_hist_dev) out.alpha_hist_dev[i] = in.alpha_hist_dev[i];
    if (out.k_hist_dev) out.k_hist_dev[i] = in.k_hist_dev[i];
    if (out.keff_iters_hist_dev) out.keff_iters_hist_dev[i] = in.keff_iters_hist_dev[i];
  }
}

struct AlphaWS {
  MatMeta Ha;
  AlphaState *st;
  double *kk;
  int *kit, *kst;
  float *kscr;
  // internal report (see KeffWS): alpha, k, iterations, status, histories
  double *oa, *ok, *oah, *okh;
  int *oit, *ost, *oith;
  char *sub;
  size_t sub_cap;
};

tt_status carve_alpha(const MatMeta &H, const MatMeta &V, const MatMeta &S, const MatMeta &F, const VecMeta &psi,
                      const VecMeta &z, const alpha_opts &o, Arena &ar, AlphaWS &W) {
  const int d = H.d;
  if (V.d != d) return fail(TT_ERR_SHAPE, "alpha_secant: number of cores differ");
  for (int k = 0; k < d; ++k)
    if (V.m[k] != H.m[k] || V.n[k] != H.n[k]) return fail(TT_ERR_SHAPE, "alpha_secant: V and H shapes differ");
  std::memset(&W, 0, sizeof(W));
  W.Ha = H;
  long long off = 0;
  for (int k = 0; k <= d; ++k) W.Ha.Rcap[k] = (k == 0 || k == d) ? 1 : H.Rcap[k] + V.Rcap[k];
  for (int k = 0; k < d; ++k) {
    W.Ha.off[k] = off;
    off += (long long)W.Ha.Rcap[k] * H.m[k] * H.n[k] * W.Ha.Rcap[k + 1];
  }
  W.Ha.data = ar.take<double>(off);
  W.Ha.R = ar.take<int>(d + 1);
  W.st = ar.take<AlphaState>(1);
  W.kk = ar.take<double>(1);
  W.kit = ar.take<int>(1);
  W.kst = ar.take<int>(1);
  W.kscr = ar.take<float>(KIND_SCRATCH_FLOATS);
  W.oa = ar.take<double>(1);
  W.ok = ar.take<double>(1);
  W.oah = ar.take<double>(ALPHA_HIST);
  W.okh = ar.take<double>(ALPHA_HIST);
  W.oit = ar.take<int>(1);
  W.ost = ar.take<int>(1);
  W.oith = ar.take<int>(ALPHA_HIST);
  size_t mx = keff_ws_bytes(W.Ha, S, F, psi, z, o.keff);
  if (mx == 0) return fail(TT_ERR_SHAPE, "alpha_secant: k-eff operands rejected");
  { Arena c; round_meta(mat_as_vec(W.Ha), 0.0, 1, nullptr, nullptr, 0, c, nullptr); mx = c.used > mx ? c.used : mx; }
  W.sub_cap = mx;
  W.sub = ar.take<char>(mx);
  return TT_OK;
}

}  // namespace

size_t alpha_ws_bytes(const MatMeta &H, const MatMeta &V, const MatMeta &S, const MatMeta &F, const VecMeta &psi,
                      const VecMeta &z, const alpha_opts &o) {
  Arena ar;
  AlphaWS W;
  if (carve_alpha(H, V, S, F, psi, z, o, ar, W) != TT_OK) return 0;
  return ar.used;
}

tt_status alpha_meta(const MatMeta &H0, const MatMeta &V0, const MatMeta &S0, const MatMeta &F0, const VecMeta &psi,
                     const VecMeta &z, const alpha_opts &o, const alpha_report &rep, Arena &ar, cudaStream_t s) {
  AlphaWS W;
  const Arena ar0 = ar;
  TT_TRY(carve_alpha(H0, V0, S0, F0, psi, z, o, ar, W));
  if (!ar.base) return TT_OK;
  if (!ar.ok()) return fail(TT_ERR_CAPACITY, "alpha_secant: workspace too small");
  if (o.max_alpha < 1 || !(o.tol > 0.0)) return fail(TT_ERR_ARG, "alpha_secant: max_alpha >= 1, tol > 0");
  MatMeta H = H0, V = V0, S = S0, F = F0;
  if (!V.kinds_set) TT_TRY(detect_core_kinds(V, W.kscr, s));
  TT_TRY(detect_ops_kinds(H, S, F, W.kscr, s));
  for (int k = 0; k < H.d; ++k) W.Ha.kind[k] = H.kind[k] && V.kind[k];   // H + alpha V^{-1}: block sum
  W.Ha.kinds_set = 1;
  const VecMeta hv = mat_as_vec(H), vv = mat_as_vec(V), av = mat_as_vec(W.Ha);
  keff_report kr;
  std::memset(&kr, 0, sizeof(kr));
  kr.k_dev = W.kk; kr.iters_dev = W.kit; kr.hist_cap = 0; kr.status_dev = W.kst;
  alpha_report ir;
  ir.alpha_dev = W.oa; ir.k_dev = W.ok; ir.iters_dev = W.oit; ir.alpha_hist_dev = W.oah; ir.k_hist_dev = W.okh;
  ir.keff_iters_hist_dev = W.oith; ir.hist_cap = ALPHA_HIST; ir.status_dev = W.ost;
  auto copy_out = [&]() -> tt_status {
    int n = rep.hist_cap < ALPHA_HIST ? rep.hist_cap : ALPHA_HIST;
    n = n < o.max_alpha ? n : o.max_alpha;
    alpha_copy_out_kernel<<<1, 256, 0, s>>>(ir, rep, n < 0 ? 0 : n);
    return check_launch("alpha report");
  };
  // one secant step: H_alpha, the k-eff solve warm-started from the previous Psi
  // and k (the first from k0 = st->k = 1), the device update of alpha
  auto step = [&]() -> tt_status {
    TT_TRY(add_meta(hv, &W.st->one, vv, &W.st->a, av, s));
    { Arena a; a.base = W.sub; a.cap = W.sub_cap; TT_TRY(round_meta(av, o.eps_op, 1 << 30, nullptr, nullptr, 0, a, s)); }
    cudaMemsetAsync(W.kst, 0, sizeof(int), s);
    { Arena a; a.base = W.sub; a.cap = W.sub_cap; TT_TRY(keff_body(W.Ha, S, F, psi, z, &W.st->k, o.keff, kr, a, s)); }
    alpha_update_kernel<<<1, 1, 0, s>>>(W.st, W.kk, W.kit, W.kst, o.alpha1, o.tol, o.max_alpha, ir.alpha_hist_dev,
                                        ir.k_hist_dev, ir.keff_iters_hist_dev, ir.hist_cap, ir.alpha_dev,
                                        ir.k_dev, ir.iters_dev, ir.status_dev);
    return check_launch("alpha iteration");
  };
  auto all = [&]() -> tt_status {
    alpha_init_kernel<<<1, 1, 0, s>>>(W.st, o.alpha0);
    if (device_loops(s))   // K11: the secant loop as a conditional WHILE node
      return dev_while(s, [&](cudaGraphConditionalHandle h) -> tt_status {
        TT_TRY(step());
        return cond_from_flag(h, &W.st->flag, s);
      });
    for (int t = 0; t < o.max_alpha; ++t) {
      TT_TRY(step());
      int hflag = 0;
      TT_TRY(read_back(&hflag, &W.st->flag, sizeof(int), s));
      TT_TRY(check_launch("alpha iteration"));
      if (hflag) break;
    }
    return check_launch("alpha_secant");
  };
  if (graph_mode() < 2 || stream_capturing(s)) {
    TT_TRY(all());
    return copy_out();
  }
  gmres_fused_grid();
  GraphKey key;
  key.add(H); key.add(V); key.add(S); key.add(F); key.add(psi); key.add(z);
  const double dd[6] = {o.alpha0, o.alpha1, o.tol, o.eps_op, o.keff.tol_k, o.keff.tol_res};
  const double de[2] = {o.keff.eps_round, o.keff.eps_solve};
  const int ii[11] = {o.max_alpha, o.keff.max_outer, o.keff.rmax, o.keff.max_sweeps, o.keff.kickrank,
                      o.keff.gmres_restart, o.keff.gmres_max_restarts, o.keff.local_dense_max, o.keff.matvec,
                      o.keff.mv_max_sweeps, o.keff.warm};
  key.add(dd); key.add(de); key.add(ii); key.add(ar0.base); key.add(ar0.cap);
  TT_TRY(run_captured(key, s, all));
  return copy_out();
}

}  // namespace tt

using namespace tt;

extern "C" size_t amen_workspace(const tt_mat *A, const tt_vec *b, const tt_vec *x, const tt_vec *z,
                                 const amen_opts *o) {
  MatMeta Am;
  VecMeta bm, xm, zm;
  if (!o || make_mat_meta(A, Am) || make_vec_meta(b, bm) || make_vec_meta(x, xm) || make_vec_meta(z, zm)) return 0;
  return amen_ws_bytes(Am, bm, xm, zm, o->gmres_restart, o->local_dense_max);
}

extern "C" tt_status amen_solve(const tt_mat *A, const tt_vec *b, tt_vec *x, tt_vec *z, const amen_opts *o,
                                int32_t *sweeps_dev, double *res_dev, void *ws, size_t wsb, tt_stream s) {
  MatMeta Am;
  VecMeta bm, xm, zm;
  TT_TRY(make_mat_meta(A, Am));
  TT_TRY(make_vec_meta(b, bm));
  TT_TRY(make_vec_meta(x, xm));
  TT_TRY(make_vec_meta(z, zm));
  if (!o || !ws) return fail(TT_ERR_ARG, "amen_solve: NULL options or workspace");
  if (o->max_sweeps < 1 || o->rmax < 1 || o->gmres_max_restarts < 1)
    return fail(TT_ERR_ARG, "amen_solve: max_sweeps, rmax, gmres_max_restarts must be >= 1");
  AmenOpts ao;
  ao.eps = o->eps;
  ao.local_tol = o->local_tol;
  ao.max_sweeps = o->max_sweeps;
  ao.rmax = o->rmax;
  ao.restart = o->gmres_restart;
  ao.max_restarts = o->gmres_max_restarts;
  ao.dense_max = o->local_dense_max;
  Arena ar;
  ar.base = (char *)ws;
  ar.cap = wsb;
  return amen_solve_meta(Am, bm, xm, zm, ao, sweeps_dev, res_dev, nullptr, ar, (cudaStream_t)s);
}

extern "C" size_t amen_mv_workspace(const tt_mat *A, const tt_vec *b, const tt_vec *y, const tt_vec *z) {
  MatMeta Am;
  VecMeta bm, ym, zm;
  if (make_mat_meta(A, Am) || make_vec_meta(b, bm) || make_vec_meta(y, ym) || make_vec_meta(z, zm)) return 0;
  return amen_mv_ws_bytes(Am, bm, ym, zm);
}

extern "C" tt_status amen_mv(const tt_mat *A, const tt_vec *b, tt_vec *y, tt_vec *z, double eps, int32_t max_sweeps,
                             int32_t rmax, int32_t *sweeps_dev, void *ws, size_t wsb, tt_stream s) {
  MatMeta Am;
  VecMeta bm, ym, zm;
  TT_TRY(make_mat_meta(A, Am));
  TT_TRY(make_vec_meta(b, bm));
  TT_TRY(make_vec_meta(y, ym));
  TT_TRY(make_vec_meta(z, zm));
  if (!ws) return fail(TT_ERR_ARG, "amen_mv: NULL workspace");
  Arena ar;
  ar.base = (char *)ws;
  ar.cap = wsb;
  return amen_mv_meta(Am, bm, ym, zm, eps, max_sweeps, rmax, sweeps_dev, ar, (cudaStream_t)s);
}

extern "C" size_t keff_workspace(const tt_mat *H, const tt_mat *S, const tt_mat *F, const tt_vec *psi,
                                 const tt_vec *z, const keff_opts *o) {
  MatMeta Hm, Sm, Fm;
  VecMeta pm, zm;
  if (!o || make_mat_meta(H, Hm) || make_mat_meta(S, Sm) || make_mat_meta(F, Fm) || make_vec_meta(psi, pm) ||
      make_vec_meta(z, zm))
    return 0;
  return keff_ws_bytes(Hm, Sm, Fm, pm, zm, *o);
}

extern "C" tt_status keff_fixed_point(const tt_mat *H, const tt_mat *S, const tt_mat *F, tt_vec *psi, tt_vec *z,
                                      double k0, const keff_opts *o, keff_report *rep, void *ws, size_t wsb,
                                      tt_stream s) {
  MatMeta Hm, Sm, Fm;
  VecMeta pm, zm;
  TT_TRY(make_mat_meta(H, Hm));
  TT_TRY(make_mat_meta(S, Sm));
  TT_TRY(make_mat_meta(F, Fm));
  TT_TRY(make_vec_meta(psi, pm));
  TT_TRY(make_vec_meta(z, zm));
  if (!o || !rep || !ws) return fail(TT_ERR_ARG, "keff_fixed_point: NULL options, report or workspace");
  if (o->max_outer < 1 || o->rmax < 1 || o->max_sweeps < 1 || o->gmres_max_restarts < 1 ||
      ((o->matvec == 1 || o->tol_res >= 0.0) && o->mv_max_sweeps < 1))
    return fail(TT_ERR_ARG, "keff_fixed_point: iteration limits must be >= 1");
  if (!rep->k_dev || !rep->iters_dev || !rep->status_dev)
    return fail(TT_ERR_ARG, "keff_fixed_point: k_dev, iters_dev and status_dev are required");
  Arena ar;
  ar.base = (char *)ws;
  ar.cap = wsb;
  return keff_meta(Hm, Sm, Fm, pm, zm, k0, *o, *rep, ar, (cudaStream_t)s);
}

extern "C" size_t alpha_workspace(const tt_mat *H, const tt_mat *V, const tt_mat *S, const tt_mat *F,
                                  const tt_vec *psi, const tt_vec *z, const alpha_opts *o) {
  MatMeta Hm, Vm, Sm, Fm;
  VecMeta pm, zm;
  if (!o || make_mat_meta(H, Hm) || make_mat_meta(V, Vm) || make_mat_meta(S, Sm) || make_mat_meta(F, Fm) ||
      make_vec_meta(psi, pm) || make_vec_meta(z, zm))
    return 0;
  return alpha_ws_bytes(Hm, Vm, Sm, Fm, pm, zm, *o);
}

extern "C" tt_status alpha_secant(const tt_mat *H, const tt_mat *V, const tt_mat *S, const tt_mat *F, tt_vec *psi,
                                  tt_vec *z, const alpha_opts *o, alpha_report *rep, void *ws, size_t wsb,
                                  tt_stream s) {
  MatMeta Hm, Vm, Sm, Fm;
  VecMeta pm, zm;
  TT_TRY(make_mat_meta(H, Hm));
  TT_TRY(make_mat_meta(V, Vm));
  TT_TRY(make_mat_meta(S, Sm));
  TT_TRY(make_mat_meta(F, Fm));
  TT_TRY(make_vec_meta(psi, pm));
  TT_TRY(make_vec_meta(z, zm));
  if (!o || !rep || !ws) return fail(TT_ERR_ARG, "alpha_secant: NULL options, report or workspace");
  const keff_opts &k = o->keff;
  if (k.max_outer < 1 || k.rmax < 1 || k.max_sweeps < 1 || k.gmres_max_restarts < 1 ||
      (k.matvec == 1 && k.mv_max_sweeps < 1))
    return fail(TT_ERR_ARG, "alpha_secant: k-eff iteration limits must be >= 1");
  Arena ar;
  ar.base = (char *)ws;
  ar.cap = wsb;
  return alpha_meta(Hm, Vm, Sm, Fm, pm, zm, *o, *rep, ar, (cudaStream_t)s);
}
