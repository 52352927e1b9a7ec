// Host-side factor matrices of the rank-1 per-octant terms of H, S, F
// (§3.2), written independently of the oracle.  One-off
// setup: the caller uploads the factors and sums / rounds them on the device
// with tt_add and tt_round.  Readings: Z3 full-L integral, Z4 full
// scattering matrix, Z5 chi nu_sigma_f^T, Z6 boundary rows as displayed, Z7
// octant-shifted row->cell map, Z12 vertices, Z34 painted boxes.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "tt_common.cuh"

namespace {

struct Mat {
  int n;
  std::vector<double> a;  // column-major n x n
  explicit Mat(int n_) : n(n_), a((size_t)n_ * n_, 0.0) {}
  double &at(int i, int j) { return a[(size_t)i + (size_t)n * j]; }
};

// D^+ (P:1094-1101): (1/h)(ψ_i - ψ_{i-1}) rows, row 0 = ψ_0/h.  D^- (P:1106-1113).
Mat diff(int s, int n, double h) {
  Mat M(n);
  for (int i = 0; i < n; ++i) {
    if (s > 0) {
      M.at(i, i) = 1.0 / h;
      if (i > 0) M.at(i, i - 1) = -1.0 / h;
    } else {
      M.at(i, i) = -1.0 / h;
      if (i + 1 < n) M.at(i, i + 1) = 1.0 / h;
    }
  }
  return M;
}

// Ip^+ / Ip^- (P:1130-1148); no-BC variants zero the inflow row.
Mat interp(int s, int n, bool noBC) {
  Mat M(n);
  for (int i = 0; i < n; ++i) {
    M.at(i, i) = 0.5;
    if (s > 0 && i > 0) M.at(i, i - 1) = 0.5;
    if (s < 0 && i + 1 < n) M.at(i, i + 1) = 0.5;
  }
  if (noBC) {
    const int row = s > 0 ? 0 : n - 1;
    for (int j = 0; j < n; ++j) M.at(row, j) = 0.0;
  }
  return M;
}

// rows whose (octant-shifted, clamped) cell lies in [lo, hi)  (Z7, Z34)
Mat row_indicator(int s, int n, int lo, int hi) {
  Mat M(n);
  for (int i = 0; i < n; ++i) {
    int c = i - (s > 0 ? 1 : 0);
    c = c < 0 ? 0 : (c > n - 2 ? n - 2 : c);
    M.at(i, i) = (c >= lo && c < hi) ? 1.0 : 0.0;
  }
  return M;
}

Mat mul(const Mat &A, const Mat &B) {
  Mat C(A.n);
  for (int j = 0; j < A.n; ++j)
    for (int k = 0; k < A.n; ++k) {
      const double b = B.a[(size_t)k + (size_t)A.n * j];
      if (b == 0.0) continue;
      for (int i = 0; i < A.n; ++i) C.a[(size_t)i + (size_t)A.n * j] += A.a[(size_t)i + (size_t)A.n * k] * b;
    }
  return C;
}

struct Term {
  Mat fx, fy, fz, fa, fg;
};

}  // namespace

// ------------------------------------------------ Alg. 1 ---
// Device QTT-matrix of a 2^l x 2^l factor: the tensor T(i_0, .., i_{l-1}) with
// mode index i_t = (row bit t) + 2 (column bit t) (bits LSB first, Z28) is
// written as an EXACT TT with index-forwarding cores — cores t < h carry the
// digits i_0..i_t in their right rank index, cores t > h carry i_t..i_{l-1} in
// their left rank index, core h = floor(l/2) holds the n^2 entries of the
// factor — ranks 4^min(t, l-t) (<= n); tt_round of that TT to eps is the TT-SVD
// of T (rounding an exact TT = TT-SVD with the same per-bond rule, Oseledets
// 2011 / reading Z21), i.e. Alg. 1's "compute G_k's QTT-matrix format".
namespace tt {
namespace {
__global__ void qtt_forward_kernel(const VecMeta q, int l, int n, const double *__restrict__ M) {
  const int t = blockIdx.y, h = l / 2;
  auto rk = [&](int b) { int e = b < l - b ? b : l - b; return 1 << (2 * e); };
  const int r0 = rk(t), r1 = rk(t + 1);
  double *core = q.data + q.off[t];
  const long long total = (long long)r0 * 4 * r1;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int a = (int)(e % r0);
    const long long rest = e / r0;
    const int i = (int)(rest % 4), b = (int)(rest / 4);
    double v;
    if (t < h) {          // left forwarding: b = a + r0 i
      v = (b == a + r0 * i) ? 1.0 : 0.0;
    } else if (t > h) {   // right forwarding: a = i + 4 b
      v = (a == i + 4 * b) ? 1.0 : 0.0;
    } else {              // data core: a = digits 0..h-1, b = digits h+1..l-1
      int row = 0, col = 0, s = 0;
      for (int k = 0; k < h; ++k, ++s) {
        const int dg = (a >> (2 * k)) & 3;
        row |= (dg & 1) << s;
        col |= (dg >> 1) << s;
      }
      row |= (i & 1) << s;
      col |= (i >> 1) << s;
      ++s;
      for (int k = 0; k < l - h - 1; ++k, ++s) {
        const int dg = (b >> (2 * k)) & 3;
        row |= (dg & 1) << s;
        col |= (dg >> 1) << s;
      }
      v = M[row + (long long)n * col];
    }
    core[e] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    q.r[t] = r0;
    if (t == l - 1) q.r[t + 1] = 1;
  }
}

tt_status qtt_check(int32_t n, const VecMeta &qm, int &l) {
  l = 0;
  while ((1 << l) < n) ++l;
  if (n < 2 || (1 << l) != n) return fail(TT_ERR_ARG, "tt_qtt_matrix_dev: n must be a power of two >= 2");
  if (qm.d != l) return fail(TT_ERR_SHAPE, "tt_qtt_matrix_dev: q must have log2(n) cores");
  for (int t = 0; t < l; ++t) {
    const int e = t < l - t ? t : l - t;
    if (qm.n[t] != 4) return fail(TT_ERR_SHAPE, "tt_qtt_matrix_dev: q modes must be 4");
    if (qm.rcap[t] < (1 << (2 * e))) return fail(TT_ERR_CAPACITY, "tt_qtt_matrix_dev: rank capacity below 4^min(t, l-t)");
  }
  return TT_OK;
}
}  // namespace
}  // namespace tt

extern "C" size_t tt_qtt_matrix_dev_workspace(const tt_vec *q) {
  tt::VecMeta qm;
  if (tt::make_vec_meta(q, qm) != TT_OK) return 0;
  tt::Arena ar;
  tt::round_meta(qm, 0.0, 1, nullptr, nullptr, 0, ar, nullptr);
  return ar.used;
}

extern "C" tt_status tt_qtt_matrix_dev(int32_t n, const double *M, double eps, tt_vec *q, void *ws, size_t wsb,
                                       tt_stream s) {
  tt::VecMeta qm;
  TT_TRY(tt::make_vec_meta(q, qm));
  int l = 0;
  TT_TRY(tt::qtt_check(n, qm, l));
  if (!M || !ws) return tt::fail(TT_ERR_ARG, "tt_qtt_matrix_dev: NULL matrix or workspace");
  const cudaStream_t st = (cudaStream_t)s;
  tt::qtt_forward_kernel<<<dim3(64, l), 256, 0, st>>>(qm, l, n, M);
  TT_TRY(tt::check_launch("qtt_forward"));
  tt::Arena ar;
  ar.base = (char *)ws;
  ar.cap = wsb;
  return tt::round_meta(qm, eps, 1 << 30, nullptr, nullptr, 0, ar, st);
}

// 1-D slab: the 3-D construction restricted to the x factor, the
// two half-range blocks (mu < 0, mu > 0) playing the octants.  Homogeneous
// material; each term writes [F_x (nv^2), F_angle (L^2), F_group (G^2)].
extern "C" int32_t tt_transport_terms_1d(int32_t op, int32_t nv, double extent, int32_t G, int32_t L,
                                         const double *mu, const double *w, const double *sigma_t,
                                         const double *sigma_s, const double *nu_sigma_f, const double *chi,
                                         double *out) {
  if (op < 0 || op > 2 || nv < 2 || G < 1 || L < 1 || !mu || !w || !sigma_t || !sigma_s || !nu_sigma_f || !chi) {
    tt::set_error("tt_transport_terms_1d: invalid argument");
    return -1;
  }
  const double h = extent / (nv - 1);
  std::vector<Mat> fac;
  int nt = 0;
  for (int sx : {-1, 1}) {
    Mat Cb(L), Q(L), Intg(L);
    for (int l = 0; l < L; ++l) {
      if ((mu[l] > 0) != (sx > 0)) continue;
      Cb.at(l, l) = 1.0;
      Q.at(l, l) = mu[l];
      for (int lp = 0; lp < L; ++lp) Intg.at(l, lp) = w[lp];
    }
    Mat E(G);
    if (op == 0) {
      Mat IG(G);
      for (int g = 0; g < G; ++g) { IG.at(g, g) = 1.0; E.at(g, g) = sigma_t[g]; }
      fac.push_back(diff(sx, nv, h)); fac.push_back(Q); fac.push_back(IG);
      fac.push_back(interp(sx, nv, false)); fac.push_back(Cb); fac.push_back(E);
      nt += 2;
    } else {
      for (int g = 0; g < G; ++g)
        for (int gp = 0; gp < G; ++gp)
          E.at(g, gp) = (op == 1) ? sigma_s[g + (size_t)G * gp] : chi[g] * nu_sigma_f[gp];
      fac.push_back(interp(sx, nv, true)); fac.push_back(Intg); fac.push_back(E);
      nt += 1;
    }
  }
  if (out) {
    double *p = out;
    for (const Mat &M : fac) {
      std::memcpy(p, M.a.data(), M.a.size() * sizeof(double));
      p += M.a.size();
    }
  }
  return nt;
}

static int32_t transport_terms_impl(int32_t op, int32_t nv, double extent, int32_t G, int32_t L, const double *mu,
                                    const double *eta, const double *xi, const double *w, int32_t nmat,
                                    const double *sigma_t, const double *sigma_s, const double *nu_sigma_f,
                                    const double *chi, int32_t nbox, const int32_t *box_lo, const int32_t *box_hi,
                                    const int32_t *box_mat, int32_t reflective, double *out);

extern "C" int32_t tt_transport_terms(int32_t op, int32_t nv, double extent, int32_t G, int32_t L, const double *mu,
                                      const double *eta, const double *xi, const double *w, int32_t nmat,
                                      const double *sigma_t, const double *sigma_s, const double *nu_sigma_f,
                                      const double *chi, int32_t nbox, const int32_t *box_lo, const int32_t *box_hi,
                                      const int32_t *box_mat, double *out) {
  return transport_terms_impl(op, nv, extent, G, L, mu, eta, xi, w, nmat, sigma_t, sigma_s, nu_sigma_f, chi, nbox,
                              box_lo, box_hi, box_mat, 0, out);
}

// Reflective variant of configs[0] (reading Z15; not in the paper): the H
// terms of octant b are restricted to its interior rows (no axis on an inflow
// face); every inflow-face row carries psi_l - psi_refl(l) = 0, where refl
// negates the cosine of the first inflow axis in (x, y, z) order:
//   sum_b sum_a E^a_x (x) E^a_y (x) E^a_z (x) (C_b - R_{a,b}) (x) I_G.
// S and F are unchanged (their inflow-face rows are already zero).
extern "C" int32_t tt_transport_terms_reflective(int32_t op, int32_t nv, double extent, int32_t G, int32_t L,
                                                 const double *mu, const double *eta, const double *xi,
                                                 const double *w, int32_t nmat, const double *sigma_t,
                                                 const double *sigma_s, const double *nu_sigma_f, const double *chi,
                                                 int32_t nbox, const int32_t *box_lo, const int32_t *box_hi,
                                                 const int32_t *box_mat, double *out) {
  return transport_terms_impl(op, nv, extent, G, L, mu, eta, xi, w, nmat, sigma_t, sigma_s, nu_sigma_f, chi, nbox,
                              box_lo, box_hi, box_mat, 1, out);
}

static int32_t transport_terms_impl(int32_t op, int32_t nv, double extent, int32_t G, int32_t L, const double *mu,
                                    const double *eta, const double *xi, const double *w, int32_t nmat,
                                    const double *sigma_t, const double *sigma_s, const double *nu_sigma_f,
                                    const double *chi, int32_t nbox, const int32_t *box_lo, const int32_t *box_hi,
                                    const int32_t *box_mat, int32_t reflective, double *out) {
  if (op < 0 || op > 2 || nv < 2 || G < 1 || L < 1 || nmat < 1 || nbox < 0 || !mu || !eta || !xi || !w || !sigma_t ||
      !sigma_s || !nu_sigma_f || !chi || (nbox > 0 && (!box_lo || !box_hi || !box_mat))) {
    tt::set_error("tt_transport_terms: invalid argument");
    return -1;
  }
  const double h = extent / (nv - 1);
  // parent material of each box: the material painted at its first cell before it (nested/disjoint boxes)
  std::vector<int> parent(nbox, 0);
  for (int t = 0; t < nbox; ++t) {
    int p = 0;
    for (int u = 0; u < t; ++u) {
      bool inside = true;
      for (int a = 0; a < 3; ++a)
        inside = inside && box_lo[3 * t + a] >= box_lo[3 * u + a] && box_lo[3 * t + a] < box_hi[3 * u + a];
      if (inside) p = box_mat[u];
    }
    parent[t] = p;
  }
  std::vector<Term> terms;
  auto push = [&](const Mat &fx, const Mat &fy, const Mat &fz, const Mat &fa, const Mat &fg) {
    terms.push_back(Term{fx, fy, fz, fa, fg});
  };
  for (int b = 0; b < 8; ++b) {
    const int sx = (b & 1) ? 1 : -1, sy = (b & 2) ? 1 : -1, sz = (b & 4) ? 1 : -1;
    auto in_oct = [&](int l) {
      return ((mu[l] > 0) == (sx > 0)) && ((eta[l] > 0) == (sy > 0)) && ((xi[l] > 0) == (sz > 0));
    };
    Mat Cb(L), Qmu(L), Qeta(L), Qxi(L), Intg(L);
    for (int l = 0; l < L; ++l) {
      if (!in_oct(l)) continue;
      Cb.at(l, l) = 1.0;
      Qmu.at(l, l) = mu[l];
      Qeta.at(l, l) = eta[l];
      Qxi.at(l, l) = xi[l];
      for (int lp = 0; lp < L; ++lp) Intg.at(l, lp) = w[lp];   // Z3 full-L
    }
    Mat Dx = diff(sx, nv, h), Dy = diff(sy, nv, h), Dz = diff(sz, nv, h);
    Mat Ix = interp(sx, nv, false), Iy = interp(sy, nv, false), Iz = interp(sz, nv, false);
    Mat Nx = interp(sx, nv, true), Ny = interp(sy, nv, true), Nz = interp(sz, nv, true);
    auto energy = [&](int kind, int m1, int m0) {  // kind 0: diag sigma_t, 1: sigma_s, 2: chi nuSf^T; m1 - m0 (m0 < 0: none)
      Mat E(G);
      for (int g = 0; g < G; ++g)
        for (int gp = 0; gp < G; ++gp) {
          double v = 0.0;
          if (kind == 0) {
            if (g == gp) v = sigma_t[m1 * G + g] - (m0 >= 0 ? sigma_t[m0 * G + g] : 0.0);
          } else if (kind == 1) {
            v = sigma_s[(size_t)m1 * G * G + g + (size_t)G * gp] - (m0 >= 0 ? sigma_s[(size_t)m0 * G * G + g + (size_t)G * gp] : 0.0);
          } else {
            v = chi[g] * (nu_sigma_f[m1 * G + gp] - (m0 >= 0 ? nu_sigma_f[m0 * G + gp] : 0.0));
          }
          E.at(g, gp) = v;
        }
      return E;
    };
    auto nonzero = [](const Mat &M) {
      for (double v : M.a)
        if (v != 0.0) return true;
      return false;
    };
    if (op == 0) {
      Mat IG(G);
      for (int g = 0; g < G; ++g) IG.at(g, g) = 1.0;
      const size_t first = terms.size();
      push(Dx, Iy, Iz, Qmu, IG);                  // H_x^{TT,b}
      push(Ix, Dy, Iz, Qeta, IG);                 // H_y^{TT,b}
      push(Ix, Iy, Dz, Qxi, IG);                  // H_z^{TT,b}
      push(Ix, Iy, Iz, Cb, energy(0, 0, -1));     // H_sigma^{TT,b}
      for (int t = 0; t < nbox; ++t) {
        Mat E = energy(0, box_mat[t], parent[t]);
        if (!nonzero(E)) continue;
        push(mul(row_indicator(sx, nv, box_lo[3 * t], box_hi[3 * t]), Ix),
             mul(row_indicator(sy, nv, box_lo[3 * t + 1], box_hi[3 * t + 1]), Iy),
             mul(row_indicator(sz, nv, box_lo[3 * t + 2], box_hi[3 * t + 2]), Iz), Cb, E);
      }
      if (reflective) {
        // interior-row masks of this octant (vertex not on its inflow face)
        Mat Px(nv), Py(nv), Pz(nv), Ox(nv), Oy(nv), Oz(nv), Id(nv);
        for (int i = 0; i < nv; ++i) {
          Id.at(i, i) = 1.0;
          Px.at(i, i) = (i != (sx > 0 ? 0 : nv - 1)) ? 1.0 : 0.0;
          Py.at(i, i) = (i != (sy > 0 ? 0 : nv - 1)) ? 1.0 : 0.0;
          Pz.at(i, i) = (i != (sz > 0 ? 0 : nv - 1)) ? 1.0 : 0.0;
          Ox.at(i, i) = 1.0 - Px.at(i, i);
          Oy.at(i, i) = 1.0 - Py.at(i, i);
          Oz.at(i, i) = 1.0 - Pz.at(i, i);
        }
        for (size_t t = first; t < terms.size(); ++t) {
          terms[t].fx = mul(Px, terms[t].fx);
          terms[t].fy = mul(Py, terms[t].fy);
          terms[t].fz = mul(Pz, terms[t].fz);
        }
        // face rows, by first inflow axis a: psi_l - psi_{refl_a(l)} = 0
        for (int a = 0; a < 3; ++a) {
          Mat Ang(L);
          for (int l = 0; l < L; ++l) {
            if (!in_oct(l)) continue;
            double t3[3] = {mu[l], eta[l], xi[l]};
            t3[a] = -t3[a];
            int best = 0;
            double bd = 1e300;
            for (int lp = 0; lp < L; ++lp) {
              const double d0 = mu[lp] - t3[0], d1 = eta[lp] - t3[1], d2 = xi[lp] - t3[2];
              const double dd = d0 * d0 + d1 * d1 + d2 * d2;
              if (dd < bd) { bd = dd; best = lp; }
            }
            Ang.at(l, l) += 1.0;
            Ang.at(l, best) -= 1.0;
          }
          if (a == 0) push(Ox, Id, Id, Ang, IG);
          else if (a == 1) push(Px, Oy, Id, Ang, IG);
          else push(Px, Py, Oz, Ang, IG);
        }
      }
    } else {
      const int kind = op == 1 ? 1 : 2;          // S (Z4) / F (Z5)
      push(Nx, Ny, Nz, Intg, energy(kind, 0, -1));
      for (int t = 0; t < nbox; ++t) {
        Mat E = energy(kind, box_mat[t], parent[t]);
        if (!nonzero(E)) continue;
        push(mul(row_indicator(sx, nv, box_lo[3 * t], box_hi[3 * t]), Nx),
             mul(row_indicator(sy, nv, box_lo[3 * t + 1], box_hi[3 * t + 1]), Ny),
             mul(row_indicator(sz, nv, box_lo[3 * t + 2], box_hi[3 * t + 2]), Nz), Intg, E);
      }
    }
  }
  if (out) {
    double *p = out;
    for (const Term &t : terms) {
      for (const Mat *M : {&t.fx, &t.fy, &t.fz, &t.fa, &t.fg}) {
        std::memcpy(p, M->a.data(), M->a.size() * sizeof(double));
        p += M->a.size();
      }
    }
  }
  return (int32_t)terms.size();
}

// Velocity operator V^{-1} of the alpha problem (eq.
// Discretized_alphaNTE P:341-349): per octant (bci) the rank-1 term
//   diag(1/v) o (C_b (x) I) o Ip_z o Ip_y o Ip_x
// (the collision term's structure with sigma_t -> 1/v, uniform in space).
// dim 3: terms [F_x, F_y, F_z, F_angle, F_group]; reflective (Z15) restricts
// them to the octant's interior rows (face rows carry only the reflection).
// dim 1: terms [F_x, F_angle, F_group] over the two half-range blocks.
extern "C" int32_t tt_velocity_terms(int32_t dim, int32_t nv, int32_t G, int32_t L, const double *mu,
                                     const double *eta, const double *xi, const double *inv_v, int32_t reflective,
                                     double *out) {
  if ((dim != 1 && dim != 3) || nv < 2 || G < 1 || L < 1 || !mu || !inv_v ||
      (dim == 3 && (!eta || !xi)) || (dim == 1 && reflective)) {
    tt::set_error("tt_velocity_terms: invalid argument");
    return -1;
  }
  Mat E(G);
  for (int g = 0; g < G; ++g) E.at(g, g) = inv_v[g];
  std::vector<const Mat *> order;
  std::vector<Mat> keep;
  keep.reserve(8 * 5);
  const int nb = dim == 3 ? 8 : 2;
  for (int b = 0; b < nb; ++b) {
    const int sx = (b & 1) ? 1 : -1, sy = (b & 2) ? 1 : -1, sz = (b & 4) ? 1 : -1;
    Mat Cb(L);
    for (int l = 0; l < L; ++l) {
      bool in = (mu[l] > 0) == (sx > 0);
      if (dim == 3) in = in && ((eta[l] > 0) == (sy > 0)) && ((xi[l] > 0) == (sz > 0));
      if (in) Cb.at(l, l) = 1.0;
    }
    if (dim == 1) {
      keep.push_back(interp(sx, nv, false));
      keep.push_back(Cb);
      keep.push_back(E);
      continue;
    }
    Mat Ix = interp(sx, nv, false), Iy = interp(sy, nv, false), Iz = interp(sz, nv, false);
    if (reflective) {
      Mat Px(nv), Py(nv), Pz(nv);
      for (int i = 0; i < nv; ++i) {
        Px.at(i, i) = (i != (sx > 0 ? 0 : nv - 1)) ? 1.0 : 0.0;
        Py.at(i, i) = (i != (sy > 0 ? 0 : nv - 1)) ? 1.0 : 0.0;
        Pz.at(i, i) = (i != (sz > 0 ? 0 : nv - 1)) ? 1.0 : 0.0;
      }
      Ix = mul(Px, Ix); Iy = mul(Py, Iy); Iz = mul(Pz, Iz);
    }
    keep.push_back(Ix); keep.push_back(Iy); keep.push_back(Iz); keep.push_back(Cb); keep.push_back(E);
  }
  if (out) {
    double *p = out;
    for (const Mat &M : keep) {
      std::memcpy(p, M.a.data(), M.a.size() * sizeof(double));
      p += M.a.size();
    }
  }
  (void)order;
  return nb;
}
