// Host-side factor matrices of the rank-1 per-octant terms of H, S, F
// (§3.2), written independently of the oracle.  One-off
// setup: the caller uploads the factors and sums / rounds them on the device
// with tt_add and tt_round.  Readings: Z3 full-L integral, Z4 full
// scattering matrix, Z5 chi nu_sigma_f^T, Z6 boundary rows as displayed, Z7
// octant-shifted row->cell map, Z12 vertices, Z34 painted boxes.
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

extern "C" int32_t tt_transport_terms(int32_t op, int32_t nv, double extent, int32_t G, int32_t L, const double *mu,
                                      const double *eta, const double *xi, const double *w, int32_t nmat,
                                      const double *sigma_t, const double *sigma_s, const double *nu_sigma_f,
                                      const double *chi, int32_t nbox, const int32_t *box_lo, const int32_t *box_hi,
                                      const int32_t *box_mat, double *out) {
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
