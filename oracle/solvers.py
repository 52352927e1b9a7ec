"""ORACLE (test infrastructure only) — eigenvalue drivers and the AMEn solve.

  keff_dense_power   eq. k_eff_fixed_points with exact solves (LU)
  keff_dense_ges     dominant generalised eigenpair of (H - S) psi = (1/k) F psi (GES)
  gmres              plain restarted GMRES (Saad), modified Gram-Schmidt + Givens
  amen_solve         ALS/AMEn for H x = b in TT (reading Z20)
  keff_tt            eq. TT_k_eff_fixed_points with readings Z16-Z19
  alpha_secant       eq. alpha_eig_fixed_points / TT_alpha_eig_fixed_points
                      with the secant reading Z32, around any k-eff solver
"""
from __future__ import annotations

import math
import numpy as np
import scipy.linalg as sla

from . import tt as ott

# ------------------------------------------------------------ dense ---


def keff_dense_power(H, S, F, psi0=None, k0=1.0, tol=1e-12, max_it=10000, minnorm=False):
    """Eq. 8: psi' = H^{-1} (S + F/k) psi, k' = k sum(F psi') / sum(F psi).
    minnorm=True uses minimum-norm least-squares solves (reflective variant, Z15)."""
    N = H.shape[0]
    psi = np.ones(N) if psi0 is None else psi0.copy()
    k = k0
    if minnorm:
        Hp = np.linalg.pinv(H, rcond=1e-12)
        solve = lambda r: Hp @ r
    else:
        lu = sla.lu_factor(H)
        solve = lambda r: sla.lu_solve(lu, r)
    hist = []
    for it in range(1, max_it + 1):
        src = S @ psi + (F @ psi) / k
        new = solve(src)
        knew = k * np.sum(F @ new) / np.sum(F @ psi)
        psi = new / np.linalg.norm(new)
        hist.append(knew)
        if abs(knew - k) < tol:
            k = knew
            break
        k = knew
    return k, psi, hist


def keff_dense_ges(H, S, F):
    """Dominant eigenvalue of (H - S)^{-1} F (generalised eigenproblem of eq. OpFormkNTE)."""
    M = np.linalg.solve(H - S, F)
    ev, V = np.linalg.eig(M)
    i = int(np.argmax(ev.real))
    return float(ev[i].real), V[:, i].real


# ------------------------------------------------------------ GMRES ---


def gmres(apply, b, x0, tol=1e-12, restart=60, max_restarts=200):
    """Restarted GMRES(m) (Saad & Schultz), modified Gram-Schmidt, Givens rotations.
    Stops when ||b - A x|| <= tol ||b||.  Returns (x, rel_res, iterations)."""
    bn = np.linalg.norm(b)
    if bn == 0.0:
        return np.zeros_like(b), 0.0, 0
    x = x0.copy()
    its = 0
    rel = np.inf
    for _ in range(max_restarts):
        r = b - apply(x)
        beta = np.linalg.norm(r)
        rel = beta / bn
        if rel <= tol:
            break
        m = restart
        V = np.zeros((m + 1, b.size))
        Hh = np.zeros((m + 1, m))
        cs = np.zeros(m); sn = np.zeros(m)
        g = np.zeros(m + 1); g[0] = beta
        V[0] = r / beta
        j_done = 0
        for j in range(m):
            w = apply(V[j])
            for i in range(j + 1):
                Hh[i, j] = w @ V[i]
                w = w - Hh[i, j] * V[i]
            Hh[j + 1, j] = np.linalg.norm(w)
            if Hh[j + 1, j] > 0:
                V[j + 1] = w / Hh[j + 1, j]
            for i in range(j):
                t = cs[i] * Hh[i, j] + sn[i] * Hh[i + 1, j]
                Hh[i + 1, j] = -sn[i] * Hh[i, j] + cs[i] * Hh[i + 1, j]
                Hh[i, j] = t
            den = math.hypot(Hh[j, j], Hh[j + 1, j])
            cs[j] = Hh[j, j] / den if den > 0 else 1.0
            sn[j] = Hh[j + 1, j] / den if den > 0 else 0.0
            Hh[j, j] = den
            Hh[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            its += 1
            j_done = j + 1
            if abs(g[j + 1]) / bn <= tol:
                break
        y = sla.solve_triangular(Hh[:j_done, :j_done], g[:j_done])
        x = x + V[:j_done].T @ y
    r = b - apply(x)
    return x, np.linalg.norm(r) / bn, its


# ------------------------------------------------------------- AMEn ---


def _local_solve(Phi, Ak, Psi, rhs, x0, tol, dense_max, restart):
    ra, m, rap = rhs.shape
    N = rhs.size
    bvec = rhs.reshape(-1, order="F")
    if N <= dense_max:
        B = ott.local_matrix(Phi, Ak, Psi)
        try:
            sol = np.linalg.solve(B, bvec)
        except np.linalg.LinAlgError:                     # reading Z35
            mu = 1e-12 * np.linalg.norm(B)
            sol = np.linalg.solve(B + mu * np.eye(N), bvec)
    else:
        shape = x0.shape

        def app(v):
            return ott.local_apply(Phi, Ak, Psi, v.reshape(shape, order="F")).reshape(-1, order="F")
        sol, _, _ = gmres(app, bvec, x0.reshape(-1, order="F"), tol=tol, restart=restart)
    return sol.reshape(ra, m, rap, order="F")


def amen_solve(A, b, x0, z0, eps=1e-8, max_sweeps=20, rmax=10**9, dense_max=2000,
               local_tol=None, restart=60, trunc=True, verbose=False):
    """AMEn for A x = b in TT (Dolgov & Savostyanov; P:1520-1531 'amen_solve'),
    Galerkin local systems with orthonormal frames (reading Z20):
      * x0: initial guess TT; z0: initial residual-approximation TT (its ranks are
        the kickrank); both are inputs (random draws are passed in).
      * sweeps alternate left->right and right->left; at core k: solve the local
        system (dense if size <= dense_max, else GMRES), truncate by SVD with
        delta = eps ||x_k|| / sqrt(d-1), update the residual core z_k, enrich the
        solution core with the residual projected onto (x frames | z frames),
        re-orthogonalise with QR and move the centre.
      * stop after a sweep whose max local residual (measured before each local
        solve) is <= eps, or whose max relative change of the local solution
        ||x_k^new - x_k^old|| / ||x_k^new|| is <= eps (the solution-change exit of
        TT-Toolbox amen_solve; reading Z20).
    Returns (x, info)."""
    d = len(A)
    x, _ = ott.tt_orthogonalize_rl(x0)
    z, _ = ott.tt_orthogonalize_rl(z0)
    ltol = eps * 0.1 if local_tol is None else local_tol
    one3 = np.ones((1, 1, 1)); one2 = np.ones((1, 1))
    PhiA = [None] * (d + 2); Phib = [None] * (d + 2)
    PhZA = [None] * (d + 2); PhZb = [None] * (d + 2)
    PhiA[0] = one3; Phib[0] = one2; PhZA[0] = one3; PhZb[0] = one2
    PhiA[d + 1] = one3; Phib[d + 1] = one2; PhZA[d + 1] = one3; PhZb[d + 1] = one2
    # index convention here: Phi*[k] (k = 0..d+1) with cores 1-based; left
    # interface over cores 1..k stored at [k], right interface over k..d at [k].
    for k in range(d, 1, -1):
        PhiA[k] = ott.right_update(PhiA[k + 1], x[k - 1], A[k - 1], x[k - 1])
        Phib[k] = ott.right_update_vec(Phib[k + 1], x[k - 1], b[k - 1])
        PhZA[k] = ott.right_update(PhZA[k + 1], z[k - 1], A[k - 1], x[k - 1])
        PhZb[k] = ott.right_update_vec(PhZb[k + 1], z[k - 1], b[k - 1])
    hist = []
    dx_hist = []
    direction = +1
    sweeps = 0
    for sweep in range(max_sweeps):
        sweeps += 1
        maxres = 0.0
        maxdx = 0.0
        order = range(1, d + 1) if direction > 0 else range(d, 0, -1)
        for k in order:
            Ak, bk = A[k - 1], b[k - 1]
            rhs = ott.local_rhs(Phib[k - 1], bk, Phib[k + 1])
            nrhs = np.linalg.norm(rhs)
            Ax = ott.local_apply(PhiA[k - 1], Ak, PhiA[k + 1], x[k - 1])
            res = np.linalg.norm(Ax - rhs) / nrhs if nrhs > 0 else 0.0
            maxres = max(maxres, res)
            sol = _local_solve(PhiA[k - 1], Ak, PhiA[k + 1], rhs, x[k - 1], ltol, dense_max, restart)
            nsol = np.linalg.norm(sol)
            maxdx = max(maxdx, np.linalg.norm(sol - x[k - 1]) / nsol if nsol > 0 else 0.0)
            r0, n, r1 = sol.shape
            last = (k == d) if direction > 0 else (k == 1)
            if last:
                x[k - 1] = sol
                continue
            if direction > 0:
                M = sol.reshape(r0 * n, r1, order="F")
                U, s, Vt = np.linalg.svd(M, full_matrices=False)
                rr = ott.trunc_rank(s, eps * np.linalg.norm(s) / math.sqrt(d - 1), rmax) if trunc else len(s)
                U = U[:, :rr]; SV = s[:rr, None] * Vt[:rr]
                xk = U.reshape(r0, n, rr, order="F")
                xfull = (U @ SV).reshape(r0, n, r1, order="F")
                # residual core for z (z frames on both sides)
                crz = ott.local_rhs(PhZb[k - 1], bk, PhZb[k + 1]) - \
                    ott.local_apply(PhZA[k - 1], Ak, PhZA[k + 1], xfull)
                z0_, zn, z1_ = crz.shape
                Qz, _ = np.linalg.qr(crz.reshape(z0_ * zn, z1_, order="F"))
                z[k - 1] = Qz.reshape(z0_, zn, Qz.shape[1], order="F")
                # fix rank consistency of z_{k+1} (its left rank must match)
                if z[k].shape[0] != Qz.shape[1]:
                    zk1 = np.zeros((Qz.shape[1],) + z[k].shape[1:])
                    mm = min(Qz.shape[1], z[k].shape[0])
                    zk1[:mm] = z[k][:mm]
                    z[k] = zk1
                # enrichment: residual with x frames on the left, z frames on the right
                crs = ott.local_rhs(Phib[k - 1], bk, PhZb[k + 1]) - \
                    ott.local_apply(PhiA[k - 1], Ak, PhZA[k + 1], xfull)
                Ue = np.concatenate([U, crs.reshape(r0 * n, -1, order="F")], axis=1)
                Q, R = np.linalg.qr(Ue)
                q = Q.shape[1]
                SVe = R[:, :rr] @ SV                               # q x r1
                x[k - 1] = Q.reshape(r0, n, q, order="F")
                x[k] = np.einsum("cb,bjd->cjd", SVe, x[k])
                PhiA[k] = ott.left_update(PhiA[k - 1], x[k - 1], Ak, x[k - 1])
                Phib[k] = ott.left_update_vec(Phib[k - 1], x[k - 1], bk)
                PhZA[k] = ott.left_update(PhZA[k - 1], z[k - 1], Ak, x[k - 1])
                PhZb[k] = ott.left_update_vec(PhZb[k - 1], z[k - 1], bk)
            else:
                M = sol.reshape(r0, n * r1, order="F")
                U, s, Vt = np.linalg.svd(M, full_matrices=False)
                rr = ott.trunc_rank(s, eps * np.linalg.norm(s) / math.sqrt(d - 1), rmax) if trunc else len(s)
                US = U[:, :rr] * s[:rr]; Vt = Vt[:rr]
                xfull = (US @ Vt).reshape(r0, n, r1, order="F")
                crz = ott.local_rhs(PhZb[k - 1], bk, PhZb[k + 1]) - \
                    ott.local_apply(PhZA[k - 1], Ak, PhZA[k + 1], xfull)
                z0_, zn, z1_ = crz.shape
                Qz, _ = np.linalg.qr(crz.reshape(z0_, zn * z1_, order="F").T)
                z[k - 1] = Qz.T.reshape(Qz.shape[1], zn, z1_, order="F")
                if z[k - 2].shape[2] != Qz.shape[1]:
                    zk1 = np.zeros(z[k - 2].shape[:2] + (Qz.shape[1],))
                    mm = min(Qz.shape[1], z[k - 2].shape[2])
                    zk1[:, :, :mm] = z[k - 2][:, :, :mm]
                    z[k - 2] = zk1
                crs = ott.local_rhs(PhZb[k - 1], bk, Phib[k + 1]) - \
                    ott.local_apply(PhZA[k - 1], Ak, PhiA[k + 1], xfull)
                Ve = np.concatenate([Vt, crs.reshape(crs.shape[0], n * r1, order="F")], axis=0)
                Q, R = np.linalg.qr(Ve.T)                          # (n r1) x q
                q = Q.shape[1]
                USe = US @ R[:, :rr].T                             # r0 x q
                x[k - 1] = Q.T.reshape(q, n, r1, order="F")
                x[k - 2] = np.einsum("aib,bc->aic", x[k - 2], USe)
                PhiA[k] = ott.right_update(PhiA[k + 1], x[k - 1], Ak, x[k - 1])
                Phib[k] = ott.right_update_vec(Phib[k + 1], x[k - 1], bk)
                PhZA[k] = ott.right_update(PhZA[k + 1], z[k - 1], Ak, x[k - 1])
                PhZb[k] = ott.right_update_vec(PhZb[k + 1], z[k - 1], bk)
        hist.append(maxres)
        dx_hist.append(maxdx)
        if verbose:
            print(f"amen sweep {sweep} dir {direction} maxres {maxres:.3e} ranks {ott.ranks(x)}")
        if maxres <= eps or maxdx <= eps:
            break
        direction = -direction
    return x, {"res_hist": hist, "dx_hist": dx_hist, "sweeps": sweeps}


# ------------------------------------------------------------ amen_mv ---


def amen_mv(A, b, y0, z0, eps=1e-8, max_sweeps=20, rmax=10**9):
    """Fit-based matvec y ~ A b (P:1489-1494 eqn:mv_obj, P:1501-1506 'amen_mv';
    NEXT-1): minimise ||A b - y|| one core at a time without forming the rank R r
    product.  With orthonormal frames of y the local minimiser is the projection
      y_k = Phi^{yAb}_{k-1} A_k Psi^{yAb}_{k+1} b_k
    (Phi^{yAb} = interfaces with test y, operator A, trial b).  Then, as in
    amen_solve: SVD truncation (delta = eps ||y_k|| / sqrt(d-1), rmax), residual
    core z_k = proj_z (A b - y) with z frames on both sides, enrichment of y_k by
    the residual projected on (y frames | z frames), QR, carry.  Sweeps alternate;
    stop when the max relative change of a local core is <= eps.
    Returns (y, info)."""
    d = len(A)
    y, _ = ott.tt_orthogonalize_rl(y0)
    z, _ = ott.tt_orthogonalize_rl(z0)
    one3 = np.ones((1, 1, 1)); one2 = np.ones((1, 1))
    YA = [None] * (d + 2); ZA = [None] * (d + 2); ZY = [None] * (d + 2)
    YA[0] = YA[d + 1] = one3; ZA[0] = ZA[d + 1] = one3; ZY[0] = ZY[d + 1] = one2
    for k in range(d, 1, -1):
        YA[k] = ott.right_update(YA[k + 1], y[k - 1], A[k - 1], b[k - 1])
        ZA[k] = ott.right_update(ZA[k + 1], z[k - 1], A[k - 1], b[k - 1])
        ZY[k] = ott.right_update_vec(ZY[k + 1], z[k - 1], y[k - 1])
    direction = +1
    dx_hist = []
    sweeps = 0
    for sweep in range(max_sweeps):
        sweeps += 1
        maxdx = 0.0
        order = range(1, d + 1) if direction > 0 else range(d, 0, -1)
        for k in order:
            Ak, bk = A[k - 1], b[k - 1]
            sol = ott.local_apply(YA[k - 1], Ak, YA[k + 1], bk)          # projection of A b
            nsol = np.linalg.norm(sol)
            old = y[k - 1]
            if old.shape == sol.shape:
                maxdx = max(maxdx, np.linalg.norm(sol - old) / nsol if nsol > 0 else 0.0)
            else:
                maxdx = max(maxdx, 1.0)
            r0, n, r1 = sol.shape
            last = (k == d) if direction > 0 else (k == 1)
            if last:
                y[k - 1] = sol
                continue
            if direction > 0:
                M = sol.reshape(r0 * n, r1, order="F")
                U, s, Vt = np.linalg.svd(M, full_matrices=False)
                rr = ott.trunc_rank(s, eps * np.linalg.norm(s) / math.sqrt(d - 1), rmax)
                U = U[:, :rr]; SV = s[:rr, None] * Vt[:rr]
                yfull = (U @ SV).reshape(r0, n, r1, order="F")
                crz = ott.local_apply(ZA[k - 1], Ak, ZA[k + 1], bk) - ott.local_rhs(ZY[k - 1], yfull, ZY[k + 1])
                z0_, zn, z1_ = crz.shape
                Qz, _ = np.linalg.qr(crz.reshape(z0_ * zn, z1_, order="F"))
                z[k - 1] = Qz.reshape(z0_, zn, Qz.shape[1], order="F")
                if z[k].shape[0] != Qz.shape[1]:
                    zk1 = np.zeros((Qz.shape[1],) + z[k].shape[1:])
                    mm = min(Qz.shape[1], z[k].shape[0])
                    zk1[:mm] = z[k][:mm]
                    z[k] = zk1
                # enrichment: (y frames | z frames) projection of A b - y
                crs = ott.local_apply(YA[k - 1], Ak, ZA[k + 1], bk) - \
                    np.einsum("aib,cb->aic", yfull, ZY[k + 1])
                Ue = np.concatenate([U, crs.reshape(r0 * n, -1, order="F")], axis=1)
                Q, R = np.linalg.qr(Ue)
                y[k - 1] = Q.reshape(r0, n, Q.shape[1], order="F")
                y[k] = np.einsum("cb,bjd->cjd", R[:, :rr] @ SV, y[k])
                YA[k] = ott.left_update(YA[k - 1], y[k - 1], Ak, bk)
                ZA[k] = ott.left_update(ZA[k - 1], z[k - 1], Ak, bk)
                ZY[k] = ott.left_update_vec(ZY[k - 1], z[k - 1], y[k - 1])
            else:
                M = sol.reshape(r0, n * r1, order="F")
                U, s, Vt = np.linalg.svd(M, full_matrices=False)
                rr = ott.trunc_rank(s, eps * np.linalg.norm(s) / math.sqrt(d - 1), rmax)
                US = U[:, :rr] * s[:rr]; Vt = Vt[:rr]
                yfull = (US @ Vt).reshape(r0, n, r1, order="F")
                crz = ott.local_apply(ZA[k - 1], Ak, ZA[k + 1], bk) - ott.local_rhs(ZY[k - 1], yfull, ZY[k + 1])
                z0_, zn, z1_ = crz.shape
                Qz, _ = np.linalg.qr(crz.reshape(z0_, zn * z1_, order="F").T)
                z[k - 1] = Qz.T.reshape(Qz.shape[1], zn, z1_, order="F")
                if z[k - 2].shape[2] != Qz.shape[1]:
                    zk1 = np.zeros(z[k - 2].shape[:2] + (Qz.shape[1],))
                    mm = min(Qz.shape[1], z[k - 2].shape[2])
                    zk1[:, :, :mm] = z[k - 2][:, :, :mm]
                    z[k - 2] = zk1
                crs = ott.local_apply(ZA[k - 1], Ak, YA[k + 1], bk) - \
                    np.einsum("ab,bic->aic", ZY[k - 1], yfull)
                Ve = np.concatenate([Vt, crs.reshape(crs.shape[0], n * r1, order="F")], axis=0)
                Q, R = np.linalg.qr(Ve.T)
                y[k - 1] = Q.T.reshape(Q.shape[1], n, r1, order="F")
                y[k - 2] = np.einsum("aib,bc->aic", y[k - 2], US @ R[:, :rr].T)
                YA[k] = ott.right_update(YA[k + 1], y[k - 1], Ak, bk)
                ZA[k] = ott.right_update(ZA[k + 1], z[k - 1], Ak, bk)
                ZY[k] = ott.right_update_vec(ZY[k + 1], z[k - 1], y[k - 1])
        dx_hist.append(maxdx)
        if maxdx <= eps:
            break
        direction = -direction
    return y, {"dx_hist": dx_hist, "sweeps": sweeps}


# ------------------------------------------------------------ k-eff ---


def keff_tt(H, S, F, psi0, z0, k0=1.0, tol_k=1e-10, max_outer=200, eps_round=1e-12,
            eps_solve=1e-11, rmax=10**9, max_sweeps=20, dense_max=2000, verbose=False, matvec="exact",
            mv_max_sweeps=10):
    """Eq. TT_k_eff_fixed_points with readings Z16-Z19:
        B = round(S Psi + (1/k) F Psi);  H Psi' = B (AMEn, warm start Psi);
        k' = k <f, Psi'> / <f, Psi>  with f = F^T 1  (Z18);  Psi <- Psi'/||Psi'||.
    matvec="amen_mv": B = amen_mv(S + (1/k) F, Psi) to eps_round, warm-started
    from the previous B (the paper's product).
    Returns (k, Psi, history)."""
    modes = [c.shape[2] for c in F]
    ones = [np.ones((1, n, 1)) for n in modes]
    f, _ = ott.tt_round(ott.tt_matvec_fast(ott.ttm_transpose(F), ones), 1e-14)
    psi, _ = ott.tt_round(psi0, eps_round, rmax)
    nrm = ott.tt_norm(psi)
    psi = ott.tt_scale(psi, 1.0 / nrm)
    k = k0
    s_old = ott.tt_dot(f, psi)
    hist = []
    B = psi
    rows = [c.shape[1] for c in S]
    cols = [c.shape[2] for c in S]
    for tau in range(1, max_outer + 1):
        if matvec == "amen_mv":
            SF = ott.tt_as_ttm(ott.tt_add(ott.ttm_as_tt(S), ott.tt_scale(ott.ttm_as_tt(F), 1.0 / k)), rows, cols)
            B, _ = amen_mv(SF, psi, B, z0, eps=eps_round, max_sweeps=mv_max_sweeps, rmax=rmax)
        else:
            SP, _ = ott.tt_round(ott.tt_matvec_fast(S, psi), eps_round, rmax)
            FP, _ = ott.tt_round(ott.tt_matvec_fast(F, psi), eps_round, rmax)
            B, _ = ott.tt_round(ott.tt_add(SP, ott.tt_scale(FP, 1.0 / k)), eps_round, rmax)
        new, info = amen_solve(H, B, psi, z0, eps=eps_solve, max_sweeps=max_sweeps, rmax=rmax,
                               dense_max=dense_max)
        s_new = ott.tt_dot(f, new)
        if s_old == 0.0:
            raise ZeroDivisionError("no fission source: <f, Psi> = 0")
        knew = k * s_new / s_old
        nn = ott.tt_norm(new)
        psi = ott.tt_scale(new, 1.0 / nn)
        s_old = s_new / nn
        hist.append({"k": knew, "sweeps": info["sweeps"], "ranks": ott.ranks(psi)})
        if verbose:
            print(tau, knew, info["sweeps"], ott.ranks(psi))
        if abs(knew - k) <= tol_k:
            k = knew
            break
        k = knew
    return k, psi, hist


# ------------------------------------------------------------ alpha ---


def alpha_secant(keff_of_alpha, alpha0=0.0, alpha1=0.01, tol=1e-10, max_it=50):
    """Alpha-eigenvalue outer loop.  keff_of_alpha(alpha)
    solves the k-eff problem [alpha V^{-1} + H] Psi = [S + F/k] Psi and returns k.
    alpha^(0) = 0, alpha^(1) = 0.01; then the secant step on
    f(alpha) = k_eff(alpha) - 1 (reading Z32; the printed update at P:1434 and
    P:1444 is dimensionally inconsistent):
        alpha^(t+1) = alpha^(t) + (1 - k^(t)) (alpha^(t) - alpha^(t-1)) / (k^(t) - k^(t-1)).
    Stops when |k^(t) - 1| <= tol.  Returns (alpha, k, history [(alpha, k)])."""
    a_prev, a = alpha0, alpha1
    k_prev = keff_of_alpha(a_prev)
    hist = [(a_prev, k_prev)]
    if abs(k_prev - 1.0) <= tol:
        return a_prev, k_prev, hist
    k = keff_of_alpha(a)
    hist.append((a, k))
    for _ in range(max_it):
        if abs(k - 1.0) <= tol:
            return a, k, hist
        if abs(k - k_prev) < 1e-14:
            raise RuntimeError("alpha secant stagnated: |k(t) - k(t-1)| < 1e-14")
        a_next = a + (1.0 - k) * (a - a_prev) / (k - k_prev)
        a_prev, k_prev = a, k
        a = a_next
        k = keff_of_alpha(a)
        hist.append((a, k))
    raise RuntimeError("alpha secant did not converge")


def alpha_dense(H, V, S, F, tol=1e-10, tol_k=1e-13, minnorm=False):
    """alpha_secant with dense k-eff solves (LU / minimum norm) of H + alpha V^{-1}."""
    def keff(a):
        k, _, _ = keff_dense_power(H + a * V, S, F, tol=tol_k, minnorm=minnorm)
        return k
    return alpha_secant(keff, tol=tol)


def alpha_tt(H, V, S, F, psi0, z0, tol=1e-9, eps_op=1e-13, **keff_kw):
    """alpha_secant with TT k-eff solves (keff_tt) of round(H + alpha V^{-1})
    (TT_alpha_eig_fixed_points); each k-eff solve starts from psi0."""
    def keff(a):
        Ha = ott.tt_as_ttm(ott.tt_round(ott.tt_add(ott.ttm_as_tt(H), ott.tt_scale(ott.ttm_as_tt(V), a)),
                                        eps_op)[0],
                           [c.shape[1] for c in H], [c.shape[2] for c in H])
        k, _, _ = keff_tt(Ha, S, F, psi0, z0, **keff_kw)
        return k
    return alpha_secant(keff, tol=tol)
