"""ORACLE (test infrastructure only) — TT algebra in plain fp64 NumPy.

Cores are NumPy arrays:
  TT-vector core  G_k : shape (r_{k-1}, n_k, r_k)          PAPER.md P:492-512 (eqn:TT_def_element)
  TT-matrix core  A_k : shape (R_{k-1}, m_k, n_k, R_k)     PAPER.md P:670-692 (eqn:TT-matrix-componentwise)
with (i_k, j_k) = (row/output, column/input), P:654-656 (reading Z27).
The full tensor is linearised with the FIRST core fastest (reading Z28):
  lin(i_1..i_d) = i_1 + n_1 (i_2 + n_2 (... )).
No blocking, fusion or reordering beyond the textbook definitions.
"""
from __future__ import annotations

import math
import numpy as np

# ----------------------------------------------------------------- basics ---


def ranks(cores):
    return [c.shape[0] for c in cores] + [cores[-1].shape[-1]]


def modes(cores):
    return [c.shape[1] for c in cores]


def tt_full(cores) -> np.ndarray:
    """Dense vector of a TT-vector, eqn:TT-vector:
    X(i_1..i_d) = G_1(i_1) G_2(i_2) ... G_d(i_d)."""
    T = np.ones((1, 1))                       # [lin so far, alpha]
    for G in cores:
        r0, n, r1 = G.shape
        N = T.shape[0]
        new = np.zeros((N, n, r1))
        for i in range(n):
            new[:, i, :] = T @ G[:, i, :]     # matrix product of the slices
        T = new.reshape(N * n, r1, order="F")  # lin' = lin + N * i
    return T[:, 0]


def ttm_full(cores) -> np.ndarray:
    """Dense matrix of a TT-matrix, eqn:TT-matrix-compact:
    A(i, j) = A_1(i_1, j_1) ... A_d(i_d, j_d), rows/cols linearised first-fastest."""
    T = np.ones((1, 1, 1))                    # [row lin, col lin, alpha]
    for A in cores:
        R0, m, n, R1 = A.shape
        Nr, Nc = T.shape[0], T.shape[1]
        new = np.zeros((Nr, m, Nc, n, R1))
        for i in range(m):
            for j in range(n):
                new[:, i, :, j, :] = np.einsum("rca,ab->rcb", T, A[:, i, j, :])
        T = new.reshape(Nr * m, Nc * n, R1, order="F")
    return T[:, :, 0]


def rank1_ttm(factors):
    """eqn:TT_matrices: A = A_1 o A_2 o ... o A_d, each core [1,m,n,1]."""
    return [np.asarray(F, dtype=np.float64).reshape(1, F.shape[0], F.shape[1], 1) for F in factors]


# ------------------------------------------------------------- exact ops ---


def tt_matvec(A, X):
    """Exact TT matvec (P:1501-1506 'explicit and exact algorithm').
    Y_k[rho, i, rho'] = sum_j A_k[a, i, j, a'] X_k[b, j, b'],
    rho = a + R_{k-1} b, rho' = a' + R_k b' (operator rank fastest)."""
    assert len(A) == len(X)
    Y = []
    for Ak, Xk in zip(A, X):
        R0, m, n, R1 = Ak.shape
        r0, nx, r1 = Xk.shape
        if n != nx:
            raise ValueError("shape mismatch")
        Yk = np.zeros((R0 * r0, m, R1 * r1))
        for a in range(R0):
            for b in range(r0):
                for a1 in range(R1):
                    for b1 in range(r1):
                        # sum over j: A[a,:,:,a1] @ X[b,:,b1]
                        Yk[a + R0 * b, :, a1 + R1 * b1] = Ak[a, :, :, a1] @ Xk[b, :, b1]
        Y.append(Yk)
    return Y


def tt_matvec_fast(A, X):
    """Same result as tt_matvec via one einsum per core (for sizes where the loop
    form is slow).  Pinned to tt_matvec element by element in tests."""
    Y = []
    for Ak, Xk in zip(A, X):
        R0, m, n, R1 = Ak.shape
        r0, _, r1 = Xk.shape
        T = np.einsum("aijc,bjd->abicd", Ak, Xk)          # [a, b, i, a', b']
        Y.append(T.reshape(R0 * r0, m, R1 * r1, order="F"))  # rho = a + R0 b
    return Y


def tt_add(X, Y):
    """Sum of TT tensors: block-diagonal core concatenation, ranks add."""
    d = len(X)
    if d != len(Y) or modes(X) != modes(Y):
        raise ValueError("shape mismatch")
    if d == 1:
        return [X[0] + Y[0]]
    Z = []
    for k in range(d):
        a0, n, a1 = X[k].shape
        b0, _, b1 = Y[k].shape
        if k == 0:
            C = np.zeros((1, n, a1 + b1))
            C[:, :, :a1] = X[k]; C[:, :, a1:] = Y[k]
        elif k == d - 1:
            C = np.zeros((a0 + b0, n, 1))
            C[:a0] = X[k]; C[a0:] = Y[k]
        else:
            C = np.zeros((a0 + b0, n, a1 + b1))
            C[:a0, :, :a1] = X[k]; C[a0:, :, a1:] = Y[k]
        Z.append(C)
    return Z


def tt_scale(X, c):
    Z = [G.copy() for G in X]
    Z[0] = Z[0] * c
    return Z


def ttm_as_tt(A):
    """View a TT-matrix as a TT-vector with mode m_k n_k (row index fastest)."""
    return [Ak.reshape(Ak.shape[0], Ak.shape[1] * Ak.shape[2], Ak.shape[3], order="F") for Ak in A]


def tt_as_ttm(X, rows, cols):
    return [Xk.reshape(Xk.shape[0], m, n, Xk.shape[2], order="F") for Xk, m, n in zip(X, rows, cols)]


def ttm_transpose(A):
    return [np.transpose(Ak, (0, 2, 1, 3)).copy() for Ak in A]


def tt_dot(X, Y) -> float:
    """<X, Y> by left-to-right chain contraction (P:395/P:1409 use sums)."""
    W = np.ones((1, 1))                       # [alpha_X, alpha_Y]
    for Xk, Yk in zip(X, Y):
        W = np.einsum("ab,aic,bid->cd", W, Xk, Yk)
    return float(W[0, 0])


def tt_sum(X) -> float:
    """Sum of all entries = <X, ones>."""
    W = np.ones((1,))
    for Xk in X:
        W = np.einsum("a,aib->b", W, Xk)
    return float(W[0])


def tt_norm(X) -> float:
    return math.sqrt(max(tt_dot(X, X), 0.0))


# ------------------------------------------------- orthogonalize / round ---


def tt_orthogonalize_rl(X):
    """Right-to-left orthogonalization: for k = d..2,
    Householder QR (LAPACK geqrf/orgqr via numpy) of the transposed right
    unfolding M^T = Q R, (n_k r_k) x r_{k-1}; core k <- Q^T; core k-1 <- core k-1 x_3 R^T.
    Returns (cores, norm) with norm = ||core_1||_F = ||X||_F."""
    Y = [G.copy() for G in X]
    d = len(Y)
    for k in range(d - 1, 0, -1):
        r0, n, r1 = Y[k].shape
        M = Y[k].reshape(r0, n * r1, order="F")          # right unfolding
        Q, R = np.linalg.qr(M.T)                          # economy: Q (n r1 x q), R (q x r0)
        q = Q.shape[1]
        Y[k] = Q.T.reshape(q, n, r1, order="F")
        Y[k - 1] = np.einsum("aib,cb->aic", Y[k - 1], R)
    return Y, float(np.linalg.norm(Y[0]))


def tt_orthogonalize_lr(X):
    """Left-to-right mirror: QR of the left unfolding (r_{k-1} n_k) x r_k."""
    Y = [G.copy() for G in X]
    d = len(Y)
    for k in range(d - 1):
        r0, n, r1 = Y[k].shape
        M = Y[k].reshape(r0 * n, r1, order="F")
        Q, R = np.linalg.qr(M)
        q = Q.shape[1]
        Y[k] = Q.reshape(r0, n, q, order="F")
        Y[k + 1] = np.einsum("cb,bjd->cjd", R, Y[k + 1])
    return Y, float(np.linalg.norm(Y[-1]))


def trunc_rank(s, delta, rmax):
    """Reading Z21: r' = smallest r >= 1 with sum_{i>r} s_i^2 <= delta^2, then min(r', rmax)."""
    s = np.asarray(s)
    p = len(s)
    tail = 0.0
    r = p
    # walk from the end: drop s_i while the accumulated tail stays <= delta^2
    for i in range(p - 1, 0, -1):
        if tail + s[i] ** 2 <= delta ** 2:
            tail += s[i] ** 2
            r = i
        else:
            break
    return max(1, min(r, rmax))


def tt_round(X, eps, rmax=10**9):
    """TT rounding (P:776 'rank reduction step').
    Right-to-left QR orthogonalization, delta = eps ||X|| / sqrt(d-1), then
    left-to-right truncated SVD of the left unfoldings.
    Returns (cores, info) with info = {'sv': [bond singular values],
    'discarded_sq': [tail energies], 'norm': ||X||}."""
    d = len(X)
    Y, nrm = tt_orthogonalize_rl(X)
    info = {"sv": [], "discarded_sq": [], "norm": nrm}
    if d == 1:
        return Y, info
    delta = eps * nrm / math.sqrt(d - 1)
    for k in range(d - 1):
        r0, n, r1 = Y[k].shape
        M = Y[k].reshape(r0 * n, r1, order="F")
        U, s, Vt = np.linalg.svd(M, full_matrices=False)
        rnew = trunc_rank(s, delta, rmax)
        info["sv"].append(s.copy())
        info["discarded_sq"].append(float(np.sum(s[rnew:] ** 2)))
        Y[k] = U[:, :rnew].reshape(r0, n, rnew, order="F")
        SV = s[:rnew, None] * Vt[:rnew, :]
        Y[k + 1] = np.einsum("cb,bjd->cjd", SV, Y[k + 1])
    return Y, info


def tt_svd(T, dims, eps, rmax=10**9):
    """TT-SVD of a full tensor (standard sequential truncated SVDs; used by Alg. 1
    P:1330-1349 line 'Compute G_k's QTT-matrix format').  T is the dense vector
    linearised first-index-fastest over dims."""
    d = len(dims)
    nrm = np.linalg.norm(T)
    delta = eps * nrm / math.sqrt(max(d - 1, 1))
    cores = []
    C = np.asarray(T, dtype=np.float64).reshape(-1, order="F")
    r0 = 1
    for k in range(d - 1):
        M = C.reshape(r0 * dims[k], -1, order="F")
        U, s, Vt = np.linalg.svd(M, full_matrices=False)
        r = trunc_rank(s, delta, rmax)
        cores.append(U[:, :r].reshape(r0, dims[k], r, order="F"))
        C = (s[:r, None] * Vt[:r, :])
        r0 = r
    cores.append(C.reshape(r0, dims[-1], 1, order="F"))
    return cores


# ------------------------------------------------- interfaces / local op ---
# Orientation: Phi_k[alpha, gamma, beta] with
# alpha = test (Y) rank, gamma = operator rank, beta = trial (X) rank.
# Phi_k is the left interface over cores 1..k (Phi_0 = [[[1]]]); Psi_k the right
# interface over cores k..d (Psi_{d+1} = [[[1]]]).  Local system at core k uses
# Phi_{k-1} and Psi_{k+1} (P:1517-1519 'fix all but one TT core').


def left_update(Phi, Yk, Ak, Xk):
    """Phi_k[a',g',b'] = sum Phi_{k-1}[a,g,b] Y_k[a,i,a'] A_k[g,i,j,g'] X_k[b,j,b'],
    as three pairwise contractions (library tensordot), in this order:
    over a, then over (g, i), then over (b, j)."""
    T1 = np.tensordot(Phi, Yk, axes=([0], [0]))              # [g, b, i, a']
    T2 = np.tensordot(T1, Ak, axes=([0, 2], [0, 1]))         # [b, a', j, g']
    return np.tensordot(T2, Xk, axes=([0, 2], [0, 1]))       # [a', g', b']


def right_update(Psi, Yk, Ak, Xk):
    """Psi_k[a,g,b] = sum Psi_{k+1}[a',g',b'] Y_k[a,i,a'] A_k[g,i,j,g'] X_k[b,j,b'];
    contractions over b', then (j, g'), then (i, a')."""
    T1 = np.tensordot(Xk, Psi, axes=([2], [2]))              # [b, j, a', g']
    T2 = np.tensordot(T1, Ak, axes=([1, 3], [2, 3]))         # [b, a', g, i]
    out = np.tensordot(Yk, T2, axes=([1, 2], [3, 1]))        # [a, b, g]
    return np.transpose(out, (0, 2, 1))


def left_update_vec(phi, Yk, Bk):
    """phi_k[a',b'] = sum phi_{k-1}[a,b] Y_k[a,i,a'] B_k[b,i,b'] (vector interface)."""
    T1 = np.tensordot(phi, Yk, axes=([0], [0]))              # [b, i, a']
    return np.tensordot(T1, Bk, axes=([0, 1], [0, 1]))       # [a', b']


def right_update_vec(psi, Yk, Bk):
    """psi_k[a,b] = sum psi_{k+1}[a',b'] Y_k[a,i,a'] B_k[b,i,b']."""
    T1 = np.tensordot(Bk, psi, axes=([2], [1]))              # [b, i, a']
    return np.tensordot(Yk, T1, axes=([1, 2], [1, 2]))       # [a, b]


def local_apply(Phi, Ak, Psi, x):
    """y[a,i,a'] = sum Phi[a,g,b] A[g,i,j,g'] Psi[a',g',b'] x[b,j,b']:
    (1) x x Psi over b'; (2) x A over (j, g'); (3) x Phi over (b, g)."""
    T1 = np.tensordot(x, Psi, axes=([2], [2]))               # [b, j, a', g']
    T2 = np.tensordot(T1, Ak, axes=([1, 3], [2, 3]))         # [b, a', g, i]
    y = np.tensordot(Phi, T2, axes=([1, 2], [2, 0]))         # [a, a', i]
    return np.transpose(y, (0, 2, 1))


def local_rhs(phi, Bk, psi):
    """rhs[a,i,a'] = sum phi[a,b] B[b,i,b'] psi[a',b']."""
    T1 = np.tensordot(Bk, psi, axes=([2], [1]))              # [b, i, a']
    return np.tensordot(phi, T1, axes=([1], [0]))            # [a, i, a']


def local_matrix(Phi, Ak, Psi):
    """Dense local matrix B[(a,i,a'), (b,j,b')] (column-major row/col linearisation)."""
    ra, R0, rb = Phi.shape
    rap, R1, rbp = Psi.shape
    _, m, n, _ = Ak.shape
    T = np.tensordot(Phi, Ak, axes=([1], [0]))               # [a, b, i, j, g']
    T = np.tensordot(T, Psi, axes=([4], [1]))                # [a, b, i, j, a', b']
    T = np.transpose(T, (0, 2, 4, 1, 3, 5))                  # [a, i, a', b, j, b']
    return T.reshape(ra * m * rap, rb * n * rbp, order="F")


def frames_dense(X, k):
    """Dense frame matrix X_{!=k} of size N x (r_{k-1} n_k r_k) (0-based k), so that
    vec(X) = X_{!=k} vec(X_k).  Used only by pins."""
    d = len(X)
    left = np.ones((1, 1))
    for G in X[:k]:
        r0, n, r1 = G.shape
        new = np.zeros((left.shape[0], n, r1))
        for i in range(n):
            new[:, i, :] = left @ G[:, i, :]
        left = new.reshape(left.shape[0] * n, r1, order="F")       # [lin_left, alpha]
    right = np.ones((1, 1))
    for G in reversed(X[k + 1:]):
        r0, n, r1 = G.shape
        new = np.zeros((r0, n, right.shape[1]))
        for i in range(n):
            new[:, i, :] = G[:, i, :] @ right
        right = new.reshape(r0, n * right.shape[1], order="F")      # [alpha, lin_right]
    r0, n, r1 = X[k].shape
    NL, NR = left.shape[0], right.shape[1]
    F = np.einsum("la,ij,bm->limajb", left, np.eye(n), right)        # [lL, i, lR, a, j, b]
    F = F.reshape(NL * n * NR, r0 * n * r1, order="F")
    return F
