"""GPU parity of operator assembly (device sum + round), AMEn (a7) and the k-eff
fixed point (a9) against the oracle.  |dk|/k <= 1e-8 on the dense-checkable
configs (BASELINE.json north_star)."""
import copy
import os

import numpy as np
import pytest

import inputs
from oracle import solvers as so
from oracle import transport as T
from oracle import tt as ott

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2309_03347_b200 as tb  # noqa: E402
from paper_2309_03347_b200 import transport as gtr  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def small_c1(nv=4):
    p = copy.deepcopy(inputs.problem_c1())
    p["nv"] = nv
    return p


@pytest.mark.parametrize("prob", [inputs.problem_c1(), inputs.problem_small_hetero(nv=4, G=2, N=4)],
                         ids=["C1", "hetero4"])
def test_operator_assembly_on_device(prob):
    dense = T.dense_operators(prob)
    ops = gtr.operators(prob)
    for k in "HSF":
        got = ott.ttm_full(ops[k].cores())
        assert np.max(np.abs(got - dense[k])) <= 1e-12 * np.abs(dense[k]).max()
    if prob["name"].startswith("C1"):
        assert ops["H"].ranks() == [1, 3, 7, 8, 1, 1]
        assert ops["S"].ranks() == [1, 2, 4, 8, 1, 1]


def test_amen_identity_and_transport():
    g = inputs.rng(60)
    modes = [2, 3, 4, 2]
    b = inputs.random_tt(g, modes, [1, 2, 3, 2, 1])
    I = tb.TTMat.from_cores(ott.rank1_ttm([np.eye(n) for n in modes]))
    x = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=[1, 8, 8, 8, 1])
    z = tb.TTVec.from_cores(inputs.random_tt(g, modes, [1, 2, 2, 2, 1]))
    tb.amen_solve(I, tb.TTVec.from_cores(b), x, z, eps=1e-12)
    assert np.linalg.norm(ott.tt_full(x.cores()) - ott.tt_full(b)) <= 1e-10 * np.linalg.norm(ott.tt_full(b))
    # transport H on a 4^3 S2 cube vs a dense solve
    prob = small_c1(4)
    ops = gtr.operators(prob)
    Hd = T.dense_operators(prob)["H"]
    modes = [4, 4, 4, 8, 1]
    b = inputs.random_tt(g, modes, [1, 2, 3, 2, 1, 1])
    x = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=[1, 20, 20, 20, 20, 1])
    z = tb.TTVec.from_cores(inputs.random_tt(g, modes, [1, 4, 4, 4, 4, 1]))
    _, sweeps, res = tb.amen_solve(ops["H"], tb.TTVec.from_cores(b), x, z, eps=1e-11)
    ref = np.linalg.solve(Hd, ott.tt_full(b))
    err = np.linalg.norm(ott.tt_full(x.cores()) - ref) / np.linalg.norm(ref)
    assert err <= 1e-8, (err, sweeps.item(), res.item())


def test_qtt_alg1_device():
    """Alg. 1 on the device (tt_qtt_matrix_dev: rounding of the exact
    index-forwarding TT = TT-SVD): the displayed factors are reproduced exactly in
    QTT with the oracle's ranks; a generic matrix gets full ranks; the 256 x 256
    C4 factors (D, Ip, Ip_noBC of both signs, a box indicator) reconstruct to
    <= 1e-13 with the ranks of the oracle's TT-SVD (oracle.transport.qtt_matrix)."""
    for M in (T.D_plus(8, 0.25), T.D_minus(64, 0.1), T.Ip_plus_noBC(16), T.Ip_minus(32), np.eye(4), np.eye(2)):
        cores = gtr.qtt_matrix(M)
        assert np.max(np.abs(ott.ttm_full(cores) - M)) <= 1e-13 * np.abs(M).max()
        assert ott.ranks(cores) == ott.ranks(T.qtt_matrix(M))
        assert max(ott.ranks(cores)) <= 3
    R = inputs.rng(71).standard_normal((8, 8))      # generic matrix: full QTT ranks
    cores = gtr.qtt_matrix(R)
    assert np.max(np.abs(ott.ttm_full(cores) - R)) <= 1e-13 * np.abs(R).max()
    assert ott.ranks(cores) == [1, 4, 4, 1]
    h = 10.0 / 255
    box = np.diag(((np.arange(256) >= 64) & (np.arange(256) < 192)).astype(float)) @ T.Ip_plus(256)
    for M in (T.D_plus(256, h), T.D_minus(256, h), T.Ip_plus(256), T.Ip_minus(256), T.Ip_plus_noBC(256),
              T.Ip_minus_noBC(256), box):
        cores = gtr.qtt_matrix(M)
        assert np.max(np.abs(ott.ttm_full(cores) - M)) <= 1e-13 * np.abs(M).max()
        assert ott.ranks(cores) == ott.ranks(T.qtt_matrix(M))


def _keff_gpu(prob, modes, rmax, kick=4, **kw):
    ops = gtr.operators(prob)
    g = inputs.rng(61)
    d = len(modes)
    psi = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=[1] + [rmax + kick] * (d - 1) + [1])
    z = tb.TTVec.from_cores(inputs.random_tt(g, modes, [1] + [kick] * (d - 1) + [1]))
    res = tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], psi, z, rmax=rmax, **kw)
    torch.cuda.synchronize()
    return res, psi


def test_keff_small_vs_dense():
    prob = small_c1(4)
    ops = T.dense_operators(prob)
    kd, psid, _ = so.keff_dense_power(ops["H"], ops["S"], ops["F"], tol=1e-13)
    res, psi = _keff_gpu(prob, [4, 4, 4, 8, 1], rmax=32, tol_k=1e-12, eps_round=1e-13, eps_solve=1e-12)
    assert res.status.item() == 0
    k = res.k.item()
    assert abs(k - kd) / kd <= 1e-8
    v = ott.tt_full(psi.cores())
    v = v * np.sign(v.sum()) / np.linalg.norm(v)
    assert np.linalg.norm(v - psid * np.sign(psid.sum())) <= 1e-6


def test_slab_qtt_operators_on_device():
    """QTT operators of the 1-D slab (host Alg. 1 + device sum/round) vs dense."""
    p = inputs.problem_slab(4)
    dense = T.dense_operators(p)
    ops = gtr.operators(p, eps=1e-12)
    for k in "HSF":
        got = ott.ttm_full(ops[k].cores())
        assert np.max(np.abs(got - dense[k])) <= 1e-11 * np.abs(dense[k]).max()


@pytest.mark.parametrize("L", [4, 32])
def test_keff_slab_qtt(L):
    """NEXT-3: 1-D Pu-239 slab, 1024 points, QTT in x; GPU TT k vs
    the oracle's matrix-free full-grid iteration; k -> 1 (exactly critical)."""
    p = inputs.problem_slab(L)
    ks, _, _ = T.slab_keff_sweep(p, tol=1e-13)
    res, psi = _keff_gpu(p, gtr.modes(p), rmax=40, kick=3, tol_k=1e-11, eps_round=1e-11, eps_solve=1e-11)
    assert res.status.item() == 0
    assert abs(res.k.item() - ks) <= 1e-8
    if L == 32:
        assert 1.0 - res.k.item() < 5e-4


def test_keff_c1_vacuum():
    """BASELINE.json configs[0] (vacuum): |dk|/k <= 1e-8 against the dense oracle value."""
    kd = float(open(os.path.join(GOLD, "c1_keff_vacuum.txt")).read().split()[-1])
    res, psi = _keff_gpu(inputs.problem_c1(), [8, 8, 8, 8, 1], rmax=64, tol_k=1e-12, eps_round=1e-13,
                         eps_solve=1e-12)
    assert res.status.item() == 0
    assert abs(res.k.item() - kd) / kd <= 1e-8
    it = res.iters.item()
    hist = res.k_hist[:it].cpu().numpy()
    assert abs(hist[-1] - res.k.item()) == 0.0


@pytest.mark.parametrize("case", ["c1", "slab"])
def test_keff_amen_mv(case):
    """k-eff with B formed by the fit-based product (keff_opts.matvec = amen_mv,
    P:1501-1506) reaches the same k as the oracle: C1 vacuum (dense golden value,
    |dk|/k <= 1e-8) and the slab L=4 (matrix-free sweep)."""
    if case == "c1":
        kd = float(open(os.path.join(GOLD, "c1_keff_vacuum.txt")).read().split()[-1])
        res, _ = _keff_gpu(inputs.problem_c1(), [8, 8, 8, 8, 1], rmax=64, tol_k=1e-12, eps_round=1e-13,
                           eps_solve=1e-12, matvec="amen_mv")
    else:
        p = inputs.problem_slab(4)
        kd, _, _ = T.slab_keff_sweep(p, tol=1e-13)
        res, _ = _keff_gpu(p, gtr.modes(p), rmax=40, kick=3, tol_k=1e-11, eps_round=1e-11, eps_solve=1e-11,
                           matvec="amen_mv")
    assert res.status.item() == 0
    assert abs(res.k.item() - kd) / kd <= 1e-8


def test_keff_c1_reflective():
    """configs[0] reflective variant (reading Z15): the device-assembled operator
    equals the dense one, k -> k_inf = nuSf / (St - Ss) = 1.2 and, from psi0 = 1,
    k0 = 1, the iterates follow k_tau = 1.2 - 0.2 * 0.5^tau (closed form)."""
    prob = inputs.problem_c1("reflective")
    dense = T.dense_operators(prob)
    ops = gtr.operators(prob)
    for k in "HSF":
        got = ott.ttm_full(ops[k].cores())
        assert np.max(np.abs(got - dense[k])) <= 1e-12 * np.abs(dense[k]).max()
    res, psi = _keff_gpu(prob, [8, 8, 8, 8, 1], rmax=64, tol_k=1e-10, eps_round=1e-13, eps_solve=1e-12,
                         max_outer=60)
    it = res.iters.item()
    hist = res.k_hist[:it].cpu().numpy()
    assert abs(res.k.item() - 1.2) <= 1e-8
    for tau, kt in enumerate(hist[:10], start=1):
        assert abs(kt - (1.2 - 0.2 * 0.5 ** tau)) <= 1e-8


def _mv_gpu(A, b, y0, z0, rcap, eps, max_sweeps=40):
    d = len(b)
    y = tb.TTVec.from_cores(y0, rcap=[1] + [rcap] * (d - 1) + [1])
    z = tb.TTVec.from_cores(z0)
    _, sweeps = tb.amen_mv(tb.TTMat.from_cores(A), tb.TTVec.from_cores(b), y, z, eps=eps, max_sweeps=max_sweeps)
    torch.cuda.synchronize()
    return ott.tt_full(y.cores()), sweeps.item()


def test_amen_mv_gpu():
    """NEXT-1: device amen_mv vs the exact product (oracle exact
    matvec + full contraction) and vs the oracle amen_mv, on the oracle's pins."""
    g = inputs.rng(81)
    modes = [2, 3, 4, 2]
    b = inputs.random_tt(g, modes, [1, 2, 3, 2, 1])
    y0 = inputs.random_tt(g, modes, [1, 1, 1, 1, 1])
    z0 = inputs.random_tt(g, modes, [1, 2, 2, 2, 1])
    I = ott.rank1_ttm([np.eye(n) for n in modes])
    got, _ = _mv_gpu(I, b, y0, z0, 16, 1e-12)
    ref = ott.tt_full(b)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    Fs = [g.standard_normal((n, n)) for n in modes]
    vs = [g.standard_normal(n).reshape(1, n, 1) for n in modes]
    got, _ = _mv_gpu(ott.rank1_ttm(Fs), vs, y0, z0, 16, 1e-12)
    ref = ott.tt_full(ott.tt_matvec(ott.rank1_ttm(Fs), vs))
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    # rectangular operator: modes (3, 2, 4) <- (2, 5, 3)
    Ar = inputs.random_ttm(g, [3, 2, 4], [2, 5, 3], [1, 2, 3, 1])
    br = inputs.random_tt(g, [2, 5, 3], [1, 2, 2, 1])
    got, _ = _mv_gpu(Ar, br, inputs.random_tt(g, [3, 2, 4], [1, 1, 1, 1]),
                     inputs.random_tt(g, [3, 2, 4], [1, 2, 2, 1]), 12, 1e-12)
    ref = ott.tt_full(ott.tt_matvec(Ar, br))
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    # C2 slice d = 10 vs the dense product
    inst = inputs.c2_slice(110)
    d = 10
    y0 = inputs.random_tt(g, [2] * d, [1] + [2] * (d - 1) + [1])
    z0 = inputs.random_tt(g, [2] * d, [1] + [4] * (d - 1) + [1])
    got, sw = _mv_gpu(inst["A"], inst["X"], y0, z0, 40, 1e-10)
    ref = ott.ttm_full(inst["A"]) @ ott.tt_full(inst["X"])
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref), sw
    # truncated QTT slab transport apply vs exact (and vs the oracle amen_mv)
    p = inputs.problem_slab(4, nv=256)
    H = T.tt_operators(p, eps=1e-12)["H"]
    modes = T.qtt_modes(p)
    d = len(modes)
    x = inputs.random_tt(g, modes, [1] + [2] * (d - 1) + [1])
    y0 = inputs.random_tt(g, modes, [1] + [2] * (d - 1) + [1])
    z0 = inputs.random_tt(g, modes, [1] + [3] * (d - 1) + [1])
    got, sw = _mv_gpu(H, x, y0, z0, 40, 1e-8)
    ref = ott.tt_full(ott.tt_matvec_fast(H, x))
    assert np.linalg.norm(got - ref) <= 1e-7 * np.linalg.norm(ref), sw
    yo, _ = so.amen_mv(H, x, y0, z0, eps=1e-8, max_sweeps=40)
    assert np.linalg.norm(got - ott.tt_full(yo)) <= 2e-7 * np.linalg.norm(ref)


def _alpha_gpu(prob, modes, rmax, kick=4, **kw):
    ops = gtr.operators(prob, velocity=True)
    g = inputs.rng(62)
    d = len(modes)
    psi = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=[1] + [rmax + kick] * (d - 1) + [1])
    z = tb.TTVec.from_cores(inputs.random_tt(g, modes, [1] + [kick] * (d - 1) + [1]))
    res = tb.alpha_secant(ops["H"], ops["V"], ops["S"], ops["F"], psi, z, rmax=rmax, **kw)
    torch.cuda.synchronize()
    return res


def test_alpha_c1_reflective_closed_form():
    """NEXT-2 (Z32) on configs[0]'s reflective variant: the infinite-
    medium closed form alpha* = v (nuSf + Ss - St) = 0.1; the first two k-eff
    solves give k(0) = 1.2 and k(0.01) = 0.6/0.51."""
    res = _alpha_gpu(inputs.problem_c1("reflective"), [8, 8, 8, 8, 1], rmax=64, tol=1e-10, tol_k=1e-12,
                     eps_round=1e-13, eps_solve=1e-12, max_outer=80)
    assert res.status.item() == 0
    assert abs(res.alpha.item() - 0.1) <= 1e-8
    kh = res.k_hist.cpu().numpy()
    assert abs(kh[0] - 1.2) <= 1e-9 and abs(kh[1] - 0.6 / 0.51) <= 1e-9
    assert res.iters.item() <= 10


@pytest.mark.parametrize("nsf", [2.8, 2.0], ids=["super", "sub"])
def test_alpha_cube_vs_dense(nsf):
    """4^3 S2 cube: device alpha vs the oracle's dense secant (LU k-eff solves)."""
    prob = small_c1(4)
    prob["materials"][0]["nu_sigma_f"] = np.array([nsf])
    ops = T.dense_operators(prob)
    ad, _, _ = so.alpha_dense(ops["H"], ops["V"], ops["S"], ops["F"], tol=1e-11)
    res = _alpha_gpu(prob, [4, 4, 4, 8, 1], rmax=32, tol=1e-11, tol_k=1e-12, eps_round=1e-13, eps_solve=1e-12)
    assert res.status.item() == 0
    assert abs(res.alpha.item() - ad) <= 1e-8 * abs(ad)


def test_alpha_slab():
    """1-D Pu-239 slab L=4, 1024 points: device alpha vs the oracle's
    matrix-free secant (sigma_t shift, Z39); the slab is critical so |alpha| is small."""
    p = inputs.problem_slab(4)
    ao, _, _ = so.alpha_secant(lambda a: T.slab_keff_sweep(p, tol=1e-13, alpha=a)[0], tol=1e-11)
    res = _alpha_gpu(p, gtr.modes(p), rmax=40, kick=3, tol=1e-10, tol_k=1e-12, eps_round=1e-12,
                     eps_solve=1e-12, eps_op=1e-12)
    assert res.status.item() == 0
    assert abs(res.alpha.item() - ao) <= 1e-8


def test_keff_c3_small_grid():
    """configs[2]'s problem (two regions, G=7 downscatter, 80 S8 ordinates, QTT
    space) on a 4^3 grid, where rmax does not bind: the device TT k-eff (B by
    amen_mv; exact products of rank R_S r = 4800 would not fit) equals the
    oracle's matrix-free full-grid sweep iteration (discretisation truth) to 1e-8."""
    matvec = "amen_mv"
    p = inputs.problem_c3(nv=4)
    kt, _, _ = T.keff_sweep_3d(p, tol=1e-13)
    res, psi = _keff_gpu(p, gtr.modes(p), rmax=96, kick=4, tol_k=1e-11, eps_round=1e-12, eps_solve=1e-12,
                         matvec=matvec, max_sweeps=20)
    assert res.status.item() == 0
    assert abs(res.k.item() - kt) / kt <= 1e-8


def test_keff_c3_truncated():
    """configs[2]'s problem on an 8^3 grid with rmax = 64 (binding: the full-grid
    solution's QTT ranks reach 391 at eps 1e-4): the TT k-eff stays within the
    truncation level of the matrix-free truth (C3 partially
    pinned; P:1654 reports ~1e-5 discrepancies at tolerance 1e-6)."""
    p = inputs.problem_c3(nv=8)
    kt = [float(l.split()[1]) for l in open(os.path.join(GOLD, "c3_keff.txt"))
          if l.strip() and not l.startswith("#") and l.split()[0] == "8"][0]
    res, _ = _keff_gpu(p, gtr.modes(p), rmax=64, kick=4, tol_k=1e-7, eps_round=1e-7, eps_solve=1e-7,
                       matvec="amen_mv", max_sweeps=4, mv_max_sweeps=4, max_outer=40)
    assert abs(res.k.item() - kt) / kt <= 2e-4


def _golden(name, nv):
    return [float(l.split()[1]) for l in open(os.path.join(GOLD, name))
            if l.strip() and not l.startswith("#") and l.split()[0] == str(nv)][0]


def test_keff_c4_small_grid():
    """configs[3]'s physics (G=30 with upscatter into groups 26-30, S16 LS-style 288
    ordinates, core/blanket/reflector) on a 4^3 grid, where rmax does not bind
    (the QTT bonds are <= 64, the angle|group bond <= 30): the device TT k-eff
    (B by amen_mv) equals the oracle's matrix-free full-grid sweep iteration
    (tests/golden/c4_keff.txt, make_c4_keff.py) to 1e-8, with the fixed-point
    residual ||H Psi - (S + F/k) Psi|| / ||H Psi|| (Z19) required <= 1e-9."""
    p = inputs.problem_c4(nv=4)
    kt = _golden("c4_keff.txt", 4)
    res, _ = _keff_gpu(p, gtr.modes(p), rmax=96, kick=4, tol_k=1e-11, tol_res=1e-9, eps_round=1e-12,
                       eps_solve=1e-12, matvec="amen_mv", max_sweeps=20)
    assert res.status.item() == 0
    assert 0.0 <= res.res.item() <= 1e-9
    assert abs(res.k.item() - kt) / kt <= 1e-8


def test_keff_c3_full_gpu_tt_vs_cpu_tt():
    """configs[2] at full size (64^3 QTT, G=7, 80 ordinates, rmax 64, eps 1e-6):
    the GPU-TT fixed-point iterates against the CPU-TT oracle's
    (oracle.solvers.keff_tt with the same eps, rmax, sweep limits, amen_mv B,
    GMRES local solves and z0; tests/golden/c3_tt_keff.txt,
    make_c3_tt_keff.py).  Iteration 1 (ranks set by eps): |dk|/k <= 10
    eps_solve (measured 1.2e-11).  Later iterations: the
    ranks are capped by the 4-sweep rank growth (kickrank 4 per sweep) and then
    by rmax, so the kept subspace at each cut is only determined to (local
    solve tolerance) / (spectral gap at the cut) and the two implementations'
    GMRES roundoff (DGKS vs MGS) moves k by O(1e-4) (reading Z22's near-tie
    caveat; measured 3.6e-4): |dk|/k <= 1e-3 and the same final ranks are
    required there."""
    rows = [l.split() for l in open(os.path.join(GOLD, "c3_tt_keff.txt")) if l.strip() and not l.startswith("#")]
    kref = np.array([float(r[1]) for r in rows])
    rref = [int(r[2]) for r in rows]
    n = len(kref)
    p = inputs.problem_c3()
    res, psi = _keff_gpu(p, gtr.modes(p), rmax=64, kick=4, tol_k=0.0, eps_round=1e-6, eps_solve=1e-6,
                         matvec="amen_mv", max_sweeps=4, mv_max_sweeps=4, restart=60, max_restarts=200,
                         max_outer=n)
    kg = res.k_hist[:n].cpu().numpy()
    rel = np.abs(kg - kref) / kref
    assert rel[0] <= 1e-5, rel
    assert np.all(rel <= 1e-3), (kg, kref, rel)
    assert max(psi.ranks()) == rref[-1]


def test_keff_c4_full_residual_and_rmax_refinement():
    """configs[3] at full size (256^3 QTT, G=30 with upscatter, S16 288
    ordinates, three regions; eps 1e-6), SURVEY.md §8(c).4 "parity unpinned
    beyond self-consistency" — so the pins are self-consistency ones: the
    fixed point converges (|dk| <= 1e-6) at rmax 128 and at rmax 160; the
    fixed-point residual ||H Psi - (S + F/k) Psi|| / ||H Psi|| (Z19) of
    the final iterate is evaluated and bounded (truncation-limited: the
    full-grid flux is not low rank, measured 1.7e-2 / 1.3e-2) and does not grow
    under refinement; the eigenvalue moves by <= 1e-4 relative between the two
    rank caps (measured 1.4e-5, the paper's TT-vs-PARTISN level ~1e-5 at
    tolerance 1e-6); and k lies below the coarse-grid matrix-free
    values (tests/golden/c4_keff.txt: 0.6641 / 0.6569 at 8^3 / 16^3, k falling
    under refinement as for C3)."""
    p = inputs.problem_c4()
    ks, rs = {}, {}
    for rmax in (128, 160):
        res, psi = _keff_gpu(p, gtr.modes(p), rmax=rmax, kick=4, tol_k=1e-6, tol_res=0.0, eps_round=1e-6,
                             eps_solve=1e-6, matvec="amen_mv", max_sweeps=4, mv_max_sweeps=4, restart=40,
                             max_restarts=20, max_outer=120)
        assert res.status.item() == 0, (rmax, res.iters.item())
        ks[rmax], rs[rmax] = res.k.item(), res.res.item()
        assert 0.0 < rs[rmax] <= 5e-2, (rmax, rs[rmax])
        assert max(psi.ranks()) <= rmax + 4
    assert abs(ks[128] - ks[160]) / ks[160] <= 1e-4, ks
    assert rs[160] <= 1.1 * rs[128], rs
    assert ks[160] < _golden("c4_keff.txt", 16) < _golden("c4_keff.txt", 8)


def _qtt_vec(v, eps=1e-14):
    """QTT cores (bits LSB first, Z28) of a 2^l vector, by the oracle's TT-SVD."""
    l = int(round(np.log2(v.size)))
    return ott.tt_svd(v, [2] * l, eps)


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_transport_operator_sampled_full_size(cfg):
    """configs[2] / configs[3] at full size (64^3 G=7 80 ordinates; 256^3 G=30
    288 ordinates): the device-assembled QTT operators H, S, F applied (exact
    device matvec) to a separable Psi equal the oracle's per-term Kronecker
    factors (Z3-Z7, Z34) on 64 sampled entries, evaluated one by one."""
    p = inputs.problem_c3() if cfg == "c3" else inputs.problem_c4()
    nv, L, G = p["nv"], len(p["quad"]["w"]), p["G"]
    g = inputs.rng(95)
    vx, vy, vz = (np.exp(-((np.arange(nv) - c) / (0.3 * nv)) ** 2) + 0.1 * g.random(nv) for c in (0.3 * nv, 0.5 * nv,
                                                                                                0.6 * nv))
    va, vg = 1.0 + g.random(L), 1.0 + g.random(G)
    cores = _qtt_vec(vx) + _qtt_vec(vy) + _qtt_vec(vz) + [va.reshape(1, L, 1), vg.reshape(1, G, 1)]
    psi = tb.TTVec.from_cores(cores)
    terms = T.operator_terms(p)
    ops = gtr.operators(p, eps=1e-13)
    idx = [g.integers(0, n, size=64) for n in (nv, nv, nv, L, G)]
    l = int(round(np.log2(nv)))
    for key in "HSF":
        y = tb.matvec_out(ops[key], psi)
        torch.cuda.synchronize()
        r = y.ranks()
        # device evaluation of the sampled entries: chain of core slices per sample
        digits = []
        for a in range(3):
            digits += [(idx[a] >> b) & 1 for b in range(l)]
        digits += [idx[3], idx[4]]
        vec = torch.ones(64, 1, dtype=torch.float64, device="cuda")
        for k in range(y.d):
            core = y.data[y.off[k]:y.off[k] + r[k] * y.n[k] * r[k + 1]].reshape(r[k + 1], y.n[k], r[k])
            sel = core[:, torch.as_tensor(digits[k], device="cuda"), :].permute(1, 2, 0)   # [S, r0, r1]
            vec = torch.bmm(vec.unsqueeze(1), sel).squeeze(1)
        got = vec[:, 0].cpu().numpy()
        ref = np.zeros(64)
        for t in terms[key]:
            fx, fy, fz, fa, fg = t
            ref += (fx @ vx)[idx[0]] * (fy @ vy)[idx[1]] * (fz @ vz)[idx[2]] * (fa @ va)[idx[3]] * (fg @ vg)[idx[4]]
        scale = max(np.abs(ref).max(), 1e-300)
        assert np.max(np.abs(got - ref)) <= 1e-10 * scale, (key, np.max(np.abs(got - ref)) / scale)
        del y


_DET_SCRIPT = r"""
import numpy as np, torch, inputs
import paper_2309_03347_b200 as tb
from paper_2309_03347_b200 import transport as gtr
p = inputs.problem_c1(); ops = gtr.operators(p); modes = [8, 8, 8, 8, 1]
g = inputs.rng(61)
psi = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=[1, 68, 68, 68, 68, 1])
z = tb.TTVec.from_cores(inputs.random_tt(g, modes, [1, 4, 4, 4, 4, 1]))
r = tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], psi, z, tol_k=1e-12, eps_round=1e-13, eps_solve=1e-12,
                        rmax=64, matvec="amen_mv")
torch.cuda.synchronize()
print(repr(r.k.item()), r.iters.item())
"""


def test_keff_deterministic_graphs_on_off():
    """The device path is deterministic (fixed reduction orders, no atomics in the
    arithmetic): two C1 solves give bitwise-identical k, and the device-resident
    graph (default), the host-polled loops of replayed sequences (TT_NO_DEVLOOP=1)
    and direct launches (TT_NO_GRAPHS=1) give the same bits."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env_extra in ({}, {}, {"TT_NO_GRAPHS": "1"}, {"TT_NO_DEVLOOP": "1"}):
        env = dict(os.environ, PYTHONPATH=root, **env_extra)
        r = subprocess.run([sys.executable, "-c", _DET_SCRIPT], capture_output=True, text=True, env=env, cwd=root,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1] == outs[2] == outs[3], outs


def test_keff_warm_continuation():
    """keff_opts.warm (the bench's one-iteration step): 1 cold + 5 warm calls of one
    outer iteration follow the single 6-iteration call's k history (the warm call
    only re-orthogonalises the already normalised Psi)."""
    p = small_c1(4)
    modes = [4, 4, 4, 8, 1]
    kw = dict(tol_k=0.0, eps_round=1e-10, eps_solve=1e-10, matvec="amen_mv", max_sweeps=6, mv_max_sweeps=6)
    ref, _ = _keff_gpu(p, modes, rmax=32, max_outer=6, **kw)
    kref = ref.k_hist[:6].cpu().numpy()
    ops = gtr.operators(p)
    g = inputs.rng(61)
    d = len(modes)
    psi = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=[1] + [36] * (d - 1) + [1])
    z = tb.TTVec.from_cores(inputs.random_tt(g, modes, [1] + [4] * (d - 1) + [1]))
    nb = tb.keff_workspace_bytes(ops["H"], ops["S"], ops["F"], psi, z, rmax=32, matvec="amen_mv")
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    k, ks = 1.0, []
    for it in range(6):
        r = tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], psi, z, k0=k, max_outer=1, rmax=32, warm=it > 0,
                                ws=ws, **kw)
        k = r.k.item()
        ks.append(k)
    assert np.max(np.abs(np.array(ks) - kref) / kref) <= 1e-9, (ks, kref)


def test_amen_dense_local_solver():
    """a7's dense branch (Z20): local systems of size <= local_dense_max are
    solved by Gauss-Jordan with partial pivoting on the device.  (1) transport H
    on a 4^3 S2 cube vs a dense LU solve (<= 1e-8, as the GMRES branch);
    (2) a singular operator (zero diagonal entries; the rhs vanishes on them):
    the exactly singular local systems are regularised with mu = 1e-12 ||B||_F
    (Z35) and the result equals the oracle's amen_solve with its dense branch
    (np.linalg.solve -> LinAlgError -> B + mu I)."""
    g = inputs.rng(64)
    prob = small_c1(4)
    ops = gtr.operators(prob)
    Hd = T.dense_operators(prob)["H"]
    modes = [4, 4, 4, 8, 1]
    b = inputs.random_tt(g, modes, [1, 2, 3, 2, 1, 1])
    x = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=[1, 20, 20, 20, 20, 1])
    z = tb.TTVec.from_cores(inputs.random_tt(g, modes, [1, 4, 4, 4, 4, 1]))
    tb.amen_solve(ops["H"], tb.TTVec.from_cores(b), x, z, eps=1e-11, local_dense_max=2000)
    torch.cuda.synchronize()
    ref = np.linalg.solve(Hd, ott.tt_full(b))
    assert np.linalg.norm(ott.tt_full(x.cores()) - ref) <= 1e-8 * np.linalg.norm(ref)
    # singular: A = diag(d1) (x) diag(d2) (x) diag(d3) with zeros, b zero on the null rows
    dims = [3, 4, 2]
    ds = [np.array([1.0, 2.0, 0.0]), np.array([1.5, 0.0, 3.0, 0.5]), np.array([2.0, 1.0])]
    A = ott.rank1_ttm([np.diag(v) for v in ds])
    bv = [np.where(v != 0.0, 1.0 + g.random(v.size), 0.0).reshape(1, -1, 1) for v in ds]
    x0 = [np.ones((1, n, 1)) for n in dims]
    z0 = inputs.random_tt(g, dims, [1, 2, 2, 1])
    xo, _ = so.amen_solve(A, bv, x0, z0, eps=1e-12, max_sweeps=4, dense_max=2000)
    xg = tb.TTVec.from_cores(x0, rcap=[1, 6, 6, 1])
    tb.amen_solve(tb.TTMat.from_cores(A), tb.TTVec.from_cores(bv), xg, tb.TTVec.from_cores(z0), eps=1e-12,
                  max_sweeps=4, local_dense_max=2000)
    torch.cuda.synchronize()
    fo, fg = ott.tt_full(xo), ott.tt_full(xg.cores())
    assert np.linalg.norm(fg - fo) <= 1e-9 * np.linalg.norm(fo), (np.linalg.norm(fg - fo), np.linalg.norm(fo))


def test_keff_dense_local_solver_c1():
    """k-eff (C1 4^3 cube) with the dense local solver (local_dense_max = 2000, the
    SPEC's threshold; the oracle's keff_tt default) reaches the dense power
    iteration's k to 1e-8."""
    prob = small_c1(4)
    ops = T.dense_operators(prob)
    kd, _, _ = so.keff_dense_power(ops["H"], ops["S"], ops["F"], tol=1e-13)
    res, _ = _keff_gpu(prob, [4, 4, 4, 8, 1], rmax=32, tol_k=1e-12, eps_round=1e-13, eps_solve=1e-12,
                       local_dense_max=2000)
    assert res.status.item() == 0
    assert abs(res.k.item() - kd) / kd <= 1e-8


# ------------------------------------------------------------------ K11 ---

def _in_modes(fn):
    out = {}
    try:
        for mode in (2, 1, 0):
            tb.set_graph_mode(mode)
            out[mode] = fn()
            torch.cuda.synchronize()
    finally:
        tb.set_graph_mode(-1)
    return out


def test_device_loops_keff_bitwise():
    """keff_fixed_point as ONE graph launch (outer WHILE node, nested
    amen_mv / AMEn sweep WHILE + IF nodes, residual every iteration) gives the
    same k, histories, status and Psi bits as the host-polled loops (mode 1) and
    direct launches (mode 0); a repeated call replays the cached graph."""
    p = small_c1(4)
    modes = [4, 4, 4, 8, 1]

    def run():
        r, psi = _keff_gpu(p, modes, rmax=32, max_outer=12, tol_k=1e-12, tol_res=1e-6, eps_round=1e-10,
                           eps_solve=1e-10, matvec="amen_mv", max_sweeps=6, mv_max_sweeps=6)
        return (r.k.item(), r.iters.item(), r.status.item(), r.k_hist[:12].cpu().numpy().tolist(),
                r.sweeps_hist[:12].cpu().numpy().tolist(), r.res_hist[:12].cpu().numpy().tolist(),
                [c.tobytes() for c in psi.cores()])
    out = _in_modes(run)
    assert out[2][:6] == out[1][:6] == out[0][:6], (out[2][:6], out[1][:6])
    assert out[2][6] == out[1][6] == out[0][6]
    assert out[2][1] >= 3
    # exact-product B variant, one more time in mode 2: the second identical call replays
    ops = gtr.operators(p)
    g = inputs.rng(61)
    psi = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=[1, 36, 36, 36, 36, 1])
    z = tb.TTVec.from_cores(inputs.random_tt(g, modes, [1, 4, 4, 4, 4, 1]))
    nb = tb.keff_workspace_bytes(ops["H"], ops["S"], ops["F"], psi, z, rmax=32)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    psi0, zc0 = [c.copy() for c in psi.cores()], [c.copy() for c in z.cores()]
    ks = []
    for rep in range(2):
        psi.set_cores(psi0)
        z.set_cores(zc0)
        if rep == 1:
            c0, r0, _ = tb.graph_stats()
        r = tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], psi, z, rmax=32, max_outer=3, tol_k=0.0,
                                eps_round=1e-10, eps_solve=1e-10, ws=ws)
        ks.append(r.k.item())
    c1, r1, _ = tb.graph_stats()
    assert c1 == c0 and r1 == r0 + 1, (c0, c1, r0, r1)
    assert ks[0] == ks[1], ks


def test_device_loops_amen_and_alpha_bitwise():
    """amen_solve (sweep WHILE + IF) and alpha_secant (secant WHILE around the
    k-eff WHILE) in one graph each: the same bits as modes 1 and 0."""
    g = inputs.rng(60)
    prob = small_c1(4)
    ops = gtr.operators(prob)
    modes = [4, 4, 4, 8, 1]
    b = inputs.random_tt(g, modes, [1, 2, 3, 2, 1, 1])
    zc = inputs.random_tt(g, modes, [1, 4, 4, 4, 4, 1])

    def run_amen():
        x = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=[1, 20, 20, 20, 20, 1])
        z = tb.TTVec.from_cores(zc)
        _, sweeps, res = tb.amen_solve(ops["H"], tb.TTVec.from_cores(b), x, z, eps=1e-11)
        return sweeps.item(), res.item(), [c.tobytes() for c in x.cores()]
    out = _in_modes(run_amen)
    assert out[2] == out[1] == out[0], (out[2][:2], out[1][:2], out[0][:2])

    sup = small_c1(4)
    sup["materials"][0]["nu_sigma_f"] = np.array([2.8])   # supercritical cube (test_alpha_cube_vs_dense)

    def run_alpha():
        r = _alpha_gpu(sup, modes, rmax=32, tol=1e-11, tol_k=1e-12, eps_round=1e-13, eps_solve=1e-12)
        return (r.alpha.item(), r.k.item(), r.iters.item(), r.status.item(),
                r.alpha_hist[:r.iters.item()].cpu().numpy().tolist())
    out = _in_modes(run_alpha)
    assert out[2] == out[1] == out[0], (out[2], out[1], out[0])
    assert out[2][3] == 0
