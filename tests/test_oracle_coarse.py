"""Pins of the p = 1 coarse level and the hybrid V(1,1) cycle (oracle/coarse.py).  CPU only."""
import numpy as np
import pytest

import rm_inputs as ri
from oracle.basis1d import fdm_basis
from oracle.coarse import CoarseLevel, embed_1d, prolongation, smoother_colours, vcycle
from oracle.fem import P_FAM, Space, assemble
from oracle.solver import Problem


def make(w, **kw):
    return Problem(w.space, w.p, w.nx, w.ny, w.nz, ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w),
                   w.gamma_d, decomposition=w.decomposition, factorization=w.factorization, **kw)


@pytest.mark.parametrize("p", [1, 2, 3, 7, 15])
def test_embedding_reproduces_the_lowest_order_functions(p):
    """sum_j E[c p + j, c + a] s_j(x) = phi_a(x) on cell c (closed form (1 -+ x)/2), and the DP
    constant maps to the constant."""
    f = fdm_basis(p)
    E = embed_1d(p, P_FAM, 3).toarray()
    x = np.linspace(-1, 1, 11)
    s, _ = f.tab_s(x)
    for c in range(3):
        for a, phi in enumerate(((1 - x) / 2, (1 + x) / 2)):
            coef = E[c * p:c * p + p + 1, c + a]
            np.testing.assert_allclose(s @ coef, phi, atol=1e-13)
    Ed = embed_1d(p, "D", 3).toarray()
    r = f.tab_r(x)
    for c in range(3):
        np.testing.assert_allclose(r @ Ed[c * p:c * p + p, c], np.full_like(x, 2 ** -0.5), atol=1e-13)


@pytest.mark.parametrize("k,p", [(0, 3), (0, 4), (1, 3), (2, 3)])
def test_galerkin_identity_cartesian(k, p):
    """V_{h,1} is a subspace of V_{h,p} and both quadratures are exact on Cartesian cells, so
    R_0 A_p R_0^T equals the p = 1 rediscretisation A_0 (a wrong embedding coefficient fails)."""
    n = 2
    w = ri.CONFIGS[2].with_mesh(n)
    X = ri.vertex_coords(w)
    al = np.exp(np.linspace(-1, 1, n ** 3)).reshape(n, n, n)
    be = np.full((n, n, n), 0.3)
    Ap = assemble(Space(k, p, n, n, n), X, al, be)
    A1 = assemble(Space(k, 1, n, n, n), X, al, be).toarray()
    E = prolongation(k, p, n, n, n)
    G = (E.T @ Ap @ E).toarray()
    assert np.abs(G - A1).max() < 1e-12 * np.abs(A1).max()


def test_smoother_colours_bound_lambda_max():
    """Reading G20: lambda_max(S A) equals the colour count N_c (vertex stars: 8)."""
    w = ri.CONFIGS[1].with_mesh(3)
    pb = make(w)
    x = ri.uniform_vector(1, 9, pb.space.ndof)
    x[pb.constrained] = 0
    for _ in range(100):
        y = pb.precondition(pb.apply(x))
        lam = np.linalg.norm(y) / np.linalg.norm(x)
        x = y / np.linalg.norm(y)
    assert smoother_colours(0, "pafw") == 8 and abs(lam - 8.0) < 1e-3


@pytest.mark.parametrize("cfg,p,n", [(1, 3, 3), (3, 2, 2), (4, 2, 2), (5, 3, 2)])
def test_vcycle_symmetric_positive(cfg, p, n):
    w = ri.CONFIGS[cfg].with_mesh(n).with_p(p)
    pb = make(w, coarse=True)
    a = ri.uniform_vector(cfg, 0, pb.space.ndof); a[pb.constrained] = 0
    b = ri.uniform_vector(cfg, 3, pb.space.ndof); b[pb.constrained] = 0
    Ma, Mb = pb.cycle(a), pb.cycle(b)
    assert abs(b @ Ma - a @ Mb) < 1e-11 * abs(a @ Ma)
    assert a @ Ma > 0 and b @ Mb > 0


def test_p1_converges_in_one_iteration():
    """p = 1: the coarse space is the whole space, so the cycle ends with the exact solve and CG
    stops after one iteration (tab:hgrad-iter row p = 1, l = 0: "1/1")."""
    for cfg in (1, 2):
        w = ri.CONFIGS[cfg].with_mesh(3).with_p(1)
        pb = make(w, coarse=True)
        f = ri.uniform_vector(cfg, 0, pb.space.ndof); f[pb.constrained] = 0
        _, it, rel = pb.pcg(f)
        assert it == 1 and rel <= 1e-8


def test_coarse_pcg_counts_scale_invariant_and_p_robust():
    """With the coarse level: counts depend only on alpha / beta and stay flat in p
    (tab:hgrad-iter Cartesian: 14 / 12 / 10 at p = 3 / 7 / 15)."""
    its = []
    for p in (2, 3, 4, 5):
        w = ri.CONFIGS[1].with_mesh(3).with_p(p)
        pb = make(w, coarse=True)
        f = ri.uniform_vector(1, 0, pb.space.ndof); f[pb.constrained] = 0
        _, it, rel = pb.pcg(f)
        assert rel <= 1e-8
        its.append(it)
    assert max(its) - min(its) <= 3 and max(its) <= 20, its
    w = ri.CONFIGS[2].with_mesh(3).with_p(3)
    counts = []
    for c in (1.0, 1e3):
        pb = Problem(0, 3, 3, 3, 3, ri.vertex_coords(w), c * ri.cell_alpha(w), c * ri.cell_beta(w), w.gamma_d,
                     coarse=True)
        f = ri.uniform_vector(2, 0, pb.space.ndof); f[pb.constrained] = 0
        counts.append(pb.pcg(f)[1])
    assert counts[0] == counts[1]


def test_coarse_level_reduces_iterations():
    """The coarse level removes the one-level method's mesh dependence: fewer iterations."""
    w = ri.CONFIGS[1].with_mesh(4).with_p(3)
    f = None
    its = []
    for coarse in (False, True):
        pb = make(w, coarse=coarse)
        if f is None:
            f = ri.uniform_vector(1, 0, pb.space.ndof); f[pb.constrained] = 0
        its.append(pb.pcg(f)[1])
    assert its[1] < its[0], its
