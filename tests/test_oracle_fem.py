"""Pins of the oracle's spaces and operators (oracle/fem.py) to closed forms, special cases and
the de Rham structure fixed by PAPER.md.  CPU only."""
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp

import rm_inputs as ri
from oracle.basis1d import fdm_basis, gauss_rule
from oracle.fem import (FAMILIES, Space, assemble, assemble_aux, aux_element_matrix, element_matrix,
                        global_derivative, ref_derivative_pattern_or_values)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def unit_cell(h=(1.0, 1.0, 1.0)):
    X = np.zeros((2, 2, 2, 3))
    for az in range(2):
        for ay in range(2):
            for ax in range(2):
                X[az, ay, ax] = (ax * h[0], ay * h[1], az * h[2])
    return X


def grid(n, perturb=0.0, cfg=9):
    w = ri.Workload(cfg, 0, 1, n, n, n, "one", 1.0, 0, perturb, "pafw", "chol")
    return ri.vertex_coords(w)


def test_single_cell_p2():
    g = json.load(open(os.path.join(GOLD, "cell_values.json")))
    for key in ("single_cell_p2", "single_cell_p2_b"):
        c = g[key]
        A = element_matrix(0, 2, unit_cell(), c["alpha"], c["beta"])
        assert abs(A[13, 13] - eval(c["value"])) < 1e-13


def test_q1_2x2x2_center():
    c = json.load(open(os.path.join(GOLD, "cell_values.json")))["q1_2x2x2_center"]
    s = Space(0, 1, 2, 2, 2)
    X = grid(2)
    A = assemble(s, X, np.full((2, 2, 2), c["alpha"]), np.full((2, 2, 2), c["beta"])).toarray()
    free = ~s.constrained_mask(ri.GAMMA_ALL)
    assert free.sum() == 1
    i = np.flatnonzero(free)[0]
    assert abs(A[i, i] - eval(c["value"])) < 1e-14


@pytest.mark.parametrize("k,p,n", [(0, 2, 2), (1, 2, 2), (2, 2, 2), (0, 3, 3)])
def test_dof_counts(k, p, n):
    s = Space(k, p, n, n, n)
    nloc = {0: (p + 1) ** 3, 1: 3 * p * (p + 1) ** 2, 2: 3 * (p + 1) * p ** 2}[k]
    assert s.nloc == nloc
    # global: every cell DoF appears, shared ones once
    seen = np.zeros(s.ndof, dtype=int)
    for cz in range(n):
        for cy in range(n):
            for cx in range(n):
                seen[s.cell_dofs(cx, cy, cz)] += 1
    assert seen.min() >= 1


def test_constant_function_hgrad():
    # K c = 0 and c^T M c = |Omega| for the constant function (any mesh, no Dirichlet)
    p = 3
    s = Space(0, p, 2, 2, 2)
    X = grid(2, perturb=0.1)
    K = assemble(s, X, np.ones((2, 2, 2)), np.zeros((2, 2, 2)))
    M = assemble(s, X, np.zeros((2, 2, 2)), np.ones((2, 2, 2)))
    f = fdm_basis(p)
    xq, wq = gauss_rule(p + 2)
    sq, _ = f.tab_s(xq)
    c1 = np.ones(p + 1); c1[1:p] = wq @ sq[:, 1:p]
    # global coefficients of 1: per direction the 1D coefficient pattern, periodic in cells
    L = 2 * p + 1
    c1d = np.array([c1[i % p] if i % p else 1.0 for i in range(L)])
    c = np.einsum("z,y,x->zyx", c1d, c1d, c1d).ravel()
    assert np.abs(K @ c).max() < 1e-12
    assert abs(c @ M @ c - 1.0) < 1e-12


@pytest.mark.parametrize("p", [2, 3])
def test_patch_test_x1_perturbed(p):
    """u = x_1 is in Q_p on trilinear cells: u^T K u = alpha |Omega|, u^T M u = beta/3,
    exact because the integrands are polynomials GLL integrates exactly."""
    n = 2
    s = Space(0, p, n, n, n)
    X = grid(n, perturb=0.1, cfg=7)
    alpha, beta = 2.0, 3.0
    K = assemble(s, X, np.full((n,) * 3, alpha), np.zeros((n,) * 3))
    M = assemble(s, X, np.zeros((n,) * 3), np.full((n,) * 3, beta))
    f = fdm_basis(p)
    xq, wq = gauss_rule(p + 2)
    sq, _ = f.tab_s(xq)
    phi0, phi1 = (1 - xq) / 2, (1 + xq) / 2
    m0, m1 = np.ones(p + 1), np.ones(p + 1)
    m0[1:p] = (wq * phi0) @ sq[:, 1:p]; m0[p] = 0.0
    m1[1:p] = (wq * phi1) @ sq[:, 1:p]; m1[0] = 0.0
    u = np.zeros(s.ndof)
    for cz in range(n):
        for cy in range(n):
            for cx in range(n):
                coef = np.zeros((p + 1,) * 3)
                for az in range(2):
                    for ay in range(2):
                        for ax in range(2):
                            v = X[cz + az, cy + ay, cx + ax, 0]
                            coef += v * np.einsum("z,y,x->zyx", (m0, m1)[az], (m0, m1)[ay], (m0, m1)[ax])
                u[s.cell_dofs(cx, cy, cz)] = coef.ravel()
    assert abs(u @ K @ u - alpha * 1.0) < 1e-11
    assert abs(u @ M @ u - beta / 3.0) < 1e-11


@pytest.mark.parametrize("p", [2, 3])
def test_discrete_complex_exact(p):
    D0 = global_derivative(0, p, 2, 3, 2)
    D1 = global_derivative(1, p, 2, 3, 2)
    D2 = global_derivative(2, p, 2, 3, 2)
    assert abs(D1 @ D0).max() == 0.0
    assert abs(D2 @ D1).max() == 0.0
    # and the element-level reference derivative agrees with the quadrature curl of a gradient
    d0 = ref_derivative_pattern_or_values(0, p, True)
    d1 = ref_derivative_pattern_or_values(1, p, True)
    assert np.abs(d1 @ d0).max() < 1e-12


def test_interior_relations_eq_gradbasis():
    p = 2
    f = fdm_basis(p)
    D0 = global_derivative(0, p, 1, 1, 1).toarray()
    s0, s1 = Space(0, p, 1, 1, 1), Space(1, p, 1, 1, 1)
    col = 13  # psi_111
    nz = np.flatnonzero(np.abs(D0[:, col]) > 1e-14)
    assert len(nz) == 3
    np.testing.assert_allclose(D0[nz, col], math.sqrt(2.5), rtol=1e-13)
    # one nonzero in each component block
    off = s1.offsets()
    assert [int(np.searchsorted(off, i, side="right") - 1) for i in nz] == [0, 1, 2]


@pytest.mark.parametrize("k,p", [(0, 3), (1, 2), (1, 3), (2, 2), (2, 3)])
def test_interior_block_nnz(k, p):
    """On a Cartesian cell the interior block couples each interior DoF to at most d (k=1,2) or
    one (k=0) interior DoF; computed by quadrature, unmasked."""
    A = element_matrix(k, p, unit_cell((0.5, 0.7, 1.1)), 1.3, 0.4)
    s = Space(k, p, 1, 1, 1)
    interior = np.zeros(s.nloc, dtype=bool)
    o = 0
    for fam in FAMILIES[k]:
        sz = [p + 1 if f_ == "P" else p for f_ in fam]
        Z, Y, X = np.meshgrid(range(sz[2]), range(sz[1]), range(sz[0]), indexing="ij")
        inn = np.ones(Z.shape, dtype=bool)
        for d, Aa in enumerate((X, Y, Z)):
            if fam[d] == "P":
                inn &= (Aa > 0) & (Aa < p)
        interior[o:o + inn.size] = inn.ravel()
        o += inn.size
    Aii = A[np.ix_(interior, interior)]
    nnz = (np.abs(Aii) > 1e-12 * np.abs(A).max()).sum(axis=1)
    assert nnz.max() <= (1 if k == 0 else 3)


def test_symmetry_and_aux_equals_A_cartesian():
    w = ri.Workload(5, 0, 3, 2, 2, 2, "logu22", 1.0, 63, 0.0, "pafw", "icc_sc")
    X, al, be = ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w)
    s = Space(0, 3, 2, 2, 2)
    A = assemble(s, X, al, be)
    P, _ = assemble_aux(s, X, al, be)
    assert abs(A - A.T).max() < 1e-13 * abs(A).max()
    assert abs(P - A).max() < 1e-13 * abs(A).max()    # exact in the separable case


def test_aux_perturbed_spd_and_limit():
    p = 3
    Xc = unit_cell((0.5, 0.5, 0.5))
    rng = np.random.default_rng(0)
    d = rng.uniform(-1, 1, Xc.shape)
    PK0 = aux_element_matrix(p, Xc, 1.0, 1.0)
    AK0 = element_matrix(0, p, Xc, 1.0, 1.0)
    assert np.abs(PK0 - AK0).max() < 1e-12 * np.abs(AK0).max()
    prev = None
    for eps in (1e-2, 1e-3, 1e-4):
        PK = aux_element_matrix(p, Xc + eps * 0.5 * d, 1.0, 1.0)
        assert np.abs(PK - PK.T).max() < 1e-13 * np.abs(PK).max()
        err = np.abs(PK - PK0).max()
        if prev is not None:
            assert err < 0.2 * prev          # P -> A continuously as the perturbation -> 0
        prev = err
    # positive semidefinite cell matrix; SPD once Dirichlet/mass present (beta > 0)
    assert np.linalg.eigvalsh(PK).min() > 0


def test_hcurl_hdiv_mass_stiffness_scaling():
    """Cartesian scalings of SURVEY §8(a) row a2: k=1 mass ~ beta h/2, curl-curl ~ alpha 2/h;
    k=2 mass ~ beta 2/h, div-div ~ alpha (2/h)^3 -- checked as ratios between two cell sizes."""
    for k, (mexp, kexp) in {0: (3, 1), 1: (1, -1), 2: (-1, -3)}.items():
        p = 2
        M1 = element_matrix(k, p, unit_cell((1, 1, 1)), 0.0, 1.0)
        M2 = element_matrix(k, p, unit_cell((0.5, 0.5, 0.5)), 0.0, 1.0)
        K1 = element_matrix(k, p, unit_cell((1, 1, 1)), 1.0, 0.0)
        K2 = element_matrix(k, p, unit_cell((0.5, 0.5, 0.5)), 1.0, 0.0)
        np.testing.assert_allclose(M2, M1 * 0.5 ** mexp, atol=1e-13 * np.abs(M1).max() * 8)
        np.testing.assert_allclose(K2, K1 * 0.5 ** kexp, atol=1e-12 * np.abs(K1).max() * 8)


def test_aux_operator_on_a_sheared_affine_cell_equals_the_equivalent_box():
    """Pin of the auxiliary operator beyond axis-aligned cells (eq:sum-factorization_approx,
    P:732-739): on an AFFINE cell x = b + J xi with a non-diagonal J the metric is constant, so
    P_K = alpha |J| sum_m (J^-1 J^-T)_mm S_m + beta |J| M (only the metric's diagonal enters).  That
    is exactly the TRUE operator of the axis-aligned box with half-sizes j_m = (J^-1 J^-T)_mm^(-1/2)
    and coefficients (alpha, beta) |J| / prod(j), computed through the independent element_matrix
    path (itself pinned by closed forms above).  Using J^T J instead of J^-1 J^-T, a transposed J or a
    misplaced weight fails this."""
    import numpy as np
    from oracle.fem import aux_element_matrix, element_matrix
    p, alpha, beta = 3, 1.7, 0.6
    J = np.array([[0.30, 0.05, -0.02], [0.04, 0.25, 0.06], [-0.03, 0.02, 0.20]])
    b = np.array([0.5, 0.4, 0.3])
    Xc = np.zeros((2, 2, 2, 3))
    for az in range(2):
        for ay in range(2):
            for ax in range(2):
                Xc[az, ay, ax] = b + J @ np.array([2 * ax - 1, 2 * ay - 1, 2 * az - 1], dtype=float)
    G = np.linalg.inv(J) @ np.linalg.inv(J).T
    d = abs(np.linalg.det(J))
    jm = 1.0 / np.sqrt(np.diag(G))
    Xb = np.zeros((2, 2, 2, 3))
    for az in range(2):
        for ay in range(2):
            for ax in range(2):
                Xb[az, ay, ax] = np.array([2 * ax - 1, 2 * ay - 1, 2 * az - 1], dtype=float) * jm
    s = d / np.prod(jm)
    P = aux_element_matrix(p, Xc, alpha, beta)
    A = element_matrix(0, p, Xb, alpha * s, beta * s)
    assert np.abs(P - A).max() <= 1e-12 * np.abs(A).max()
    # and the true operator of the sheared cell is NOT this (the off-diagonal metric matters)
    At = element_matrix(0, p, Xc, alpha, beta)
    assert np.abs(At - A).max() > 1e-3 * np.abs(A).max()


@pytest.mark.parametrize("p", [2, 3])
def test_aux_operator_on_a_non_affine_cell_equals_its_definition(p):
    """eq:sum-factorization_approx on a genuinely trilinear (non-affine) cell, from the
    definition with the TRUE weighted mass matrices: diag(M-bar) = diag(G-bar^-T M G-bar^-1) with
    M^0_beta and M^1_alpha assembled by quadrature (element_matrix; their pullbacks are pinned by
    the discrete complex on trilinear cells and the box closed forms), then
    P_K = G0^T diag(M-bar^0) G0 + (G1 D)^T diag(M-bar^1) (G1 D).  aux_element_matrix computes the
    diagonals by sum factorisation with squared broken-basis tables and (J^-1 J^-T)_mm: a wrong
    metric entry, table or square fails here (the off-diagonal metric terms of M^1 drop out of
    its broken-basis diagonal)."""
    from oracle.fem import broken_G3, ref_derivative_pattern_or_values
    rng = np.random.default_rng(7 + p)
    Xc = np.zeros((2, 2, 2, 3))                                  # [az][ay][ax][xyz]
    for az in range(2):
        for ay in range(2):
            for ax in range(2):
                Xc[az, ay, ax] = 0.5 * np.array([ax, ay, az], dtype=float)
    Xc += rng.uniform(-0.08, 0.08, Xc.shape)                     # every vertex moved: non-affine
    alpha, beta = 1.7, 0.6
    M0 = element_matrix(0, p, Xc, 0.0, beta)                     # (psi, beta psi)_K
    M1 = element_matrix(1, p, Xc, 0.0, alpha)                    # (F Psi, alpha F Psi)_K, covariant pullback
    G0, G1 = broken_G3(0, p), broken_G3(1, p)
    d0 = np.diag(np.linalg.solve(G0.T, np.linalg.solve(G0.T, M0.T).T))   # diag(G0^-T M0 G0^-1)
    d1 = np.diag(np.linalg.solve(G1.T, np.linalg.solve(G1.T, M1.T).T))
    D = ref_derivative_pattern_or_values(0, p, values=True)
    D = D.toarray() if hasattr(D, "toarray") else np.asarray(D)
    Db = G1 @ D
    P_def = G0.T @ np.diag(d0) @ G0 + Db.T @ np.diag(d1) @ Db
    P = aux_element_matrix(p, Xc, alpha, beta)
    assert np.abs(P - P_def).max() < 1e-12 * np.abs(P_def).max()
    # and it is not the true operator (the cell is not Cartesian): P differs from A off its pattern
    A = element_matrix(0, p, Xc, alpha, beta)
    assert np.abs(A - P).max() > 1e-3 * np.abs(A).max()
