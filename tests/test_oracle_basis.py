"""Pins of the oracle's 1D element (oracle/basis1d.py) to closed forms and invariants fixed by
PAPER.md §2.2-§2.3 (not to the oracle itself).  CPU only."""
import json
import math
import os

import numpy as np
import pytest

from oracle.basis1d import fdm_basis, gauss_rule, gll_rule, lagrange, pattern_A, pattern_B, pattern_D

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def ev(s, p=None):
    if isinstance(s, (int, float)):
        return float(s)
    return float(eval(s, {"sqrt": math.sqrt, "p": p}))


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


@pytest.mark.parametrize("n", [2, 3, 4])
def test_gll_closed_forms(n):
    g = load("gll.json")[f"n{n}"]
    x, w = gll_rule(n)
    np.testing.assert_allclose(x, [ev(v) for v in g["x"]], atol=1e-15)
    np.testing.assert_allclose(w, [ev(v) for v in g["w"]], atol=1e-15)


@pytest.mark.parametrize("n", [5, 8, 12, 24])
def test_gll_exactness_degree(n):
    # exact for degree 2n-3 (monomial integrals), not for 2n-2 (x^{2n-2} is even)
    x, w = gll_rule(n)
    for d in range(0, 2 * n - 2):
        exact = 0.0 if d % 2 else 2.0 / (d + 1)
        assert abs(w @ x ** d - exact) < 1e-13
    if n <= 8:   # degree 2n-2 is not integrated exactly (error shrinks fast with n)
        d = 2 * n - 2
        assert abs(w @ x ** d - 2.0 / (d + 1)) > 1e-9


def test_lagrange_small():
    V, dV = lagrange(np.array([-1.0, 0.0, 1.0]), np.array([0.5]))
    np.testing.assert_allclose(V[0], [-1 / 8, 3 / 4, 3 / 8], atol=1e-15)
    V, dV = lagrange(np.array([-1.0, 1.0]), np.array([0.0]))
    np.testing.assert_allclose(V[0], [0.5, 0.5]); np.testing.assert_allclose(dV[0], [-0.5, 0.5])


def test_p1_closed_forms():
    g = load("fdm_closed_forms.json")["p1"]
    f = fdm_basis(1)
    np.testing.assert_allclose(f.B, [[ev(v) for v in r] for r in g["B"]], atol=1e-15)
    np.testing.assert_allclose(f.A, [[ev(v) for v in r] for r in g["A"]], atol=1e-15)
    np.testing.assert_allclose(f.D, [[ev(v) for v in r] for r in g["D"]], atol=1e-15)


def test_p2_closed_forms():
    g = load("fdm_closed_forms.json")["p2"]
    f = fdm_basis(2)
    assert abs(f.lam[1] - 2.5) < 1e-13
    s, ds = f.tab_s(np.array([0.0]))
    assert abs(s[0, 1] - ev(g["s1_at_0"])) < 1e-14
    assert abs(s[0, 0] - ev(g["s0_at_0"])) < 1e-14
    # the closed-form functions themselves at random points
    x = np.linspace(-1, 1, 7)
    s, _ = f.tab_s(x)
    np.testing.assert_allclose(s[:, 1], math.sqrt(15) / 4 * (1 - x ** 2), atol=1e-14)
    np.testing.assert_allclose(s[:, 0], (5 * x ** 2 - 4 * x - 1) / 8, atol=1e-14)
    np.testing.assert_allclose(f.B, [[ev(v) for v in r] for r in g["B"]], atol=1e-14)
    np.testing.assert_allclose(f.A, [[ev(v) for v in r] for r in g["A"]], atol=1e-13)
    np.testing.assert_allclose(f.D, [[ev(v) for v in r] for r in g["D"]], atol=1e-14)


def test_p3_eigenvalues():
    g = load("fdm_closed_forms.json")["p3"]
    f = fdm_basis(3)
    np.testing.assert_allclose(f.lam[1:3], [ev(v) for v in g["lambda"]], rtol=1e-13)


@pytest.mark.parametrize("p", [2, 3, 4, 6, 7, 8, 15])
def test_fdm_invariants(p):
    f = fdm_basis(p)
    I = slice(1, p)
    lam = f.lam[1:p]
    # eq:eigs: S_II^T B S_II = I, S_II^T A S_II = Lambda (relative to lambda_max)
    Sii = f.S[I, I]
    np.testing.assert_allclose(Sii.T @ f.Bgll[I, I] @ Sii, np.eye(p - 1), atol=1e-12)
    np.testing.assert_allclose(Sii.T @ f.Agll[I, I] @ Sii / lam.max(), np.diag(lam) / lam.max(), atol=1e-12)
    assert np.all(np.diff(lam) > 0)                   # reading G3 ascending
    # B-hat: diagonal + (0,p) only with the closed forms of the interface block
    off = np.where(pattern_B(p), 0.0, f.B)
    assert np.abs(off).max() < 1e-13
    np.testing.assert_allclose(f.B[0, 0], 2 / (p * (p + 2)), rtol=1e-12)
    np.testing.assert_allclose(f.B[p, p], 2 / (p * (p + 2)), rtol=1e-12)
    np.testing.assert_allclose(f.B[0, p], (-1) ** (p + 1) * 2 / (p * (p + 1) * (p + 2)), rtol=1e-10)
    np.testing.assert_allclose(np.diag(f.B)[I], 1.0, atol=1e-12)
    # A-hat: interior block diagonal = Lambda
    offA = np.where(pattern_A(p), 0.0, f.A)
    assert np.abs(offA).max() < 1e-10 * lam.max()
    np.testing.assert_allclose(np.diag(f.A)[I], lam, rtol=1e-12)
    # D-hat interior columns: single entry lambda_j^{1/2} (eq:gradbasis); D^T D = A (DP basis orthonormal)
    offD = np.where(pattern_D(p), 0.0, f.D)
    assert np.abs(offD).max() < 1e-11 * math.sqrt(lam.max())
    np.testing.assert_allclose([f.D[j, j] for j in range(1, p)], np.sqrt(lam), rtol=1e-12)
    np.testing.assert_allclose(f.D.T @ f.D, f.A, atol=1e-12 * lam.max())
    assert abs(f.D[0, 0] + 1 / math.sqrt(2)) < 1e-12 and abs(f.D[0, p] - 1 / math.sqrt(2)) < 1e-12
    # r-hat orthonormal including r0
    xq, wq = gauss_rule(p + 2)
    R = f.tab_r(xq)
    np.testing.assert_allclose(R.T @ (wq[:, None] * R), np.eye(p), atol=1e-12)
    # duality: (s_i, s_j) = 0 for i interior, j interface; s_j(+-1) = delta
    s, ds = f.tab_s(np.array([-1.0, 1.0]))
    np.testing.assert_allclose(s[0], np.eye(p + 1)[0], atol=1e-13)
    np.testing.assert_allclose(s[1], np.eye(p + 1)[p], atol=1e-13)
    # sign reading G3: s_j'(-1) > 0, well separated from 0
    assert ds[0, 1:p].min() > 1.0
    # constant function: coefficients c = [1, (s_j,1), 1] ; D c = 0 ; c^T B c = |I| = 2
    sq, _ = f.tab_s(xq)
    c = np.ones(p + 1)
    c[1:p] = wq @ sq[:, 1:p]
    assert np.abs(f.D @ c).max() < 1e-12
    assert abs(c @ f.B @ c - 2.0) < 1e-12
    # G-bar: transformed interface Gram = I (reading G4), interior block identity
    G = f.G
    Gi = np.linalg.inv(G)
    np.testing.assert_allclose(Gi.T @ f.B @ Gi, np.eye(p + 1), atol=1e-12)
    np.testing.assert_allclose(G[I, I], np.eye(p - 1), atol=0)
