"""Oracle: 1D FDM element of arXiv 2211.14284 (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Everything here follows PAPER.md §2.2-§2.3 step by step:

  gll_rule            GLL nodes/weights ("Lagrange interpolants ... GLL points").
  gauss_rule          Gauss-Legendre rule (library primitive), used only for exact 1D
                      integrals of polynomial products.
  lagrange            product-formula Lagrange basis and derivative on given nodes.
  fdm_basis(p)        * A^GLL, B^GLL by exact quadrature,
                      * the interior generalized eigenproblem eq:eigs solved
                        with LAPACK's symmetric-definite routine (P:430-432 uses dsygv),
                      * S_GG = I, S_GI = 0, S_IG = -S_II S_II^T B^GLL_IG,
                      * B-hat, A-hat,
                      * r-hat_0 = lambda_0^{-1/2}, r-hat_j = lambda_j^{-1/2} s'_j,
                      * D-hat_ij = (r-hat_i, s'_j) (Fig 2.2c),
                      * G-bar (broken transform) with the Loewdin reading G4.
  Readings: G3 eigenvalues ascending, eigenvector sign s'_j(-1) > 0;
  G4 G-bar_GG = B-hat_GG^{1/2} (symmetric square root).

Pinned by tests/test_oracle_basis.py (closed forms at p=1,2,3, GLL tables, invariants).
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache
import math

import numpy as np
import scipy.linalg


def legendre_and_derivs(n: int, x: np.ndarray):
    """L_n(x), L_n'(x), L_n''(x) by the three-term recurrence (textbook)."""
    x = np.asarray(x, dtype=np.float64)
    p0, p1 = np.ones_like(x), x.copy()
    if n == 0:
        return p0, np.zeros_like(x), np.zeros_like(x)
    for k in range(1, n):
        p0, p1 = p1, ((2 * k + 1) * x * p1 - k * p0) / (k + 1)
    # p1 = L_n, p0 = L_{n-1};  (1-x^2) L_n' = n (L_{n-1} - x L_n)
    with np.errstate(divide="ignore", invalid="ignore"):
        d1 = n * (p0 - x * p1) / (1.0 - x * x)
        d2 = (2.0 * x * d1 - n * (n + 1) * p1) / (1.0 - x * x)
    return p1, d1, d2


def gll_rule(n: int):
    """n-point Gauss-Lobatto-Legendre rule on [-1,1]: nodes ascending, weights."""
    if n < 2:
        raise ValueError("GLL needs n >= 2")
    m = n - 1
    if n == 2:
        x = np.array([-1.0, 1.0])
    else:
        # interior nodes = roots of L_m'; start from the library roots, polish by Newton
        inner = np.sort(np.polynomial.legendre.Legendre.basis(m).deriv().roots().real)
        for _ in range(4):
            _, d1, d2 = legendre_and_derivs(m, inner)
            inner = inner - d1 / d2
        x = np.concatenate([[-1.0], inner, [1.0]])
    Lm, _, _ = legendre_and_derivs(m, x)
    Lm[0], Lm[-1] = (-1.0) ** m, 1.0
    w = 2.0 / (n * (n - 1) * Lm ** 2)
    return x, w


def gauss_rule(n: int):
    x, w = np.polynomial.legendre.leggauss(n)
    return x, w


def lagrange(nodes: np.ndarray, x: np.ndarray):
    """values[q, j] = l_j(x_q), derivs[q, j] = l_j'(x_q) by the product formula."""
    nodes = np.asarray(nodes, dtype=np.float64)
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    n = len(nodes)
    V = np.ones((len(x), n))
    dV = np.zeros((len(x), n))
    for j in range(n):
        others = [m for m in range(n) if m != j]
        den = np.prod([nodes[j] - nodes[m] for m in others])
        for m in others:
            V[:, j] *= (x - nodes[m])
        for k in others:
            t = np.ones_like(x)
            for m in others:
                if m != k:
                    t = t * (x - nodes[m])
            dV[:, j] += t
        V[:, j] /= den
        dV[:, j] /= den
    return V, dV


@dataclass
class FDM1D:
    p: int
    nodes: np.ndarray      # GLL nodes xi_0..xi_p
    S: np.ndarray          # (p+1, p+1): S[i, j] = s_j(xi_i)
    lam: np.ndarray        # (p+1,) lam[0] = |I| = 2, lam[j] = (s_j', s_j') for j in 1..p-1, lam[p] unused (nan)
    B: np.ndarray          # FDM mass  (s_i, s_j)
    A: np.ndarray          # FDM stiffness (s_i', s_j')
    D: np.ndarray          # (p, p+1) D-hat_ij = (r_i, s_j')
    G: np.ndarray          # (p+1, p+1) broken transform G-bar (P space); DP space uses identity
    Bgll: np.ndarray
    Agll: np.ndarray

    def tab_s(self, x):
        """s_j(x), s_j'(x): shape (len(x), p+1)."""
        V, dV = lagrange(self.nodes, x)
        return V @ self.S, dV @ self.S

    def tab_r(self, x):
        """r_j(x), shape (len(x), p): r_0 = 2^{-1/2}, r_j = lam_j^{-1/2} s_j'."""
        _, ds = self.tab_s(x)
        x = np.atleast_1d(x)
        R = np.empty((len(x), self.p))
        R[:, 0] = 1.0 / math.sqrt(2.0)
        for j in range(1, self.p):
            R[:, j] = ds[:, j] / math.sqrt(self.lam[j])
        return R

    def tab_sbar(self, x):
        """Broken P basis s-bar = s G-bar^{-1}: interface functions orthonormalised."""
        s, ds = self.tab_s(x)
        Gi = np.linalg.inv(self.G)
        return s @ Gi, ds @ Gi


@lru_cache(maxsize=None)
def fdm_basis(p: int) -> FDM1D:
    if p < 1:
        raise ValueError("p >= 1")
    nodes, _ = gll_rule(p + 1)
    xq, wq = gauss_rule(p + 2)                      # exact for degree 2p+3 >= 2p
    L, dL = lagrange(nodes, xq)
    Bgll = L.T @ (wq[:, None] * L)                  # (l_i, l_j)
    Agll = dL.T @ (wq[:, None] * dL)                # (l_i', l_j')
    I = list(range(1, p))
    G_ = [0, p]
    S = np.zeros((p + 1, p + 1))
    S[np.ix_(G_, G_)] = np.eye(2)                   # S_GG = I, S_GI = 0
    lam = np.full(p + 1, np.nan)
    lam[0] = 2.0                                    # lambda_0 = |I-hat|
    if p >= 2:
        vals, vecs = scipy.linalg.eigh(Agll[np.ix_(I, I)], Bgll[np.ix_(I, I)])  # eq:eigs
        order = np.argsort(vals)                    # G3: ascending
        vals, vecs = vals[order], vecs[:, order]
        # G3 sign: s_j'(-1) > 0 ; s_j'(-1) = sum_i l_i'(-1) S_ij (only interior rows of S_II)
        _, dLm1 = lagrange(nodes, np.array([-1.0]))
        slope = dLm1[0, I] @ vecs
        vecs = vecs * np.where(slope < 0, -1.0, 1.0)[None, :]
        S[np.ix_(I, I)] = vecs
        lam[1:p] = vals
        S[np.ix_(I, G_)] = -vecs @ vecs.T @ Bgll[np.ix_(I, G_)]
    B = S.T @ Bgll @ S
    A = S.T @ Agll @ S
    fdm = FDM1D(p, nodes, S, lam, B, A, np.zeros((p, p + 1)), np.eye(p + 1), Bgll, Agll)
    # D-hat_ij = (r_i, s_j') by exact quadrature (degree 2p-2)
    s, ds = fdm.tab_s(xq)
    R = fdm.tab_r(xq)
    fdm.D = R.T @ (wq[:, None] * ds)
    # G-bar: identity on interior, symmetric square root of the interface Gram on {0,p}
    BGG = B[np.ix_(G_, G_)]
    ev, Q = np.linalg.eigh(BGG)
    G = np.eye(p + 1)
    G[np.ix_(G_, G_)] = Q @ np.diag(np.sqrt(ev)) @ Q.T
    fdm.G = G
    return fdm


# ---- symbolic 1D sparsity (used to define structural patterns, never values) -------------
def pattern_B(p: int) -> np.ndarray:
    """Structural pattern of B-hat: diagonal plus (0,p),(p,0)."""
    P = np.eye(p + 1, dtype=bool)
    P[0, p] = P[p, 0] = True
    return P


def pattern_A(p: int) -> np.ndarray:
    """Structural pattern of A-hat: interior block diagonal (eq:fdmbasis), rows/cols 0,p full."""
    P = np.eye(p + 1, dtype=bool)
    P[0, :] = P[p, :] = P[:, 0] = P[:, p] = True
    return P


def pattern_D(p: int) -> np.ndarray:
    """Structural pattern of D-hat (p x p+1): interior column j has the single entry (j,j)
    (eq:gradbasis); columns 0 and p are full (Fig 2.2c)."""
    P = np.zeros((p, p + 1), dtype=bool)
    for j in range(1, p):
        P[j, j] = True
    P[:, 0] = P[:, p] = True
    return P


def pattern_G(p: int) -> np.ndarray:
    return pattern_B(p)
