"""Oracle: the p = 1 coarse level and the hybrid V(1,1) cycle (TEST INFRASTRUCTURE ONLY).

Follows PAPER.md:
  * eq:asm-afw / eq:asm-hiptmair: the coarse term R_0^T A_0^{-1} R_0, with A_0 "the
    stiffness matrix for the original bilinear form a^k rediscretized with the lowest-order
    element (p = 1)" and R_0 "the restriction matrix from (V^k_{h,p})^* to (V^k_{h,1})^*" -- the
    transpose of the embedding V^k_{h,1} -> V^k_{h,p} written in the FDM reference values.
  * "they combine patches additively within each level, and the levels are combined
    multiplicatively in a V(1,1)-cycle".

Embedding (per direction, tensor-product structure of eq:hgrad-basis..eq:hdiv-basis):
  P family  (n p + 1) x (n + 1): the lowest-order functions phi_0 = (1 - x)/2, phi_1 = (1 + x)/2 of
            cell c expressed in the FDM basis s_0..s_p of that cell.  s_j(-1) = delta_j0,
            s_j(1) = delta_jp and the interior s_j are L2-orthonormal and L2-orthogonal to s_0, s_p
            (B-hat has zeros outside diag U (0,p)), so the vertex coefficients are the
            vertex values and the interior ones are (s_j, phi_a) (exact Gauss quadrature).
  DP family (n p) x n: the p = 1 DP function r_0 = 2^{-1/2} is the degree-p r_0 itself.
A_0 is assembled by oracle.fem at p = 1 (GLL quadrature with ceil(3 * 2 / 2) = 3 points, reading
G1) with the fine problem's coefficients and Dirichlet set; constrained DoFs are held at zero.

Hybrid V(1,1) (reading G20): with S the additive patch sum of the fine level (the
preconditioner of oracle.solver, potential stage included) and C_0 = R_0^T A_0^{-1} R_0,
    z_1 = w S r,   z_2 = z_1 + C_0 (r - A z_1),   z = z_2 + w S (r - A z_2)
with the smoother damping w = 1 / N_c, N_c = the number of patch colours of the level (8 vertex,
12 edge, 6 face stars; the PH potential stage adds its own): each colour is a sum of A-orthogonal
projections onto A-orthogonal subspaces, so lambda_max(S A) <= N_c and I - w S A is a contraction;
the cycle is then symmetric positive definite.

Pins (tests/test_oracle_coarse.py): the embedding reproduces the lowest-order functions exactly
(closed form at sample points); Galerkin identity R_0 A_p R_0^T = A_0 on Cartesian cells (the forms
are the same and both quadratures are exact there); the cycle is symmetric; for p = 1 the coarse
space is the whole space and PCG converges in one iteration (the "1/1" row); PCG counts
are invariant under (alpha, beta) -> c (alpha, beta).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg
import scipy.sparse as sp

from .basis1d import fdm_basis, gauss_rule
from .fem import P_FAM, Space, assemble


def embed_1d(p: int, fam: str, ncell: int) -> sp.csr_matrix:
    """Global 1D embedding of the p = 1 family into the degree-p family (rows fine, cols coarse)."""
    if fam != P_FAM:
        E = sp.lil_matrix((ncell * p, ncell))
        for c in range(ncell):
            E[c * p, c] = 1.0
        return E.tocsr()
    f = fdm_basis(p)
    xq, wq = gauss_rule(p + 2)
    s, _ = f.tab_s(xq)
    phi = np.stack([(1 - xq) / 2, (1 + xq) / 2], axis=1)   # phi_0, phi_1 at the Gauss points
    inner = (s * wq[:, None]).T @ phi                        # (s_j, phi_a)
    E = sp.lil_matrix((ncell * p + 1, ncell + 1))
    for c in range(ncell):
        E[c * p, c] = 1.0
        E[c * p + p, c + 1] = 1.0
        for j in range(1, p):
            E[c * p + j, c] = inner[j, 0]
            E[c * p + j, c + 1] = inner[j, 1]
    return E.tocsr()


def prolongation(k: int, p: int, nx: int, ny: int, nz: int) -> sp.csr_matrix:
    """R_0^T: V^k_{h,1} -> V^k_{h,p} on reference values, block-diagonal over components, each a
    Kronecker product of the 1D embeddings (x fastest)."""
    sp_p = Space(k, p, nx, ny, nz)
    n = (nx, ny, nz)
    blocks = []
    for fam in sp_p.fams:
        Ex, Ey, Ez = (embed_1d(p, fam[d], n[d]) for d in range(3))
        blocks.append(sp.kron(Ez, sp.kron(Ey, Ex, format="csr"), format="csr"))
    return sp.block_diag(blocks, format="csr")


def smoother_colours(k: int, decomposition: str) -> int:
    """N_c of reading G20: patch colours of the primary family plus the potential family."""
    prim = {0: 8, 1: 12, 2: 6}[0 if decomposition == "pafw" else k]
    pot = 0 if (decomposition == "pafw" or k == 0) else {1: 8, 2: 12}[k]
    return prim + pot


class CoarseLevel:
    """C_0 = R_0^T A_0^{-1} R_0 for a oracle.solver.Problem (dense Cholesky of the free A_0)."""

    def __init__(self, pb):
        self.space1 = Space(pb.k, 1, pb.nx, pb.ny, pb.nz)
        self.con1 = self.space1.constrained_mask(pb.gamma_d)
        self.free1 = np.flatnonzero(~self.con1)
        A0 = assemble(self.space1, pb.X, pb.alpha, pb.beta).tocsr()
        self.A0 = A0[self.free1][:, self.free1].toarray()
        self.L = np.linalg.cholesky(self.A0)
        self.E = prolongation(pb.k, pb.p, pb.nx, pb.ny, pb.nz)
        self.free = pb.free

    def apply(self, r):
        r = np.where(self.free, r, 0.0)
        b = (self.E.T @ r)[self.free1]
        y = scipy.linalg.solve_triangular(self.L, b, lower=True)
        x = scipy.linalg.solve_triangular(self.L.T, y, lower=False)
        xc = np.zeros(self.space1.ndof)
        xc[self.free1] = x
        return np.where(self.free, self.E @ xc, 0.0)


def vcycle(pb, coarse: CoarseLevel, r, omega):
    """Hybrid V(1,1): z = M r (module header)."""
    z1 = omega * pb.precondition(r)
    z2 = z1 + coarse.apply(r - pb.apply(z1))
    return z2 + omega * pb.precondition(r - pb.apply(z2))
