"""Pins of the oracle's patches and patch factors (oracle/patches.py).  CPU only."""
import math

import numpy as np
import pytest
import scipy.sparse as sp

import rm_inputs as ri
from oracle.fem import Space, assemble, assemble_aux
from oracle.patches import DenseCholeskyPatch, ICCSCPatch, all_patches, entities, icc_masked, patch_dofs


def test_entity_counts():
    s = Space(0, 2, 2, 2, 2)
    assert len(entities(s, 0)) == 27 and len(entities(s, 1)) == 54 and len(entities(s, 2)) == 36


@pytest.mark.parametrize("p", [2, 3, 5])
def test_full_star_sizes(p):
    """Interior stars on a 3x3x3 mesh: vertex (2p-1)^3 (k=0); NCE x-edge p(2p-1)^2+4p(p-1)(2p-1);
    NCF x-face p^2(6p-5) (SURVEY App. A worked counts)."""
    n = 3
    none = np.zeros(Space(0, p, n, n, n).ndof, dtype=bool)
    g, _ = patch_dofs(Space(0, p, n, n, n), (("node", 1), ("node", 1), ("node", 1)), none)
    assert len(g) == (2 * p - 1) ** 3
    s1 = Space(1, p, n, n, n)
    g, _ = patch_dofs(s1, (("cell", 1), ("node", 1), ("node", 1)), np.zeros(s1.ndof, dtype=bool))
    assert len(g) == p * (2 * p - 1) ** 2 + 4 * p * (p - 1) * (2 * p - 1)
    s2 = Space(2, p, n, n, n)
    g, _ = patch_dofs(s2, (("node", 1), ("cell", 1), ("cell", 1)), np.zeros(s2.ndof, dtype=bool))
    assert len(g) == p * p * (6 * p - 5)


def test_star_cells_and_boundary_clipping():
    p = 3
    s = Space(0, p, 2, 2, 2)
    con = s.constrained_mask(ri.GAMMA_X0)
    # corner vertex at x=0 (Dirichlet): x window 1..p-1, y,z windows 0..p-1 (Neumann)
    g, grp = patch_dofs(s, (("node", 0), ("node", 0), ("node", 0)), con)
    assert len(g) == (p - 1) * p * p
    # vertex x=2 (Neumann side): window 2p-(p-1)..2p -> p entries
    g, _ = patch_dofs(s, (("node", 2), ("node", 1), ("node", 1)), con)
    assert len(g) == p * (2 * p - 1) ** 2
    # all stars together cover every free DoF
    cover = np.zeros(s.ndof, dtype=int)
    for ent, g, grp in all_patches(s, 0, con):
        cover[g] += 1
    assert (cover[~con] >= 1).all() and (cover[con] == 0).all()
    assert cover.max() == 8


def test_pinned_order_groups():
    p = 3
    s = Space(0, p, 2, 2, 2)
    none = np.zeros(s.ndof, dtype=bool)
    g, grp = patch_dofs(s, (("node", 1), ("node", 1), ("node", 1)), none)
    assert np.all(np.diff(grp) >= 0)
    assert (grp == 0).sum() == 8 * (p - 1) ** 3
    assert (grp == 1).sum() == 12 * (p - 1) ** 2
    assert (grp == 2).sum() == 6 * (p - 1)
    assert (grp == 3).sum() == 1


def _brute_masked_icc(a, mask):
    n = a.shape[0]
    L = np.zeros_like(a)
    for j in range(n):
        L[j, j] = math.sqrt(a[j, j] - sum(L[j, k] ** 2 for k in range(j)))
        for i in range(j + 1, n):
            if mask[i, j]:
                L[i, j] = (a[i, j] - sum(L[i, k] * L[j, k] for k in range(j))) / L[j, j]
    return L


def _aux_problem(p, n=2, perturb=0.1):
    w = ri.Workload(5, 0, p, n, n, n, "one", 1.0, 0, perturb, "pafw", "icc_sc")
    s = Space(0, p, n, n, n)
    P, S = assemble_aux(s, ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w))
    return s, P, S


def test_icc_full_pattern_equals_cholesky():
    s, P, S = _aux_problem(2)
    g, grp = patch_dofs(s, (("node", 1), ("node", 1), ("node", 1)), np.zeros(s.ndof, dtype=bool))
    A = P[g][:, g].toarray()
    full = sp.csr_matrix(np.tril(np.ones_like(A)))
    L = icc_masked(sp.csr_matrix(A), full).toarray()
    np.testing.assert_allclose(L, np.linalg.cholesky(A), atol=1e-12 * np.abs(A).max())


@pytest.mark.parametrize("p", [2, 3])
def test_icc_sc_matches_brute_force_definition(p):
    s, P, S = _aux_problem(p)
    g, grp = patch_dofs(s, (("node", 1), ("node", 1), ("node", 1)), np.zeros(s.ndof, dtype=bool))
    A = P[g][:, g]
    pat = S[g][:, g]
    f = ICCSCPatch(A.tocsr(), pat.tocsr(), grp == 0)
    Lb = _brute_masked_icc(A.toarray(), f.mask.toarray() != 0)
    np.testing.assert_allclose(f.L.toarray(), Lb, atol=1e-12 * np.abs(Lb).max())
    assert f.sigma == 0.0


def test_icc_sc_equals_interior_elimination_then_icc0_of_schur():
    """With interiors first and P_II diagonal, ICC-SC = exact interior elimination followed by
    ICC(0) on the patch Schur complement (SURVEY §8(c) step 7 note)."""
    p = 3
    s, P, S = _aux_problem(p)
    g, grp = patch_dofs(s, (("node", 1), ("node", 1), ("node", 1)), np.zeros(s.ndof, dtype=bool))
    A = P[g][:, g].toarray()
    pat = S[g][:, g].toarray() != 0
    I = grp == 0
    G = ~I
    assert np.count_nonzero(A[np.ix_(I, I)] - np.diag(np.diag(A[np.ix_(I, I)]))) == 0
    f = ICCSCPatch(sp.csr_matrix(A), sp.csr_matrix(pat.astype(float)), I)
    Sc = A[np.ix_(G, G)] - A[np.ix_(G, I)] @ np.diag(1 / np.diag(A[np.ix_(I, I)])) @ A[np.ix_(I, G)]
    patS = pat[np.ix_(G, G)] | ((pat[np.ix_(G, I)].astype(int) @ pat[np.ix_(I, G)].astype(int)) != 0)
    LS = _brute_masked_icc(Sc, patS)
    np.testing.assert_allclose(f.L.toarray()[np.ix_(G, G)], LS, atol=1e-11 * np.abs(LS).max())


def test_face_star_zero_fill():
    """H(div) face-star patch matrices in the FDM basis: Cholesky has no fill."""
    p = 3
    n = 3
    s = Space(2, p, n, n, n)
    X = ri.vertex_coords(ri.Workload(4, 2, p, n, n, n, "one", 1e-2, 63, 0.0, "ph", "chol"))
    A = assemble(s, X, np.ones((n,) * 3), np.full((n,) * 3, 1e-2))
    con = s.constrained_mask(ri.GAMMA_ALL)
    g, _ = patch_dofs(s, (("node", 1), ("cell", 1), ("cell", 1)), con)
    Af = A[g][:, g].toarray()
    L = np.linalg.cholesky(Af)
    tol = 1e-12 * np.abs(L).max()
    assert np.count_nonzero(np.abs(L) > tol) == np.count_nonzero(np.abs(np.tril(Af)) > 1e-12 * np.abs(Af).max())


def test_dense_cholesky_patch_solve():
    rng = np.random.default_rng(1)
    M = rng.standard_normal((20, 20))
    A = M @ M.T + 20 * np.eye(20)
    b = rng.standard_normal(20)
    np.testing.assert_allclose(DenseCholeskyPatch(A).solve(b), np.linalg.solve(A, b), rtol=1e-12)
