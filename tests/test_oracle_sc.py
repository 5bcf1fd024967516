"""Pins of the statically condensed decomposition SC-PAFW (oracle/solver.py precondition_sc,
eq:sc-pafw / eq:schur / eq:sc-asm-afw; row f2 for k = 0).  CPU only."""
import dataclasses

import numpy as np
import pytest

import rm_inputs as ri
from oracle.solver import Problem


def make(w, **kw):
    return Problem(w.space, w.p, w.nx, w.ny, w.nz, ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w),
                   w.gamma_d, decomposition=kw.pop("decomposition", w.decomposition),
                   factorization=kw.pop("factorization", w.factorization), **kw)


def vec(pb, cfg, s):
    v = ri.uniform_vector(cfg, s, pb.space.ndof)
    v[pb.constrained] = 0.0
    return v


def test_sc_single_patch_is_exact_solve():
    """Interior-only stars on 2x2x2 with Dirichlet everywhere: one vertex star holds every interface
    DoF, so S_v = S and eq:schur is the exact inverse (one sweep solves A u = f)."""
    w = ri.CONFIGS[1].with_mesh(2)
    pb = make(w, decomposition="sc-pafw", interior_only=True)
    f = vec(pb, 1, 0)
    u = pb.relax(f, np.zeros_like(f))
    assert np.abs(pb.apply(u) - f).max() < 1e-11 * np.abs(f).max()


@pytest.mark.parametrize("cfg,p,n", [(1, 3, 3), (2, 4, 3), (5, 3, 2)])
def test_sc_interface_part_equals_the_patch_elimination(cfg, p, n):
    """The interface part of SC-PAFW equals that of PAFW: each star's block elimination with its
    interiors first computes S_v^{-1} (r_G - A_GI A_II^{-1} r_I) on its interface (LDL^T, eq:LDU),
    because every cell carrying a star's interface DoF is a star cell.  (Exact: both factorizations;
    ICC-SC: ICC(0) of S_v = the masked ICC with interiors first, reading G19.)  The interiors
    differ: SC solves them once, c_I = A_II^{-1}(r_I - A_IG c_G)."""
    w = ri.CONFIGS[cfg].with_mesh(n).with_p(p)
    a = make(w)
    b = make(w, decomposition="sc-pafw")
    r = vec(a, cfg, 0)
    ca, cb = a.precondition(r), b.precondition(r)
    _, I, dI, _ = b.sc_data()
    G = np.setdiff1d(np.flatnonzero(a.free), I)
    assert np.abs(ca[G] - cb[G]).max() < 1e-11 * np.abs(ca).max()
    At = b.sc_data()[0]
    cI = (r[I] - At[I] @ cb) / dI + (At[I][:, I] @ cb[I]) / dI   # r_I - A_IG c_G (c_G = cb on G)
    assert np.abs(cb[I] - cI).max() < 1e-11 * np.abs(cb).max()
    assert np.abs(ca[I] - cb[I]).max() > 1e-6 * np.abs(ca).max()   # the interiors do differ


@pytest.mark.parametrize("cfg,p,n", [(1, 3, 3), (5, 3, 2)])
def test_sc_symmetric_and_fewer_iterations(cfg, p, n):
    """SC-PAFW is symmetric and converges like the non-condensed decomposition (one-level: equal
    counts within 2 -- the harmonic subspaces overlap less; the paper's 14 -> 11 at
    p = 3 is with its own level smoother in the hybrid cycle, which it does not state)."""
    w = ri.CONFIGS[cfg].with_mesh(n).with_p(p)
    b = make(w, decomposition="sc-pafw")
    x, y = vec(b, cfg, 0), vec(b, cfg, 3)
    assert abs(y @ b.precondition(x) - x @ b.precondition(y)) < 1e-11 * abs(x @ b.precondition(x))
    its = []
    for dec in ("pafw", "sc-pafw"):
        pb = make(w, decomposition=dec)
        _, it, rel = pb.pcg(vec(pb, cfg, 0))
        assert rel <= 1e-8
        its.append(it)
    assert abs(its[1] - its[0]) <= 2, its


# ------------------------------------------------------------------ SC-PH (k = 1, 2)
SCPH_CASES = [(3, 3, 2), (4, 3, 2), (3, 2, 3)]


@pytest.mark.parametrize("cfg,p,n", SCPH_CASES)
def test_scph_schur_identity_is_the_exact_inverse(cfg, p, n):
    """eq:schur with the oracle's own pieces: R_I^T A_II^{-1} R_I + R_G^T S^{-1} R_G = A^{-1} (a wrong
    sign in R_G, a transposed coupling or a wrong interior set breaks it)."""
    import scipy.sparse.linalg as spla
    w = ri.CONFIGS[cfg].with_mesh(n).with_p(p)
    pb = make(w, decomposition="sc-ph")
    A, I, G, AIIinv, S, _, _, _ = pb.sc_ph_data()
    r = vec(pb, cfg, 0)
    yI = AIIinv @ r[I]
    rG = r[G] - A[G][:, I] @ yI
    cG = spla.spsolve(S.tocsc(), rG)
    c = np.zeros_like(r)
    c[G] = cG
    c[I] = yI - AIIinv @ (A[I][:, G] @ cG)
    # backward error, scaled by kappa(A_II): with beta = 1e-2 the H(div) interior blocks reach
    # kappa ~ 5e4 and c_I = y_I - A_II^{-1} A_IG c_G cancels terms ~ 1/beta larger than the result
    kap = np.linalg.cond(A[I][:, I].toarray())
    assert np.linalg.norm(A @ c - r) < 1e-11 * max(1.0, kap) * np.linalg.norm(r)
    # the interior blocks are <= 3x3 (remark P:1061-1066): A_II^{-1} has A_II's pattern
    assert AIIinv.nnz == A[I][:, I].nnz


@pytest.mark.parametrize("cfg,p,n", SCPH_CASES)
def test_scph_star_interface_parts_equal_the_ph_star_eliminations(cfg, p, n):
    """eq:LDU per star: the interface part of each k-star's exact solve A_i^{-1} R_i r equals
    S_i^{-1} R~_i R_G r, and for the potential stage the interface part of each (k-1)-star's solve
    with B applied to an interface-only vector t equals B~_j^{-1} R~_j t (every cell carrying a
    star's interface DoF is a star cell)."""
    w = ri.CONFIGS[cfg].with_mesh(n).with_p(p)
    ph = make(w, decomposition="ph")
    sc = make(w, decomposition="sc-ph")
    A, I, G, AIIinv, S, prim, Dt, pot = sc.sc_ph_data()
    r = vec(sc, cfg, 0)
    rG = r[G] - A[G][:, I] @ (AIIinv @ r[I])
    ca = np.zeros_like(r)
    for g, P_ in ph.patch_solvers():
        ca[g] += P_.solve(r[g])
    cG = np.zeros(len(G))
    for loc, P_ in prim:
        cG[loc] += P_.solve(rG[loc])
    # forward differences of two exact eliminations ~ kappa eps (H(div), beta = 1e-2: kappa(A_II) ~ 5e4)
    tol = 1e-10 * max(1.0, np.linalg.cond(A[I][:, I].toarray()))
    assert np.abs(ca[G] - cG).max() < tol * np.abs(cG).max()
    D, pcon, sol = ph.potential()
    from oracle.solver import interior_mask
    from oracle.fem import Space
    pspace = Space(w.space - 1, w.p, w.nx, w.ny, w.nz)
    Gb = np.flatnonzero(~pcon & ~interior_mask(pspace))
    t = np.zeros(D.shape[1])
    t[Gb] = Dt.T @ rG
    sa = np.zeros_like(t)
    for g, P_ in sol:
        sa[g] += P_.solve(t[g])
    sb = np.zeros(len(Gb))
    for loc, P_ in pot:
        sb[loc] += P_.solve(t[Gb][loc])
    assert np.abs(sa[Gb] - sb).max() < tol * np.abs(sb).max()
    # d of an interior (k-1)-form bubble is an interior k-form bubble: D_GI = 0, so D~ = D_GG is
    # the whole action of d on interface potentials seen by the interface
    Ib = np.flatnonzero(~pcon & interior_mask(pspace))
    assert abs(D[G][:, Ib]).max() == 0.0


@pytest.mark.parametrize("cfg", [3, 4])
def test_scph_symmetric_robust_in_beta_and_needs_the_potential_stage(cfg):
    """S_PH^{-1} is symmetric; PCG iteration counts stay flat as beta -> 0 (the potential stage
    carries the kernel of d) and grow without it."""
    w = ri.CONFIGS[cfg].with_mesh(3).with_p(3)
    its = {}
    for beta in (1.0, 1e-4):
        pb = make(w, decomposition="sc-ph")
        pb.beta = np.full_like(pb.beta, beta)
        x, y = vec(pb, cfg, 0), vec(pb, cfg, 3)
        assert abs(y @ pb.precondition(x) - x @ pb.precondition(y)) < 1e-10 * abs(x @ pb.precondition(x))
        _, it, rel = pb.pcg(vec(pb, cfg, 0))
        assert rel <= 1e-8
        its[beta] = it
    assert its[1e-4] <= its[1.0] + 4, its
    pb = make(w, decomposition="sc-ph")
    pb.beta = np.full_like(pb.beta, 1e-4)
    pb.precondition = lambda r: pb.precondition_sc_ph(r, potential_stage=False)
    _, it, _ = pb.pcg(vec(pb, cfg, 0), maxit=4 * its[1e-4] + 20)
    assert it > 2 * its[1e-4], (it, its)
