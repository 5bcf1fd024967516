"""Pins of the oracle's sweep and PCG (oracle/solver.py) to properties the paper and the
algebra fix.  CPU only."""
import numpy as np
import pytest

import rm_inputs as ri
from oracle.solver import Problem


def make(w, **kw):
    return Problem(w.space, w.p, w.nx, w.ny, w.nz, ri.vertex_coords(w), ri.cell_alpha(w),
                   ri.cell_beta(w), w.gamma_d, decomposition=kw.pop("decomposition", w.decomposition),
                   factorization=kw.pop("factorization", w.factorization), **kw)


def vec(pb, cfg, s):
    v = ri.uniform_vector(cfg, s, pb.space.ndof)
    v[pb.constrained] = 0.0
    return v


def test_interior_only_single_patch_is_exact_solve():
    """RM_INTERIOR_ONLY on 2x2x2 with Dirichlet everywhere: one patch covering all free DoFs,
    so one sweep with omega=1 from u=0 solves A u = f exactly."""
    w = ri.CONFIGS[1].with_mesh(2)
    pb = make(w, interior_only=True)
    assert len(pb.patch_solvers()) == 1
    f = vec(pb, 1, 0)
    u = pb.relax(f, np.zeros_like(f))
    assert np.abs(pb.apply(u) - f).max() < 1e-12 * np.abs(f).max() * 10
    _, it, _ = pb.pcg(f)
    assert it == 1


@pytest.mark.parametrize("cfg,p,n", [(1, 3, 3), (2, 3, 3), (3, 2, 2), (4, 2, 2), (5, 2, 2)])
def test_sweep_linear_and_symmetric(cfg, p, n):
    w = ri.CONFIGS[cfg].with_mesh(n).with_p(p)
    pb = make(w)
    f, u = vec(pb, cfg, 0), vec(pb, cfg, 3)
    # linear in (f, u)
    a, b = 0.7, -1.3
    lhs = pb.relax(a * f, a * u) + pb.relax(b * f, b * u)
    rhs = pb.relax((a + b) * f, (a + b) * u)
    assert np.abs(lhs - rhs).max() < 1e-11 * np.abs(rhs).max()
    # the preconditioner is symmetric: v^T P^{-1} w = w^T P^{-1} v
    v2 = vec(pb, cfg, 7)
    assert abs(v2 @ pb.precondition(f) - f @ pb.precondition(v2)) < 1e-11 * abs(f @ pb.precondition(f))
    # fixed point: the exact solution is not moved by a sweep
    x, it, rel = pb.pcg(f, rtol=1e-13)
    np.testing.assert_allclose(pb.relax(f, x), x, atol=1e-8 * np.abs(x).max())


def test_pcg_scale_invariance():
    """Iteration counts depend only on alpha/beta."""
    w = ri.CONFIGS[2].with_mesh(3).with_p(3)
    pb = make(w)
    f = vec(pb, 2, 0)
    _, it1, _ = pb.pcg(f)
    pb2 = Problem(w.space, w.p, 3, 3, 3, ri.vertex_coords(w), 1e3 * ri.cell_alpha(w), 1e3 * ri.cell_beta(w),
                  w.gamma_d)
    _, it2, _ = pb2.pcg(f)
    assert it1 == it2


def test_pcg_p_robust_hgrad():
    its = []
    for p in (2, 3, 4):
        w = ri.CONFIGS[1].with_mesh(3).with_p(p)
        pb = make(w)
        _, it, rel = pb.pcg(vec(pb, 1, 0))
        assert rel <= 1e-8
        its.append(it)
    assert max(its) - min(its) <= 3


def test_pcg_solves_system():
    w = ri.CONFIGS[1]
    pb = make(w)
    f = vec(pb, 1, 0)
    x, it, rel = pb.pcg(f)
    assert rel <= 1e-8 and 5 <= it <= 40
    r = f - pb.apply(x)
    assert np.linalg.norm(r) < 1e-6 * np.linalg.norm(f)
