"""Helpers shared by the GPU parity tests (test infrastructure)."""
import numpy as np

import rm_inputs as ri


def setup_product(w, **kw):
    import paper_2211_14284_b200 as rmb
    coords = None if w.perturb == 0 else ri.vertex_coords(w)
    return rmb.rm_setup(w.nx, w.ny, w.nz, w.p, w.space, ri.cell_alpha(w).ravel(), ri.cell_beta(w).ravel(),
                        w.gamma_d, coords=coords,
                        decomposition=kw.pop("decomposition", {"ph": rmb.RM_PH, "sc-pafw": rmb.RM_SC_PAFW, "sc-ph": rmb.RM_SC_PH}.get(w.decomposition, rmb.RM_PAFW)),
                        factorization=kw.pop("factorization", rmb.RM_ICC_SC if w.factorization == "icc_sc" else rmb.RM_CHOL),
                        **kw)


def setup_oracle(w, **kw):
    from oracle.solver import Problem
    return Problem(w.space, w.p, w.nx, w.ny, w.nz, ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w),
                   w.gamma_d, decomposition=w.decomposition, factorization=w.factorization, **kw)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def oracle_noise_floor(w, f, u):
    """Relative L2 difference of the oracle's own sweep with the Cartesian cell matrices from
    quadrature vs from the box closed form (identical in exact arithmetic; oracle only,
    scripts/cfg4_conditioning.py): the round-off floor two exact implementations share."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    import oracle.fem as fem
    from cfg4_conditioning import closed_form_parts
    a = setup_oracle(w).relax(f, u)
    fem._cartesian_parts.cache_clear()
    orig = fem._cartesian_parts
    fem._cartesian_parts = closed_form_parts
    try:
        b = setup_oracle(w).relax(f, u)
    finally:
        fem._cartesian_parts = orig
        fem._cartesian_parts.cache_clear()
    return rel(b, a)
