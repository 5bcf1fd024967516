"""Helpers shared by the GPU parity tests (test infrastructure)."""
import numpy as np

import rm_inputs as ri


def setup_product(w, **kw):
    import paper_2211_14284_b200 as rmb
    coords = None if w.perturb == 0 else ri.vertex_coords(w)
    return rmb.rm_setup(w.nx, w.ny, w.nz, w.p, w.space, ri.cell_alpha(w).ravel(), ri.cell_beta(w).ravel(),
                        w.gamma_d, coords=coords,
                        decomposition=kw.pop("decomposition", rmb.RM_PH if w.decomposition == "ph" else rmb.RM_PAFW),
                        factorization=kw.pop("factorization", rmb.RM_ICC_SC if w.factorization == "icc_sc" else rmb.RM_CHOL),
                        **kw)


def setup_oracle(w, **kw):
    from oracle.solver import Problem
    return Problem(w.space, w.p, w.nx, w.ny, w.nz, ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w),
                   w.gamma_d, decomposition=w.decomposition, factorization=w.factorization, **kw)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
