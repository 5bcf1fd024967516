"""Derivation of the H(div) (cfg4 shapes) parity tolerance -- calls only the oracle.

Two correct fp64 implementations of an exact patch solve differ by about kappa(A_i) * eps
relative: their patch matrices already differ by O(eps) entrywise (different, equally exact
assembly arithmetic) and the solve amplifies that by the condition number.  The face-star
matrices of H(div) with beta = 1e-2 (BASELINE cfg4) are rank-deficient div-div blocks plus a
small mass, so kappa grows to 1e5-1e7 and the north-star 1e-11 is below what any pair of fp64
implementations can agree to.  This script
  1. computes kappa_max over the distinct primary (face-star) and potential (edge-star)
     patch matrices of the GPU parity shapes,
  2. demonstrates the effect inside the oracle alone: the same sweep with the Cartesian cell
     matrices assembled by the box closed form (Kronecker products of the 1D tables,
     tests/test_oracle_pins.py::test_box_cell_matrices_closed_form) instead of quadrature --
     identical in exact arithmetic -- differs from the quadrature oracle by ~kappa eps,
and writes tests/golden/cfg4_conditioning.json (read by tests/test_gpu_parity.py, whose cfg4
tolerance is kappa_max * eps).
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import rm_inputs as ri  # noqa: E402
import oracle.fem as fem  # noqa: E402
from oracle.basis1d import fdm_basis  # noqa: E402
from oracle.solver import Problem  # noqa: E402

EPS = np.finfo(np.float64).eps


def kappa_max(mats):
    seen, km = set(), 0.0
    for A in mats:
        h = hashlib.sha1(np.round(A, 12).tobytes()).hexdigest()
        if h in seen:
            continue
        seen.add(h)
        ev = np.linalg.eigvalsh(A)
        km = max(km, ev[-1] / ev[0])
    return km


def closed_form_parts(k, p, hx, hy, hz):
    """(M, K) of an axis-aligned box by the closed form (Kronecker products)."""
    f = fdm_basis(p)
    h = (hx, hy, hz)
    detJ = hx * hy * hz / 8.0

    def mass(kk):
        blocks = []
        for m, fam in enumerate(fem.FAMILIES[kk]):
            t = [f.B if fm == fem.P_FAM else np.eye(p) for fm in fam]
            s = {0: detJ, 1: detJ * (2.0 / h[m]) ** 2 if kk == 1 else 0, 2: (h[m] / 2.0) ** 2 / detJ if kk == 2 else 0,
                 3: 1.0 / detJ}[kk]
            blocks.append(s * fem.kron3(t[2], t[1], t[0]))
        n = sum(b.shape[0] for b in blocks)
        out = np.zeros((n, n))
        o = 0
        for b in blocks:
            out[o:o + b.shape[0], o:o + b.shape[0]] = b
            o += b.shape[0]
        return out

    Dk = fem.ref_derivative_pattern_or_values(k, p, values=True)
    return mass(k), Dk.T @ mass(k + 1) @ Dk


def main():
    out = {}
    for n, p in [(2, 3), (3, 4), (5, 3), (2, 8)]:
        w = ri.CONFIGS[4].with_mesh(n).with_p(p)
        pb = Problem(w.space, w.p, n, n, n, ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w), w.gamma_d,
                     decomposition="ph")
        A = pb.A
        kf = kappa_max([A[g][:, g].toarray() for g, _ in pb.patch_solvers()])
        D, pcon, sol = pb.potential()
        kp = kappa_max([S.L @ S.L.T for _, S in sol])
        f = ri.uniform_vector(w.cfg, 0, pb.space.ndof); f[pb.constrained] = 0
        u = ri.uniform_vector(w.cfg, 3, pb.space.ndof); u[pb.constrained] = 0
        ref = pb.relax(f, u)
        # the same sweep, cell matrices from the closed form
        fem._cartesian_parts.cache_clear()
        orig = fem._cartesian_parts
        fem._cartesian_parts = closed_form_parts
        try:
            pb2 = Problem(w.space, w.p, n, n, n, ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w), w.gamma_d,
                          decomposition="ph")
            alt = pb2.relax(f, u)
        finally:
            fem._cartesian_parts = orig
        d = float(np.linalg.norm(alt - ref) / np.linalg.norm(ref))
        key = f"{n}^3-p{p}"
        out[key] = {"kappa_face_star_max": kf, "kappa_potential_max": kp, "kappa_max": max(kf, kp),
                    "kappa_eps": max(kf, kp) * EPS, "oracle_vs_closed_form_assembly_sweep_rel": d}
        print(key, out[key], flush=True)
    path = os.path.join(ROOT, "tests", "golden", "cfg4_conditioning.json")
    json.dump({"source": "scripts/cfg4_conditioning.py (oracle only)", "cases": out}, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
