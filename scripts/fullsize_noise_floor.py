"""Oracle noise floor of the full-size sampled H(curl) / H(div) sweep (oracle only).

The sampled sweep of tests/test_gpu_parity.py::test_full_size_hcurl_hdiv_sampled is recomputed
with the Cartesian cell matrices from the box closed form (Kronecker products of the 1D tables,
pinned in tests/test_oracle_pins.py) instead of quadrature -- identical in exact arithmetic.  The
difference is the round-off amplification of the patch solves at full size (kappa grows like the
stiffness / mass ratio ~ (alpha / beta) p^4 / h^2).  Writes tests/golden/fullsize_noise_floor.json.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import rm_inputs as ri  # noqa: E402
import oracle.fem as fem  # noqa: E402
from oracle.fem import Space  # noqa: E402
from oracle.solver import sampled_relax_ph  # noqa: E402
from cfg4_conditioning import closed_form_parts  # noqa: E402


def rows_of(w, sp_):
    off = sp_.offsets()
    rows = []
    for m in range(3):
        Lz, Ly, Lx = sp_.comp_shape(m)
        x, y, z = 12 * w.p + 2, 11 * w.p + 1, 13 * w.p
        rows += [off[m] + ((z + dz) * Ly + y + dy) * Lx + x + dx for dx, dy, dz in ((0, 0, 0), (-2, 1, 0))]
    return rows


def main():
    out = {}
    for cfg in (3, 4):
        w = ri.CONFIGS[cfg]
        sp_ = Space(w.space, w.p, w.nx, w.ny, w.nz)
        n = sp_.ndof
        f = ri.uniform_vector(w.cfg, 0, n)
        u = ri.uniform_vector(w.cfg, 3, n)
        rows = rows_of(w, sp_)
        args = (sp_, ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w), w.gamma_d, f, u, rows, 1.0)
        a = sampled_relax_ph(*args)
        fem._cartesian_parts.cache_clear()
        orig = fem._cartesian_parts
        fem._cartesian_parts = closed_form_parts
        try:
            b = sampled_relax_ph(*args)
        finally:
            fem._cartesian_parts = orig
        d = float(np.abs(a - b).max() / np.abs(a).max())
        out[f"cfg{cfg}"] = {"rows": len(rows), "oracle_vs_closed_form_assembly_maxabs_rel": d}
        print(cfg, out[f"cfg{cfg}"], flush=True)
    json.dump({"source": "scripts/fullsize_noise_floor.py (oracle only)", "cases": out},
              open(os.path.join(ROOT, "tests", "golden", "fullsize_noise_floor.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
