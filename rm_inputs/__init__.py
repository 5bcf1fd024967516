"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no basis, no operator, no layout
rule): it only names the BASELINE.json workloads and draws random numbers of a given
shape with a fixed recipe, so the CPU oracle (`oracle/`) and the CUDA path
(`paper_2211_14284_b200/`) can be fed identical inputs without sharing code.

Recipe (DESIGN.md §"Inputs"):
  * generator: numpy PCG64, seed = 1000*cfg + s, one independent stream per s:
      s=0 right-hand side f, s=1 coefficient alpha, s=2 vertex perturbation, s=3 u_in.
  * vectors: U[-1, 1) i.i.d., one value per DoF of the whole layout (constrained
    entries included); the caller zeroes constrained entries with its own mask.
  * alpha (cfg2): 10**U[-2, 2) per cell, C-order [z][y][x]  (BASELINE.json configs[1]).
  * perturbation (cfg5): U[-0.1h, 0.1h) per coordinate, drawn for every vertex of the
    global (nz+1)(ny+1)(nx+1) grid in C-order [z][y][x][xyz], applied to interior
    vertices only (BASELINE.json configs[4]).
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

# space codes follow the paper's form degree k: 0 H(grad), 1 H(curl), 2 H(div)
HGRAD, HCURL, HDIV = 0, 1, 2
# Gamma_D bitmask: bit0 x=0, bit1 x=1, bit2 y=0, bit3 y=1, bit4 z=0, bit5 z=1
GAMMA_ALL = 0x3F
GAMMA_X0 = 0x01


@dataclass(frozen=True)
class Workload:
    cfg: int             # 1..5, BASELINE.json configs[cfg-1]
    space: int           # k
    p: int
    nx: int
    ny: int
    nz: int
    alpha: str           # "one" | "logu22" (10**U[-2,2) per cell)
    beta: float
    gamma_d: int
    perturb: float       # relative amplitude (fraction of h) of the interior-vertex jitter; 0 = Cartesian
    decomposition: str   # "pafw" (vertex stars) | "ph" (k-stars + potential)
    factorization: str   # "chol" | "icc_sc"
    alpha_value: float = 1.0

    def with_mesh(self, nx: int, ny: int | None = None, nz: int | None = None) -> "Workload":
        ny = nx if ny is None else ny
        nz = nx if nz is None else nz
        return replace(self, nx=nx, ny=ny, nz=nz)

    def with_p(self, p: int) -> "Workload":
        return replace(self, p=p)

    @property
    def ncells(self) -> int:
        return self.nx * self.ny * self.nz


# BASELINE.json "configs", in order.
CONFIGS = {
    1: Workload(1, HGRAD, 3, 4, 4, 4, "one", 1.0, GAMMA_ALL, 0.0, "pafw", "chol"),
    2: Workload(2, HGRAD, 7, 32, 32, 32, "logu22", 1.0, GAMMA_X0, 0.0, "pafw", "chol"),
    3: Workload(3, HCURL, 6, 24, 24, 24, "one", 1.0, GAMMA_ALL, 0.0, "ph", "chol"),
    4: Workload(4, HDIV, 8, 24, 24, 24, "one", 1e-2, GAMMA_ALL, 0.0, "ph", "chol"),
    5: Workload(5, HGRAD, 15, 16, 16, 16, "one", 1.0, GAMMA_ALL, 0.1, "pafw", "icc_sc"),
}


def rng(cfg: int, s: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(1000 * cfg + s))


def uniform_vector(cfg: int, s: int, n: int) -> np.ndarray:
    """n values U[-1,1) from stream s (0 = RHS f, 3 = u_in)."""
    return rng(cfg, s).uniform(-1.0, 1.0, size=n)


def cell_alpha(w: Workload) -> np.ndarray:
    """Per-cell alpha, C-order [z][y][x], shape (nz, ny, nx)."""
    if w.alpha == "one":
        return np.full((w.nz, w.ny, w.nx), w.alpha_value)
    if w.alpha == "logu22":
        e = rng(w.cfg, 1).uniform(-2.0, 2.0, size=(w.nz, w.ny, w.nx))
        return 10.0 ** e
    raise ValueError(w.alpha)


def cell_beta(w: Workload) -> np.ndarray:
    return np.full((w.nz, w.ny, w.nx), w.beta)


def vertex_coords(w: Workload) -> np.ndarray:
    """Vertex coordinates of the unit cube grid, shape (nz+1, ny+1, nx+1, 3), [x,y,z] last.

    Cell widths h_d = 1/n_d.  With w.perturb > 0 every interior vertex moves by
    U[-perturb*h_d, perturb*h_d) per coordinate d (boundary vertices never move).
    """
    z, y, x = np.meshgrid(np.linspace(0.0, 1.0, w.nz + 1), np.linspace(0.0, 1.0, w.ny + 1),
                          np.linspace(0.0, 1.0, w.nx + 1), indexing="ij")
    X = np.stack([x, y, z], axis=-1)
    if w.perturb > 0.0:
        h = np.array([1.0 / w.nx, 1.0 / w.ny, 1.0 / w.nz])
        d = rng(w.cfg, 2).uniform(-1.0, 1.0, size=X.shape) * (w.perturb * h)
        interior = np.zeros(X.shape[:3], dtype=bool)
        interior[1:-1, 1:-1, 1:-1] = True
        X = X + d * interior[..., None]
    return X
