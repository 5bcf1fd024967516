"""Oracle: star patches and patch solves (TEST INFRASTRUCTURE ONLY).

  * star of an entity and V_h|_{star j} = {v : support(v) in star j}, realised on
    the structured layout by per-direction windows:
        P family,  vertex-type direction at node v : v p-(p-1) .. v p+(p-1)
        DP family, vertex-type direction at node v : v p-p     .. v p+p-1
        P family,  cell-type direction (cell c)     : c p+1     .. c p+p-1
        DP family, cell-type direction (cell c)     : c p       .. c p+p-1
    clipped to the mesh; constrained DoFs removed; empty patches dropped (reading G5).
  * patch matrices A_i = R_i A R_i^T as dense submatrices.
  * patch DoF order (reading G6): group (interior, face, edge, vertex = number of P-family
    indices that are multiples of p), then component, then global (z, y, x) lexicographic.
  * exact Cholesky by dense LAPACK Cholesky.
  * ICC on the static-condensation pattern: the masked definition
        L_jj = sqrt(a_jj - sum_{k<j} L_jk^2),
        L_ij = (a_ij - sum_{k<j} L_ik L_jk) / L_jj   if (i,j) in pattern, else 0,
    pattern = tril(pattern(P_v)) U tril(pattern(P_GI P_IG)) taken structurally, with the
    breakdown restart of reading G7 (shift sigma diag, sigma0 = 1e-10 max diag, doubling).

Pins: tests/test_oracle_patches.py (star sizes, dense vs masked-ICC with a full pattern,
interior-only 2x2x2 single patch = exact solve, face-star zero fill).
"""
from __future__ import annotations

from dataclasses import dataclass
import math

import numpy as np
import scipy.linalg
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .fem import FAMILIES, P_FAM, Space


def entities(space: Space, dim: int):
    """Entities of dimension dim as per-direction specs (("node", v) | ("cell", c)) x 3."""
    n = (space.nx, space.ny, space.nz)
    out = []
    if dim == 0:
        for vz in range(n[2] + 1):
            for vy in range(n[1] + 1):
                for vx in range(n[0] + 1):
                    out.append((("node", vx), ("node", vy), ("node", vz)))
    elif dim == 1:        # edges along direction e
        for e in range(3):
            rng = [range(n[d] + 1) if d != e else range(n[d]) for d in range(3)]
            for iz in rng[2]:
                for iy in rng[1]:
                    for ix in rng[0]:
                        idx = (ix, iy, iz)
                        out.append(tuple(("cell", idx[d]) if d == e else ("node", idx[d]) for d in range(3)))
    elif dim == 2:        # faces normal to direction f
        for f in range(3):
            rng = [range(n[d] + 1) if d == f else range(n[d]) for d in range(3)]
            for iz in rng[2]:
                for iy in rng[1]:
                    for ix in rng[0]:
                        idx = (ix, iy, iz)
                        out.append(tuple(("node", idx[d]) if d == f else ("cell", idx[d]) for d in range(3)))
    else:
        raise ValueError(dim)
    return out


def window(spec, fam, p, ncell):
    kind, v = spec
    if fam == P_FAM:
        lo, hi = (v * p - (p - 1), v * p + (p - 1)) if kind == "node" else (v * p + 1, v * p + p - 1)
        lo, hi = max(lo, 0), min(hi, ncell * p)
    else:
        lo, hi = (v * p - p, v * p + p - 1) if kind == "node" else (v * p, v * p + p - 1)
        lo, hi = max(lo, 0), min(hi, ncell * p - 1)
    return np.arange(lo, hi + 1)


def patch_dofs(space: Space, ent, constrained: np.ndarray):
    """Free global DoFs of V_h|_{star ent}, in the pinned order (reading G6)."""
    n = (space.nx, space.ny, space.nz)
    off = space.offsets()
    p = space.p
    keys, idxs = [], []
    for m, fam in enumerate(space.fams):
        Lz, Ly, Lx = space.comp_shape(m)
        w = [window(ent[d], fam[d], p, n[d]) for d in range(3)]
        Z, Y, X = np.meshgrid(w[2], w[1], w[0], indexing="ij")
        g = off[m] + (Z * Ly + Y) * Lx + X
        grp = np.zeros(Z.shape, dtype=np.int64)
        for d, A in enumerate((X, Y, Z)):
            if fam[d] == P_FAM:
                grp += (A % p == 0)
        g, grp, Z, Y, X = (a.ravel() for a in (g, grp, Z, Y, X))
        keep = ~constrained[g]
        idxs.append(g[keep])
        keys.append(np.stack([grp[keep], np.full(keep.sum(), m), Z[keep], Y[keep], X[keep]], axis=1))
    g = np.concatenate(idxs)
    key = np.concatenate(keys)
    order = np.lexsort(key.T[::-1])
    return g[order], key[order, 0]


def all_patches(space: Space, dim: int, constrained, interior_only=False):
    out = []
    n = (space.nx, space.ny, space.nz)
    for ent in entities(space, dim):
        if interior_only:
            bad = any(s[0] == "node" and (s[1] == 0 or s[1] == n[d]) for d, s in enumerate(ent))
            if bad:
                continue
        g, grp = patch_dofs(space, ent, constrained)
        if len(g):
            out.append((ent, g, grp))
    return out


# ------------------------------------------------------------------------------ factors
class DenseCholeskyPatch:
    """Exact patch solve A_i^{-1} by dense Cholesky."""

    def __init__(self, A_i: np.ndarray):
        self.L = np.linalg.cholesky(A_i)

    def solve(self, b):
        y = scipy.linalg.solve_triangular(self.L, b, lower=True)
        return scipy.linalg.solve_triangular(self.L.T, y, lower=False)


def icc_masked(a: sp.csr_matrix, pattern: sp.csr_matrix):
    """Row-by-row (up-looking) masked incomplete Cholesky with the definition in the module
    header.  a: symmetric CSR, pattern: boolean CSR containing the lower-triangular mask
    (diagonal included).  Returns L (CSR, lower) or raises FloatingPointError at breakdown."""
    n = a.shape[0]
    a = a.tocsr()
    pat = pattern.tocsr()
    rows = []                          # rows[i] = dict j -> L_ij (j <= i)
    diag = np.zeros(n)
    for i in range(n):
        cols = pat.indices[pat.indptr[i]:pat.indptr[i + 1]]
        cols = np.sort(cols[cols <= i])
        arow = dict(zip(a.indices[a.indptr[i]:a.indptr[i + 1]], a.data[a.indptr[i]:a.indptr[i + 1]]))
        Li = {}
        for j in cols:
            if j == i:
                s = arow.get(i, 0.0) - sum(v * v for v in Li.values())
                if not s > 0.0:
                    raise FloatingPointError(f"non-positive pivot at row {i}")
                Li[i] = math.sqrt(s)
            else:
                Lj = rows[j]
                s = arow.get(j, 0.0)
                # sum over k < j of L_ik L_jk
                if len(Li) < len(Lj):
                    s -= sum(v * Lj[k] for k, v in Li.items() if k in Lj and k < j)
                else:
                    s -= sum(v * Li[k] for k, v in Lj.items() if k in Li and k < j)
                Li[j] = s / Lj[j]
        rows.append(Li)
        diag[i] = Li[i]
    r, c, v = [], [], []
    for i, Li in enumerate(rows):
        for j, val in Li.items():
            r.append(i); c.append(j); v.append(val)
    return sp.csr_matrix((v, (r, c)), shape=(n, n))


class ICCSCPatch:
    """ICC on the static-condensation pattern with the reading-G7 restart."""

    def __init__(self, A_i: sp.csr_matrix, pat_i: sp.csr_matrix, interior: np.ndarray):
        I = np.flatnonzero(interior)
        G = np.flatnonzero(~interior)
        patb = (pat_i != 0).astype(np.int64).tocsr()
        PGI = patb[G][:, I]
        fill = (PGI @ PGI.T).tocoo()
        extra = sp.csr_matrix((np.ones(fill.nnz), (G[fill.row], G[fill.col])), shape=A_i.shape)
        mask = sp.tril(((patb + extra) != 0).astype(np.int64), format="csr")
        self.mask = mask
        self.sigma = 0.0
        A = A_i.tocsr()
        while True:
            try:
                self.L = icc_masked(A if self.sigma == 0.0 else A + self.sigma * sp.diags(A_i.diagonal()), mask)
                break
            except FloatingPointError:
                if self.sigma == 0.0:
                    self.sigma = 1e-10
                else:
                    self.sigma *= 2.0
                if self.sigma > 1e-2:
                    raise
        self.LT = self.L.T.tocsr()

    def solve(self, b):
        y = spla.spsolve_triangular(self.L, b, lower=True)
        return spla.spsolve_triangular(self.LT, y, lower=False)
