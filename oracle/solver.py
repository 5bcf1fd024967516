"""Oracle: residual, one additive Schwarz relaxation sweep, PCG (TEST INFRASTRUCTURE ONLY).

  sweep (eq:asm-afw and eq:asm-hiptmair without the p=1 coarse
  term, reading G10):
      r     = f - A u                                      (true A)
      c     = sum_i R_i^T A_i^{-1} R_i r                   (eq:asm-afw / first sum of eq:asm-hiptmair)
      PH:   c += D (sum_j R_j^T B_j^{-1} R_j) D^T r         (eq:asm-hiptmair)
            B = D^T A D (k=1), B = D^T A D + eps_s beta M^{k-1} (k=2, remark P:916-927, reading G8)
      u_out = u + omega c                                   (reading G9)
  For the auxiliary-operator variant the patch matrices come from P instead of A.
  With `coarse`, PCG's preconditioner is the hybrid V(1,1) cycle with the p = 1 coarse level
  (oracle/coarse.py, reading G20).
  PCG: zero initial guess, stop at the first k with
      sqrt(r_k^T z_k) <= rtol sqrt(r_0^T z_0)  (natural P^{-1} norm), iters = k (reading G15).

Constrained DoFs (Dirichlet) are held at zero: all operators act on the free DoFs.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import math

import numpy as np
import scipy.sparse as sp

from .fem import Space, assemble, assemble_aux, apply_matfree, global_derivative
from .patches import DenseCholeskyPatch, ICCSCPatch, all_patches

EPS_S = 1e-3   # reading G8: eps_s = 1e-3 of the potential-space mass


@dataclass
class Problem:
    k: int
    p: int
    nx: int
    ny: int
    nz: int
    X: np.ndarray            # vertex coordinates (nz+1, ny+1, nx+1, 3)
    alpha: np.ndarray        # (nz, ny, nx)
    beta: np.ndarray
    gamma_d: int
    decomposition: str = "pafw"      # "pafw" | "ph"
    factorization: str = "chol"      # "chol" | "icc_sc"
    interior_only: bool = False
    matfree: bool = False            # apply A cell by cell (large p) instead of via CSR
    potential_shift: float = EPS_S   # eps_s of reading G8 (k = 2 PH)
    coarse: bool = False             # p = 1 coarse level + hybrid V(1,1) in pcg / cycle (oracle.coarse)
    space: Space = field(init=False)
    constrained: np.ndarray = field(init=False)
    free: np.ndarray = field(init=False)

    def __post_init__(self):
        self.space = Space(self.k, self.p, self.nx, self.ny, self.nz)
        self.constrained = self.space.constrained_mask(self.gamma_d)
        self.free = ~self.constrained
        self._A = None
        self._patches = None
        self._pot = None
        self._coarse = None

    # ---------------------------------------------------------------- operator
    @property
    def A(self) -> sp.csr_matrix:
        """Global A with constrained rows/columns zeroed (constrained DoFs held at 0)."""
        if self._A is None:
            A = assemble(self.space, self.X, self.alpha, self.beta)
            Pf = sp.diags(self.free.astype(np.float64))
            self._A = (Pf @ A @ Pf).tocsr()
        return self._A

    def apply(self, u):
        """v = A u on free DoFs, zero on constrained rows."""
        u = np.where(self.free, u, 0.0)
        if self.matfree:
            v = apply_matfree(self.space, self.X, self.alpha, self.beta, u)
        else:
            v = self.A @ u
        return np.where(self.free, v, 0.0)

    def residual(self, f, u):
        return np.where(self.free, f - self.apply(u), 0.0)

    # ---------------------------------------------------------------- patches
    def _patch_dim(self):
        return 0 if self.decomposition == "pafw" else self.k

    def patch_solvers(self):
        if self._patches is not None:
            return self._patches
        dim = self._patch_dim()
        pats = all_patches(self.space, dim, self.constrained, self.interior_only)
        out = []
        if self.factorization == "chol":
            A = self.A
            for ent, g, grp in pats:
                Ai = A[g][:, g].toarray()
                out.append((g, DenseCholeskyPatch(Ai)))
        elif self.factorization == "icc_sc":
            assert self.k == 0
            Paux, Spat = assemble_aux(self.space, self.X, self.alpha, self.beta)
            for ent, g, grp in pats:
                Ai = Paux[g][:, g].tocsr()
                pat = Spat[g][:, g].tocsr()
                out.append((g, ICCSCPatch(Ai, pat, grp == 0)))
        else:
            raise ValueError(self.factorization)
        self._patches = out
        return out

    def potential(self):
        """PH potential stage data: D (primal <- potential), the potential problem and its
        patch solvers on the stars of (k-1)-entities."""
        if self._pot is not None:
            return self._pot
        assert self.decomposition == "ph" and self.k >= 1
        kp = self.k - 1
        D = global_derivative(kp, self.p, self.nx, self.ny, self.nz)
        pspace = Space(kp, self.p, self.nx, self.ny, self.nz)
        pcon = pspace.constrained_mask(self.gamma_d)
        Pf = sp.diags((~pcon).astype(np.float64))
        Af = assemble(self.space, self.X, self.alpha, self.beta)     # unconstrained A^k
        B = D.T @ Af @ D
        if self.k == 2:
            M = assemble(pspace, self.X, np.zeros_like(self.alpha), self.beta)
            B = B + self.potential_shift * M
        B = (Pf @ B @ Pf).tocsr()
        pats = all_patches(pspace, kp, pcon, self.interior_only)
        sol = []
        for ent, g, grp in pats:
            sol.append((g, DenseCholeskyPatch(B[g][:, g].toarray())))
        self._pot = (D.tocsr(), pcon, sol)
        return self._pot

    # ---------------------------------------------------------------- sweep
    def precondition(self, r):
        """c = P^{-1} r (the additive Schwarz sum), r zero on constrained DoFs."""
        c = np.zeros_like(r)
        for g, S in self.patch_solvers():
            c[g] += S.solve(r[g])
        if self.decomposition == "ph" and self.k >= 1:
            D, pcon, sol = self.potential()
            t = D.T @ r
            s = np.zeros(D.shape[1])
            for g, S in sol:
                s[g] += S.solve(t[g])
            c += D @ s
        return np.where(self.free, c, 0.0)

    def cycle(self, r):
        """The PCG preconditioner: the one-level additive sweep, or with `coarse` the hybrid
        V(1,1) cycle of oracle.coarse."""
        if not self.coarse:
            return self.precondition(r)
        from .coarse import CoarseLevel, smoother_colours, vcycle
        if self._coarse is None:
            self._coarse = CoarseLevel(self)
        return vcycle(self, self._coarse, r, 1.0 / smoother_colours(self.k, self.decomposition))

    def relax(self, f, u, omega=1.0):
        r = self.residual(f, u)
        return u + omega * self.precondition(r)

    def pcg(self, f, rtol=1e-8, maxit=500):
        f = np.where(self.free, f, 0.0)
        x = np.zeros_like(f)
        r = f.copy()
        z = self.cycle(r)
        rz = float(r @ z)
        rz0 = rz
        if rz0 == 0.0:
            return x, 0, 0.0
        pdir = z.copy()
        for it in range(1, maxit + 1):
            q = self.apply(pdir)
            a = rz / float(pdir @ q)
            x += a * pdir
            r -= a * q
            z = self.cycle(r)
            rz_new = float(r @ z)
            rel = math.sqrt(max(rz_new, 0.0) / rz0)
            if rel <= rtol:
                return x, it, rel
            pdir = z + (rz_new / rz) * pdir
            rz = rz_new
        return x, maxit, rel


def sampled_relax(space: Space, X, alpha, beta, gamma_d, f, u, rows, omega=1.0):
    """u_out[rows] of one PAFW exact-Cholesky sweep (k = 0), computed only from the star
    patches that contain those rows, each assembled from its own cells (no global matrix):
    for every patch i containing row g:  u_out[g] += omega * (A_i^{-1} R_i (f - A u))[g].
    Used for full-size sampled parity (the same definitions as Problem.relax)."""
    from .fem import cell_rows_apply, dof_coords, local_matrix
    from .patches import patch_dofs
    constrained = space.constrained_mask(gamma_d)
    u = np.where(constrained, 0.0, u)
    f = np.where(constrained, 0.0, f)
    n = (space.nx, space.ny, space.nz)
    out = u[np.asarray(rows)].copy()
    cache = {}
    for t, g in enumerate(rows):
        if constrained[g]:
            continue
        _, ix, iy, iz = dof_coords(space, int(g))
        cand = [[v for v in (i // space.p - 1, i // space.p, i // space.p + 1) if 0 <= v <= n[d]]
                for d, i in enumerate((ix, iy, iz))]
        for vz in cand[2]:
            for vy in cand[1]:
                for vx in cand[0]:
                    ent = (("node", vx), ("node", vy), ("node", vz))
                    if ent not in cache:
                        gp, _ = patch_dofs(space, ent, constrained)
                        cache[ent] = gp
                    gp = cache[ent]
                    where = np.flatnonzero(gp == g)
                    if not len(where):
                        continue
                    key = ("x",) + ent
                    if key not in cache:
                        r = f[gp] - cell_rows_apply(space, X, alpha, beta, u, gp)
                        Ai = local_matrix(space, X, alpha, beta, gp)
                        cache[key] = DenseCholeskyPatch(Ai).solve(r)
                    out[t] += omega * cache[key][where[0]]
    return out
