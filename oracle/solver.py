"""Oracle: residual, one additive Schwarz relaxation sweep, PCG (TEST INFRASTRUCTURE ONLY).

  sweep (eq:asm-afw and eq:asm-hiptmair without the p=1 coarse
  term, reading G10):
      r     = f - A u                                      (true A)
      c     = sum_i R_i^T A_i^{-1} R_i r                   (eq:asm-afw / first sum of eq:asm-hiptmair)
      PH:   c += D (sum_j R_j^T B_j^{-1} R_j) D^T r         (eq:asm-hiptmair)
            B = the discretization of a^k(d phi, d psi) = the (k-1)-form operator with
            (alpha', beta') = (beta, 0) (k=1) or (beta, eps_s beta) (k=2, remark P:916-927, G8)
      u_out = u + omega c                                   (reading G9)
  SC-PAFW / SC-PH (eq:sc-asm-afw / eq:sc-asm-hiptmair, eq:schur): c = R_I^T A_II^{-1} R_I r +
      R_G^T S^{-1}_{PAFW|PH} R_G r with patches on interface DoFs only (precondition_sc,
      precondition_sc_ph).
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

from .fem import P_FAM, Space, assemble, assemble_aux, apply_matfree, global_derivative
from .patches import DenseCholeskyPatch, ICCSCPatch, all_patches, icc_masked


class _TriangularPair:
    """Solve with L L^T for a sparse lower triangular L (ICC factor)."""

    def __init__(self, L):
        import scipy.sparse.linalg as spla
        self._spla = spla
        self.L = L.tocsr()
        self.LT = self.L.T.tocsr()

    def solve(self, b):
        y = self._spla.spsolve_triangular(self.L, b, lower=True)
        return self._spla.spsolve_triangular(self.LT, y, lower=False)

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
    decomposition: str = "pafw"      # "pafw" | "ph" | "sc-pafw" (k = 0, eq:sc-asm-afw) | "sc-ph" (k >= 1, eq:sc-asm-hiptmair)
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
        self._sc = None
        self._scph = None

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
        return self.k if self.decomposition in ("ph", "sc-ph") else 0

    def patch_solvers(self):
        if self._patches is not None:
            return self._patches
        dim = self._patch_dim()
        pats = all_patches(self.space, dim, self.constrained, self.interior_only)
        out = []
        # the factorization option applies to the scalar (H(grad)) patch problems: the primary
        # patches for k = 0, the PH potential patches for k = 1; the k-star patches
        # of k = 1, 2 are always factored exactly (their Cholesky has optimal fill)
        if self.factorization == "chol" or self.k >= 1:
            A = self.A
            for ent, g, grp in pats:
                Ai = A[g][:, g].toarray()
                out.append((g, DenseCholeskyPatch(Ai)))
        elif self.factorization == "icc_sc":
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
        assert self.decomposition in ("ph", "sc-ph") and self.k >= 1
        kp = self.k - 1
        D = global_derivative(kp, self.p, self.nx, self.ny, self.nz)
        pspace = Space(kp, self.p, self.nx, self.ny, self.nz)
        pcon = pspace.constrained_mask(self.gamma_d)
        Pf = sp.diags((~pcon).astype(np.float64))
        # B "obtained as the discretization of a^k(d^{k-1} phi, d^{k-1} psi)": since
        # d^k d^{k-1} = 0 this form is (d phi, beta d psi), i.e. the (k-1)-form operator with
        # coefficients (alpha', beta') = (beta, 0), assembled directly by quadrature (+ the k = 2
        # shift eps_s beta M^{k-1}, remark P:916-927, reading G8).  Forming D^T A D instead is equal
        # in exact arithmetic but carries the round-off of D^T (alpha K^k) D ~ eps |K^k|, which grows
        # like (alpha / beta) h^-2 (tests/test_oracle_pins.py pins the equality).
        shift = self.potential_shift if self.k == 2 else 0.0
        B = assemble(pspace, self.X, self.beta, shift * self.beta)
        B = (Pf @ B @ Pf).tocsr()
        self._pot_B = B
        pats = all_patches(pspace, kp, pcon, self.interior_only)
        sol = []
        if self.factorization == "icc_sc" and kp == 0:
            # "On the auxiliary scalar-valued problem posed on the vertex star, we employ the
            # incomplete Cholesky factorization described above": ICC on the
            # static-condensation pattern of the potential vertex-star matrices, with the
            # structural pattern of the H(grad) operator (auxiliary pattern = Cartesian pattern)
            _, Spat = assemble_aux(pspace, self.X, self.beta, shift * self.beta)
            for ent, g, grp in pats:
                sol.append((g, ICCSCPatch(B[g][:, g].tocsr(), Spat[g][:, g].tocsr(), grp == 0)))
        else:
            for ent, g, grp in pats:
                sol.append((g, DenseCholeskyPatch(B[g][:, g].toarray())))
        self._pot = (D.tocsr(), pcon, sol)
        return self._pot

    # ---------------------------------------------------------- statically condensed (SC-PAFW)
    def sc_data(self):
        """SC-PAFW (eq:sc-pafw, eq:schur, eq:sc-asm-afw; k = 0): the operator the patches are
        built from (A on Cartesian cells, the auxiliary P with ICC-SC), its interior set I = the
        cell-interior DoFs (A_II is diagonal for k = 0), and per vertex star the
        interface DoFs with a factor of S_v = A_v,GG - A_v,GI A_v,II^{-1} A_v,IG -- exact dense
        Cholesky, or ICC(0) on S_v's own structural pattern for SC-ICC (reading G19)."""
        if self._sc is not None:
            return self._sc
        assert self.k == 0
        if self.factorization == "icc_sc":
            At, Spat = assemble_aux(self.space, self.X, self.alpha, self.beta)
            Pf = sp.diags(self.free.astype(np.float64))
            At = (Pf @ At @ Pf).tocsr()
        else:
            At, Spat = self.A, None
        n = self.space.ndof
        ids = np.arange(n)
        Lz, Ly, Lx = self.space.comp_shape(0)
        p = self.p
        interior = (ids % Lx % p != 0) & ((ids // Lx) % Ly % p != 0) & (ids // (Lx * Ly) % p != 0)
        I = np.flatnonzero(interior & self.free)
        dI = At.diagonal()[I]
        pats = all_patches(self.space, 0, self.constrained, self.interior_only)
        out = []
        for ent, g, grp in pats:
            gI, gG = g[grp == 0], g[grp != 0]
            if len(gG) == 0:
                continue
            AGG = At[gG][:, gG].toarray()
            AGI = At[gG][:, gI].toarray()
            Sv = AGG - AGI @ (AGI.T / At.diagonal()[gI][:, None])
            if Spat is None:
                out.append((gG, DenseCholeskyPatch(Sv)))
            else:
                pb_ = (Spat != 0).astype(np.int64).tocsr()
                PGG, PGI = pb_[gG][:, gG], pb_[gG][:, gI]
                mask = sp.tril(((PGG + PGI @ PGI.T) != 0).astype(np.int64), format="csr")
                L = icc_masked(sp.csr_matrix(Sv), mask)
                out.append((gG, _TriangularPair(L)))
        self._sc = (At, I, dI, out)
        return self._sc

    def precondition_sc(self, r):
        """c = R_I^T A_II^{-1} R_I r + R_G^T (sum_v R_v^T S_v^{-1} R_v) R_G r (eq:schur, eq:sc-asm-afw
        without the coarse term), R_G = [-A_GI A_II^{-1}, I]."""
        At, I, dI, pats = self.sc_data()
        r = np.where(self.free, r, 0.0)
        yI = r[I] / dI
        rG = r.copy()
        rG[I] = 0.0
        rG -= At[:, I] @ yI
        rG[I] = 0.0
        cG = np.zeros_like(r)
        for gG, S in pats:
            cG[gG] += S.solve(rG[gG])
        c = cG.copy()
        c[I] = (r[I] - (At[I] @ cG)) / dI
        return np.where(self.free, c, 0.0)

    # ------------------------------------------------------------ statically condensed (SC-PH)
    def sc_ph_data(self):
        """SC-PH (eq:sc-ph, eq:schur, eq:sc-asm-hiptmair; k = 1, 2, exact factors): the interior set I
        (cell-interior DoFs) and interface G of V^k with A_II^{-1} (block diagonal, blocks
        <= 3x3, remark P:1061-1066) and S = A_GG - A_GI A_II^{-1} A_IG (eq:LDU); per k-star the
        interface DoFs and a Cholesky factor of S_i = R~_i S R~_i^T; D~ = D_GG, the derivative
        tabulated between the interface DoFs of V^{k-1} and V^k; and per (k-1)-star a factor of
        B~_j = R~_j S_B R~_j^T, S_B the interface Schur complement of the potential matrix B (the
        discretization of a^k(d phi, d psi) = PH's B)."""
        if self._scph is not None:
            return self._scph
        import scipy.sparse.linalg as spla
        assert self.k >= 1 and self.factorization == "chol", "SC-PH: k = 1, 2 with exact factors"
        A = self.A
        I = np.flatnonzero(self.free & interior_mask(self.space))
        G = np.flatnonzero(self.free & ~interior_mask(self.space))
        AIIinv = spla.inv(A[I][:, I].tocsc()).tocsr()
        S = (A[G][:, G] - A[G][:, I] @ AIIinv @ A[I][:, G]).tocsr()
        gpos = np.full(self.space.ndof, -1)
        gpos[G] = np.arange(len(G))
        prim = []
        for ent, g, grp in all_patches(self.space, self.k, self.constrained, self.interior_only):
            loc = gpos[g[grp != 0]]
            if len(loc):
                prim.append((loc, DenseCholeskyPatch(S[loc][:, loc].toarray())))
        D, pcon, _ = self.potential()
        B = self._pot_B
        pspace = Space(self.k - 1, self.p, self.nx, self.ny, self.nz)
        Ib = np.flatnonzero(~pcon & interior_mask(pspace))
        Gb = np.flatnonzero(~pcon & ~interior_mask(pspace))
        BIIinv = spla.inv(B[Ib][:, Ib].tocsc()).tocsr()
        SB = (B[Gb][:, Gb] - B[Gb][:, Ib] @ BIIinv @ B[Ib][:, Gb]).tocsr()
        bpos = np.full(pspace.ndof, -1)
        bpos[Gb] = np.arange(len(Gb))
        pot = []
        for ent, g, grp in all_patches(pspace, self.k - 1, pcon, self.interior_only):
            loc = bpos[g[grp != 0]]
            if len(loc):
                pot.append((loc, DenseCholeskyPatch(SB[loc][:, loc].toarray())))
        Dt = D[G][:, Gb].tocsr()
        self._scph = (A, I, G, AIIinv, S, prim, Dt, pot)
        return self._scph

    def precondition_sc_ph(self, r, potential_stage=True):
        """c = R_I^T A_II^{-1} R_I r + R_G^T S_PH^{-1} R_G r (eq:schur, eq:sc-asm-hiptmair without the
        coarse term), S_PH^{-1} = sum_i R~_i^T S_i^{-1} R~_i + D~ (sum_j R~_j^T B~_j^{-1} R~_j) D~^T,
        R_G = [-A_GI A_II^{-1}, I]."""
        A, I, G, AIIinv, S, prim, Dt, pot = self.sc_ph_data()
        r = np.where(self.free, r, 0.0)
        yI = AIIinv @ r[I]
        rG = r[G] - A[G][:, I] @ yI
        cG = np.zeros(len(G))
        for loc, P_ in prim:
            cG[loc] += P_.solve(rG[loc])
        if potential_stage:
            t = Dt.T @ rG
            s_ = np.zeros(Dt.shape[1])
            for loc, P_ in pot:
                s_[loc] += P_.solve(t[loc])
            cG += Dt @ s_
        c = np.zeros_like(r)
        c[G] = cG
        c[I] = yI - AIIinv @ (A[I][:, G] @ cG)
        return np.where(self.free, c, 0.0)

    # ---------------------------------------------------------------- sweep
    def precondition(self, r):
        """c = P^{-1} r (the additive Schwarz sum), r zero on constrained DoFs."""
        if self.decomposition == "sc-pafw":
            return self.precondition_sc(r)
        if self.decomposition == "sc-ph":
            return self.precondition_sc_ph(r)
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


def interior_mask(space: Space) -> np.ndarray:
    """Cell-interior DoFs of a space (I = E^d): every P-family index off the cell
    boundaries (index % p != 0); DP-family indices are interior to their cell."""
    p = space.p
    out = np.zeros(space.ndof, dtype=bool)
    off = space.offsets()
    for m, fam in enumerate(space.fams):
        Lz, Ly, Lx = space.comp_shape(m)
        iz, iy, ix = np.meshgrid(np.arange(Lz), np.arange(Ly), np.arange(Lx), indexing="ij")
        ok = np.ones((Lz, Ly, Lx), dtype=bool)
        for idx, f in zip((ix, iy, iz), fam):
            if f == P_FAM:
                ok &= idx % p != 0
        out[off[m]:off[m + 1]] = ok.ravel()
    return out


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


def sampled_relax_ph(space: Space, X, alpha, beta, gamma_d, f, u, rows, omega=1.0, potential_shift=EPS_S):
    """u_out[rows] of one PH exact-Cholesky sweep (k = 1, 2; eq:asm-hiptmair without the coarse
    term) computed only from the patches that reach those rows, each assembled from its own cells
    (no global matrix; full-size sampled parity):
        u_out[g] = u[g] + omega ( sum_{i contains g} (A_i^{-1} R_i r)[g] + sum_h D[g, h] s[h] ),
        s[h] = sum_{j contains h} (B_j^{-1} R_j D^T r)[h],   r = f - A u,
    with B_j the potential patch matrix, assembled as the (k-1)-form operator with coefficients
    (beta, 0) (k = 1) or (beta, eps_s beta) (k = 2) -- equal to R_j D^T A D R_j^T (+ eps_s beta M)
    (pinned in tests/test_oracle_pins.py::test_potential_operator_is_the_lower_form_operator)."""
    from .fem import cell_rows_apply, derivative_entries, dof_coords, local_matrix
    from .patches import entities, patch_dofs
    k, p = space.k, space.p
    n = (space.nx, space.ny, space.nz)
    con = space.constrained_mask(gamma_d)
    u = np.where(con, 0.0, u)
    f = np.where(con, 0.0, f)
    pspace = Space(k - 1, p, *n)
    pcon = pspace.constrained_mask(gamma_d)
    beta_p = potential_shift * beta if k == 2 else np.zeros_like(beta)
    rcache = {}

    def resid(gs):
        need = [int(g) for g in gs if int(g) not in rcache and not con[int(g)]]
        if need:
            Au = cell_rows_apply(space, X, alpha, beta, u, need)
            for g, v in zip(need, Au):
                rcache[g] = f[g] - v
        return np.array([0.0 if con[int(g)] else rcache[int(g)] for g in gs])

    def near_entities(sp_, dim, g):
        _, ix, iy, iz = dof_coords(sp_, int(g))
        cand = []
        for ent in _entities_near(sp_, dim, (ix, iy, iz)):
            cand.append(ent)
        return cand

    pcache, scache = {}, {}

    def prim_correction(g):
        tot = 0.0
        for ent in near_entities(space, k, g):
            if ent not in pcache:
                pcache[ent] = [patch_dofs(space, ent, con)[0], None]
            gp, z = pcache[ent]
            w = np.flatnonzero(gp == g)
            if not len(w):
                continue
            if z is None:
                Ai = local_matrix(space, X, alpha, beta, gp)
                z = pcache[ent][1] = DenseCholeskyPatch(Ai).solve(resid(gp))
            tot += z[w[0]]
        return tot

    def s_value(h):
        tot = 0.0
        for ent in near_entities(pspace, k - 1, h):
            if ent not in scache:
                scache[ent] = [patch_dofs(pspace, ent, pcon)[0], None]
            gp, z = scache[ent]
            w = np.flatnonzero(gp == h)
            if not len(w):
                continue
            if z is None:
                # t = (D^T r) on the patch: column entries of D
                cols = [derivative_entries(k - 1, p, *n, int(hh), by="col") for hh in gp]
                need = sorted({g2 for ce in cols for g2 in ce})
                rmap = dict(zip(need, resid(need)))
                t = np.array([sum(v * rmap[g2] for g2, v in ce.items()) for ce in cols])
                Bj = local_matrix(pspace, X, beta, beta_p, gp)
                z = scache[ent][1] = DenseCholeskyPatch(Bj).solve(t)
            tot += z[w[0]]
        return tot

    out = u[np.asarray(rows)].copy()
    for t_, g in enumerate(rows):
        g = int(g)
        if con[g]:
            continue
        c = prim_correction(g)
        for h, dv in derivative_entries(k - 1, p, *n, g, by="row").items():
            if not pcon[h]:
                c += dv * s_value(h)
        out[t_] += omega * c
    return out


def _entities_near(sp_, dim, idx):
    """Entities of dimension dim whose star can contain a DoF at structured indices idx: node or
    cell coordinates within one cell of the DoF in every direction."""
    from .patches import entities
    p = sp_.p
    n = (sp_.nx, sp_.ny, sp_.nz)
    lo = [max(0, i // p - 1) for i in idx]
    hi = [min(n[d], idx[d] // p + 1) for d, i in enumerate(idx)]
    out = []
    for ent in _entities_cached(sp_, dim):
        if all(lo[d] <= ent[d][1] <= hi[d] for d in range(3)):
            out.append(ent)
    return out


_ENT_CACHE = {}


def _entities_cached(sp_, dim):
    from .patches import entities
    key = (sp_, dim)
    if key not in _ENT_CACHE:
        _ENT_CACHE[key] = entities(sp_, dim)
    return _ENT_CACHE[key]
