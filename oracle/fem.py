"""Oracle: de Rham spaces on structured hexahedral meshes (TEST INFRASTRUCTURE ONLY).

Follows PAPER.md step by step:
  * tensor-product bases psi, Psi^(m), Phi^(m), phi                (eq:hgrad-basis..eq:ltwo-basis)
  * pullbacks F^k (identity, J^{-T}, J/detJ, 1/detJ) and d F^k = F^{k+1} d-hat
  * cell matrices [A_K]_ij = a^k(F^k psi_i, F^k psi_j)              (eq:common_weak_formulation)
    evaluated by GLL quadrature with ceil(3(p+1)/2) points per direction (reading G1)
  * global assembly with reference values as DoFs in the structured layout of
    SURVEY.md App. A (reading G16): per component, C-order [Z][Y][X] with X fastest; per
    direction a P family (n p + 1 entries, shared at multiples of p) or a DP family (n p).
  * Dirichlet: a DoF is constrained iff one of its P-family indices lies on a Gamma_D plane.
  * the auxiliary operator P_K = G^T diag(M-bar_beta) G + D-bar^T diag(M-bar_alpha) D-bar
    (eq:sum-factorization_approx) for k = 0.
  * the tabulated exterior derivative D as a global sparse matrix.

Curl sign (reading G17): the standard curl is used; eq:curlbasis as printed is its negative.
Every output of the method (A, C^T M C, D B^{-1} D^T) is invariant under curl -> -curl.

Pins: tests/test_oracle_fem.py (31/8 single cell, Q1 2x2x2 value 4/3 a + b/27, constants,
u = x_1 patch test on perturbed cells, complex property, interior nnz bounds, P = A on
Cartesian cells, the auxiliary operator of a sheared AFFINE cell = the true operator of the
equivalent box, and on NON-AFFINE cells its definition eq:sum-factorization_approx evaluated with
the true quadrature mass matrices: diag(G-bar^-T M G-bar^-1)).
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache
import math

import numpy as np
import scipy.sparse as sp

from .basis1d import fdm_basis, gll_rule, pattern_B, pattern_D

P_FAM, D_FAM = "P", "D"
FAMILIES = {
    0: [(P_FAM, P_FAM, P_FAM)],
    1: [(D_FAM, P_FAM, P_FAM), (P_FAM, D_FAM, P_FAM), (P_FAM, P_FAM, D_FAM)],
    2: [(P_FAM, D_FAM, D_FAM), (D_FAM, P_FAM, D_FAM), (D_FAM, D_FAM, P_FAM)],
    3: [(D_FAM, D_FAM, D_FAM)],
}


def nq_for(p: int) -> int:
    """Reading G1: ceil(3(p+1)/2) GLL points per direction."""
    return (3 * (p + 1) + 1) // 2


# ------------------------------------------------------------------------------ layout
@dataclass(frozen=True)
class Space:
    k: int
    p: int
    nx: int
    ny: int
    nz: int

    @property
    def fams(self):
        return FAMILIES[self.k]

    def length(self, fam, d):
        n = (self.nx, self.ny, self.nz)[d]
        return n * self.p + 1 if fam == P_FAM else n * self.p

    def comp_shape(self, m):
        fx, fy, fz = self.fams[m]
        return (self.length(fz, 2), self.length(fy, 1), self.length(fx, 0))

    def comp_size(self, m):
        return int(np.prod(self.comp_shape(m)))

    def offsets(self):
        o = [0]
        for m in range(len(self.fams)):
            o.append(o[-1] + self.comp_size(m))
        return o

    @property
    def ndof(self):
        return self.offsets()[-1]

    def local_sizes(self, m):
        p = self.p
        return tuple(p + 1 if f == P_FAM else p for f in self.fams[m])  # (x, y, z)

    @property
    def nloc(self):
        return sum(int(np.prod(self.local_sizes(m))) for m in range(len(self.fams)))

    def cell_dofs(self, cx, cy, cz):
        """Global indices of the cell's DoFs in the local element order
        (component-major, then z, y, x with x fastest)."""
        out = []
        off = self.offsets()
        p = self.p
        for m in range(len(self.fams)):
            sx, sy, sz = self.local_sizes(m)
            Lz, Ly, Lx = self.comp_shape(m)
            iz = cz * p + np.arange(sz)
            iy = cy * p + np.arange(sy)
            ix = cx * p + np.arange(sx)
            g = off[m] + (iz[:, None, None] * Ly + iy[None, :, None]) * Lx + ix[None, None, :]
            out.append(g.ravel())
        return np.concatenate(out)

    def constrained_mask(self, gamma_d: int) -> np.ndarray:
        mask = np.zeros(self.ndof, dtype=bool)
        off = self.offsets()
        n = (self.nx, self.ny, self.nz)
        for m, fam in enumerate(self.fams):
            Lz, Ly, Lx = self.comp_shape(m)
            cm = np.zeros((Lz, Ly, Lx), dtype=bool)
            for d in range(3):
                if fam[d] != P_FAM:
                    continue
                last = n[d] * self.p
                sl_lo = [slice(None)] * 3
                sl_hi = [slice(None)] * 3
                ax = 2 - d  # array axis of direction d
                sl_lo[ax] = 0
                sl_hi[ax] = last
                if gamma_d & (1 << (2 * d)):
                    cm[tuple(sl_lo)] = True
                if gamma_d & (1 << (2 * d + 1)):
                    cm[tuple(sl_hi)] = True
            mask[off[m]:off[m + 1]] = cm.ravel()
        return mask


# ------------------------------------------------------------------------ 1D tables / kron
def kron3(Tz, Ty, Tx):
    """Tensor product with x fastest (local order z, y, x)."""
    return np.kron(Tz, np.kron(Ty, Tx))


@lru_cache(maxsize=None)
def quad_tables(p: int, nq: int):
    """1D tables at the nq GLL points: s, s', r."""
    f = fdm_basis(p)
    xq, wq = gll_rule(nq)
    s, ds = f.tab_s(xq)
    r = f.tab_r(xq)
    return xq, wq, s, ds, r


def _fam_tab(fam, s, r):
    return s if fam == P_FAM else r


def comp_value_tables(k, p, nq, m, qz_slice=None):
    """(points, n_m) value table and dict d -> derivative table (only P directions) of
    component m's scalar factor f, for quadrature points (qz in qz_slice, qy, qx)."""
    xq, wq, s, ds, r = quad_tables(p, nq)
    fx, fy, fz = FAMILIES[k][m]
    Tx, Ty, Tz = _fam_tab(fx, s, r), _fam_tab(fy, s, r), _fam_tab(fz, s, r)
    if qz_slice is not None:
        Tz = Tz[qz_slice]
    V = kron3(Tz, Ty, Tx)
    dV = {}
    if fx == P_FAM:
        dV[0] = kron3(Tz, Ty, ds)
    if fy == P_FAM:
        dV[1] = kron3(Tz, ds, Tx)
    if fz == P_FAM:
        dsz = ds if qz_slice is None else ds[qz_slice]
        dV[2] = kron3(dsz, Ty, Tx)
    return V, dV


def reference_fields(k, p, nq, qz_slice=None):
    """Reference value field Vhat (points, ncomp_v, n) and reference derivative field
    dhat (points, ncomp_d, n) of the element basis, for k = 0, 1, 2."""
    sizes = [int(np.prod([(p + 1) if f == P_FAM else p for f in fam])) for fam in FAMILIES[k]]
    n = sum(sizes)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    npts = None
    comps = []
    for m in range(len(FAMILIES[k])):
        V, dV = comp_value_tables(k, p, nq, m, qz_slice)
        comps.append((V, dV))
        npts = V.shape[0]
    if k == 0:
        V, dV = comps[0]
        val = V[:, None, :]
        der = np.stack([dV[0], dV[1], dV[2]], axis=1)  # grad-hat
        return val, der
    val = np.zeros((npts, 3, n))
    for m in range(3):
        val[:, m, offs[m]:offs[m + 1]] = comps[m][0]
    if k == 1:
        der = np.zeros((npts, 3, n))
        # curl(f e_x) = (0, d_z f, -d_y f); curl(f e_y) = (-d_z f, 0, d_x f); curl(f e_z) = (d_y f, -d_x f, 0)
        _, d = comps[0]
        der[:, 1, offs[0]:offs[1]] = d[2]
        der[:, 2, offs[0]:offs[1]] = -d[1]
        _, d = comps[1]
        der[:, 0, offs[1]:offs[2]] = -d[2]
        der[:, 2, offs[1]:offs[2]] = d[0]
        _, d = comps[2]
        der[:, 0, offs[2]:offs[3]] = d[1]
        der[:, 1, offs[2]:offs[3]] = -d[0]
        return val, der
    if k == 2:
        der = np.zeros((npts, 1, n))
        for m in range(3):
            der[:, 0, offs[m]:offs[m + 1]] = comps[m][1][m]
        return val, der
    raise ValueError(k)


# ------------------------------------------------------------------------------ geometry
def trilinear_geometry(Xc: np.ndarray, xq: np.ndarray, qz_slice=None):
    """Jacobian J (points, 3, 3) with J[:, i, d] = d x_i / d xhat_d, for the trilinear map
    F(xhat) = sum_a X_a prod_d phi_{a_d}(xhat_d), phi_0 = (1-t)/2, phi_1 = (1+t)/2.
    Xc: (2, 2, 2, 3) vertices indexed [az][ay][ax]."""
    t = xq
    phi = np.stack([(1 - t) / 2, (1 + t) / 2], axis=1)    # (nq, 2)
    dphi = np.stack([-0.5 * np.ones_like(t), 0.5 * np.ones_like(t)], axis=1)
    tz = phi if qz_slice is None else phi[qz_slice]
    dtz = dphi if qz_slice is None else dphi[qz_slice]
    # points ordered (qz, qy, qx)
    Jx = np.einsum("zc,yb,xa,cbai->zyxi", tz, phi, dphi, Xc)
    Jy = np.einsum("zc,yb,xa,cbai->zyxi", tz, dphi, phi, Xc)
    Jz = np.einsum("zc,yb,xa,cbai->zyxi", dtz, phi, phi, Xc)
    J = np.stack([Jx, Jy, Jz], axis=-1)                   # [..., i, d]
    return J.reshape(-1, 3, 3)


def pullback_fields(k, val, der, J):
    """Physical value and d^k fields from reference ones."""
    detJ = np.linalg.det(J)
    if k == 0:
        Jit = np.linalg.inv(J).transpose(0, 2, 1)          # J^{-T}
        return val, np.einsum("qij,qjn->qin", Jit, der), detJ
    if k == 1:
        Jit = np.linalg.inv(J).transpose(0, 2, 1)
        pv = np.einsum("qij,qjn->qin", Jit, val)
        pd = np.einsum("qij,qjn->qin", J, der) / detJ[:, None, None]
        return pv, pd, detJ
    if k == 2:
        pv = np.einsum("qij,qjn->qin", J, val) / detJ[:, None, None]
        pd = der / detJ[:, None, None]
        return pv, pd, detJ
    raise ValueError(k)


def element_matrix(k, p, Xc, alpha, beta, nq=None):
    """Dense cell matrix [A_K]_ij = (F psi_i, beta F psi_j)_K + (F d psi_i, alpha F d psi_j)_K
    by GLL quadrature (eq:form-reference-values)."""
    nq = nq or nq_for(p)
    xq, wq = gll_rule(nq)
    A = None
    for qz in range(nq):
        sl = slice(qz, qz + 1)
        val, der = reference_fields(k, p, nq, sl)
        J = trilinear_geometry(Xc, xq, sl)
        pv, pd, detJ = pullback_fields(k, val, der, J)
        w = (wq[qz] * np.outer(wq, wq)).ravel() * detJ
        # sum_q w_q beta F psi_n(q) . F psi_m(q) (and the same for d): as matrix products (BLAS)
        Mq = sum(pv[:, c, :].T @ ((w * beta)[:, None] * pv[:, c, :]) for c in range(pv.shape[1]))
        Kq = sum(pd[:, c, :].T @ ((w * alpha)[:, None] * pd[:, c, :]) for c in range(pd.shape[1]))
        A = Mq + Kq if A is None else A + Mq + Kq
    return A


def element_apply(k, p, Xc, alpha, beta, u_loc, nq=None):
    """A_K u_loc by quadrature without forming A_K: V^T W (V u) (same sums as element_matrix)."""
    nq = nq or nq_for(p)
    xq, wq = gll_rule(nq)
    out = np.zeros_like(u_loc)
    for qz in range(nq):
        sl = slice(qz, qz + 1)
        val, der = reference_fields(k, p, nq, sl)
        J = trilinear_geometry(Xc, xq, sl)
        pv, pd, detJ = pullback_fields(k, val, der, J)
        w = (wq[qz] * np.outer(wq, wq)).ravel() * detJ
        uv = np.einsum("qcn,n->qc", pv, u_loc)
        ud = np.einsum("qcn,n->qc", pd, u_loc)
        out += np.einsum("qcn,qc->n", pv, (w * beta)[:, None] * uv)
        out += np.einsum("qcn,qc->n", pd, (w * alpha)[:, None] * ud)
    return out


# ------------------------------------------------------------------ symbolic cell patterns
def _I(n):
    return np.eye(n, dtype=np.int64)


def ref_derivative_pattern_or_values(k, p, values: bool):
    """Cell-level reference exterior derivative d-hat^k as a matrix (rows: V^{k+1} local
    order, cols: V^k local order), built from D-hat Kronecker products (P:565-586,
    standard curl sign).  values=False gives the 0/1 structural pattern."""
    f = fdm_basis(p)
    Dh = f.D if values else pattern_D(p).astype(np.int64)
    IP = np.eye(p + 1) if values else _I(p + 1)
    ID = np.eye(p) if values else _I(p)
    Z = lambda r, c: np.zeros((r, c))
    if k == 0:
        blocks = [[kron3(IP, IP, Dh)], [kron3(IP, Dh, IP)], [kron3(Dh, IP, IP)]]
    elif k == 1:
        # NCE comps: x (D,P,P), y (P,D,P), z (P,P,D); NCF comps: x (P,D,D), y (D,P,D), z (D,D,P)
        nce = [(p) * (p + 1) ** 2] * 3
        ncf = [(p + 1) * p * p] * 3
        bx = [None, -kron3(Dh, ID, IP), kron3(ID, Dh, IP)]      # d_y u_z - d_z u_y
        by = [kron3(Dh, IP, ID), None, -kron3(ID, IP, Dh)]      # d_z u_x - d_x u_z
        bz = [-kron3(IP, Dh, ID), kron3(IP, ID, Dh), None]      # d_x u_y - d_y u_x
        blocks = []
        for r, row in enumerate([bx, by, bz]):
            blocks.append([b if b is not None else Z(ncf[r], nce[c]) for c, b in enumerate(row)])
        if not values:
            blocks = [[np.abs(b) for b in row] for row in blocks]
    elif k == 2:
        blocks = [[kron3(ID, ID, Dh), kron3(ID, Dh, ID), kron3(Dh, ID, ID)]]
    else:
        raise ValueError(k)
    M = np.block(blocks)
    return M if values else (M != 0)


def mass_pattern(k, p):
    """Structural pattern of the Cartesian mass matrix of V^k: Kronecker of B-hat (P) and I (DP)."""
    PB = pattern_B(p).astype(np.int64)
    mats = []
    for fam in FAMILIES[k]:
        t = [PB if fm == P_FAM else _I(p) for fm in fam]
        mats.append(kron3(t[2], t[1], t[0]))
    n = sum(m.shape[0] for m in mats)
    out = np.zeros((n, n), dtype=bool)
    o = 0
    for m in mats:
        out[o:o + m.shape[0], o:o + m.shape[0]] = m != 0
        o += m.shape[0]
    return out


@lru_cache(maxsize=16)
def cartesian_cell_pattern(k, p):
    """Structural pattern of A_K on Cartesian cells: pattern(M^k) U pattern(D^T M^{k+1} D)
    (eq:sum-factorization)."""
    Mk = mass_pattern(k, p).astype(np.int64)
    D = ref_derivative_pattern_or_values(k, p, values=False).astype(np.int64)
    Mk1 = mass_pattern(k + 1, p).astype(np.int64)
    return (Mk + D.T @ Mk1 @ D) != 0


# --------------------------------------------------------------------------- assembly
def cell_vertices(X, cx, cy, cz):
    return X[cz:cz + 2, cy:cy + 2, cx:cx + 2, :]


def is_axis_aligned(Xc, tol=1e-14):
    lo = Xc[0, 0, 0]
    hi = Xc[1, 1, 1]
    for az in range(2):
        for ay in range(2):
            for ax in range(2):
                expect = np.array([(lo, hi)[ax][0], (lo, hi)[ay][1], (lo, hi)[az][2]])
                if np.abs(Xc[az, ay, ax] - expect).max() > tol:
                    return False
    return True


@lru_cache(maxsize=512)
def _cartesian_parts(k, p, hx, hy, hz):
    """(M, K) cell matrices for alpha=beta=1 on an axis-aligned box with sides h, by
    quadrature, with structurally-zero entries set to exact zero."""
    Xc = np.zeros((2, 2, 2, 3))
    for az in range(2):
        for ay in range(2):
            for ax in range(2):
                Xc[az, ay, ax] = (ax * hx, ay * hy, az * hz)
    M = element_matrix(k, p, Xc, 0.0, 1.0)
    K = element_matrix(k, p, Xc, 1.0, 0.0)
    pat = cartesian_cell_pattern(k, p)
    return np.where(pat, M, 0.0), np.where(pat, K, 0.0)


def assemble(space: Space, X: np.ndarray, alpha: np.ndarray, beta: np.ndarray) -> sp.csr_matrix:
    """Global matrix over ALL DoFs (constraints not yet removed)."""
    rows, cols, vals = [], [], []
    for cz in range(space.nz):
        for cy in range(space.ny):
            for cx in range(space.nx):
                Xc = cell_vertices(X, cx, cy, cz)
                a, b = alpha[cz, cy, cx], beta[cz, cy, cx]
                if is_axis_aligned(Xc):
                    h = Xc[1, 1, 1] - Xc[0, 0, 0]
                    M, K = _cartesian_parts(space.k, space.p, float(h[0]), float(h[1]), float(h[2]))
                    AK = b * M + a * K
                else:
                    AK = element_matrix(space.k, space.p, Xc, a, b)
                g = space.cell_dofs(cx, cy, cz)
                r, c = np.nonzero(AK)
                rows.append(g[r]); cols.append(g[c]); vals.append(AK[r, c])
    n = space.ndof
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))


def apply_matfree(space: Space, X, alpha, beta, u):
    """v = A u cell by cell by quadrature, without forming any matrix (used at high p)."""
    v = np.zeros_like(u)
    for cz in range(space.nz):
        for cy in range(space.ny):
            for cx in range(space.nx):
                g = space.cell_dofs(cx, cy, cz)
                Xc = cell_vertices(X, cx, cy, cz)
                v[g] += element_apply(space.k, space.p, Xc, alpha[cz, cy, cx], beta[cz, cy, cx], u[g])
    return v


def dof_coords(space: Space, g):
    """(component, ix, iy, iz) of a global DoF index."""
    off = space.offsets()
    m = int(np.searchsorted(off, g, side="right") - 1)
    Lz, Ly, Lx = space.comp_shape(m)
    r = g - off[m]
    return m, r % Lx, (r // Lx) % Ly, r // (Lx * Ly)


def cells_containing(space: Space, g):
    """Cells whose closure carries the basis function of DoF g (structured layout rule)."""
    m, ix, iy, iz = dof_coords(space, g)
    n = (space.nx, space.ny, space.nz)
    per = []
    for d, i in enumerate((ix, iy, iz)):
        if space.fams[m][d] == D_FAM or i % space.p:
            per.append([i // space.p])
        else:
            per.append([c for c in (i // space.p - 1, i // space.p) if 0 <= c < n[d]])
    return [(cx, cy, cz) for cz in per[2] for cy in per[1] for cx in per[0]]


def _cell_matrix(space, X, alpha, beta, cx, cy, cz):
    Xc = cell_vertices(X, cx, cy, cz)
    if is_axis_aligned(Xc):
        h = Xc[1, 1, 1] - Xc[0, 0, 0]
        M, K = _cartesian_parts(space.k, space.p, float(h[0]), float(h[1]), float(h[2]))
        return beta[cz, cy, cx] * M + alpha[cz, cy, cx] * K
    return element_matrix(space.k, space.p, Xc, alpha[cz, cy, cx], beta[cz, cy, cx])


def local_matrix(space: Space, X, alpha, beta, g):
    """A[g][:, g] assembled only from the cells carrying those DoFs (no global matrix)."""
    g = np.asarray(g)
    pos = {int(v): i for i, v in enumerate(g)}
    cells = set()
    for v in g:
        cells.update(cells_containing(space, int(v)))
    A = np.zeros((len(g), len(g)))
    for (cx, cy, cz) in sorted(cells):
        cd = space.cell_dofs(cx, cy, cz)
        loc = np.array([pos.get(int(v), -1) for v in cd])
        sel = np.flatnonzero(loc >= 0)
        AK = _cell_matrix(space, X, alpha, beta, cx, cy, cz)
        A[np.ix_(loc[sel], loc[sel])] += AK[np.ix_(sel, sel)]
    return A


def cell_rows_apply(space: Space, X, alpha, beta, u, rows):
    """(A u)[rows] computed only from the cells that contain those DoFs (sampled parity)."""
    rows = np.asarray(rows)
    out = np.zeros(len(rows))
    cells = set()
    for r in rows:
        cells.update(cells_containing(space, int(r)))
    for (cx, cy, cz) in sorted(cells):
        g = space.cell_dofs(cx, cy, cz)
        Xc = cell_vertices(X, cx, cy, cz)
        if is_axis_aligned(Xc):
            h = Xc[1, 1, 1] - Xc[0, 0, 0]
            M, K = _cartesian_parts(space.k, space.p, float(h[0]), float(h[1]), float(h[2]))
            vloc = (beta[cz, cy, cx] * M + alpha[cz, cy, cx] * K) @ u[g]
        else:
            vloc = element_apply(space.k, space.p, Xc, alpha[cz, cy, cx], beta[cz, cy, cx], u[g])
        pos = {int(gi): i for i, gi in enumerate(g)}
        for t, r in enumerate(rows):
            if int(r) in pos:
                out[t] += vloc[pos[int(r)]]
    return out


# -------------------------------------------------------------------- global derivative D
@lru_cache(maxsize=16)
def derivative_blocks(k, p, nx, ny, nz):
    """The blocks of the tabulated d^k : V^k_h -> V^{k+1}_h on reference values: per
    direction the 1D global D-hat (row c p + a = sum_i D-hat[a, i] at column c p + i) or an
    identity, Kronecker-combined like eq:gradbasis/eq:curlbasis/eq:divbasis (standard curl sign).
    Returns [(row component, column component, sign, (Z, Y, X) 1D sparse factors)]."""
    f = fdm_basis(p)
    n = (nx, ny, nz)

    def D1(d):
        L = n[d]
        rows, cols, vals = [], [], []
        for c in range(L):
            for a in range(p):
                for i in range(p + 1):
                    if f.D[a, i] != 0.0:
                        rows.append(c * p + a); cols.append(c * p + i); vals.append(f.D[a, i])
        return sp.csr_matrix((vals, (rows, cols)), shape=(L * p, L * p + 1))

    def I(fam, d):
        return sp.identity(n[d] * p + 1 if fam == P_FAM else n[d] * p, format="csr")

    Dx, Dy, Dz = D1(0), D1(1), D1(2)
    Pp = lambda d: I(P_FAM, d)   # noqa: E731
    Dd = lambda d: I(D_FAM, d)   # noqa: E731
    if k == 0:
        return [(0, 0, 1.0, (Pp(2), Pp(1), Dx)), (1, 0, 1.0, (Pp(2), Dy, Pp(0))), (2, 0, 1.0, (Dz, Pp(1), Pp(0)))]
    if k == 1:
        # source comps: x (D,P,P), y (P,D,P), z (P,P,D); curl x = d_y u_z - d_z u_y, ...
        return [(0, 1, -1.0, (Dz, Dd(1), Pp(0))), (0, 2, 1.0, (Dd(2), Dy, Pp(0))),
                (1, 0, 1.0, (Dz, Pp(1), Dd(0))), (1, 2, -1.0, (Dd(2), Pp(1), Dx)),
                (2, 0, -1.0, (Pp(2), Dy, Dd(0))), (2, 1, 1.0, (Pp(2), Dd(1), Dx))]
    if k == 2:
        return [(0, 0, 1.0, (Dd(2), Dd(1), Dx)), (0, 1, 1.0, (Dd(2), Dy, Dd(0))), (0, 2, 1.0, (Dz, Dd(1), Dd(0)))]
    raise ValueError(k)


@lru_cache(maxsize=16)
def _derivative_blocks_t(k, p, nx, ny, nz):
    """derivative_blocks with every 1D factor transposed (column access)."""
    return [(r, c, sg, tuple(M.T.tocsr() for M in f)) for r, c, sg, f in derivative_blocks(k, p, nx, ny, nz)]


def _csr_row(M, i):
    a, b = M.indptr[i], M.indptr[i + 1]
    return list(zip(M.indices[a:b].tolist(), M.data[a:b].tolist()))


def global_derivative(k, p, nx, ny, nz) -> sp.csr_matrix:
    """d^k as one sparse matrix (rows V^{k+1}, columns V^k): the blocks of derivative_blocks."""
    blocks = derivative_blocks(k, p, nx, ny, nz)
    nr = 1 + max(b[0] for b in blocks)
    nc = 1 + max(b[1] for b in blocks)
    grid = [[None] * nc for _ in range(nr)]
    for r, c, sg, (Z, Y, X) in blocks:
        grid[r][c] = sg * sp.kron(Z, sp.kron(Y, X, format="csr"), format="csr")
    return sp.bmat(grid, format="csr")


def derivative_entries(k, p, nx, ny, nz, index, by="row"):
    """Entries of one row (by="row") or one column (by="col") of global_derivative without forming
    it: {other index: value}, from the same Kronecker blocks."""
    blocks = derivative_blocks(k, p, nx, ny, nz) if by == "row" else _derivative_blocks_t(k, p, nx, ny, nz)
    rsp, csp = Space(k + 1, p, nx, ny, nz), Space(k, p, nx, ny, nz)
    own, oth = (rsp, csp) if by == "row" else (csp, rsp)
    oo, ot = own.offsets(), oth.offsets()
    m = int(np.searchsorted(oo, index, side="right") - 1)
    Lz, Ly, Lx = own.comp_shape(m)
    r = index - oo[m]
    iz, iy, ix = r // (Lx * Ly), (r // Lx) % Ly, r % Lx
    out = {}
    for br, bc, sg, (Z, Y, X) in blocks:
        if (br if by == "row" else bc) != m:
            continue
        mo = bc if by == "row" else br
        Tz, Ty, Tx = oth.comp_shape(mo)
        rz, ry, rx = (_csr_row(Z, iz), _csr_row(Y, iy), _csr_row(X, ix))
        for cz, vz in rz:
            for cy, vy in ry:
                for cx, vx in rx:
                    g = ot[mo] + (cz * Ty + cy) * Tx + cx
                    out[g] = out.get(g, 0.0) + sg * vz * vy * vx
    return out


# ---------------------------------------------------------------- auxiliary operator (k=0)
def broken_G3(k, p):
    """G-bar for V^k on the cell: block-diagonal over components, Kronecker of G-bar_1D (P
    directions) and identity (DP directions)."""
    f = fdm_basis(p)
    blocks = []
    for fam in FAMILIES[k]:
        t = [f.G if fm == P_FAM else np.eye(p) for fm in fam]
        blocks.append(kron3(t[2], t[1], t[0]))
    n = sum(b.shape[0] for b in blocks)
    G = np.zeros((n, n))
    o = 0
    for b in blocks:
        G[o:o + b.shape[0], o:o + b.shape[0]] = b
        o += b.shape[0]
    return G


def _kron3_sparse(Tz, Ty, Tx):
    """kron3 as a sparse matrix (same ordering, x fastest); for the high-p Kronecker factors."""
    return sp.kron(sp.csr_matrix(Tz), sp.kron(sp.csr_matrix(Ty), sp.csr_matrix(Tx), format="csr"), format="csr")


def broken_G3_sparse(k, p):
    """broken_G3 as a sparse matrix (the same Kronecker products; dense would be 11,520^2 at p = 15)."""
    f = fdm_basis(p)
    blocks = []
    for fam in FAMILIES[k]:
        t = [f.G if fm == P_FAM else np.eye(p) for fm in fam]
        blocks.append(_kron3_sparse(t[2], t[1], t[0]))
    return sp.block_diag(blocks, format="csr")


def grad_ref_sparse(p):
    """The reference gradient d-hat^0 (V^0 -> V^1 local orders) as a sparse matrix: the same blocks
    as ref_derivative_pattern_or_values(0, p, values=True), eq:gradbasis."""
    f = fdm_basis(p)
    IP = np.eye(p + 1)
    return sp.vstack([_kron3_sparse(IP, IP, f.D), _kron3_sparse(IP, f.D, IP), _kron3_sparse(f.D, IP, IP)], format="csr")


def aux_element_matrix(p, Xc, alpha, beta, nq=None, sparse=False):
    """P_K for k=0 (eq:sum-factorization_approx):
        diag(M-bar^0_beta)_a       = sum_q w_q beta detJ psi-bar_a^2
        diag(M-bar^1_alpha)_(m,a)  = sum_q w_q alpha detJ (J^{-1} J^{-T})_mm Psi-bar^(m)_a^2
        P_K = G0^T diag(M0) G0 + (G1 D)^T diag(M1) (G1 D)
    with psi-bar, Psi-bar the broken (interface-orthonormalised) bases."""
    nq = nq or nq_for(p)
    f = fdm_basis(p)
    xq, wq = gll_rule(nq)
    sb, _ = f.tab_sbar(xq)
    r = f.tab_r(xq)
    diag0 = np.zeros((p + 1) ** 3)
    diag1 = [np.zeros(p * (p + 1) ** 2) for _ in range(3)]
    for qz in range(nq):
        sl = slice(qz, qz + 1)
        J = trilinear_geometry(Xc, xq, sl)
        detJ = np.linalg.det(J)
        Ji = np.linalg.inv(J)
        JiJit = np.einsum("qij,qkj->qik", Ji, Ji)
        w = (wq[qz] * np.outer(wq, wq)).ravel() * detJ
        V0 = kron3(sb[sl], sb, sb)
        diag0 += (w * beta) @ (V0 ** 2)
        tabs = [kron3(sb[sl], sb, r), kron3(sb[sl], r, sb), kron3(r[sl], sb, sb)]
        for m in range(3):
            diag1[m] += (w * alpha * JiJit[:, m, m]) @ (tabs[m] ** 2)
    G0 = broken_G3_sparse(0, p)
    Db = broken_G3_sparse(1, p) @ grad_ref_sparse(p)
    d1 = np.concatenate(diag1)
    PK = G0.T @ sp.diags(diag0) @ G0 + Db.T @ sp.diags(d1) @ Db
    return PK.tocsr() if sparse else PK.toarray()


def aux_cell_pattern(p):
    """Structural pattern of P_K: pattern(G)^T pattern(G) U pattern(G1 D)^T pattern(G1 D)
    (0/1 Kronecker products, sparse)."""
    # G-bar_1D pattern is B-hat's pattern (identity + (0,p) corner)
    PB = pattern_B(p).astype(np.int64)
    G0 = _kron3_sparse(PB, PB, PB)
    blocks = []
    for fam in FAMILIES[1]:
        t = [PB if fm == P_FAM else _I(p) for fm in fam]
        blocks.append(_kron3_sparse(t[2], t[1], t[0]))
    G1 = sp.block_diag(blocks, format="csr")
    PD = pattern_D(p).astype(np.int64)
    IP = _I(p + 1)
    D = sp.vstack([_kron3_sparse(IP, IP, PD), _kron3_sparse(IP, PD, IP), _kron3_sparse(PD, IP, IP)], format="csr")
    Db = G1 @ D
    return ((G0.T @ G0 + Db.T @ Db) != 0).toarray()


def assemble_aux(space: Space, X, alpha, beta):
    """Global auxiliary operator P (k = 0) over all DoFs, structural pattern kept exact."""
    assert space.k == 0
    pat = aux_cell_pattern(space.p)
    rows, cols, vals, prow, pcol = [], [], [], [], []
    for cz in range(space.nz):
        for cy in range(space.ny):
            for cx in range(space.nx):
                Xc = cell_vertices(X, cx, cy, cz)
                PK = aux_element_matrix(space.p, Xc, alpha[cz, cy, cx], beta[cz, cy, cx], sparse=True)
                g = space.cell_dofs(cx, cy, cz)
                r, c = np.nonzero(pat)
                rows.append(g[r]); cols.append(g[c]); vals.append(np.asarray(PK[r, c]).ravel())
    n = space.ndof
    R, C, V = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    P = sp.csr_matrix((V, (R, C)), shape=(n, n))
    S = sp.csr_matrix((np.ones_like(V), (R, C)), shape=(n, n))
    S.data[:] = 1.0
    return P, S
