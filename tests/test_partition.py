"""Z-slab partition on CPU.

1. The exchange plan of `rm_partition` (the product's host arithmetic, include/rm.h): neighbours'
   send / receive ranges coincide plane by plane in global terms, owned DoF planes and owned
   vertex layers partition the global ones exactly once.
2. A world_size-2 `gloo` run of the distributed sweep: each rank builds its LOCAL problem from
   the plan, fills its forward halos from the neighbour (planes it does not own start as NaN),
   computes r = f - A u on the local mesh (oracle apply), the local patch correction with the
   product's host emulator restricted to the owned vertex layers (the same patch filter the device
   setup uses), reverse-adds the correction planes, and updates its owned planes.  The result
   must equal the single-domain oracle sweep (partition invariance, up to summation order).
"""
import ctypes
import dataclasses
import os
import socket
import sys
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "native"))

import rm_inputs as ri  # noqa: E402
import paper_2211_14284_b200 as rmb  # noqa: E402


def _splits(nz, G):
    b = [nz * g // G for g in range(G + 1)]
    return [(b[g], b[g + 1]) for g in range(G)]


@pytest.mark.parametrize("nz,G,p,gamma", [(4, 2, 3, 63), (9, 3, 4, 31), (8, 4, 2, 0), (12, 5, 7, 63), (6, 6, 3, 47)])
def test_partition_plan_consistency(nz, G, p, gamma):
    nx, ny = 3, 2
    parts = [rmb.rm_partition(nx, ny, nz, p, 0, gamma, g, G, *_splits(nz, G)[g]) for g in range(G)]
    gplane = lambda P, j: P["z_cell0"] * p + j   # noqa: E731
    owned_planes, owned_layers = [], []
    for g, P in enumerate(parts):
        owned_planes += [gplane(P, j) for j in range(P["own_lo"], P["own_hi"])]
        owned_layers += [P["z_cell0"] + v for v in range(P["v_lo"], P["v_hi"])]
        assert P["plane_len"] == (nx * p + 1) * (ny * p + 1)
        # Gamma_D: x, y bits kept; z bits only on the true boundary ranks
        assert P["gamma_local"] & 0xF == gamma & 0xF
        assert bool(P["gamma_local"] & 0x10) == (g == 0 and bool(gamma & 0x10))
        assert bool(P["gamma_local"] & 0x20) == (g == G - 1 and bool(gamma & 0x20))
        if g + 1 < G:
            Q = parts[g + 1]
            fwd_up = [gplane(P, j) for j in range(*P["fwd_send_hi"])]
            assert fwd_up == [gplane(Q, j) for j in range(*Q["fwd_recv_lo"])] and len(fwd_up) == p
            fwd_dn = [gplane(Q, j) for j in range(*Q["fwd_send_lo"])]
            assert fwd_dn == [gplane(P, j) for j in range(*P["fwd_recv_hi"])] and len(fwd_dn) == 1
            rev = [gplane(Q, j) for j in range(*Q["rev_send_lo"])]
            assert rev == [gplane(P, j) for j in range(*P["rev_recv_hi"])] and len(rev) == p - 1
            # what a rank receives it does not own, what it sends it owns
            assert all(pl not in range(gplane(P, P["own_lo"]), gplane(P, P["own_hi"])) for pl in fwd_dn)
            assert all(pl in range(gplane(P, P["own_lo"]), gplane(P, P["own_hi"])) for pl in fwd_up)
            assert all(pl in range(gplane(P, P["own_lo"]), gplane(P, P["own_hi"])) for pl in rev)
    assert sorted(owned_planes) == list(range(nz * p + 1))
    assert sorted(owned_layers) == list(range(nz + 1))


@pytest.mark.parametrize("nz,G,p", [(4, 2, 3), (9, 3, 4), (6, 6, 2)])
def test_partition_plan_consistency_dp_components(nz, G, p):
    """H(curl) / H(div) components with a DP family in z (nz p planes, plane c p + a in cell layer
    c, no shared plane): forward / reverse ranges of neighbours coincide plane by plane, owned
    planes partition the global ones."""
    parts = [rmb.rm_partition(3, 2, nz, p, 1, 63, g, G, *_splits(nz, G)[g]) for g in range(G)]
    gplane = lambda P, j: P["z_cell0"] * p + j   # noqa: E731
    owned = []
    for g, P in enumerate(parts):
        owned += [gplane(P, j) for j in range(P["dp_own_lo"], P["dp_own_hi"])]
        if g + 1 < G:
            Q = parts[g + 1]
            up = [gplane(P, j) for j in range(*P["dp_fwd_send_hi"])]
            assert up == [gplane(Q, j) for j in range(*Q["dp_fwd_recv_lo"])] and len(up) == p
            rev = [gplane(Q, j) for j in range(*Q["dp_rev_send_lo"])]
            assert rev == [gplane(P, j) for j in range(*P["dp_rev_recv_hi"])] and len(rev) == p
            assert all(pl in range(gplane(P, P["dp_own_lo"]), gplane(P, P["dp_own_hi"])) for pl in up + rev)
        else:
            assert P["dp_fwd_send_hi"] == (0, 0) and P["dp_rev_recv_hi"] == (0, 0)
    assert sorted(owned) == list(range(nz * p))


def test_partition_rejects_bad_ranges():
    with pytest.raises(rmb.RmError):
        rmb.rm_partition(2, 2, 4, 3, 0, 63, 1, 2, 0, 2)   # rank 1 must not start at 0... it may not end before nz
    with pytest.raises(rmb.RmError):
        rmb.rm_partition(2, 2, 4, 3, 0, 63, 0, 2, 1, 2)   # rank 0 must start at layer 0


# ------------------------------------------------------------------ distributed sweep over gloo
CASES = {
    "q3-chol-dirichlet": (dataclasses.replace(ri.CONFIGS[1].with_mesh(2), nz=4), 0),
    "q3-chol-neumann-top": (dataclasses.replace(ri.CONFIGS[1].with_mesh(2), nz=4, gamma_d=0x1F), 0),
    "q3-iccsc-trilinear": (dataclasses.replace(ri.CONFIGS[5].with_mesh(2).with_p(3), nz=4), 1),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, case, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    import build_emu
    from oracle.solver import Problem
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w, fact = CASES[case]
    p, nx, ny, nz = w.p, w.nx, w.ny, w.nz
    X = ri.vertex_coords(w).reshape(nz + 1, ny + 1, nx + 1, 3)
    al, be = ri.cell_alpha(w), ri.cell_beta(w)
    gp = Problem(0, p, nx, ny, nz, X, al, be, w.gamma_d, factorization="icc_sc" if fact else "chol")
    n = gp.space.ndof
    f = ri.uniform_vector(w.cfg, 0, n); f[gp.constrained] = 0
    u = ri.uniform_vector(w.cfg, 3, n); u[gp.constrained] = 0
    zb, ze = _splits(nz, world)[rank]
    P = rmb.rm_partition(nx, ny, nz, p, 0, w.gamma_d, rank, world, zb, ze)
    L, z0, nzl = P["plane_len"], P["z_cell0"], P["nz_local"]
    g0 = z0 * p * L
    nloc = (nzl * p + 1) * L
    own = slice(P["own_lo"] * L, P["own_hi"] * L)
    # local vectors: owned planes from the global data, everything else NaN until received
    fl = np.full(nloc, np.nan); ul = np.full(nloc, np.nan)
    fl[own] = f[g0:g0 + nloc][own]; ul[own] = u[g0:g0 + nloc][own]

    def xfer(vec, send, recv, peer):
        reqs, buf = [], None
        if send[1] > send[0]:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(vec[send[0] * L:send[1] * L])), peer))
        if recv[1] > recv[0]:
            buf = torch.empty((recv[1] - recv[0]) * L, dtype=torch.float64)
            reqs.append(dist.irecv(buf, peer))
        for r_ in reqs:
            r_.wait()
        return buf

    for vec in (fl, ul):   # forward halos
        if rank > 0:
            b = xfer(vec, P["fwd_send_lo"], P["fwd_recv_lo"], rank - 1)
            vec[P["fwd_recv_lo"][0] * L:P["fwd_recv_lo"][1] * L] = b.numpy()
        if rank < world - 1:
            b = xfer(vec, P["fwd_send_hi"], P["fwd_recv_hi"], rank + 1)
            vec[P["fwd_recv_hi"][0] * L:P["fwd_recv_hi"][1] * L] = b.numpy()
    assert np.isfinite(fl).all() and np.isfinite(ul).all(), "forward halo left planes unfilled"
    # local problem: residual with the oracle, owned-patch correction with the product's host code
    Xl = X[z0:z0 + nzl + 1]
    lp = Problem(0, p, nx, ny, nzl, Xl, al[z0:z0 + nzl], be[z0:z0 + nzl], P["gamma_local"])
    r = lp.residual(fl, ul)
    emu = ctypes.CDLL(build_emu.build())
    D = ctypes.POINTER(ctypes.c_double)
    dp = lambda a: a.ctypes.data_as(D)   # noqa: E731
    alc = np.ascontiguousarray(al[z0:z0 + nzl].ravel()); bec = np.ascontiguousarray(be[z0:z0 + nzl].ravel())
    cart = w.perturb == 0
    Xc = None if cart else np.ascontiguousarray(Xl.ravel())
    hz = np.ascontiguousarray(np.diff(Xl[:, 0, 0, 2]))
    c = np.zeros(nloc)
    err = ctypes.create_string_buffer(256)
    rc = emu.emu_precondition_zv(0, p, nx, ny, nzl, ctypes.c_uint(P["gamma_local"]), dp(alc), ctypes.c_longlong(alc.size),
                                 dp(bec), ctypes.c_longlong(bec.size), None if cart else dp(Xc), 0, fact, P["v_lo"],
                                 P["v_hi"], dp(hz) if cart else None, dp(r), dp(c), err, 256)
    assert rc == 0, err.value
    # reverse-add of the corrections on the neighbour's planes
    if rank > 0:
        xfer(c, P["rev_send_lo"], (0, 0), rank - 1)
    if rank < world - 1:
        b = xfer(c, (0, 0), P["rev_recv_hi"], rank + 1)
        c[P["rev_recv_hi"][0] * L:P["rev_recv_hi"][1] * L] += b.numpy()
    uo = ul + c
    ref = gp.relax(f, u)[g0:g0 + nloc]
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.stack([uo[own], ref[own]]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", list(CASES))
def test_slab_sweep_gloo_world2(case):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank_main, args=(2, _free_port(), case, d), nprocs=2, join=True)
        for rank in range(2):
            got, ref = np.load(os.path.join(d, f"r{rank}.npy"))
            assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), (case, rank)


# ------------------------------------------------------- H(curl) / H(div) slabs (PH) over gloo
PH_CASES = {
    "nce3-ph": dataclasses.replace(ri.CONFIGS[3].with_mesh(2).with_p(3), nz=4),
    "ncf3-ph": dataclasses.replace(ri.CONFIGS[4].with_mesh(2).with_p(3), nz=4),
    "nce3-ph-neumann-top": dataclasses.replace(ri.CONFIGS[3].with_mesh(2).with_p(3), nz=4, gamma_d=0x1F),
}


def comp_views(gsp, lsp, z_cell0, p):
    """Per component: (global slice of the local planes, local slice, plane length, DP-in-z flag)."""
    from oracle.fem import P_FAM
    out = []
    go, lo = gsp.offsets(), lsp.offsets()
    for m in range(len(lsp.fams)):
        Lz, Ly, Lx = lsp.comp_shape(m)
        Lm = Ly * Lx
        g0 = go[m] + z_cell0 * p * Lm
        out.append((slice(g0, g0 + Lz * Lm), slice(lo[m], lo[m] + Lz * Lm), Lm, lsp.fams[m][2] != P_FAM))
    return out


def _rank_main_ph(rank, world, port, case, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    import build_emu
    from oracle.fem import Space, global_derivative
    from oracle.solver import EPS_S, Problem
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = PH_CASES[case]
    k, p, nx, ny, nz = w.space, w.p, w.nx, w.ny, w.nz
    X = ri.vertex_coords(w)
    al, be = ri.cell_alpha(w), ri.cell_beta(w)
    gp = Problem(k, p, nx, ny, nz, X, al, be, w.gamma_d, decomposition="ph")
    n = gp.space.ndof
    f = ri.uniform_vector(w.cfg, 0, n); f[gp.constrained] = 0
    u = ri.uniform_vector(w.cfg, 3, n); u[gp.constrained] = 0
    zb, ze = _splits(nz, world)[rank]
    P = rmb.rm_partition(nx, ny, nz, p, k, w.gamma_d, rank, world, zb, ze)
    z0, nzl = P["z_cell0"], P["nz_local"]
    lsp = Space(k, p, nx, ny, nzl)
    views = comp_views(gp.space, lsp, z0, p)
    nloc = lsp.ndof
    rng = lambda dp, key: P[("dp_" if dp else "") + key]   # noqa: E731
    fl = np.full(nloc, np.nan); ul = np.full(nloc, np.nan)
    for gs, ls, Lm, dp in views:
        lo, hi = rng(dp, "own_lo"), rng(dp, "own_hi")
        own = slice(ls.start + lo * Lm, ls.start + hi * Lm)
        fl[own] = f[gs][lo * Lm:hi * Lm]
        ul[own] = u[gs][lo * Lm:hi * Lm]

    def xfer(send, recv, peer):
        reqs, bufs = [], []
        for s_ in send:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(s_)), peer))
        for nr in recv:
            b = torch.empty(nr, dtype=torch.float64)
            bufs.append(b)
            reqs.append(dist.irecv(b, peer))
        for r_ in reqs:
            r_.wait()
        return [b.numpy() for b in bufs]

    def planes(vec, ls, Lm, rg):
        return vec[ls.start + rg[0] * Lm:ls.start + rg[1] * Lm]

    for vec in (fl, ul):   # forward halos, per component
        for peer, sk, rk in ((rank - 1, "fwd_send_lo", "fwd_recv_lo"), (rank + 1, "fwd_send_hi", "fwd_recv_hi")):
            if not 0 <= peer < world:
                continue
            sends, recvs, where = [], [], []
            for gs, ls, Lm, dp in views:
                sr = (0, 0) if (dp and sk == "fwd_send_lo") else rng(dp, sk)
                rr = (0, 0) if (dp and rk == "fwd_recv_hi") else rng(dp, rk)
                if sr[1] > sr[0]:
                    sends.append(planes(vec, ls, Lm, sr))
                if rr[1] > rr[0]:
                    recvs.append((rr[1] - rr[0]) * Lm)
                    where.append((ls, Lm, rr))
            got = xfer(sends, recvs, peer)
            for (ls, Lm, rr), b in zip(where, got):
                vec[ls.start + rr[0] * Lm:ls.start + rr[1] * Lm] = b
    assert np.isfinite(fl).all() and np.isfinite(ul).all(), "forward halo left planes unfilled"
    Xl = X[z0:z0 + nzl + 1]
    lp = Problem(k, p, nx, ny, nzl, Xl, al[z0:z0 + nzl], be[z0:z0 + nzl], P["gamma_local"], decomposition="ph")
    r = lp.residual(fl, ul)
    emu = ctypes.CDLL(build_emu.build())
    Dp = ctypes.POINTER(ctypes.c_double)
    dptr = lambda a: a.ctypes.data_as(Dp)   # noqa: E731
    hz = np.ascontiguousarray(np.diff(Xl[:, 0, 0, 2]))
    err = ctypes.create_string_buffer(256)

    def family(kk, alpha, beta, rhs):
        out = np.zeros_like(rhs)
        a_, b_ = np.ascontiguousarray(alpha.ravel()), np.ascontiguousarray(beta.ravel())
        rc = emu.emu_precondition_zv(kk, p, nx, ny, nzl, ctypes.c_uint(P["gamma_local"]), dptr(a_),
                                     ctypes.c_longlong(a_.size), dptr(b_), ctypes.c_longlong(b_.size), None, kk, 0,
                                     P["v_lo"], P["v_hi"], dptr(hz), dptr(np.ascontiguousarray(rhs)), dptr(out), err, 256)
        assert rc == 0, err.value
        return out

    alc, bec = al[z0:z0 + nzl], be[z0:z0 + nzl]
    c = family(k, alc, bec, r)                                  # owned k-star patches
    D = global_derivative(k - 1, p, nx, ny, nzl)
    pcon = Space(k - 1, p, nx, ny, nzl).constrained_mask(P["gamma_local"])
    t = D.T @ r
    t[pcon] = 0.0
    s_ = family(k - 1, bec, (EPS_S if k == 2 else 0.0) * bec, t)   # owned potential patches
    c += np.where(lp.constrained, 0.0, D @ s_)
    # reverse-add of the corrections on the neighbour's planes, per component
    for peer, sk, rk in ((rank - 1, "rev_send_lo", None), (rank + 1, None, "rev_recv_hi")):
        if not 0 <= peer < world:
            continue
        sends, recvs, where = [], [], []
        for gs, ls, Lm, dp in views:
            if sk:
                sr = rng(dp, sk)
                if sr[1] > sr[0]:
                    sends.append(planes(c, ls, Lm, sr))
            if rk:
                rr = rng(dp, rk)
                if rr[1] > rr[0]:
                    recvs.append((rr[1] - rr[0]) * Lm)
                    where.append((ls, Lm, rr))
        got = xfer(sends, recvs, peer)
        for (ls, Lm, rr), b in zip(where, got):
            c[ls.start + rr[0] * Lm:ls.start + rr[1] * Lm] += b
    uo = ul + c
    ref = gp.relax(f, u)
    got_own, ref_own = [], []
    for gs, ls, Lm, dp in views:
        lo, hi = rng(dp, "own_lo"), rng(dp, "own_hi")
        got_own.append(uo[ls.start + lo * Lm:ls.start + hi * Lm])
        ref_own.append(ref[gs][lo * Lm:hi * Lm])
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.stack([np.concatenate(got_own), np.concatenate(ref_own)]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", list(PH_CASES))
def test_slab_sweep_ph_gloo_world2(case):
    """H(curl) / H(div) PH sweep over a world-2 gloo partition: per-component forward halos (P and
    DP families in z), owned k-star and potential patches (the product's host code), the potential
    stage on the local mesh, per-component reverse-add; the owned planes equal the single-domain
    oracle sweep."""
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank_main_ph, args=(2, _free_port(), case, d), nprocs=2, join=True)
        for rank in range(2):
            got, ref = np.load(os.path.join(d, f"r{rank}.npy"))
            assert np.abs(got - ref).max() <= 1e-11 * max(1.0, np.abs(ref).max()), (case, rank, np.abs(got - ref).max())
