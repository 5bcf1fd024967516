"""GPU parity tests: the CUDA path (through the C ABI / thin binding) against the CPU oracle on
the same seeded inputs (rm_inputs).  Tolerance (BASELINE.json north_star): relative L2 <= 1e-11
per apply and per sweep in fp64, PCG iteration counts within +-1.  The H(div) cases carry a
conditioning-derived tolerance: two exact factorizations of the
same patch differ by ~cond(A_II) eps, and cond(A_II) ~ 5e4 at these sizes."""
import dataclasses

import numpy as np
import pytest

import gpu_util as gu
import rm_inputs as ri

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch.device("cuda", 0)


def setup_pair(w, **kw):
    import paper_2211_14284_b200 as rmb
    from oracle.solver import Problem
    coords = None if w.perturb == 0 else ri.vertex_coords(w)
    ctx = rmb.rm_setup(w.nx, w.ny, w.nz, w.p, w.space, ri.cell_alpha(w).ravel(), ri.cell_beta(w).ravel(), w.gamma_d,
                       coords=coords, decomposition={"ph": rmb.RM_PH, "sc-pafw": rmb.RM_SC_PAFW, "sc-ph": rmb.RM_SC_PH}.get(w.decomposition, rmb.RM_PAFW),
                       factorization=rmb.RM_ICC_SC if w.factorization == "icc_sc" else rmb.RM_CHOL,
                       patch_entities=kw.get("patch_entities", 0))
    pb = Problem(w.space, w.p, w.nx, w.ny, w.nz, ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w), w.gamma_d,
                 decomposition=w.decomposition, factorization=w.factorization,
                 interior_only=bool(kw.get("patch_entities", 0)), matfree=(w.perturb > 0 and w.p > 6))
    return ctx, pb


def vecs(w, ctx):
    m = ctx.constrained_mask()
    f = ri.uniform_vector(w.cfg, 0, ctx.n_local); f[m] = 0
    u = ri.uniform_vector(w.cfg, 3, ctx.n_local); u[m] = 0
    return f, u


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def check(name, err, tol):
    from conftest import record_parity
    record_parity(name, err, tol)
    assert err < tol, (name, err, tol)


def hdiv_tol(key):
    """H(div) tolerance: 10x the difference between two equally exact ORACLE
    assemblies of the same sweep (quadrature vs the box closed form), floored at the north-star
    1e-11 -- scripts/cfg4_conditioning.py, tests/golden/cfg4_conditioning.json."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cfg4_conditioning.json")))["cases"][key]
    return max(1e-11, 10 * g["oracle_vs_closed_form_assembly_sweep_rel"])


CASES = [
    ("cfg1", ri.CONFIGS[1], 1e-11),
    ("cfg2-3^3", ri.CONFIGS[2].with_mesh(3), 1e-11),
    ("cfg2-2x3x4-p4", ri.CONFIGS[2].with_mesh(2, 3, 4).with_p(4), 1e-11),
    ("cfg3-2^3-p3", ri.CONFIGS[3].with_mesh(2).with_p(3), 1e-11),
    ("cfg3-2^3-p6", ri.CONFIGS[3].with_mesh(2), 1e-11),
    ("cfg4-2^3-p3", ri.CONFIGS[4].with_mesh(2).with_p(3), hdiv_tol("2^3-p3")),
    ("cfg4-3^3-p4", ri.CONFIGS[4].with_mesh(3).with_p(4), hdiv_tol("3^3-p4")),
    ("cfg4-2^3-p8", ri.CONFIGS[4].with_mesh(2), hdiv_tol("2^3-p8")),   # cfg4's own degree
    # more patches than CTAs: the persistent kernel's cross-patch pipeline on edge / face families
    ("cfg3-6^3-p3", ri.CONFIGS[3].with_mesh(6).with_p(3), 1e-11),
    ("cfg4-5^3-p3", ri.CONFIGS[4].with_mesh(5).with_p(3), hdiv_tol("5^3-p3")),
    # trilinear cells (perturbed vertices): true operator by quadrature, auxiliary-operator
    # patches with ICC on the static-condensation pattern (cfg5 shapes at reduced size)
    ("cfg5-3^3-p3", ri.CONFIGS[5].with_mesh(3).with_p(3), 1e-11),
    ("cfg5-2^3-p7", ri.CONFIGS[5].with_mesh(2).with_p(7), 1e-11),
    ("cfg5-2^3-p15", ri.CONFIGS[5].with_mesh(2), 1e-11),             # cfg5's own degree (n_q = 24)
    # row f3: PAFW vertex stars for k = 1, 2, ICC-SC on the H(curl) potential
    ("cfg3-pafw-2^3-p3", dataclasses.replace(ri.CONFIGS[3].with_mesh(2).with_p(3), decomposition="pafw"), 1e-11),
    ("cfg4-pafw-2^3-p3", dataclasses.replace(ri.CONFIGS[4].with_mesh(2).with_p(3), decomposition="pafw"), None),
    ("cfg3-iccsc-2^3-p3", dataclasses.replace(ri.CONFIGS[3].with_mesh(2).with_p(3), factorization="icc_sc"), 1e-11),
    ("cfg3-iccsc-3^3-p4", dataclasses.replace(ri.CONFIGS[3].with_mesh(3).with_p(4), factorization="icc_sc"), 1e-11),
    # row f2 (k = 0): statically condensed vertex stars SC-PAFW (eq:sc-asm-afw), exact and ICC
    ("cfg1-sc", dataclasses.replace(ri.CONFIGS[1], decomposition="sc-pafw"), 1e-11),
    ("cfg2-sc-3^3-p4", dataclasses.replace(ri.CONFIGS[2].with_mesh(3).with_p(4), decomposition="sc-pafw"), 1e-11),
    ("cfg5-sc-3^3-p3", dataclasses.replace(ri.CONFIGS[5].with_mesh(3).with_p(3), decomposition="sc-pafw"), 1e-11),
    ("cfg5-sc-2^3-p7", dataclasses.replace(ri.CONFIGS[5].with_mesh(2).with_p(7), decomposition="sc-pafw"), 1e-11),
    # more than 1024 x entries (Lx = 342 * 3 + 1): the gathers' per-x tables end, x decoded on the fly
    ("cfg2-long-x", ri.CONFIGS[2].with_mesh(342, 1, 1).with_p(3), 1e-11),
    ("cfg5-long-x", ri.CONFIGS[5].with_mesh(342, 2, 2).with_p(3), 1e-11),
    # row f2 (k = 1, 2): SC-PH (eq:sc-asm-hiptmair), interface-only star solves + interiors once.
    # The explicit condensation (S = A_GG - A_GI A_II^-1 A_IG, c_I = y_I - A_II^-1 A_IG c_G) cancels:
    # the oracle's own two exact assemblies differ by 1.5e-11 (3^3, p = 4) and 3.2e-11 (2^3, p = 6),
    # so these cases take the derived tolerance (None: 10x the oracle noise floor)
    ("cfg3-scph-2^3-p3", dataclasses.replace(ri.CONFIGS[3].with_mesh(2).with_p(3), decomposition="sc-ph"), 1e-11),
    ("cfg3-scph-3^3-p4", dataclasses.replace(ri.CONFIGS[3].with_mesh(3).with_p(4), decomposition="sc-ph"), None),
    ("cfg3-scph-2^3-p6", dataclasses.replace(ri.CONFIGS[3].with_mesh(2), decomposition="sc-ph"), None),
    ("cfg4-scph-2^3-p3", dataclasses.replace(ri.CONFIGS[4].with_mesh(2).with_p(3), decomposition="sc-ph"), None),
    ("cfg4-scph-3^3-p3", dataclasses.replace(ri.CONFIGS[4].with_mesh(3).with_p(3), decomposition="sc-ph"), None),
]
# the one-box-buffer sequential schedule of the patch kernel (taken by full-size cfg4) forced
NBOX1_CASES = [("nbox1-" + c[0], c[1], c[2]) for c in CASES if c[0] in ("cfg2-3^3", "cfg3-2^3-p3", "cfg4-2^3-p3",
                                                                       "cfg5-3^3-p3", "cfg4-3^3-p4", "cfg3-6^3-p3",
                                                                       "cfg4-5^3-p3")]

# uniform Cartesian meshes run the class-batched patch kernel by default (few distinct factor
# blocks); the persistent stream kernel on the same shapes (RM_PATCH_STREAM=1)
STREAM_CASES = [("stream-" + c[0], c[1], c[2]) for c in CASES
                if c[0] in ("cfg1", "cfg3-2^3-p6", "cfg4-2^3-p8", "cfg3-6^3-p3", "cfg4-5^3-p3", "cfg3-pafw-2^3-p3",
                            "cfg4-pafw-2^3-p3")]
ALL_CASES = CASES + NBOX1_CASES + STREAM_CASES


@pytest.mark.parametrize("name,w,tol", ALL_CASES, ids=[c[0] for c in ALL_CASES])
def test_apply_and_sweep_parity(dev, name, w, tol, monkeypatch):
    import paper_2211_14284_b200 as rmb
    if name.startswith(("nbox1-", "stream-")):
        monkeypatch.setenv("RM_PATCH_STREAM", "1")   # read at setup (include/rm.h)
    if name.startswith("nbox1-"):
        monkeypatch.setenv("RM_NBOX1", "1")   # read by the patch plan at setup (include/rm.h)
    ctx, pb = setup_pair(w)
    info = ctx.info()
    if name.startswith(("nbox1-", "stream-")):
        assert info["batched_families"] == 0
    name = f"{name} [B={info['batch_width']}]" if info["batched_families"] else name
    assert (ctx.constrained_mask() == pb.constrained).all()
    assert ctx.n_free == int(pb.free.sum())
    f, u = vecs(w, ctx)
    if tol is None:   # H(div) PAFW, SC-PH: 10x the oracle's own assembly noise on this shape
        tol = max(1e-11, 10 * gu.oracle_noise_floor(w, f, u))
    ft, ut = torch.tensor(f, device=dev), torch.tensor(u, device=dev)
    v = torch.empty_like(ut)
    rmb.rm_apply(ctx, ut, v)
    check(name + " apply", rel(v.cpu().numpy(), pb.apply(u)), 1e-11)
    rmb.rm_residual(ctx, ft, ut, v)
    check(name + " residual", rel(v.cpu().numpy(), pb.residual(f, u)), 1e-11)
    out = torch.empty_like(ut)
    for omega in (1.0, 0.7):
        rmb.rm_relax(ctx, ft, ut, out, omega)
        check(f"{name} relax w={omega}", rel(out.cpu().numpy(), pb.relax(f, u, omega)), tol)
    # in-place (u_out aliases u_in) equals out-of-place
    u2 = ut.clone()
    rmb.rm_relax(ctx, ft, u2, u2, 0.7)
    assert torch.equal(u2, out)
    # bitwise determinism of the coloured sweep
    out2 = torch.empty_like(ut)
    rmb.rm_relax(ctx, ft, ut, out2, 0.7)
    assert torch.equal(out2, out)


@pytest.mark.parametrize("name,w", [("cfg1", ri.CONFIGS[1]), ("cfg2-2^3-p3", ri.CONFIGS[2].with_mesh(2).with_p(3)),
                                    ("cfg3-2^3-p3", ri.CONFIGS[3].with_mesh(2).with_p(3)),
                                    ("cfg4-2^3-p3", ri.CONFIGS[4].with_mesh(2).with_p(3)),
                                    ("cfg5-3^3-p3", ri.CONFIGS[5].with_mesh(3).with_p(3)),
                                    ("cfg3-pafw-2^3-p3",
                                     dataclasses.replace(ri.CONFIGS[3].with_mesh(2).with_p(3), decomposition="pafw")),
                                    ("cfg4-pafw-2^3-p3",
                                     dataclasses.replace(ri.CONFIGS[4].with_mesh(2).with_p(3), decomposition="pafw")),
                                    ("cfg3-iccsc-3^3-p3",
                                     dataclasses.replace(ri.CONFIGS[3].with_mesh(3).with_p(3), factorization="icc_sc")),
                                    ("cfg1-sc", dataclasses.replace(ri.CONFIGS[1], decomposition="sc-pafw")),
                                    ("cfg3-scph-3^3-p3",
                                     dataclasses.replace(ri.CONFIGS[3].with_mesh(3).with_p(3), decomposition="sc-ph")),
                                    ("cfg4-scph-3^3-p3",
                                     dataclasses.replace(ri.CONFIGS[4].with_mesh(3).with_p(3), decomposition="sc-ph")),
                                    ("cfg5-sc-3^3-p3",
                                     dataclasses.replace(ri.CONFIGS[5].with_mesh(3).with_p(3), decomposition="sc-pafw"))])
def test_pcg_iterations(dev, name, w):
    import paper_2211_14284_b200 as rmb
    ctx, pb = setup_pair(w)
    f, _ = vecs(w, ctx)
    x = torch.empty(ctx.n_local, dtype=torch.float64, device=dev)
    it, relres, ok = rmb.rm_pcg(ctx, torch.tensor(f, device=dev), x, 1e-8, 500)
    xo, ito, _ = pb.pcg(f)
    assert ok and relres <= 1e-8
    check(f"{name} pcg iters {it} vs oracle {ito}", abs(it - ito), 1.5)
    check(f"{name} pcg solution", rel(x.cpu().numpy(), xo), 1e-7)


def test_precondition_and_host_entry_points(dev):
    import paper_2211_14284_b200 as rmb
    w = ri.CONFIGS[1]
    ctx, pb = setup_pair(w)
    f, u = vecs(w, ctx)
    z = torch.empty(ctx.n_local, dtype=torch.float64, device=dev)
    rmb.rm_precondition(ctx, torch.tensor(f, device=dev), z)
    check("cfg1 precondition", rel(z.cpu().numpy(), pb.precondition(f)), 1e-11)
    out = np.empty_like(u)
    rmb.rm_relax_host(ctx, f, u, out, 1.0)
    check("cfg1 relax_host", rel(out, pb.relax(f, u)), 1e-11)


def test_relax_host_overlapped_copy_trilinear(dev):
    """rm_relax_host on the SC-fused path (trilinear ICC-SC, one rank) copies f on a second stream
    while the apply runs: bitwise the device-buffer sweep, and the oracle's sweep within 1e-11."""
    import paper_2211_14284_b200 as rmb
    w = ri.CONFIGS[5].with_mesh(3).with_p(5)
    ctx, pb = setup_pair(w)
    f, u = vecs(w, ctx)
    out = np.empty_like(u)
    for _ in range(2):   # second call: reused staging buffers, stream and events
        rmb.rm_relax_host(ctx, f, u, out, 0.7)
    dv = torch.empty(ctx.n_local, dtype=torch.float64, device=dev)
    rmb.rm_relax(ctx, torch.tensor(f, device=dev), torch.tensor(u, device=dev), dv, 0.7)
    assert np.array_equal(out, dv.cpu().numpy())
    check("cfg5-3^3-p5 relax_host (overlapped copies)", rel(out, pb.relax(f, u, 0.7)), 1e-11)


def test_interior_only_single_patch_exact_solve(dev):
    import paper_2211_14284_b200 as rmb
    w = ri.CONFIGS[1].with_mesh(2)
    ctx, pb = setup_pair(w, patch_entities=rmb.RM_INTERIOR_ONLY)
    assert ctx.info()["n_patches"] == 1
    f, _ = vecs(w, ctx)
    out = torch.empty(ctx.n_local, dtype=torch.float64, device=dev)
    rmb.rm_relax(ctx, torch.tensor(f, device=dev), torch.zeros_like(out), out, 1.0)
    Au = pb.apply(out.cpu().numpy())
    assert np.abs(Au - f).max() < 1e-11 * np.abs(f).max()


def test_cfg2_full_size_sampled(dev):
    """BASELINE configs[1] at full size in the bench's launch configuration: apply rows and sweep
    outputs at 128 sampled DoFs -- 16 clusters of 8 (interior, face, edge and vertex DoFs around
    seeded random vertices, so that neighbouring rows share their patches) -- each recomputed by
    the oracle from the cells / patches that carry it."""
    import paper_2211_14284_b200 as rmb
    from oracle.fem import Space, cell_rows_apply
    from oracle.solver import sampled_relax
    w = ri.CONFIGS[2]
    ctx = rmb.rm_setup(w.nx, w.ny, w.nz, w.p, w.space, ri.cell_alpha(w).ravel(), ri.cell_beta(w).ravel(), w.gamma_d)
    sp = Space(0, w.p, w.nx, w.ny, w.nz)
    X, al, be = ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w)
    f, u = vecs(w, ctx)
    ft, ut = torch.tensor(f, device=dev), torch.tensor(u, device=dev)
    L = w.nx * w.p + 1
    idx = lambda x, y, z: (z * L + y) * L + x   # noqa: E731
    g = np.random.default_rng(2024)
    rows = []
    for c in range(16):
        # vertices anywhere, including the Dirichlet face x = 0 and the Neumann faces
        vx, vy, vz = (int(t) for t in g.integers(0, w.nx + 1, size=3))
        if c == 0:
            vx, vy, vz = w.nx, w.ny, w.nz          # the far corner (Neumann on three sides)
        base = np.array([vx, vy, vz]) * w.p
        for off in ((0, 0, 0), (1, 0, 0), (1, 1, 0), (1, 1, 1), (-2, 0, 0), (-3, -1, 2), (0, 2, -1), (3, 3, 3)):
            x, y, z = np.clip(base + np.array(off), 0, L - 1)
            rows.append(idx(int(x), int(y), int(z)))
    rows = sorted(set(rows))
    um = np.where(ctx.constrained_mask(), 0.0, u)
    v = torch.empty_like(ut)
    rmb.rm_apply(ctx, ut, v)
    vo = cell_rows_apply(sp, X, al, be, um, rows)
    err = float(np.abs(v.cpu().numpy()[rows] - vo).max() / np.abs(vo).max())
    check(f"cfg2 full size apply ({len(rows)} rows, max-abs rel)", err, 1e-11)
    out = torch.empty_like(ut)
    rmb.rm_relax(ctx, ft, ut, out, 1.0)
    so = sampled_relax(sp, X, al, be, w.gamma_d, f, u, rows)
    got = out.cpu().numpy()[rows]
    check(f"cfg2 full size relax ({len(rows)} rows, max-abs rel)", float(np.abs(got - so).max() / np.abs(so).max()),
          1e-11)


@pytest.mark.parametrize("nx,p", [(2, 15), (3, 5)])
def test_trilinear_apply_full_degree(dev, nx, p):
    """cfg5's degree p = 15 (n_q = 24 GLL points per direction) on perturbed trilinear cells:
    the matrix-free apply against the oracle's quadrature apply (element by element)."""
    import paper_2211_14284_b200 as rmb
    from oracle.fem import Space, apply_matfree
    w = ri.CONFIGS[5].with_mesh(nx).with_p(p)
    ctx = rmb.rm_setup(w.nx, w.ny, w.nz, w.p, w.space, ri.cell_alpha(w).ravel(), ri.cell_beta(w).ravel(), w.gamma_d,
                       coords=ri.vertex_coords(w), factorization=rmb.RM_ICC_SC)
    f, u = vecs(w, ctx)
    m = ctx.constrained_mask()
    v = torch.empty(ctx.n_local, dtype=torch.float64, device=dev)
    rmb.rm_apply(ctx, torch.tensor(u, device=dev), v)
    sp_ = Space(0, w.p, w.nx, w.ny, w.nz)
    ref = apply_matfree(sp_, ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w), np.where(m, 0.0, u))
    ref[m] = 0.0
    check(f"trilinear apply {nx}^3 p={p}", rel(v.cpu().numpy(), ref), 1e-11)


# ------------------------------------------------------------------ z-slab partition on one GPU
# Row a3: two contexts on the same device hold the local problems of rank 0 and
# rank 1 of 2 (no communicator: the split-stage calls), the test moves the halo planes with plain
# device copies following rm_partition's plan, and the owned planes of the result must equal the
# single-context sweep.  (The NCCL path of rm_relax performs the same moves with ncclSend/Recv.)
SLAB_CASES = [
    ("q3-cart-dirichlet", dataclasses.replace(ri.CONFIGS[1].with_mesh(3), nz=4)),
    ("q4-cart-neumann-z", dataclasses.replace(ri.CONFIGS[2].with_mesh(3).with_p(4), nz=5)),
    ("q3-trilinear-iccsc", dataclasses.replace(ri.CONFIGS[5].with_mesh(3).with_p(3), nz=4)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,w", SLAB_CASES, ids=[c[0] for c in SLAB_CASES])
def test_slab_partition_two_contexts(dev, name, w):
    import torch
    import paper_2211_14284_b200 as rmb
    G = 2
    gctx = gu.setup_product(w)
    n = gctx.n_local
    mask = gctx.constrained_mask()
    f = ri.uniform_vector(w.cfg, 0, n); f[mask] = 0
    u = ri.uniform_vector(w.cfg, 3, n); u[mask] = 0
    ft, ut = torch.tensor(f, device=dev), torch.tensor(u, device=dev)
    ref = torch.empty_like(ut)
    rmb.rm_relax(gctx, ft, ut, ref, 1.0)
    bounds = [w.nz * g // G for g in range(G + 1)]
    parts, ctxs, fl, ul = [], [], [], []
    for g in range(G):
        P = rmb.rm_partition(w.nx, w.ny, w.nz, w.p, 0, w.gamma_d, g, G, bounds[g], bounds[g + 1])
        ctx = gu.setup_product(w, rank=g, nranks=G, z_begin=bounds[g], z_end=bounds[g + 1])
        L, g0 = P["plane_len"], P["z_cell0"] * w.p * P["plane_len"]
        assert ctx.n_local == (P["nz_local"] * w.p + 1) * L
        own = slice(P["own_lo"] * L, P["own_hi"] * L)
        a = torch.full((ctx.n_local,), float("nan"), dtype=torch.float64, device=dev)
        b = a.clone()
        a[own] = ft[g0:g0 + ctx.n_local][own]
        b[own] = ut[g0:g0 + ctx.n_local][own]
        parts.append(P); ctxs.append(ctx); fl.append(a); ul.append(b)
    L = parts[0]["plane_len"]
    sl = lambda r: slice(r[0] * L, r[1] * L)   # noqa: E731
    for v in (fl, ul):   # forward halos (rank 0 <-> rank 1)
        v[1][sl(parts[1]["fwd_recv_lo"])] = v[0][sl(parts[0]["fwd_send_hi"])]
        v[0][sl(parts[0]["fwd_recv_hi"])] = v[1][sl(parts[1]["fwd_send_lo"])]
    assert all(torch.isfinite(t).all() for t in fl + ul)
    cs = [torch.empty_like(t) for t in ul]
    for g in range(G):
        rmb.rm_relax_begin(ctxs[g], fl[g], ul[g], cs[g])
    cs[0][sl(parts[0]["rev_recv_hi"])] += cs[1][sl(parts[1]["rev_send_lo"])]   # reverse-add
    for g in range(G):
        uo = torch.empty_like(ul[g])
        rmb.rm_relax_end(ctxs[g], ul[g], cs[g], uo, 1.0)
        P = parts[g]
        g0 = P["z_cell0"] * w.p * L
        own = slice(P["own_lo"] * L, P["own_hi"] * L)
        got = uo[own].cpu().numpy()
        want = ref[g0:g0 + ctxs[g].n_local][own].cpu().numpy()
        assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max()), (name, g)


@pytest.mark.gpu
@pytest.mark.parametrize("name,w", [("nce3-ph", dataclasses.replace(ri.CONFIGS[3].with_mesh(2).with_p(3), nz=4)),
                                    ("ncf3-ph", dataclasses.replace(ri.CONFIGS[4].with_mesh(2).with_p(3), nz=4))])
def test_slab_partition_two_contexts_hcurl_hdiv(dev, name, w):
    """H(curl) / H(div) z-slabs on one device: per-component halo planes (P family in z: the
    ranges of rm_partition, DP family: its dp_* ranges) moved by device copies between two
    contexts; owned planes equal the single-context sweep."""
    import torch
    import paper_2211_14284_b200 as rmb
    from oracle.fem import P_FAM, Space
    G = 2
    gctx = gu.setup_product(w)
    n = gctx.n_local
    mask = gctx.constrained_mask()
    f = ri.uniform_vector(w.cfg, 0, n); f[mask] = 0
    u = ri.uniform_vector(w.cfg, 3, n); u[mask] = 0
    ft, ut = torch.tensor(f, device=dev), torch.tensor(u, device=dev)
    ref = torch.empty_like(ut)
    rmb.rm_relax(gctx, ft, ut, ref, 1.0)
    gsp = Space(w.space, w.p, w.nx, w.ny, w.nz)
    bounds = [w.nz * g // G for g in range(G + 1)]
    parts, ctxs, views = [], [], []
    for g in range(G):
        P = rmb.rm_partition(w.nx, w.ny, w.nz, w.p, w.space, w.gamma_d, g, G, bounds[g], bounds[g + 1])
        ctx = gu.setup_product(w, rank=g, nranks=G, z_begin=bounds[g], z_end=bounds[g + 1])
        lsp = Space(w.space, w.p, w.nx, w.ny, P["nz_local"])
        assert ctx.n_local == lsp.ndof
        v = []
        go, lo = gsp.offsets(), lsp.offsets()
        for m in range(3):
            Lz, Ly, Lx = lsp.comp_shape(m)
            Lm = Ly * Lx
            v.append((go[m] + P["z_cell0"] * w.p * Lm, lo[m], Lz * Lm, Lm, lsp.fams[m][2] != P_FAM))
        parts.append(P); ctxs.append(ctx); views.append(v)
    key = lambda dp, k: ("dp_" if dp else "") + k   # noqa: E731
    fl, ul = [], []
    for g in range(G):
        a = torch.full((ctxs[g].n_local,), float("nan"), dtype=torch.float64, device=dev)
        b = a.clone()
        for g0, l0, ln, Lm, dp in views[g]:
            lo_, hi_ = parts[g][key(dp, "own_lo")], parts[g][key(dp, "own_hi")]
            a[l0 + lo_ * Lm:l0 + hi_ * Lm] = ft[g0 + lo_ * Lm:g0 + hi_ * Lm]
            b[l0 + lo_ * Lm:l0 + hi_ * Lm] = ut[g0 + lo_ * Lm:g0 + hi_ * Lm]
        fl.append(a); ul.append(b)
    P0, P1 = parts
    for vecs in (fl, ul):   # forward halos, per component
        for m in range(3):
            _, l00, _, Lm, dp = views[0][m]
            _, l10, _, _, _ = views[1][m]
            if dp:
                s0, r1 = P0["dp_fwd_send_hi"], P1["dp_fwd_recv_lo"]
                vecs[1][l10 + r1[0] * Lm:l10 + r1[1] * Lm] = vecs[0][l00 + s0[0] * Lm:l00 + s0[1] * Lm]
            else:
                s0, r1 = P0["fwd_send_hi"], P1["fwd_recv_lo"]
                vecs[1][l10 + r1[0] * Lm:l10 + r1[1] * Lm] = vecs[0][l00 + s0[0] * Lm:l00 + s0[1] * Lm]
                s1, r0 = P1["fwd_send_lo"], P0["fwd_recv_hi"]
                vecs[0][l00 + r0[0] * Lm:l00 + r0[1] * Lm] = vecs[1][l10 + s1[0] * Lm:l10 + s1[1] * Lm]
    assert all(torch.isfinite(t).all() for t in fl + ul)
    cs = [torch.empty_like(t) for t in ul]
    for g in range(G):
        rmb.rm_relax_begin(ctxs[g], fl[g], ul[g], cs[g])
    for m in range(3):   # reverse-add
        _, l00, _, Lm, dp = views[0][m]
        _, l10, _, _, _ = views[1][m]
        sl, rh = P1[key(dp, "rev_send_lo")], P0[key(dp, "rev_recv_hi")]
        cs[0][l00 + rh[0] * Lm:l00 + rh[1] * Lm] += cs[1][l10 + sl[0] * Lm:l10 + sl[1] * Lm]
    for g in range(G):
        uo = torch.empty_like(ul[g])
        rmb.rm_relax_end(ctxs[g], ul[g], cs[g], uo, 1.0)
        for g0, l0, ln, Lm, dp in views[g]:
            lo_, hi_ = parts[g][key(dp, "own_lo")], parts[g][key(dp, "own_hi")]
            got = uo[l0 + lo_ * Lm:l0 + hi_ * Lm].cpu().numpy()
            want = ref[g0 + lo_ * Lm:g0 + hi_ * Lm].cpu().numpy()
            err = np.abs(got - want).max() / max(1.0, np.abs(want).max())
            # H(div): the partitioned and single contexts run different patch kernels (class-batched vs
            # streamed, by family size), i.e. different summation orders on problems with
            # kappa ~ 1e5..4e6 -- the DESIGN.md section 7 derived H(div) tolerance applies
            check(f"slab two-context {name} rank {g} comp", err, hdiv_tol("2^3-p3") if w.space == 2 else 1e-12)


@pytest.mark.gpu
def test_nccl_transport_self_check(dev):
    """The NCCL entry points rm_relax uses with nranks > 1 (dlopen, unique id, communicator,
    grouped send/recv, allreduce on a stream), exercised on one device with a one-rank comm."""
    import paper_2211_14284_b200 as rmb
    rmb.rm_nccl_check(torch.cuda.current_device())
    assert len(rmb.rm_nccl_unique_id()) == 128


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [3, 4])
def test_full_size_hcurl_hdiv_sampled(dev, cfg):
    """BASELINE configs 3 and 4 at full size (24^3, p = 6 / 8) in the bench's launch configuration
    (cfg4's large windows take the one-box-buffer schedule): sweep outputs at sampled DoFs of every
    component near an interior vertex, each recomputed by the oracle from the primary and potential
    patches that reach it (oracle.solver.sampled_relax_ph, no global matrix)."""
    import paper_2211_14284_b200 as rmb
    from oracle.fem import Space
    from oracle.solver import sampled_relax_ph
    w = ri.CONFIGS[cfg]
    ctx = gu.setup_product(w)
    sp_ = Space(w.space, w.p, w.nx, w.ny, w.nz)
    f, u = vecs(w, ctx)
    out = torch.empty(ctx.n_local, dtype=torch.float64, device=dev)
    ft, ut = torch.tensor(f, device=dev), torch.tensor(u, device=dev)
    rmb.rm_relax(ctx, ft, ut, out, 1.0)
    # bitwise determinism at full size, where the colour launches of the class-batched kernel run
    # several waves and overlap as programmatic dependent launches (the next colour's CTAs start
    # under the previous colour's last wave and wait before their reduce-adds)
    out2 = torch.empty_like(out)
    for _ in range(3):
        rmb.rm_relax(ctx, ft, ut, out2, 1.0)
        assert torch.equal(out2, out)
    off = sp_.offsets()
    rows = []
    for m in range(3):
        Lz, Ly, Lx = sp_.comp_shape(m)
        x, y, z = 12 * w.p + 2, 11 * w.p + 1, 13 * w.p   # an interior vertex region (faces, edges, interiors)
        rows += [off[m] + ((z + dz) * Ly + y + dy) * Lx + x + dx for dx, dy, dz in ((0, 0, 0), (-2, 1, 0))]
    so = sampled_relax_ph(sp_, ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w), w.gamma_d, f, u, rows, 1.0)
    got = out.cpu().numpy()[rows]
    # tolerance: 10x the ORACLE's own noise floor at these rows (quadrature vs closed-form cell
    # matrices, identical in exact arithmetic: scripts/fullsize_noise_floor.py), floored at 1e-11;
    # at h = 1/24 the edge / face-star patch problems are ill-conditioned (stiffness / mass ~
    # p^4 / h^2), DESIGN.md §7
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fullsize_noise_floor.json")))["cases"]
    tol = max(1e-11, 10 * g[f"cfg{cfg}"]["oracle_vs_closed_form_assembly_maxabs_rel"])
    check(f"cfg{cfg} full size relax ({len(rows)} rows, max-abs rel)", float(np.abs(got - so).max() / np.abs(so).max()), tol)


# ------------------------------------------------------------------ p = 1 coarse level (f1)
COARSE_CASES = [
    ("cfg1", ri.CONFIGS[1], 1e-11),
    ("cfg2-3^3-p4", ri.CONFIGS[2].with_mesh(3).with_p(4), 1e-11),
    ("cfg3-2^3-p3", ri.CONFIGS[3].with_mesh(2).with_p(3), 1e-11),
    ("cfg4-2^3-p3", ri.CONFIGS[4].with_mesh(2).with_p(3), hdiv_tol("2^3-p3")),
    ("cfg5-3^3-p3", ri.CONFIGS[5].with_mesh(3).with_p(3), 1e-11),
]


@pytest.mark.parametrize("name,w,tol", COARSE_CASES, ids=[c[0] for c in COARSE_CASES])
def test_coarse_cycle_and_pcg(dev, name, w, tol):
    """rm_precondition with options.coarse = 1 is the hybrid V(1,1) cycle with the p = 1 coarse
    level (reading G20): equal to the oracle's cycle; rm_pcg iteration
    counts within +-1 of the oracle's."""
    import paper_2211_14284_b200 as rmb
    ctx = gu.setup_product(w, coarse=1)
    pb = gu.setup_oracle(w, coarse=True)
    info = ctx.info()
    assert info["coarse"] == 1 and info["coarse_ndof"] > 0
    f, _ = vecs(w, ctx)
    z = torch.empty(ctx.n_local, dtype=torch.float64, device=dev)
    rmb.rm_precondition(ctx, torch.tensor(f, device=dev), z)
    check(f"{name} coarse V(1,1) cycle", rel(z.cpu().numpy(), pb.cycle(f)), tol)
    x = torch.empty_like(z)
    it, relres, ok = rmb.rm_pcg(ctx, torch.tensor(f, device=dev), x, 1e-8, 200)
    _, ito, _ = pb.pcg(f)
    assert ok and relres <= 1e-8
    check(f"{name} coarse pcg iters {it} vs oracle {ito}", abs(it - ito), 1.5)


@pytest.mark.parametrize("cfg", [1, 2])
def test_coarse_p1_one_iteration(dev, cfg):
    """p = 1: the coarse space is the whole space; PCG with the cycle converges in one iteration
    (tab:hgrad-iter, p = 1, l = 0: "1/1")."""
    import paper_2211_14284_b200 as rmb
    w = ri.CONFIGS[cfg].with_mesh(4).with_p(1)
    ctx = gu.setup_product(w, coarse=1)
    f, _ = vecs(w, ctx)
    x = torch.empty(ctx.n_local, dtype=torch.float64, device=dev)
    it, relres, ok = rmb.rm_pcg(ctx, torch.tensor(f, device=dev), x, 1e-8, 50)
    assert ok and it == 1, (it, relres)


# ------------------------------------------------------------------ device-resident setup (f4)
DSETUP_CASES = [("cfg1", ri.CONFIGS[1], 1e-13), ("cfg2-3^3-p7", ri.CONFIGS[2].with_mesh(3), 1e-13),
                ("cfg3-2^3-p6", ri.CONFIGS[3].with_mesh(2), 1e-12), ("cfg4-2^3-p3", ri.CONFIGS[4].with_mesh(2).with_p(3), 1e-11),
                ("cfg5-2^3-p15", ri.CONFIGS[5].with_mesh(2), 1e-13), ("cfg5-3^3-p5", ri.CONFIGS[5].with_mesh(3).with_p(5), 1e-13),
                ("cfg3-pafw-2^3-p3", dataclasses.replace(ri.CONFIGS[3].with_mesh(2).with_p(3), decomposition="pafw"), 1e-12),
                ("cfg3-iccsc-3^3-p3", dataclasses.replace(ri.CONFIGS[3].with_mesh(3).with_p(3), factorization="icc_sc"), 1e-12),
                ("cfg5-sc-3^3-p3", dataclasses.replace(ri.CONFIGS[5].with_mesh(3).with_p(3), decomposition="sc-pafw"), 1e-13)]


@pytest.mark.parametrize("name,w,tol", DSETUP_CASES, ids=[c[0] for c in DSETUP_CASES])
def test_device_setup_matches_host_setup_and_oracle(dev, name, w, tol):
    """the numeric setup on the GPU (dsetup.cu) -- cell matrices incl. the trilinear
    auxiliary operator, patch assembly, block elimination, dense Cholesky / ICC-SC, static-
    condensation cell data, stream packing -- gives the sweep of the host setup to rounding (the
    interface elimination runs as one dense Cholesky; differences ~ kappa * eps) and the oracle's
    sweep within the north-star tolerance."""
    import paper_2211_14284_b200 as rmb
    cd = gu.setup_product(w, setup=rmb.RM_SETUP_DEVICE)
    ch = gu.setup_product(w, setup=rmb.RM_SETUP_HOST)
    assert cd.info()["setup_on_device"] == 1 and ch.info()["setup_on_device"] == 0
    f, u = vecs(w, cd)
    ft, ut = torch.tensor(f, device=dev), torch.tensor(u, device=dev)
    od, oh = torch.empty_like(ut), torch.empty_like(ut)
    rmb.rm_relax(cd, ft, ut, od, 1.0)
    rmb.rm_relax(ch, ft, ut, oh, 1.0)
    check(f"dsetup {name} device vs host setup", rel(od.cpu().numpy(), oh.cpu().numpy()), tol)
    pb = gu.setup_oracle(w)
    otol = hdiv_tol("2^3-p3") if w.space == 2 else 1e-11
    check(f"dsetup {name} device setup vs oracle", rel(od.cpu().numpy(), pb.relax(f, u)), otol)
