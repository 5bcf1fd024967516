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
                       coords=coords, decomposition=rmb.RM_PH if w.decomposition == "ph" else rmb.RM_PAFW,
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


CASES = [
    ("cfg1", ri.CONFIGS[1], 1e-11),
    ("cfg2-3^3", ri.CONFIGS[2].with_mesh(3), 1e-11),
    ("cfg2-2x3x4-p4", ri.CONFIGS[2].with_mesh(2, 3, 4).with_p(4), 1e-11),
    ("cfg3-2^3-p3", ri.CONFIGS[3].with_mesh(2).with_p(3), 1e-11),
    ("cfg3-2^3-p6", ri.CONFIGS[3].with_mesh(2), 1e-11),
    ("cfg4-2^3-p3", ri.CONFIGS[4].with_mesh(2).with_p(3), 1e-10),
    ("cfg4-3^3-p4", ri.CONFIGS[4].with_mesh(3).with_p(4), 1e-10),
    # trilinear cells (perturbed vertices): true operator by quadrature, auxiliary-operator
    # patches with ICC on the static-condensation pattern (cfg5 shapes at reduced size)
    ("cfg5-3^3-p3", ri.CONFIGS[5].with_mesh(3).with_p(3), 1e-11),
    ("cfg5-2^3-p7", ri.CONFIGS[5].with_mesh(2).with_p(7), 1e-11),
]


@pytest.mark.parametrize("name,w,tol", CASES, ids=[c[0] for c in CASES])
def test_apply_and_sweep_parity(dev, name, w, tol):
    import paper_2211_14284_b200 as rmb
    ctx, pb = setup_pair(w)
    assert (ctx.constrained_mask() == pb.constrained).all()
    assert ctx.n_free == int(pb.free.sum())
    f, u = vecs(w, ctx)
    ft, ut = torch.tensor(f, device=dev), torch.tensor(u, device=dev)
    v = torch.empty_like(ut)
    rmb.rm_apply(ctx, ut, v)
    assert rel(v.cpu().numpy(), pb.apply(u)) < 1e-11
    rmb.rm_residual(ctx, ft, ut, v)
    assert rel(v.cpu().numpy(), pb.residual(f, u)) < 1e-11
    out = torch.empty_like(ut)
    for omega in (1.0, 0.7):
        rmb.rm_relax(ctx, ft, ut, out, omega)
        assert rel(out.cpu().numpy(), pb.relax(f, u, omega)) < tol
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
                                    ("cfg5-3^3-p3", ri.CONFIGS[5].with_mesh(3).with_p(3))])
def test_pcg_iterations(dev, name, w):
    import paper_2211_14284_b200 as rmb
    ctx, pb = setup_pair(w)
    f, _ = vecs(w, ctx)
    x = torch.empty(ctx.n_local, dtype=torch.float64, device=dev)
    it, relres, ok = rmb.rm_pcg(ctx, torch.tensor(f, device=dev), x, 1e-8, 500)
    xo, ito, _ = pb.pcg(f)
    assert ok and relres <= 1e-8
    assert abs(it - ito) <= 1
    assert rel(x.cpu().numpy(), xo) < 1e-7


def test_precondition_and_host_entry_points(dev):
    import paper_2211_14284_b200 as rmb
    w = ri.CONFIGS[1]
    ctx, pb = setup_pair(w)
    f, u = vecs(w, ctx)
    z = torch.empty(ctx.n_local, dtype=torch.float64, device=dev)
    rmb.rm_precondition(ctx, torch.tensor(f, device=dev), z)
    assert rel(z.cpu().numpy(), pb.precondition(f)) < 1e-11
    out = np.empty_like(u)
    rmb.rm_relax_host(ctx, f, u, out, 1.0)
    assert rel(out, pb.relax(f, u)) < 1e-11


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
    outputs sampled at interior, face, edge and vertex DoFs, each recomputed by the oracle from
    the cells / patches that carry it."""
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
    idx = lambda x, y, z: (z * L + y) * L + x
    rows = [idx(100, 101, 102), idx(105, 101, 102), idx(105, 105, 102), idx(105, 105, 105), idx(224, 3, 8), idx(1, 224, 224)]
    v = torch.empty_like(ut)
    rmb.rm_apply(ctx, ut, v)
    vo = cell_rows_apply(sp, X, al, be, np.where(ctx.constrained_mask(), 0.0, u), rows)
    np.testing.assert_allclose(v.cpu().numpy()[rows], vo, rtol=1e-12, atol=1e-12 * np.abs(vo).max())
    out = torch.empty_like(ut)
    rmb.rm_relax(ctx, ft, ut, out, 1.0)
    so = sampled_relax(sp, X, al, be, w.gamma_d, f, u, rows[:4])
    got = out.cpu().numpy()[rows[:4]]
    assert np.abs(got - so).max() < 1e-11 * np.abs(so).max()


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
    assert rel(v.cpu().numpy(), ref) < 1e-11


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
def test_nccl_transport_self_check(dev):
    """The NCCL entry points rm_relax uses with nranks > 1 (dlopen, unique id, communicator,
    grouped send/recv, allreduce on a stream), exercised on one device with a one-rank comm."""
    import paper_2211_14284_b200 as rmb
    rmb.rm_nccl_check(torch.cuda.current_device())
    assert len(rmb.rm_nccl_unique_id()) == 128


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [3, 4])
def test_full_size_hcurl_hdiv_configs_sweep(dev, cfg):
    """BASELINE configs 3 and 4 at full size (24^3, p = 6 / 8): the patch plans fit (cfg4's ~95 KB
    window boxes run with one box buffer and the sequential schedule) and a sweep is finite and
    non-trivial.  (Parity of these paths is tested on the small shapes above, also with
    RM_NBOX1=1 forcing the one-buffer schedule.)"""
    import paper_2211_14284_b200 as rmb
    w = ri.CONFIGS[cfg]
    ctx = gu.setup_product(w)
    n = ctx.n_local
    mask = ctx.constrained_mask()
    f = ri.uniform_vector(w.cfg, 0, n); f[mask] = 0
    ft = torch.tensor(f, device=dev)
    u = torch.zeros_like(ft)
    rmb.rm_relax(ctx, ft, u, u, 1.0)
    uh = u.cpu().numpy()
    assert np.isfinite(uh).all() and np.abs(uh).max() > 0
    assert np.abs(uh[mask]).max() == 0.0
