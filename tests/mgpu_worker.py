"""Worker of tests/test_multigpu.py (one process per GPU under torch.distributed.run).

Every rank sets up (a) the single-domain problem on its own GPU and (b) its z-slab of the same
global problem with an NCCL communicator (options.nccl_id: halos, reverse-add and PCG allreduces
inside the library), then checks that the owned planes of rm_apply / rm_relax / rm_precondition /
rm_pcg equal the single-domain results (SURVEY 8(e) partition invariance)."""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2211_14284_b200 as rmb  # noqa: E402
import rm_inputs as ri  # noqa: E402


def setup(w, **kw):
    coords = None if w.perturb == 0 else ri.vertex_coords(w)
    return rmb.rm_setup(w.nx, w.ny, w.nz, w.p, w.space, ri.cell_alpha(w).ravel(), ri.cell_beta(w).ravel(), w.gamma_d,
                        coords=coords, factorization=rmb.RM_ICC_SC if w.factorization == "icc_sc" else rmb.RM_CHOL,
                        decomposition=rmb.RM_PH if w.decomposition == "ph" else rmb.RM_PAFW,
                        device=torch.cuda.current_device(), **kw)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    dev = torch.device("cuda", torch.cuda.current_device())
    cases = [dataclasses.replace(ri.CONFIGS[1].with_mesh(3), nz=2 * world),
             dataclasses.replace(ri.CONFIGS[2].with_mesh(3).with_p(4), nz=2 * world),
             dataclasses.replace(ri.CONFIGS[5].with_mesh(3).with_p(3), nz=2 * world),
             dataclasses.replace(ri.CONFIGS[3].with_mesh(2).with_p(3), nz=2 * world),
             dataclasses.replace(ri.CONFIGS[4].with_mesh(2).with_p(3), nz=2 * world)]
    bad = 0
    for w in cases:
        g = setup(w)
        n, mask = g.n_local, g.constrained_mask()
        f = ri.uniform_vector(w.cfg, 0, n); f[mask] = 0
        u = ri.uniform_vector(w.cfg, 3, n); u[mask] = 0
        ft, ut = torch.tensor(f, device=dev), torch.tensor(u, device=dev)
        ref_relax, ref_apply, ref_z = torch.empty_like(ut), torch.empty_like(ut), torch.empty_like(ut)
        rmb.rm_relax(g, ft, ut, ref_relax, 0.8)
        rmb.rm_apply(g, ut, ref_apply)
        rmb.rm_precondition(g, ft, ref_z)
        ref_x = torch.empty_like(ut)
        it_ref, _, _ = rmb.rm_pcg(g, ft, ref_x, 1e-8, 300)
        zb, ze = w.nz * rank // world, w.nz * (rank + 1) // world
        P = rmb.rm_partition(w.nx, w.ny, w.nz, w.p, w.space, w.gamma_d, rank, world, zb, ze)
        nid = [rmb.rm_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        ctx = setup(w, rank=rank, nranks=world, z_begin=zb, z_end=ze, nccl_id=nid[0])
        assert ctx.info()["comm_nranks"] == world
        from oracle.fem import P_FAM, Space
        gsp, lsp = Space(w.space, w.p, w.nx, w.ny, w.nz), Space(w.space, w.p, w.nx, w.ny, P["nz_local"])
        comps = []
        for m in range(len(lsp.fams)):
            Lz, Ly, Lx = lsp.comp_shape(m)
            dp = lsp.fams[m][2] != P_FAM
            comps.append((gsp.offsets()[m] + P["z_cell0"] * w.p * Ly * Lx, lsp.offsets()[m], Lz * Ly * Lx, Ly * Lx,
                          P["dp_own_lo" if dp else "own_lo"], P["dp_own_hi" if dp else "own_hi"]))

        def loc(t):   # the local planes of a global vector (halo planes overwritten in place by the call)
            return torch.cat([t[g0:g0 + ln] for g0, l0, ln, Lm, lo, hi in comps]).clone()

        def owned(t):
            return torch.cat([t[l0 + lo * Lm:l0 + hi * Lm] for g0, l0, ln, Lm, lo, hi in comps])
        out = torch.empty(ctx.n_local, dtype=torch.float64, device=dev)
        res = {}
        rmb.rm_relax(ctx, loc(ft), loc(ut), out, 0.8)
        res["relax"] = (owned(out), owned(loc(ref_relax)))
        out2 = torch.empty_like(out)
        rmb.rm_apply(ctx, loc(ut), out2)
        res["apply"] = (owned(out2), owned(loc(ref_apply)))
        out3 = torch.empty_like(out)
        rmb.rm_precondition(ctx, loc(ft), out3)
        res["precondition"] = (owned(out3), owned(loc(ref_z)))
        x = torch.empty_like(out)
        it, _, _ = rmb.rm_pcg(ctx, loc(ft), x, 1e-8, 300)
        res["pcg"] = (owned(x), owned(loc(ref_x)))
        for k, (a, b) in res.items():
            e = float((a - b).abs().max() / b.abs().max())
            tol = 1e-12 if k != "pcg" else 1e-7
            ok = e <= tol
            bad += not ok
            print(f"[rank {rank}] cfg{w.cfg} p={w.p} {k}: max-abs rel {e:.2e} (tol {tol:.0e}) {'ok' if ok else 'FAIL'}", flush=True)
        ok = abs(it - it_ref) <= 1
        bad += not ok
        print(f"[rank {rank}] cfg{w.cfg} pcg iterations {it} vs single-domain {it_ref} {'ok' if ok else 'FAIL'}", flush=True)
        ctx.close()
        g.close()
    t = torch.tensor([bad], device=dev)
    dist.all_reduce(t)
    dist.destroy_process_group()
    sys.exit(1 if int(t.item()) else 0)


if __name__ == "__main__":
    main()
