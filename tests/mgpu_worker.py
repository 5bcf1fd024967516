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
                        device=torch.cuda.current_device(), **kw)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    dev = torch.device("cuda", torch.cuda.current_device())
    cases = [dataclasses.replace(ri.CONFIGS[1].with_mesh(3), nz=2 * world),
             dataclasses.replace(ri.CONFIGS[2].with_mesh(3).with_p(4), nz=2 * world),
             dataclasses.replace(ri.CONFIGS[5].with_mesh(3).with_p(3), nz=2 * world)]
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
        P = rmb.rm_partition(w.nx, w.ny, w.nz, w.p, 0, w.gamma_d, rank, world, zb, ze)
        nid = [rmb.rm_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        ctx = setup(w, rank=rank, nranks=world, z_begin=zb, z_end=ze, nccl_id=nid[0])
        assert ctx.info()["comm_nranks"] == world
        L = P["plane_len"]
        g0 = P["z_cell0"] * w.p * L
        own = slice(P["own_lo"] * L, P["own_hi"] * L)
        loc = lambda t: t[g0:g0 + ctx.n_local].clone()   # noqa: E731  (halo planes overwritten in place)
        out = torch.empty(ctx.n_local, dtype=torch.float64, device=dev)
        res = {}
        rmb.rm_relax(ctx, loc(ft), loc(ut), out, 0.8)
        res["relax"] = (out[own], loc(ref_relax)[own])
        out2 = torch.empty_like(out)
        rmb.rm_apply(ctx, loc(ut), out2)
        res["apply"] = (out2[own], loc(ref_apply)[own])
        out3 = torch.empty_like(out)
        rmb.rm_precondition(ctx, loc(ft), out3)
        res["precondition"] = (out3[own], loc(ref_z)[own])
        x = torch.empty_like(out)
        it, _, _ = rmb.rm_pcg(ctx, loc(ft), x, 1e-8, 300)
        res["pcg"] = (x[own], loc(ref_x)[own])
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
