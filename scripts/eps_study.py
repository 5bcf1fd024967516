import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import rm_inputs as ri
import paper_2211_14284_b200 as rmb
from gpu_util import setup_product, setup_oracle, rel
dev = torch.device('cuda')
for p, n in [(3, 2), (4, 3)]:
    w = ri.CONFIGS[4].with_mesh(n).with_p(p)
    for eps in [1e-6, 1e-4, 1e-3, 1e-2]:
        ctx = setup_product(w, potential_shift=eps)
        pb = setup_oracle(w, potential_shift=eps)
        m = ctx.constrained_mask()
        f = ri.uniform_vector(4, 0, ctx.n_local); f[m] = 0
        u = ri.uniform_vector(4, 3, ctx.n_local); u[m] = 0
        uo = torch.empty(ctx.n_local, dtype=torch.float64, device=dev)
        rmb.rm_relax(ctx, torch.tensor(f, device=dev), torch.tensor(u, device=dev), uo, 1.0)
        x = torch.empty_like(uo)
        it, rr, ok = rmb.rm_pcg(ctx, torch.tensor(f, device=dev), x)
        _, ito, _ = pb.pcg(f)
        print(f'p={p} n={n} eps={eps:g} relax rel {rel(uo.cpu().numpy(), pb.relax(f, u)):.2e} iters gpu {it} oracle {ito}', flush=True)
