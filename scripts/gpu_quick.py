import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import rm_inputs as ri
import paper_2211_14284_b200 as rmb
from gpu_util import setup_product, setup_oracle, rel
dev = torch.device('cuda')
for name, w, kw in [('cfg1', ri.CONFIGS[1], {}), ('cfg2-3^3', ri.CONFIGS[2].with_mesh(3), {}),
                    ('cfg3-2^3p3', ri.CONFIGS[3].with_mesh(2).with_p(3), {}), ('cfg4-2^3p3', ri.CONFIGS[4].with_mesh(2).with_p(3), {})]:
    t = time.time()
    ctx = setup_product(w)
    pb = setup_oracle(w)
    n = ctx.n_local
    mask = ctx.constrained_mask()
    print(name, 'n', n, 'mask ok', bool((mask == pb.constrained).all()), 'info', ctx.info())
    f = ri.uniform_vector(w.cfg, 0, n); f[mask] = 0
    u = ri.uniform_vector(w.cfg, 3, n); u[mask] = 0
    ft = torch.tensor(f, device=dev); ut = torch.tensor(u, device=dev); vt = torch.empty_like(ut)
    rmb.rm_apply(ctx, ut, vt); torch.cuda.synchronize()
    print('  apply rel', rel(vt.cpu().numpy(), pb.apply(u)))
    uo = torch.empty_like(ut)
    rmb.rm_relax(ctx, ft, ut, uo, 1.0); torch.cuda.synchronize()
    print('  relax rel', rel(uo.cpu().numpy(), pb.relax(f, u)))
    x = torch.empty_like(ut)
    it, rr, ok = rmb.rm_pcg(ctx, ft, x, 1e-8, 500)
    _, ito, _ = pb.pcg(f)
    print('  pcg', it, rr, ok, 'oracle', ito, 'time', time.time() - t)
