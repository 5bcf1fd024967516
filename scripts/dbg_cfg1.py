import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import rm_inputs as ri
import paper_2211_14284_b200 as rmb
from gpu_util import setup_product, setup_oracle, rel
w = ri.CONFIGS[1]
ctx = setup_product(w)
n = ctx.n_local
mask = ctx.constrained_mask()
f = ri.uniform_vector(w.cfg, 0, n); f[mask] = 0
u = ri.uniform_vector(w.cfg, 3, n); u[mask] = 0
dev = torch.device('cuda')
ft = torch.tensor(f, device=dev); ut = torch.tensor(u, device=dev); uo = torch.empty_like(ut)
rmb.rm_relax(ctx, ft, ut, uo, 1.0); torch.cuda.synchronize()
pb = setup_oracle(w)
print('relax rel', rel(uo.cpu().numpy(), pb.relax(f, u)))
