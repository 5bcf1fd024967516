import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import rm_inputs as ri
import paper_2211_14284_b200 as rmb
from gpu_util import setup_product, setup_oracle, rel
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = ri.CONFIGS[2].with_mesh(n)
ctx = setup_product(w)
print(ctx.info(), flush=True)
m = ctx.constrained_mask()
f = ri.uniform_vector(2, 0, ctx.n_local); f[m] = 0
u = ri.uniform_vector(2, 3, ctx.n_local); u[m] = 0
dev = torch.device('cuda')
uo = torch.empty(ctx.n_local, dtype=torch.float64, device=dev)
rmb.rm_relax(ctx, torch.tensor(f, device=dev), torch.tensor(u, device=dev), uo, 1.0)
torch.cuda.synchronize()
pb = setup_oracle(w)
print('relax rel', rel(uo.cpu().numpy(), pb.relax(f, u)), flush=True)
