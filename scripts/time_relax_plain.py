"""Time rm_relax WITHOUT the library's per-kernel timing events (bench.py keeps them on inside its
timed region for the roofline): python scripts/time_relax_plain.py CFG [steps]."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import rm_inputs as ri
import paper_2211_14284_b200 as rmb
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import gpu_util as gu

cfg = int(sys.argv[1]); steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = ri.CONFIGS[cfg]
ctx = gu.setup_product(w)
dev = torch.device("cuda", 0)
n = ctx.n_local
mask = ctx.constrained_mask()
f = ri.uniform_vector(w.cfg, 0, n); f[mask] = 0
u = ri.uniform_vector(w.cfg, 3, n); u[mask] = 0
ft, ut = torch.tensor(f, device=dev), torch.tensor(u, device=dev)
uo = torch.empty_like(ut)
for _ in range(3):
    rmb.rm_relax(ctx, ft, ut, uo, 1.0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    rmb.rm_relax(ctx, ft, ut, uo, 1.0)
e1.record()
torch.cuda.synchronize()
print(f"cfg{cfg} plain rm_relax: {e0.elapsed_time(e1) / steps:.3f} ms per sweep ({steps} sweeps, no library timing events)")
