"""Quick GPU check: H(curl)/H(div) sweeps with more patches than CTAs vs the oracle (diagnostic)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import rm_inputs as ri
import paper_2211_14284_b200 as rmb
from gpu_util import setup_product, setup_oracle, rel
dev = torch.device("cuda")
for cfg, n, p, nbox1 in [(3, 6, 3, 0), (3, 6, 3, 1), (4, 5, 3, 0), (4, 5, 3, 1), (3, 4, 6, 0)]:
    if nbox1: os.environ["RM_NBOX1"] = "1"
    else: os.environ.pop("RM_NBOX1", None)
    w = ri.CONFIGS[cfg].with_mesh(n).with_p(p)
    ctx = setup_product(w); pb = setup_oracle(w)
    m = ctx.constrained_mask()
    f = ri.uniform_vector(cfg, 0, ctx.n_local); f[m] = 0
    u = ri.uniform_vector(cfg, 3, ctx.n_local); u[m] = 0
    out = torch.empty(ctx.n_local, dtype=torch.float64, device=dev)
    rmb.rm_relax(ctx, torch.tensor(f, device=dev), torch.tensor(u, device=dev), out, 1.0)
    ref = pb.relax(f, u)
    got = out.cpu().numpy()
    e = np.abs(got - ref)
    print(f"cfg{cfg} {n}^3 p={p} nbox1={nbox1}: rel L2 {rel(got, ref):.2e}  max-abs rel {e.max() / np.abs(ref).max():.2e} at {int(e.argmax())}", flush=True)
    # the preconditioner alone
    z = torch.empty_like(out)
    rmb.rm_precondition(ctx, torch.tensor(f, device=dev), z)
    print(f"   precondition rel L2 {rel(z.cpu().numpy(), pb.precondition(f)):.2e}", flush=True)
