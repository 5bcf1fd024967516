"""SC-PH product vs oracle, stage by stage (debug; GPU)."""
import dataclasses, sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np, torch
import rm_inputs as ri
import gpu_util as gu
import paper_2211_14284_b200 as rmb
from oracle.solver import interior_mask

w = dataclasses.replace(ri.CONFIGS[3].with_mesh(2).with_p(3), decomposition="sc-ph")
ctx = gu.setup_product(w)
pb = gu.setup_oracle(w)
A, I, G, AIIinv, S, prim, Dt, pot = pb.sc_ph_data()
n = ctx.n_local
dev = torch.device("cuda", 0)
def prod(r):
    z = torch.empty(n, dtype=torch.float64, device=dev)
    rmb.rm_precondition(ctx, torch.tensor(r, device=dev), z)
    return z.cpu().numpy()
def orac(r, pot_stage=True):
    return pb.precondition_sc_ph(r, potential_stage=pot_stage)
rng = np.random.default_rng(0)
for name, sel in (("interior-only r", I), ("interface-only r", G)):
    r = np.zeros(n); r[sel] = rng.uniform(-1, 1, len(sel))
    zp, zo = prod(r), orac(r)
    zo_np = orac(r, False)
    for part, idx in (("G", G), ("I", I)):
        print(name, part, "prod-oracle", np.abs(zp[idx] - zo[idx]).max() / np.abs(zo[idx]).max(),
              "| prod-oracle(no pot)", np.abs(zp[idx] - zo_np[idx]).max() / np.abs(zo_np[idx]).max())
# y = A_II^-1 r_I check via interior-only r with no patches: c_I for r interior-only when c_G = 0?
