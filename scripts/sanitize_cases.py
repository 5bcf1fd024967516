"""Small sweeps of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
H(grad) exact (cfg1), H(curl) PH (edge stars + potential), H(div) PH, trilinear ICC-SC, SC-PAFW,
the coarse V(1,1) cycle in PCG.  Exit code 0 = every call returned RM_OK."""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import paper_2211_14284_b200 as rmb  # noqa: E402
import rm_inputs as ri  # noqa: E402
from gpu_util import setup_product  # noqa: E402

dev = torch.device("cuda")
cases = [("cfg1", ri.CONFIGS[1], {}),
         ("cfg3-2^3-p3", ri.CONFIGS[3].with_mesh(2).with_p(3), {}),
         ("cfg4-2^3-p3", ri.CONFIGS[4].with_mesh(2).with_p(3), {}),
         ("cfg5-2^3-p3", ri.CONFIGS[5].with_mesh(2).with_p(3), {}),
         ("cfg1-sc", dataclasses.replace(ri.CONFIGS[1], decomposition="sc-pafw"), {}),
         ("cfg1-coarse", ri.CONFIGS[1].with_mesh(3), {"coarse": 1})]
only = sys.argv[1:]
for name, w, kw in cases:
    if only and name not in only:
        continue
    ctx = setup_product(w, **kw)
    m = ctx.constrained_mask()
    f = ri.uniform_vector(w.cfg, 0, ctx.n_local); f[m] = 0
    ft = torch.tensor(f, device=dev)
    u = torch.zeros_like(ft)
    rmb.rm_relax(ctx, ft, u, u, 1.0)
    v = torch.empty_like(u)
    rmb.rm_apply(ctx, u, v)
    if kw.get("coarse"):
        it, rel, ok = rmb.rm_pcg(ctx, ft, u, 1e-8, 50)
        print(name, "pcg", it, ok, flush=True)
    torch.cuda.synchronize()
    print(name, "ok", flush=True)
