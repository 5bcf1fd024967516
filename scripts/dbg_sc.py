# debug: GPU preconditioner vs host emulator for an ICC-SC family, split interior / interface DoFs
import sys, ctypes, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo/tests/native')
import rm_inputs as ri
import paper_2211_14284_b200 as rmb
import build_emu
import os
w = ri.CONFIGS[5].with_mesh(3).with_p(3)
cart = os.environ.get("CART") == "1"
if cart:
    from dataclasses import replace
    w = replace(w, perturb=0.0)
ctx = rmb.rm_setup(w.nx, w.ny, w.nz, w.p, w.space, ri.cell_alpha(w).ravel(), ri.cell_beta(w).ravel(), w.gamma_d,
                   coords=None if cart else ri.vertex_coords(w), factorization=rmb.RM_ICC_SC)
n = ctx.n_local; m = ctx.constrained_mask()
r = ri.uniform_vector(w.cfg, 0, n); r[m] = 0
z = torch.empty(n, dtype=torch.float64, device='cuda')
rmb.rm_precondition(ctx, torch.tensor(r, device='cuda'), z)
zg = z.cpu().numpy()
lib = ctypes.CDLL(build_emu.build())
D = ctypes.POINTER(ctypes.c_double)
dp = lambda a: a.ctypes.data_as(D)
al = np.ascontiguousarray(ri.cell_alpha(w).ravel()); be = np.ascontiguousarray(ri.cell_beta(w).ravel())
X = np.ascontiguousarray(ri.vertex_coords(w).ravel())
ze = np.zeros(n); err = ctypes.create_string_buffer(256); st = (ctypes.c_longlong * 6)()
lib.emu_precondition.argtypes = [ctypes.c_int] * 5 + [ctypes.c_uint, D, ctypes.c_longlong, D, ctypes.c_longlong, D,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_int, D, D, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_longlong)]
rc = lib.emu_precondition(0, w.p, w.nx, w.ny, w.nz, w.gamma_d, dp(al), al.size, dp(be), be.size, None if cart else dp(X), 0, 1, 0, dp(r), dp(ze), err, 256, st)
L = w.nx * w.p + 1
idx = np.arange(n); x = idx % L; y = (idx // L) % L; zz = idx // (L * L)
inter = (x % w.p != 0) & (y % w.p != 0) & (zz % w.p != 0)
xp = (x % w.p == 0); yp = (y % w.p == 0) & ~xp; zp = (zz % w.p == 0) & ~xp & ~(y % w.p == 0)
for name, sel in [('interior', inter), ('interface', ~inter), ('x-planes', xp), ('y-planes(not x)', yp), ('z-planes(only)', zp)]:
    d = np.abs(zg[sel] - ze[sel]).max(); print(name, 'max abs diff', d, 'max |ze|', np.abs(ze[sel]).max())
bad = np.argsort(-np.abs(zg - ze))[:8]
for b in bad: print('dof', b, (x[b], y[b], zz[b]), 'gpu', zg[b], 'emu', ze[b])
if os.environ.get("RM_DEBUG_SC_PRE") or os.environ.get("RM_DEBUG_Q") == "2":
    lib.emu_sc_pre.argtypes = [ctypes.c_int] * 4 + [ctypes.c_uint, D, ctypes.c_longlong, D, ctypes.c_longlong, D, D, D]
    rs = np.zeros(n)
    lib.emu_sc_pre(w.p, w.nx, w.ny, w.nz, w.gamma_d, dp(al), al.size, dp(be), be.size, None if cart else dp(X), dp(r), dp(rs))
    d = np.abs(zg - rs); d[m] = 0
    print('SC pre: max diff (meaningful only with RM_DEBUG_SC_PRE)', d.max())
    for b in np.argsort(-d)[:5]: print('  dof', b, (x[b], y[b], zz[b]), 'gpu', zg[b], 'emu', rs[b], 'r', r[b])
if os.environ.get("RM_DEBUG_Q"):
    # compare every finished patch box: GPU dump (librm rm_debug_box) vs emulator dump (RM_DEBUG_EMU_PATCH file)
    rl = ctypes.CDLL(rmb.LIB_PATH)
    buf = np.zeros(1 << 22)
    rl.rm_debug_box.argtypes = [D, ctypes.c_int]
    print('dump rc', rl.rm_debug_box(dp(buf), buf.size))
    recs = [l.split() for l in open(os.environ["RM_DEBUG_EMU_PATCH"])]
    bt = len(recs[0]) - 9
    dev = buf[:(len(recs)) * (bt + 9)].reshape(len(recs), bt + 9)
    key = {tuple(int(v) for v in dev[q, :9]): q for q in range(len(recs))}
    nbad = 0
    for rec in recs:
        po = tuple(int(v) for v in rec[:9]); e = np.array([float(v) for v in rec[9:]])
        q = key.get(po)
        if q is None: print('no device patch for', po); continue
        d = np.abs(dev[q, 9:] - e)
        if d.max() > 1e-10:
            nbad += 1
            if nbad <= 6:
                bad = np.nonzero(d > 1e-10)[0]
                print('patch', po, 'q', q, 'bad box idx', bad[:20].tolist(), 'dev', dev[q, 9 + bad[:4]], 'emu', e[bad[:4]])
    print('bad patches', nbad, 'of', len(recs), 'box_total', bt)
if os.environ.get("RM_DEBUG_Q") == "2":
    # loaded boxes vs the emulator's condensed residual (RM_DEBUG_SC_PRE must be set too)
    import ctypes as C2
    box = np.array(rmb_box := None) if False else None
    Ls = L
    bx = [(2, 5, 5), (6, 1, 5), (6, 5, 1)]
    nb = 0
    for q in range(dev.shape[0] // 2 if False else 64):
        po = [int(v) for v in dev[q, :9]]
        off = 0; offs = [0, 64, 96]
        for m in range(3):
            o = po[3 * m:3 * m + 3]; X, Y, Z = bx[m]
            for z_ in range(Z):
                for y_ in range(Y):
                    for x_ in range(X):
                        g = (o[0] + x_, o[1] + y_, o[2] + z_)
                        want = rs[g[0] + Ls * (g[1] + Ls * g[2])] if all(0 <= c < Ls for c in g) else 0.0
                        got = dev[q, 9 + offs[m] + x_ + X * (y_ + Y * z_)]
                        if abs(got - want) > 1e-12:
                            nb += 1
                            if nb < 10: print('load mismatch q', q, po, 'sub', m, (x_, y_, z_), 'got', got, 'want', want)
    print('load mismatches', nb)
if os.environ.get("RM_DEBUG_Q") == "3":
    for q in range(64):
        po = [int(v) for v in dev[q, :9]]
        if po[:3] in ([6, 7, 7], [2, 7, 7], [6, 4, 4]):
            nrec = int(dev[q, 9]); print('patch', po, 'icc pieces', nrec)
            for j in range(min(nrec, 14)): print('   ', dev[q, 10 + 8 * j: 18 + 8 * j])
