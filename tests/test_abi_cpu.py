"""CPU-side checks of the product: the C-ABI library loads and exports every symbol that
include/rm.h declares (no compute calls -- there is no GPU here), and the product's host setup
(FDM basis, Kronecker term lists, patch classes, elimination programs, ICC-SC, packing) re-enacted
on the host by tests/native/emu.cpp agrees with the oracle."""
import ctypes
import os
import re
import sys

import numpy as np
import pytest

import rm_inputs as ri

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "rm.h")


def header_functions():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:rm_status|void|const char \*)\s*(rm_\w+)\s*\(", src, re.M)))


def test_header_declares_the_boundary():
    fns = header_functions()
    for f in ("rm_setup", "rm_apply", "rm_relax", "rm_pcg", "rm_destroy", "rm_layout", "rm_last_error"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    from paper_2211_14284_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    for f in header_functions():
        assert hasattr(lib, f), f
    # the binding loads the same in-tree library
    import paper_2211_14284_b200 as rmb
    assert os.path.samefile(rmb.LIB_PATH, lib_path)
    assert rmb.exported_symbols() == header_functions()


def test_library_is_sm100a_only():
    from paper_2211_14284_b200 import build
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", build.build()], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass      # TMA bulk copies feed the dense patch phase


def test_setup_errors_without_gpu_are_reported_not_raised():
    import paper_2211_14284_b200 as rmb
    with pytest.raises(rmb.RmError):
        rmb.rm_setup(2, 2, 2, 0, 0, [1.0], [1.0], 63)          # p = 0 is invalid
    with pytest.raises(rmb.RmError):
        rmb.rm_setup(2, 2, 2, 3, 0, [1.0, 2.0], [1.0], 63)     # alpha size neither 1 nor ncells
    with pytest.raises(rmb.RmError):
        rmb.rm_setup(2, 2, 2, 3, 0, [1.0], [1.0], 63, decomposition=rmb.RM_SC_PH)   # SC-PH is k = 1, 2


# ------------------------------------------------------------------ host re-enactment vs oracle
@pytest.fixture(scope="module")
def emu():
    sys.path.insert(0, os.path.join(ROOT, "tests", "native"))
    import build_emu
    lib = ctypes.CDLL(build_emu.build())
    D = ctypes.POINTER(ctypes.c_double)
    lib.emu_precondition.argtypes = [ctypes.c_int] * 5 + [ctypes.c_uint, D, ctypes.c_longlong, D, ctypes.c_longlong, D,
                                                          ctypes.c_int, ctypes.c_int, ctypes.c_int, D, D, ctypes.c_char_p,
                                                          ctypes.c_int, ctypes.POINTER(ctypes.c_longlong)]
    lib.emu_basis.argtypes = [ctypes.c_int] + [D] * 6
    return lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


@pytest.mark.parametrize("p", [2, 3, 7, 15])
def test_product_basis_matches_oracle(emu, p):
    from oracle.basis1d import fdm_basis
    n = p + 1
    S, lam, B, A, D, G = (np.zeros(n * n), np.zeros(n), np.zeros(n * n), np.zeros(n * n), np.zeros(p * n), np.zeros(n * n))
    emu.emu_basis(p, _dp(S), _dp(lam), _dp(B), _dp(A), _dp(D), _dp(G))
    f = fdm_basis(p)
    np.testing.assert_allclose(S.reshape(n, n), f.S, atol=1e-12)
    np.testing.assert_allclose(lam[1:p], f.lam[1:p], rtol=1e-12)
    np.testing.assert_allclose(D.reshape(p, n), f.D, atol=1e-11 * max(1, np.sqrt(f.lam[1:p].max() if p > 1 else 1)))
    np.testing.assert_allclose(G.reshape(n, n), f.G, atol=1e-14)


CASES = [
    ("cfg1", ri.CONFIGS[1], 0, 0, 0),
    ("cfg2-3^3p4", ri.CONFIGS[2].with_mesh(3).with_p(4), 0, 0, 0),
    ("cfg1-2^3-interior", ri.CONFIGS[1].with_mesh(2), 0, 0, 1),
    ("cfg3-edge-2^3p3", ri.CONFIGS[3].with_mesh(2).with_p(3), 1, 0, 0),
    ("cfg4-face-2^3p3", ri.CONFIGS[4].with_mesh(2).with_p(3), 2, 0, 0),
    ("cfg3-vertex-2^3p3", ri.CONFIGS[3].with_mesh(2).with_p(3), 0, 0, 0),
    ("cfg5-icc-2^3p3", ri.CONFIGS[5].with_mesh(2).with_p(3), 0, 1, 0),
    ("cfg5-icc-3^3p5", ri.CONFIGS[5].with_mesh(3).with_p(5), 0, 1, 0),   # levels wider than one 32-row piece
]


@pytest.mark.parametrize("name,w,dim,fact,interior", CASES, ids=[c[0] for c in CASES])
def test_product_patch_programs_match_oracle(emu, name, w, dim, fact, interior):
    from oracle.solver import Problem
    pb = Problem(w.space, w.p, w.nx, w.ny, w.nz, ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w), w.gamma_d,
                 decomposition="pafw" if dim == 0 else "ph", factorization="icc_sc" if fact else "chol",
                 interior_only=bool(interior))
    nd = pb.space.ndof
    r = ri.uniform_vector(w.cfg, 0, nd)
    r[pb.constrained] = 0
    al = np.ascontiguousarray(ri.cell_alpha(w).ravel())
    be = np.ascontiguousarray(ri.cell_beta(w).ravel())
    coords = None if w.perturb == 0 else np.ascontiguousarray(ri.vertex_coords(w).ravel())
    z = np.zeros(nd)
    err = ctypes.create_string_buffer(256)
    st = (ctypes.c_longlong * 6)()
    rc = emu.emu_precondition(w.space, w.p, w.nx, w.ny, w.nz, w.gamma_d, _dp(al), al.size, _dp(be), be.size,
                              None if coords is None else _dp(coords), dim, fact, interior, _dp(r), _dp(z), err, 256, st)
    assert rc == 0, err.value
    zo = np.zeros(nd)
    for g, S in pb.patch_solvers():
        zo[g] += S.solve(r[g])
    tol = 1e-11
    if w.space == 2:   # H(div): 10x the oracle's own assembly noise (tests/golden/cfg4_conditioning.json)
        import json
        g = json.load(open(os.path.join(ROOT, "tests", "golden", "cfg4_conditioning.json")))["cases"]
        tol = max(1e-11, 10 * g[f"{w.nx}^3-p{w.p}"]["oracle_vs_closed_form_assembly_sweep_rel"])
    assert np.linalg.norm(z - zo) / np.linalg.norm(zo) < tol


# ------------------------------------------------------------ algorithmic factor size (rm_info)
@pytest.mark.parametrize("name,k,p,n,gamma,dim,fact,interior,total,largest", [
    # SURVEY 8(a) rows a5/a6 [V]: cfg1 sum of nnz(L) = 51,121; a full cfg2 vertex patch (Q7,
    # (2p-1)^3 = 2197 DoFs) 70,183; a full cfg5 ICC-SC mask (Q15, 24,389 DoFs) 160,889
    ("cfg1", 0, 3, 4, 63, 0, 0, 0, 51121, None),
    ("cfg2-full-patch", 0, 7, 2, 0, 0, 0, 1, 70183, 70183),
    ("cfg5-full-patch-iccsc", 0, 15, 2, 0, 0, 1, 1, 160889, 160889),
])
def test_algorithmic_factor_nnz_matches_survey(emu, name, k, p, n, gamma, dim, fact, interior, total, largest):
    """The roofline's algorithmic bytes (bench.py) count nnz(L) of the exact Cholesky factor in
    the pinned order (reading G6), or of the ICC-SC mask, per patch -- not the product's stored
    format.  Checked against the counts SURVEY.md 8(a) verified independently."""
    emu.emu_family_nnz.argtypes = [ctypes.c_int] * 5 + [ctypes.c_uint] + [ctypes.c_int] * 3 + [
        ctypes.POINTER(ctypes.c_longlong), ctypes.c_char_p, ctypes.c_int]
    out = (ctypes.c_longlong * 3)()
    err = ctypes.create_string_buffer(256)
    assert emu.emu_family_nnz(k, p, n, n, n, gamma, dim, fact, interior, out, err, 256) == 0, err.value
    assert out[0] == total
    if largest is not None:
        assert out[2] == largest


# ------------------------------------------------------------ p = 1 coarse level (host factor)
@pytest.mark.parametrize("name,w", [
    ("q3-dirichlet", ri.CONFIGS[1].with_mesh(3)),
    ("q4-neumann-logalpha", ri.CONFIGS[2].with_mesh(3).with_p(4)),
    ("nce3", ri.CONFIGS[3].with_mesh(2).with_p(3)),
    ("ncf3", ri.CONFIGS[4].with_mesh(2).with_p(3)),
    ("q3-trilinear", ri.CONFIGS[5].with_mesh(3).with_p(3)),
])
def test_product_coarse_level_matches_oracle(emu, name, w):
    """The product's host coarse setup (A_0 assembly incl. the trilinear Q1 element matrix, the
    block-tridiagonal Cholesky, the embedding tables) re-enacted by tests/native/emu.cpp equals the
    oracle's R_0^T A_0^{-1} R_0 (oracle/coarse.py)."""
    from oracle.coarse import CoarseLevel
    from oracle.solver import Problem
    pb = Problem(w.space, w.p, w.nx, w.ny, w.nz, ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w), w.gamma_d,
                 decomposition=w.decomposition, factorization=w.factorization)
    r = ri.uniform_vector(w.cfg, 0, pb.space.ndof)
    r[pb.constrained] = 0
    al = np.ascontiguousarray(ri.cell_alpha(w).ravel())
    be = np.ascontiguousarray(ri.cell_beta(w).ravel())
    coords = None if w.perturb == 0 else np.ascontiguousarray(ri.vertex_coords(w).ravel())
    D = ctypes.POINTER(ctypes.c_double)
    emu.emu_coarse.argtypes = [ctypes.c_int] * 5 + [ctypes.c_uint, D, ctypes.c_longlong, D, ctypes.c_longlong, D, D, D,
                                                    ctypes.c_char_p, ctypes.c_int]
    z = np.zeros_like(r)
    err = ctypes.create_string_buffer(256)
    rc = emu.emu_coarse(w.space, w.p, w.nx, w.ny, w.nz, w.gamma_d, _dp(al), al.size, _dp(be), be.size,
                        None if coords is None else _dp(coords), _dp(r), _dp(z), err, 256)
    assert rc == 0, err.value
    zo = CoarseLevel(pb).apply(r)
    assert np.linalg.norm(z - zo) / np.linalg.norm(zo) < 1e-11


@pytest.mark.parametrize("n,p", [(2, 3), (3, 4)])
def test_product_icc_sc_potential_matches_oracle(emu, n, p):
    """Row f3: ICC on the static-condensation pattern for the H(curl) PH potential vertex stars
     -- the product's k = 0 ICC-SC family on Cartesian cells with the potential
    coefficients (alpha', beta') = (beta, 0), re-enacted on the host, equals the oracle's potential
    patch solves (oracle.solver.Problem.potential with factorization icc_sc)."""
    from oracle.solver import Problem
    w = ri.CONFIGS[3].with_mesh(n).with_p(p)
    beta = np.full((n, n, n), 0.7)
    pb = Problem(1, p, n, n, n, ri.vertex_coords(w), np.ones((n, n, n)), beta, w.gamma_d, decomposition="ph",
                 factorization="icc_sc")
    D, pcon, sol = pb.potential()
    t = ri.uniform_vector(3, 5, D.shape[1])
    t[pcon] = 0
    so = np.zeros_like(t)
    for g, S in sol:
        so[g] += S.solve(t[g])
    al = np.ascontiguousarray(beta.ravel())
    be = np.zeros_like(al)
    z = np.zeros_like(t)
    err = ctypes.create_string_buffer(256)
    st = (ctypes.c_longlong * 10)()
    rc = emu.emu_precondition(0, p, n, n, n, w.gamma_d, _dp(al), al.size, _dp(be), be.size, None, 0, 1, 0, _dp(t),
                              _dp(z), err, 256, st)
    assert rc == 0, err.value
    assert np.linalg.norm(z - so) / np.linalg.norm(so) < 1e-11


@pytest.mark.parametrize("name,w", [
    ("cfg1-sc-chol", ri.CONFIGS[1].with_mesh(3)),
    ("cfg2-sc-chol-logalpha", ri.CONFIGS[2].with_mesh(3).with_p(4)),
    ("cfg5-sc-icc", ri.CONFIGS[5].with_mesh(2).with_p(3)),
    ("cfg5-sc-icc-3^3p5", ri.CONFIGS[5].with_mesh(3).with_p(5)),
])
def test_product_sc_pafw_matches_oracle(emu, name, w):
    """Row f2 (k = 0): SC-PAFW (eq:sc-asm-afw) -- the product's family with the interior
    corrections zeroed in the boxes (exact program) or n_K = 1 (ICC-SC program) and the post step
    c_I = A_II^{-1}(r_I - A_IG c_G), re-enacted on the host, equals the oracle's definition."""
    from oracle.solver import Problem
    pb = Problem(w.space, w.p, w.nx, w.ny, w.nz, ri.vertex_coords(w), ri.cell_alpha(w), ri.cell_beta(w), w.gamma_d,
                 decomposition="sc-pafw", factorization=w.factorization)
    r = ri.uniform_vector(w.cfg, 0, pb.space.ndof)
    r[pb.constrained] = 0
    al = np.ascontiguousarray(ri.cell_alpha(w).ravel())
    be = np.ascontiguousarray(ri.cell_beta(w).ravel())
    coords = None if w.perturb == 0 else np.ascontiguousarray(ri.vertex_coords(w).ravel())
    z = np.zeros_like(r)
    err = ctypes.create_string_buffer(256)
    st = (ctypes.c_longlong * 10)()
    fact = 1 if w.factorization == "icc_sc" else 0
    rc = emu.emu_precondition(0, w.p, w.nx, w.ny, w.nz, w.gamma_d, _dp(al), al.size, _dp(be), be.size,
                              None if coords is None else _dp(coords), 0, fact, 2, _dp(r), _dp(z), err, 256, st)
    assert rc == 0, err.value
    zo = pb.precondition(r)
    assert np.linalg.norm(z - zo) / np.linalg.norm(zo) < 1e-11


# ------------------------------------------------------------------ device numeric setup (f4)
NUMPROG_CASES = [
    ("cfg1", ri.CONFIGS[1], 0, 0),
    ("cfg2-3^3p4", ri.CONFIGS[2].with_mesh(3).with_p(4), 0, 0),
    ("cfg2-2^3p7", ri.CONFIGS[2].with_mesh(2), 0, 0),
    ("cfg3-edge-2^3p3", ri.CONFIGS[3].with_mesh(2).with_p(3), 1, 0),
    ("cfg3-vertex-2^3p3", ri.CONFIGS[3].with_mesh(2).with_p(3), 0, 0),
    ("cfg4-face-2^3p3", ri.CONFIGS[4].with_mesh(2).with_p(3), 2, 0),
    ("cfg5-icc-2^3p3", ri.CONFIGS[5].with_mesh(2).with_p(3), 0, 1),
    ("cfg5-icc-3^3p5", ri.CONFIGS[5].with_mesh(3).with_p(5), 0, 1),
]


@pytest.mark.parametrize("name,w,dim,fact", NUMPROG_CASES, ids=[c[0] for c in NUMPROG_CASES])
def test_device_numeric_program_reenacted_equals_host_factorization(emu, name, w, dim, fact):
    """The program the GPU setup executes (dsetup.cu: assembly lists, level-0 records, Schur targets,
    dense Cholesky of the interface in position order, level recipes, final inverse / ICC(0), stream
    map), re-enacted on the host, reproduces every value block of the host factorization
    (factor_patch) to rounding: a wrong index anywhere in the program moves some value by O(1)."""
    D = ctypes.POINTER(ctypes.c_double)
    emu.emu_numeric_program_check.argtypes = [ctypes.c_int] * 5 + [ctypes.c_uint, D, ctypes.c_longlong, D,
                                                                     ctypes.c_longlong, D, ctypes.c_int, ctypes.c_int, D,
                                                                     ctypes.c_char_p, ctypes.c_int]
    al = np.ascontiguousarray(ri.cell_alpha(w).ravel())
    be = np.ascontiguousarray(ri.cell_beta(w).ravel())
    coords = None if w.perturb == 0 else np.ascontiguousarray(ri.vertex_coords(w).ravel())
    rel = np.zeros(1)
    err = ctypes.create_string_buffer(256)
    rc = emu.emu_numeric_program_check(w.space, w.p, w.nx, w.ny, w.nz, w.gamma_d, _dp(al), al.size, _dp(be), be.size,
                                       None if coords is None else _dp(coords), dim, fact, _dp(rel), err, 256)
    assert rc == 0, err.value
    # the interface elimination order differs (one dense Cholesky instead of sparse levels + dense final
    # block): rounding only; H(div) blocks carry kappa ~1e5
    print(f"{name}: max |device program - host| / max|value| = {rel[0]:.2e}")
    assert 0 <= rel[0] < (1e-9 if w.space == 2 else 1e-11), rel[0]
