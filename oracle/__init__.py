"""CPU ORACLE for arXiv 2211.14284 -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 implementation of what one multigrid relaxation
sweep computes, written from /root/reference/PAPER.md.  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import it.  The product path (`paper_2211_14284_b200/`) never imports,
calls or links anything here; the two share no code (only `rm_inputs`, which holds
no arithmetic of the method).

Modules
  basis1d   GLL rule, FDM 1D basis (eq:fdmbasis, eq:eigs), DP basis, D-hat, G-bar.
  fem       structured de Rham layouts, element matrices by quadrature through the
            pullbacks, global assembly, the auxiliary operator (eq:sum-factorization_approx).
  patches   star patches, patch matrices, dense Cholesky / masked ICC-SC solves.
  solver    residual, additive Schwarz sweep (eq:asm-afw / eq:asm-hiptmair without the
            coarse term), PCG with the natural-norm stopping rule.

Parity status per function is stated in each module header and in DESIGN.md.
"""
