"""CPU oracle for the Anderson shift-and-invert / Jacobi-Davidson hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_math_0508111_b200/`) may import, call, link or execute anything under
`oracle/`.  Only `tests/`, `__graft_entry__.smoke()`, `bench.py`'s
`cpu_baseline` leg / `--impl reference` arm and `scripts/make_golden.py` use it.

The oracle is a plain, slow, obviously-correct fp64 implementation written
from PAPER.md (arxiv math/0508111, Schenk, Bollhoefer, Roemer) and the
readings listed in DESIGN.md section 3.  It shares no code with the CUDA path.

Modules
-------
anderson  Eq. (eigenequation): disorder generator,
          site index, sparse matrix, matrix-free stencil.
eigs      eigenpairs nearest a shift: dense diagonalisation (tiny L) and plain
          shift-and-invert Lanczos (sect. 4.1) with a direct
          inner solve (larger L).
mlildl    the symmetric multilevel incomplete LDL^T preconditioner
          (sect. 7) in the independent-set reading of
          DESIGN.md sect. 3.3.
sqmr      simplified QMR (sect. 4.2 / 7.4).

Parity status: every function is pinned by `tests/test_oracle_*.py` against
closed forms / invariants / brute force, see DESIGN.md sect. 5 for the list.
"""
