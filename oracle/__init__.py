"""CPU oracle for the SCSF hot path — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct fp64 implementations of what the CUDA path
computes, written from PAPER.md (arXiv 2510.23215) and sharing no code with
`paper_2510_23215_b200/` (neither side imports the other).  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import anything from here; the product path never does.

Modules
  sort     Alg. 2: naive truncated DFT, Frobenius
           distances, greedy nearest-neighbour order with strict `<`.
  operator the oracle's own flux-form FD assembly (
           DESIGN.md reading R20) into explicit sparse / dense / banded forms.
  eig      the plain definition of the solve result (PAPER.md:143-150, 336,
           341): the L eigenpairs of smallest |lambda| of each operator,
           independently of order and warm start — cyclic Jacobi for tiny
           dense matrices, shift-invert block Lanczos otherwise.
  checks   residual metric, orthonormality, subspace sines,
           clusters, Sylvester inertia (completeness) and Loewner bounds.

Pins: tests/test_oracle_*.py (marker "not gpu") — closed-form Laplacian
spectra, the paper's printed Eq. 2 and App. B matrices, FFT/Parseval
identities, brute-force raw-field greedy, library eigh on tiny inputs,
inertia counts.  See DESIGN.md §4 for the pin of every function.
"""
