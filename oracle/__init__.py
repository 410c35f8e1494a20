"""CPU fp64 ORACLE for the superfast-CUR hot path of arXiv 1710.07946 — TEST INFRASTRUCTURE.

This package is a plain, slow, obviously-correct numpy (fp64 / complex128) restatement of
what the hot path computes, written from PAPER.md before any kernel existed.  It is NOT
part of the product: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  It shares no code with
``paper_1710_07946_b200`` (the CUDA path) and imports nothing from it; the only common
dependency is ``synth`` (seeded input generators, no method arithmetic).

Citations: ``P:n`` = line n of /root/reference/PAPER.md (LaTeX; labels in parentheses).
Every ambiguity resolved here is listed in DESIGN.md §2 ("readings", C1–C23).

Modules
  transforms  H_{n,d} and Ω_{n,d} by the paper's recursions + their closed forms
  lra         sketch (Alg 10.2 stage 1), maxvol (Alg D.2 stage 1 + Alg D.1), C-A loops
              (Remark rerfnhmt), canonical nucleus (Alg 3.1), residual, sampled residual

Pinned by tests/test_oracle_*.py (-m "not gpu"): recursion = closed form = library DFT,
HᵀH = 2^d·I, maxvol vs brute-force volume search, dominance, volume monotonicity,
exactness W = CUR (Thm thcandec), Eckart–Young floor, SPEC nucleus examples.
Parity unpinned: pivots beyond the numerical rank (noise-determined), and the exact value
of ρ for configs 2/3 beyond its floor — see DESIGN.md §5.
"""
from . import transforms, lra  # noqa: F401
