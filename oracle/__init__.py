"""CPU fp64 oracle for RQI-PCGTLS-MP (Oktay & Carson, arXiv 2305.19028).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
`cpu_baseline` / `--impl reference` legs may import anything from this package.
The product path (paper_2305_19028_b200/) never imports it and shares no code,
headers, tables or helpers with it; the only shared module is tlsgen/ (seeded
input generators, no method arithmetic).

Layout
  rounding.py   fp64 -> fp16 / bf16 / fp32 round-to-nearest-even (PAPER.md
                Table 2, l.435-447; readings R4, R12)
  exact.py      the definitional TLS result from the SVD of [A, b]
                (§1 l.58-63) and the reduced "arrow" model pin
  rqi.py        the algorithmic oracle: scaling, u_f Gram, Cholesky, the
                preconditioner solves, PCGTLS (Alg. 3, l.186-204, both operator
                forms), RQI-PCGTLS-MP (Alg. 4, l.221-258) with the psi stop
                (l.260-265) and the DESIGN.md stop reading
  perfmodel.py  the paper's cost model (§3.2 l.409-417)

Every function cites the passage it follows.  Parity status of each function
is listed in DESIGN.md §"Oracle pins"; the only "parity unpinned" items are
the bitwise u_f Gram and R~ (tensor-core accumulation order is
implementation-defined), pinned instead by a closed-form error bound.
"""
from . import rounding, exact, rqi, perfmodel  # noqa: F401
