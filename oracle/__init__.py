"""FP64 CPU oracle for the FMM-BEM hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg, --impl reference)
may import, call, link or execute anything under oracle/.  The product path
(paper_1007_4591_b200/) never imports it and fails loudly when its CUDA library is
missing.  The oracle shares no code with the CUDA path.

Contents (each function cites the PAPER.md passage it follows; readings in DESIGN.md):
  bem.py           panels + quadrature (O1), constants (O2), E (O3), K' (O4), V (O5),
                   dense LU + GMRES (O6), C (O7), energy (O8), BIBEE (O9), binding (O10),
                   relative L2 (O11)
  closed_forms.py  Born, Kirkwood and BIBEE-on-sphere series (O12)
  direct.c         plain FP64 OpenMP direct sums used by bem.py

Pins: tests/test_oracle_*.py (marker "not gpu").  Parity status per function is listed
in DESIGN.md Sec. "Oracle and pins"; every function has at least one pin that does not
restate its own formula.
"""
from . import bem, closed_forms  # noqa: F401
