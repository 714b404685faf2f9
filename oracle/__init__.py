"""QuaRot CPU oracle — TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct CPU definition of what the
QuaRot online quantized-linear hot path computes (arXiv 2404.00456).  It exists
to *judge* the CUDA path, never to serve it:

* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it.
* It shares no code with ``paper_2404_00456_b200`` (the CUDA path) and imports
  nothing from it.  The only shared module is ``synth`` (seeded input
  generators, which contain none of the method's arithmetic).
* Arithmetic is NumPy fp64 (reals) / int64 (integers).  fp16 inputs are exact in
  fp64.  Each function cites the PAPER.md line (``P:<n>``) and the SURVEY.md §8(c)
  reading (``Z<n>``) it implements.

Citation convention: ``P:<n>`` = /root/reference/PAPER.md line n (the paper's
LaTeX source), ``S:<n>`` = SPEC.md line n.  Readings Z1..Z20 are listed in
DESIGN.md §3.

Parity pins live in ``tests/test_oracle_*.py``.  Functions without an external
pin say "parity unpinned" in their docstring; DESIGN.md lists them.
"""

from . import hadamard, quant, gemm, kv, layer, glue, attention  # noqa: F401
