"""TEST INFRASTRUCTURE ONLY -- CPU oracles for the latsum hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package; the product (``paper_1405_2270_b200``) never
does. Two oracles live here:

* ``restatement()`` -- ``liblatsum_oracle.so``, a plain-C restatement of the
  reference algorithm (``latsum_oracle.c``, each function citing the
  reference file:line it follows).
* ``reference()`` -- ``_ref/libref_latsum_v{3,4}.so``, the reference's own
  headers compiled unmodified (``ref_capi.cpp``); present wherever
  ``oracle/Makefile`` ran with ``/root/reference`` available (the built .so
  travels to the GPU box, the reference sources do not).
"""
from .binding import reference, restatement, ref_available  # noqa: F401
