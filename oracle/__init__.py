"""CPU oracle for the SHIRO distributed SpMM hot path (arXiv 2512.20178).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import,
call, link or execute anything under ``oracle/``.  The product path in
``paper_2512_20178_b200/`` never touches it, and the two share no code: the
only module both sides use is the seeded input generator ``shiro_gen``, which
holds none of the method's arithmetic.

Every function cites the PAPER.md (P:line) or SPEC.md (S:line) passage it
follows.  Readings of silent / ambiguous passages are listed in DESIGN.md
("Readings") and referenced here as R<n>.
"""
from .oracle import *  # noqa: F401,F403
