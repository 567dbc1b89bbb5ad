"""CPU oracle for the CKKS hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product package
``paper_2104_03152_b200`` never imports it and shares no code with it.
"""
from .oracle import OracleContext, OCt, cdt_table, build_oracle  # noqa: F401
