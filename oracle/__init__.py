"""Parity CHECKERS for the LaMM hot path — test infrastructure only.

* ``ref()``    — the unmodified reference (``/root/reference/proj/core``) compiled
  into ``oracle/_ref/liblamm_ref.so`` by ``oracle/Makefile``.
* ``port()``   — the plain-C restatement ``oracle/lamm_oracle.c`` (pinned
  bit-exact to ``ref()`` by ``tests/test_oracle_pin.py``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. The product package
``paper_2505_22208_b200`` never does.
"""
from .binding import OracleLib, ref, port, ref_available  # noqa: F401
