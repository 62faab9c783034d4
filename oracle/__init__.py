"""CPU oracle for the DDCCANet fit/transform path — TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference package's hot path
(``ddccanet`` 0.1.0, /root/reference/pkg/src/ddccanet). Every function cites
the reference file:line it restates.

Who may use it (and nobody else):
  * ``tests/``                      — as the parity checker;
  * ``__graft_entry__.smoke()``     — to check one small CUDA invocation;
  * ``bench.py``                    — the ``cpu_baseline`` leg and the
                                      ``--impl reference`` arm (it is the
                                      reference's CPU algorithm, timed).

The product package ``paper_2209_13027_b200`` never imports this package;
the product path fails loudly when its CUDA library is missing.

Pinning: ``tests/test_oracle_golden.py`` checks this port against golden
vectors produced by running the unmodified reference in the build container
(``tests/golden/make_golden.py`` → ``tests/golden/*.npz``) and against the
known-answer tests of the reference's own test suite (pkg/tests/*.py).
Parity status: PINNED (golden fixtures from the reference itself).
"""

from .port import *  # noqa: F401,F403
from .port import __all__  # noqa: F401
