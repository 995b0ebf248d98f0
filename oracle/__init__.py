"""CPU oracle for the DSO hot path — TEST INFRASTRUCTURE ONLY.

Two checkers, both loaded with ctypes:

* ``port()`` — ``oracle/liboracle.so``, the plain-C double-precision
  restatement of the reference (``oracle/dso_oracle.c``; every function cites
  the reference file:line it follows);
* ``ref()``  — ``oracle/_ref/libdso_ref.so``, the reference's own
  ``proj/src/optimizer.cpp`` and headers compiled in place by
  ``oracle/Makefile`` (see ``oracle/ref_shim.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this package.  The product package never does.
"""

from .oracle import Port, Ref, port, ref, build  # noqa: F401
