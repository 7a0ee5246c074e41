"""TEST INFRASTRUCTURE ONLY -- the checkers for the B200 path.

* ``hec_oracle.c`` (``_build/libhecoracle.so``): plain-C restatement of the
  reference path, each function citing the reference file:line it follows.
* ``_ref/libhecref.so``: the reference library itself, compiled from
  /root/reference/proj/src by ``oracle/Makefile`` (present when it was built in
  a container that has the reference; the .so travels with the snapshot).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's reference / cpu_baseline
legs may import this package. The product never does.
"""
from .oracle import Oracle, Reference, load_oracle, load_reference  # noqa: F401
