"""CPU oracle for the segregated transpose convolution -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the CPU baseline.  The product path (``paper_2209_03704_b200``) never does.

Two back ends, both loaded with ctypes:

* ``liboracle.so`` -- plain-C restatement of the reference algorithm
  (``oracle/segconv_oracle.c``; each function cites the reference file:line).
  Parity status: pinned against ``tests/golden`` (made by the reference).
* ``_ref/libsegconv_ref.so`` -- the reference's own headers behind an
  ``extern "C"`` shim (``oracle/ref_harness.cpp``), built in this container
  from ``/root/reference`` and shipped as a prebuilt file.
"""
from .oracle import *  # noqa: F401,F403
