"""CPU oracle for the MDRQ scan hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / the timed CPU baseline.  The product package
``paper_1801_03644_b200`` never imports it: there is no CPU fallback.

Three layers, each pinned against the next (see tests/test_oracle.py):

* ``numpy`` restatements -- :func:`brute_ids` (the reference test suite's own
  independent oracle, pkg/tests/test_scan.py:22-28), :func:`packbits_mask`
  (pkg/tests/test_kernels.py:109), :func:`chunk_spans` (scan.py:43-52),
  :func:`mask_to_ids` (scan.py:85-88) ...;
* ``libmdrq_oracle.so`` -- a C restatement of the reference's Cython kernels
  (oracle/mdrq_oracle.c cites each file:line), OpenMP-parallel batch
  counting for the full-size configs;
* ``_ref/`` -- the reference's own ``_kernels_cy`` module, cythonized and
  compiled from /root/reference by oracle/Makefile (git-ignored, shipped to
  the GPU box as a prebuilt .so).  Used to pin the restatement and as the
  ``kind: "reference"`` CPU baseline.
"""

from .oracle import *  # noqa: F401,F403
from .oracle import __all__  # noqa: F401
