"""TEST INFRASTRUCTURE ONLY: CPU oracle for the HHFFBPA / BPA hot path.

A restatement of the reference algorithm (/root/reference/pkg/src/hhsar)
in numpy + a small OpenMP C library (oracle_kernels.c).  It is the checker
for the CUDA product path and the timed CPU baseline in bench.py; nothing in
``paper_2506_23568_b200`` imports it.  It is pinned against golden vectors
produced by the reference itself (tests/golden/make_golden.py).
"""

from .pipeline import *  # noqa: F401,F403
