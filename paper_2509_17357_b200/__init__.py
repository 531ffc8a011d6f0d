"""Cronus partial-prefill serving (arXiv 2509.17357), B200-native hot path.

C++ scheduler + sm_100a CUDA kernels in libcronus_b200.so; this package is the thin
Python mirror used by tests and bench.py.
"""
from . import engine  # noqa: F401
