"""paper_2602_10541_b200 -- B200-native hot path of Fast-LSQ (arxiv 2602.10541).

Closed-form assembly of the PDE operator matrix A_ij = L[phi_j](x_i) for sinusoidal random
features (Eq. 2), stacked with weighted BC/IC rows and the rhs (Eq. 3,
P:L118-124), plus the least-squares solve and evaluation of Algorithm 1.

The compute path is libfls.so (hand-written sm_100a CUDA behind the C ABI in include/fls.h);
this package is the thin ctypes binding (``fls``) plus multi-GPU plumbing (``dist``).
"""
from ._abi import FlsError, load as _load_lib  # noqa: F401

__all__ = ["FlsError"]
