"""B200-native hot path of Skrull (arXiv 2505.19609): DACP/GDS-scheduled packed varlen
causal attention (fwd+bwd) with CP K/V all-gather and dK/dV reduce-scatter.

The product is the C-ABI library `libskrull.so` (include/skrull.h). `skrull.py` is a thin
ctypes binding with the same function names (argument marshalling only); `cp.py` drives
one CP step through it. No CPU fallback: importing the binding without the built library
raises.
"""
__all__ = ["skrull"]
