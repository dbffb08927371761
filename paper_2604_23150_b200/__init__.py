"""moeplace_b200: B200-native MoE routing-and-placement hot path
(arxiv/paper_2604_23150). See DESIGN.md.

The compute path is libmoeplace_b200.so (hand-written sm_100a CUDA behind the
C ABI in include/moeplace_b200.h); this package is its host-side mirror of the
reference's moeplace:: interface. There is no CPU fallback.
"""
from . import _abi, errors  # noqa: F401
from ._abi import LIB_PATH  # noqa: F401

__all__ = ["LIB_PATH", "errors"]


def load():
    """Loads the shared library (raises if it was not built)."""
    return _abi.lib()
