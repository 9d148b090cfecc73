"""podracer-b200: B200-native pod hot path of ElegantRL-podracer (arXiv 2112.05923).

The product is libprb.so (csrc/, sm_100a CUDA behind the prb_* C ABI in
include/prb.h); ``podracer`` is the Python mirror of the reference API on top.
"""
from . import _lib  # noqa: F401

__version__ = "0.1.0"


def load():
    """Load the native library (raises ImportError when it was not built)."""
    return _lib.lib()
