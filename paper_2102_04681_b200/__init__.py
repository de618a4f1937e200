"""B200-native implementation of the Spice SNN hot path (arXiv 2102.04681).

The compute path lives in ``libspice.so`` (CUDA kernels for sm_100a behind the C ABI of
``include/spice.h``); ``spice`` is its ctypes binding.  Build with
``python -m paper_2102_04681_b200.build``.
"""
from .spice import Network, SpiceError, lib  # noqa: F401
