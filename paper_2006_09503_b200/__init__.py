"""p2bw: B200-native PipeDream-2BW training engine.

Python mirror of the reference's pipesim API for the pipelined training path,
bound over the C-ABI of libp2bw.so (include/p2bw.h).  See DESIGN.md.
"""
from ._lib import P2bwError, lib  # noqa: F401
