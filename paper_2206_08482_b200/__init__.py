"""B200-native GMI-DRL data-parallel PPO iteration (arXiv 2206.08482).

Host-side Python mirror of the reference's gmux API over the C-ABI in
include/gmi.h (libgmi.so, built in-tree).  See DESIGN.md.
"""
from ._lib import GmiError, lib  # noqa: F401
