"""B200-native SOLAR loading planner (arXiv 2211.00224) — drop-in for the
reference ``loadsched`` hot path: shuffle -> reuse matrix -> epoch order ->
{remap, balance, clairvoyant eviction} step loop -> per-rank replay -> HBM
batch gather, all as hand-written sm_100a kernels behind a C ABI
(include/lsg.h)."""
from ._lib import LIB_PATH, LsgError, lib  # noqa: F401
from .loadsched import *  # noqa: F401,F403

__version__ = "0.1.0"
