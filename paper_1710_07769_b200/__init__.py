"""B200-native builder of the row inner-product graph G_RIP (arXiv 1710.07769)
and the cutsize of a block-row partition.

The compute path is librig.so (hand-written sm_100a CUDA behind the C ABI in
include/rig.h); this package is its thin Python binding plus the multi-GPU
plumbing (torch.distributed).  Importing ``paper_1710_07769_b200.rig`` fails
loudly when librig.so has not been built: there is no CPU fallback.
"""
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "librig.so")

__all__ = ["PKG_DIR", "LIB_PATH"]
