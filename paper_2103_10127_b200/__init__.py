"""paper_2103_10127_b200 -- B200-native restricted additive Vanka (RAV)
geometric multigrid for Taylor-Hood Stokes systems (arXiv 2103.10127).

The compute path is libravgmg.so (CUDA, sm_100a) behind the C-ABI of
include/ravgmg.h; ``ravgmg`` is its thin ctypes binding.
"""
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libravgmg.so")


def load():
    """Import the binding (loads libravgmg.so; raises if it cannot)."""
    from . import ravgmg
    return ravgmg
