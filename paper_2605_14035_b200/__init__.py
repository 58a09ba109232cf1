"""paper_2605_14035_b200 — B200-native ℓFEM assembly (arxiv/paper_2605_14035).

The product is liblfem.so (C ABI, include/lfem.h) with hand-written sm_100a
CUDA kernels; `lfem` is its thin Python binding.  This package never
imports the test oracle (oracle/).
"""
from . import lfem  # noqa: F401
from .lfem import *  # noqa: F401,F403
