"""paper_2406_11235_b200 -- B200-native QTIP (arXiv 2406.11235) inference hot path.

The product is libqtip.so (include/qtip.h): fused trellis-decode GEMV/GEMM with RHT in/out,
hand-written for sm_100a.  This package holds its sources (csrc/), the in-tree build
(build.py), the ctypes binding (qtip.py), a layer wrapper (layer.py) and the row-sharded
multi-GPU wrapper (sharded.py).  PyTorch supplies device memory, streams and process
groups only.
"""
from . import qtip  # noqa: F401
