"""B200-native 2DGS camera + LiDAR renderer (hot path of arXiv 2503.11731).

C-ABI: include/gsr.h, implemented by libgsr.so (csrc/*.cu, sm_100a).
Python: `gsr` (ctypes binding, same names as the C-ABI), `render.Renderer`
(buffer management), `dist` (frame-sharded multi-GPU batches).
"""
from . import gsr  # noqa: F401

__all__ = ["gsr"]
