"""PG-SAG (arXiv 2501.01677) masked tile rasterizer, forward and backward, on B200.

The product is libpgsag.so (sm_100a CUDA kernels behind the C ABI in
include/pgsag.h).  This package is its thin Python binding:
  _lib    ctypes declarations of the ABI (marshalling only)
  raster  buffer ownership + the four calls on the current torch stream
  train   NEXT-3 training iteration (losses + Adam) over the same ABI
  shard   sub-region assignment / per-rank statistics (multi-GPU plumbing)
  build   in-tree nvcc build of libpgsag.so
There is no CPU fallback; the oracle lives in /oracle and is test-only.
"""
from . import _lib  # noqa: F401
from ._lib import PgsagError, lib, version  # noqa: F401


def __getattr__(name):
    if name in ("Rasterizer", "GaussianTensors", "camera_from", "make_camera"):
        from . import raster
        return getattr(raster, name)
    if name in ("Trainer", "AdamConfig"):
        from . import train
        return getattr(train, name)
    raise AttributeError(name)
