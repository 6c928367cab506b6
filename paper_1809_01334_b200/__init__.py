"""B200-native forest-of-octrees raycasting hot path (arXiv 1809.01334).

The product is librc.so (CUDA, sm_100a) behind the C ABI of include/rc.h;
`rc` is its thin ctypes binding and `dist` the torch.distributed plumbing of
the multi-GPU tile exchange.
"""
from . import rc  # noqa: F401

__all__ = ["rc"]
