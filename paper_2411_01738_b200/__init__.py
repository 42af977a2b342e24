"""B200-native USP attention hot path of xDiT (arXiv 2411.01738).

The product is the C-ABI library ``libxdit_usp.so`` (include/xdit_usp.h: tcgen05/TMEM/TMA attention,
LSE merge and Ulysses pack/unpack kernels for sm_100a, NCCL for the all-to-all and ring P2P).
This package is its thin Python binding (``usp``), the in-tree build (``build``) and the seeded
synthetic input generators (``inputs``).  Importing the package does not load the library; the
first call into ``usp`` does, and raises if it was not built -- there is no CPU fallback.
"""
from . import usp  # noqa: F401
from .usp import Comm, RowMap, XditError, attention, plan, shard  # noqa: F401

__all__ = ["usp", "Comm", "RowMap", "XditError", "attention", "plan", "shard"]
