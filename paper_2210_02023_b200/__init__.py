"""B200-native embedding hot path of DreamShard (arXiv 2210.02023).

The package is a thin host mirror (api.py) of the reference's interface over
the in-tree CUDA library `_shardplan_b200.so` (C-ABI: include/shardplan_b200.h).
"""
from .api import *  # noqa: F401,F403
from .api import __all__  # noqa: F401
