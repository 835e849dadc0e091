"""paper_2601_04719_b200 — B200-native (sm_100a) per-channel symmetric INT8
quantization of FP32 KV-cache keys (arxiv 2601.04719).

The product is libkvq.so (C ABI: include/kvq.h).  ``kvq`` is its thin Python
binding; ``dist`` holds the token-sharding helpers used by bench.py.
"""
from . import kvq  # noqa: F401  (loads libkvq.so; raises if it cannot)
from .kvq import *  # noqa: F401,F403

__version__ = "0.1.0"
