"""paper_2601_04719_b200 — B200-native (sm_100a) per-channel symmetric INT8
quantization of FP32 KV-cache keys (arxiv 2601.04719).

The product is libkvq.so (C ABI: include/kvq.h).  ``kvq`` is its thin Python
binding (importing it loads libkvq.so and raises if it cannot); ``dist`` holds
the token-sharding helpers used by bench.py; ``build`` compiles libkvq.so.
"""
import importlib

__version__ = "0.1.0"
__all__ = ["kvq", "dist", "build"]


def __getattr__(name):
    if name in __all__:
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
