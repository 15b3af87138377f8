"""SynerDiff (arXiv 2605.08835) data-parallel hot path on B200 (sm_100a).

The product is libsynerdiff.so (include/sd_api.h); this package only builds it (`build.py`),
binds it (`binding.py`, ctypes) and wraps it for torch-allocated buffers (`engine.py`).
It never imports `oracle/` and has no CPU fallback.
"""
from . import binding  # noqa: F401
from .build import LIB  # noqa: F401
