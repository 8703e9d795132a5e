"""B200-native stage-execution backend for vLLM-Omni-style disaggregated serving.

The product is native: libomni_dev.so (sm_100a kernels, C ABI include/omni_dev.h)
and libomni_serve.so (C++ stage-graph control plane, C ABI include/omni_serve.h).
This package only locates/loads them (ctypes) and mirrors the reference's
interface names for tests and bench.py. There is no Python or CPU compute path.
"""
from ._native import dev_lib, serve_lib, OmniError, check  # noqa: F401

__all__ = ["dev_lib", "serve_lib", "OmniError", "check"]
