"""B200-native GSI subgraph matching (arXiv 1906.03420) — C-ABI library + thin binding.

The product is ``lib/libgsi_b200.so`` (include/gsi.h); ``gsi`` is its ctypes binding.
Importing this package never touches ``oracle/`` and never falls back to the CPU."""
from . import gsi  # noqa: F401  (raises ImportError if the CUDA library was not built)
from .gsi import (GsiError, build, query, prepare, gsi_build_graph, gsi_query, gsi_query_prepare,  # noqa: F401
                  gsi_query_run, gsi_graph_info_get, gsi_device_count, gsi_version)

__all__ = ["gsi", "GsiError", "build", "query", "prepare", "gsi_build_graph", "gsi_query", "gsi_query_prepare",
           "gsi_query_run", "gsi_graph_info_get", "gsi_device_count", "gsi_version"]
