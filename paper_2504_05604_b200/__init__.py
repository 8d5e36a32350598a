"""B200-native matrix-free SIMP hot path (PyTopo3D, arXiv 2504.05604).

The product is libtopo.so (include/topo.h): hand-written sm_100a CUDA kernels
behind a C ABI.  `topo` is the thin ctypes binding; there is no CPU fallback.
"""
from . import topo  # noqa: F401  (raises ImportError if libtopo.so is not built)
from .topo import Problem, TopoError, element_stiffness  # noqa: F401
