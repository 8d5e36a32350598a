"""B200-native matrix-free SIMP hot path (PyTopo3D, arXiv 2504.05604).

The product is libtopo.so (include/topo.h): hand-written sm_100a CUDA kernels
behind a C ABI.  `topo` is the thin ctypes binding; there is no CPU fallback
(importing `topo` without the built library raises ImportError).  The
binding is loaded lazily so that `python -m paper_2504_05604_b200.build` works
before the library exists.
"""
import importlib

__all__ = ["topo", "Problem", "TopoError", "element_stiffness"]


def __getattr__(name):
    if name == "topo":
        return importlib.import_module(".topo", __name__)
    if name in ("Problem", "TopoError", "element_stiffness"):
        return getattr(importlib.import_module(".topo", __name__), name)
    raise AttributeError(name)
