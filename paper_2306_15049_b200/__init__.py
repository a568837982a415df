"""B200-native (sm_100a, fp64) hot path of arXiv 2306.15049: recycled CG for the
shifted family (A + gamma_l E_k) x = b of edge-preserving image reconstruction.

    csrc/        CUDA kernels + the C ABI (include/rsk.h), built into librsk.so
    _lib.py      ctypes loader (fails loudly when librsk.so is missing)
    rsk.py       thin binding with the C names (argument marshalling only)
    pipeline.py  outer IRN loop (Alg. 5) orchestrating librsk calls
    build.py     nvcc build (-gencode arch=compute_100a,code=sm_100a)
"""
from . import _lib  # noqa: F401

__all__ = ["Handle", "GpuSolver", "load"]


def load():
    return _lib.load()


def __getattr__(name):
    if name == "Handle":
        from .rsk import Handle
        return Handle
    if name == "GpuSolver":
        from .pipeline import GpuSolver
        return GpuSolver
    raise AttributeError(name)
