"""vmfilt-b200: B200-native hot path of `vmfilt` (Kennedy, arXiv 1912.07133).

Separable IIR/FIR blur -> [1,-2,1] Laplacian -> threshold + NMS blob
extraction on hand-written sm_100a CUDA kernels behind a C ABI
(include/vmfilt_b200.h, libvmfilt_b200.so).  The Python layer mirrors the
reference's engine API (engine.py) so it is a drop-in.
"""
from . import design, filters, synth  # noqa: F401
from .errors import FilterError, StabilityError  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # engine / detect import torch; load them lazily
    if name in ("engine", "detect", "blob", "shard"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
