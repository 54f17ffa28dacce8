"""B200-native RFPF Cholesky (Gustavson, Wasniewski, Dongarra, Langou).

Drop-in for the reference package ``rfpk`` on its hot path: ``layout``,
``convert``, ``rfp``, ``packed`` and ``kernels`` mirror the reference modules
of the same names; data lives in CUDA tensors and every operation runs as
hand-written sm_100a kernels behind the C ABI in ``include/rfpk_b200.h``
(``librfpk_b200.so``).  There is no CPU fallback.
"""

from . import layout  # noqa: F401  (pure host geometry; importable without a GPU)

__all__ = ["layout", "convert", "rfp", "packed", "kernels", "__version__"]
__version__ = "0.1.0"


def __getattr__(name):
    import importlib

    if name in ("convert", "rfp", "packed", "kernels", "_capi"):
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
