"""B200-native Chung–Lu generator (Alam & Khan, arXiv:1406.1215).

The hot path of the reference ``clgen`` library — the per-source edge-skipping
sampler ``edges_from_source`` driven over UCP partitions — rebuilt as
hand-written sm_100a CUDA kernels behind a C ABI (``include/clgen_dev.h``).
This package is the host-side mirror of the reference's ``clgen::`` API.
"""
from ._lib import error  # noqa: F401

__all__ = ["error", "api"]


def __getattr__(name):
    if name == "api":
        import importlib
        return importlib.import_module(__name__ + ".api")
    raise AttributeError(name)
