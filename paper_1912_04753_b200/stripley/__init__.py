"""Host-side mirror of the reference's C++ API for the K pair path.

Module and symbol names follow ``stripley::geom``, ``stripley::est``,
``stripley::sim`` and ``stripley::rt`` (proj/core/include/stripley/*.hpp), with
the same argument meaning and the same ``std::invalid_argument`` messages
(raised here as ``ValueError``).  Every estimation call runs on the device
through ``libstk.so``; there is no CPU fallback.
"""
from . import device, est, geom, rt, sim  # noqa: F401

__all__ = ["device", "est", "geom", "rt", "sim"]
