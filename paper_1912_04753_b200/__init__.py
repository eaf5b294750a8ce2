"""paper_1912_04753_b200 — B200-native space-time Ripley's K pair path.

The reference (stripley, arXiv 1912.04753) keeps its public entry points; this
package re-provides them over ``libstk.so`` (hand-written sm_100a kernels behind
the C ABI in ``include/stk.h``):

    from paper_1912_04753_b200.stripley import geom, est, sim, rt

mirrors ``stripley::geom`` / ``est`` / ``sim`` / ``rt`` (proj/core/include/stripley/).
"""
from ._lib import LIB_PATH, load  # noqa: F401

__all__ = ["LIB_PATH", "load"]
