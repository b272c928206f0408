"""B200-native DLPM / D^2LPM decision path (arXiv 2501.14312).

Hand-written sm_100a CUDA kernels behind a C ABI (include/fairsched_b200.h,
libfsb200.so) with drop-in Python adapters for the reference `fairsched`
plug points.  See DESIGN.md.
"""
from ._lib import FsError, load  # noqa: F401

__all__ = ["FsError", "load", "install", "uninstall"]


def install():
    from .plugin import install as _install
    _install()


def uninstall():
    from .plugin import uninstall as _uninstall
    _uninstall()
