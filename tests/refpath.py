"""Locate an importable copy of the reference `fairsched` package (the caller
side of the drop-in boundary: Simulator, Worker, runner).

Search order: already importable, ./baseline/_ref (installed by build()),
/root/reference/pkg/src (build container only)."""
import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def import_fairsched():
    try:
        return importlib.import_module("fairsched")
    except ImportError:
        pass
    for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(cand, "fairsched")):
            sys.path.insert(0, cand)
            return importlib.import_module("fairsched")
    return None
