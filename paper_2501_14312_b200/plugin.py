"""Install the B200 decision path behind the reference's own plug points.

The reference resolves its policy classes from module globals at call time
(make_local_policy -> `Dlpm`, local_policies.py:198-209; make_dispatcher ->
`D2lpm`, global_policies.py:164-181) and Worker builds its cache through
`fairsched.worker.RadixTree` (worker.py:11, 72).  install() rebinds exactly
those names, so `fairsched.runner.run_experiment` (and every caller of the
factories) runs unchanged on the GPU path; config validation still sees the
names "dlpm" / "lpm" / "d2lpm".  Nothing in the reference is edited.
"""
from __future__ import annotations

import importlib

from .policies import GpuD2lpm, GpuDlpm, GpuLpm, GpuThresholdRouter, GpuVtc
from .radix import DeviceRadixTree

_SAVED = {}

_BINDINGS = (
    ("fairsched.local_policies", "Dlpm", GpuDlpm),
    ("fairsched.local_policies", "Lpm", GpuLpm),
    ("fairsched.local_policies", "Vtc", GpuVtc),
    ("fairsched.global_policies", "D2lpm", GpuD2lpm),
    ("fairsched.global_policies", "ThresholdRouter", GpuThresholdRouter),
    ("fairsched.global_policies", "RadixTree", DeviceRadixTree),
    ("fairsched.worker", "RadixTree", DeviceRadixTree),
    ("fairsched.radix", "RadixTree", DeviceRadixTree),
    ("fairsched", "RadixTree", DeviceRadixTree),
)


_WORKER_SAVED = {}


def install(host_fast_path: bool = True) -> None:
    """Route fairsched's DLPM / LPM / D2LPM / RadixTree through the GPU.
    host_fast_path: also give workers running these policies the host
    bookkeeping fast path (paper_2501_14312_b200.hostpath)."""
    from ._lib import load

    load()  # fail loudly now if the CUDA extension is missing
    for mod_name, attr, obj in _BINDINGS:
        mod = importlib.import_module(mod_name)
        key = (mod_name, attr)
        if key not in _SAVED:
            _SAVED[key] = getattr(mod, attr)
        setattr(mod, attr, obj)
    # the reference's native-kernel seam reports which implementation runs the
    # prefix compares (speedups.py:8-22): with the drop-in installed every walk
    # is on the device, common_prefix_len itself is never called by the path
    sp = importlib.import_module("fairsched.speedups")
    if ("fairsched.speedups", "KERNEL_IMPL") not in _SAVED:
        _SAVED[("fairsched.speedups", "KERNEL_IMPL")] = sp.KERNEL_IMPL
    sp.KERNEL_IMPL = "cuda"
    if host_fast_path and not _WORKER_SAVED:
        from . import hostpath
        _WORKER_SAVED.update(hostpath.install(importlib.import_module("fairsched.worker").Worker,
                                              importlib.import_module("fairsched.requests").Trace))


def uninstall() -> None:
    for (mod_name, attr), obj in list(_SAVED.items()):
        setattr(importlib.import_module(mod_name), attr, obj)
    _SAVED.clear()
    if _WORKER_SAVED:
        from . import hostpath
        hostpath.uninstall(dict(_WORKER_SAVED))
        _WORKER_SAVED.clear()


def installed() -> bool:
    return bool(_SAVED)
