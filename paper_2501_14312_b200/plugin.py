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


def install(host_fast_path: bool = True, placement: str = "shared", devices=None, verifiers: bool = True) -> None:
    """Route fairsched's DLPM / LPM / VTC / D2LPM / threshold routing and
    RadixTree through the GPU.
    host_fast_path: also give workers running these policies the host
    bookkeeping fast path (paper_2501_14312_b200.hostpath).
    placement: "shared" (one context) or "per_worker" (worker w's cache, queue
    and counters on devices[w % len(devices)] with its own context, the
    dispatcher on devices[0]; runtime.set_placement).
    verifiers: also run metrics.py's service-gap verifiers on the GPU
    (paper_2501_14312_b200.verify; runner.verify_run calls them through the
    module, runner.py:383-440)."""
    from ._lib import load
    from . import runtime

    load()  # fail loudly now if the CUDA extension is missing
    runtime.set_placement(placement, devices)
    wmod = importlib.import_module("fairsched.worker")
    if ("fairsched.worker", "Worker.__init__") not in _SAVED:
        orig_init = wmod.Worker.__init__
        _SAVED[("fairsched.worker", "Worker.__init__")] = orig_init

        def __init__(self, sim, wid, *a, **kw):
            # Worker builds its RadixTree in __init__ (worker.py:72): tell the
            # device tree whose cache it is
            runtime.set_current_worker(wid)
            try:
                orig_init(self, sim, wid, *a, **kw)
            finally:
                runtime.set_current_worker(None)
        __init__.__wrapped__ = orig_init
        wmod.Worker.__init__ = __init__
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
    if verifiers:
        from . import verify
        mmod = importlib.import_module("fairsched.metrics")
        for name in verify.REBOUND:
            key = ("fairsched.metrics", name)
            if key not in _SAVED:
                _SAVED[key] = getattr(mmod, name)
            setattr(mmod, name, getattr(verify, name))
    if host_fast_path and not _WORKER_SAVED:
        from . import hostpath
        _WORKER_SAVED.update(hostpath.install(importlib.import_module("fairsched.worker").Worker,
                                              importlib.import_module("fairsched.requests").Trace))


def uninstall() -> None:
    for (mod_name, attr), obj in list(_SAVED.items()):
        if attr == "Worker.__init__":
            importlib.import_module(mod_name).Worker.__init__ = obj
        else:
            setattr(importlib.import_module(mod_name), attr, obj)
    _SAVED.clear()
    from . import runtime
    runtime.set_placement("shared")
    if _WORKER_SAVED:
        from . import hostpath
        hostpath.uninstall(dict(_WORKER_SAVED))
        _WORKER_SAVED.clear()


def installed() -> bool:
    return bool(_SAVED)
