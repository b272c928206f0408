"""Per-process device runtime shared by every drop-in object.

* one `Context` per CUDA device (token arena + request table),
* a request registry mapping the reference's token tuples (Request.input_tokens,
  requests.py:22-32) to device request ids -- each tuple is uploaded once,
* a client registry (client name -> dense id, shared by all workers and the
  dispatcher of the device),
* order-maintenance labels for the LPM tie-break key (arrival, rid)
  (local_policies.py:17): the device keeps each worker queue in label order so
  the per-fill sort only has to order by match length.
"""
from __future__ import annotations

import os
import threading

import numpy as np
from sortedcontainers import SortedList

from .device import Context

_LABEL_GAP = 1 << 32


class OrderLabels:
    """64-bit labels whose integer order equals the order of their keys.

    New keys take the midpoint of their neighbours' labels; when a gap is
    exhausted every label is respaced (returned so the caller re-uploads)."""

    def __init__(self):
        self._keys = SortedList()
        self._label = {}

    def __len__(self):
        return len(self._keys)

    def label(self, key):
        return self._label[key]

    def add(self, key):
        """Insert key; returns (label, relabeled) where relabeled is None or a dict."""
        if key in self._label:
            return self._label[key], None
        keys = self._keys
        i = keys.bisect_left(key)
        lo = self._label[keys[i - 1]] if i > 0 else None
        hi = self._label[keys[i]] if i < len(keys) else None
        if lo is None and hi is None:
            lab = 0
        elif hi is None:
            lab = lo + _LABEL_GAP
        elif lo is None:
            lab = hi - _LABEL_GAP
        elif hi - lo >= 2:
            lab = (lo + hi) // 2
        else:
            lab = None
        keys.add(key)
        if lab is not None:
            self._label[key] = lab
            return lab, None
        for j, k in enumerate(keys):
            self._label[k] = j * _LABEL_GAP
        return self._label[key], dict(self._label)


class DeviceRuntime:
    def __init__(self, device: int = 0):
        self.device = device
        self.ctx = Context(device, arena_tokens=1 << 22, max_requests=1 << 16)
        self._by_tuple = {}      # id(tokens) -> (device id, tokens)  (strong ref keeps id stable)
        self._by_key = {}        # (arrival, rid) -> device id: a request's own row
        self._tok_of_id = {}     # device id -> token tuple it was uploaded from
        self._key_of_id = {}     # device id -> (arrival, rid) label key
        self._did_at = {}        # arena offset of a request row -> device id
        self._client_of = {}     # device id -> client id stored in the request table
        self.clients = {}        # client name -> dense id
        self.client_names = []
        self.labels = OrderLabels()

    # -- clients ---------------------------------------------------------
    def client_id(self, name) -> int:
        cid = self.clients.get(name)
        if cid is None:
            cid = len(self.client_names)
            self.clients[name] = cid
            self.client_names.append(name)
        return cid

    # -- requests ----------------------------------------------------------
    def lookup(self, tokens):
        hit = self._by_tuple.get(id(tokens))
        if hit is not None and hit[1] is tokens:
            return hit[0]
        return None

    def did_at(self, off):
        """Device id of the request row starting at arena offset `off` (None if unknown)."""
        return self._did_at.get(int(off))

    def tokens_of(self, did):
        """The token tuple a device id was uploaded from (None if unknown)."""
        return self._tok_of_id.get(did)

    def upload(self, tokens, client=None, arrival=None, rid=None) -> int:
        """Device id of a token sequence; uploads it on first sight.  When
        (arrival, rid) are given the request gets its own row and its LPM
        tie-break label: requests are identified by (arrival, rid), not by
        their token tuple -- Trace.materialize can hand two requests the same
        tuple object (a ``req:`` child with an empty suffix gets
        ``base[:len(base)] + ()``, which CPython returns as ``base`` itself,
        requests.py:148-156), and each must keep its own queue entry."""
        key = (arrival, rid) if rid is not None else None
        if key is not None:
            did = self._by_key.get(key)
            # a key hit is the same request only if it carries the same token
            # tuple: the runtime outlives one run_experiment, and a later run's
            # request can reuse an earlier run's (arrival, rid)
            if did is not None and self._tok_of_id.get(did) is tokens:
                if client is not None:
                    self._set_client(did, client)
                return did
        did = self.lookup(tokens)
        if did is not None and key is not None and self._key_of_id.get(did, key) != key:
            did = None  # the tuple belongs to another request: this one gets its own row
        if did is None:
            if not isinstance(tokens, tuple):
                tokens = tuple(tokens)
            lab = 0
            relabeled = None
            if key is not None:
                lab, relabeled = self.labels.add(key)
            cid = self.client_id(client) if client is not None else 0
            did = self.ctx.add_request(np.fromiter(tokens, dtype=np.int64, count=len(tokens)), cid, lab)
            if self.lookup(tokens) is None:
                self._by_tuple[id(tokens)] = (did, tokens)
            self._tok_of_id[did] = tokens
            self._did_at[self.ctx.request_info(did)[0]] = did
            self._client_of[did] = cid
            if key is not None:
                self._key_of_id[did] = key
                self._by_key[key] = did
            if relabeled is not None:
                self._push_labels()
            return did
        if key is not None:
            lab, relabeled = self.labels.add(key)
            self._key_of_id[did] = key
            self._by_key[key] = did
            if relabeled is not None:
                self._push_labels()
            else:
                self.ctx.set_labels(np.array([did], np.int32), np.array([lab], np.int64))
        if client is not None:
            self._set_client(did, client)
        return did

    def _set_client(self, did, client):
        # a token sequence first seen by a routing index (e.g. the reference's
        # ThresholdRouter walking the device tree) was uploaded without its
        # client; the worker's enqueue supplies it
        cid = self.client_id(client)
        if self._client_of.get(did) != cid:
            self.ctx.set_clients(np.array([did], np.int32), np.array([cid], np.int32))
            self._client_of[did] = cid

    def _push_labels(self):
        ids = np.fromiter(self._key_of_id.keys(), dtype=np.int32, count=len(self._key_of_id))
        labs = np.array([self.labels.label(self._key_of_id[i]) for i in ids], dtype=np.int64)
        self.ctx.set_labels(ids, labs)


_RUNTIMES = {}

# Placement of the drop-in's device state (plugin.install(placement=...)):
#   "shared"     -- every worker's tree and the dispatcher on one context of
#                   FS_B200_DEVICE (default);
#   "per_worker" -- worker w gets its own context on devices[w % len(devices)]
#                   (one GPU per data-parallel worker, runner.py:272-289), the
#                   dispatcher its own on devices[0]; eviction notices cross
#                   contexts by request identity (DeviceRadixTree.evict_notify).
_PLACEMENT = {"mode": "shared", "devices": None}
_CURRENT = threading.local()  # worker id whose Worker.__init__ is running (plugin)


def set_placement(mode: str = "shared", devices=None) -> None:
    if mode not in ("shared", "per_worker"):
        raise ValueError(f"unknown placement {mode!r}")
    _PLACEMENT["mode"] = mode
    _PLACEMENT["devices"] = list(devices) if devices is not None else None


def _devices():
    devs = _PLACEMENT["devices"]
    if devs:
        return devs
    env = os.environ.get("FS_B200_DEVICES")
    if env:
        return [int(x) for x in env.split(",") if x.strip()]
    try:
        import torch
        n = torch.cuda.device_count()
    except Exception:
        n = 0
    return list(range(max(n, 1)))


def set_current_worker(wid) -> None:
    _CURRENT.wid = wid


def current_worker():
    return getattr(_CURRENT, "wid", None)


def get_runtime(device: int | None = None, key=None) -> DeviceRuntime:
    """The runtime (context) for `device` (default FS_B200_DEVICE); `key`
    separates several contexts on one device (per-worker placement)."""
    if device is None:
        device = int(os.environ.get("FS_B200_DEVICE", "0"))
    k = (device, key)
    rt = _RUNTIMES.get(k)
    if rt is None:
        rt = DeviceRuntime(device)
        _RUNTIMES[k] = rt
    return rt


def runtime_for_worker(wid=None) -> DeviceRuntime:
    """Runtime of worker `wid`'s tree (the Worker being built when None)."""
    wid = current_worker() if wid is None else wid
    if _PLACEMENT["mode"] != "per_worker" or wid is None:
        return get_runtime()
    devs = _devices()
    return get_runtime(devs[int(wid) % len(devs)], ("worker", int(wid)))


def runtime_for_dispatcher() -> DeviceRuntime:
    if _PLACEMENT["mode"] != "per_worker":
        return get_runtime()
    return get_runtime(_devices()[0], ("dispatcher",))


def runtime_of_ctx(ctx):
    for rt in _RUNTIMES.values():
        if rt.ctx is ctx:
            return rt
    return None


def reset_runtimes():
    """Drop every device runtime (tests use this between independent runs)."""
    for rt in _RUNTIMES.values():
        rt.ctx.close()
    _RUNTIMES.clear()
