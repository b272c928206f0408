"""Drop-in policy objects for the reference plug points.

GpuDlpm / GpuLpm satisfy the LocalPolicy protocol (local_policies.py:20-55,
66-136); GpuD2lpm satisfies the Dispatcher protocol (global_policies.py:28-58,
88-132).  Their decisions are computed on the GPU (fs_worker_fill /
fs_dispatch); the Python objects keep the reference-visible state (`q`,
`client_list`, `refill_counts`, `queue_size`, `records`) as mirrors of the
device state, and the reference Worker keeps doing its own host bookkeeping.

Requires a worker built with DeviceRadixTree (plugin.install() rebinds
fairsched.worker.RadixTree); with any other worker they raise TypeError -- no
CPU fallback.
"""
from __future__ import annotations

import sys
from dataclasses import dataclass

import numpy as np

from .device import DispatcherDev, WorkerDev
from .radix import DeviceRadixTree, EvictedPath
from .runtime import get_runtime


class _TrackedDict(dict):
    """dict that remembers keys written from outside (tests and callers may
    poke counters directly, e.g. test_local_policies.py:96, test_global_policies.py:279)."""

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        self.dirty = set()

    def __setitem__(self, k, v):
        super().__setitem__(k, v)
        self.dirty.add(k)

    def update(self, *a, **kw):
        for k, v in dict(*a, **kw).items():
            self[k] = v

    def setdefault(self, k, v=None):
        if k not in self:
            self[k] = v
        return self[k]

    def _set(self, k, v):  # internal mirror write
        dict.__setitem__(self, k, v)


def _dispatch_record_cls():
    mod = sys.modules.get("fairsched.global_policies")
    if mod is not None and hasattr(mod, "DispatchRecord"):
        return mod.DispatchRecord
    return DispatchRecord


@dataclass
class DispatchRecord:  # global_policies.py:18-25
    rid: str
    client: str
    worker: int
    match_len: int
    matched_workers: tuple
    time: int


# ---------------------------------------------------------------------------
# local policies
# ---------------------------------------------------------------------------


class _GpuLocalPolicy:
    name = "base"
    _policy = "lpm"

    def __init__(self, quantum: int = 1):
        self.worker = None
        self.quantum = quantum
        self._dev = None
        self._rt = None
        self._pending = []      # requests enqueued since the last fill
        self._req_of = {}       # device id -> Request
        self._known_n = 0

    def attach(self, worker) -> None:
        self.worker = worker

    # -- device binding --------------------------------------------------
    def _device(self) -> WorkerDev:
        if self._dev is None:
            w = self.worker
            tree = getattr(w, "tree", None)
            if not isinstance(tree, DeviceRadixTree):
                raise TypeError(
                    f"{type(self).__name__} runs on the GPU and needs a worker whose tree is a "
                    f"DeviceRadixTree (paper_2501_14312_b200.plugin.install()); got {type(tree).__name__}")
            self._rt = tree._rt
            self._dev = WorkerDev(self._rt.ctx, tree.device_trie, self._policy, self.quantum, w.params.M,
                                  w.output_reserve, w.weights.w_e, w.weights.w_q,
                                  max_clients=max(256, len(self._rt.client_names) + 1))
        return self._dev

    def _flush_enqueues(self):
        if not self._pending:
            return
        dev = self._device()
        rt = self._rt
        ids = []
        for req in self._pending:
            did = rt.upload(req.input_tokens, req.client, req.arrival, req.rid)
            self._req_of[did] = req
            ids.append(did)
        dev.reserve_clients(len(rt.client_names) + 1)
        dev.enqueue(np.asarray(ids, np.int32))
        self._pending.clear()

    def on_request_enqueued(self, req, was_active: bool) -> None:
        self._pending.append(req)

    # -- one schedule step ----------------------------------------------
    def fill(self) -> None:
        w = self.worker
        dev = self._device()
        self._flush_enqueues()
        self._push_counters()
        res = dev.fill(w.sim.now, w.generated_total, w._reserved_headroom())
        tree = w.tree
        for k in range(len(res.adm_req)):
            did = int(res.adm_req[k])
            req = self._req_of.pop(did)
            tree._arm(res, k, did)
            try:
                entry = w.try_admit(req)
            finally:
                tree._disarm()
            if entry is None or entry.match_len != int(res.adm_mlen[k]):
                raise RuntimeError(
                    f"device admission of {req.rid} disagrees with the reference Worker.can_add "
                    f"(entry={entry!r}, device mlen={int(res.adm_mlen[k])})")
            self._on_admitted(req, entry)
        self._pull_counters()
        self.last_fill = res

    def _on_admitted(self, req, entry):
        pass

    def _push_counters(self):
        pass

    def _pull_counters(self):
        pass

    def on_outputs(self, counts) -> None:
        pass

    def counters(self):
        return None


class GpuLpm(_GpuLocalPolicy):
    """Lpm (local_policies.py:66-71) on the device."""

    name = "lpm"
    _policy = "lpm"

    def __init__(self):
        super().__init__(1)


class GpuDlpm(_GpuLocalPolicy):
    """Dlpm (local_policies.py:74-136) on the device."""

    name = "dlpm"
    _policy = "dlpm"

    def __init__(self, quantum: int):
        if quantum <= 0:
            raise ValueError("quantum must be positive")
        super().__init__(quantum)
        self.q = _TrackedDict()
        self.client_list = []
        self.refill_counts = {}

    def on_request_enqueued(self, req, was_active: bool) -> None:
        if req.client not in self.q:  # local_policies.py:88-92
            self.q._set(req.client, 0)
            self.refill_counts[req.client] = 0
            self.client_list.append(req.client)
        super().on_request_enqueued(req, was_active)

    def _push_counters(self):
        dev = self._device()
        rt = self._rt
        if self._known_n < len(self.client_list) or self.q.dirty:
            for c in self.client_list:
                rt.client_id(c)
            dev.reserve_clients(len(rt.client_names) + 1)
        if self._known_n < len(self.client_list):
            new = [rt.client_id(c) for c in self.client_list[self._known_n:]]
            dev.mark_known(np.asarray(new, np.int32))
            self._known_n = len(self.client_list)
        if self.q.dirty:
            for c in self.q.dirty:
                if c in self.q:
                    dev.set_counter(rt.client_id(c), int(self.q[c]))
            self.q.dirty.clear()

    def _pull_counters(self):
        q, rf, _ = self._dev.counters()
        for c in self.client_list:
            cid = self._rt.client_id(c)
            self.q._set(c, int(q[cid]))
            self.refill_counts[c] = int(rf[cid])

    def check_refill(self, queued_clients) -> bool:
        """local_policies.py:94-106, evaluated by the device kernel."""
        dev = self._device()
        self._push_counters()
        refilled = dev.check_refill(np.asarray([self._rt.client_id(c) for c in queued_clients], np.int32))
        self._pull_counters()
        return refilled

    def on_outputs(self, counts) -> None:
        """local_policies.py:130-133 (mirror + device delta for the next fill)."""
        if not counts:
            return
        dev = self._device()
        w_q = self.worker.weights.w_q
        cids, ns = [], []
        for client, n in counts.items():
            self.q._set(client, self.q[client] - w_q * n)
            cids.append(self._rt.client_id(client))
            ns.append(n)
        dev.outputs(np.asarray(cids, np.int32), np.asarray(ns, np.int64))

    def counters(self):
        return dict(self.q)


# ---------------------------------------------------------------------------
# D2LPM dispatcher
# ---------------------------------------------------------------------------


class GpuD2lpm:
    """D2lpm (global_policies.py:88-132) with the routing index, q_{i,w} and the
    SelectWorker chain on the device."""

    name = "d2lpm"
    uses_global_tree = True

    def __init__(self, worker_ids, quantum, weights):
        if quantum <= 0:
            raise ValueError("quantum must be positive")
        self.worker_ids = list(worker_ids)
        self.queue_size = _TrackedDict({w: 0 for w in self.worker_ids})
        self.queue_size.dirty.clear()
        self.records = []
        self.quantum = quantum
        self.weights = weights
        self.q = _TrackedDict()
        self._ids = sorted(self.worker_ids)   # device worker index order == id order (_min_queue tie-break)
        self._rt = get_runtime()
        self._dev = DispatcherDev(self._rt.ctx, len(self._ids), quantum, weights.w_e, weights.w_q,
                                  max_clients=max(256, len(self._rt.client_names) + 1))
        self.tree = DeviceRadixTree(track_workers=True, n_workers=len(self._ids), runtime=self._rt,
                                    worker_ids=self._ids, _trie=self._dev.trie)

    # -- mirrors ------------------------------------------------------------
    def counter(self, client, worker) -> int:
        return self.q.get((client, worker), 0)

    def _cid(self, client) -> int:
        cid = self._rt.client_id(client)
        self._dev.reserve_clients(cid + 1)
        return cid

    def _push(self):
        if self.q.dirty:
            for key in self.q.dirty:
                if key in self.q:
                    c, w = key
                    self._dev.set_counter(self._cid(c), self._ids.index(w), int(self.q[key]))
            self.q.dirty.clear()
        if self.queue_size.dirty:
            for w in self.queue_size.dirty:
                self._dev.set_queue_size(self._ids.index(w), int(self.queue_size[w]))
            self.queue_size.dirty.clear()

    def _pull_row(self, client, cid):
        row, present = self._dev.counters(cid)
        for i, w in enumerate(self._ids):
            if present[i]:
                self.q._set((client, w), int(row[i]))

    def _mask(self, matched) -> int:
        m = 0
        for w in matched:
            if w in self._ids:
                m |= 1 << self._ids.index(w)
        return m

    # -- protocol -------------------------------------------------------------
    def select_worker(self, matched, client) -> int:
        """global_policies.py:107-114 on the device."""
        self._push()
        cid = self._cid(client)
        idx, _ = self._dev.select(cid, self._mask(matched))
        self._pull_row(client, cid)
        return self._ids[idx]

    def select(self, req, now):
        match_len, matched = self.tree.longest_match_workers(req.input_tokens, now=now)
        wid = self.select_worker(matched, req.client)
        return wid, match_len, matched

    def dispatch(self, req, now):
        """Dispatcher.dispatch (global_policies.py:40-46) as one device call:
        match, SelectWorker, queue_size += 1, q -= w_e*input_len, index insert."""
        self._push()
        cid = self._cid(req.client)
        did = self._rt.upload(req.input_tokens, req.client, req.arrival, req.rid)
        w, m, mask, _ = self._dev.dispatch(np.array([did], np.int32), np.array([cid], np.int32),
                                           np.array([now], np.int64))
        wid = self._ids[int(w[0])]
        matched = tuple(sorted(self._ids[b] for b in range(len(self._ids)) if int(mask[0]) >> b & 1))
        self.queue_size._set(wid, self.queue_size[wid] + 1)
        self._pull_row(req.client, cid)
        rec = _dispatch_record_cls()(req.rid, req.client, wid, int(m[0]), matched, now)
        self.records.append(rec)
        return rec

    def after_dispatch(self, req, wid, now) -> None:
        """global_policies.py:121-124 (only reached when called directly)."""
        key = (req.client, wid)
        self.q[key] = self.counter(req.client, wid) - self.weights.w_e * req.input_len
        self._push()
        self.tree.insert(req.input_tokens, now=now, worker=wid)

    def on_finish(self, client, worker, output_tokens, now) -> None:
        """global_policies.py:126-129 + Dispatcher.on_finish (51-52)."""
        self._push()
        self._dev.finish(self._cid(client), self._ids.index(worker), output_tokens)
        self.q._set((client, worker), self.counter(client, worker) - self.weights.w_q * output_tokens)
        self.queue_size._set(worker, self.queue_size[worker] - 1)

    def on_eviction(self, path, keep_len, worker, notice_time, now) -> None:
        self.tree.evict_notify(path, worker, keep_len, notice_time)

    def _min_queue(self, candidates) -> int:
        return min(candidates, key=lambda w: (self.queue_size[w], w))


__all__ = ["GpuDlpm", "GpuLpm", "GpuD2lpm", "DispatchRecord", "EvictedPath"]
