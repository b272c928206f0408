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
from .runtime import get_runtime, runtime_for_dispatcher


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


class GpuVtc(_GpuLocalPolicy):
    """Vtc (local_policies.py:139-195): the fill -- least-served client first,
    its earliest request, can_add, admit, full-input charge -- on the device
    (k_vtc); the enqueue-time counter lift and the output charge are the
    reference's host logic, pushed to the device before each fill."""

    name = "vtc"
    _policy = "vtc"

    def __init__(self):
        super().__init__(1)
        self.counter = _TrackedDict()
        self._ranked = -1

    def _active_clients(self):
        w = self.worker
        q = w.queue
        active = set(q._clients) if hasattr(q, "_clients") else {r.client for r in q}
        active.update(e.request.client for e in w.batch.values())
        return active

    def on_request_enqueued(self, req, was_active: bool) -> None:
        i = req.client  # local_policies.py:158-166
        if not was_active:
            others = self._active_clients() - {i}
            known = [self.counter[j] for j in others if j in self.counter]
            lift = min(known) if known else 0
            self.counter[i] = max(self.counter.get(i, 0), lift)
        else:
            self.counter.setdefault(i, 0)
        super().on_request_enqueued(req, was_active)

    def _push_counters(self):
        dev = self._device()
        rt = self._rt
        for c in self.counter.dirty:
            rt.client_id(c)
        dev.reserve_clients(len(rt.client_names) + 1)
        if self._ranked != len(rt.client_names):
            # sorted(queued, key=(counter, name)) tie-break: the names' order
            names = rt.client_names
            order = sorted(range(len(names)), key=lambda k: str(names[k]))
            ranks = np.zeros(len(names), np.int32)
            ranks[np.asarray(order, np.int64)] = np.arange(len(names), dtype=np.int32)
            dev.set_client_ranks(ranks)
            self._ranked = len(names)
        for c in self.counter.dirty:
            if c in self.counter:
                dev.set_counter(rt.client_id(c), int(self.counter[c]))
        self.counter.dirty.clear()

    def _pull_counters(self):
        q, _, _ = self._dev.counters()
        for c in self.counter:
            self.counter._set(c, int(q[self._rt.client_id(c)]))

    def on_outputs(self, counts) -> None:
        """local_policies.py:191-194 (mirror + device delta for the next fill)."""
        if not counts:
            return
        dev = self._device()
        w_q = self.worker.weights.w_q
        cids, ns = [], []
        for client, n in counts.items():
            self.counter._set(client, self.counter.get(client, 0) + w_q * n)
            cids.append(self._rt.client_id(client))
            ns.append(n)
        dev.outputs(np.asarray(cids, np.int32), np.asarray(ns, np.int64))

    def counters(self):
        return dict(self.counter)


# ---------------------------------------------------------------------------
# Routers on the device index (D2LPM, ThresholdRouter)
# ---------------------------------------------------------------------------


def _arrival_run(now):
    """The reference runner's pending arrivals at `now`, in processing order.

    Events are processed by (time, kind, seq) (engine.py:106-116) and
    REQUEST_ARRIVAL ranks first within a timestamp (engine.py:40-45), so the
    arrivals already queued at `now` are dispatched back to back: no finish,
    step or eviction notice -- nothing else that touches the dispatcher --
    can come between them (notices of fills triggered by these arrivals are
    scheduled events of a later rank).  Found through the runner's `arrive`
    frame (runner.py:305-317); None when not called from it."""
    f = sys._getframe(1)
    for _ in range(4):  # _arrival_run <- dispatch <- arrive
        f = f.f_back
        if f is None or f.f_code.co_name == "arrive":
            break
    if f is None or f.f_code.co_name != "arrive" or "sim" not in f.f_locals or \
            not f.f_globals.get("__name__", "").endswith("runner"):
        return None
    sim = f.f_locals["sim"]
    heap = getattr(sim, "_heap", None)
    if heap is None:
        return None
    mod = sys.modules.get("fairsched.requests")
    req_cls = getattr(mod, "Request", None)
    run = []
    for t, kind, seq, ev in heap:
        if t != now or kind != 0 or getattr(ev, "cancelled", False):
            continue
        cb = ev.callback
        d = getattr(cb, "__defaults__", None)
        if not d or (req_cls is not None and not isinstance(d[0], req_cls)):
            return None  # an arrival we cannot identify: no batching
        run.append((seq, d[0]))
    run.sort(key=lambda x: x[0])
    return [r for _, r in run]


class _GpuRouter:
    """Dispatcher protocol (global_policies.py:28-58) over fs_dispatcher: the
    tagged routing index, queue sizes (and D2LPM's q_{i,w}) on the device.

    dispatch() of the first arrival of a same-timestamp run dispatches the
    whole run in one device call (parallel batch-start matches,
    then the serial chain); the following dispatch() calls of that run are
    answered from it, in order.  Anything else arriving first is refused
    (RuntimeError) rather than answered from a diverged state."""

    uses_global_tree = True
    _policy = "d2lpm"

    def __init__(self, worker_ids, quantum=1, weights=None):
        self.worker_ids = list(worker_ids)
        self.queue_size = _TrackedDict({w: 0 for w in self.worker_ids})
        self.queue_size.dirty.clear()
        self.records = []
        self.q = _TrackedDict()
        self._ids = sorted(self.worker_ids)   # device worker index order == id order (_min_queue tie-break)
        self._rt = runtime_for_dispatcher()
        w_e, w_q = (weights.w_e, weights.w_q) if weights is not None else (1, 2)
        self._dev = DispatcherDev(self._rt.ctx, len(self._ids), quantum, w_e, w_q,
                                  max_clients=max(256, len(self._rt.client_names) + 1))
        self.tree = DeviceRadixTree(track_workers=True, n_workers=len(self._ids), runtime=self._rt,
                                    worker_ids=self._ids, _trie=self._dev.trie)
        self._ahead = []      # (request, now, (wid, mlen, matched)) dispatched ahead, in order
        self.batched = 0      # arrivals answered from a batch (diagnostic)

    # -- mirrors ------------------------------------------------------------
    def _cid(self, client) -> int:
        cid = self._rt.client_id(client)
        self._dev.reserve_clients(cid + 1)
        return cid

    def _push(self):
        if self.queue_size.dirty:
            for w in self.queue_size.dirty:
                self._dev.set_queue_size(self._ids.index(w), int(self.queue_size[w]))
            self.queue_size.dirty.clear()

    def _pull_row(self, client, cid):
        pass

    def _mask(self, matched) -> int:
        m = 0
        for w in matched:
            if w in self._ids:
                m |= 1 << self._ids.index(w)
        return m

    def _guard(self):
        if self._ahead:
            raise RuntimeError("dispatcher called between the arrivals of a same-timestamp run it "
                               "dispatched ahead (not the reference runner's event order)")

    # -- protocol -------------------------------------------------------------
    def select(self, req, now):
        raise NotImplementedError

    def dispatch(self, req, now):
        """Dispatcher.dispatch (global_policies.py:40-46) on the device:
        match, select, queue_size += 1, after_dispatch (D2LPM: q -= w_e*input_len;
        both: tagged index insert)."""
        if self._ahead:
            r0, t0, res = self._ahead[0]
            if r0 is not req or t0 != now:
                raise RuntimeError("arrival order differs from the same-timestamp run dispatched ahead")
            self._ahead.pop(0)
            self.batched += 1
        else:
            run = _arrival_run(now) or []
            batch = [req] + [r for r in run if r is not req]
            results = self._dispatch_batch(batch, now)
            res = results[0]
            self._ahead = [(r, now, x) for r, x in zip(batch[1:], results[1:])]
        wid, mlen, matched = res
        self.queue_size._set(wid, self.queue_size[wid] + 1)
        rec = _dispatch_record_cls()(req.rid, req.client, wid, mlen, matched, now)
        self.records.append(rec)
        return rec

    def _dispatch_batch(self, batch, now):
        self._push()
        cids = [self._cid(r.client) for r in batch]
        dids = [self._rt.upload(r.input_tokens, r.client, r.arrival, r.rid) for r in batch]
        w, m, mask, _ = self._dev.dispatch(np.asarray(dids, np.int32), np.asarray(cids, np.int32),
                                           np.full(len(batch), now, np.int64))
        out = []
        for k, r in enumerate(batch):
            wid = self._ids[int(w[k])]
            matched = tuple(sorted(self._ids[b] for b in range(len(self._ids)) if int(mask[k]) >> b & 1))
            out.append((wid, int(m[k]), matched))
        for r, cid in zip(batch, cids):
            self._pull_row(r.client, cid)
        return out

    def after_dispatch(self, req, wid, now) -> None:
        self._guard()
        self.tree.insert(req.input_tokens, now=now, worker=wid)

    def on_finish(self, client, worker, output_tokens, now) -> None:
        """Dispatcher.on_finish (global_policies.py:51-52) (+ D2lpm's charge)."""
        self._guard()
        self._push()
        self._dev.finish(self._cid(client), self._ids.index(worker), output_tokens)
        self.queue_size._set(worker, self.queue_size[worker] - 1)

    def on_eviction(self, path, keep_len, worker, notice_time, now) -> None:
        self._guard()
        self.tree.evict_notify(path, worker, keep_len, notice_time)

    def _min_queue(self, candidates) -> int:
        return min(candidates, key=lambda w: (self.queue_size[w], w))


class GpuD2lpm(_GpuRouter):
    """D2lpm (global_policies.py:88-132) with the routing index, q_{i,w} and the
    SelectWorker chain on the device."""

    name = "d2lpm"

    def __init__(self, worker_ids, quantum, weights):
        if quantum <= 0:
            raise ValueError("quantum must be positive")
        super().__init__(worker_ids, quantum, weights)
        self.quantum = quantum
        self.weights = weights

    def counter(self, client, worker) -> int:
        return self.q.get((client, worker), 0)

    def _push(self):
        if self.q.dirty:
            for key in self.q.dirty:
                if key in self.q:
                    c, w = key
                    self._dev.set_counter(self._cid(c), self._ids.index(w), int(self.q[key]))
            self.q.dirty.clear()
        super()._push()

    def _pull_row(self, client, cid):
        row, present = self._dev.counters(cid)
        for i, w in enumerate(self._ids):
            if present[i]:
                self.q._set((client, w), int(row[i]))

    def select_worker(self, matched, client) -> int:
        """global_policies.py:107-114 on the device."""
        self._guard()
        self._push()
        cid = self._cid(client)
        idx, _ = self._dev.select(cid, self._mask(matched))
        self._pull_row(client, cid)
        return self._ids[idx]

    def select(self, req, now):
        self._guard()
        match_len, matched = self.tree.longest_match_workers(req.input_tokens, now=now)
        wid = self.select_worker(matched, req.client)
        return wid, match_len, matched

    def after_dispatch(self, req, wid, now) -> None:
        """global_policies.py:121-124 (only reached when called directly)."""
        self._guard()
        key = (req.client, wid)
        self.q[key] = self.counter(req.client, wid) - self.weights.w_e * req.input_len
        self._push()
        self.tree.insert(req.input_tokens, now=now, worker=wid)

    def on_finish(self, client, worker, output_tokens, now) -> None:
        """global_policies.py:126-129 + Dispatcher.on_finish (51-52)."""
        super().on_finish(client, worker, output_tokens, now)
        self.q._set((client, worker), self.counter(client, worker) - self.weights.w_q * output_tokens)


class GpuThresholdRouter(_GpuRouter):
    """ThresholdRouter (global_policies.py:135-161): locality when the matched
    fraction of the input reaches theta, else the least-loaded worker -- the
    match, the select and the tagged insert in the device dispatch chain
    (fs_dispatcher_set_policy FS_DISPATCH_THRESHOLD), batched like D2LPM."""

    name = "threshold"

    def __init__(self, worker_ids, theta):
        if not 0.0 <= theta <= 1.0:
            raise ValueError("theta must be in [0, 1]")
        super().__init__(worker_ids)
        self.theta = theta
        self._dev.set_policy("threshold", theta)

    def select(self, req, now):
        self._guard()
        match_len, matched = self.tree.longest_match_workers(req.input_tokens, now=now)
        if matched and req.input_len > 0 and match_len / req.input_len >= self.theta:
            wid = self._min_queue(sorted(matched))
        else:
            wid = self._min_queue(self.worker_ids)
        return wid, match_len, matched


__all__ = ["GpuDlpm", "GpuLpm", "GpuVtc", "GpuD2lpm", "GpuThresholdRouter", "DispatchRecord", "EvictedPath"]
