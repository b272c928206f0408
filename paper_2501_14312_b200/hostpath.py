"""Host bookkeeping fast path around the reference Worker.

With the decisions on the GPU, the reference Worker's own list bookkeeping is
the next wall in a serving run: `queue.remove(req)` is O(N) per admission
(worker.py:127), `enqueue` scans the queue for the client's activity
(worker.py:142-147), and the monitor's `has_admissible_waiting`
(worker.py:137-138, runner.py:354) probes the queued requests one by one --
one device round trip each on the device tree.  For workers whose policy is
one of this package's GPU policies:

* `FastQueue` replaces `worker.queue` (same iteration order, O(1) append /
  remove, per-client counts);
* `enqueue` answers `was_active` from the per-client counts (the batch scan is
  kept as is);
* `has_admissible_waiting` evaluates `Worker.can_add` (worker.py:100-109) for
  the whole queue from ONE batched device probe (fs_trie_match without
  stamps), in numpy;
* `Trace.materialize` (requests.py:134-161, run once per experiment by
  runner.py:247) takes its tokens from the device SHA-256 expander (k_expand,
  SURVEY §8f.2) instead of hashlib in Python.

Each is the reference computation restated exactly (same results, same side
effects -- probe has none); every other worker keeps the reference methods.
Installed and removed by plugin.install() / uninstall().
"""
from __future__ import annotations

import numpy as np

# below this queue length the reference's per-request probes are as cheap
_BATCH_PROBE_MIN = 8


class FastQueue:
    """list[Request] replacement: insertion order, O(1) remove by identity."""

    __slots__ = ("_d", "_clients")

    def __init__(self, items=()):
        self._d = {}
        self._clients = {}
        for r in items:
            self.append(r)

    def append(self, r) -> None:
        self._d[id(r)] = r
        self._clients[r.client] = self._clients.get(r.client, 0) + 1

    def remove(self, r) -> None:
        x = self._d.pop(id(r), None)
        if x is None:
            # list.remove semantics: the first element equal to r
            for k, v in self._d.items():
                if v == r:
                    x = self._d.pop(k)
                    break
            else:
                raise ValueError("FastQueue.remove(x): x not in queue")
        n = self._clients[x.client] - 1
        if n:
            self._clients[x.client] = n
        else:
            del self._clients[x.client]

    def has_client(self, client) -> bool:
        return client in self._clients

    def __iter__(self):
        return iter(list(self._d.values()))

    def __len__(self) -> int:
        return len(self._d)

    def __bool__(self) -> bool:
        return bool(self._d)

    def __contains__(self, r) -> bool:
        return id(r) in self._d or any(v == r for v in self._d.values())

    def __getitem__(self, i):
        return list(self._d.values())[i]

    def __repr__(self) -> str:
        return f"FastQueue({list(self._d.values())!r})"


def _gpu_worker(w) -> bool:
    from .policies import _GpuLocalPolicy
    return isinstance(getattr(w, "policy", None), _GpuLocalPolicy)


def _queue(w):
    q = w.queue
    if type(q) is list:
        q = FastQueue(q)
        w.queue = q
    return q


def make_enqueue(orig):
    def enqueue(self, req) -> None:
        # Worker.enqueue (worker.py:142-147)
        if not _gpu_worker(self):
            return orig(self, req)
        q = _queue(self)
        was_active = q.has_client(req.client) or any(
            e.request.client == req.client for e in self.batch.values())
        q.append(req)
        self.policy.on_request_enqueued(req, was_active)
        self.maybe_step()
    enqueue.__wrapped__ = orig
    return enqueue


def make_has_admissible_waiting(orig):
    def has_admissible_waiting(self) -> bool:
        # any(self.can_add(r) for r in self.queue)  (worker.py:137-138, 100-109)
        from .radix import DeviceRadixTree
        tree = self.tree
        if not _gpu_worker(self) or not isinstance(tree, DeviceRadixTree) or tree._armed is not None \
                or len(self.queue) < _BATCH_PROBE_MIN:
            return orig(self)
        reqs = list(self.queue)
        mlen, unpinned = tree.probe_many([r.input_tokens for r in reqs])
        lens = np.fromiter((r.input_len for r in reqs), np.int64, len(reqs))
        extend = lens - mlen
        footprint = tree.pinned_tokens + unpinned + extend
        reserve = self._reserved_headroom() + self.output_reserve
        ok = footprint + self.generated_total + reserve <= self.params.M
        cap = tree.capacity
        if cap:  # `footprint > (capacity or footprint)` is never true without a capacity
            ok &= footprint <= cap
        return bool(ok.any())
    has_admissible_waiting.__wrapped__ = orig
    return has_admissible_waiting


def host_tokens(records):
    """Every record's input tokens (Trace.materialize's recipe,
    requests.py:134-161, same errors) generated on the device by k_expand
    (SHA-256 per 8-token block, requests.py:89-102) and read back as tuples."""
    from .device import Context
    from .trace import add_segments, resolve
    segs, rids, clients, arrivals, out_lens = resolve(records)
    lens = segs.lens().astype(np.int64)
    n = len(rids)
    if n == 0:
        return [], rids, out_lens
    rows = (lens + 3) & ~3  # 16-B aligned rows, back to back (fs_requests_add_expanded)
    total = int(rows.sum())
    ctx = Context(int(__import__("os").environ.get("FS_B200_DEVICE", "0")), arena_tokens=total + 1024,
                  max_requests=n + 16)
    try:
        ids = add_segments(ctx, segs, np.zeros(n, np.int32), np.zeros(n, np.int64))
        base, _ = ctx.request_info(int(ids[0]))
        flat = ctx.arena_read(base, total) if total else np.zeros(0, np.int32)
        last, _ = ctx.request_info(int(ids[-1]))
        offs = np.zeros(n, np.int64)
        offs[1:] = np.cumsum(rows[:-1])
        if last - base != offs[-1]:
            raise RuntimeError("unexpected arena placement of materialized requests")
    finally:
        ctx.close()
    vals = flat.tolist()
    toks = [tuple(vals[o:o + l]) for o, l in zip(offs.tolist(), lens.tolist())]
    return toks, rids, out_lens


def make_materialize(orig):
    def materialize(self):
        # Trace.materialize (requests.py:134-161) with the tokens from the device
        from fairsched.requests import Request
        toks, rids, out_lens = host_tokens(self.records)
        requests = [Request(rid=rec.rid, client=rec.client, input_tokens=tk, arrival=rec.arrival_time,
                            parent=rec.parent_id) for rec, tk in zip(self.records, toks)]
        return requests, out_lens
    materialize.__wrapped__ = orig
    return materialize


_PATCHES = (("enqueue", make_enqueue), ("has_admissible_waiting", make_has_admissible_waiting))


def install(worker_cls, trace_cls=None) -> dict:
    saved = {}
    for name, make in _PATCHES:
        orig = getattr(worker_cls, name)
        saved[(worker_cls, name)] = orig
        setattr(worker_cls, name, make(orig))
    if trace_cls is not None:
        saved[(trace_cls, "materialize")] = trace_cls.materialize
        trace_cls.materialize = make_materialize(trace_cls.materialize)
    return saved


def uninstall(saved: dict) -> None:
    for (cls, name), orig in saved.items():
        setattr(cls, name, orig)
