"""Thin object wrappers over the C ABI (numpy in, numpy out).

These are the handles the drop-in adapters (radix.py, policies.py) and the
benchmark use.  No scheduling logic lives here.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from ._lib import P32, P64, PU64, PU8, call


def _p32(a):
    return a.ctypes.data_as(P32)


def _p64(a):
    return a.ctypes.data_as(P64)


def _pu64(a):
    return a.ctypes.data_as(PU64)


def _pu8(a):
    return a.ctypes.data_as(PU8)


def host_register(arr: np.ndarray) -> None:
    """Page-lock a numpy buffer for DMA uploads (fs_host_register); keep the
    array alive and call host_unregister before it is freed."""
    L.load()
    call("fs_host_register", arr.ctypes.data_as(C.c_void_p), arr.nbytes)


def host_unregister(arr: np.ndarray) -> None:
    call("fs_host_unregister", arr.ctypes.data_as(C.c_void_p))


class Context:
    """One CUDA device: token arena + request table (fs_ctx)."""

    def __init__(self, device: int | str = 0, arena_tokens: int = 1 << 22, max_requests: int = 1 << 16):
        if isinstance(device, str):  # "cuda:N" / "cuda"
            device = int(device.split(":")[1]) if ":" in device else 0
        L.load()
        h = C.c_void_p()
        call("fs_ctx_create", device, arena_tokens, max_requests, C.byref(h))
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            L.load().fs_ctx_destroy(self._h)
            self._h = None

    def add_requests(self, flat: np.ndarray, offsets: np.ndarray, lens: np.ndarray,
                     clients: np.ndarray | None = None, labels: np.ndarray | None = None) -> np.ndarray:
        n = len(lens)
        flat = np.ascontiguousarray(flat, dtype=np.int32)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        lens = np.ascontiguousarray(lens, dtype=np.int32)
        cl = np.ascontiguousarray(clients if clients is not None else np.zeros(n), dtype=np.int32)
        lb = np.ascontiguousarray(labels if labels is not None else np.zeros(n), dtype=np.int64)
        out = np.zeros(max(n, 1), np.int32)
        if flat.size == 0:
            flat = np.zeros(1, np.int32)
        call("fs_requests_add", self._h, n, _p32(flat), _p64(offsets), _p32(lens), _p32(cl), _p64(lb), _p32(out))
        return out[:n]

    def add_request(self, tokens, client: int = 0, label: int = 0) -> int:
        a = np.ascontiguousarray(np.asarray(tokens, dtype=np.int64).reshape(-1))
        if a.size and (a.min() < 0 or a.max() >= 2 ** 31):
            raise L.FsError(L.FS_ERR_TOKEN_RANGE, "fs_requests_add", "token id outside [0, 2^31)")
        a = a.astype(np.int32)
        return int(self.add_requests(a, np.zeros(1, np.int64), np.array([a.size], np.int32),
                                     np.array([client], np.int32), np.array([label], np.int64))[0])

    def set_labels(self, ids: np.ndarray, labels: np.ndarray) -> None:
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        labels = np.ascontiguousarray(labels, dtype=np.int64)
        call("fs_requests_set_labels", self._h, len(ids), _p32(ids), _p64(labels))

    def set_clients(self, ids: np.ndarray, clients: np.ndarray) -> None:
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        cl = np.ascontiguousarray(clients, dtype=np.int32)
        call("fs_requests_set_clients", self._h, len(ids), _p32(ids), _p32(cl))

    def arena_read(self, off: int, n: int) -> np.ndarray:
        out = np.zeros(max(n, 1), np.int32)
        call("fs_arena_read", self._h, off, n, _p32(out))
        return out[:n]

    def request_info(self, rid: int):
        off = C.c_int64(); ln = C.c_int32()
        call("fs_request_info", self._h, rid, C.byref(off), C.byref(ln))
        return off.value, ln.value

    def request_tokens(self, rid: int) -> np.ndarray:
        off, ln = self.request_info(rid)
        return self.arena_read(off, ln)

    def sync(self):
        call("fs_ctx_sync", self._h)


@dataclass
class Records:
    """Eviction records (radix.py:217-249) as arena references."""
    src: np.ndarray
    length: np.ndarray
    keep: np.ndarray

    def __len__(self):
        return len(self.src)

    @staticmethod
    def empty():
        return Records(np.zeros(0, np.int64), np.zeros(0, np.int32), np.zeros(0, np.int32))


class Trie:
    """One device RadixTree (fs_trie)."""

    def __init__(self, ctx: Context, capacity=None, track_workers=False, n_workers=0, _handle=None):
        self.ctx = ctx
        self.capacity = capacity
        if _handle is not None:
            self._h = _handle
            self._owned = False
        else:
            h = C.c_void_p()
            call("fs_trie_create", ctx.handle, -1 if capacity is None else capacity,
                 1 if track_workers else 0, n_workers, C.byref(h))
            self._h = h
            self._owned = True

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._owned and self._h:
            L.load().fs_trie_destroy(self._h)
        self._h = None

    def stats(self):
        u = C.c_int64(); p = C.c_int64(); s = C.c_int64(); n = C.c_int64()
        call("fs_trie_stats", self._h, C.byref(u), C.byref(p), C.byref(s), C.byref(n))
        return u.value, p.value, s.value, n.value

    def match(self, ids, now: int = 0, stamp: bool = True):
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        n = len(ids)
        m = np.zeros(max(n, 1), np.int32); cv = np.zeros(max(n, 1), np.int32)
        call("fs_trie_match", self._h, n, _p32(ids), now, 1 if stamp else 0, _p32(m), _p32(cv))
        return m[:n], cv[:n]

    def read_records(self, n: int) -> Records:
        """Records of this trie's last operation (fs_trie_read_records)."""
        src = np.zeros(max(n, 1), np.int64); ln = np.zeros(max(n, 1), np.int32); kp = np.zeros(max(n, 1), np.int32)
        if n:
            call("fs_trie_read_records", self._h, 0, n, _p64(src), _p32(ln), _p32(kp))
        return Records(src[:n], ln[:n], kp[:n])

    def _op(self, name, *args):
        rs = L.FsRecords(0, None, None, None, 0)
        err = None
        try:
            call(name, self._h, *args, C.byref(rs))
        except L.FsError as e:
            if e.code != L.FS_ERR_CACHE_FULL:
                raise
            err = e
        return self.read_records(rs.n_rec), err

    def insert(self, rid: int, now: int = 0, worker: int = -1):
        """-> (new_len, path node, Records, CacheFull error or None)"""
        nl = C.c_int32(); node = C.c_int32()
        recs, err = self._op("fs_trie_insert", rid, now, worker, C.byref(nl), C.byref(node))
        return nl.value, node.value, recs, err

    def admit(self, rid: int, now: int = 0):
        """-> (mlen, path node, Records, CacheFull error or None)"""
        m = C.c_int32(); node = C.c_int32()
        recs, err = self._op("fs_trie_admit", rid, now, C.byref(m), C.byref(node))
        return m.value, node.value, recs, err

    def pin(self, node: int):
        call("fs_trie_pin", self._h, node)

    def unpin(self, node: int):
        call("fs_trie_unpin", self._h, node)

    def unpin_many(self, nodes):
        nodes = np.ascontiguousarray(nodes, dtype=np.int32)
        call("fs_trie_unpin_many", self._h, len(nodes), _p32(nodes))

    def unpin_many_async(self, nodes):
        """unpin_many without waiting (fs_trie_unpin_many_async): errors and the
        device time surface at the next fill_end / last_ms / unpin_many."""
        nodes = np.ascontiguousarray(nodes, dtype=np.int32)
        call("fs_trie_unpin_many_async", self._h, len(nodes), _p32(nodes))

    def evict_lru(self, needed: int) -> Records:
        recs, err = self._op("fs_trie_evict_lru", needed)
        return recs

    def longest_match_workers(self, rid: int, now: int = 0):
        m = C.c_int32(); mask = C.c_uint64()
        call("fs_trie_longest_match_workers", self._h, rid, now, C.byref(m), C.byref(mask))
        return m.value, mask.value

    def evict_notify(self, path_src: int, path_len: int, worker: int, keep_len: int, notice_time: int):
        call("fs_trie_evict_notify", self._h, path_src, path_len, worker, keep_len, notice_time)

    def last_ms(self) -> float:
        """Device time of the last unpin_many (fs_trie_last_ms)."""
        v = C.c_float()
        call("fs_trie_last_ms", self._h, C.byref(v))
        return v.value

    def evict_notify_many(self, src, length, worker, keep, when):
        """A round's notices in order, one launch (fs_trie_evict_notify_many)."""
        src = np.ascontiguousarray(src, dtype=np.int64)
        n = len(src)
        if n == 0:
            return
        ln = np.ascontiguousarray(length, dtype=np.int32)
        wk = np.ascontiguousarray(worker, dtype=np.int32)
        kp = np.ascontiguousarray(keep, dtype=np.int32)
        wh = np.ascontiguousarray(when, dtype=np.int64)
        call("fs_trie_evict_notify_many", self._h, n, _p64(src), _p32(ln), _p32(wk), _p32(kp), _p64(wh))

    def export(self):
        n = C.c_int64()
        call("fs_trie_export", self._h, 0, C.byref(n), None, None, None, None, None, None, None)
        k = max(n.value, 1)
        src = np.zeros(k, np.int64); st = np.zeros(k, np.int32); en = np.zeros(k, np.int32)
        par = np.zeros(k, np.int32); ref = np.zeros(k, np.int32); la = np.zeros(k, np.int64)
        wm = np.zeros(k, np.uint64)
        call("fs_trie_export", self._h, k, C.byref(n), _p64(src), _p32(st), _p32(en), _p32(par), _p32(ref),
             _p64(la), _pu64(wm))
        m = n.value
        return {"src": src[:m], "start": st[:m], "end": en[:m], "parent": par[:m], "ref": ref[:m],
                "last_access": la[:m], "wmask": wm[:m]}

    def dump(self, worker_ids=None):
        """RadixTree.dump (radix.py:306-318): pre-order, children by first token."""
        tab = self.export()
        par = tab["parent"]
        alive = [i for i in range(1, len(par)) if par[i] >= 0]
        paths = {}
        firsts = {}
        for i in alive:
            paths[i] = self.ctx.arena_read(int(tab["src"][i]), int(tab["end"][i]))
            firsts[i] = int(paths[i][tab["start"][i]])
        kids = {}
        for i in alive:
            kids.setdefault(int(par[i]), []).append(i)
        out = []

        def rec(node):
            for ch in sorted(kids.get(node, ()), key=lambda x: firsts[x]):
                wm = int(tab["wmask"][ch])
                ws = [w for w in range(64) if wm >> w & 1]
                if worker_ids is not None:
                    ws = sorted(worker_ids[w] for w in ws)
                out.append((tuple(int(x) for x in paths[ch]), int(tab["ref"][ch]), tuple(ws),
                            int(tab["last_access"][ch])))
                rec(ch)

        rec(0)
        return out


@dataclass
class FillResult:
    adm_req: np.ndarray
    adm_mlen: np.ndarray
    adm_unpinned: np.ndarray
    adm_pinned_before: np.ndarray
    adm_node: np.ndarray
    adm_rec_end: np.ndarray
    records: Records
    n_queued: int
    used: int
    pinned: int
    device_ms: float
    phases_ms: list = field(default_factory=list)
    stats: list = field(default_factory=list)  # fs_worker_last_stats
    stats_ext: list = field(default_factory=list)  # fs_worker_last_stats_ext


def launch_count() -> int:
    return int(L.load().fs_launch_count())


class WorkerDev:
    """DLPM / LPM policy state + queue mirror of one worker (fs_worker)."""

    def __init__(self, ctx: Context, trie: Trie, policy: str, quantum: int, M: int, output_reserve: int,
                 w_e: int, w_q: int, max_clients: int = 256):
        h = C.c_void_p()
        call("fs_worker_create", ctx.handle, trie.handle, {"dlpm": 0, "lpm": 1, "vtc": 2}[policy], quantum or 1, M,
             output_reserve, w_e, w_q, max_clients, C.byref(h))
        self._h = h
        self.ctx = ctx
        self.trie = trie
        self.max_clients = max_clients
        self._cap = 0
        self._alloc(1024)

    def _alloc(self, cap):
        self._cap = cap
        self._req = np.zeros(cap, np.int32); self._mlen = np.zeros(cap, np.int32)
        self._unp = np.zeros(cap, np.int64); self._pinb = np.zeros(cap, np.int64)
        self._node = np.zeros(cap, np.int32); self._rend = np.zeros(cap, np.int64)
        if not hasattr(self, "_rcap"):
            self._rec_alloc(4096)

    def _rec_alloc(self, cap):
        # eviction records come back with the fill (one transfer set, one sync)
        self._rcap = cap
        self._rsrc = np.zeros(cap, np.int64); self._rlen = np.zeros(cap, np.int32); self._rkeep = np.zeros(cap, np.int32)

    def close(self):
        if self._h:
            L.load().fs_worker_destroy(self._h)
            self._h = None

    def reserve_clients(self, n: int):
        if n > self.max_clients:
            call("fs_worker_reserve_clients", self._h, n)
            self.max_clients = max(n, 2 * self.max_clients)

    def enqueue(self, ids):
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        call("fs_worker_enqueue", self._h, len(ids), _p32(ids))

    def mark_known(self, clients):
        c = np.ascontiguousarray(clients, dtype=np.int32)
        call("fs_worker_mark_known", self._h, len(c), _p32(c))

    def outputs(self, clients, counts):
        c = np.ascontiguousarray(clients, dtype=np.int32)
        n = np.ascontiguousarray(counts, dtype=np.int64)
        call("fs_worker_outputs", self._h, len(c), _p32(c), _p64(n))

    def set_counter(self, client: int, q: int):
        call("fs_worker_set_counter", self._h, client, q)

    def check_refill(self, clients) -> bool:
        c = np.ascontiguousarray(clients, dtype=np.int32)
        r = C.c_int()
        call("fs_worker_check_refill", self._h, len(c), _p32(c), C.byref(r))
        return bool(r.value)

    def counters(self, n: int | None = None):
        n = self.max_clients if n is None else n
        q = np.zeros(max(n, 1), np.int64); rf = np.zeros(max(n, 1), np.int64); kn = np.zeros(max(n, 1), np.uint8)
        call("fs_worker_counters", self._h, n, _p64(q), _p64(rf), _pu8(kn))
        return q[:n], rf[:n], kn[:n]

    def device_counters(self, n: int):
        q = np.zeros(max(n, 1), np.int64); rf = np.zeros(max(n, 1), np.int64)
        call("fs_worker_device_counters", self._h, n, _p64(q), _p64(rf))
        return q[:n], rf[:n]

    def set_client_ranks(self, ranks):
        """Vtc's name tie-break: rank of each dense client id's name."""
        r = np.ascontiguousarray(ranks, dtype=np.int32)
        call("fs_worker_set_client_ranks", self._h, len(r), _p32(r))

    def set_k1_full(self, full: bool) -> None:
        """Re-match every queued request from the root each fill (ablation of the
        incremental match; identical decisions)."""
        call("fs_worker_set_option", self._h, 1, 1 if full else 0)

    def queue_len(self) -> int:
        n = C.c_int64()
        call("fs_worker_queue_len", self._h, C.byref(n))
        return n.value

    def fill(self, now: int, generated_total: int, headroom: int) -> FillResult:
        res = self._result_struct()
        call("fs_worker_fill", self._h, now, generated_total, headroom, C.byref(res))
        return self._result(res)

    def fill_begin(self, now: int, generated_total: int, headroom: int) -> None:
        """Launch a fill and return at once (fs_worker_fill_begin): context
        uploads may run until fill_end; this worker and its tree are busy."""
        res = self._result_struct()
        call("fs_worker_fill_begin", self._h, now, generated_total, headroom)
        self._res = res

    def fill_end(self) -> FillResult:
        res, self._res = getattr(self, "_res", None), None
        if res is None:
            res = self._result_struct()  # nothing in flight: the call below reports it
        call("fs_worker_fill_end", self._h, C.byref(res))
        return self._result(res)

    def _result_struct(self):
        qlen = self.queue_len()
        if qlen + 1 > self._cap:
            self._alloc(max(qlen + 1, 2 * self._cap))
        res = L.FsFillResult()
        res.cap_adm = self._cap
        res.adm_req = _p32(self._req); res.adm_mlen = _p32(self._mlen); res.adm_unpinned = _p64(self._unp)
        res.adm_pinned_before = _p64(self._pinb); res.adm_path_node = _p32(self._node)
        res.adm_rec_end = _p64(self._rend)
        res.recs = L.FsRecords(self._rcap, _p64(self._rsrc), _p32(self._rlen), _p32(self._rkeep), 0)
        return res

    def _result(self, res) -> FillResult:
        nr = res.recs.n_rec
        if nr <= self._rcap:
            recs = Records(self._rsrc[:nr].copy(), self._rlen[:nr].copy(), self._rkeep[:nr].copy())
        else:
            recs = self.trie.read_records(nr)
            self._rec_alloc(2 * nr)
        ph = (C.c_float * 4)()
        call("fs_worker_last_phases", self._h, ph)
        st = (C.c_int64 * 24)()
        call("fs_worker_last_stats", self._h, st)
        sx = (C.c_int64 * 8)()
        call("fs_worker_last_stats_ext", self._h, sx)
        a = res.n_adm
        return FillResult(self._req[:a].copy(), self._mlen[:a].copy(), self._unp[:a].copy(),
                          self._pinb[:a].copy(), self._node[:a].copy(), self._rend[:a].copy(),
                          recs, res.n_queued, res.used, res.pinned, res.device_ms, list(ph), list(st), list(sx))


class DispatcherDev:
    """D2LPM counters + global routing index (fs_dispatcher)."""

    def __init__(self, ctx: Context, D: int, quantum: int, w_e: int, w_q: int, max_clients: int = 256):
        h = C.c_void_p()
        call("fs_dispatcher_create", ctx.handle, D, quantum, w_e, w_q, max_clients, C.byref(h))
        self._h = h
        self.ctx = ctx
        self.D = D
        self.max_clients = max_clients
        self.trie = Trie(ctx, _handle=L.load().fs_dispatcher_tree(h))

    def close(self):
        if self._h:
            L.load().fs_dispatcher_destroy(self._h)
            self._h = None

    def reserve_clients(self, n: int):
        if n > self.max_clients:
            call("fs_dispatcher_reserve_clients", self._h, n)
            self.max_clients = max(n, 2 * self.max_clients)

    def set_policy(self, policy: str, theta: float = 0.5):
        """"d2lpm" (default) or "threshold" (ThresholdRouter, global_policies.py:135-161)."""
        call("fs_dispatcher_set_policy", self._h, {"d2lpm": 0, "threshold": 1}[policy], float(theta))

    def dispatch(self, ids, clients, nows):
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        cl = np.ascontiguousarray(clients, dtype=np.int32)
        nw = np.ascontiguousarray(nows, dtype=np.int64)
        n = len(ids)
        w = np.zeros(max(n, 1), np.int32); m = np.zeros(max(n, 1), np.int32)
        mk = np.zeros(max(n, 1), np.uint64); rd = np.zeros(max(n, 1), np.int64)
        call("fs_dispatch", self._h, n, _p32(ids), _p32(cl), _p64(nw), _p32(w), _p32(m), _pu64(mk), _p64(rd))
        return w[:n], m[:n], mk[:n], rd[:n]

    @staticmethod
    def prematch_record_bytes() -> int:
        return int(L.load().fs_prematch_record_bytes())

    def prematch(self, ids, dev_out_ptr: int):
        """Batch-start matches of `ids` (one rank's slice of an arrival batch)
        written to device memory at dev_out_ptr (fs_dispatch_prematch)."""
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        call("fs_dispatch_prematch", self._h, len(ids), _p32(ids), C.c_void_p(dev_out_ptr))

    def dispatch_prematched(self, ids, clients, nows, dev_pre_ptr: int):
        """fs_dispatch with the batch's all-gathered prematch records."""
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        cl = np.ascontiguousarray(clients, dtype=np.int32)
        nw = np.ascontiguousarray(nows, dtype=np.int64)
        n = len(ids)
        w = np.zeros(max(n, 1), np.int32); m = np.zeros(max(n, 1), np.int32)
        mk = np.zeros(max(n, 1), np.uint64); rd = np.zeros(max(n, 1), np.int64)
        call("fs_dispatch_prematched", self._h, n, _p32(ids), _p32(cl), _p64(nw), C.c_void_p(dev_pre_ptr), _p32(w),
             _p32(m), _pu64(mk), _p64(rd))
        return w[:n], m[:n], mk[:n], rd[:n]

    def last_profile(self) -> np.ndarray:
        """SM cycles of the last dispatch chain (fs_dispatch_last_profile)."""
        p = np.zeros(16, np.int64)
        call("fs_dispatch_last_profile", self._h, _p64(p))
        return p

    def select(self, client: int, mask: int):
        w = C.c_int32(); r = C.c_int64()
        call("fs_dispatch_select", self._h, client, mask, C.byref(w), C.byref(r))
        return w.value, r.value

    def finish(self, client: int, worker: int, out: int):
        call("fs_dispatch_finish", self._h, client, worker, out)

    def finish_many(self, clients, workers, outs):
        cl = np.ascontiguousarray(clients, dtype=np.int32)
        if len(cl) == 0:
            return
        wk = np.ascontiguousarray(workers, dtype=np.int32)
        ot = np.ascontiguousarray(outs, dtype=np.int64)
        call("fs_dispatch_finish_many", self._h, len(cl), _p32(cl), _p32(wk), _p64(ot))

    def set_counter(self, client: int, worker: int, q: int):
        call("fs_dispatch_set_counter", self._h, client, worker, q)

    def set_queue_size(self, worker: int, size: int):
        call("fs_dispatch_set_queue_size", self._h, worker, size)

    def counters(self, client: int):
        q = np.zeros(self.D, np.int64); pr = np.zeros(self.D, np.uint8)
        call("fs_dispatch_counters", self._h, client, _p64(q), _pu8(pr))
        return q, pr

    def queue_sizes(self):
        s = np.zeros(self.D, np.int64)
        call("fs_dispatch_queue_sizes", self._h, _p64(s))
        return s

    def device_counters(self, n_clients: int):
        n = n_clients * self.D
        q = np.zeros(max(n, 1), np.int64); pr = np.zeros(max(n, 1), np.uint8); qs = np.zeros(self.D, np.int64)
        call("fs_dispatch_device_counters", self._h, n, _p64(q), _pu8(pr), _p64(qs))
        return q[:n], pr[:n], qs
