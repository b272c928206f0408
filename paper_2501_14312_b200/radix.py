"""DeviceRadixTree: the reference RadixTree surface (radix.py:48-340) on the device trie.

Every structural operation runs on the GPU through the C ABI; this class only
translates Python token tuples to device request ids, keeps host mirrors of
used/pinned tokens, and fires `on_evict` for the eviction records the device
emitted (radix.py:247-249), in order.

Replay mode: a device-side DLPM fill (policies.GpuDlpm) performs all of its
admissions on the GPU and then lets the unchanged reference Worker.try_admit
(worker.py:112-135) run its host bookkeeping.  While an admission is armed,
probe()/admit()/pinned_tokens answer with the values the device observed at
that admission, and any disagreement with the reference's can_add raises.
"""
from __future__ import annotations

import sys
from collections.abc import Sequence

import numpy as np

from .device import Trie
from .runtime import get_runtime, runtime_for_worker, runtime_of_ctx


class CacheFull(Exception):
    """Raised when the budget cannot admit the tokens (radix.py:19-20)."""


_BOTH = {}


def _cache_full_cls():
    # when the reference is loaded, raise a type that is both its CacheFull and
    # this module's, so `except CacheFull` keeps working for callers of either
    # (reference code, and code written against this module before the
    # reference was imported)
    mod = sys.modules.get("fairsched.radix")
    ref = getattr(mod, "CacheFull", None) if mod is not None else None
    if ref is None or ref is CacheFull:
        return CacheFull
    cls = _BOTH.get(ref)
    if cls is None:
        cls = _BOTH[ref] = type("CacheFull", (ref, CacheFull), {"__module__": ref.__module__})
    return cls


class EvictedPath(Sequence):
    """Lazy token path of an eviction record: arena[src : src+n] on the device.

    Compares equal to the tuple of its tokens.  The D2LPM drop-in passes it to
    the device evict_notify by reference, without copying tokens to the host."""

    __slots__ = ("_ctx", "src", "n", "_t")

    def __init__(self, ctx, src: int, n: int):
        self._ctx = ctx
        self.src = int(src)
        self.n = int(n)
        self._t = None

    def tokens(self) -> tuple:
        if self._t is None:
            self._t = tuple(int(x) for x in self._ctx.arena_read(self.src, self.n))
        return self._t

    def __len__(self):
        return self.n

    def __getitem__(self, i):
        return self.tokens()[i]

    def __iter__(self):
        return iter(self.tokens())

    def __eq__(self, other):
        if isinstance(other, EvictedPath):
            return self.tokens() == other.tokens()
        if isinstance(other, (tuple, list)):
            return self.tokens() == tuple(other)
        return NotImplemented

    def __hash__(self):
        return hash(self.tokens())

    def __repr__(self):
        return f"EvictedPath({self.tokens()!r})"


class DevicePath(list):
    """Path handle of insert/admit: [deepest node id] (radix.py:164-172 only
    ever uses path[-1]; splits keep the deepest node's identity)."""


class DeviceRadixTree:
    def __init__(self, capacity=None, track_workers=False, *, n_workers=64, runtime=None, worker_ids=None,
                 _trie=None):
        self.capacity = capacity
        self.track_workers = track_workers
        self.on_evict = None
        # a worker's cache lives on that worker's context (plugin placement)
        self._rt = runtime or (get_runtime() if track_workers else runtime_for_worker())
        self._t = _trie if _trie is not None else Trie(self._rt.ctx, capacity, track_workers,
                                                      n_workers if track_workers else 0)
        self._worker_ids = worker_ids  # tag index -> worker id (global index of a dispatcher)
        self._armed = None

    # -- host mirrors ------------------------------------------------------
    @property
    def used_tokens(self) -> int:
        return self._t.stats()[0]

    @property
    def pinned_tokens(self) -> int:
        if self._armed is not None:
            res, k = self._armed
            return int(res.adm_pinned_before[k])
        return self._t.stats()[1]

    @property
    def device_trie(self) -> Trie:
        return self._t

    def _rid(self, tokens) -> int:
        return self._rt.upload(tokens)

    def _tag(self, worker):
        if worker is None:
            return -1
        if self._worker_ids is not None:
            return self._worker_ids.index(worker)
        return int(worker)

    def _fire(self, recs) -> list:
        ctx = self._rt.ctx
        out = []
        for s, n, k in zip(recs.src, recs.length, recs.keep):
            out.append((EvictedPath(ctx, int(s), int(n)), int(k)))
        if self.on_evict is not None:
            for path, keep in out:
                self.on_evict(path, keep, len(path) - keep)
        return out

    # -- replay (device fill -> reference try_admit) -----------------------
    def _arm(self, res, k: int, rid: int):
        self._armed = (res, k)
        self._armed_rid = rid

    def _disarm(self):
        self._armed = None

    def _check_armed(self, tokens):
        # the armed request's own row, or another row of the very same tuple
        # (two requests may share one tuple object: runtime.DeviceRuntime.upload)
        if self._rt.lookup(tokens) != self._armed_rid and self._rt.tokens_of(self._armed_rid) is not tokens:
            raise RuntimeError("device fill replay desynchronised: try_admit called for a different request")

    # -- traversal (radix.py:83-110) ---------------------------------------
    def match_prefix(self, tokens, now=0, update_access=True):
        m, _ = self._t.match([self._rid(tokens)], now, stamp=update_access)
        return int(m[0]), []

    def probe(self, tokens):
        if self._armed is not None:
            self._check_armed(tokens)
            res, k = self._armed
            return int(res.adm_mlen[k]), int(res.adm_unpinned[k])
        m, cov = self._t.match([self._rid(tokens)], 0, stamp=False)
        return int(m[0]), int(m[0] - cov[0])

    def probe_many(self, token_seqs):
        """probe() of many sequences in one device call (no stamps, no side
        effects): (mlen, matched-unpinned) as int64 arrays."""
        m, cov = self._t.match([self._rid(t) for t in token_seqs], 0, stamp=False)
        m = m.astype(np.int64)
        return m, m - cov.astype(np.int64)

    def longest_match_workers(self, tokens, now=0):
        m, mask = self._t.longest_match_workers(self._rid(tokens), now)
        ws = {w for w in range(64) if mask >> w & 1}
        if self._worker_ids is not None:
            ws = {self._worker_ids[w] for w in ws}
        return m, ws

    # -- structure edits (radix.py:128-192) --------------------------------
    def insert(self, tokens, now=0, worker=None):
        nl, node, recs, err = self._t.insert(self._rid(tokens), now,
                                              self._tag(worker) if self.track_workers else -1)
        self._fire(recs)
        if err is not None:
            raise _cache_full_cls()(f"cannot free {nl} tokens")
        return nl, DevicePath([node] if node >= 0 else [])

    def pin(self, path) -> None:
        if path:
            self._t.pin(int(path[-1]))

    def unpin(self, path) -> None:
        if path:
            try:
                self._t.unpin(int(path[-1]))
            except Exception as e:  # radix.py:183
                raise AssertionError(str(e)) from e

    def admit(self, tokens, now=0):
        if self._armed is not None:
            self._check_armed(tokens)
            res, k = self._armed
            lo = int(res.adm_rec_end[k - 1]) if k > 0 else 0
            hi = int(res.adm_rec_end[k])
            from .device import Records
            sub = Records(res.records.src[lo:hi], res.records.length[lo:hi], res.records.keep[lo:hi])
            self._fire(sub)
            node = int(res.adm_node[k])
            self._armed = None
            return int(res.adm_mlen[k]), DevicePath([node] if node >= 0 else [])
        m, node, recs, err = self._t.admit(self._rid(tokens), now)
        self._fire(recs)
        if err is not None:
            raise _cache_full_cls()("cannot free tokens")
        return m, DevicePath([node] if node >= 0 else [])

    # -- eviction (radix.py:210-302) ---------------------------------------
    def evict_lru(self, needed, protect=None):
        if protect:
            raise ValueError("evict_lru with a protect set is internal to insert (radix.py:149)")
        recs = self._t.evict_lru(needed)
        out = self._fire(recs)
        return [(p.tokens(), k) for p, k in out]

    def evict_notify(self, path_tokens, worker, keep_len, notice_time) -> None:
        if isinstance(path_tokens, EvictedPath) and path_tokens._ctx is self._rt.ctx:
            src, n = path_tokens.src, path_tokens.n
        elif isinstance(path_tokens, EvictedPath) and self._cross_ctx(path_tokens) is not None:
            # a notice from a worker on another context (per-worker placement):
            # the path is a prefix of a request both sides hold -- no token copy
            src, n = self._cross_ctx(path_tokens), path_tokens.n
        else:
            rid = self._rid(path_tokens)
            src, n = self._rt.ctx.request_info(rid)
        w = self._tag(worker) if (self._worker_ids is None or worker in self._worker_ids) else -1
        self._t.evict_notify(src, n, w, keep_len, notice_time)

    def _cross_ctx(self, p):
        """Arena offset, on this tree's context, of the request whose row holds
        EvictedPath p on another context (None when unknown here)."""
        other = runtime_of_ctx(p._ctx)
        if other is None:
            return None
        did = other.did_at(p.src)
        toks = other.tokens_of(did) if did is not None else None
        if toks is None:
            return None
        mine = self._rt.lookup(toks)
        if mine is None:
            mine = self._rt.upload(toks)
        return int(self._rt.ctx.request_info(mine)[0])

    # -- diagnostics (radix.py:306-340) ------------------------------------
    def dump(self):
        return self._t.dump(self._worker_ids)

    def check(self) -> None:
        tab = self._t.export()
        par = tab["parent"]
        alive = [i for i in range(1, len(par)) if par[i] >= 0]
        total = sum(int(tab["end"][i] - tab["start"][i]) for i in alive)
        pinned = sum(int(tab["end"][i] - tab["start"][i]) for i in alive if tab["ref"][i] > 0)
        used, pin, _, _ = self._t.stats()
        assert total == used, f"used_tokens {used} != sum of edges {total}"
        assert pinned == pin
        assert all(tab["ref"][i] >= 0 for i in alive)
        if self.capacity is not None:
            assert used <= self.capacity
        firsts = {}
        for i in alive:
            key = (int(par[i]), int(self._rt.ctx.arena_read(int(tab["src"][i]) + int(tab["start"][i]), 1)[0]))
            assert key not in firsts, "sibling edges must start with distinct tokens"
            firsts[key] = i


def tokens_array(tokens) -> np.ndarray:
    return np.fromiter(tokens, dtype=np.int64, count=len(tokens))
