"""TEST INFRASTRUCTURE ONLY -- ctypes front-end of the CPU oracle (fs_oracle.c).

The oracle is a literal C restatement of the reference decision path
(`fairsched` radix.py / local_policies.py / global_policies.py / worker.py,
arXiv 2501.14312).  Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline leg import this module; the product package never does.

Parity of the oracle against the reference is pinned by
tests/test_oracle_golden.py (golden op traces recorded from the real reference
by tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
U64P = C.POINTER(C.c_uint64)
U8P = C.POINTER(C.c_uint8)

OR_OK = 0
OR_CACHE_FULL = 3


class OracleCacheFull(Exception):
    """Mirror of fairsched.radix.CacheFull (radix.py:19-20)."""


def build() -> None:
    src = os.path.join(_HERE, "fs_oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        sig = {
            "or_tree_new": (C.c_void_p, [C.c_int64, C.c_int, C.c_int]),
            "or_tree_free": (None, [C.c_void_p]),
            "or_tree_used": (C.c_int64, [C.c_void_p]),
            "or_tree_pinned": (C.c_int64, [C.c_void_p]),
            "or_tree_seq": (C.c_int64, [C.c_void_p]),
            "or_common_prefix_len": (C.c_int32, [I32P, C.c_int32, C.c_int32, I32P, C.c_int32, C.c_int32]),
            "or_match_prefix": (C.c_int32, [C.c_void_p, I32P, C.c_int32, C.c_int64, C.c_int]),
            "or_probe": (C.c_int32, [C.c_void_p, I32P, C.c_int32, I64P]),
            "or_longest_match_workers": (C.c_int32, [C.c_void_p, I32P, C.c_int32, C.c_int64, U64P]),
            "or_insert": (C.c_int, [C.c_void_p, I32P, C.c_int32, C.c_int64, C.c_int, U64P, I32P]),
            "or_pin": (None, [C.c_void_p, C.c_uint64]),
            "or_unpin": (C.c_int, [C.c_void_p, C.c_uint64]),
            "or_admit": (C.c_int, [C.c_void_p, I32P, C.c_int32, C.c_int64, I32P, U64P]),
            "or_evict_lru": (C.c_int64, [C.c_void_p, C.c_int64]),
            "or_records_count": (C.c_int64, [C.c_void_p]),
            "or_record_len": (C.c_int32, [C.c_void_p, C.c_int64]),
            "or_record_keep": (C.c_int32, [C.c_void_p, C.c_int64]),
            "or_record_path": (None, [C.c_void_p, C.c_int64, I32P]),
            "or_evict_notify": (None, [C.c_void_p, I32P, C.c_int32, C.c_int, C.c_int32, C.c_int64]),
            "or_dump": (C.c_int64, [C.c_void_p, I64P, C.c_int64]),
            "or_worker_new": (C.c_void_p, [C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int64, C.c_int32]),
            "or_worker_free": (None, [C.c_void_p]),
            "or_worker_tree": (C.c_void_p, [C.c_void_p]),
            "or_worker_q": (I64P, [C.c_void_p]),
            "or_worker_refills": (I64P, [C.c_void_p]),
            "or_worker_on_enqueue": (None, [C.c_void_p, C.c_int32]),
            "or_worker_on_outputs": (None, [C.c_void_p, C.c_int32, C.c_int64]),
            "or_worker_check_refill": (C.c_int, [C.c_void_p, U8P]),
            "or_worker_fill": (C.c_int64, [C.c_void_p, I32P, I64P, I32P, I32P, I64P, C.c_int32, C.c_int64,
                                           C.c_int64, C.c_int64, I32P, I32P, I64P, I64P, U64P, I64P, I32P]),
            "or_fill_records_count": (C.c_int64, []),
            "or_fill_record_len": (C.c_int32, [C.c_int64]),
            "or_fill_record_keep": (C.c_int32, [C.c_int64]),
            "or_fill_record_path": (None, [C.c_int64, I32P]),
            "or_d2_new": (C.c_void_p, [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int32]),
            "or_d2_free": (None, [C.c_void_p]),
            "or_d2_tree": (C.c_void_p, [C.c_void_p]),
            "or_d2_q": (I64P, [C.c_void_p]),
            "or_d2_qset": (U8P, [C.c_void_p]),
            "or_d2_queue_size": (I64P, [C.c_void_p]),
            "or_d2_dispatch": (C.c_int, [C.c_void_p, I32P, C.c_int32, C.c_int32, C.c_int64, I32P, I32P, U64P]),
            "or_d2_finish": (None, [C.c_void_p, C.c_int32, C.c_int, C.c_int64]),
            "or_d2_eviction": (None, [C.c_void_p, I32P, C.c_int32, C.c_int32, C.c_int, C.c_int64]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _arr(tokens) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32).reshape(-1))
    return a


def _p32(a: np.ndarray):
    return a.ctypes.data_as(I32P)


def _p64(a: np.ndarray):
    return a.ctypes.data_as(I64P)


def parse_dump(buf: np.ndarray) -> list:
    """Decode or_dump's flat layout into RadixTree.dump() tuples (radix.py:306-318)."""
    out = []
    i = 0
    n = len(buf)
    while i < n:
        plen = int(buf[i]); i += 1
        path = tuple(int(x) for x in buf[i:i + plen]); i += plen
        ref = int(buf[i]); i += 1
        nw = int(buf[i]); i += 1
        workers = tuple(int(x) for x in buf[i:i + nw]); i += nw
        la = int(buf[i]); i += 1
        out.append((path, ref, workers, la))
    return out


def _dump_tree(ptr) -> list:
    L = lib()
    need = L.or_dump(ptr, None, 0)
    buf = np.zeros(max(need, 1), dtype=np.int64)
    L.or_dump(ptr, _p64(buf), need)
    return parse_dump(buf[:need])


class OracleTree:
    """RadixTree surface (radix.py:48-340) over the C oracle."""

    def __init__(self, capacity=None, track_workers=False, n_workers=64, _ptr=None, _owned=True):
        L = lib()
        self._ptr = _ptr if _ptr is not None else L.or_tree_new(-1 if capacity is None else capacity,
                                                              1 if track_workers else 0, n_workers)
        self._owned = _owned and _ptr is None
        self.capacity = capacity
        self.track_workers = track_workers

    def __del__(self):
        if getattr(self, "_owned", False) and self._ptr:
            lib().or_tree_free(self._ptr)
            self._ptr = None

    @property
    def used_tokens(self) -> int:
        return lib().or_tree_used(self._ptr)

    @property
    def pinned_tokens(self) -> int:
        return lib().or_tree_pinned(self._ptr)

    @property
    def seq(self) -> int:
        return lib().or_tree_seq(self._ptr)

    def match_prefix(self, tokens, now=0, update_access=True):
        a = _arr(tokens)
        return lib().or_match_prefix(self._ptr, _p32(a), len(a), now, 1 if update_access else 0), None

    def probe(self, tokens):
        a = _arr(tokens)
        unp = C.c_int64(0)
        m = lib().or_probe(self._ptr, _p32(a), len(a), C.byref(unp))
        return m, unp.value

    def longest_match_workers(self, tokens, now=0):
        a = _arr(tokens)
        mask = C.c_uint64(0)
        m = lib().or_longest_match_workers(self._ptr, _p32(a), len(a), now, C.byref(mask))
        return m, {w for w in range(64) if mask.value >> w & 1}

    def _records(self):
        L = lib()
        out = []
        for i in range(L.or_records_count(self._ptr)):
            n = L.or_record_len(self._ptr, i)
            buf = np.zeros(max(n, 1), dtype=np.int32)
            L.or_record_path(self._ptr, i, _p32(buf))
            out.append((tuple(int(x) for x in buf[:n]), L.or_record_keep(self._ptr, i)))
        return out

    def insert(self, tokens, now=0, worker=None):
        a = _arr(tokens)
        h = C.c_uint64(0)
        nl = C.c_int32(0)
        st = lib().or_insert(self._ptr, _p32(a), len(a), now, -1 if worker is None else worker,
                             C.byref(h), C.byref(nl))
        self.last_records = self._records()
        if st == OR_CACHE_FULL:
            raise OracleCacheFull(f"cannot free {nl.value} tokens")
        return nl.value, h.value

    def pin(self, handle):
        lib().or_pin(self._ptr, handle)

    def unpin(self, handle):
        if lib().or_unpin(self._ptr, handle) != 0:
            raise AssertionError("unpin underflow")

    def admit(self, tokens, now=0):
        a = _arr(tokens)
        m = C.c_int32(0)
        h = C.c_uint64(0)
        st = lib().or_admit(self._ptr, _p32(a), len(a), now, C.byref(m), C.byref(h))
        self.last_records = self._records()
        if st == OR_CACHE_FULL:
            raise OracleCacheFull("admit")
        return m.value, h.value

    def evict_lru(self, needed):
        lib().or_evict_lru(self._ptr, needed)
        return self._records()

    def evict_notify(self, path_tokens, worker, keep_len, notice_time):
        a = _arr(path_tokens)
        lib().or_evict_notify(self._ptr, _p32(a), len(a), worker, keep_len, notice_time)

    def dump(self):
        return _dump_tree(self._ptr)


class OracleWorker:
    """One worker's local tree + Dlpm/Lpm policy state (local_policies.py:74-136,
    worker.py:87-135) over the C oracle.  Clients are dense ints."""

    def __init__(self, capacity, M, output_reserve, w_e, w_q, policy, quantum, n_clients):
        self.L = lib()
        self.n_clients = n_clients
        self._ptr = self.L.or_worker_new(capacity, M, output_reserve, w_e, w_q,
                                         1 if policy == "lpm" else 0, quantum or 1, n_clients)
        self.tree = OracleTree(_ptr=self.L.or_worker_tree(self._ptr), _owned=False)
        self.tree.capacity = capacity

    def __del__(self):
        if getattr(self, "_ptr", None):
            self.L.or_worker_free(self._ptr)
            self._ptr = None

    def q(self) -> np.ndarray:
        return np.ctypeslib.as_array(self.L.or_worker_q(self._ptr), shape=(self.n_clients,)).copy()

    def set_q(self, c, v):
        self.L.or_worker_q(self._ptr)[c] = v

    def refills(self) -> np.ndarray:
        return np.ctypeslib.as_array(self.L.or_worker_refills(self._ptr), shape=(self.n_clients,)).copy()

    def on_enqueue(self, client: int):
        self.L.or_worker_on_enqueue(self._ptr, client)

    def on_outputs(self, client: int, n: int):
        self.L.or_worker_on_outputs(self._ptr, client, n)

    def check_refill(self, queued_clients) -> bool:
        flags = np.zeros(max(self.n_clients, 1), dtype=np.uint8)
        for c in queued_clients:
            flags[c] = 1
        return bool(self.L.or_worker_check_refill(self._ptr, flags.ctypes.data_as(U8P)))

    def fill(self, tokens: np.ndarray, offsets: np.ndarray, lens: np.ndarray, clients: np.ndarray,
             labels: np.ndarray, now: int, generated_total: int, headroom: int):
        """Returns dict with admissions (queue positions), mlen, unpinned, pinned_before,
        handles, per-admission record ends, records, sort-time mlen."""
        nq = len(lens)
        n = max(nq, 1)
        pos = np.zeros(n, np.int32); ml = np.zeros(n, np.int32); unp = np.zeros(n, np.int64)
        pb = np.zeros(n, np.int64); h = np.zeros(n, np.uint64); re = np.zeros(n, np.int64)
        sm = np.zeros(n, np.int32)
        tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        lens = np.ascontiguousarray(lens, dtype=np.int32)
        clients = np.ascontiguousarray(clients, dtype=np.int32)
        labels = np.ascontiguousarray(labels, dtype=np.int64)
        A = self.L.or_worker_fill(self._ptr, _p32(tokens), _p64(offsets), _p32(lens), _p32(clients),
                                  _p64(labels), nq, now, generated_total, headroom,
                                  _p32(pos), _p32(ml), _p64(unp), _p64(pb), h.ctypes.data_as(U64P),
                                  _p64(re), _p32(sm))
        if A < 0:
            raise OracleCacheFull("fill")
        recs = []
        for i in range(self.L.or_fill_records_count()):
            ln = self.L.or_fill_record_len(i)
            buf = np.zeros(max(ln, 1), dtype=np.int32)
            self.L.or_fill_record_path(i, _p32(buf))
            recs.append((buf[:ln].copy(), self.L.or_fill_record_keep(i)))
        return {
            "pos": pos[:A].copy(), "mlen": ml[:A].copy(), "unpinned": unp[:A].copy(),
            "pinned_before": pb[:A].copy(), "handles": [int(x) for x in h[:A]],
            "rec_end": re[:A].copy(), "records": recs, "sort_mlen": sm[:nq].copy(),
        }

    def unpin(self, handle):
        self.tree.unpin(handle)


class OracleD2lpm:
    """D2lpm dispatcher state over the C oracle (global_policies.py:88-132).
    Worker ids are 0..D-1; clients are dense ints."""

    def __init__(self, D, quantum, w_e, w_q, n_clients):
        self.L = lib()
        self.D = D
        self.n_clients = n_clients
        self._ptr = self.L.or_d2_new(D, quantum, w_e, w_q, n_clients)
        self.tree = OracleTree(_ptr=self.L.or_d2_tree(self._ptr), _owned=False)

    def __del__(self):
        if getattr(self, "_ptr", None):
            self.L.or_d2_free(self._ptr)
            self._ptr = None

    def dispatch(self, tokens, client, now):
        a = _arr(tokens)
        w = C.c_int32(0); m = C.c_int32(0); mask = C.c_uint64(0)
        self.L.or_d2_dispatch(self._ptr, _p32(a), len(a), client, now, C.byref(w), C.byref(m), C.byref(mask))
        return w.value, m.value, tuple(x for x in range(64) if mask.value >> x & 1)

    def on_finish(self, client, w, out):
        self.L.or_d2_finish(self._ptr, client, w, out)

    def on_eviction(self, path, keep_len, w, notice_time):
        a = _arr(path)
        self.L.or_d2_eviction(self._ptr, _p32(a), len(a), keep_len, w, notice_time)

    def q(self) -> dict:
        n = self.n_clients * self.D
        q = np.ctypeslib.as_array(self.L.or_d2_q(self._ptr), shape=(n,))
        s = np.ctypeslib.as_array(self.L.or_d2_qset(self._ptr), shape=(n,))
        return {(c, w): int(q[c * self.D + w]) for c in range(self.n_clients) for w in range(self.D)
                if s[c * self.D + w]}

    def queue_size(self) -> list:
        return list(np.ctypeslib.as_array(self.L.or_d2_queue_size(self._ptr), shape=(self.D,)))


def common_prefix_len(a, a_off, b, b_off) -> int:
    x = _arr(a); y = _arr(b)
    return lib().or_common_prefix_len(_p32(x), len(x), a_off, _p32(y), len(y), b_off)
