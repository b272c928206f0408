"""ctypes binding of libfsb200.so (include/fairsched_b200.h).

Loading never falls back to a CPU path: if the shared library is missing the
import raises, and every call that needs a GPU fails with FS_ERR_CUDA.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FS_LIB_PATH") or os.path.join(HERE, "libfsb200.so")  # override: build experiments

FS_OK = 0
FS_ERR_INVALID = 1
FS_ERR_CUDA = 2
FS_ERR_CACHE_FULL = 3
FS_ERR_TOKEN_RANGE = 4
FS_ERR_NOMEM = 5
FS_ERR_INTERNAL = 6
FS_ERR_UNDERFLOW = 7

vp = C.c_void_p
i32, i64, u64, u8 = C.c_int32, C.c_int64, C.c_uint64, C.c_uint8
P32, P64, PU64, PU8 = C.POINTER(i32), C.POINTER(i64), C.POINTER(u64), C.POINTER(u8)
PF = C.POINTER(C.c_float)
PP = C.POINTER(vp)
PI = C.POINTER(C.c_int)


class FsRecords(C.Structure):
    _fields_ = [("rec_cap", i64), ("rec_src", P64), ("rec_len", P32), ("rec_keep", P32), ("n_rec", i64)]


class FsFillResult(C.Structure):
    _fields_ = [
        ("cap_adm", i64),
        ("adm_req", P32),
        ("adm_mlen", P32),
        ("adm_unpinned", P64),
        ("adm_pinned_before", P64),
        ("adm_path_node", P32),
        ("adm_rec_end", P64),
        ("recs", FsRecords),
        ("n_adm", i64),
        ("n_queued", i64),
        ("used", i64),
        ("pinned", i64),
        ("device_ms", C.c_float),
    ]


PREC = C.POINTER(FsRecords)
PFILL = C.POINTER(FsFillResult)

SIGNATURES = {
    "fs_last_error": (C.c_char_p, []),
    "fs_version": (C.c_int, []),
    "fs_device_count": (C.c_int, [PI]),
    "fs_host_register": (C.c_int, [vp, i64]),
    "fs_host_unregister": (C.c_int, [vp]),
    "fs_ctx_create": (C.c_int, [C.c_int, i64, i64, PP]),
    "fs_ctx_destroy": (C.c_int, [vp]),
    "fs_ctx_sync": (C.c_int, [vp]),
    "fs_requests_add": (C.c_int, [vp, i64, P32, P64, P32, P32, P64, P32]),
    "fs_requests_add_expanded": (C.c_int, [vp, i64, P64, P32, P32, i64, PU8, P64, P32, P32, P64, P32]),
    "fs_requests_set_labels": (C.c_int, [vp, i64, P32, P64]),
    "fs_requests_set_clients": (C.c_int, [vp, i64, P32, P32]),
    "fs_requests_count": (C.c_int, [vp, P64]),
    "fs_request_info": (C.c_int, [vp, i32, P64, P32]),
    "fs_arena_read": (C.c_int, [vp, i64, i64, P32]),
    "fs_trie_create": (C.c_int, [vp, i64, C.c_int, C.c_int, PP]),
    "fs_trie_destroy": (C.c_int, [vp]),
    "fs_trie_stats": (C.c_int, [vp, P64, P64, P64, P64]),
    "fs_trie_match": (C.c_int, [vp, i64, P32, i64, C.c_int, P32, P32]),
    "fs_trie_read_records": (C.c_int, [vp, i64, i64, P64, P32, P32]),
    "fs_trie_insert": (C.c_int, [vp, i32, i64, i32, P32, P32, PREC]),
    "fs_trie_admit": (C.c_int, [vp, i32, i64, P32, P32, PREC]),
    "fs_trie_pin": (C.c_int, [vp, i32]),
    "fs_trie_unpin": (C.c_int, [vp, i32]),
    "fs_trie_unpin_many": (C.c_int, [vp, i64, P32]),
    "fs_trie_unpin_many_async": (C.c_int, [vp, i64, P32]),
    "fs_trie_last_ms": (C.c_int, [vp, PF]),
    "fs_trie_evict_lru": (C.c_int, [vp, i64, PREC]),
    "fs_trie_longest_match_workers": (C.c_int, [vp, i32, i64, P32, PU64]),
    "fs_trie_evict_notify": (C.c_int, [vp, i64, i32, i32, i32, i64]),
    "fs_trie_evict_notify_many": (C.c_int, [vp, i64, P64, P32, P32, P32, P64]),
    "fs_trie_last_notify_profile": (C.c_int, [vp, P64]),
    "fs_trie_export": (C.c_int, [vp, i64, P64, P64, P32, P32, P32, P32, P64, PU64]),
    "fs_worker_create": (C.c_int, [vp, vp, C.c_int, i64, i64, i64, i64, i64, i32, PP]),
    "fs_worker_destroy": (C.c_int, [vp]),
    "fs_worker_enqueue": (C.c_int, [vp, i64, P32]),
    "fs_worker_outputs": (C.c_int, [vp, i64, P32, P64]),
    "fs_worker_check_refill": (C.c_int, [vp, i64, P32, PI]),
    "fs_worker_counters": (C.c_int, [vp, i32, P64, P64, PU8]),
    "fs_worker_set_counter": (C.c_int, [vp, i32, i64]),
    "fs_worker_reserve_clients": (C.c_int, [vp, i32]),
    "fs_worker_mark_known": (C.c_int, [vp, i64, P32]),
    "fs_worker_fill": (C.c_int, [vp, i64, i64, i64, PFILL]),
    "fs_worker_fill_begin": (C.c_int, [vp, i64, i64, i64]),
    "fs_worker_fill_end": (C.c_int, [vp, PFILL]),
    "fs_worker_last_phases": (C.c_int, [vp, PF]),
    "fs_worker_last_gaps": (C.c_int, [vp, PF]),
    "fs_worker_set_option": (C.c_int, [vp, C.c_int, i64]),
    "fs_worker_last_stats": (C.c_int, [vp, P64]),
    "fs_dispatcher_set_policy": (C.c_int, [vp, C.c_int32, C.c_double]),
    "fs_worker_set_client_ranks": (C.c_int, [vp, C.c_int32, P32]),
    "fs_worker_last_stats_ext": (C.c_int, [vp, P64]),
    "fs_launch_count": (i64, []),
    "fs_worker_queue_len": (C.c_int, [vp, P64]),
    "fs_worker_device_counters": (C.c_int, [vp, i32, P64, P64]),
    "fs_dispatcher_create": (C.c_int, [vp, C.c_int, i64, i64, i64, i32, PP]),
    "fs_dispatcher_destroy": (C.c_int, [vp]),
    "fs_dispatcher_tree": (vp, [vp]),
    "fs_dispatch": (C.c_int, [vp, i64, P32, P32, P64, P32, P32, PU64, P64]),
    "fs_prematch_record_bytes": (C.c_int, []),
    "fs_dispatch_prematch": (C.c_int, [vp, i64, P32, vp]),
    "fs_dispatch_prematched": (C.c_int, [vp, i64, P32, P32, P64, vp, P32, P32, PU64, P64]),
    "fs_dispatch_finish": (C.c_int, [vp, i32, i32, i64]),
    "fs_dispatch_finish_many": (C.c_int, [vp, i64, P32, P32, P64]),
    "fs_dispatch_counters": (C.c_int, [vp, i32, P64, PU8]),
    "fs_dispatch_queue_sizes": (C.c_int, [vp, P64]),
    "fs_dispatch_select": (C.c_int, [vp, i32, u64, P32, P64]),
    "fs_dispatch_set_counter": (C.c_int, [vp, i32, i32, i64]),
    "fs_dispatch_set_queue_size": (C.c_int, [vp, i32, i64]),
    "fs_dispatcher_reserve_clients": (C.c_int, [vp, i32]),
    "fs_dispatch_last_profile": (C.c_int, [vp, P64]),
    "fs_dispatch_device_counters": (C.c_int, [vp, i64, P64, PU8, P64]),
    "fs_verify_pairs": (C.c_int, [C.c_int, i32, P64, P64, P64, P64, P64, P64, C.c_int, P64, P64, P64, P32]),
    "fs_verify_vs_any": (C.c_int, [C.c_int, i32, P64, P64, P64, P64, P64, P64, i64, P32, P64, P64, P64, P32]),
}

_lib = None


class FsError(RuntimeError):
    def __init__(self, code: int, fn: str, msg: str):
        super().__init__(f"{fn} failed with status {code}: {msg}")
        self.code = code


def load():
    """Load libfsb200.so (build it with __graft_entry__.build() / python -m paper_2501_14312_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("FS_LIB_PATH") and not hasattr(lib, name):
            continue  # an older build under A/B comparison: calls to it fail loudly
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def call(name: str, *args) -> None:
    """Call an fs_* status-returning entry point; raise FsError on failure."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != FS_OK:
        msg = lib.fs_last_error()
        raise FsError(rc, name, msg.decode() if msg else "")
