"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's token universe.

Restates, with hashlib, the three functions that turn a trace into token ids
(`fairsched/requests.py`, arXiv 2501.14312):

* `token_block`   -- `_token_block`  requests.py:89-92
* `expand_tokens` -- `expand_tokens` requests.py:95-102
* `materialize`   -- `Trace.materialize` requests.py:134-161 (tokens and
  output lengths; no Request objects)

Pinned by tests/test_materialize.py against tests/golden/tokens.json, which
tests/golden/make_golden_tokens.py recorded from the real reference.  Only
tests/ and bench.py's CPU leg use this module; the product materializes on the
device (paper_2501_14312_b200/trace.py -> fs_requests_add_expanded).
"""
from __future__ import annotations

import hashlib


def token_block(namespace: str, block: int) -> tuple:
    # requests.py:89-92: sha256(f"{namespace}#{block}") -> 8 big-endian words % 2^31
    d = hashlib.sha256(f"{namespace}#{block}".encode()).digest()
    return tuple(int.from_bytes(d[i:i + 4], "big") % (1 << 31) for i in range(0, 32, 4))


def expand_tokens(namespace: str, length: int) -> tuple:
    # requests.py:95-102: blocks 0, 1, ... until >= length, then out[:length]
    out = []
    b = 0
    while len(out) < length:
        out.extend(token_block(namespace, b))
        b += 1
    return tuple(out[:length])


def materialize(records) -> tuple:
    """requests.py:134-161 over records exposing rid, shared_prefix_id,
    prefix_len, input_token_count, true_output_len (objects or dicts).
    Returns ({rid: tokens} in record order, {rid: true_output_len})."""
    inputs = {}
    out_lens = {}
    order = []
    for rec in records:
        g = rec.get if isinstance(rec, dict) else (lambda k, r=rec: getattr(r, k))
        rid, spid, plen = g("rid"), g("shared_prefix_id"), g("prefix_len")
        if spid.startswith("req:"):
            base = inputs[spid[4:]]
            if plen > len(base):
                raise ValueError(f"{rid}: prefix_len exceeds parent input")
            prefix = base[:plen]
        else:
            prefix = expand_tokens(spid, plen)
        suffix_len = g("input_token_count") - plen
        if suffix_len < 0:
            raise ValueError(f"{rid}: prefix_len exceeds input_token_count")
        toks = prefix + expand_tokens(f"sfx:{rid}", suffix_len)
        inputs[rid] = toks
        out_lens[rid] = g("true_output_len")
        order.append((rid, toks))
    return order, out_lens


def expand_segments(segs, out=None):
    """All requests of a paper_2501_14312_b200.trace.Segments, expanded by the C
    restatement (oracle/tokens.c, pthreads): returns (flat int32 tokens, offsets
    int64[n+1]).  Same tokens as expand_tokens per segment.  `out`: an int32
    buffer to expand into (at least the total token count; lets a caller lay
    several streams out back to back without a copy)."""
    import ctypes as C
    import os
    import subprocess

    import numpy as np

    here = os.path.dirname(os.path.abspath(__file__))
    lib_path = os.path.join(here, "libtokens.so")
    src = os.path.join(here, "tokens.c")
    if not os.path.exists(lib_path) or os.path.getmtime(lib_path) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", here, "libtokens.so"], check=True)
    lib = C.CDLL(lib_path)
    fn = lib.or_expand_segments
    fn.restype = C.c_int64
    n = len(segs.seg_first) - 1
    sf = np.ascontiguousarray(segs.seg_first, np.int64)
    sn = np.ascontiguousarray(segs.seg_ns, np.int32)
    sl = np.ascontiguousarray(segs.seg_len, np.int32)
    nb = np.ascontiguousarray(segs.ns_bytes, np.uint8)
    no = np.ascontiguousarray(segs.ns_off, np.int64)
    nl = np.ascontiguousarray(segs.ns_len, np.int32)
    total = int(sl.astype(np.int64).sum())
    if out is None:
        out = np.zeros(max(total, 1), np.int32)
    assert out.dtype == np.int32 and out.flags.c_contiguous and len(out) >= total
    offs = np.zeros(n + 1, np.int64)
    P = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
    fn(C.c_int64(n), P(sf, C.c_int64), P(sn, C.c_int32), P(sl, C.c_int32), P(nb, C.c_uint8), P(no, C.c_int64),
       P(nl, C.c_int32), P(out, C.c_int32), P(offs, C.c_int64))
    return out[:total], offs
