"""TEST INFRASTRUCTURE ONLY -- restatement of the reference trace materializer.

Rebuilds the exact token sequences the reference assigns to trace records
(requests.py:89-102 `_token_block` / `expand_tokens`, requests.py:134-161
`Trace.materialize`) so golden op traces can be stored as compact trace
records instead of raw tokens.  Pinned by the per-run token digests stored in
tests/golden/*.json.
"""
from __future__ import annotations

import hashlib
from functools import lru_cache

import numpy as np


@lru_cache(maxsize=1 << 16)
def _block(namespace: str, block: int) -> tuple:
    # requests.py:89-92: 8 big-endian uint32 words of sha256("ns#block") mod 2^31
    d = hashlib.sha256(f"{namespace}#{block}".encode()).digest()
    return tuple(int.from_bytes(d[i:i + 4], "big") & 0x7FFFFFFF for i in range(0, 32, 4))


def expand(namespace: str, length: int) -> list:
    # requests.py:95-102
    out = []
    b = 0
    while len(out) < length:
        out.extend(_block(namespace, b))
        b += 1
    return out[:length]


def materialize(records: list) -> dict:
    """records: dicts with TraceRecord fields (requests.py:70-86).
    Returns rid -> np.int32 token array (requests.py:134-161)."""
    inputs = {}
    for rec in records:
        sp = rec["shared_prefix_id"]
        if sp.startswith("req:"):
            base = inputs[sp[4:]]
            prefix = list(base[: rec["prefix_len"]])
        else:
            prefix = expand(sp, rec["prefix_len"])
        suffix = expand(f"sfx:{rec['rid']}", rec["input_token_count"] - rec["prefix_len"])
        inputs[rec["rid"]] = np.asarray(prefix + suffix, dtype=np.int32)
    return inputs


def tokens_digest(inputs: dict) -> str:
    h = hashlib.sha256()
    for rid in sorted(inputs):
        h.update(rid.encode())
        h.update(np.ascontiguousarray(inputs[rid], dtype="<i4").tobytes())
    return h.hexdigest()
