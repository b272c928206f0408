"""Trace materialization into the device token arena.

The reference expands every TraceRecord into a Python tuple of token ids
(`Trace.materialize`, requests.py:134-161; `expand_tokens` / `_token_block`,
requests.py:89-102): one SHA-256 per 8 tokens, in Python -- about 80 minutes
and 65 GB for a 1M-request, 8k-token queue.  Here the host only resolves
each record into *segments* -- leading slices `expand_tokens(ns, n)` of one
namespace -- and the device generates the tokens in place
(`fs_requests_add_expanded`, k_expand: a warp per segment, a lane per
8-token SHA-256 block).

Resolution follows Trace.materialize exactly:
  * shared_prefix_id "req:<rid>": the prefix is the parent's first prefix_len
    tokens, i.e. the parent's segments truncated (KeyError for an unknown
    parent, ValueError when prefix_len exceeds the parent's input);
  * any other id: expand_tokens(shared_prefix_id, prefix_len);
  * then expand_tokens(f"sfx:{rid}", input_token_count - prefix_len)
    (ValueError when negative).
"""
from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from ._lib import P32, P64, PU8, call


@dataclass
class Segments:
    """Requests as concatenations of namespace slices (the ABI's layout)."""
    seg_first: np.ndarray   # int64 [n+1]
    seg_ns: np.ndarray      # int32 [nseg]
    seg_len: np.ndarray     # int32 [nseg]
    ns_bytes: np.ndarray    # uint8, UTF-8 namespaces back to back
    ns_off: np.ndarray      # int64 [n_ns]
    ns_len: np.ndarray      # int32 [n_ns]

    @property
    def n(self) -> int:
        return len(self.seg_first) - 1

    def lens(self) -> np.ndarray:
        c = np.concatenate([[0], np.cumsum(self.seg_len, dtype=np.int64)])
        return (c[self.seg_first[1:]] - c[self.seg_first[:-1]]).astype(np.int64)

    def slice(self, a: int, b: int) -> "Segments":
        s0, s1 = int(self.seg_first[a]), int(self.seg_first[b])
        return Segments(self.seg_first[a:b + 1] - s0, self.seg_ns[s0:s1], self.seg_len[s0:s1],
                        self.ns_bytes, self.ns_off, self.ns_len)


class NamespaceTable:
    def __init__(self):
        self.index = {}
        self.chunks = []
        self.off = []
        self.lens = []
        self.total = 0

    def add(self, ns: str) -> int:
        k = self.index.get(ns)
        if k is None:
            b = ns.encode()
            k = len(self.off)
            self.index[ns] = k
            self.chunks.append(b)
            self.off.append(self.total)
            self.lens.append(len(b))
            self.total += len(b)
        return k

    def arrays(self):
        data = np.frombuffer(b"".join(self.chunks) or b"\0", dtype=np.uint8).copy()
        return data, np.asarray(self.off, np.int64), np.asarray(self.lens, np.int32)


def _field(rec, k):
    return rec[k] if isinstance(rec, dict) else getattr(rec, k)


def _truncate(segs, n):
    """Python slice [:n] of a segment list (n may be negative, like a tuple slice)."""
    total = sum(l for _, l in segs)
    if n < 0:
        n = max(0, total + n)
    out, acc = [], 0
    for ns, l in segs:
        if acc >= n:
            break
        take = min(l, n - acc)
        out.append((ns, take))
        acc += take
    return out


def resolve(records) -> tuple:
    """Trace.materialize's token recipe for every record, as Segments.
    Returns (segments, rids, clients(str), arrivals, output_lens dict)."""
    table = NamespaceTable()
    inputs = {}
    seg_first = [0]
    seg_ns, seg_len = [], []
    rids, clients, arrivals = [], [], []
    out_lens = {}
    for rec in records:
        rid = _field(rec, "rid")
        spid = _field(rec, "shared_prefix_id")
        plen = int(_field(rec, "prefix_len"))
        if spid.startswith("req:"):
            base = inputs[spid[4:]]
            if plen > sum(l for _, l in base):
                raise ValueError(f"{rid}: prefix_len exceeds parent input")
            segs = _truncate(base, plen)
        else:
            segs = [(table.add(spid), plen)] if plen > 0 else []
        suffix = int(_field(rec, "input_token_count")) - plen
        if suffix < 0:
            raise ValueError(f"{rid}: prefix_len exceeds input_token_count")
        if suffix > 0:
            segs = segs + [(table.add(f"sfx:{rid}"), suffix)]
        inputs[rid] = segs
        for ns, l in segs:
            seg_ns.append(ns)
            seg_len.append(l)
        seg_first.append(len(seg_ns))
        rids.append(rid)
        clients.append(_field(rec, "client"))
        arrivals.append(int(_field(rec, "arrival_time")))
        out_lens[rid] = int(_field(rec, "true_output_len"))
    data, off, ln = table.arrays()
    segs = Segments(np.asarray(seg_first, np.int64), np.asarray(seg_ns, np.int32), np.asarray(seg_len, np.int32),
                    data, off, ln)
    return segs, rids, clients, arrivals, out_lens


def load_jsonl(path: str) -> list:
    """Trace.load (requests.py:123-126): one TraceRecord JSON object per line."""
    with open(path) as fh:
        return [json.loads(line) for line in fh if line.strip()]


def add_segments(ctx, segs: Segments, clients: np.ndarray, labels: np.ndarray | None = None,
                 chunk: int = 1 << 16) -> np.ndarray:
    """Generate the requests' tokens in `ctx`'s arena; returns device request ids."""
    n = segs.n
    clients = np.ascontiguousarray(clients, dtype=np.int32)
    labels = np.ascontiguousarray(labels if labels is not None else np.arange(n), dtype=np.int64)
    ids = np.zeros(max(n, 1), np.int32)
    data = np.ascontiguousarray(segs.ns_bytes, dtype=np.uint8)
    off = np.ascontiguousarray(segs.ns_off, dtype=np.int64)
    ln = np.ascontiguousarray(segs.ns_len, dtype=np.int32)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        s = segs.slice(a, b)
        sf = np.ascontiguousarray(s.seg_first, np.int64)
        sn = np.ascontiguousarray(s.seg_ns, np.int32)
        sl = np.ascontiguousarray(s.seg_len, np.int32)
        if sn.size == 0:
            sn = np.zeros(1, np.int32)
            sl = np.zeros(1, np.int32)
        out = np.zeros(b - a, np.int32)
        call("fs_requests_add_expanded", ctx.handle, b - a, sf.ctypes.data_as(P64), sn.ctypes.data_as(P32),
             sl.ctypes.data_as(P32), len(off), data.ctypes.data_as(PU8), off.ctypes.data_as(P64),
             ln.ctypes.data_as(P32), clients[a:b].ctypes.data_as(P32), labels[a:b].ctypes.data_as(P64),
             out.ctypes.data_as(P32))
        ids[a:b] = out
    return ids[:n]


def materialize(records, ctx, client_ids: dict | None = None) -> tuple:
    """Trace.materialize (requests.py:134-161) into the device arena.

    Returns (request ids, rids, output_lens {rid: n}, client_ids {name: dense id}).
    Labels are the (arrival_time, rid) rank within this batch -- the LPM
    tie-break order (local_policies.py:17)."""
    segs, rids, clients, arrivals, out_lens = resolve(records)
    client_ids = {} if client_ids is None else client_ids
    dense = np.asarray([client_ids.setdefault(c, len(client_ids)) for c in clients], np.int32)
    order = sorted(range(len(rids)), key=lambda i: (arrivals[i], rids[i]))
    labels = np.empty(len(rids), np.int64)
    labels[order] = np.arange(len(rids), dtype=np.int64)
    ids = add_segments(ctx, segs, dense, labels)
    return ids, rids, out_lens, client_ids
