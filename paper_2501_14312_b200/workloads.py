"""Synthetic shared-prefix request queues.

Token ids are uniform in [0, 2^31) (requests.py:92), drawn with numpy PCG64;
the prefix structure is drawn with Python `random`, both from the config seed,
so every consumer (the CUDA path, the CPU oracle, the reference) sees the
same requests.  Returned as flat arrays ready for fs_requests_add.
"""
from __future__ import annotations

import bisect
import random
from dataclasses import dataclass

import numpy as np


@dataclass
class Queue:
    flat: np.ndarray      # int32 tokens, requests back to back
    offsets: np.ndarray   # int64 start of each request in flat
    lens: np.ndarray      # int32
    clients: np.ndarray   # int32 dense client ids
    arrival: np.ndarray   # int64 trace arrival (us)
    rids: list            # request ids (str); (arrival, rid) order == labels order
    labels: np.ndarray    # int64 rank of (arrival, rid)

    def __len__(self):
        return len(self.lens)

    def tokens(self, i) -> np.ndarray:
        o = int(self.offsets[i])
        return self.flat[o:o + int(self.lens[i])]


@dataclass
class SharedPrefixSpec:
    n: int = 65536
    clients: int = 100
    docs: int = 256
    zipf_s: float = 1.1
    len_lo: int = 1024
    len_hi: int = 4096
    doc_lo: int = 512
    doc_hi: int = 4032
    seed: int = 2


def config2(n: int = 65536, seed: int = 2) -> SharedPrefixSpec:
    """Config 2: DLPM single worker, 100 clients, 64k queued, 1-4k-token prompts,
    prefixes = Zipf(1.1)-chosen document over 256 docs of U[512, 4032] tokens."""
    return SharedPrefixSpec(n=n, seed=seed)


def config3(n: int = 262144, seed: int = 3) -> SharedPrefixSpec:
    """Config 3: D2LPM D=8 workers, 200 clients, 256k queued -- the config-2
    generator (1-4k-token prompts, Zipf(1.1) document prefixes)."""
    return SharedPrefixSpec(n=n, clients=200, seed=seed)


def build_docs(spec: SharedPrefixSpec):
    pr = random.Random(spec.seed)
    g = np.random.Generator(np.random.PCG64(spec.seed))
    doc_len = [pr.randint(spec.doc_lo, spec.doc_hi) for _ in range(spec.docs)]
    docs = [g.integers(0, 2 ** 31, size=dl, dtype=np.int64).astype(np.int32) for dl in doc_len]
    w = [1.0 / (k + 1) ** spec.zipf_s for k in range(spec.docs)]
    cum = []
    acc = 0.0
    for x in w:
        acc += x
        cum.append(acc)
    return docs, cum


def shared_prefix_queue(spec: SharedPrefixSpec, first: int = 0, count: int | None = None,
                        arrival: int = 0, docs=None, stream_seed: int | None = None) -> Queue:
    """Requests [first, first+count) of the spec's stream.  Request i draws its
    length, document and client from a per-request Python RNG and its unique
    suffix from a per-batch PCG64 stream, so slices are reproducible."""
    count = spec.n if count is None else count
    if docs is None:
        docs = build_docs(spec)
    doc_tok, cum = docs
    total_w = cum[-1]
    pr = random.Random(spec.seed * 1_000_003 + first)
    g = np.random.Generator(np.random.PCG64((spec.seed if stream_seed is None else stream_seed) * 7919 + first))
    L = np.empty(count, np.int64)
    D = np.empty(count, np.int64)
    C = np.empty(count, np.int32)
    for i in range(count):
        L[i] = pr.randint(spec.len_lo, spec.len_hi)
        D[i] = bisect.bisect_left(cum, pr.random() * total_w)
        C[i] = pr.randrange(spec.clients)
    doc_len = np.array([len(d) for d in doc_tok], np.int64)
    P = np.minimum(doc_len[D], L - 1)
    suf = L - P
    offsets = np.zeros(count, np.int64)
    offsets[1:] = np.cumsum(L[:-1])
    flat = np.empty(int(L.sum()), np.int32)
    sfx = g.integers(0, 2 ** 31, size=int(suf.sum()), dtype=np.int64).astype(np.int32)
    so = 0
    for i in range(count):
        o = offsets[i]
        p = P[i]
        flat[o:o + p] = doc_tok[D[i]][:p]
        s = suf[i]
        flat[o + p:o + p + s] = sfx[so:so + s]
        so += s
    rids = [f"r{first + i:08d}" for i in range(count)]
    arr = np.full(count, arrival, np.int64)
    # (arrival, rid) rank; zero-padded rids sort numerically
    labels = (np.int64(arrival) << 32) + np.arange(first, first + count, dtype=np.int64)
    return Queue(flat, offsets, L.astype(np.int32), C, arr, rids, labels)


# ---------------------------------------------------------------------------
# Config 5: 1M queued 8k-token requests over a deep prefix tree.
# ---------------------------------------------------------------------------

@dataclass
class DeepTreeSpec:
    n: int = 1 << 20
    clients: int = 200
    branching: int = 4
    depth: int = 6
    level_tokens: int = 1024
    length: int = 8192
    seed: int = 5


def config5(n: int = 1 << 20, seed: int = 5) -> DeepTreeSpec:
    """Config 5: branching-4, depth-6 prefix tree of 1024-token levels, a unique
    tail to 8192 tokens, 200 clients, seed 5."""
    return DeepTreeSpec(n=n, seed=seed)


def deep_tree_segments(spec: DeepTreeSpec, first: int = 0, count: int | None = None, stream: int = 0):
    """Requests [first, first+count) of the config-5 stream as device segments.

    Request i walks a random root-to-depth path of the tree; level l of node k
    (heap numbering, root 0) is expand_tokens(f"c5n:{k}", level_tokens) and the
    tail is expand_tokens(f"sfx:c5r{stream}.{i:08d}", length - depth*level_tokens),
    i.e. the reference's own token universe (requests.py:89-102).
    Returns (Segments, clients int32, labels int64)."""
    from .trace import Segments
    count = spec.n - first if count is None else count
    g = np.random.Generator(np.random.PCG64(spec.seed * 7919 + first + 1_000_003 * stream))
    digits = g.integers(0, spec.branching, size=(count, spec.depth), dtype=np.int64)
    clients = g.integers(0, spec.clients, size=count, dtype=np.int64).astype(np.int32)
    n_nodes = sum(spec.branching ** l for l in range(spec.depth + 1))
    node_ns = [f"c5n:{k}".encode() for k in range(n_nodes)]
    tail_ns = ("".join(f"sfx:c5r{stream}.{first + i:08d}" for i in range(count))).encode()
    tail_w = len(f"sfx:c5r{stream}.{0:08d}")
    node_off = np.zeros(n_nodes, np.int64)
    node_len = np.array([len(b) for b in node_ns], np.int32)
    node_off[1:] = np.cumsum(node_len[:-1])
    node_bytes = b"".join(node_ns)
    ns_bytes = np.frombuffer(node_bytes + tail_ns, np.uint8).copy()
    ns_off = np.concatenate([node_off, len(node_bytes) + tail_w * np.arange(count, dtype=np.int64)])
    ns_len = np.concatenate([node_len, np.full(count, tail_w, np.int32)])
    tail = spec.length - spec.depth * spec.level_tokens
    per = spec.depth + (1 if tail > 0 else 0)
    seg_ns = np.empty((count, per), np.int32)
    seg_len = np.empty((count, per), np.int32)
    node = np.zeros(count, np.int64)
    for l in range(spec.depth):
        node = node * spec.branching + digits[:, l] + 1
        seg_ns[:, l] = node
        seg_len[:, l] = spec.level_tokens
    if tail > 0:
        seg_ns[:, spec.depth] = n_nodes + np.arange(count)
        seg_len[:, spec.depth] = tail
    segs = Segments(np.arange(count + 1, dtype=np.int64) * per, seg_ns.reshape(-1), seg_len.reshape(-1),
                    ns_bytes, ns_off, ns_len)
    labels = (np.int64(stream) << 40) + np.arange(first, first + count, dtype=np.int64)
    return segs, clients, labels


def segments_namespaces(segs) -> list:
    """Decode the namespace string of every segment (tests / oracle side)."""
    b = segs.ns_bytes.tobytes()
    return [b[int(segs.ns_off[k]):int(segs.ns_off[k]) + int(segs.ns_len[k])].decode() for k in segs.seg_ns]
