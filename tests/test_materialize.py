"""Trace materialization: the reference's token universe
(_token_block / expand_tokens / Trace.materialize, requests.py:89-161).

CPU: the oracle restatement against golden vectors recorded from the real
reference (tests/golden/make_golden_tokens.py), and the host-side segment
resolution (paper_2501_14312_b200.trace.resolve) expanded by the oracle.
GPU: the device generator k_expand (fs_requests_add_expanded) against the
same goldens, at up to 7-digit block numbers, and on config-5 slices."""
import gzip
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import materialize as OM
from paper_2501_14312_b200.trace import Segments, resolve
from paper_2501_14312_b200.workloads import config5, deep_tree_segments, segments_namespaces

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tokens.json")))


def digest(toks) -> str:
    return hashlib.sha256(json.dumps([int(x) for x in toks], separators=(",", ":")).encode()).hexdigest()


def oracle_expand_segments(segs: Segments) -> list:
    names = segments_namespaces(segs)
    out = []
    for i in range(segs.n):
        toks = []
        for s in range(int(segs.seg_first[i]), int(segs.seg_first[i + 1])):
            toks.extend(OM.expand_tokens(names[s], int(segs.seg_len[s])))
        out.append(toks)
    return out


# ------------------------------------------------------------------ CPU

def test_oracle_token_blocks():
    for ns, b, toks in GOLD["blocks"]:
        assert list(OM.token_block(ns, b)) == toks, (ns, b)


def test_oracle_expand():
    for ns, n, toks in GOLD["expand"]:
        assert list(OM.expand_tokens(ns, n)) == toks, (ns, n)


@pytest.mark.parametrize("t", GOLD["traces"], ids=[t["name"] for t in GOLD["traces"]])
def test_oracle_materialize(t):
    order, _ = OM.materialize(t["records"])
    assert [digest(x) for _, x in order] == t["digests"]


@pytest.mark.parametrize("t", GOLD["traces"], ids=[t["name"] for t in GOLD["traces"]])
def test_resolve_segments(t):
    segs, rids, clients, arrivals, outs = resolve(t["records"])
    assert rids == [r["rid"] for r in t["records"]]
    assert list(segs.lens()) == t["lens"]
    assert [digest(x) for x in oracle_expand_segments(segs)] == t["digests"]
    assert outs == {r["rid"]: r["true_output_len"] for r in t["records"]}


def test_resolve_errors_match_reference():
    base = {"client": "c", "arrival_time": 0, "true_output_len": 1, "parent_id": None}
    recs = [dict(base, rid="p", shared_prefix_id="ns", prefix_len=4, input_token_count=10)]
    with pytest.raises(ValueError):
        resolve(recs + [dict(base, rid="c", shared_prefix_id="req:p", prefix_len=11, input_token_count=12)])
    with pytest.raises(ValueError):
        resolve([dict(base, rid="x", shared_prefix_id="ns", prefix_len=5, input_token_count=4)])
    with pytest.raises(KeyError):
        resolve([dict(base, rid="y", shared_prefix_id="req:missing", prefix_len=1, input_token_count=4)])
    # Python slice semantics of a negative prefix_len (requests.py:145-151)
    odd = recs + [dict(base, rid="n", shared_prefix_id="req:p", prefix_len=-3, input_token_count=2)]
    segs, *_ = resolve(odd)
    order, _ = OM.materialize(odd)
    assert [digest(x) for x in oracle_expand_segments(segs)] == [digest(x) for _, x in order]


def test_c_restatement_matches_hashlib():
    """oracle/tokens.c (used for large CPU samples) == the hashlib restatement
    == the reference goldens."""
    for t in GOLD["traces"]:
        segs, *_ = resolve(t["records"])
        flat, offs = OM.expand_segments(segs)
        got = [flat[offs[i]:offs[i + 1]] for i in range(segs.n)]
        assert [digest(x) for x in got] == t["digests"]
    segs, _, _ = deep_tree_segments(config5(), first=7, count=5)
    flat, offs = OM.expand_segments(segs)
    want = oracle_expand_segments(segs)
    assert [list(flat[offs[i]:offs[i + 1]]) for i in range(5)] == [list(w) for w in want]


def test_config5_structure():
    spec = config5()
    segs, clients, labels = deep_tree_segments(spec, first=100, count=64)
    assert list(segs.lens()) == [8192] * 64
    names = segments_namespaces(segs)
    assert names[0].startswith("c5n:") and names[6] == "sfx:c5r0.00000100"
    assert clients.min() >= 0 and clients.max() < spec.clients
    # slices of the stream are reproducible
    s2, c2, _ = deep_tree_segments(spec, first=100, count=64)
    assert np.array_equal(s2.seg_ns, segs.seg_ns) and np.array_equal(c2, clients)


# ------------------------------------------------------------------ GPU

def _ctx():
    from paper_2501_14312_b200.device import Context
    return Context(0, arena_tokens=1 << 22, max_requests=1 << 12)


def _read(ctx, ids):
    out = []
    for i in ids:
        off, ln = ctx.request_info(int(i))
        out.append(ctx.arena_read(off, ln))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("t", GOLD["traces"], ids=[t["name"] for t in GOLD["traces"]])
def test_gpu_materialize_trace(t):
    from paper_2501_14312_b200.trace import materialize
    ctx = _ctx()
    ids, rids, outs, cl = materialize(t["records"], ctx)
    toks = _read(ctx, ids)
    assert [len(x) for x in toks] == t["lens"]
    assert [digest(x) for x in toks] == t["digests"]
    ctx.close()


@pytest.mark.gpu
def test_gpu_expand_golden_blocks():
    """Every golden (namespace, block) through a segment long enough to reach
    it: covers every padding regime and 1..7-digit block numbers."""
    from paper_2501_14312_b200.device import Context
    from paper_2501_14312_b200.trace import NamespaceTable, add_segments
    ctx = Context(0, arena_tokens=1 << 26, max_requests=1 << 10)
    small = [(ns, b, toks) for ns, b, toks in GOLD["blocks"] if b <= 12345]
    big = [(ns, b, toks) for ns, b, toks in GOLD["blocks"] if b > 12345 and ns in ("a", "x" * 64)]
    tab = NamespaceTable()
    reqs = [(tab.add(ns), 8 * (b + 1)) for ns, b, _ in small + big]
    data, off, ln = tab.arrays()
    segs = Segments(np.arange(len(reqs) + 1, dtype=np.int64), np.array([r[0] for r in reqs], np.int32),
                    np.array([r[1] for r in reqs], np.int32), data, off, ln)
    ids = add_segments(ctx, segs, np.zeros(len(reqs), np.int32), chunk=8)
    for (ns, b, toks), i in zip(small + big, ids):
        o, n = ctx.request_info(int(i))
        got = ctx.arena_read(o + 8 * b, 8)
        assert list(got) == toks, (ns, b)
    ctx.close()


@pytest.mark.gpu
def test_gpu_expand_lengths():
    from paper_2501_14312_b200.trace import add_segments
    ctx = _ctx()
    for ns, n, toks in GOLD["expand"]:
        segs, *_ = resolve([{"rid": "r", "client": "c", "arrival_time": 0, "true_output_len": 1,
                             "shared_prefix_id": ns, "prefix_len": n, "input_token_count": n}])
        ids = add_segments(ctx, segs, np.zeros(1, np.int32))
        assert list(_read(ctx, ids)[0]) == toks, (ns, n)
    ctx.close()


@pytest.mark.gpu
def test_gpu_config5_slice_matches_oracle():
    from paper_2501_14312_b200.trace import add_segments
    ctx = _ctx()
    segs, clients, labels = deep_tree_segments(config5(), first=4096, count=24)
    ids = add_segments(ctx, segs, clients, labels, chunk=7)
    got = _read(ctx, ids)
    want = oracle_expand_segments(segs)
    for g, w in zip(got, want):
        assert list(g) == list(w)
    ctx.close()
