"""fs_worker_fill_begin / fs_worker_fill_end: the split fill decides exactly
what fs_worker_fill decides, context uploads may run while it is in flight,
and every other call on the worker or its tree is refused until _end."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(seed):
    from paper_2501_14312_b200.device import Context, Trie, WorkerDev
    rng = np.random.default_rng(seed)
    n, L = 300, 48
    base = rng.integers(0, 1000, L)
    toks = []
    for i in range(n):
        k = int(rng.integers(1, L))
        toks.append(np.concatenate([base[:k], rng.integers(0, 1000, int(rng.integers(1, 24)))]).astype(np.int32))
    flat = np.concatenate(toks)
    lens = np.array([len(t) for t in toks], np.int32)
    offs = np.zeros(n, np.int64)
    offs[1:] = np.cumsum(lens[:-1])
    clients = rng.integers(0, 6, n).astype(np.int32)
    ctx = Context(0, arena_tokens=1 << 18, max_requests=1 << 12)
    trie = Trie(ctx, 900)
    w = WorkerDev(ctx, trie, "dlpm", 400, 1200, 4, 1, 2, max_clients=8)
    return ctx, trie, w, (flat, offs, lens, clients)


def _upload(ctx, data, a, b):
    flat, offs, lens, clients = data
    o0 = int(offs[a])
    return ctx.add_requests(flat[o0:int(offs[b - 1] + lens[b - 1])], offs[a:b] - o0, lens[a:b], clients[a:b],
                            np.arange(a, b, dtype=np.int64))


def test_split_fill_matches_fill_and_guards():
    from paper_2501_14312_b200._lib import FsError
    c1, t1, w1, d = _setup(3)
    c2, t2, w2, _ = _setup(3)
    w1.enqueue(_upload(c1, d, 0, 100))
    w2.enqueue(_upload(c2, d, 0, 100))
    nxt = 100
    prev1, prev2 = [], []
    for k in range(8):
        now = 1000 * (k + 1)
        if prev1:
            t1.unpin_many(np.asarray(prev1, np.int32))
            t2.unpin_many_async(np.asarray(prev2, np.int32))  # settled by the fill below
        r1 = w1.fill(now, 0, 0)
        w2.fill_begin(now, 0, 0)
        # refused while the fill is in flight
        with pytest.raises(FsError):
            w2.enqueue(np.zeros(1, np.int32))
        with pytest.raises(FsError):
            t2.unpin_many(np.zeros(1, np.int32))
        with pytest.raises(FsError):
            w2.fill_begin(now, 0, 0)
        # ... but uploads run concurrently with it
        ids2 = _upload(c2, d, nxt, nxt + 25)
        r2 = w2.fill_end()
        ids1 = _upload(c1, d, nxt, nxt + 25)
        assert ids1.tolist() == ids2.tolist()
        nxt += 25
        assert r1.adm_req.tolist() == r2.adm_req.tolist(), f"step {k}"
        assert r1.adm_mlen.tolist() == r2.adm_mlen.tolist(), f"step {k}"
        assert (r1.used, r1.pinned) == (r2.used, r2.pinned)
        assert r1.records.src.tolist() == r2.records.src.tolist()
        w1.enqueue(ids1)
        w2.enqueue(ids2)
        prev1, prev2 = r1.adm_node.tolist(), r2.adm_node.tolist()
    with pytest.raises(FsError):
        w2.fill_end()  # nothing in flight
    for w, t, c in ((w1, t1, c1), (w2, t2, c2)):
        w.close()
        t.close()
        c.close()


def test_async_unpin_reports_underflow():
    from paper_2501_14312_b200._lib import FsError
    c, t, w, d = _setup(5)
    w.enqueue(_upload(c, d, 0, 60))
    r = w.fill(1000, 0, 0)
    nodes = r.adm_node.astype(np.int32)
    assert len(nodes) > 0
    t.unpin_many_async(nodes)
    assert t.last_ms() >= 0.0  # settles: fine
    t.unpin_many_async(nodes[:1])  # the same path again: below zero
    with pytest.raises(FsError):
        t.last_ms()
    w.close()
    t.close()
    c.close()
