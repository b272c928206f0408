"""Partitioned batch-start matching for multi-GPU D2LPM: the
records of an arrival batch computed in slices (as N ranks would, then
all-gathered) and handed to fs_dispatch_prematched give exactly the
decisions, match lengths, worker masks and refill rounds of fs_dispatch
(global_policies.py:40-46, 107-124), batch after batch, with finishes and
eviction notices changing the routing index in between."""
import numpy as np
import pytest

import cluster_oracle as co

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sliced_prematch_dispatches_like_fs_dispatch(world):
    import torch
    from paper_2501_14312_b200.device import Context, DispatcherDev

    q = co.workload()
    ctx = Context(0, arena_tokens=int(q.lens.sum()) + 4 * len(q) + 1024, max_requests=len(q) + 16)
    ids = np.asarray(ctx.add_requests(q.flat, q.offsets, q.lens, q.clients, q.labels), np.int32)
    D = 4
    a = DispatcherDev(ctx, D, co.Q_W, co.W_E, co.W_Q, max_clients=co.SPEC.clients)
    b = DispatcherDev(ctx, D, co.Q_W, co.W_E, co.W_Q, max_clients=co.SPEC.clients)
    rec = DispatcherDev.prematch_record_bytes()
    rng = np.random.default_rng(world)
    pos, now = 0, 0
    while pos < len(q):
        n = int(min(len(q) - pos, rng.integers(1, 200)))
        sl = ids[pos:pos + n]
        cl = q.clients[pos:pos + n].astype(np.int32)
        nows = np.full(n, now, np.int64)
        wa = a.dispatch(sl, cl, nows)
        chunk = max(1, -(-n // world))
        buf = torch.zeros(world * chunk * rec, dtype=torch.uint8, device="cuda:0")
        for r in range(world):
            lo, hi = min(n, r * chunk), min(n, (r + 1) * chunk)
            if hi > lo:
                b.prematch(sl[lo:hi], buf.data_ptr() + r * chunk * rec)
        torch.cuda.synchronize()
        wb = b.dispatch_prematched(sl, cl, nows, buf.data_ptr())
        for x, y in zip(wa, wb):
            assert np.array_equal(x, y)
        # finishes and eviction notices between batches (same on both)
        for k in range(0, n, 3):
            a.finish(int(cl[k]), int(wa[0][k]), 8)
            b.finish(int(cl[k]), int(wb[0][k]), 8)
        if n > 4:
            off, ln = ctx.request_info(int(sl[n // 2]))
            a.trie.evict_notify(off, ln, int(wa[0][n // 2]), ln // 2, now)
            b.trie.evict_notify(off, ln, int(wb[0][n // 2]), ln // 2, now)
        pos += n
        now += 1000
    for x, y in zip(a.device_counters(co.SPEC.clients), b.device_counters(co.SPEC.clients)):
        assert np.array_equal(x, y)
    ea, eb = a.trie.export(), b.trie.export()
    for k in ea:
        assert np.array_equal(ea[k], eb[k]), k
    a.close(); b.close(); ctx.close()
