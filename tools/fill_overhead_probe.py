"""Probe (not a test): where the Python fill wrapper spends host time."""
import ctypes as C
import sys
import time

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2501_14312_b200 import _lib as L  # noqa: E402
from paper_2501_14312_b200.device import _p32, _p64  # noqa: E402

wl = bench.make_workload("c5", 0, 0, 40)
g = bench.GpuSteps(wl, 0)
now = 0
for _ in range(4):
    now += bench.STEP_US
    g.step(now)
w = g.w
T = {}
def tick(k, t0):
    T[k] = T.get(k, 0) + time.perf_counter() - t0
    return time.perf_counter()
for _ in range(10):
    now += bench.STEP_US
    # completion + arrivals exactly as GpuSteps.step, then the wrapper by parts
    t = time.perf_counter()
    n_prev = len(g.prev_nodes)
    if n_prev:
        import numpy as np
        cl, cnt = np.unique(g.prev_clients, return_counts=True)
        w.outputs(cl.astype(np.int32), (cnt * 8).astype(np.int64))
        g.trie.unpin_many(g.prev_nodes)
    t = tick("complete", t)
    p = g.pool
    a, b = g.pool_next, g.pool_next + n_prev
    o0 = int(p.offsets[a]); o1 = int(p.offsets[b - 1] + p.lens[b - 1])
    ids = g.ctx.add_requests(p.flat[o0:o1], p.offsets[a:b] - o0, p.lens[a:b], p.clients[a:b], p.labels[a:b])
    g.pool_next = b
    t = tick("add_requests", t)
    w.enqueue(ids)
    t = tick("enqueue", t)
    qlen = w.queue_len()
    res = L.FsFillResult()
    res.cap_adm = w._cap
    res.adm_req = _p32(w._req); res.adm_mlen = _p32(w._mlen); res.adm_unpinned = _p64(w._unp)
    res.adm_pinned_before = _p64(w._pinb); res.adm_path_node = _p32(w._node); res.adm_rec_end = _p64(w._rend)
    res.recs = L.FsRecords(0, None, None, None, 0)
    t = tick("prep", t)
    L.call("fs_worker_fill", w._h, now, 0, 0, C.byref(res))
    t = tick("c_fill", t)
    recs = w.trie.read_records(res.recs.n_rec)
    t = tick("read_records", t)
    na = res.n_adm
    g.prev_nodes = w._node[:na].astype(np.int32)
    g.prev_clients = np.asarray([g.clients[int(i)] for i in w._req[:na]], np.int32)
    t = tick("post", t)
for k, v in T.items():
    print(f"{k:14s} {1000 * v / 10:.3f} ms")
