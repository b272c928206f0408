"""Replay backend driving the CUDA path through its C ABI (device.py wrappers).

Implements the backend interface of tests/replay.py so the golden serving
traces recorded from the reference run against libfsb200.so exactly as they
run against the CPU oracle.
"""
from __future__ import annotations

import numpy as np

from paper_2501_14312_b200.device import Context, DispatcherDev, Trie, WorkerDev


class GpuBackend:
    def __init__(self, device: int = 0):
        self.ctx = Context(device, arena_tokens=1 << 20, max_requests=1 << 14)
        self.ids = {}   # rid -> device request id
        self.rid_of = {}

    def close(self):
        self.ctx.close()

    def bind(self, tab):
        # a new run: rids are only unique within one run
        self.tab = tab
        self.ids = {}
        self.rid_of = {}

    def upload(self, rid, tab):
        did = self.ids.get(rid)
        if did is None:
            did = self.ctx.add_request(tab.tokens(rid), tab.client_of[rid], tab.label[rid])
            self.ids[rid] = did
            self.rid_of[did] = rid
        return did

    def make_worker(self, wid, cap, M, R, w_e, w_q, policy, quantum, n_clients):
        trie = Trie(self.ctx, cap)
        dev = WorkerDev(self.ctx, trie, policy, quantum, M, R, w_e, w_q, max_clients=max(n_clients, 1))
        return _GpuWorker(self, trie, dev)

    def make_d2(self, D, quantum, w_e, w_q, n_clients):
        return _GpuD2(self, DispatcherDev(self.ctx, D, quantum, w_e, w_q, max_clients=max(n_clients, 1)))


class _GpuWorker:
    def __init__(self, be, trie, dev):
        self.be = be
        self.trie = trie
        self.dev = dev
        self.seen = []

    def enqueue(self, rid, tab):
        c = tab.client_of[rid]
        if c not in self.seen:
            self.seen.append(c)
        self.dev.enqueue(np.array([self.be.upload(rid, tab)], np.int32))

    def fill(self, queue, tab, now, gen, headroom):
        r = self.dev.fill(now, gen, headroom)
        ctx = self.be.ctx
        adm = []
        for did, m in zip(r.adm_req, r.adm_mlen):
            rid = self.be.rid_of[int(did)]
            adm.append((rid, int(m), int(len(tab.tokens(rid)) - m)))
        recs = [(ctx.arena_read(int(s), int(n)), int(k))
                for s, n, k in zip(r.records.src, r.records.length, r.records.keep)]
        q, rf, _ = self.dev.counters()
        dq, drf = self.dev.device_counters(len(q))
        assert (dq == q).all() and (drf == rf).all(), "device counters != host mirror"
        used, pinned, _, _ = self.trie.stats()
        assert (used, pinned) == (r.used, r.pinned)
        return {
            "admissions": adm,
            "handles": [int(x) for x in r.adm_node],
            "records": recs,
            "q": {c: int(q[c]) for c in self.seen},
            "refills": {c: int(rf[c]) for c in self.seen},
            "used": used,
            "pinned": pinned,
            "dump": self.trie.dump,
            "fill": r,
        }

    def on_outputs(self, client, n):
        self.dev.outputs(np.array([client], np.int32), np.array([n], np.int64))

    def unpin(self, h):
        self.trie.unpin(h)

    def dump(self):
        return self.trie.dump()


class _GpuD2:
    def __init__(self, be, dev):
        self.be = be
        self.dev = dev
        self.n_clients = dev.max_clients

    def dispatch(self, tokens, client, now, rid=None):
        did = self.be.upload(rid, self.be.tab)
        w, m, mask, _ = self.dev.dispatch(np.array([did], np.int32), np.array([client], np.int32),
                                          np.array([now], np.int64))
        matched = tuple(b for b in range(64) if int(mask[0]) >> b & 1)
        return int(w[0]), int(m[0]), matched

    def on_finish(self, client, w, out):
        self.dev.finish(client, w, out)

    def on_eviction(self, path, keep, w, notice_time, ref=None):
        rid, n = ref[0], ref[1]
        off, _ = self.be.ctx.request_info(self.be.ids[rid])
        self.dev.trie.evict_notify(off, n, w, keep, notice_time)

    def q(self):
        out = {}
        for c in range(self.n_clients):
            row, pr = self.dev.counters(c)
            for w in range(self.dev.D):
                if pr[w]:
                    out[(c, w)] = int(row[w])
        return out

    def dump(self):
        return self.dev.trie.dump()
