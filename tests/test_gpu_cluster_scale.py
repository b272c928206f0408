"""Config 3 (BASELINE.json configs[2]) parity at its full size: D2LPM with D=8
workers, 200 clients and 262,144 queued requests (the config-2 generator:
1-4k-token prompts, Zipf(1.1) document prefixes), per-worker M = capacity =
65,536, q_u_frac = q_w_frac = 0.5, reserve 8.

The GPU side holds all eight workers' tries, queues and deficit counters plus
the dispatcher (global routing index with worker tags, q_{i,w}, queue sizes)
on one device and drives them through the C ABI: the 262,144 requests are
dispatched at t=0 (global_policies.py:40-46, 107-124), then every round
completes the previous batch (Dlpm.on_outputs + unpin; D2lpm.on_finish),
applies each worker's eviction notices to the routing index (on_eviction ->
evict_notify, radix.py:254-302), dispatches as many arrivals as were admitted
and runs one DLPM fill per worker (local_policies.py:108-128).  The oracle side
is the same rounds on the C restatement (tests/cluster_oracle.SingleCluster:
OracleD2lpm + eight OracleWorkers).  Every dispatch decision, every worker's
admissions in order, the per-worker deficit counters and refills after every
round, and the final q_{i,w} and queue sizes must be identical."""
import numpy as np
import pytest

import cluster_oracle as co

pytestmark = pytest.mark.gpu

NQ = 262144
EXTRA = 16384
D = 8
ROUNDS = 6
STEP_US = 10_000


def params():
    M = CAP = 65536
    L_INPUT = 4096
    U = 1 * L_INPUT + 2 * M
    q = max(1, round(0.5 * U))  # runner.py:127, 131 (banker's rounding; U is even)
    return co.Params(M=M, CAP=CAP, RESERVE=8, W_E=1, W_Q=2, Q_U=q, Q_W=q, n_clients=200)


class GpuCluster:
    """All D workers and the dispatcher on one GPU, SingleCluster's rounds."""

    def __init__(self, q, D, p, device=0):
        from paper_2501_14312_b200.device import Context, DispatcherDev, Trie, WorkerDev
        self.q, self.D, self.p = q, D, p
        tot = int(q.lens.sum()) + 4 * len(q) + 1024
        self.ctx = Context(device, arena_tokens=tot, max_requests=len(q) + 16)
        self.ids = np.asarray(self.ctx.add_requests(q.flat, q.offsets, q.lens, q.clients, q.labels), np.int32)
        assert np.array_equal(self.ids, np.arange(len(q), dtype=np.int32))
        self.tries = [Trie(self.ctx, p.CAP) for _ in range(D)]
        self.workers = [WorkerDev(self.ctx, t, "dlpm", p.Q_U, p.M, p.RESERVE, p.W_E, p.W_Q, max_clients=p.n_clients)
                        for t in self.tries]
        self.d = DispatcherDev(self.ctx, D, p.Q_W, p.W_E, p.W_Q, max_clients=p.n_clients)
        self.prev = [None] * D
        self.notices = [None] * D
        self.next_arrival = 0
        self.n_notices = 0

    def _dispatch(self, arrivals, now, batch=1 << 16):
        idx = np.asarray(arrivals, np.int64)
        ws = []
        for a in range(0, len(idx), batch):
            j = idx[a:a + batch]
            w, _, _, _ = self.d.dispatch(self.ids[j], self.q.clients[j], np.full(len(j), now, np.int64))
            ws.append(np.asarray(w, np.int32))
        ws = np.concatenate(ws) if ws else np.zeros(0, np.int32)
        for r in range(self.D):
            mine = idx[ws == r]
            if len(mine):
                self.workers[r].enqueue(self.ids[mine])
        return ws

    def seed(self, arrivals, now):
        return self._dispatch(arrivals, now)

    def round(self, now, take):
        p = self.p
        n_adm = 0
        for r in range(self.D):
            if self.prev[r] is not None and len(self.prev[r][0]):
                adm, nodes = self.prev[r]
                cl, cnt = np.unique(self.q.clients[adm], return_counts=True)
                self.workers[r].outputs(cl.astype(np.int32), (cnt * p.out_tokens).astype(np.int64))
                self.tries[r].unpin_many(nodes)
        for r in range(self.D):
            if self.prev[r] is not None and len(self.prev[r][0]):
                adm = self.prev[r][0]
                n = len(adm)
                self.d.finish_many(self.q.clients[adm].astype(np.int32), np.full(n, r, np.int32),
                                   np.full(n, p.out_tokens, np.int64))
                n_adm += n
            nt = self.notices[r]
            if nt is not None and len(nt.src):
                self.d.trie.evict_notify_many(nt.src, nt.length, np.full(len(nt.src), r, np.int32), nt.keep,
                                              np.full(len(nt.src), nt.now, np.int64))
        arrivals = take(self.next_arrival, n_adm)
        self.next_arrival += len(arrivals)
        ws = self._dispatch(arrivals, now)
        out = []
        for r in range(self.D):
            res = self.workers[r].fill(now, 0, 0)
            adm = np.asarray(res.adm_req, np.int64)
            self.prev[r] = (adm, np.asarray(res.adm_node, np.int32))
            rec = res.records
            rec.now = now
            self.notices[r] = rec
            self.n_notices += len(rec.src)
            out.append([int(x) for x in adm])
        return out, ws

    def close(self):
        for w in self.workers:
            w.close()
        for t in self.tries:
            t.close()
        self.d.close()
        self.ctx.close()


def test_config3_d2lpm_d8_256k():
    from paper_2501_14312_b200.workloads import build_docs, config3, shared_prefix_queue
    p = params()
    spec = config3(NQ + EXTRA, seed=3)
    q = shared_prefix_queue(spec, docs=build_docs(spec))

    def take(first, n):
        return list(range(NQ + first, min(len(q), NQ + first + n)))

    o = co.SingleCluster(q, D, p=p)
    g = GpuCluster(q, D, p)
    try:
        seed_o = o.seed(list(range(NQ)), 0)
        seed_g = g.seed(list(range(NQ)), 0)
        assert np.array_equal(seed_o, seed_g), "initial dispatch of the 256k queue differs"
        assert set(seed_g.tolist()) == set(range(D))
        total_adm = 0
        for k in range(ROUNDS):
            now = (k + 1) * STEP_US
            adm_o, ws_o = o.round(now, take)
            adm_g, ws_g = g.round(now, take)
            assert np.array_equal(ws_o, ws_g), f"round {k}: dispatch decisions differ"
            for r in range(D):
                assert adm_g[r] == adm_o[r], f"round {k} worker {r}: admissions differ"
                qg, rfg, _ = g.workers[r].counters(p.n_clients)
                qo = o.workers[r].ow.q()[:p.n_clients]
                assert np.array_equal(qg, qo), f"round {k} worker {r}: deficit counters differ"
                assert np.array_equal(rfg, o.workers[r].ow.refills()[:p.n_clients]), f"round {k} worker {r}: refills"
            total_adm += sum(len(a) for a in adm_o)
        qd, present, qsize = g.d.device_counters(p.n_clients)
        assert [int(x) for x in qsize] == [int(x) for x in o.od.queue_size()]
        qo = o.od.q()
        got = {(c, w): int(qd[c * D + w]) for c in range(p.n_clients) for w in range(D) if present[c * D + w]}
        assert got == qo, "q_{i,w} differ"
        assert total_adm > ROUNDS * D
        assert g.n_notices > 0, "eviction notices must flow into the routing index"
    finally:
        g.close()
