"""TEST INFRASTRUCTURE ONLY -- the CPU oracle driven through the synthetic
serving loop used by bench.py and the scale parity tests.

One step = (1) the previous step's batch completes: every admitted request is
charged its output tokens (Dlpm.on_outputs, local_policies.py:130-133) and its
path is unpinned (worker.py:209-213); (2) requests that arrived since the last
step are enqueued (local_policies.py:88-92); (3) one schedule step
(Dlpm.fill, local_policies.py:108-128) over the whole queue.
"""
from __future__ import annotations

import time

import numpy as np

from .oracle import OracleWorker


class OracleSteps:
    def __init__(self, q, capacity, M, R, w_e, w_q, quantum, n_clients, policy="dlpm", out_tokens=8):
        self.q = q                      # workloads.Queue holding every request that will ever arrive
        self.ow = OracleWorker(capacity, M, R, w_e, w_q, policy, quantum, n_clients)
        self.pending = []               # queue indices, enqueue order
        self.prev = []                  # (handle, client) of the last step's admissions
        self.out_tokens = out_tokens
        self.w_q = w_q
        self.fill_s = 0.0
        self.decisions = 0

    def enqueue(self, idx):
        for i in idx:
            self.ow.on_enqueue(int(self.q.clients[i]))
            self.pending.append(int(i))

    def step(self, now):
        for h, c in self.prev:
            self.ow.on_outputs(c, self.out_tokens)
            self.ow.unpin(h)
        idx = np.asarray(self.pending, np.int64)
        t0 = time.perf_counter()
        r = self.ow.fill(self.q.flat, self.q.offsets[idx], self.q.lens[idx], self.q.clients[idx],
                         self.q.labels[idx], now, 0, 0)
        self.fill_s += time.perf_counter() - t0
        self.decisions += len(idx)
        adm = [int(idx[p]) for p in r["pos"]]
        gone = set(adm)
        self.pending = [i for i in self.pending if i not in gone]
        self.prev = [(h, int(self.q.clients[i])) for h, i in zip(r["handles"], adm)]
        return {"admitted": adm, "mlen": [int(x) for x in r["mlen"]], "q": self.ow.q(),
                "refills": self.ow.refills(), "records": r["records"], "n": len(idx),
                "used": self.ow.tree.used_tokens, "pinned": self.ow.tree.pinned_tokens}
