"""Test infrastructure for the multi-GPU D^2LPM protocol (paper_2501_14312_b200.cluster).

* OracleRank -- the protocol backend of one rank on the CPU oracle (its worker
  and its own dispatcher replica), so the distributed protocol itself can run
  under gloo with world size 2 on CPU.
* SingleCluster -- the same rounds in one process with ONE dispatcher and all
  workers: the semantics the replicated protocol must reproduce exactly.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from oracle.oracle import OracleD2lpm, OracleWorker
from paper_2501_14312_b200.cluster import NOTICE_COLS
from paper_2501_14312_b200.workloads import SharedPrefixSpec, build_docs, shared_prefix_queue

SPEC = SharedPrefixSpec(n=1600, clients=12, docs=16, zipf_s=1.1, len_lo=64, len_hi=256, doc_lo=32, doc_hi=200,
                        seed=7)
M = 2048
CAP = 2048
RESERVE = 4
W_E, W_Q = 1, 2
L_INPUT = 256
U = W_E * L_INPUT + W_Q * M
Q_U = max(1, round(0.5 * U))
Q_W = max(1, round(0.5 * U))
N_SEED = 700
ROUNDS = 12
STEP_US = 10_000


@dataclass
class Params:
    """Serving parameters of one cluster run (per-worker M / capacity, the
    resolved quanta -- runner.py:127, 131 -- and the client count)."""
    M: int = M
    CAP: int = CAP
    RESERVE: int = RESERVE
    W_E: int = W_E
    W_Q: int = W_Q
    Q_U: int = Q_U
    Q_W: int = Q_W
    n_clients: int = SPEC.clients
    out_tokens: int = 8


DEFAULT = Params()


def workload():
    return shared_prefix_queue(SPEC, docs=build_docs(SPEC))


def stream(q):
    def take(first, n):
        return list(range(N_SEED + first, min(len(q), N_SEED + first + n)))
    return take


class _OracleWorkerSide:
    def __init__(self, rank, q, p=DEFAULT):
        self.rank = rank
        self.q = q
        self.ow = OracleWorker(p.CAP, p.M, p.RESERVE, p.W_E, p.W_Q, "dlpm", p.Q_U, p.n_clients)
        self._by_first = {}  # first token -> admitted request indices (notice -> source request)
        self.pending = []
        self.admitted = []

    def enqueue(self, mine):
        for i in mine:
            self.ow.on_enqueue(int(self.q.clients[i]))
            self.pending.append(int(i))

    def complete(self, handles, clients, out):
        for h, c in zip(handles, clients):
            self.ow.on_outputs(int(c), out)
            self.ow.unpin(h)

    def _src_of(self, path):
        n = len(path)
        cand = self._by_first.get(int(path[0]), []) if n else self.admitted
        for i in reversed(cand):
            t = self.q.tokens(i)
            if len(t) >= n and np.array_equal(t[:n], path):
                return i
        raise AssertionError("evicted path is not a prefix of an admitted request")

    def fill(self, now):
        q = self.q
        idx = np.asarray(self.pending, np.int64)
        r = self.ow.fill(q.flat, q.offsets[idx], q.lens[idx], q.clients[idx], q.labels[idx], now, 0, 0)
        adm = [int(idx[p]) for p in r["pos"]]
        gone = set(adm)
        self.pending = [i for i in self.pending if i not in gone]
        self.admitted.extend(adm)
        for i in adm:
            t = q.tokens(i)
            if len(t):
                self._by_first.setdefault(int(t[0]), []).append(i)
        notices = np.zeros((len(r["records"]), NOTICE_COLS), np.int64)
        for k, (path, keep) in enumerate(r["records"]):
            notices[k] = (self._src_of(path), len(path), keep, self.rank, now)
        return adm, r["handles"], [int(q.clients[i]) for i in adm], notices, len(idx), 0.0


class OracleRank(_OracleWorkerSide):
    """One rank: its worker and its own replica of the dispatcher."""

    def __init__(self, rank, q, D, p=DEFAULT):
        super().__init__(rank, q, p)
        self.od = OracleD2lpm(D, p.Q_W, p.W_E, p.W_Q, p.n_clients)

    def dispatch(self, arrivals, now):
        return np.array([self.od.dispatch(self.q.tokens(i), int(self.q.clients[i]), now)[0] for i in arrivals],
                        np.int32)

    def dispatcher_finish(self, client, worker, out):
        self.od.on_finish(client, worker, out)

    def dispatcher_notice(self, src, ln, keep, worker, emitted):
        self.od.on_eviction(self.q.tokens(src)[:ln], keep, worker, emitted)

    def dispatcher_state(self, n_clients):
        return self.od.q(), self.od.queue_size()


class SingleCluster:
    """All workers and one dispatcher in one process, same round structure."""

    def __init__(self, q, D, pipelined=False, p=DEFAULT):
        self.q = q
        self.D = D
        self.p = p
        self.pipelined = pipelined
        self.late = [[] for _ in range(D)]
        self.workers = [_OracleWorkerSide(r, q, p) for r in range(D)]
        self.od = OracleD2lpm(D, p.Q_W, p.W_E, p.W_Q, p.n_clients)
        self.prev = [[] for _ in range(D)]
        self.notices = [np.zeros((0, NOTICE_COLS), np.int64) for _ in range(D)]
        self.next_arrival = 0

    def _dispatch(self, arrivals, now, late=False):
        ws = []
        for i in arrivals:
            w = self.od.dispatch(self.q.tokens(i), int(self.q.clients[i]), now)[0]
            if late:
                self.late[w].append(i)
            else:
                self.workers[w].enqueue([i])
            ws.append(w)
        return np.array(ws, np.int32)

    def seed(self, arrivals, now):
        return self._dispatch(arrivals, now)

    def round(self, now, take):
        n_adm = 0
        fins = []
        for r, wk in enumerate(self.workers):
            prev = self.prev[r]
            if prev:
                wk.complete([h for _, _, h in prev], [c for _, c, _ in prev], self.p.out_tokens)
            fins.append([(c, r, self.p.out_tokens) for _, c, _ in prev])
        for r in range(self.D):
            for c, w, out in fins[r]:
                self.od.on_finish(c, w, out)
            n_adm += len(fins[r])
            for src, ln, keep, worker, emitted in self.notices[r]:
                self.od.on_eviction(self.q.tokens(int(src))[: int(ln)], int(keep), int(worker), int(emitted))
        arrivals = take(self.next_arrival, n_adm)
        self.next_arrival += len(arrivals)
        if self.pipelined:
            for r, wk in enumerate(self.workers):  # last round's arrivals join now
                if self.late[r]:
                    wk.enqueue(self.late[r])
                self.late[r] = []
        ws = self._dispatch(arrivals, now, late=self.pipelined)
        out = []
        for r, wk in enumerate(self.workers):
            adm, handles, clients, notices, nq, _ = wk.fill(now)
            self.prev[r] = list(zip(adm, clients, handles))
            self.notices[r] = notices
            out.append(adm)
        return out, ws


def run_single(D, pipelined=False):
    q = workload()
    c = SingleCluster(q, D, pipelined)
    take = stream(q)
    seed_ws = c.seed(list(range(N_SEED)), 0)
    rounds = []
    n_notices = 0
    for k in range(ROUNDS):
        adm, ws = c.round((k + 1) * STEP_US, take)
        n_notices += sum(len(x) for x in c.notices)
        rounds.append({"admitted": adm, "dispatched": ws.tolist()})
    return {"seed": seed_ws.tolist(), "rounds": rounds, "q": c.od.q(), "qsize": c.od.queue_size(),
            "n_notices": n_notices}


def run_rank(rank, comm, backend, pipelined=False):
    """Drive one rank through the protocol; returns its view of every round."""
    from paper_2501_14312_b200.cluster import ClusterRank
    q = backend.q
    cr = ClusterRank(backend, comm, out_tokens=8, pipelined=pipelined)
    take = stream(q)
    seed_ws = cr.seed(list(range(N_SEED)), 0)
    rounds = []
    for k in range(ROUNDS):
        rr = cr.round((k + 1) * STEP_US, take)
        rounds.append({"admitted": rr.admitted, "dispatched": np.asarray(rr.dispatched).tolist()})
    return {"seed": np.asarray(seed_ws).tolist(), "rounds": rounds}


def gloo_main(rank, world, port, out_dir, kind, pipelined=False):
    """Entry of one spawned rank (world size `world`, gloo on 127.0.0.1)."""
    import json
    import os
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch.distributed as dist
    from paper_2501_14312_b200.cluster import TorchComm
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        q = workload()
        if kind == "oracle":
            be = OracleRank(rank, q, world)
        else:
            be = make_gpu_rank(rank, q, world, "cuda:0")
        res = run_rank(rank, TorchComm("cpu"), be, pipelined)
        st = be.dispatcher_state(SPEC.clients)
        res["qsize"] = [int(x) for x in st[-1]]
        with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
            json.dump(res, f)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def make_gpu_rank(rank, q, D, device):
    from paper_2501_14312_b200.cluster import GpuRank
    return GpuRank(rank, device, q, D, M, CAP, RESERVE, W_E, W_Q, Q_U, Q_W, SPEC.clients)
