"""D^2LPM across GPUs: one worker per GPU, a replicated dispatcher.

The dispatcher's state -- the global routing index, q_{i,w} and queue sizes
(global_policies.py:88-132) -- is a deterministic state machine.  Every rank
keeps a replica on its own GPU and feeds it the same inputs in the same
order, so every replica makes the same decisions without exchanging them.
The only inputs that originate on one rank are the events of its worker --
request finishes (D2lpm.on_finish, global_policies.py:126-129) and eviction
notices (D2lpm.on_eviction -> evict_notify, radix.py:254-302) -- so each round
has exactly one exchange step: an all-gather of those records (NCCL over
NVLink on GPUs, gloo in the CPU tests), applied by every rank in rank order.

One round at time `now` (the synchronous serving loop of bench.py, cluster-wide):
  1. the batch admitted by each worker in the previous round completes: output
     charge (Dlpm.on_outputs) and unpin on its own GPU; finish records
     (client, worker, output tokens) are produced;
  2. exchange: all-gather finish records and the previous round's eviction
     notices (arena offset, path length, keep_len, worker, emission time);
     every replica applies them rank by rank;
  3. as many requests arrive as were admitted cluster-wide in the previous
     round (a deterministic shared stream); every replica dispatches them in
     order (Dispatcher.dispatch, global_policies.py:40-46) and each rank
     enqueues the ones routed to it;
  4. every rank runs one DLPM fill of its own queue.

Requests are uploaded to every rank in the same order, so arena offsets -- and
therefore eviction-notice paths -- are identical on all ranks.  Backends and
the transport are pluggable: `GpuRank` drives the CUDA library; the CPU tests
drive the oracle through the same protocol.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# record layouts exchanged every round (int64 columns)
FIN_COLS = 3      # client, worker, output tokens
NOTICE_COLS = 5   # arena src, path length, keep_len, worker, emission time


@dataclass
class RoundResult:
    admitted: list            # request indices admitted on this rank
    dispatched: np.ndarray    # worker chosen for each arrival of the round (all ranks agree)
    n_queued: int             # requests this rank's fill evaluated
    n_arrivals: int
    fill_ms: float = 0.0
    extra: dict = field(default_factory=dict)


class LocalComm:
    """Single-process transport (world size 1)."""

    rank = 0
    world = 1

    def all_gather_rows(self, rows: np.ndarray) -> list:
        return [rows]


class TorchComm:
    """torch.distributed transport: counts, then padded rows (NCCL or gloo)."""

    def __init__(self, device: str = "cpu"):
        import torch
        import torch.distributed as dist
        self.torch = torch
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = device

    def all_gather_rows(self, rows: np.ndarray) -> list:
        torch, dist = self.torch, self.dist
        cols = rows.shape[1]
        n = torch.tensor([rows.shape[0]], dtype=torch.int64, device=self.device)
        ns = [torch.zeros_like(n) for _ in range(self.world)]
        dist.all_gather(ns, n)
        counts = [int(x.item()) for x in ns]
        m = max(max(counts), 1)
        buf = torch.zeros((m, cols), dtype=torch.int64, device=self.device)
        if rows.shape[0]:
            buf[: rows.shape[0]] = torch.from_numpy(np.ascontiguousarray(rows, dtype=np.int64)).to(self.device)
        outs = [torch.zeros_like(buf) for _ in range(self.world)]
        dist.all_gather(outs, buf)
        return [o[:c].cpu().numpy() for o, c in zip(outs, counts)]


class ClusterRank:
    """Protocol driver of one rank.  `backend` provides the worker and the
    dispatcher replica (see GpuRank / the oracle backend in tests)."""

    def __init__(self, backend, comm, out_tokens: int = 8):
        self.be = backend
        self.comm = comm
        self.out_tokens = out_tokens
        self.prev = []            # (request index, client, path handle) admitted last round
        self.notices = np.zeros((0, NOTICE_COLS), np.int64)
        self.last_cluster_admitted = 0
        self.next_arrival = 0

    def seed(self, arrivals: list, now: int) -> np.ndarray:
        """Initial burst: dispatch `arrivals` everywhere, enqueue mine."""
        return self._dispatch(arrivals, now)

    def _dispatch(self, arrivals, now) -> np.ndarray:
        if not arrivals:
            return np.zeros(0, np.int32)
        workers = self.be.dispatch(arrivals, now)
        mine = [a for a, w in zip(arrivals, workers) if w == self.comm.rank]
        if mine:
            self.be.enqueue(mine)
        return workers

    def round(self, now: int, arrival_stream) -> RoundResult:
        be, comm = self.be, self.comm
        # 1. completion of last round's batch on this worker
        fin = np.zeros((len(self.prev), FIN_COLS), np.int64)
        if self.prev:
            clients = np.array([c for _, c, _ in self.prev], np.int64)
            fin[:, 0] = clients
            fin[:, 1] = comm.rank
            fin[:, 2] = self.out_tokens
            be.complete([h for _, _, h in self.prev], clients, self.out_tokens)
        # 2. exchange and apply in rank order (finishes, then notices)
        rows = np.zeros((fin.shape[0] + self.notices.shape[0], 1 + NOTICE_COLS), np.int64)
        rows[: fin.shape[0], 0] = 0
        rows[: fin.shape[0], 1:1 + FIN_COLS] = fin
        rows[fin.shape[0]:, 0] = 1
        rows[fin.shape[0]:, 1:] = self.notices
        gathered = comm.all_gather_rows(rows)
        n_adm_cluster = 0
        for part in gathered:
            f = part[part[:, 0] == 0]
            for client, worker, out in f[:, 1:1 + FIN_COLS]:
                be.dispatcher_finish(int(client), int(worker), int(out))
            n_adm_cluster += len(f)
            for src, ln, keep, worker, emitted in part[part[:, 0] == 1][:, 1:]:
                be.dispatcher_notice(int(src), int(ln), int(keep), int(worker), int(emitted))
        # 3. arrivals, dispatched identically on every replica
        arrivals = arrival_stream(self.next_arrival, n_adm_cluster)
        self.next_arrival += len(arrivals)
        workers = self._dispatch(arrivals, now)
        # 4. local fill
        adm, handles, clients, notices, nq, ms = be.fill(now)
        self.prev = list(zip(adm, clients, handles))
        self.notices = notices
        return RoundResult(adm, workers, nq, len(arrivals), ms)


class GpuRank:
    """CUDA backend of one rank: its worker (local trie + DLPM queue) and a
    dispatcher replica, both on this rank's GPU, through the C ABI."""

    def __init__(self, rank, device, queue, D, M, capacity, reserve, w_e, w_q, q_u, q_w, n_clients):
        from .device import Context, DispatcherDev, Trie, WorkerDev
        self.rank = rank
        self.q = queue
        tot = int(queue.lens.sum()) + 4 * len(queue) + 1024
        self.ctx = Context(device, arena_tokens=tot, max_requests=len(queue) + 16)
        # every rank uploads the whole stream in the same order: identical arena offsets
        self.ids = self.ctx.add_requests(queue.flat, queue.offsets, queue.lens, queue.clients, queue.labels)
        self.trie = Trie(self.ctx, capacity)
        self.w = WorkerDev(self.ctx, self.trie, "dlpm", q_u, M, reserve, w_e, w_q, max_clients=n_clients)
        self.d = DispatcherDev(self.ctx, D, q_w, w_e, w_q, max_clients=n_clients)
        self.now_dispatch = 0

    def dispatch(self, arrivals, now):
        idx = np.asarray(arrivals, np.int64)
        w, _, _, _ = self.d.dispatch(self.ids[idx], self.q.clients[idx], np.full(len(idx), now, np.int64))
        return w

    def enqueue(self, mine):
        self.w.enqueue(self.ids[np.asarray(mine, np.int64)])

    def complete(self, handles, clients, out_tokens):
        cl, cnt = np.unique(np.asarray(clients, np.int32), return_counts=True)
        self.w.outputs(cl.astype(np.int32), (cnt * out_tokens).astype(np.int64))
        self.trie.unpin_many(np.asarray(handles, np.int32))

    def dispatcher_finish(self, client, worker, out):
        self.d.finish(client, worker, out)

    def dispatcher_notice(self, src, ln, keep, worker, emitted):
        self.d.trie.evict_notify(src, ln, worker, keep, emitted)

    def fill(self, now):
        r = self.w.fill(now, 0, 0)
        adm = [int(x) for x in r.adm_req]  # device ids == stream indices (uploaded in order)
        notices = np.zeros((len(r.records), NOTICE_COLS), np.int64)
        if len(r.records):
            notices[:, 0] = r.records.src
            notices[:, 1] = r.records.length
            notices[:, 2] = r.records.keep
            notices[:, 3] = self.rank
            notices[:, 4] = now
        return adm, [int(x) for x in r.adm_node], [int(self.q.clients[i]) for i in adm], notices, r.n_queued, \
            r.device_ms

    def dispatcher_state(self, n_clients):
        q, present, qsize = self.d.device_counters(n_clients)
        return q, present, qsize
