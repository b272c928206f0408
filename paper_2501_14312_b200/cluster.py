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

    def all_gather_tensor(self, t):
        """Concatenation of every rank's equal-size device tensor t, on t's
        device (NCCL: one all_gather_into_tensor over NVLink; gloo: through
        host memory).  Complete when it returns."""
        torch, dist = self.torch, self.dist
        if dist.get_backend() == "nccl":
            out = torch.empty(self.world * t.numel(), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(out, t)
        else:
            parts = [torch.empty(t.numel(), dtype=t.dtype) for _ in range(self.world)]
            dist.all_gather(parts, t.cpu())
            out = torch.cat(parts).to(t.device)
        if t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()  # the library reads it on its own stream
        return out

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
    dispatcher replica (see GpuRank / the oracle backend in tests).

    pipelined: a round's arrivals are dispatched while the workers fill and
    join the queues of the NEXT round's fill (they arrive just after this
    round's step).  The dispatcher sees exactly the same inputs in the same
    order; only the local enqueue moves one round later.  With a backend whose
    dispatcher has its own CUDA stream (`concurrent_dispatch`), the dispatcher
    side runs on a second host thread concurrently with the fill."""

    def __init__(self, backend, comm, out_tokens: int = 8, max_arrivals: int | None = None,
                 pipelined: bool = False):
        self.be = backend
        self.max_arrivals = max_arrivals
        self.comm = comm
        self.out_tokens = out_tokens
        self.pipelined = pipelined
        self._pool = None
        if pipelined and getattr(backend, "concurrent_dispatch", False):
            from concurrent.futures import ThreadPoolExecutor
            self._pool = ThreadPoolExecutor(1)
        self._late = []           # pipelined arrivals routed here, enqueued at the next round
        self.prev = []            # (request index, client, path handle) admitted last round
        self.notices = np.zeros((0, NOTICE_COLS), np.int64)
        self.next_arrival = 0
        self.t_exchange = 0.0  # host wall seconds: all-gather, apply, dispatch
        self.t_apply = 0.0
        self.t_dispatch = 0.0
        self.t_fill = 0.0     # host wall of the fill call
        self.t_complete = 0.0  # host wall of step 1 (unpin + output accounting of the last batch)
        self.t_upload = 0.0   # host wall of the arrivals' upload (pipelined, before the fill)
        self.t_overlap = 0.0  # per round: max(fill, dispatcher side) when pipelined, else their sum

    def seed(self, arrivals: list, now: int) -> np.ndarray:
        """Initial burst: dispatch `arrivals` everywhere, enqueue mine."""
        return self._dispatch(arrivals, now)[0]

    def _dispatch(self, arrivals, now, enqueue=True):
        if not arrivals:
            return np.zeros(0, np.int32), []
        if self.comm.world > 1 and getattr(self.be, "prematch_partitioned", False):
            # the batch-start matches split 1/N across the ranks, one all-gather
            workers = self.be.dispatch(arrivals, now, comm=self.comm)
        else:
            workers = self.be.dispatch(arrivals, now)
        mine = [a for a, w in zip(arrivals, workers) if w == self.comm.rank]
        if mine and enqueue:
            self.be.enqueue(mine)
        return workers, mine

    def round(self, now: int, arrival_stream) -> RoundResult:
        import time
        be, comm = self.be, self.comm
        tc = time.perf_counter()
        # 1. completion of last round's batch on this worker
        fin = np.zeros((len(self.prev), FIN_COLS), np.int64)
        if self.prev:
            clients = np.array([c for _, c, _ in self.prev], np.int64)
            fin[:, 0] = clients
            fin[:, 1] = comm.rank
            fin[:, 2] = self.out_tokens
            be.complete([h for _, _, h in self.prev], clients, self.out_tokens)
        # 2. exchange; every replica applies the records in rank order (finishes, then notices)
        rows = np.zeros((fin.shape[0] + self.notices.shape[0], 1 + NOTICE_COLS), np.int64)
        rows[: fin.shape[0], 0] = 0
        rows[: fin.shape[0], 1:1 + FIN_COLS] = fin
        rows[fin.shape[0]:, 0] = 1
        rows[fin.shape[0]:, 1:] = self.notices
        t0 = time.perf_counter()
        self.t_complete += t0 - tc
        gathered = comm.all_gather_rows(rows)
        t1 = time.perf_counter()
        n_adm_cluster = sum(int((part[:, 0] == 0).sum()) for part in gathered)
        n_arr = n_adm_cluster if self.max_arrivals is None else min(n_adm_cluster, self.max_arrivals)
        arrivals = arrival_stream(self.next_arrival, n_arr)
        self.next_arrival += len(arrivals)

        def dispatcher_side():
            ta = time.perf_counter()
            batched = hasattr(be, "dispatcher_apply")
            for part in gathered:
                f = part[part[:, 0] == 0]
                nt = part[part[:, 0] == 1][:, 1:]
                if batched:
                    be.dispatcher_apply(f[:, 1:1 + FIN_COLS], nt)
                    continue
                for client, worker, out in f[:, 1:1 + FIN_COLS]:
                    be.dispatcher_finish(int(client), int(worker), int(out))
                for src, ln, keep, worker, emitted in nt:
                    be.dispatcher_notice(int(src), int(ln), int(keep), int(worker), int(emitted))
            tb = time.perf_counter()
            # 3. arrivals, dispatched identically on every replica
            ws, mine = self._dispatch(arrivals, now, enqueue=not self.pipelined)
            return ws, mine, tb - ta, time.perf_counter() - tb

        if self.pipelined:
            if self._late:
                be.enqueue(self._late)  # last round's arrivals join this round's queue
            if arrivals and hasattr(be, "prepare"):
                # arrival uploads go out before the fill is launched: an H2D issued
                # while another thread waits on the fill stalls in the driver
                tp = time.perf_counter()
                be.prepare(arrivals)
                self.t_upload += time.perf_counter() - tp
            fut = self._pool.submit(dispatcher_side) if self._pool is not None else None
            if fut is None:
                workers, mine, ta, td = dispatcher_side()
            # 4. local fill (concurrently with the dispatcher chain on its own stream)
            tf = time.perf_counter()
            adm, handles, clients, notices, nq, ms = be.fill(now)
            tf = time.perf_counter() - tf
            if fut is not None:
                workers, mine, ta, td = fut.result()
                self.t_overlap += time.perf_counter() - t1
            else:
                self.t_overlap += ta + td + tf
            self._late = mine
        else:
            workers, mine, ta, td = dispatcher_side()
            # 4. local fill
            tf = time.perf_counter()
            adm, handles, clients, notices, nq, ms = be.fill(now)
            tf = time.perf_counter() - tf
            self.t_overlap += ta + td + tf
        self.t_fill += tf
        self.t_exchange += t1 - t0
        self.t_apply += ta
        self.t_dispatch += td
        self.prev = list(zip(adm, clients, handles))
        self.notices = notices
        return RoundResult(adm, workers, nq, len(arrivals), ms)


def partitioned_prematch(d, ids, comm, device):
    """The batch-start matches of an arrival batch (ids in arrival order), split
    1/N across the ranks: rank r matches arrivals [r*chunk, (r+1)*chunk) on its
    replica of the routing index (fs_dispatch_prematch); one all-gather of the
    fixed-size records hands every replica the whole batch in arrival order.
    Every replica holds the same index, so every slice is what any replica
    would have computed.  Returns the gathered device tensor."""
    import torch
    from .device import DispatcherDev
    rec = DispatcherDev.prematch_record_bytes() if device is not None else d.record_bytes
    n = len(ids)
    chunk = max(1, -(-n // comm.world))
    lo = min(n, comm.rank * chunk)
    hi = min(n, lo + chunk)
    # device None: host memory (tests of the exchange with a host-side matcher)
    local = torch.zeros(chunk * rec, dtype=torch.uint8, device=f"cuda:{device}" if device is not None else "cpu")
    if hi > lo:
        d.prematch(ids[lo:hi], local.data_ptr())
    return comm.all_gather_tensor(local)


class GpuRank:
    """CUDA backend of one rank: its worker (local trie + DLPM queue) and a
    dispatcher replica, both on this rank's GPU, through the C ABI."""

    concurrent_dispatch = True  # the dispatcher replica has its own CUDA stream

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

    prematch_partitioned = True

    def dispatch(self, arrivals, now, comm=None):
        idx = np.asarray(arrivals, np.int64)
        nows = np.full(len(idx), now, np.int64)
        if comm is None:
            w, _, _, _ = self.d.dispatch(self.ids[idx], self.q.clients[idx], nows)
        else:
            pre = partitioned_prematch(self.d, self.ids[idx], comm, self.ctx.device)
            w, _, _, _ = self.d.dispatch_prematched(self.ids[idx], self.q.clients[idx], nows, pre.data_ptr())
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


class GpuStreamRank:
    """CUDA backend of one rank for the benchmark's serving loop: the workload's
    initial queue materialized on the device (identical order on every rank, so
    arena offsets and eviction-notice paths agree) plus a host pool of later
    arrivals uploaded as they arrive.  Stream index i < nq is initial request i;
    nq + k is pool request k."""

    concurrent_dispatch = True  # the dispatcher replica has its own CUDA stream

    def __init__(self, rank, device, wl, D, w_e, w_q, q_w, n_clients):
        from .device import Context, DispatcherDev, Trie, WorkerDev
        self.rank = rank
        self.wl = wl
        self.pool = wl.pool
        tot = wl.queue_tokens + int(self.pool.lens.sum()) + 4 * (wl.nq + len(self.pool)) + 1024
        self.ctx = Context(device, arena_tokens=tot, max_requests=wl.nq + len(self.pool) + 16)
        ids, clients = wl.put_initial(self.ctx)
        self.ids = np.full(wl.nq + len(self.pool), -1, np.int32)
        self.clients = np.zeros(wl.nq + len(self.pool), np.int32)
        self.ids[:wl.nq] = ids
        self.clients[:wl.nq] = clients
        self.clients[wl.nq:] = self.pool.clients
        self.uploaded = wl.nq
        self.trie = Trie(self.ctx, wl.CAP)
        self.w = WorkerDev(self.ctx, self.trie, "dlpm", wl.quantum(), wl.M, wl.reserve, w_e, w_q,
                           max_clients=n_clients)
        self.d = DispatcherDev(self.ctx, D, q_w, w_e, w_q, max_clients=n_clients)
        # arrivals upload straight from the page-locked pool (one DMA per round)
        from .device import host_register
        self.pool.flat = np.ascontiguousarray(self.pool.flat, dtype=np.int32)
        host_register(self.pool.flat)
        self.h2d = 0
        self.fill_ms = 0.0
        self.disp_s = 0.0
        self.upload_s = 0.0
        self.disp_prof = np.zeros(16, np.int64)
        self.n_queued = 0
        self.n_dispatched = 0

    def _ensure(self, upto):
        if upto <= self.uploaded:
            return
        p, nq = self.pool, self.wl.nq
        a, b = self.uploaded - nq, upto - nq
        o0 = int(p.offsets[a])
        o1 = int(p.offsets[b - 1] + p.lens[b - 1])
        self.ids[self.uploaded:upto] = self.ctx.add_requests(p.flat[o0:o1], p.offsets[a:b] - o0, p.lens[a:b],
                                                             p.clients[a:b], p.labels[a:b])
        self.h2d += (o1 - o0) * 4 + (b - a) * 24
        self.uploaded = upto

    def arrival_stream(self, first, count):
        nq = self.wl.nq
        count = max(0, min(count, len(self.pool) - first))
        return list(range(nq + first, nq + first + count))

    def prepare(self, arrivals):
        import time
        tu = time.perf_counter()
        self._ensure(int(max(arrivals)) + 1)
        self.upload_s += time.perf_counter() - tu

    prematch_partitioned = True

    def dispatch(self, arrivals, now, batch=1 << 16, comm=None):
        import time
        idx = np.asarray(arrivals, np.int64)
        tu = time.perf_counter()
        self._ensure(int(idx.max()) + 1)
        t0 = time.perf_counter()
        self.upload_s += t0 - tu
        out = []
        for a in range(0, len(idx), batch):
            j = idx[a:a + batch]
            nows = np.full(len(j), now, np.int64)
            if comm is None:
                w, _, _, _ = self.d.dispatch(self.ids[j], self.clients[j], nows)
            else:
                tp = time.perf_counter()
                pre = partitioned_prematch(self.d, self.ids[j], comm, self.ctx.device)
                self.prematch_s = getattr(self, "prematch_s", 0.0) + time.perf_counter() - tp
                w, _, _, _ = self.d.dispatch_prematched(self.ids[j], self.clients[j], nows, pre.data_ptr())
            out.append(w)
            self.disp_prof += self.d.last_profile()
        self.disp_s += time.perf_counter() - t0
        self.n_dispatched += len(idx)
        return np.concatenate(out)

    def enqueue(self, mine):
        self.w.enqueue(self.ids[np.asarray(mine, np.int64)])

    def complete(self, handles, clients, out_tokens):
        cl, cnt = np.unique(np.asarray(clients, np.int32), return_counts=True)
        self.w.outputs(cl.astype(np.int32), (cnt * out_tokens).astype(np.int64))
        self.trie.unpin_many_async(np.asarray(handles, np.int32))  # settled by this round's fill
        self.h2d += cl.nbytes + cnt.nbytes + 4 * len(handles)

    def dispatcher_apply(self, fin, notices):
        if len(fin):
            self.d.finish_many(fin[:, 0], fin[:, 1], fin[:, 2])
        if len(notices):
            self.d.trie.evict_notify_many(notices[:, 0], notices[:, 1], notices[:, 3], notices[:, 2], notices[:, 4])
            import ctypes as C
            from ._lib import call
            pr = np.zeros(4, np.int64)
            call("fs_trie_last_notify_profile", self.d.trie._h, pr.ctypes.data_as(C.POINTER(C.c_int64)))
            self.notice_prof = getattr(self, "notice_prof", np.zeros(4, np.int64)) + pr
            self.n_notices = getattr(self, "n_notices", 0) + len(notices)

    def fill(self, now):
        r = self.w.fill(now, 0, 0)
        self.fill_ms += r.device_ms
        self.n_queued += r.n_queued
        adm_ids = np.asarray(r.adm_req, np.int64)
        # device id -> stream index (uploads are in stream order: ids are increasing)
        adm = np.searchsorted(self.ids[:self.uploaded], adm_ids).tolist()
        notices = np.zeros((len(r.records), NOTICE_COLS), np.int64)
        if len(r.records):
            notices[:, 0] = r.records.src
            notices[:, 1] = r.records.length
            notices[:, 2] = r.records.keep
            notices[:, 3] = self.rank
            notices[:, 4] = now
        return adm, [int(x) for x in r.adm_node], [int(self.clients[i]) for i in adm], notices, r.n_queued, \
            r.device_ms

    def close(self):
        from .device import host_unregister
        host_unregister(self.pool.flat)
        self.w.close()
        self.trie.close()
        self.d.close()
        self.ctx.close()
