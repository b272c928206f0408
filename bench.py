"""Benchmark: DLPM / D2LPM scheduling decisions/s (BASELINE.json metric, "at
1M-request queue") on config 5 by default -- 1M queued 8k-token requests over a
deep shared-prefix tree (`--workload c2` for configs[1], the 64k queue) -- plus
the prefix-match kernel's roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one pass of the decision path over the resident queue, driven the
way the reference's serving loop drives it:
  1. the previous step's batch completes: output charge w_q*8 per request
     (Dlpm.on_outputs) and unpin of its paths (worker.py:209-213);
  2. as many new requests arrive as were admitted (uploaded from page-locked
     host memory through the C ABI, Worker.enqueue -> on_request_enqueued);
  3. one schedule step over the whole queue (Dlpm.fill): K1 match + LRU stamp
     of every queued request, K2 sort, K3/K4 deficit-gated admission with
     radix insert / split / LRU evict / pin.
Decisions per step = queued requests evaluated.  `value` is device time
(CUDA events inside the library, inputs resident); `e2e` is host wall time of
the same public-API calls including the H2D upload of arrivals and the D2H of
the admission results.
N>1 (torchrun): one DLPM worker per GPU with its own 1M queue (weak scaling;
the local fill has no cross-worker exchange), then -- reported under
`d2lpm_cluster` -- D2LPM across the same GPUs: one shared 1M queue dispatched
by a replicated dispatcher, one NCCL all-gather per round (strong scaling).
`--cluster` runs only the latter (also at N=1).
The CPU baseline is the C oracle (a literal restatement of the reference's
Dlpm.fill) on the same steps of a 65,536-request sample, on one core.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W_E, W_Q = 1, 2
STEP_US = 10_000
DEFAULT_WORKLOAD = "c5"
METRIC = "scheduling decisions/sec (DLPM schedule steps over the resident request queue)"


class Workload:
    """One BASELINE.json configuration: serving parameters, the initial queue
    (put on the device untimed) and the pool of later arrivals (host tokens,
    uploaded inside the timed steps)."""
    name = ""
    out_tokens = 8
    reserve = 8

    def quantum(self):
        return max(1, round(0.5 * (W_E * self.L_INPUT + W_Q * self.M)))  # q_u_frac 0.5 (runner.py:127)


class Config2(Workload):
    """configs[1]: one worker, 100 clients, 64k queued 1-4k-token prompts with a
    Zipf(1.1) shared-prefix tree over 256 documents."""
    name = "c2"
    M = CAP = 65536
    L_INPUT = 4096
    clients = 100

    def __init__(self, nq, rank, steps):
        from paper_2501_14312_b200.workloads import build_docs, config2, shared_prefix_queue
        self.nq = nq
        self.spec = config2(nq, seed=2 + rank)
        docs = build_docs(self.spec)
        self.q = shared_prefix_queue(self.spec, docs=docs)
        pool_n = 800 * steps + 1024
        self.pool = shared_prefix_queue(self.spec, first=nq, count=pool_n, arrival=STEP_US, docs=docs,
                                        stream_seed=self.spec.seed + 101)
        self.queue_tokens = int(self.q.lens.sum())
        self.desc = ("config2: DLPM 1 worker/GPU, 100 clients, %d queued, 1-4k-token prompts, Zipf(1.1) prefixes "
                     "over 256 docs, M=capacity=65536, q_u_frac=0.5, reserve=8" % nq)
        self.l2 = ("inputs larger than L2: each step streams every queued request's matched prefix (~240 MB) "
                   "and the queue occupies ~640 MB")

    def put_initial(self, ctx):
        ids = ctx.add_requests(self.q.flat, self.q.offsets, self.q.lens, self.q.clients, self.q.labels)
        return ids, self.q.clients.astype(np.int32)

    def cpu_sample(self, device):
        return self.q, self.pool, len(self.q)


class Config3(Config2):
    """configs[2]: the config-2 generator with 200 clients and 256k queued
    requests -- the D2LPM D=8 configuration (`--workload c3 --cluster`);
    per-worker M = capacity = 65536, q_w_frac 0.5."""
    name = "c3"
    clients = 200

    def __init__(self, nq, rank, steps):
        from paper_2501_14312_b200.workloads import build_docs, config3, shared_prefix_queue
        self.nq = nq
        self.spec = config3(nq, seed=3 + rank)
        docs = build_docs(self.spec)
        self.q = shared_prefix_queue(self.spec, docs=docs)
        pool_n = 800 * steps + 1024
        self.pool = shared_prefix_queue(self.spec, first=nq, count=pool_n, arrival=STEP_US, docs=docs,
                                        stream_seed=self.spec.seed + 101)
        self.queue_tokens = int(self.q.lens.sum())
        self.desc = ("config3: 200 clients, %d queued, 1-4k-token prompts, Zipf(1.1) prefixes over 256 docs, "
                     "per-worker M=capacity=65536, q_u_frac=q_w_frac=0.5, reserve=8" % nq)
        self.l2 = "inputs larger than L2: the queue occupies %.1f GB" % (self.queue_tokens * 4 / 1e9)


class Config5(Workload):
    """configs[4] at D=1: 1M queued 8k-token requests over a branching-4, depth-6
    prefix tree of 1024-token levels (+ a unique 2048-token tail), 200 clients,
    M = capacity = 262144.  Tokens are the reference's own universe
    (expand_tokens, requests.py:89-102) generated on the device."""
    name = "c5"
    M = CAP = 262144
    L_INPUT = 8192
    clients = 200
    CPU_NQ = 65536

    def __init__(self, nq, rank, steps, device=0, cpu_only=False):
        from paper_2501_14312_b200.workloads import config5
        self.nq = nq
        self.spec = config5(nq, seed=5 + rank)
        self.pool_n = 160 * steps + 512
        self.cpu_only = cpu_only  # reference arm: build every token on the host (oracle/tokens.c)
        self.pool = self._host_queue(device, stream=1, first=0, count=self.pool_n, arrival=STEP_US)
        self.queue_tokens = nq * self.spec.length
        self.desc = ("config5 at D=1: DLPM, 200 clients, %d queued 8192-token prompts, branching-4 depth-6 prefix "
                     "tree of 1024-token levels + unique 2048-token tail, M=capacity=262144, q_u_frac=0.5, "
                     "reserve=8; tokens = expand_tokens (sha256) generated on device" % nq)
        self.l2 = "inputs larger than L2: the queue occupies %.1f GB; each step streams every queued request's " \
                  "matched prefix" % (self.queue_tokens * 4 / 1e9)

    def _host_queue(self, device, stream, first, count, arrival, cpu=False):
        """Host token buffers of a slice of the stream: materialized on the device
        and read back (the GPU arm's arrivals), or by the CPU restatement
        oracle/tokens.c (the CPU baseline's sample, the reference arm)."""
        from paper_2501_14312_b200.workloads import Queue, deep_tree_segments
        segs, clients, labels = deep_tree_segments(self.spec, first=first, count=count, stream=stream)
        lens = segs.lens()
        rids = [f"c5r{stream}.{first + i:08d}" for i in range(count)]
        if cpu or self.cpu_only:
            from oracle.materialize import expand_segments
            flat, offs = expand_segments(segs)
            return Queue(flat, offs[:-1].copy(), lens.astype(np.int32), clients, np.full(count, arrival, np.int64),
                         rids, labels)
        from paper_2501_14312_b200.device import Context
        from paper_2501_14312_b200.trace import add_segments
        tmp = Context(device, arena_tokens=int(lens.sum()) + 4 * count + 1024, max_requests=count + 16)
        try:
            ids = add_segments(tmp, segs, clients, labels)
            off0, _ = tmp.request_info(int(ids[0]))
            offl, lnl = tmp.request_info(int(ids[-1]))
            raw = tmp.arena_read(off0, offl + lnl - off0)
            offs = np.array([tmp.request_info(int(i))[0] - off0 for i in ids], np.int64)
        finally:
            tmp.close()
        return Queue(raw, offs, lens.astype(np.int32), clients, np.full(count, arrival, np.int64), rids, labels)

    def put_initial(self, ctx):
        from paper_2501_14312_b200.trace import add_segments
        from paper_2501_14312_b200.workloads import deep_tree_segments
        segs, clients, labels = deep_tree_segments(self.spec, first=0, count=self.nq, stream=0)
        return add_segments(ctx, segs, clients, labels), clients

    def cpu_sample(self, device):
        n = min(self.nq, self.CPU_NQ)
        return self._host_queue(device, stream=0, first=0, count=n, arrival=0, cpu=True), self.pool, n


def make_workload(name, nq, rank, steps, device=0, world=1, cpu_only=False):
    if name == "c2":
        return Config2(nq or 65536, rank, steps * world)
    if name == "c3":
        return Config3(nq or 262144, rank, steps * world)
    if name == "c5":
        return Config5(nq or (1 << 20), rank, steps * world, device=device, cpu_only=cpu_only)
    raise SystemExit(f"unknown workload {name}")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class GpuSteps:
    """The synthetic serving loop on the CUDA path, through the C ABI."""

    def __init__(self, wl, device):
        from paper_2501_14312_b200.device import Context, Trie, WorkerDev
        self.wl = wl
        self.pool = wl.pool
        tot = wl.queue_tokens + int(self.pool.lens.sum()) + 4 * (wl.nq + len(self.pool)) + 1024
        self.ctx = Context(device, arena_tokens=tot, max_requests=wl.nq + len(self.pool) + 16)
        self.trie = Trie(self.ctx, wl.CAP)
        self.w = WorkerDev(self.ctx, self.trie, "dlpm", wl.quantum(), wl.M, wl.reserve, W_E, W_Q,
                           max_clients=max(128, wl.clients))
        self.ids, clients0 = wl.put_initial(self.ctx)
        # client of every device request id: the initial queue, then the pool in upload order
        self.clients = np.concatenate([np.asarray(clients0, np.int32), np.asarray(self.pool.clients, np.int32)])
        # arrivals are uploaded from page-locked host memory (DMA), like a
        # serving frontend's pinned receive buffers
        from paper_2501_14312_b200.device import host_register
        self.pool.flat = np.ascontiguousarray(self.pool.flat, dtype=np.int32)
        host_register(self.pool.flat)
        self.w.enqueue(self.ids)
        self.prev_nodes = np.zeros(0, np.int32)
        self.prev_clients = np.zeros(0, np.int32)
        self.pool_next = 0
        self.pool_ids = np.full(len(self.pool), -1, np.int32)
        self.uploaded = 0  # pool[:uploaded] is on the device
        self.h2d = 0
        self.d2h = 0
        self.unpin_ms = 0.0  # device time of the batch-completion unpins

    def step(self, now):
        n_prev = len(self.prev_nodes)
        if n_prev:
            # output tokens per finished client (Dlpm.on_outputs, local_policies.py:130-133)
            per = np.bincount(self.prev_clients)
            cl = np.flatnonzero(per).astype(np.int32)
            cnt = per[cl].astype(np.int64)
            self.w.outputs(cl, cnt * self.wl.out_tokens)
            # stream-ordered before the fill; status and device time come back with it
            self.trie.unpin_many_async(self.prev_nodes)
            self.h2d += cl.nbytes + cnt.nbytes + self.prev_nodes.nbytes
        if n_prev and self.pool_next + n_prev <= len(self.pool):
            a, b = self.pool_next, self.pool_next + n_prev
            self._upload(b)  # normally already there (uploaded during the last fill)
            self.w.enqueue(self.pool_ids[a:b])
            self.pool_next = b
        # the scheduler runs while the host uploads the next arrivals (the pool
        # in arrival order, a lookahead of twice the last admission count):
        # the copy and its scatter overlap the fill instead of preceding it
        self.w.fill_begin(now, 0, 0)
        self._upload(min(len(self.pool), self.pool_next + max(64, 2 * n_prev)))
        res = self.w.fill_end()
        if n_prev:
            self.unpin_ms += self.trie.last_ms()
        self.prev_nodes = res.adm_node.astype(np.int32)
        self.prev_clients = self.clients[np.asarray(res.adm_req, np.int64)]
        self.d2h += res.adm_req.nbytes * 6 + 8 * 128 * 2 + 64
        return res

    def _upload(self, upto):
        if upto <= self.uploaded:
            return
        a, b = self.uploaded, upto
        p = self.pool
        o0 = int(p.offsets[a])
        o1 = int(p.offsets[b - 1] + p.lens[b - 1])
        self.pool_ids[a:b] = self.ctx.add_requests(p.flat[o0:o1], p.offsets[a:b] - o0, p.lens[a:b], p.clients[a:b],
                                                   p.labels[a:b])
        self.uploaded = b
        self.h2d += (o1 - o0) * 4 + (b - a) * 24

    def close(self):
        from paper_2501_14312_b200.device import host_unregister
        host_unregister(self.pool.flat)
        self.w.close()
        self.trie.close()
        self.ctx.close()


def clocks_start():
    path = os.path.join(ROOT, "gpurun_out", "bench_clocks.csv") if os.path.isdir(os.path.join(ROOT, "gpurun_out")) \
        else "/tmp/bench_clocks.csv"
    try:
        fh = open(path, "w")
        p = subprocess.Popen(["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
                              "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                              "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                             stdout=fh, stderr=subprocess.DEVNULL)
        return p, fh, path
    except Exception:
        return None, None, None


def clocks_stop(p, fh, path, dev):
    if p is None:
        return None
    time.sleep(0.25)
    p.terminate()
    p.wait()
    fh.close()
    sm, mx, reasons = [], 0.0, set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for line in open(path):
        f = [x.strip() for x in line.split(",")]
        if len(f) < 9 or not f[0].isdigit() or int(f[0]) != dev:
            continue
        try:
            sm.append(float(f[1]))
            mx = max(mx, float(f[2]))
        except ValueError:
            continue
        for name, v in zip(names, f[5:9]):
            if v.lower() == "active":
                reasons.add(name)
    if not sm:
        return None
    return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(wl, q, pool, warmup=5, steps_max=40, budget_s=15.0):
    """C oracle (literal restatement of Dlpm.fill) on the same serving steps as
    the GPU loop, one core: `warmup` untimed steps, then timed steps until
    steps_max or the time budget."""
    from oracle.lockstep import OracleSteps
    o = OracleSteps(_concat_once(None, q, pool), wl.CAP, wl.M, wl.reserve, W_E, W_Q, wl.quantum(),
                    max(128, wl.clients), out_tokens=wl.out_tokens)
    o.enqueue(range(len(q)))
    pool_base = len(q)
    nxt = 0
    k = 0
    t0 = None
    steps = 0
    while steps < steps_max and (t0 is None or time.perf_counter() - t0 < budget_s):
        if k == warmup:
            o.fill_s, o.decisions, t0 = 0.0, 0, time.perf_counter()
        r = o.step((k + 1) * STEP_US)
        k += 1
        if k > warmup:
            steps += 1
        # arrivals, in the same pool order as the GPU loop
        n = len(r["admitted"])
        if n and nxt + n <= len(pool):
            o.enqueue(range(pool_base + nxt, pool_base + nxt + n))
            nxt += n
    return {"value": o.decisions / o.fill_s, "steps": steps, "fill_s": o.fill_s, "decisions": o.decisions}


_CAT = {}


def _concat_once(o, q, pool):
    key = (id(q), id(pool))
    if key not in _CAT:
        from paper_2501_14312_b200.workloads import Queue
        flat = np.concatenate([q.flat, pool.flat])
        offs = np.concatenate([q.offsets, pool.offsets + len(q.flat)])
        _CAT[key] = Queue(flat, offs, np.concatenate([q.lens, pool.lens]),
                          np.concatenate([q.clients, pool.clients]), np.concatenate([q.arrival, pool.arrival]),
                          q.rids + pool.rids, np.concatenate([q.labels, pool.labels]))
    return _CAT[key]


def run_cluster(args, wl, rank, world, dev, tdev, dist, clocks=True):
    """N>1: D2LPM across GPUs (paper_2501_14312_b200.cluster): one worker per
    rank, a dispatcher replica on every rank, one NCCL all-gather of finishes
    and eviction notices per round.  The workload's queue is dispatched once
    by D2LPM at t=0 (untimed), so each worker holds ~Nq/N (strong scaling);
    every round then completes the previous batch, exchanges, dispatches the
    round's arrivals on every replica and runs one DLPM fill per worker."""
    import torch
    from paper_2501_14312_b200.cluster import ClusterRank, GpuStreamRank, LocalComm, TorchComm
    from paper_2501_14312_b200.device import launch_count
    U = W_E * wl.L_INPUT + W_Q * wl.M
    q_w = max(1, round(0.5 * U))  # q_w_frac 0.5 (runner.py:131)
    be = GpuStreamRank(rank, dev, wl, world, W_E, W_Q, q_w, max(128, wl.clients))
    comm = TorchComm(tdev) if dist is not None else LocalComm()
    cr = ClusterRank(be, comm, out_tokens=wl.out_tokens, max_arrivals=args.arrivals if args.arrivals > 0 else None,
                     pipelined=True)
    t0 = time.perf_counter()
    cr.seed(list(range(wl.nq)), 0)
    seed_s = time.perf_counter() - t0
    n_seed = wl.nq
    now = 0
    for _ in range(args.warmup):
        now += STEP_US
        cr.round(now, be.arrival_stream)
    be.ctx.sync()
    if dist is not None:
        dist.barrier()
    clk = clocks_start() if (rank == 0 and clocks) else (None, None, None)
    be.fill_ms = 0.0
    be.n_queued = be.n_dispatched = 0
    be.h2d = 0
    be.disp_s = be.upload_s = 0.0
    be.disp_prof[:] = 0
    cr.t_exchange = cr.t_apply = cr.t_dispatch = cr.t_fill = cr.t_overlap = cr.t_upload = cr.t_complete = 0.0
    l0 = launch_count()
    t_start = time.perf_counter()
    for _ in range(args.steps):
        now += STEP_US
        cr.round(now, be.arrival_stream)
    be.ctx.sync()
    wall = time.perf_counter() - t_start
    launches = launch_count() - l0
    clocks = clocks_stop(*clk, dev) if (rank == 0 and clk[0] is not None) else None
    # the dispatcher side (apply + dispatch) overlaps the fill; a round's busy
    # time is completion + exchange + the longer of the two
    busy_s = cr.t_complete + cr.t_exchange + cr.t_overlap
    local = torch.tensor([busy_s, wall, float(be.n_queued), float(be.fill_ms), cr.t_exchange, cr.t_apply,
                          cr.t_dispatch, cr.t_fill, cr.t_upload, cr.t_complete], dtype=torch.float64, device=tdev)
    if dist is not None:
        mx = local.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = local.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    else:
        mx = sm = local
    if rank != 0:
        return
    decisions = float(sm[2]) + be.n_dispatched  # local decisions on every worker + dispatches (replicated: once)
    busy, wall_max = float(mx[0]), float(mx[1])
    line = {
        "metric": METRIC, "value": decisions / busy, "unit": "decisions/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * busy / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32/int64",
        "data": "synthetic",
        "config": {"workload": wl.desc.replace("at D=1: DLPM", f"D2LPM D={world}"), "nq_total": wl.nq,
                   "clients": wl.clients, "M": wl.M, "capacity": wl.CAP, "quantum_local": wl.quantum(),
                   "quantum_global": q_w, "l2": wl.l2,
                   "parallelism": f"D2LPM dp{world}: one worker per GPU, replicated dispatcher, NCCL all-gather "
                                  "of finishes + eviction notices per round",
                   "arrivals_per_round": (f"min({args.arrivals}, cluster admissions of the previous round)"
                                          if args.arrivals > 0 else "cluster admissions of the previous round")
                   + ", dispatched on every replica while the workers fill (pipelined: they join the next "
                     "round's queues)"},
        "e2e": {"value": decisions / wall_max, "unit": "decisions/s",
                "h2d_bytes_per_step": int(be.h2d / args.steps), "d2h_bytes_per_step": None},
        "gpu_launches": int(launches),
        "cluster_ms_per_step": {"fill_device": float(mx[3]) / args.steps,
                                "exchange": 1000 * float(mx[4]) / args.steps,
                                "apply": 1000 * float(mx[5]) / args.steps,
                                "dispatch": 1000 * float(mx[6]) / args.steps,
                                "fill_host_wall": 1000 * float(mx[7]) / args.steps,
                                "arrival_upload": 1000 * float(mx[8]) / args.steps,
                                "complete": 1000 * float(mx[9]) / args.steps},
        "dispatch_detail": {"upload_ms_per_step": 1000 * be.upload_s / args.steps,
                            "call_ms_per_step": 1000 * be.disp_s / args.steps,
                            "kernel_cycles_per_arrival": dict(zip(
                                ["lmw_select", "insert_walk", "evict", "leaf_stamp_repoint", "tags", "total"],
                                (be.disp_prof[[0, 1, 2, 12, 14, 15]] / max(be.n_dispatched, 1)).tolist()))},
        "local_decisions_per_step": float(sm[2]) / args.steps, "dispatches_per_step": be.n_dispatched / args.steps,
        "seed_dispatch": {"arrivals": n_seed, "seconds": seed_s},
        "notice_cycles_per_notice": (dict(zip(["walk", "collect", "edit", "repoint"],
                                              (getattr(be, "notice_prof", np.zeros(4)) /
                                               max(getattr(be, "n_notices", 0), 1)).tolist()))),
        "clocks": clocks, "host_wall_s": wall_max,
    }
    be.close()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=["c2", "c3", "c5"],
                    help="c2 = configs[1] (64k queue), c3 = configs[2] (256k queue, 200 clients; with --cluster "
                         "for D2LPM), c5 = configs[4] (1M queue, 8k prompts)")
    ap.add_argument("--nq", type=int, default=0, help="queued requests per GPU (default: the config's)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--cluster", action="store_true",
                    help="only the D2LPM cluster run (replicated dispatcher over NCCL), also at N=1")
    ap.add_argument("--no-d2lpm", action="store_true", help="N>1: skip the D2LPM cluster run")
    ap.add_argument("--no-sub", action="store_true",
                    help="N=1: skip the config-2 DLPM and config-3 D2LPM sub-results")
    ap.add_argument("--k1-full-steps", type=int, default=3,
                    help="untimed steps after the timed region with the full re-match (scan roofline)")
    ap.add_argument("--arrivals", type=int, default=128,
                    help="cluster path: arrivals per round (a fixed cluster-wide rate, the same at every N; "
                         "0 = as many as the cluster admitted last round)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    dev = local
    tdev = "cpu"
    if world > 1:
        import torch
        import torch.distributed as tdist
        ngpu = torch.cuda.device_count() if args.impl == "ours" else 0
        # one process per GPU over NCCL; ranks sharing a GPU (tests on a
        # single-GPU box) fall back to gloo for the timing plumbing
        if ngpu >= world:
            torch.cuda.set_device(local)
            tdist.init_process_group("nccl")
            tdev = f"cuda:{local}"
        else:
            tdist.init_process_group("gloo")
            dev = local % max(ngpu, 1)
        dist = tdist

    if args.impl == "reference" and rank != 0:
        return  # the reference arm runs on rank 0 only
    cluster = args.cluster
    # the cluster path dispatches ONE shared stream (rank-independent seed);
    # independent workers (N=1) use their rank's seed
    wl = make_workload(args.workload, args.nq, 0 if cluster else rank, args.steps + args.warmup, device=dev,
                       world=world if cluster else 1, cpu_only=args.impl == "reference")
    cfg = {"workload": wl.desc, "nq_per_gpu": wl.nq, "clients": wl.clients, "M": wl.M, "capacity": wl.CAP,
           "quantum": wl.quantum(), "l2": wl.l2,
           "parallelism": f"dp{args.gpus}: one DLPM worker per GPU with its own queue (the local fill has no "
                          "cross-worker exchange; D2LPM across the GPUs is the separate d2lpm_cluster run)"}

    if args.impl == "reference":
        if rank != 0:
            return
        t0 = time.perf_counter()
        q, pool, ncpu = wl.cpu_sample(dev)
        cb = cpu_baseline(wl, q, pool, warmup=args.warmup, steps_max=args.steps, budget_s=120.0)
        line = {"metric": METRIC, "value": cb["value"],
                "unit": "decisions/s", "n_gpus": args.gpus, "steps": cb["steps"], "warmup": args.warmup,
                "ms_per_step": 1000 * cb["fill_s"] / max(cb["steps"], 1), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "int32/int64", "data": "synthetic",
                "config": cfg, "impl": "reference",
                "cpu_baseline": {"value": cb["value"], "unit": "decisions/s", "cores": 1, "kind": "port",
                                 "sample": f"C oracle Dlpm.fill restatement, {cb['steps']} timed serving steps (after {args.warmup} "
                                           f"untimed) of the {ncpu}-request queue of the same config, one core"},
                "e2e": {"value": cb["value"], "unit": "decisions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import refbench
        line["cpu_baseline"].update(refbench.host_info())
        try:
            # the reference's own Python decision path (unmodified, baseline/_ref)
            line["cpu_baseline"]["reference_python"] = refbench.run()
        except Exception as exc:
            line["cpu_baseline"]["reference_python"] = {"unavailable": f"{type(exc).__name__}: {exc}"}
        line["wall_s"] = time.perf_counter() - t0
        print(json.dumps(line))
        return

    from paper_2501_14312_b200.device import launch_count
    if cluster:
        line = run_cluster(args, wl, rank, world, dev, tdev, dist)
        if line is not None:
            print(json.dumps(line))
        return
    g = GpuSteps(wl, dev)
    st = run_dlpm(g, args.steps, args.warmup, dist=dist, rank=rank, dev=dev)
    now = st["now"]
    # ablation after the timed region: the same serving steps with every queued
    # request re-matched from the root (the full streaming scan the incremental
    # match avoids); identical decisions -- reported as the scan kernel's roofline
    full_k1, full_tok, full_n = [], 0, 0
    if args.k1_full_steps > 0:
        g.w.set_k1_full(True)
        for _ in range(args.k1_full_steps):
            now += STEP_US
            r = g.step(now)
            full_k1.append(r.phases_ms[1])
            full_tok += r.stats[0]
            full_n = r.n_queued
        g.w.set_k1_full(False)
    dev_ms, wall, decisions = st["dev_ms"], st["wall"], st["decisions"]
    if dist is not None:
        import torch
        t = torch.tensor([dev_ms, wall], dtype=torch.float64, device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, wall = float(t[0]), float(t[1])
        d = torch.tensor([decisions], dtype=torch.float64, device=tdev)
        dist.all_reduce(d, op=dist.ReduceOp.SUM)
        total_decisions = float(d[0])
    else:
        total_decisions = decisions
    if world > 1 and not args.no_d2lpm:
        # the same GPUs then run D2LPM across them (replicated dispatcher, NCCL
        # exchange) on ONE shared config-5 queue: a second, separately timed run
        g.close()
        g = None
        wl2 = make_workload(args.workload, args.nq, 0, args.steps + args.warmup, device=dev, world=world)
        d2 = run_cluster(args, wl2, rank, world, dev, tdev, dist)
        del wl2
    else:
        d2 = None
    if rank != 0:
        return
    value = total_decisions / (dev_ms / 1000.0)
    e2e = total_decisions / wall
    peak, peak_kind = peaks()
    n_per_step = decisions / args.steps
    k1_avg = float(np.mean(st["k1_ms"]))
    # incremental K1: request tokens actually needed beyond each request's still-
    # valid previous match, plus per-request metadata (queue entry, row offset and
    # length, hint in/out, outputs: 88 B)
    alg_bytes = (st["alg_tok"] / args.steps) * 4 + 88 * n_per_step
    achieved = alg_bytes / (k1_avg / 1000.0) / 1e9
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from k1_traffic import lookup as traffic_lookup
    from paper_2501_14312_b200.build import source_hash
    tr = traffic_lookup(args.workload, wl.nq)
    full_roof = None
    if full_k1:
        fk = float(np.mean(full_k1))
        fb = (full_tok / len(full_k1)) * 4 + 36 * full_n  # 4*min(mlen+1, L) + 36 per request
        full_roof = {"kernel": "k_match with FS_OPT_K1_FULL (every request re-matched from the root)",
                     "bound": "hbm", "achieved": fb / (fk / 1000.0) / 1e9, "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": fb / (fk / 1000.0) / 1e9 / peak, "alg_bytes_per_launch": fb,
                     "avg_launch_ms": fk, "steps": len(full_k1),
                     "traffic": tr.get("full_scan_dram_bytes_per_launch") if tr else None}
    phases = st["phases"]
    share = phases / phases.sum()
    sched = st["sched"]
    steps = args.steps
    line = {
        "metric": METRIC,
        "value": value, "unit": "decisions/s", "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
        "ms_per_step": dev_ms / steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int32/int64", "data": "synthetic", "config": cfg,
        "e2e": {"value": e2e, "unit": "decisions/s",
                "h2d_bytes_per_step": int(st["h2d"] / steps),
                "d2h_bytes_per_step": int(st["d2h"] / steps)},
        "gpu_launches": int(st["launches"]),
        "admissions_per_step": st["adm"] / steps, "queued_per_step": n_per_step,
        "admissions_per_s": st["adm"] / (dev_ms / 1000.0),
        "roofline": {"kernel": "k_match (K1 incremental prefix match)", "bound": "hbm", "achieved": achieved,
                     "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": tr["dram_bytes_per_launch"] if tr else None,
                     "traffic_source": (tr["source"] + f" (build {tr['source_hash']})") if tr else
                     f"no ncu capture filed for build {source_hash()} / {args.workload} / nq={wl.nq} "
                     "(tools/k1_traffic.py)",
                     "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": k1_avg,
                     "note": "resumes each request from its still-valid previous match; reads only the tokens "
                             "past it, so it is latency- not bandwidth-bound; see k1_full_match_roofline for the "
                             "streaming scan"},
        "k1_full_match_roofline": full_roof,
        "phase_share": {"merge": share[0], "k1_match": share[1], "k2_sort": share[2], "k3k4_schedule": share[3],
                        "unpin": share[4]},
        "dominant_kernel": {"kernel": "k_schedule (K3/K4 admission chain, one CTA)", "share": share[3],
                            "bound": "latency (serial admission chain; see sched_profile_per_step)",
                            "avg_launch_ms": phases[3] / steps},
        "phase_ms_per_step": {"merge": phases[0] / steps, "k1_match": phases[1] / steps,
                              "k2_sort": phases[2] / steps, "k3k4_schedule": phases[3] / steps,
                              "unpin": phases[4] / steps},
        "sched_profile_per_step": {"find_cyc": sched[0] / steps, "walk_cyc": sched[1] / steps,
                                   "evict_cyc": sched[2] / steps, "tail_cyc": sched[3] / steps,
                                   "chunks": sched[4] / steps, "evict_pops": sched[5] / steps,
                                   "admit_chains": sched[6] / steps, "k1_chains": st["k1_hops"] / steps,
                                   "resumes": st["resumes"] / steps, "refill_events": st["refills"] / steps,
                                   "pop_argmin_cyc": sched[8] / steps, "pop_edit_cyc": sched[9] / steps,
                                   "pop_update_cyc": sched[10] / steps, "setup_cyc": sched[11] / steps,
                                   "grid_sweeps": sched[15] / steps, "grid_sweep_cyc": sched[14] / steps,
                                   "side_cyc": sched[12] / steps, "leaf_cyc": sched[13] / steps,
                                   "total_cyc": sched[7] / steps,
                                   "pin_cyc": st["ext"][0] / steps, "on_walk_cyc": st["ext"][1] / steps,
                                   "fev_setup_wait_cyc": st["ext"][2] / steps,
                                   "on_walk_pre_put_cyc": st["ext"][3] / steps, "on_walk_post_put_cyc": st["ext"][4] / steps,
                                   "fev_orders": st["fev"][0] / steps, "fev_cold_leaves": st["fev"][1] / steps,
                                   "fev_heap_hw": st["fev"][2] / steps, "fev_ok_fills": st["fev"][3] / steps},
        "clocks": st["clocks"], "host_wall_s": st["t_total"],
    }
    if d2 is not None:
        line["d2lpm_cluster"] = {k: d2[k] for k in ("value", "unit", "ms_per_step", "scaling", "e2e", "config",
                                                   "cluster_ms_per_step", "local_decisions_per_step",
                                                   "dispatches_per_step", "seed_dispatch",
                                                   "notice_cycles_per_notice", "gpu_launches")}
    if g is not None:
        g.close()
    if world == 1 and not args.no_sub:
        # the other single-GPU configurations, each separately timed after the
        # headline: configs[1] (64k queue, DLPM) and configs[2]'s D2LPM queue
        # (256k, 200 clients) through the dispatcher + one worker
        subs = {}
        sub_steps, sub_warm = max(3, min(args.steps, 20)), max(3, min(args.warmup, 5))
        wl2 = make_workload("c2", 0, 0, sub_steps + sub_warm, device=dev)
        g2 = GpuSteps(wl2, dev)
        s2 = run_dlpm(g2, sub_steps, sub_warm, dev=dev, clocks=False)
        g2.close()
        subs["config2_dlpm"] = {
            "workload": wl2.desc, "value": s2["decisions"] / (s2["dev_ms"] / 1000.0), "unit": "decisions/s",
            "steps": sub_steps, "warmup": sub_warm, "ms_per_step": s2["dev_ms"] / sub_steps,
            "e2e": {"value": s2["decisions"] / s2["wall"], "unit": "decisions/s",
                    "h2d_bytes_per_step": int(s2["h2d"] / sub_steps), "d2h_bytes_per_step": int(s2["d2h"] / sub_steps)},
            "admissions_per_step": s2["adm"] / sub_steps, "admissions_per_s": s2["adm"] / (s2["dev_ms"] / 1000.0),
            "k3k4_schedule_share": float(s2["phases"][3] / s2["phases"].sum()), "gpu_launches": int(s2["launches"]),
            "l2": wl2.l2}
        del wl2, g2
        import types
        wl3 = make_workload("c3", 0, 0, sub_steps + sub_warm, device=dev)
        a3 = types.SimpleNamespace(steps=sub_steps, warmup=sub_warm, gpus=1, arrivals=args.arrivals)
        d3 = run_cluster(a3, wl3, 0, 1, dev, tdev, None, clocks=False)
        subs["config3_d2lpm"] = {k: d3[k] for k in ("value", "unit", "ms_per_step", "e2e", "config",
                                                   "cluster_ms_per_step", "local_decisions_per_step",
                                                   "dispatches_per_step", "dispatch_detail", "seed_dispatch",
                                                   "notice_cycles_per_notice", "gpu_launches")}
        subs["config3_d2lpm"]["steps"], subs["config3_d2lpm"]["warmup"] = sub_steps, sub_warm
        del wl3
        try:
            # configs[3]'s post-run service-gap checks at 1000 clients
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            import verify_bench
            subs["config4_verifiers"] = verify_bench.run()
        except Exception as exc:  # needs the unmodified reference's ServiceLog (baseline/_ref)
            subs["config4_verifiers"] = {"unavailable": f"{type(exc).__name__}: {exc}"}
        line["sub_results"] = subs
    if not args.no_cpu and world == 1:
        q, pool, ncpu = wl.cpu_sample(dev)
        cb = cpu_baseline(wl, q, pool, warmup=args.warmup, steps_max=args.steps, budget_s=20.0)
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import refbench
        line["cpu_baseline"] = {"value": cb["value"], "unit": "decisions/s", "cores": 1, "kind": "port",
                                **refbench.host_info(),
                                "sample": f"C oracle (literal Dlpm.fill restatement), {cb['steps']} timed serving steps "
                                          f"(after {args.warmup} untimed) of a {ncpu}-request queue of the same config, one host core"}
        try:
            line["cpu_baseline"]["reference_python"] = refbench.run(
                normal_sizes=(4096, 16384), steady_sizes=(4096,), indebted_sizes=(1024, 2048, 4096),
                dispatch_D=(1, 8), dispatch_n=4096)
        except Exception as exc:  # the unmodified reference is optional on the GPU box
            line["cpu_baseline"]["reference_python"] = {"unavailable": f"{type(exc).__name__}: {exc}"}
    print(json.dumps(line))


def run_dlpm(g, steps, warmup, dist=None, rank=0, dev=0, clocks=True):
    """W untimed then K timed serving steps of a GpuSteps loop; per-step device
    time (CUDA events inside the library: the fill + the completion unpins)
    and host wall time of the public-API calls."""
    from paper_2501_14312_b200.device import launch_count
    now = 0
    for _ in range(warmup):
        now += STEP_US
        g.step(now)
    g.ctx.sync()
    if dist is not None:
        dist.barrier()
    clk = clocks_start() if (rank == 0 and clocks) else (None, None, None)
    l0 = launch_count()
    h2d0, d2h0 = g.h2d, g.d2h
    st = {"dev_ms": 0.0, "wall": 0.0, "decisions": 0, "adm": 0, "alg_tok": 0, "k1_ms": [], "phases": np.zeros(5),
          "sched": np.zeros(16), "k1_hops": 0, "resumes": 0, "refills": 0, "fev": np.zeros(4), "ext": np.zeros(8)}
    t_start = time.perf_counter()
    for _ in range(steps):
        now += STEP_US
        t0 = time.perf_counter()
        u0 = g.unpin_ms
        res = g.step(now)
        st["wall"] += time.perf_counter() - t0
        st["dev_ms"] += res.device_ms + (g.unpin_ms - u0)  # the fill plus the completion unpins
        st["decisions"] += res.n_queued
        st["adm"] += len(res.adm_req)
        st["alg_tok"] += res.stats[0]
        st["k1_ms"].append(res.phases_ms[1])
        st["phases"] += np.array(list(res.phases_ms) + [g.unpin_ms - u0])
        st["sched"] += np.array(res.stats[8:24], dtype=np.float64)
        st["k1_hops"] += res.stats[6]
        st["resumes"] += res.stats[4]
        st["refills"] += res.stats[3]
        f = int(res.stats[7])  # FEV: orders | cold leaves << 20 | heap high water << 40 | ok << 60
        st["ext"] += np.array(res.stats_ext, dtype=np.float64)
        st["fev"] += np.array([f & 0xfffff, (f >> 20) & 0xfffff, (f >> 40) & 0xfffff, (f >> 60) & 1])
    g.ctx.sync()
    st["t_total"] = time.perf_counter() - t_start
    st["launches"] = launch_count() - l0
    st["clocks"] = clocks_stop(*clk, dev) if (rank == 0 and clocks) else None
    st["h2d"], st["d2h"] = g.h2d - h2d0, g.d2h - d2h0
    st["now"] = now
    return st


if __name__ == "__main__":
    main()
