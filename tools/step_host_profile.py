"""Host-side breakdown of one bench serving step (GpuSteps.step) on the GPU box:
wall time of each public-API call of the step, to locate the e2e vs device gap.

    python tools/step_host_profile.py [--workload c5] [--steps 20]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import ctypes as C  # noqa: E402

import bench  # noqa: E402
from paper_2501_14312_b200._lib import call  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    wl = bench.make_workload(args.workload, 0, 0, args.steps + args.warmup + 2, device=0)
    g = bench.GpuSteps(wl, 0)
    now = 0
    for _ in range(args.warmup):
        now += bench.STEP_US
        g.step(now)
    g.ctx.sync()
    T = {}

    def timed(name, fn, *a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        T.setdefault(name, []).append(time.perf_counter() - t0)
        return r

    walls, devs = [], []
    for _ in range(args.steps):
        now += bench.STEP_US
        t_step = time.perf_counter()
        n_prev = len(g.prev_nodes)
        if n_prev:
            per = timed("bincount", np.bincount, g.prev_clients)
            cl = np.flatnonzero(per).astype(np.int32)
            timed("outputs", g.w.outputs, cl, per[cl].astype(np.int64) * g.wl.out_tokens)
            timed("unpin_async", g.trie.unpin_many_async, g.prev_nodes)
        if n_prev and g.pool_next + n_prev <= len(g.pool):
            a, b = g.pool_next, g.pool_next + n_prev
            timed("upload_pre", g._upload, b)
            timed("enqueue", g.w.enqueue, g.pool_ids[a:b])
            g.pool_next = b
        timed("fill_begin", g.w.fill_begin, now, 0, 0)
        timed("upload_next", g._upload, min(len(g.pool), g.pool_next + max(64, 2 * n_prev)))
        rs, g.w._res = g.w._res, None
        timed("fill_end_c", call, "fs_worker_fill_end", g.w._h, C.byref(rs))
        res = timed("fill_end_py", g.w._result, rs)
        gp = (C.c_float * 2)()
        call("fs_worker_last_gaps", g.w._h, gp)
        T.setdefault("dev_staging", []).append(gp[0] / 1e3)
        if gp[1] >= 0:
            T.setdefault("dev_gap_before_fill", []).append(gp[1] / 1e3)
        t0 = time.perf_counter()
        g.prev_nodes = res.adm_node.astype(np.int32)
        g.prev_clients = g.clients[np.asarray(res.adm_req, np.int64)]
        T.setdefault("post", []).append(time.perf_counter() - t0)
        walls.append(time.perf_counter() - t_step)
        devs.append(res.device_ms)
    print(f"step wall {1e3 * np.mean(walls):.3f} ms, fill device {np.mean(devs):.3f} ms")
    for k, v in T.items():
        print(f"  {k:12s} {1e6 * np.mean(v):8.1f} us  (max {1e6 * np.max(v):.1f})")
    g.close()


if __name__ == "__main__":
    main()
