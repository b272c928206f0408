"""Probe (not a test): Python-side cost of Context.add_requests."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import bench
from paper_2501_14312_b200 import device as D

wl = bench.make_workload("c5", 16384, 0, 40)
g = bench.GpuSteps(wl, 0)
p = g.pool
ctx = g.ctx
for trial in range(3):
    a, b = 80 * trial, 80 * trial + 80
    o0 = int(p.offsets[a]); o1 = int(p.offsets[b - 1] + p.lens[b - 1])
    t0 = time.perf_counter()
    args = (p.flat[o0:o1], p.offsets[a:b] - o0, p.lens[a:b], p.clients[a:b], p.labels[a:b])
    t1 = time.perf_counter()
    ids = ctx.add_requests(*args)
    t2 = time.perf_counter()
    print(f"slice {1e6*(t1-t0):.0f} us, add_requests {1e6*(t2-t1):.0f} us", flush=True)
import cProfile, pstats
a, b = 400, 480
o0 = int(p.offsets[a]); o1 = int(p.offsets[b - 1] + p.lens[b - 1])
cProfile.run("ctx.add_requests(p.flat[o0:o1], p.offsets[a:b] - o0, p.lens[a:b], p.clients[a:b], p.labels[a:b])", "/tmp/prof")
pstats.Stats("/tmp/prof").sort_stats("cumtime").print_stats(8)
