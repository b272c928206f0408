import sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np
import bench
wl = bench.make_workload("c5", 0, 0, 40)
g = bench.GpuSteps(wl, 0)
now = 0
for _ in range(4):
    now += bench.STEP_US; g.step(now)
T = {}
orig = {}
def wrap(obj, name, key):
    f = getattr(obj, name)
    def w(*a, **k):
        t0 = time.perf_counter(); r = f(*a, **k); T[key] = T.get(key, 0) + time.perf_counter() - t0; return r
    setattr(obj, name, w)
wrap(g.w, "outputs", "outputs"); wrap(g.trie, "unpin_many_async", "unpin"); wrap(g.ctx, "add_requests", "add_requests")
wrap(g.w, "enqueue", "enqueue"); wrap(g.w, "fill_begin", "fill_begin"); wrap(g.w, "fill_end", "fill_end")
wrap(g.trie, "last_ms", "last_ms")
t0 = time.perf_counter(); dev = 0
for _ in range(20):
    now += bench.STEP_US; r = g.step(now); dev += r.device_ms
wall = time.perf_counter() - t0
print("wall ms/step", 1000 * wall / 20, "fill device ms/step", dev / 20)
for k, v in T.items(): print(k, round(1000 * v / 20, 3))
