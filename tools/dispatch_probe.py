"""Probe (not a test): D2LPM dispatch-chain throughput on config-5 arrivals.

    python tools/dispatch_probe.py [n] [D]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2501_14312_b200.device import Context, DispatcherDev  # noqa: E402
from paper_2501_14312_b200.trace import add_segments  # noqa: E402
from paper_2501_14312_b200.workloads import config5, deep_tree_segments  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
D = int(sys.argv[2]) if len(sys.argv) > 2 else 8
spec = config5(n)
segs, clients, labels = deep_tree_segments(spec, 0, n)
ctx = Context(0, arena_tokens=n * 8192 + 4 * n + 1024, max_requests=n + 16)
ids = add_segments(ctx, segs, clients, labels)
U = 8192 + 2 * 262144
d = DispatcherDev(ctx, D, max(1, round(0.5 * U)), 1, 2, max_clients=256)
for batch in (256, 4096):
    pass
t0 = time.perf_counter()
done = 0
for a in range(0, n, 4096):
    b = min(n, a + 4096)
    d.dispatch(ids[a:b], clients[a:b], np.zeros(b - a, np.int64))
    done = b
    prof = d.last_profile()
    if a == 0 or b == n:
        print("cycles/arrival: lmw+select %.0f insert-walk %.0f leaf+repoint %.0f tags %.0f total %.0f"
              % tuple(x / (b - a) for x in (prof[0], prof[1], prof[12], prof[14], prof[15])))
    if time.perf_counter() - t0 > 60:
        break
ctx.sync()
dt = time.perf_counter() - t0
print(f"dispatched {done} arrivals at D={D} in {dt:.2f}s: {dt / done * 1e6:.1f} us each; "
      f"queue sizes {d.queue_sizes().tolist()}")
