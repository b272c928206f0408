"""Probe (not a test): wall clock of the reference's unchanged serving
simulator (fairsched.runner.run_experiment) with the GPU drop-in, with and
without the host bookkeeping fast path (hostpath.py), on a large bursty
trace; the event hashes must agree.

    python tools/plugin_probe.py [clients] [rate] [horizon_ms]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from refpath import import_fairsched  # noqa: E402

import_fairsched()
from fairsched.runner import config_from_dict, run_experiment  # noqa: E402
from fairsched.workload import generate_trace  # noqa: E402
from fairsched.engine import ms  # noqa: E402
from paper_2501_14312_b200 import plugin  # noqa: E402
from paper_2501_14312_b200.runtime import reset_runtimes  # noqa: E402

n_clients = int(sys.argv[1]) if len(sys.argv) > 1 else 64
rate = float(sys.argv[2]) if len(sys.argv) > 2 else 200.0
horizon = int(sys.argv[3]) if len(sys.argv) > 3 else 400
d = {"seed": 11, "horizon_ms": horizon, "latency_window_ms": 100,
     "params": {"L_input": 1024, "L_output": 32, "M": 16384, "D": 1},
     "scheduling": {"local_policy": "dlpm", "global_policy": "rr", "q_u_frac": 0.5, "q_w_frac": 0.5,
                    "output_reserve": 4},
     "clients": [dict(name=f"c{i:03d}", rate=rate, cv=4.0, prefix_len=512, suffix_len=64, output_len=8,
                      prefix_scope="program" if i % 3 else "client") for i in range(n_clients)]}
cfg = config_from_dict(d)
trace = generate_trace(cfg.clients, cfg.params, cfg.seed, ms(cfg.horizon_ms))
print(f"{len(trace.records)} requests", flush=True)
out = {}
for fast in (False, True, False, True):
    plugin.install(host_fast_path=fast)
    t0 = time.perf_counter()
    res = run_experiment(config_from_dict(d), trace)
    out[fast] = (time.perf_counter() - t0, res.log.sha256())
    plugin.uninstall()
    reset_runtimes()
    print(f"host fast path {fast}: {out[fast][0]:.2f} s  sha {out[fast][1][:16]}", flush=True)
assert out[True][1] == out[False][1]
if os.environ.get("PROBE_REFERENCE"):
    t0 = time.perf_counter()
    res = run_experiment(config_from_dict(d), trace)  # the unmodified reference (CPU)
    print(f"reference (CPU, no plugin): {time.perf_counter() - t0:.2f} s  sha {res.log.sha256()[:16]}")
if os.environ.get("PROBE_PROFILE"):
    import cProfile
    import pstats
    plugin.install()
    cProfile.run("run_experiment(config_from_dict(d), trace)", "/tmp/plugin_probe.prof")
    plugin.uninstall()
    pstats.Stats("/tmp/plugin_probe.prof").sort_stats("tottime").print_stats(15)
