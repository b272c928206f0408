"""Record reference runs for the policies OTHER than DLPM/LPM/D2LPM that still
run on the device radix tree once the plugin is installed (run in the build
container only):

    python tests/golden/make_golden_policies.py           # policies_runs.json.gz
    python tests/golden/make_golden_policies.py config4   # config4_runs.json.gz

* config-4 style comparison (SURVEY 8d cfg 4, scaled to seconds of CPU):
  one bursty trace (Gamma arrivals, cv=4), many clients, local policies
  dlpm / vtc / lpm / fcfs on the same trace (`cli compare`, cli.py:62-89);
* global routers rr / per_client_rr / threshold / d2lpm at D=2..4 with vtc and
  dlpm workers (ThresholdRouter shares the radix index, global_policies.py:135-161).

Each run stores the config, the trace and the reference event-log sha256
(engine.py:133) plus the service-gap verifier's violation counts
(metrics.py:148-174).  Fixture: policies_runs.json.gz.
"""
from __future__ import annotations

import gzip
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from fairsched.runner import config_from_dict, run_experiment  # noqa: E402
from fairsched.workload import ClientProfile, generate_trace  # noqa: E402
from fairsched.engine import ms  # noqa: E402


def bursty_clients(n, rng, L_input):
    out = []
    for i in range(n):
        prefix = rng.randrange(16, L_input // 2)
        out.append(dict(name=f"c{i:03d}", rate=rng.uniform(0.5, 2.0) * 20, cv=4.0,
                        prefix_len=prefix, suffix_len=rng.randrange(4, 24),
                        output_len=rng.randrange(2, 10), prefix_scope=rng.choice(["client", "program"])))
    return out


def config(seed, local, glob, D, clients, L_input=128, M=512, horizon=300, extra=None):
    d = {
        "seed": seed, "horizon_ms": horizon, "latency_window_ms": 100,
        "params": {"L_input": L_input, "L_output": 32, "M": M, "D": D},
        "scheduling": {"local_policy": local, "global_policy": glob, "q_u_frac": 0.5, "q_w_frac": 0.5,
                       "output_reserve": 4, "theta": 0.5},
        "clients": clients,
    }
    if extra:
        d["scheduling"].update(extra)
    return d


def config4_clients(n=1000, seed=4):
    """SURVEY 8d cfg 4: C=1000 ClientProfiles, cv=4 (bursty Gamma arrivals),
    rate ~ U[0.5, 2]/s, prefix 256-2048 tokens, suffix 64."""
    rng = random.Random(seed)
    return [dict(name=f"c{i:04d}", rate=rng.uniform(0.5, 2.0), cv=4.0, prefix_len=rng.randint(256, 2048),
                 suffix_len=64, output_len=8, prefix_scope="client") for i in range(n)]


def config4(local, horizon_ms=2000, n_clients=1000):
    """D=1, L_input 4096, M 65536, q_u_frac 0.5, seed 4; the horizon is cut to
    2 s (8,342 requests) so the CPU reference records each policy in minutes."""
    return {"seed": 4, "horizon_ms": horizon_ms, "latency_window_ms": 500,
            "params": {"L_input": 4096, "L_output": 64, "M": 65536, "D": 1},
            "scheduling": {"local_policy": local, "global_policy": "rr", "q_u_frac": 0.5, "output_reserve": 8},
            "clients": config4_clients(n_clients)}


def main_config4():
    """dlpm / vtc / lpm on the same 1000-client bursty trace (cli compare,
    cli.py:62-89): event sha256, monitor violations, counter extremes."""
    import time
    runs = []
    cfg0 = config_from_dict(config4("dlpm"))
    trace = generate_trace(cfg0.clients, cfg0.params, cfg0.seed, ms(cfg0.horizon_ms))
    recs = [json.loads(r.to_json()) for r in trace.records]
    for local in ("dlpm", "vtc", "lpm"):
        d = config4(local)
        t0 = time.time()
        res = run_experiment(config_from_dict(d), trace)
        runs.append({"name": f"config4-{local}", "config": d, "event_sha256": res.log.sha256(),
                     "violations": {k: len(v) for k, v in res.violations.items()},
                     "extremes": {k: list(v) for k, v in res.counter_extremes.items()},
                     "reference_seconds": time.time() - t0})
        print(runs[-1]["name"], runs[-1]["event_sha256"][:16], runs[-1]["reference_seconds"], flush=True)
    with gzip.open(os.path.join(HERE, "config4_runs.json.gz"), "wt") as fh:
        json.dump({"trace": recs, "runs": runs}, fh, separators=(",", ":"))


def main():
    runs = []
    rng = random.Random(4)
    # config-4 style: the same bursty trace under four local policies
    for k, (n_clients, D) in enumerate([(120, 1), (60, 1), (40, 2)]):
        clients = bursty_clients(n_clients, rng, 128)
        base = config(4000 + k, "dlpm", "rr", D, clients)
        cfg0 = config_from_dict(base)
        trace = generate_trace(cfg0.clients, cfg0.params, cfg0.seed, ms(cfg0.horizon_ms))
        for local in ("dlpm", "vtc", "lpm", "fcfs"):
            d = config(4000 + k, local, "rr", D, clients)
            res = run_experiment(config_from_dict(d), trace)
            runs.append({"name": f"cmp{k}-{local}", "config": d,
                         "trace": [json.loads(r.to_json()) for r in trace.records],
                         "event_sha256": res.log.sha256(),
                         "violations": {k2: len(v) for k2, v in res.violations.items()}})
    # global routers with device-tree workers
    for k, (glob, local, D) in enumerate([("threshold", "vtc", 2), ("threshold", "dlpm", 4), ("per_client_rr", "vtc", 3),
                                          ("rr", "fcfs", 2), ("d2lpm", "vtc", 2), ("threshold", "lpm", 3)]):
        clients = bursty_clients(rng.randrange(6, 20), rng, 128)
        d = config(4100 + k, local, glob, D, clients, extra={"theta": rng.choice([0.3, 0.5, 0.8])})
        cfg = config_from_dict(d)
        trace = generate_trace(cfg.clients, cfg.params, cfg.seed, ms(cfg.horizon_ms))
        res = run_experiment(cfg, trace)
        runs.append({"name": f"route{k}-{glob}-{local}-D{D}", "config": d,
                     "trace": [json.loads(r.to_json()) for r in trace.records],
                     "event_sha256": res.log.sha256(),
                     "violations": {k2: len(v) for k2, v in res.violations.items()}})
    with gzip.open(os.path.join(HERE, "policies_runs.json.gz"), "wt") as fh:
        json.dump({"runs": runs}, fh, separators=(",", ":"))
    print("wrote policies_runs.json.gz:", [(r["name"], len(r["trace"])) for r in runs])


if __name__ == "__main__":
    if sys.argv[1:] == ["config4"]:
        main_config4()
    else:
        main()
