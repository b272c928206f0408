"""Record reference runs whose arrivals come in same-timestamp bursts (run in
the build container only):

    python tests/golden/make_golden_burst.py

A generated bursty trace (flat programs) with its arrival times floored to a
5 ms grid, so dozens of requests arrive at the same microsecond: the runs
exercise the drop-in dispatchers' same-timestamp batches (one device call per
run of arrivals) under d2lpm and threshold routing.  Each run
stores the config, the trace and the reference event-log sha256
(engine.py:133).  Fixture: burst_runs.json.gz.
"""
from __future__ import annotations

import gzip
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from fairsched.engine import ms  # noqa: E402
from fairsched.requests import Trace, TraceRecord  # noqa: E402
from fairsched.runner import config_from_dict, run_experiment  # noqa: E402
from fairsched.workload import generate_trace  # noqa: E402


def config(seed, glob, D, local="dlpm", theta=0.5):
    rng = random.Random(seed)
    clients = [dict(name=f"b{i:02d}", rate=rng.uniform(20, 60), cv=2.0, prefix_len=rng.randrange(16, 64),
                    suffix_len=rng.randrange(4, 16), output_len=rng.randrange(2, 8),
                    prefix_scope=rng.choice(["client", "program"])) for i in range(12)]
    return {"seed": seed, "horizon_ms": 300, "latency_window_ms": 100,
            "params": {"L_input": 128, "L_output": 32, "M": 512, "D": D},
            "scheduling": {"local_policy": local, "global_policy": glob, "q_u_frac": 0.5, "q_w_frac": 0.5,
                           "output_reserve": 4, "theta": theta},
            "clients": clients}


def main():
    runs = []
    for k, (glob, D, local, theta) in enumerate([("d2lpm", 4, "dlpm", 0.5), ("d2lpm", 2, "lpm", 0.5),
                                                 ("threshold", 3, "dlpm", 0.3), ("threshold", 4, "vtc", 0.6)]):
        d = config(5100 + k, glob, D, local, theta)
        cfg = config_from_dict(d)
        trace = generate_trace(cfg.clients, cfg.params, cfg.seed, ms(cfg.horizon_ms))
        recs = []
        for r in trace.records:
            x = json.loads(r.to_json())
            x["arrival_time"] = (x["arrival_time"] // 5000) * 5000
            recs.append(x)
        recs.sort(key=lambda x: (x["arrival_time"], x["rid"].count("."), x["rid"]))
        tr = Trace([TraceRecord(**x) for x in recs])
        res = run_experiment(cfg, tr)
        same = len(recs) - len({x["arrival_time"] for x in recs})
        runs.append({"name": f"burst{k}-{glob}-{local}-D{D}", "config": d, "trace": recs,
                     "event_sha256": res.log.sha256(), "same_time_arrivals": same})
        print(runs[-1]["name"], len(recs), same, runs[-1]["event_sha256"][:16])
    with gzip.open(os.path.join(HERE, "burst_runs.json.gz"), "wt") as fh:
        json.dump({"runs": runs}, fh, separators=(",", ":"))


if __name__ == "__main__":
    main()
