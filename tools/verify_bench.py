"""Timing of the GPU service-gap verifiers (paper_2501_14312_b200.verify,
SURVEY 8f.4) at config-4 scale (1000 clients, bursty arrivals), beside the
reference's own metrics functions on a bounded sample (the reference's
pairwise check is O(C^2) Python loops; its max-min check O(C^3)).

    python tools/verify_bench.py            # prints one JSON object
"""
from __future__ import annotations

import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def bursty_case(n_clients, n_req, horizon_us, seed):
    """Lifecycle + ServiceLog shaped like a config-4 run: Gamma(cv=4) bursts per
    client, admissions after a queueing delay, a few output events each."""
    from fairsched.accounting import CostWeights, ServiceLog
    rng = random.Random(seed)
    names = [f"client{i:04d}" for i in range(n_clients)]
    life, events = {}, []
    per = max(1, n_req // n_clients)
    k = 0
    for c in names:
        t = rng.randrange(horizon_us // 10)
        for _ in range(per):
            t += int(rng.gammavariate(1 / 16, 16 * horizon_us / per))  # cv = 4
            if t >= horizon_us:
                break
            rec = {"rid": f"r{k}", "client": c, "arrival_time": t}
            k += 1
            if rng.random() < 0.95:
                adm = t + rng.randrange(0, horizon_us // 50)
                rec["admit_time"] = adm
                events.append((adm, c, rng.randrange(64, 2048)))
                for s in range(4):
                    events.append((adm + 1000 * (s + 1), c, -8))
            life[rec["rid"]] = rec
    svc = ServiceLog(CostWeights(1, 2))
    for t, c, u in sorted(events, key=lambda e: e[0]):
        if u > 0:
            svc.add_extend(t, c, u, u + 256)
        else:
            svc.add_output(t, c, -u)
    return svc, life, horizon_us + horizon_us // 10


def timed(fn, *a, **kw):
    t0 = time.perf_counter()
    r = fn(*a, **kw)
    return r, time.perf_counter() - t0


def run(n_clients=1000, n_req=40000, sample_clients=60, seed=4):
    from refpath import import_fairsched
    fs = import_fairsched()
    from fairsched import metrics
    from paper_2501_14312_b200 import verify

    out = {"clients": n_clients, "requests": n_req}
    svc, life, end = bursty_case(n_clients, n_req, 60_000_000, seed)
    verify.verify_service_bound_pairwise(svc, life, 1, end, "warm")  # context + module load
    gpu = {}
    for name in ("verify_service_bound_pairwise", "verify_service_bound_vs_nonbacklogged"):
        r, dt = timed(getattr(verify, name), svc, life, 1e9, end, name)
        gpu[name] = {"s": dt, "measured": r.measured, "detail": r.detail}
    out["gpu"] = gpu
    # the same checks by the reference and by the GPU on a bounded sample
    svc2, life2, end2 = bursty_case(sample_clients, n_req * sample_clients // n_clients, 60_000_000, seed + 1)
    samp = {"clients": sample_clients}
    for name in ("verify_service_bound_pairwise", "verify_service_bound_vs_nonbacklogged", "verify_global_max_min"):
        rr, tr = timed(getattr(metrics, name), svc2, life2, 1e9, end2, name)
        rg, tg = timed(getattr(verify, name), svc2, life2, 1e9, end2, name)
        samp[name] = {"reference_s": tr, "gpu_s": tg, "identical": rr.row() == rg.row()}
    out["sample"] = samp
    return out


if __name__ == "__main__":
    print(json.dumps(run()))
