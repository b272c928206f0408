"""CPU baseline: the reference's OWN decision path (fairsched from baseline/_ref,
Cython `common_prefix_len` when it was built) timed on this host's cores.

This is not the product and not the oracle: it imports the unmodified
reference package and times its public classes with time.perf_counter, the
way BASELINE.md section 3 asks:

* `Dlpm.fill` (local_policies.py:108-128) on a real `Worker` / `RadixTree`
  (worker.py:42-135, radix.py), config-2 generator queues (100 clients,
  1-4k-token prompts, Zipf(1.1) document prefixes, M = capacity = 65,536,
  reserve 8), Nq in {4k, 16k, 64k}:
    - normal regime, first fill: every client at q = 0, empty cache (the LPM
      sort's Nq walks, then admissions until the M budget is spent);
    - normal regime, steady fill: the next fill after that batch completed
      (warm cache, evictions; every admission pays the reference's O(Nq)
      queue.remove / pending.remove and O(batch) _reserved_headroom);
    - indebted regime (local_policies.py:116-120): no request fits the
      M-token budget and one queued client holds credit, so every indebted
      request re-scans the pending set for credit -- O(N^2);
  with the scaling exponent fitted over the sizes;
* `D2lpm.dispatch` (global_policies.py:40-46, 88-132) of 16k arrivals over
  200 clients at D = 1 and D = 8.

One core: the reference is a single-threaded event loop under the GIL.
"""
from __future__ import annotations

import math
import os
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def import_reference():
    p = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(p, "fairsched")) and p not in sys.path:
        sys.path.insert(0, p)
    import fairsched  # noqa: F401
    from fairsched import speedups
    return speedups.KERNEL_IMPL


def host_info():
    model = platform.processor() or ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def _requests(q, Request, first=0, n=None):
    n = len(q) if n is None else n
    out = []
    for i in range(first, first + n):
        toks = tuple(q.tokens(i).tolist())
        out.append(Request(rid=q.rids[i], client=f"c{int(q.clients[i]):03d}", input_tokens=toks,
                           arrival=int(q.arrival[i])))
    return out


def _worker(M=65536, reserve=8, L_input=4096, policy=None):
    from fairsched.accounting import CostWeights, ServiceLog
    from fairsched.engine import Simulator
    from fairsched.local_policies import Dlpm
    from fairsched.requests import SystemParams
    from fairsched.worker import StepTiming, Worker
    params = SystemParams(L_input=L_input, L_output=64, M=M, D=1)
    weights = CostWeights(1, 2)
    U = weights.w_e * L_input + weights.w_q * M
    pol = policy or Dlpm(max(1, round(0.5 * U)))
    sim = Simulator(seed=0)
    w = Worker(sim, 0, params, weights, StepTiming(), pol, ServiceLog(weights), {}, output_reserve=reserve)
    return w, pol, sim


def _enqueue(w, pol, reqs):
    for r in reqs:
        w.queue.append(r)
        pol.on_request_enqueued(r, False)


def _complete_batch(w, pol):
    """The admitted batch finishes: output charge and unpin (worker.py:187-213)."""
    outs = {}
    for e in w.batch.values():
        outs[e.request.client] = outs.get(e.request.client, 0) + 8
        w.tree.unpin(e.path)
    pol.on_outputs(outs)
    w.batch.clear()


def time_fill_normal(nq, seed=2, steady=True):
    from fairsched.requests import Request
    from paper_2501_14312_b200.workloads import build_docs, config2, shared_prefix_queue
    spec = config2(nq, seed=seed)
    q = shared_prefix_queue(spec, docs=build_docs(spec))
    reqs = _requests(q, Request)
    w, pol, sim = _worker()
    _enqueue(w, pol, reqs)
    sim.now = 10_000
    t0 = time.perf_counter()
    pol.fill()                   # cold cache: warms it, admits a first batch
    cold = time.perf_counter() - t0
    first = {"nq": nq, "seconds": cold, "decisions_per_s": nq / cold, "admitted": nq - len(w.queue)}
    if not steady:
        return first, None
    _complete_batch(w, pol)
    sim.now = 20_000
    n = len(w.queue)
    t0 = time.perf_counter()
    pol.fill()                   # steady state: warm cache, q as the first batch left it
    dt = time.perf_counter() - t0
    return first, {"nq": n, "seconds": dt, "decisions_per_s": n / dt, "admitted": n - len(w.queue)}


def time_fill_indebted(nq, seed=2):
    from fairsched.requests import Request
    from paper_2501_14312_b200.workloads import build_docs, config2, shared_prefix_queue
    spec = config2(nq, seed=seed)
    q = shared_prefix_queue(spec, docs=build_docs(spec))
    reqs = _requests(q, Request)
    w, pol, sim = _worker()
    _enqueue(w, pol, reqs)
    rich = reqs[0].client
    for c in pol.client_list:
        pol.q[c] = 1 if c == rich else -1
    w.generated_total = w.params.M  # nothing fits the M-token budget (worker.py:105-106)
    sim.now = 10_000
    t0 = time.perf_counter()
    pol.fill()
    dt = time.perf_counter() - t0
    assert len(w.queue) == nq
    return {"nq": nq, "seconds": dt, "decisions_per_s": nq / dt}


def time_dispatch(n=16384, D=1, clients=200, seed=3):
    from fairsched.global_policies import make_dispatcher
    from fairsched.requests import Request
    from paper_2501_14312_b200.workloads import build_docs, config3, shared_prefix_queue
    spec = config3(n, seed=seed)
    spec.clients = clients
    q = shared_prefix_queue(spec, docs=build_docs(spec))
    reqs = _requests(q, Request)
    M, L_input = 65536, 4096
    U = L_input + 2 * M
    from fairsched.accounting import CostWeights
    disp = make_dispatcher("d2lpm", list(range(D)), CostWeights(1, 2), max(1, round(0.5 * U)), 0.5)
    t0 = time.perf_counter()
    for r in reqs:
        disp.dispatch(r, 0)
    dt = time.perf_counter() - t0
    return {"arrivals": n, "D": D, "seconds": dt, "decisions_per_s": n / dt}


def _exponent(rows):
    xs = [math.log(r["nq"]) for r in rows]
    ys = [math.log(r["seconds"]) for r in rows]
    if len(xs) < 2:
        return None
    mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
    return sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)


def run(normal_sizes=(4096, 16384, 65536), steady_sizes=(4096, 16384), indebted_sizes=(1024, 2048, 4096),
        dispatch_D=(1, 8), dispatch_n=16384):
    impl = import_reference()
    t0 = time.perf_counter()
    normal, steady = [], []
    for n in normal_sizes:
        f, st = time_fill_normal(n, steady=n in steady_sizes)
        normal.append(f)
        if st is not None:
            steady.append(st)
    indebted = [time_fill_indebted(n) for n in indebted_sizes]
    disp = [time_dispatch(dispatch_n, D) for D in dispatch_D]
    return {
        "what": "reference fairsched (baseline/_ref, unmodified) Dlpm.fill on a real Worker/RadixTree and "
                "D2lpm.dispatch, time.perf_counter, one core (single-threaded event loop under the GIL)",
        "kernel_impl": impl, "cores": 1, **host_info(),
        "workload": "config-2 generator: 100 clients, 1-4k-token prompts, Zipf(1.1) over 256 docs, "
                    "M=capacity=65536, reserve 8, q_u_frac 0.5 (dispatch: config-3 generator, 200 clients)",
        "dlpm_fill_first": normal, "first_fill_exponent": _exponent(normal),
        "dlpm_fill_steady": steady, "steady_fill_exponent": _exponent(steady),
        "dlpm_fill_indebted": indebted, "indebted_exponent": _exponent(indebted),
        "d2lpm_dispatch": disp, "wall_s": time.perf_counter() - t0,
    }


if __name__ == "__main__":
    import json
    sys.path.insert(0, ROOT)
    print(json.dumps(run()))
