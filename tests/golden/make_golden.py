"""Generate golden fixtures from the REAL reference (run in the build container only).

    python tests/golden/make_golden.py

Imports `fairsched` from /root/reference/pkg/src (read-only source, Cython kernel
optional) and records, for seeded inputs:

* radix_traces.json -- random op sequences on RadixTree (local with capacity,
  global with worker tags) with every result, eviction record and dump.
* serving_traces.json -- full `run_experiment` runs with spies at the hot-path
  boundary (Worker.enqueue, policy.fill/on_outputs, RadixTree.unpin/evict_lru,
  Dispatcher.dispatch/on_finish/on_eviction) so that tests can replay exactly
  the same interaction against the oracle and the CUDA path.  Each run also
  stores the reference event-log sha256 for plugin-level parity.

The fixtures are committed; /root/reference does not exist on the GPU box.
"""
from __future__ import annotations

import gzip
import hashlib
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"


def _import_reference():
    sys.path.insert(0, REF_SRC)
    import fairsched  # noqa: F401
    return fairsched


def canon_dump(dump) -> list:
    return [[list(p), r, list(w), la] for p, r, w, la in dump]


def dump_digest(dump) -> str:
    return hashlib.sha256(json.dumps(canon_dump(dump), separators=(",", ":")).encode()).hexdigest()


# ---------------------------------------------------------------------------
# radix op traces
# ---------------------------------------------------------------------------


def radix_traces(n_local=40, n_global=40, steps=80):
    from fairsched.radix import CacheFull, RadixTree

    out = []
    for trial in range(n_local):
        rng = random.Random(7000 + trial)
        cap = rng.randrange(6, 40)
        t = RadixTree(capacity=cap)
        sink = []
        t.on_evict = lambda path, keep, ev: sink.append([list(path), keep])
        ops = []
        pins = []  # admit handles in order
        alive = []
        for step in range(steps):
            sink.clear()
            now = step + 1 + rng.randrange(3)
            ln = rng.randrange(1, 14)
            alpha = rng.choice([2, 3, 5])
            toks = [rng.randrange(alpha) for _ in range(ln)]
            u = rng.random()
            rec = {"now": now, "tokens": toks}
            if u < 0.3:
                rec["op"] = "insert"
                try:
                    nl, _path = t.insert(tuple(toks), now=now)
                    rec["new_len"] = nl
                except CacheFull:
                    rec["cache_full"] = True
            elif u < 0.45:
                rec["op"] = "match"
                rec["update"] = rng.random() < 0.8
                rec["mlen"] = t.match_prefix(tuple(toks), now=now, update_access=rec["update"])[0]
            elif u < 0.55:
                rec["op"] = "probe"
                rec["mlen"], rec["unpinned"] = t.probe(tuple(toks))
            elif u < 0.75 and len(alive) < 4:
                rec["op"] = "admit"
                try:
                    m, path = t.admit(tuple(toks), now=now)
                    rec["mlen"] = m
                    rec["pin_id"] = len(pins)
                    pins.append(path)
                    alive.append(len(pins) - 1)
                except CacheFull:
                    rec["cache_full"] = True
            elif u < 0.88 and alive:
                rec["op"] = "unpin"
                pid = alive.pop(rng.randrange(len(alive)))
                rec["pin_id"] = pid
                t.unpin(pins[pid])
            else:
                rec["op"] = "evict"
                rec["needed"] = rng.randrange(1, cap + 1)
                recs = t.evict_lru(rec["needed"])
                rec["records"] = [[list(p), k] for p, k in recs]
            if rec["op"] in ("insert", "admit"):
                # evictions inside insert are observable through on_evict (radix.py:247-249)
                rec["records"] = [list(x) for x in sink]
            rec["used"] = t.used_tokens
            rec["pinned"] = t.pinned_tokens
            rec["dump"] = canon_dump(t.dump())
            t.check()
            ops.append(rec)
        out.append({"kind": "local", "capacity": cap, "ops": ops})

    for trial in range(n_global):
        rng = random.Random(9000 + trial)
        D = rng.choice([2, 3, 4, 8])
        t = RadixTree(track_workers=True)
        ops = []
        inserted = []
        for step in range(steps):
            now = step * 2 + 1
            u = rng.random()
            if u < 0.45 or not inserted:
                base = list(rng.choice(inserted)) if inserted and rng.random() < 0.6 else []
                cut = rng.randrange(len(base) + 1) if base else 0
                toks = base[:cut] + [rng.randrange(3) for _ in range(rng.randrange(1, 8))]
                w = rng.randrange(D)
                nl, _ = t.insert(tuple(toks), now=now, worker=w)
                inserted.append(toks)
                rec = {"op": "insert", "tokens": toks, "now": now, "worker": w, "new_len": nl}
            elif u < 0.7:
                base = list(rng.choice(inserted))
                toks = base[: rng.randrange(len(base) + 1)] + [rng.randrange(3) for _ in range(rng.randrange(0, 4))]
                m, ws = t.longest_match_workers(tuple(toks), now=now)
                rec = {"op": "lmw", "tokens": toks, "now": now, "mlen": m, "workers": sorted(ws)}
            else:
                base = list(rng.choice(inserted))
                if rng.random() < 0.2:
                    base = base + [rng.randrange(3)]
                keep = rng.randrange(len(base) + 1)
                w = rng.randrange(D)
                nt = now - rng.randrange(0, 20)
                t.evict_notify(tuple(base), w, keep, nt)
                rec = {"op": "notify", "tokens": base, "worker": w, "keep_len": keep, "notice_time": nt, "now": now}
            rec["used"] = t.used_tokens
            rec["dump"] = canon_dump(t.dump())
            t.check()
            ops.append(rec)
        out.append({"kind": "global", "n_workers": D, "ops": ops})
    return out


# ---------------------------------------------------------------------------
# serving traces (full runs with boundary spies)
# ---------------------------------------------------------------------------


def _random_config(i):
    from fairsched.requests import SystemParams
    from fairsched.runner import ExperimentConfig, SchedulingConfig
    from fairsched.workload import ClientProfile

    rng = random.Random(31000 + i)
    D = [1, 1, 2, 4, 8][i % 5]
    L_input = rng.choice([64, 96, 160])
    M = rng.choice([L_input * 3, L_input * 4, L_input * 6])
    params = SystemParams(L_input=L_input, L_output=24, M=M, D=D)
    n_clients = rng.randrange(2, 8)
    clients = []
    for c in range(n_clients):
        tree = rng.random() < 0.3
        suffix = rng.randrange(3, 10)
        depth = 1 if tree else 0
        prefix = rng.randrange(8, max(9, L_input - (depth + 1) * suffix - 20))
        clients.append(
            ClientProfile(
                name=f"cl{c}",
                rate=rng.uniform(10, 45) * max(1, D / 2),
                cv=rng.uniform(0.5, 2.0),
                program="tree" if tree else "flat",
                branches=2,
                depth=depth,
                prefix_len=prefix,
                suffix_len=suffix,
                output_len=rng.randrange(2, 9),
                output_dist=rng.choice(["constant", "lognormal"]),
                prefix_scope=rng.choice(["client", "client", "program"]),
            )
        )
    if n_clients >= 2:
        clients[0].misbehavior = "S1"
    local = rng.choice(["dlpm", "dlpm", "dlpm", "lpm"])
    glob = "d2lpm" if D > 1 and rng.random() < 0.8 else "rr"
    reserve = rng.choice([0, 4, max(p.output_len for p in clients)])
    deepest = max(p.prefix_len + (p.depth + 1) * p.suffix_len for p in clients)
    cap = None
    if rng.random() < 0.4:
        cap = rng.randrange(deepest, M + 1)
    sched = SchedulingConfig(
        local_policy=local,
        global_policy=glob,
        q_u_frac=rng.choice([0.02, 0.1, 0.5, 2.0]),
        q_w_frac=rng.choice([0.02, 0.1, 0.5, 2.0]),
        chunk_size=rng.choice([8192, 8192, 32]),
        admission_interval=rng.choice([1, 1, 2]),
        output_reserve=reserve,
        cache_capacity=cap,
        eviction_notice_delay_ms=rng.choice([0.0, 0.0, 3.0]),
    )
    if L_input + reserve > M:
        sched.output_reserve = 0
    return ExperimentConfig(seed=41000 + i, horizon_ms=rng.choice([150, 250]), latency_window_ms=50,
                            params=params, scheduling=sched, clients=clients)


def record_run(cfg, trace=None):
    """Run the reference with spies; returns the op trace dict."""
    import fairsched.global_policies as GP
    import fairsched.local_policies as LP
    import fairsched.radix as RX
    import fairsched.worker as W
    from fairsched.runner import config_to_dict, run_experiment
    from fairsched.requests import Trace

    ops = []
    sink = {"recs": None}
    path_owner = {}

    saved = {}

    def patch(obj, name, fn):
        saved[(obj, name)] = getattr(obj, name)
        setattr(obj, name, fn)

    orig_enqueue = W.Worker.enqueue

    def enqueue(self, req):
        ops.append({"op": "enq", "w": self.wid, "rid": req.rid})
        return orig_enqueue(self, req)

    orig_evict = RX.RadixTree.evict_lru

    def evict_lru(self, needed, protect=None):
        recs = orig_evict(self, needed, protect)
        if sink["recs"] is not None and not self.track_workers:
            sink["recs"].extend(recs)
        return recs

    orig_unpin = RX.RadixTree.unpin

    def unpin(self, path):
        key = id(path)
        if key in path_owner:
            w, rid = path_owner.pop(key)
            ops.append({"op": "fin", "w": w, "rid": rid})
        return orig_unpin(self, path)

    def wrap_fill(cls):
        orig_fill = cls.fill

        def fill(self):
            w = self.worker
            rec = {
                "op": "fill",
                "w": w.wid,
                "now": w.sim.now,
                "generated_total": w.generated_total,
                "headroom": w._reserved_headroom(),
                "queue": [r.rid for r in w.queue],
                "batch": sorted(w.batch),
            }
            adm = []
            real = w.try_admit

            def spy(req):
                entry = real(req)
                if entry is not None:
                    adm.append([req.rid, entry.match_len, entry.extend_total])
                    path_owner[id(entry.path)] = (w.wid, req.rid)
                return entry

            w.try_admit = spy
            sink["recs"] = []
            try:
                orig_fill(self)
            finally:
                del w.try_admit
            recs = sink["recs"]
            sink["recs"] = None
            rec["admissions"] = adm
            rec["records"] = [[list(p), k] for p, k in recs]
            c = self.counters()
            rec["q"] = dict(c) if c else {}
            rec["refills"] = dict(getattr(self, "refill_counts", {}))
            rec["used"] = w.tree.used_tokens
            rec["pinned"] = w.tree.pinned_tokens
            rec["dump_sha"] = dump_digest(w.tree.dump())
            ops.append(rec)

        patch(cls, "fill", fill)

    def wrap_outputs(cls):
        orig = cls.on_outputs

        def on_outputs(self, counts):
            ops.append({"op": "out", "w": self.worker.wid, "counts": dict(counts)})
            return orig(self, counts)

        patch(cls, "on_outputs", on_outputs)

    orig_dispatch = GP.Dispatcher.dispatch

    def dispatch(self, req, now):
        d = orig_dispatch(self, req, now)
        if isinstance(self, GP.D2lpm):
            ops.append({"op": "disp", "rid": req.rid, "now": now, "worker": d.worker,
                        "mlen": d.match_len, "matched": list(d.matched_workers),
                        "qrow": {str(w): self.q.get((req.client, w)) for w in self.worker_ids
                                 if (req.client, w) in self.q}})
        return d

    orig_dfin = GP.D2lpm.on_finish

    def d_on_finish(self, client, worker, output_tokens, now):
        ops.append({"op": "dfin", "client": client, "worker": worker, "out": output_tokens, "now": now})
        return orig_dfin(self, client, worker, output_tokens, now)

    orig_dev = GP.D2lpm.on_eviction

    def d_on_eviction(self, path, keep_len, worker, notice_time, now):
        ops.append({"op": "dev", "path": list(path), "keep_len": keep_len, "worker": worker,
                    "notice_time": notice_time, "now": now})
        return orig_dev(self, path, keep_len, worker, notice_time, now)

    patch(W.Worker, "enqueue", enqueue)
    patch(RX.RadixTree, "evict_lru", evict_lru)
    patch(RX.RadixTree, "unpin", unpin)
    wrap_fill(LP.Dlpm)
    wrap_fill(LP.Lpm)
    wrap_outputs(LP.Dlpm)
    wrap_outputs(LP.LocalPolicy)
    patch(GP.Dispatcher, "dispatch", dispatch)
    patch(GP.D2lpm, "on_finish", d_on_finish)
    patch(GP.D2lpm, "on_eviction", d_on_eviction)
    try:
        result = run_experiment(cfg, trace)
    finally:
        for (obj, name), fn in saved.items():
            setattr(obj, name, fn)

    trace_obj = result.trace
    requests, _ = trace_obj.materialize()
    tok = {r.rid: r.input_tokens for r in requests}
    # Express every token path as (rid, length) so fixtures stay small.
    by_first = {}
    for r in requests:
        by_first.setdefault(r.input_tokens[:1], []).append(r)

    def path_ref(path):
        path = tuple(path)
        for r in by_first.get(path[:1], ()):
            if r.input_tokens[: len(path)] == path:
                return [r.rid, len(path)]
        raise AssertionError("path is not a request prefix")

    for op in ops:
        if op["op"] == "fill":
            op["records"] = [path_ref(p) + [k] for p, k in op["records"]]
        elif op["op"] == "dev":
            op["path"] = path_ref(op["path"])
    h = hashlib.sha256()
    for rid in sorted(tok):
        h.update(rid.encode())
        h.update(b"".join(int(x).to_bytes(4, "little") for x in tok[rid]))
    disp_q = None
    if isinstance(result.dispatcher, GP.D2lpm):
        disp_q = [[c, w, v] for (c, w), v in sorted(result.dispatcher.q.items())]
    gdump = None
    if getattr(result.dispatcher, "tree", None) is not None:
        gdump = dump_digest(result.dispatcher.tree.dump())
    return {
        "config": json.loads(json.dumps(config_to_dict(cfg))),
        "trace": [json.loads(r.to_json()) for r in trace_obj.records],
        "requests": {r.rid: {"client": r.client, "arrival": r.arrival} for r in requests},
        "tokens_sha": h.hexdigest(),
        "event_sha256": result.log.sha256(),
        "ops": ops,
        "final_dispatch_q": disp_q,
        "global_dump_sha": gdump,
        "worker_dump_sha": [dump_digest(w.tree.dump()) for w in result.workers],
        "violations": {k: len(v) for k, v in result.violations.items()},
        "extremes": {k: list(v) for k, v in result.counter_extremes.items()},
        "n_requests": len(requests),
    }


def serving_traces(n_random=60):
    from fairsched.runner import load_config

    out = []
    for name in ("example.yaml", "d2lpm_4workers.yaml"):
        cfg = load_config(os.path.join("/root/reference/pkg/configs", name))
        rec = record_run(cfg)
        rec["name"] = name
        out.append(rec)
    for i in range(n_random):
        cfg = _random_config(i)
        try:
            cfg.validate()
        except Exception:
            continue
        rec = record_run(cfg)
        rec["name"] = f"random-{i}"
        out.append(rec)
    return out


def main():
    _import_reference()
    from fairsched.speedups import KERNEL_IMPL

    rt = radix_traces()
    with gzip.open(os.path.join(HERE, "radix_traces.json.gz"), "wt") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "kernel_impl": KERNEL_IMPL, "traces": rt}, fh,
                  separators=(",", ":"))
    st = serving_traces()
    with gzip.open(os.path.join(HERE, "serving_traces.json.gz"), "wt") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "kernel_impl": KERNEL_IMPL, "runs": st}, fh,
                  separators=(",", ":"))
    n_ops = sum(len(r["ops"]) for r in st)
    print(f"radix traces: {len(rt)}; serving runs: {len(st)} ({n_ops} boundary ops)")


if __name__ == "__main__":
    main()
