"""Replay harness for the golden op traces (test infrastructure).

A serving trace (tests/golden/serving_traces.json) is the exact sequence of
calls the reference's unchanged caller (Simulator + Worker + runner) made into
the hot path during one `run_experiment`:

  enq  -- Worker.enqueue -> policy.on_request_enqueued        (worker.py:142-148)
  fill -- policy.fill with the worker state it observed         (local_policies.py:108-128)
  out  -- policy.on_outputs(counts)                             (worker.py:208)
  fin  -- tree.unpin(entry.path) at request finish              (worker.py:213)
  disp -- Dispatcher.dispatch (D2LPM)                           (global_policies.py:40-46)
  dfin -- D2lpm.on_finish                                       (global_policies.py:126-129)
  dev  -- D2lpm.on_eviction (EVICTION_NOTICE)                   (global_policies.py:131-132)

`replay_serving(run, backend)` drives any backend (the C oracle, or the CUDA
library through its C-ABI) through the same calls and asserts every recorded
result: ordered admissions with admission-time match length and extend, the
eviction records, per-client deficit counters and refill counts, tree usage,
the tree dump digest, and every D2LPM decision and counter row.
"""
from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import trace as otrace  # noqa: E402


def load_golden(name: str) -> dict:
    for cand in (name + ".gz", name):
        p = os.path.join(GOLDEN, cand)
        if os.path.exists(p):
            opener = gzip.open if p.endswith(".gz") else open
            with opener(p, "rt") as fh:
                return json.load(fh)
    raise FileNotFoundError(name)


def canon_dump(dump) -> list:
    return [[list(p), r, list(w), la] for p, r, w, la in dump]


def dump_digest(dump) -> str:
    return hashlib.sha256(json.dumps(canon_dump(dump), separators=(",", ":")).encode()).hexdigest()


class RunTable:
    """Materialized requests of one run: tokens, dense client ids, (arrival, rid) labels."""

    def __init__(self, run: dict):
        self.inputs = otrace.materialize(run["trace"])
        assert otrace.tokens_digest(self.inputs) == run["tokens_sha"], "token materializer drifted"
        reqs = run["requests"]
        self.rids = sorted(reqs)
        self.clients = sorted({reqs[r]["client"] for r in self.rids})
        self.client_id = {c: i for i, c in enumerate(self.clients)}
        order = sorted(self.rids, key=lambda r: (reqs[r]["arrival"], r))  # lpm_order tie-break
        self.label = {r: i for i, r in enumerate(order)}
        self.client_of = {r: self.client_id[reqs[r]["client"]] for r in self.rids}

    def tokens(self, rid) -> np.ndarray:
        return self.inputs[rid]

    def path(self, ref) -> np.ndarray:
        rid, n = ref[0], ref[1]
        return self.inputs[rid][:n]


def _cfg_ints(run):
    cfg = run["config"]
    p, s = cfg["params"], cfg["scheduling"]
    U = p["w_e"] * p["L_input"] + p["w_q"] * p["M"]
    q_u = s["q_u"] if s["q_u"] is not None else max(1, round(s["q_u_frac"] * U))
    q_w = s["q_w"] if s["q_w"] is not None else max(1, round(s["q_w_frac"] * U))
    cap = s["cache_capacity"] if s["cache_capacity"] is not None else p["M"]
    return p, s, q_u, q_w, cap


def replay_serving(run: dict, backend, check_dump: bool = True) -> dict:
    """Drive `backend` through the recorded ops; raise AssertionError on any diff.
    Returns simple counters (fills, admissions, ...) for reporting."""
    tab = RunTable(run)
    if hasattr(backend, "bind"):
        backend.bind(tab)
    p, s, q_u, q_w, cap = _cfg_ints(run)
    D = p["D"]
    nC = len(tab.clients)
    workers = [backend.make_worker(w, cap, p["M"], s["output_reserve"], p["w_e"], p["w_q"],
                                   s["local_policy"], q_u, nC) for w in range(D)]
    d2 = backend.make_d2(D, q_w, p["w_e"], p["w_q"], nC) if s["global_policy"] == "d2lpm" else None
    queues = [[] for _ in range(D)]
    handles = {}
    stats = {"fills": 0, "admissions": 0, "records": 0, "dispatches": 0}
    for k, op in enumerate(run["ops"]):
        kind = op["op"]
        if kind == "enq":
            rid = op["rid"]
            queues[op["w"]].append(rid)
            workers[op["w"]].enqueue(rid, tab)
        elif kind == "fill":
            w = op["w"]
            assert queues[w] == op["queue"], f"op {k}: queue mirror drifted"
            res = workers[w].fill(queues[w], tab, op["now"], op["generated_total"], op["headroom"])
            got = [[rid, m, e] for rid, m, e in res["admissions"]]
            assert got == op["admissions"], f"op {k} fill@{op['now']}: admissions\n got {got}\n exp {op['admissions']}"
            exp_recs = [(tuple(int(x) for x in tab.path(r[:2])), r[2]) for r in op["records"]]
            got_recs = [(tuple(int(x) for x in pth), keep) for pth, keep in res["records"]]
            assert got_recs == exp_recs, f"op {k}: eviction records differ"
            if s["local_policy"] == "dlpm":
                q = {tab.clients[c]: int(v) for c, v in res["q"].items()}
                assert q == op["q"], f"op {k}: q {q} != {op['q']}"
                rf = {tab.clients[c]: int(v) for c, v in res["refills"].items()}
                assert rf == op["refills"], f"op {k}: refills {rf} != {op['refills']}"
            assert res["used"] == op["used"] and res["pinned"] == op["pinned"], (
                f"op {k}: used/pinned {res['used']}/{res['pinned']} != {op['used']}/{op['pinned']}")
            if check_dump:
                assert dump_digest(res["dump"]()) == op["dump_sha"], f"op {k}: dump differs"
            for (rid, _, _), h in zip(res["admissions"], res["handles"]):
                queues[w].remove(rid)
                handles[(w, rid)] = h
            stats["fills"] += 1
            stats["admissions"] += len(got)
            stats["records"] += len(got_recs)
        elif kind == "out":
            for client, n in op["counts"].items():
                workers[op["w"]].on_outputs(tab.client_id[client], n)
        elif kind == "fin":
            workers[op["w"]].unpin(handles.pop((op["w"], op["rid"])))
        elif kind == "disp":
            rid = op["rid"]
            w, m, matched = d2.dispatch(tab.tokens(rid), tab.client_of[rid], op["now"], rid)
            assert (w, m, list(matched)) == (op["worker"], op["mlen"], op["matched"]), (
                f"op {k}: dispatch {rid} got {(w, m, matched)} exp {(op['worker'], op['mlen'], op['matched'])}")
            q = d2.q()
            c = tab.client_of[rid]
            row = {str(ww): q[(c, ww)] for ww in range(D) if (c, ww) in q}
            assert row == op["qrow"], f"op {k}: q row {row} != {op['qrow']}"
            stats["dispatches"] += 1
        elif kind == "dfin":
            d2.on_finish(tab.client_id[op["client"]], op["worker"], op["out"])
        elif kind == "dev":
            d2.on_eviction(tab.path(op["path"]), op["keep_len"], op["worker"], op["notice_time"], ref=op["path"])
        else:
            raise ValueError(kind)
    if d2 is not None and run["final_dispatch_q"] is not None:
        q = d2.q()
        exp = {(tab.client_id[c], w): v for c, w, v in run["final_dispatch_q"]}
        assert q == exp, "final D2LPM counters differ"
        if check_dump and run["global_dump_sha"] is not None:
            assert dump_digest(d2.dump()) == run["global_dump_sha"], "global index dump differs"
    if check_dump:
        for w in range(D):
            assert dump_digest(workers[w].dump()) == run["worker_dump_sha"][w], f"worker {w} final dump differs"
    return stats


# ---------------------------------------------------------------------------
# oracle backend
# ---------------------------------------------------------------------------


class OracleBackend:
    def __init__(self):
        from oracle import oracle as O
        self.O = O

    def make_worker(self, wid, cap, M, R, w_e, w_q, policy, quantum, n_clients):
        return _OracleWorker(self.O.OracleWorker(cap, M, R, w_e, w_q, policy, quantum, n_clients))

    def make_d2(self, D, quantum, w_e, w_q, n_clients):
        return _OracleD2(self.O.OracleD2lpm(D, quantum, w_e, w_q, n_clients))


class _OracleWorker:
    def __init__(self, ow):
        self.ow = ow
        self.seen = []  # Dlpm.client_list (local_policies.py:88-92)

    def enqueue(self, rid, tab):
        c = tab.client_of[rid]
        if c not in self.seen:
            self.seen.append(c)
        self.ow.on_enqueue(c)

    def fill(self, queue, tab, now, gen, headroom):
        toks = [tab.tokens(r) for r in queue]
        lens = np.array([len(t) for t in toks], np.int32)
        offs = np.zeros(len(toks), np.int64)
        if len(toks):
            offs[1:] = np.cumsum(lens[:-1])
        flat = np.concatenate(toks) if toks else np.zeros(1, np.int32)
        clients = np.array([tab.client_of[r] for r in queue], np.int32)
        labels = np.array([tab.label[r] for r in queue], np.int64)
        r = self.ow.fill(flat, offs, lens, clients, labels, now, gen, headroom)
        adm = [(queue[pos], int(m), int(lens[pos] - m)) for pos, m in zip(r["pos"], r["mlen"])]
        q = self.ow.q()
        rf = self.ow.refills()
        return {
            "admissions": adm,
            "handles": r["handles"],
            "records": r["records"],
            "q": {c: q[c] for c in self.seen},
            "refills": {c: rf[c] for c in self.seen},
            "used": self.ow.tree.used_tokens,
            "pinned": self.ow.tree.pinned_tokens,
            "dump": self.ow.tree.dump,
        }

    def on_outputs(self, client, n):
        self.ow.on_outputs(client, n)

    def unpin(self, h):
        self.ow.unpin(h)

    def dump(self):
        return self.ow.tree.dump()


class _OracleD2:
    def __init__(self, od):
        self.od = od

    def dispatch(self, tokens, client, now, rid=None):
        return self.od.dispatch(tokens, client, now)

    def on_finish(self, client, w, out):
        self.od.on_finish(client, w, out)

    def on_eviction(self, path, keep, w, notice_time, ref=None):
        self.od.on_eviction(path, keep, w, notice_time)

    def q(self):
        return self.od.q()

    def dump(self):
        return self.od.tree.dump()


# ---------------------------------------------------------------------------
# radix op traces
# ---------------------------------------------------------------------------


def replay_radix(trace: dict, make_tree, cache_full_exc) -> int:
    """Replay one radix op trace against a tree object exposing the RadixTree surface."""
    if trace["kind"] == "local":
        t = make_tree(capacity=trace["capacity"], track_workers=False, n_workers=0)
    else:
        t = make_tree(capacity=None, track_workers=True, n_workers=trace["n_workers"])
    pins = {}
    for k, op in enumerate(trace["ops"]):
        kind = op["op"]
        toks = tuple(op["tokens"])
        where = f"op {k} ({kind})"
        if kind == "insert":
            try:
                nl, _ = t.insert(toks, now=op["now"], worker=op.get("worker"))
                assert "cache_full" not in op and nl == op["new_len"], where
            except cache_full_exc:
                assert op.get("cache_full"), where
            if "records" in op:
                assert [[list(p), kk] for p, kk in t.last_records] == op["records"], where
        elif kind == "match":
            assert t.match_prefix(toks, now=op["now"], update_access=op["update"])[0] == op["mlen"], where
        elif kind == "probe":
            assert tuple(t.probe(toks)) == (op["mlen"], op["unpinned"]), where
        elif kind == "admit":
            try:
                m, h = t.admit(toks, now=op["now"])
                assert "cache_full" not in op and m == op["mlen"], where
                pins[op["pin_id"]] = h
            except cache_full_exc:
                assert op.get("cache_full"), where
            assert [[list(p), kk] for p, kk in t.last_records] == op["records"], where
        elif kind == "unpin":
            t.unpin(pins.pop(op["pin_id"]))
        elif kind == "evict":
            recs = t.evict_lru(op["needed"])
            assert [[list(p), kk] for p, kk in recs] == op["records"], where
        elif kind == "lmw":
            m, ws = t.longest_match_workers(toks, now=op["now"])
            assert (m, sorted(ws)) == (op["mlen"], op["workers"]), where
        elif kind == "notify":
            t.evict_notify(toks, op["worker"], op["keep_len"], op["notice_time"])
        else:
            raise ValueError(kind)
        assert t.used_tokens == op["used"], where
        if "pinned" in op:
            assert t.pinned_tokens == op["pinned"], where
        assert canon_dump(t.dump()) == op["dump"], where
    return len(trace["ops"])
