"""Randomized lockstep stress of the CUDA serving loop against the CPU oracle at
small sizes where every corner is hit often: tiny alphabets (heavy sharing,
deep splits), capacity below M, requests of length 1, duplicate requests,
LPM and DLPM, tiny and large quanta (refill rounds), reserves, single-request
queues and empty fills.  Every step must agree on admissions, admission-time
match lengths, eviction records, deficit counters, refill counts and
used/pinned tokens -- exercising the incremental K1 hints, the grid sweeps
and the lazy LRU index under churn."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

W_E, W_Q = 1, 2


def _requests(rng, n, alphabet, lmax, first_id):
    base = [rng.randrange(alphabet) for _ in range(lmax)]
    toks, cls = [], []
    for i in range(n):
        kind = rng.random()
        if kind < 0.1:
            t = [rng.randrange(alphabet)]                            # length 1
        elif kind < 0.2 and toks:
            t = list(toks[rng.randrange(len(toks))])                 # duplicate
        elif kind < 0.7:
            k = rng.randrange(1, lmax)                               # shared prefix + tail
            t = base[:k] + [rng.randrange(alphabet) for _ in range(rng.randrange(1, lmax // 2 + 1))]
        else:
            t = [rng.randrange(alphabet) for _ in range(rng.randrange(1, lmax + 1))]
        toks.append(t[:lmax])
        cls.append(rng.randrange(6))
    return toks, cls


def _run(seed):
    from oracle.oracle import OracleWorker
    from paper_2501_14312_b200.device import Context, Trie, WorkerDev

    rng = random.Random(seed)
    alphabet = rng.choice([2, 3, 5, 50])
    lmax = rng.choice([8, 24, 64])
    M = rng.choice([lmax * 3, lmax * 5, lmax * 9])
    cap = rng.choice([M, M, max(lmax + 1, M // 2)])
    R = rng.choice([0, 1, 4])
    policy = rng.choice(["dlpm", "dlpm", "lpm"])
    U = W_E * lmax + W_Q * M
    Q = max(1, round(rng.choice([0.02, 0.1, 0.5, 2.0]) * U))
    n0 = rng.choice([1, 5, 60, 400])
    steps = 30
    toks, cls = _requests(rng, n0 + 60 * steps, alphabet, lmax, 0)

    ctx = Context(0, arena_tokens=1 << 20, max_requests=1 << 14)
    flat = np.concatenate([np.asarray(t, np.int32) for t in toks])
    lens = np.array([len(t) for t in toks], np.int32)
    offs = np.zeros(len(toks), np.int64)
    offs[1:] = np.cumsum(lens[:-1])
    clients = np.array(cls, np.int32)
    labels = np.arange(len(toks), dtype=np.int64)
    trie = Trie(ctx, cap)
    w = WorkerDev(ctx, trie, policy, Q, M, R, W_E, W_Q, max_clients=8)
    o = OracleWorker(cap, M, R, W_E, W_Q, policy, Q, 8)
    ids = np.zeros(0, np.int32)
    pending = []
    nxt = 0
    prev = []  # (node handle gpu, handle oracle, client)
    for k in range(steps):
        now = (k + 1) * 1000
        # completion of the previous batch (a random subset finishes)
        done = [x for x in prev if rng.random() < 0.7]
        prev = [x for x in prev if x not in done]
        if done:
            cl, cnt = np.unique(np.array([c for _, _, c in done], np.int32), return_counts=True)
            w.outputs(cl, (cnt * 3).astype(np.int64))
            trie.unpin_many(np.array([g for g, _, _ in done], np.int32))
            for _, h, c in done:
                o.on_outputs(c, 3)
                o.unpin(h)
        # arrivals (none at some steps; the whole initial burst at step 0)
        na = n0 if k == 0 else rng.choice([0, 1, 7, 60])
        if na:
            a, b = nxt, min(len(toks), nxt + na)
            o0 = int(offs[a])
            new = ctx.add_requests(flat[o0:int(offs[b - 1] + lens[b - 1])], offs[a:b] - o0, lens[a:b],
                                   clients[a:b], labels[a:b])
            ids = np.concatenate([ids, new])
            w.enqueue(new)
            for i in range(a, b):
                o.on_enqueue(int(clients[i]))
                pending.append(i)
            nxt = b
        rg = w.fill(now, 0, 0)
        idx = np.asarray(pending, np.int64)
        ro = o.fill(flat, offs[idx], lens[idx], clients[idx], labels[idx], now, 0, 0)
        adm_o = [int(idx[p]) for p in ro["pos"]]
        assert [int(x) for x in rg.adm_req] == [int(ids[i]) for i in adm_o], f"seed {seed} step {k}"
        assert [int(x) for x in rg.adm_mlen] == [int(x) for x in ro["mlen"]], f"seed {seed} step {k}"
        rec_g = [(tuple(ctx.arena_read(int(s), int(n))), int(kp))
                 for s, n, kp in zip(rg.records.src, rg.records.length, rg.records.keep)]
        rec_o = [(tuple(int(x) for x in p), int(kp)) for p, kp in ro["records"]]
        assert rec_g == rec_o, f"seed {seed} step {k}"
        if policy == "dlpm":  # Lpm keeps no counters (local_policies.py:42-71)
            qg, rfg, _ = w.counters(8)
            assert (qg == o.q()[:8]).all() and (rfg == o.refills()[:8]).all(), f"seed {seed} step {k}"
        assert (rg.used, rg.pinned) == (o.tree.used_tokens, o.tree.pinned_tokens), f"seed {seed} step {k}"
        gone = set(adm_o)
        pending = [i for i in pending if i not in gone]
        prev += [(int(g), int(h), int(clients[i])) for g, h, i in zip(rg.adm_node, ro["handles"], adm_o)]
    w.close()
    trie.close()
    ctx.close()


@pytest.mark.parametrize("seed", range(96))
def test_random_lockstep(seed):
    _run(seed)
