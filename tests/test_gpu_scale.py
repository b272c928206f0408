"""Scale parity: the CUDA path against the CPU oracle on the bench's serving
loops (config 2: Zipf shared-prefix queue, 100 clients; config 5: deep prefix
tree of 8k-token prompts, 200 clients) at sizes the golden traces do not
reach -- every step's admissions, admission-time match lengths, deficit
counters, refill counts, eviction records and tree usage must be identical."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_wl(wl, steps, q_all=None, k1_full_steps=()):
    """Lockstep of the bench's serving loop (bench.GpuSteps, through the C ABI)
    and the oracle (oracle.lockstep.OracleSteps).  q_all: the whole stream
    (queue then arrival pool) as one host Queue (default: the workload's CPU
    sample, which must be the whole queue).  k1_full_steps: steps whose fill
    re-matches every request from the root (FS_OPT_K1_FULL) instead of
    resuming from the previous matches -- both modes must equal the oracle."""
    import bench
    from oracle.lockstep import OracleSteps

    if q_all is None:
        q, pool, n = wl.cpu_sample(0)
        assert n == wl.nq
        q_all = bench._concat_once(None, q, pool)
    nq = wl.nq
    pool_n = len(q_all) - nq
    g = bench.GpuSteps(wl, 0)
    o = OracleSteps(q_all, wl.CAP, wl.M, wl.reserve, bench.W_E, bench.W_Q,
                    wl.quantum(), max(128, wl.clients), out_tokens=wl.out_tokens)
    o.enqueue(range(nq))
    nc = max(128, wl.clients)
    nxt = 0
    total_adm = 0
    for k in range(steps):
        now = (k + 1) * bench.STEP_US
        g.w.set_k1_full(k in k1_full_steps)
        rg = g.step(now)
        ro = o.step(now)
        assert rg.n_queued == ro["n"], f"step {k}: queue sizes differ"
        assert [int(x) for x in rg.adm_req] == ro["admitted"], f"step {k}: admissions differ"
        assert [int(x) for x in rg.adm_mlen] == ro["mlen"], f"step {k}: match lengths differ"
        qg, rfg, _ = g.w.counters(nc)
        assert (qg == ro["q"][:nc]).all(), f"step {k}: deficit counters differ"
        assert (rfg == ro["refills"][:nc]).all(), f"step {k}: refill counts differ"
        assert (rg.used, rg.pinned) == (ro["used"], ro["pinned"]), f"step {k}: used/pinned differ"
        recs_g = [(tuple(g.ctx.arena_read(int(s), int(n))), int(kp))
                  for s, n, kp in zip(rg.records.src, rg.records.length, rg.records.keep)]
        recs_o = [(tuple(int(x) for x in p), int(kp)) for p, kp in ro["records"]]
        assert recs_g == recs_o, f"step {k}: eviction records differ"
        n = len(ro["admitted"])
        if n and nxt + n <= pool_n:
            o.enqueue(range(nq + nxt, nq + nxt + n))
            nxt += n
        total_adm += n
    assert total_adm > steps  # the loop really admits and evicts
    g.close()
    return total_adm


def test_scale_8k():
    import bench
    _run_wl(bench.Config2(8192, 9, 12), 12)


def test_scale_64k():
    import bench
    _run_wl(bench.Config2(65536, 0, 6), 6)


def test_scale_config5_64k():
    """Config 5 (deep prefix tree, 8k-token prompts, device-generated sha256
    tokens) at 64k queued requests against the oracle on the same tokens."""
    import bench
    _run_wl(bench.Config5(65536, 0, 10), 10)


def _c5_host_stream(wl):
    """The whole config-5 stream -- the wl.nq-request queue, then the arrival
    pool -- expanded on the host by oracle/tokens.c (the reference's
    expand_tokens restated, pinned by tests/golden/tokens.json) into ONE
    buffer (34 GB at 1M requests; no concatenation copy).  The pool half must
    equal the device-materialized pool the GPU loop uploads."""
    from oracle.materialize import expand_segments
    from paper_2501_14312_b200.workloads import Queue, deep_tree_segments
    sq, cq, lq = deep_tree_segments(wl.spec, first=0, count=wl.nq, stream=0)
    sp, cp, lp = deep_tree_segments(wl.spec, first=0, count=wl.pool_n, stream=1)
    tq, tp = int(sq.lens().sum()), int(sp.lens().sum())
    flat = np.empty(tq + tp, np.int32)
    _, oq = expand_segments(sq, out=flat[:tq])
    _, op = expand_segments(sp, out=flat[tq:])
    pool = wl.pool
    assert len(pool) == wl.pool_n and np.array_equal(pool.clients, cp) and np.array_equal(pool.labels, lp)
    for i in range(len(pool)):
        assert np.array_equal(pool.tokens(i), flat[tq + op[i]:tq + op[i + 1]]), f"pool request {i}"
    n = wl.nq + wl.pool_n
    return Queue(flat, np.concatenate([oq[:-1], tq + op[:-1]]), np.concatenate([sq.lens(), sp.lens()]).astype(np.int32),
                 np.concatenate([cq, cp]).astype(np.int32),
                 np.concatenate([np.zeros(wl.nq, np.int64), np.full(wl.pool_n, bench_step_us(), np.int64)]),
                 [], np.concatenate([lq, lp]))


def bench_step_us():
    import bench
    return bench.STEP_US


@pytest.mark.slow
def test_scale_config5_full_1m():
    """Config 5 at the benchmarked size: the full 1,048,576-request queue of
    8192-token prompts (8.6 G tokens in the arena: offsets past 2^31, the
    full-size position shadow, grid sweeps and chunked LRU at full size)
    against the oracle on host-expanded tokens, five serving steps; steps 2
    and 4 re-match every request from the root, the others resume from the
    previous matches (incremental K1), so both modes are checked at 1M."""
    import bench
    wl = bench.Config5(1 << 20, 0, 5)
    q_all = _c5_host_stream(wl)
    assert int(q_all.offsets[wl.nq - 1]) > (1 << 31)
    _run_wl(wl, 5, q_all=q_all, k1_full_steps=(2, 4))


def test_scale_leader_only_sweeps(monkeypatch):
    """The same parity with the grid sweep disabled (the leader CTA scans the
    queue alone): both search paths must make identical decisions."""
    import bench
    monkeypatch.setenv("FS_SCHED_HELPERS", "0")
    _run_wl(bench.Config2(8192, 9, 12), 12)
    _run_wl(bench.Config5(16384, 0, 6), 6)


def test_incremental_match_equals_full_rematch():
    """The incremental K1 (resume from each request's previous match) makes the
    same decisions as re-matching every request from the root (FS_OPT_K1_FULL),
    including when per-call tree edits between fills invalidate the hints
    (structural version bump): two workers in lockstep on identical inputs."""
    import numpy as np
    import bench
    wl = bench.Config5(16384, 0, 10)
    a = bench.GpuSteps(wl, 0)
    b = bench.GpuSteps(wl, 0)
    b.w.set_k1_full(True)
    for k in range(10):
        now = (k + 1) * bench.STEP_US
        if k in (4, 7):
            # an out-of-fill structural edit on both trees (RadixTree.evict_lru)
            ra = a.trie.evict_lru(4096)
            rb = b.trie.evict_lru(4096)
            assert list(ra.src) == list(rb.src) and list(ra.keep) == list(rb.keep)
        x, y = a.step(now), b.step(now)
        assert list(x.adm_req) == list(y.adm_req), f"step {k}"
        assert list(x.adm_mlen) == list(y.adm_mlen), f"step {k}"
        assert list(x.records.src) == list(y.records.src) and list(x.records.keep) == list(y.records.keep)
        qa, _, _ = a.w.counters(256)
        qb, _, _ = b.w.counters(256)
        assert np.array_equal(qa, qb)
        assert (x.used, x.pinned) == (y.used, y.pinned)
    assert a.w is not b.w
    a.close()
    b.close()


def test_grid_sort_path_matches_oracle():
    """The incremental order with a large B: k_sort_b's grid-wide radix path
    and k_merge_a's unstaged search over B.  FS_SB_CAP=64 (read once per
    process, hence the subprocess) sends every B past 64 entries down them."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path[:0] = ['tests', '.']\n"
            "import bench, test_gpu_scale as t\n"
            "t._run_wl(bench.Config2(8192, 9, 12), 12)\n"
            "t._run_wl(bench.Config5(16384, 0, 6), 6)\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, FS_SB_CAP="64"),
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
