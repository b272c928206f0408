"""Scale parity: the CUDA path against the CPU oracle on the config-2 serving
loop (Zipf shared-prefix queue, 100 clients) at sizes the golden traces do not
reach -- every step's admissions, admission-time match lengths, deficit
counters, refill counts, eviction records and tree usage must be identical."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(nq, steps, seed):
    import bench
    from oracle.lockstep import OracleSteps
    from paper_2501_14312_b200.workloads import build_docs, config2, shared_prefix_queue

    spec = config2(nq, seed=seed)
    docs = build_docs(spec)
    q = shared_prefix_queue(spec, docs=docs)
    pool = shared_prefix_queue(spec, first=nq, count=96 * steps + 64, arrival=bench.STEP_US, docs=docs,
                               stream_seed=seed + 101)
    g = bench.GpuSteps(q, pool, 0)
    o = OracleSteps(bench._concat_once(None, q, pool), bench.M, bench.M, bench.RESERVE, bench.W_E, bench.W_Q,
                    bench.Q_U, 128)
    o.enqueue(range(nq))
    nxt = 0
    total_adm = 0
    for k in range(steps):
        now = (k + 1) * bench.STEP_US
        rg = g.step(now)
        ro = o.step(now)
        assert [int(x) for x in rg.adm_req] == ro["admitted"], f"step {k}: admissions differ"
        assert [int(x) for x in rg.adm_mlen] == ro["mlen"], f"step {k}: match lengths differ"
        qg, rfg, _ = g.w.counters(128)
        assert (qg == ro["q"][:128]).all(), f"step {k}: deficit counters differ"
        assert (rfg == ro["refills"][:128]).all(), f"step {k}: refill counts differ"
        assert (rg.used, rg.pinned) == (ro["used"], ro["pinned"]), f"step {k}: used/pinned differ"
        recs_g = [(tuple(g.ctx.arena_read(int(s), int(n))), int(kp))
                  for s, n, kp in zip(rg.records.src, rg.records.length, rg.records.keep)]
        recs_o = [(tuple(int(x) for x in p), int(kp)) for p, kp in ro["records"]]
        assert recs_g == recs_o, f"step {k}: eviction records differ"
        n = len(ro["admitted"])
        if n and nxt + n <= len(pool):
            o.enqueue(range(nq + nxt, nq + nxt + n))
            nxt += n
        total_adm += n
    assert total_adm > steps  # the loop really admits and evicts
    g.ctx.close()
    return total_adm


def test_scale_8k():
    _run(8192, 12, 11)


def test_scale_64k():
    _run(65536, 6, 2)
