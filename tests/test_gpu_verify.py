"""GPU service-gap verifiers (csrc/fs_verify.cuh through fs_verify_pairs /
fs_verify_vs_any) against the reference's own metrics functions
(metrics.py:148-237): identical BoundReport rows -- measured value, the
window named in `detail`, applicability."""
import pytest

from refpath import import_fairsched
from verify_cases import random_case

pytestmark = pytest.mark.gpu

NAMES = ("verify_service_bound_pairwise", "verify_service_bound_vs_nonbacklogged", "verify_global_max_min")


@pytest.fixture(scope="module")
def fs():
    mod = import_fairsched()
    if mod is None:
        pytest.skip("reference package not available")
    return mod


def _row(r):
    return (r.theorem, r.measured, type(r.measured), r.bound, r.applicable, r.guaranteed, r.detail)


@pytest.mark.parametrize("seed", range(24))
def test_random_logs_match_reference(fs, seed):
    from fairsched import metrics
    from paper_2501_14312_b200 import verify

    n_clients = [1, 2, 3, 5, 8, 13][seed % 6]
    svc, life, run_end = random_case(fs, 1000 + seed, n_clients=n_clients, n_req=5 + 11 * seed,
                                     p_unadmitted=0.05 * (seed % 4))
    for name in NAMES:
        ref = getattr(metrics, name)(svc, life, 123.5, run_end, "thm-" + name, guaranteed=bool(seed % 2))
        got = getattr(verify, name)(svc, life, 123.5, run_end, "thm-" + name, guaranteed=bool(seed % 2))
        assert _row(got) == _row(ref), name


def test_verify_run_through_the_plugin(fs):
    """runner.verify_run with the drop-in installed (GPU policies and GPU
    verifiers) gives the reference's report rows on golden configurations."""
    from fairsched import metrics
    from fairsched.requests import Trace, TraceRecord
    from fairsched.runner import config_from_dict, run_experiment, verify_run
    from paper_2501_14312_b200 import plugin
    from replay import load_golden

    runs = load_golden("serving_traces.json")["runs"][:12]
    for run in runs:
        cfg = config_from_dict(run["config"])
        trace = Trace([TraceRecord(**r) for r in run["trace"]])
        plugin.install()
        try:
            result = run_experiment(cfg, trace)
            assert metrics.verify_service_bound_pairwise.__module__.endswith(".verify")
            got = [r.row() for r in verify_run(result)]
        finally:
            plugin.uninstall()
        ref = [r.row() for r in verify_run(result)]
        assert got == ref, run["name"]


def test_thousand_clients_pairwise(fs):
    """Config-4 scale (1000 clients): the GPU pairwise check against the
    reference's on a sample of client pairs' common windows."""
    from fairsched import metrics
    from paper_2501_14312_b200.verify import ServiceView

    svc, life, run_end = random_case(fs, 7, n_clients=1000, n_req=20000, horizon=200000)
    v = ServiceView(svc, life, run_end)
    gap, t1, t2, ok = v.pairs(0)
    n = len(v.clients)
    import random
    rng = random.Random(3)
    checked = 0
    for _ in range(400):
        f, g = sorted(rng.sample(range(n), 2))
        best, win = -1, None
        for lo, hi in metrics.intersect_intervals(v.intervals(f), v.intervals(g)):
            for a, b in metrics.window_grid(lo, hi):
                d = abs(svc.service_in_interval(v.clients[f], a, b) - svc.service_in_interval(v.clients[g], a, b))
                if d > best:
                    best, win = d, (a, b)
        k = f * n + g
        assert bool(ok[k]) == (win is not None)
        if win is not None:
            assert (int(gap[k]), int(t1[k]), int(t2[k])) == (best, win[0], win[1])
            checked += 1
    assert checked > 50
