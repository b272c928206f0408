"""Host side of the GPU service-gap verifiers (paper_2501_14312_b200.verify):
the vectorised backlogged intervals and window grid must be the reference's
(metrics.py:91-115) exactly -- the kernels evaluate these windows."""
import pytest

from refpath import import_fairsched
from verify_cases import random_case


@pytest.fixture(scope="module")
def fs():
    mod = import_fairsched()
    if mod is None:
        pytest.skip("reference package not available")
    return mod


@pytest.mark.parametrize("seed", range(12))
def test_backlogs_and_windows_match_reference(fs, seed):
    from fairsched import metrics
    from paper_2501_14312_b200.verify import ServiceView

    svc, life, run_end = random_case(fs, seed, n_clients=1 + seed % 7, n_req=10 + 17 * seed)
    v = ServiceView(svc, life, run_end)
    assert v.clients == metrics._clients_of(life)
    wins = []
    for i, c in enumerate(v.clients):
        ref = metrics.backlogged_intervals(life, c, run_end)
        assert v.intervals(i) == ref
        for lo, hi in ref:
            wins += [(i, t1, t2) for t1, t2 in metrics.window_grid(lo, hi)]
    wf, w1, w2 = v.grid_windows()
    assert list(zip(wf.tolist(), w1.tolist(), w2.tolist())) == wins
    # service prefix sums reproduce service_in_interval on the windows
    for f, t1, t2 in wins[:200]:
        a = v.ev_off[f]
        tm = v.ev_time[a:v.ev_off[f + 1]]
        cum = v.ev_cum[a + f:v.ev_off[f + 1] + f + 1]
        import numpy as np
        got = int(cum[np.searchsorted(tm, t2, "left")] - cum[np.searchsorted(tm, t1, "left")])
        assert got == svc.service_in_interval(v.clients[f], t1, t2)
