"""Per-worker placement of the drop-in (plugin.install(placement="per_worker")):
worker w's cache, queue and counters live on their own context of
devices[w % len(devices)] -- one GPU per data-parallel worker on an 8-GPU box
(runner.py:272-289); the D2LPM / threshold dispatcher on its own context.
Eviction notices cross contexts by request identity.  On a one-GPU box every
context shares cuda:0, which exercises the same cross-context paths.  The
reference's unchanged runner must reproduce every multi-worker golden event
hash, including configs/d2lpm_4workers.yaml (9a140969...)."""
import pytest

from refpath import import_fairsched
from replay import load_golden

pytestmark = pytest.mark.gpu

SERVING = [r for r in load_golden("serving_traces.json")["runs"] if r["config"]["params"].get("D", 1) > 1]


@pytest.fixture(scope="module")
def fs():
    mod = import_fairsched()
    if mod is None:
        pytest.skip("reference package not available (build() installs it into baseline/_ref)")
    from paper_2501_14312_b200 import plugin
    plugin.install(placement="per_worker")
    yield mod
    plugin.uninstall()


@pytest.mark.parametrize("idx", range(len(SERVING)), ids=[r["name"] for r in SERVING])
def test_per_worker_contexts(idx, fs):
    from fairsched.requests import Trace, TraceRecord
    from fairsched.runner import config_from_dict, run_experiment

    run = SERVING[idx]
    cfg = config_from_dict(run["config"])
    result = run_experiment(cfg, Trace([TraceRecord(**r) for r in run["trace"]]))
    ctxs = {id(w.tree._rt.ctx) for w in result.workers}
    assert len(ctxs) == len(result.workers), "every worker must own its context"
    if getattr(result.dispatcher, "uses_global_tree", False) and hasattr(result.dispatcher, "_rt"):
        assert id(result.dispatcher._rt.ctx) not in ctxs
    assert result.log.sha256() == run["event_sha256"]
