"""Plugin-level parity: the reference's unchanged runner (fairsched.runner.
run_experiment) with the GPU drop-in installed must reproduce the reference
event-log sha256 of every golden run (tests/golden/serving_traces.json.gz),
including configs/example.yaml (17883b93...) and d2lpm_4workers.yaml (9a140969...)."""
import pytest

from refpath import import_fairsched
from replay import load_golden

pytestmark = pytest.mark.gpu

SERVING = load_golden("serving_traces.json")["runs"]


@pytest.fixture(scope="module")
def fs():
    mod = import_fairsched()
    if mod is None:
        pytest.skip("reference package not available (build() installs it into baseline/_ref)")
    from paper_2501_14312_b200 import plugin
    plugin.install()
    yield mod
    plugin.uninstall()


@pytest.mark.parametrize("idx", range(len(SERVING)), ids=[r["name"] for r in SERVING])
def test_event_hash_matches_reference(idx, fs):
    from fairsched.requests import Trace, TraceRecord
    from fairsched.runner import config_from_dict, run_experiment
    from paper_2501_14312_b200.policies import GpuD2lpm, GpuDlpm, GpuLpm
    from paper_2501_14312_b200.radix import DeviceRadixTree

    run = SERVING[idx]
    cfg = config_from_dict(run["config"])
    trace = Trace([TraceRecord(**r) for r in run["trace"]])
    result = run_experiment(cfg, trace)
    assert all(isinstance(w.tree, DeviceRadixTree) for w in result.workers)
    assert all(isinstance(w.policy, (GpuDlpm, GpuLpm)) for w in result.workers)
    if cfg.scheduling.global_policy == "d2lpm":
        assert isinstance(result.dispatcher, GpuD2lpm)
    assert result.log.sha256() == run["event_sha256"]
    if "violations" in run:
        got = {k: len(v) for k, v in result.violations.items()}
        assert got == run["violations"]
        assert {k: list(v) for k, v in result.counter_extremes.items()} == run["extremes"]


@pytest.mark.parametrize("idx", range(min(len(SERVING), 6)), ids=[r["name"] for r in SERVING[:6]])
def test_event_hash_with_batched_probes(idx, fs, monkeypatch):
    """The host fast path (hostpath.py) on every monitor check: the batched
    can_add of has_admissible_waiting even for 1-request queues."""
    from fairsched.requests import Trace, TraceRecord
    from fairsched.runner import config_from_dict, run_experiment
    from paper_2501_14312_b200 import hostpath

    monkeypatch.setattr(hostpath, "_BATCH_PROBE_MIN", 1)
    run = SERVING[idx]
    cfg = config_from_dict(run["config"])
    result = run_experiment(cfg, Trace([TraceRecord(**r) for r in run["trace"]]))
    # (a worker that never received a request keeps its empty list)
    assert any(isinstance(w.queue, hostpath.FastQueue) for w in result.workers)
    assert all(isinstance(w.queue, hostpath.FastQueue) or not w.queue for w in result.workers)
    assert result.log.sha256() == run["event_sha256"]


_BURST = load_golden("burst_runs.json")["runs"]


@pytest.mark.parametrize("idx", range(len(_BURST)), ids=[r["name"] for r in _BURST])
def test_same_timestamp_batches(idx, fs):
    """Arrivals in same-timestamp bursts (tests/golden/make_golden_burst.py):
    the drop-in dispatcher answers each run of arrivals from ONE device
    dispatch chain and the reference event hash is unchanged."""
    from fairsched.requests import Trace, TraceRecord
    from fairsched.runner import config_from_dict, run_experiment
    from paper_2501_14312_b200.policies import GpuD2lpm, GpuThresholdRouter

    run = _BURST[idx]
    cfg = config_from_dict(run["config"])
    result = run_experiment(cfg, Trace([TraceRecord(**r) for r in run["trace"]]))
    assert isinstance(result.dispatcher, (GpuD2lpm, GpuThresholdRouter))
    assert result.log.sha256() == run["event_sha256"]
    assert result.dispatcher.batched > 0.3 * run["same_time_arrivals"]
