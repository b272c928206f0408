"""Plugin-level parity beyond DLPM/LPM/D2LPM: with the drop-in installed every
worker's RadixTree is the device tree; Vtc's fill is the device kernel k_vtc
(GpuVtc), ThresholdRouter's dispatch chain runs on the device index
(GpuThresholdRouter), FCFS and the rr / per_client_rr routers use the device
tree through the per-call operations.  The reference's
unchanged runner must reproduce the event-log sha256 and service-gap
violation counts recorded from the CPU reference
(tests/golden/make_golden_policies.py), including the config-4 style
comparison: one bursty trace (cv=4, up to 120 clients) under dlpm / vtc / lpm /
fcfs."""
import gzip
import json
import os

import pytest

from refpath import import_fairsched

pytestmark = pytest.mark.gpu

RUNS = json.load(gzip.open(os.path.join(os.path.dirname(__file__), "golden", "policies_runs.json.gz")))["runs"]


@pytest.fixture(scope="module")
def fs():
    mod = import_fairsched()
    if mod is None:
        pytest.skip("reference package not available (build() installs it into baseline/_ref)")
    from paper_2501_14312_b200 import plugin
    plugin.install()
    yield mod
    plugin.uninstall()


@pytest.mark.parametrize("idx", range(len(RUNS)), ids=[r["name"] for r in RUNS])
def test_policy_run_matches_reference(idx, fs):
    from fairsched.requests import Trace, TraceRecord
    from fairsched.runner import config_from_dict, run_experiment
    from paper_2501_14312_b200.radix import DeviceRadixTree

    run = RUNS[idx]
    cfg = config_from_dict(run["config"])
    trace = Trace([TraceRecord(**r) for r in run["trace"]])
    result = run_experiment(cfg, trace)
    assert all(isinstance(w.tree, DeviceRadixTree) for w in result.workers)
    assert result.log.sha256() == run["event_sha256"]
    assert {k: len(v) for k, v in result.violations.items()} == run["violations"]


_C4 = os.path.join(os.path.dirname(__file__), "golden", "config4_runs.json.gz")
C4 = json.load(gzip.open(_C4)) if os.path.exists(_C4) else {"trace": [], "runs": []}


@pytest.mark.parametrize("idx", range(len(C4["runs"])), ids=[r["name"] for r in C4["runs"]])
def test_config4_1000_clients(idx, fs):
    """Config 4 (BASELINE configs[3]) at its full client count: 1000 bursty
    clients (cv=4), L_input 4096, M 65536, dlpm / vtc / lpm on the same
    8,342-request trace (cli compare, cli.py:62-89) through the unchanged
    runner with the device tree: event sha256, monitor violations and the
    counter extremes recorded from the CPU reference."""
    from fairsched.requests import Trace, TraceRecord
    from fairsched.runner import config_from_dict, run_experiment
    from paper_2501_14312_b200.radix import DeviceRadixTree

    from paper_2501_14312_b200.policies import GpuDlpm, GpuLpm, GpuVtc

    run = C4["runs"][idx]
    cfg = config_from_dict(run["config"])
    result = run_experiment(cfg, Trace([TraceRecord(**r) for r in C4["trace"]]))
    assert all(isinstance(w.tree, DeviceRadixTree) for w in result.workers)
    cls = {"dlpm": GpuDlpm, "lpm": GpuLpm, "vtc": GpuVtc}[run["config"]["scheduling"]["local_policy"]]
    assert all(isinstance(w.policy, cls) for w in result.workers)  # the fill runs on the device
    assert result.log.sha256() == run["event_sha256"]
    assert {k: len(v) for k, v in result.violations.items()} == run["violations"]
    assert {k: list(v) for k, v in result.counter_extremes.items()} == run["extremes"]
