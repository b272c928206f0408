"""Debug (not a test): run one golden policy run on the CPU reference and with
the plugin, and print the first differing dispatch record."""
import gzip
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from refpath import import_fairsched  # noqa: E402

import_fairsched()
from fairsched.requests import Trace, TraceRecord  # noqa: E402
from fairsched.runner import config_from_dict, run_experiment  # noqa: E402

runs = {r["name"]: r for r in json.load(gzip.open("tests/golden/policies_runs.json.gz"))["runs"]}
run = runs[sys.argv[1]]
cfg = config_from_dict(run["config"])
trace = Trace([TraceRecord(**r) for r in run["trace"]])
ref = run_experiment(cfg, trace)
print("cpu sha", ref.log.sha256() == run["event_sha256"])
from paper_2501_14312_b200 import plugin  # noqa: E402
plugin.install()
gpu = run_experiment(config_from_dict(run["config"]), trace)
print("gpu sha", gpu.log.sha256() == run["event_sha256"])
ra, ga = ref.dispatcher.records, gpu.dispatcher.records
for i, (a, b) in enumerate(zip(ra, ga)):
    if a != b:
        print("first diff at dispatch", i, "\n ref", a, "\n gpu", b)
        break
else:
    print("dispatch records identical", len(ra), len(ga))
ev_r = ref.log.events if hasattr(ref.log, "events") else None
print(type(ref.log), [k for k in dir(ref.log) if not k.startswith("__")][:20])
ea, eb = ref.log.events, gpu.log.events
for i, (a, b) in enumerate(zip(ea, eb)):
    if a != b:
        print("first event diff at", i)
        for j in range(max(0, i - 4), i + 2):
            print(" ref", ea[j])
            print(" gpu", eb[j])
        break
