"""Debug probe: the randomized stress lockstep (tests/test_gpu_stress.py) of one
seed, printing each step's eviction records on both sides and the FEV stats."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_stress as ts  # noqa: E402

orig_fill = None


def main(seed):
    from paper_2501_14312_b200 import device
    global orig_fill
    orig_fill = device.WorkerDev.fill

    def fill(self, now, g, h):
        r = orig_fill(self, now, g, h)
        f = int(r.stats[7])
        print(f"fill now={now} adm={len(r.adm_req)} recs={[(int(a), int(b)) for a, b in zip(r.records.length, r.records.keep)]} "
              f"fev orders={f & 0xfffff} nc={(f >> 20) & 0xfffff} heap={(f >> 40) & 0xfffff} ok={(f >> 60) & 1} "
              f"used={r.used}", flush=True)
        return r
    device.WorkerDev.fill = fill
    from oracle import oracle as om
    of = om.OracleWorker.fill

    def ofill(self, *a, **k):
        r = of(self, *a, **k)
        print(f"   oracle recs={[(len(p), int(kp)) for p, kp in r['records']]} used={self.tree.used_tokens}", flush=True)
        return r
    om.OracleWorker.fill = ofill
    try:
        ts._run(seed)
        print("OK")
    except AssertionError as e:
        print("FAIL", str(e)[:300])


if __name__ == "__main__":
    main(int(sys.argv[1]))
