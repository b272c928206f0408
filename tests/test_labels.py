"""Order-maintenance labels used for the LPM tie-break (arrival, rid)
(local_policies.py:17): label order must equal key order under any insertion
order, including gap exhaustion."""
import random

from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2501_14312_b200.runtime import OrderLabels


def check(lab, keys):
    ks = sorted(set(keys))
    labels = [lab.label(k) for k in ks]
    assert labels == sorted(labels) and len(set(labels)) == len(labels)


@settings(max_examples=100, deadline=None)
@given(st.lists(st.tuples(st.integers(0, 5), st.text(min_size=0, max_size=4)), max_size=60))
def test_labels_respect_key_order(keys):
    lab = OrderLabels()
    for k in keys:
        lab.add(k)
    check(lab, keys)


def test_gap_exhaustion_relabels():
    lab = OrderLabels()
    lab.add((0, "a"))
    lab.add((0, "z"))
    rel = None
    # insert repeatedly just above the lower key: halves the same gap
    s = "a"
    for i in range(80):
        s = s + "a"
        _, r = lab.add((0, s))
        rel = rel or r
    assert rel is not None
    check(lab, [(0, "a"), (0, "z")] + [(0, "a" * (i + 2)) for i in range(80)])


def test_python_str_order_for_rids():
    # rid compares as a Python str: "c1-10" < "c1-9"
    lab = OrderLabels()
    rng = random.Random(3)
    keys = [(rng.randrange(3), f"c{rng.randrange(3)}-{rng.randrange(20)}") for _ in range(200)]
    for k in keys:
        lab.add(k)
    check(lab, keys)


class _FakeCtx:
    """Host stand-in for device.Context: enough for the request registry."""

    def __init__(self, *a, **k):
        self.rows = []

    def add_request(self, toks, cid, lab):
        self.rows.append((tuple(int(x) for x in toks), cid, lab))
        return len(self.rows) - 1

    def request_info(self, did):
        off = sum(len(r[0]) for r in self.rows[:did])
        return off, len(self.rows[did][0])

    def set_labels(self, ids, labs):
        pass

    def set_clients(self, ids, cids):
        pass


def test_request_registry_identity(monkeypatch):
    """Requests are identified by (arrival, rid) AND their token tuple: a tuple
    shared by two requests (a req: child with an empty suffix, requests.py:
    148-156) gets two rows, a later run reusing an earlier run's (arrival, rid)
    gets its own row, and a keyless upload (a routing index walking a tuple
    first) is adopted by the request that owns the tuple."""
    from paper_2501_14312_b200 import runtime
    monkeypatch.setattr(runtime, "Context", _FakeCtx)
    rt = runtime.DeviceRuntime(0)
    base = tuple([1, 2, 3])
    a = rt.upload(base, "c", 0, "r0")
    b = rt.upload(base, "c", 0, "r0.child")
    assert a != b and rt.upload(base, "c", 0, "r0") == a and rt.upload(base, "c", 0, "r0.child") == b
    assert rt.tokens_of(a) is base and rt.tokens_of(b) is base
    later = tuple([1, 2, 3])  # a new run, same (arrival, rid), new Request object
    c = rt.upload(later, "c", 0, "r0")
    assert c not in (a, b) and rt.upload(later, "c", 0, "r0") == c
    t = (7, 8)
    d = rt.upload(t)
    assert rt.upload(t, "c", 5, "x") == d and rt.upload(t) == d
