"""Host bookkeeping fast path (paper_2501_14312_b200.hostpath):
FastQueue keeps list semantics for everything the reference does with
Worker.queue (worker.py:73, 127, 137-147; local_policies.py:62-70, 155, 174;
runner.py:354)."""
from dataclasses import dataclass

import pytest

from paper_2501_14312_b200.hostpath import FastQueue


@dataclass(frozen=True)
class R:
    rid: str
    client: str


def test_order_remove_and_client_counts():
    rs = [R(f"r{i}", "ab"[i % 2]) for i in range(7)]
    q, ref = FastQueue(), []
    for r in rs:
        q.append(r)
        ref.append(r)
    assert list(q) == ref and len(q) == 7 and bool(q)
    for r in (rs[3], rs[0], rs[6]):
        q.remove(r)
        ref.remove(r)
        assert list(q) == ref
    assert q.has_client("a") and q.has_client("b")
    for r in list(ref):
        if r.client == "a":
            q.remove(r)
            ref.remove(r)
    assert not q.has_client("a") and q.has_client("b")
    assert sorted(q, key=lambda r: r.rid) == sorted(ref, key=lambda r: r.rid)
    assert q[0] == ref[0] and rs[1] in q and rs[0] not in q


def test_remove_by_equality_and_missing():
    q = FastQueue([R("x", "c"), R("y", "c")])
    q.remove(R("y", "c"))  # an equal object, not the same one (list.remove semantics)
    assert [r.rid for r in q] == ["x"]
    with pytest.raises(ValueError):
        q.remove(R("zz", "c"))
    q.remove(R("x", "c"))
    assert not q and len(q) == 0 and not q.has_client("c")


def test_iteration_is_a_snapshot():
    q = FastQueue([R(str(i), "c") for i in range(4)])
    seen = []
    for r in q:
        seen.append(r.rid)
        q.remove(r)
    assert seen == ["0", "1", "2", "3"] and not q
