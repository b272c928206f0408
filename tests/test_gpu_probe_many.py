"""DeviceRadixTree.probe_many (the batched can_add of the host fast path)
returns exactly what probe() returns one sequence at a time (radix.py:93-99),
on a tree with splits, pins and capacity evictions."""
import random

import pytest

pytestmark = pytest.mark.gpu


def test_probe_many_equals_probe():
    from paper_2501_14312_b200.radix import DeviceRadixTree
    from paper_2501_14312_b200.runtime import reset_runtimes

    rng = random.Random(7)
    base = tuple(rng.randrange(50) for _ in range(64))
    seqs = []
    for _ in range(300):
        k = rng.randrange(0, 64)
        seqs.append(base[:k] + tuple(rng.randrange(50) for _ in range(rng.randrange(1, 20))))
    tree = DeviceRadixTree(capacity=900)
    paths = []
    for i, s in enumerate(seqs[:120]):
        mlen, path = tree.admit(s, now=i)
        if rng.random() < 0.5:
            tree.unpin(path)
        else:
            paths.append(path)
        if i % 10 == 9:
            queries = rng.sample(seqs, 40)
            m, u = tree.probe_many(queries)
            one = [tree.probe(q) for q in queries]
            assert [(int(a), int(b)) for a, b in zip(m, u)] == one
    for p in paths:
        tree.unpin(p)
    m, u = tree.probe_many(seqs)
    assert [(int(a), int(b)) for a, b in zip(m, u)] == [tree.probe(q) for q in seqs]
    reset_runtimes()
