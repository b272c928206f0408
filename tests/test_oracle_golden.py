"""Pin the CPU oracle (oracle/fs_oracle.c) against golden traces recorded from
the real reference (tests/golden/make_golden.py).  CPU only."""
import pytest

from oracle import oracle as O
from replay import OracleBackend, load_golden, replay_radix, replay_serving

RADIX = load_golden("radix_traces.json")["traces"]
SERVING = load_golden("serving_traces.json")["runs"]


@pytest.mark.parametrize("idx", range(len(RADIX)))
def test_oracle_radix_trace(idx):
    replay_radix(RADIX[idx], O.OracleTree, O.OracleCacheFull)


@pytest.mark.parametrize("idx", range(len(SERVING)), ids=[r["name"] for r in SERVING])
def test_oracle_serving_trace(idx):
    stats = replay_serving(SERVING[idx], OracleBackend())
    assert stats["fills"] > 0
