"""GPU parity: the CUDA path (through the C ABI) replays every golden op trace
recorded from the reference and must reproduce every admission, eviction
record, counter, dump and dispatch decision bit-exactly."""
import pytest

from replay import load_golden, replay_radix, replay_serving

pytestmark = pytest.mark.gpu

SERVING = load_golden("serving_traces.json")["runs"]
RADIX = load_golden("radix_traces.json")["traces"]


@pytest.fixture(scope="module")
def backend():
    from gpu_backend import GpuBackend
    be = GpuBackend()
    yield be
    be.close()


@pytest.mark.parametrize("idx", range(len(SERVING)), ids=[r["name"] for r in SERVING])
def test_gpu_serving_trace(idx, backend):
    stats = replay_serving(SERVING[idx], backend)
    assert stats["fills"] > 0


@pytest.mark.parametrize("idx", range(len(RADIX)))
def test_gpu_radix_trace(idx):
    from paper_2501_14312_b200.radix import CacheFull, DeviceRadixTree
    from paper_2501_14312_b200.runtime import get_runtime

    def make_tree(capacity, track_workers, n_workers):
        t = DeviceRadixTree(capacity=capacity, track_workers=track_workers, n_workers=max(n_workers, 1),
                            runtime=get_runtime())
        sink = []
        t.on_evict = lambda path, keep, ev: sink.append((tuple(path), keep))
        t.last_sink = sink
        return _Recording(t)

    replay_radix(RADIX[idx], make_tree, CacheFull)


class _Recording:
    """Adapts DeviceRadixTree to the replay's `last_records` convention."""

    def __init__(self, t):
        self.t = t

    def __getattr__(self, k):
        return getattr(self.t, k)

    def insert(self, toks, now=0, worker=None):
        self.t.last_sink.clear()
        try:
            return self.t.insert(toks, now=now, worker=worker)
        finally:
            self.last_records = list(self.t.last_sink)

    def admit(self, toks, now=0):
        self.t.last_sink.clear()
        try:
            return self.t.admit(toks, now=now)
        finally:
            self.last_records = list(self.t.last_sink)

    def evict_lru(self, needed):
        self.t.last_sink.clear()
        return self.t.evict_lru(needed)
