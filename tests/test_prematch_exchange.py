"""The multi-GPU D2LPM batch-start match exchange (cluster.partitioned_prematch,
SURVEY 8e) over gloo with world size 2 on CPU: every rank matches its slice
of each arrival batch, one all-gather hands every rank the whole batch's
records in arrival order.  A host matcher stands in for fs_dispatch_prematch
(record = the arrival's request id and its position, so order and coverage
are checked exactly); the CUDA records are tested by test_gpu_prematch.py."""
import json
import socket

import numpy as np
import torch.multiprocessing as mp

REC = 16


class HostMatcher:
    """Writes one 16-byte record per arrival: (request id, rank-independent tag)."""
    record_bytes = REC

    def prematch(self, ids, ptr):
        import ctypes
        a = np.zeros((len(ids), 2), np.int64)
        a[:, 0] = ids
        a[:, 1] = 7
        ctypes.memmove(ptr, a.ctypes.data, a.nbytes)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, out_dir):
    import os
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    import torch.distributed as dist
    from paper_2501_14312_b200.cluster import TorchComm, partitioned_prematch
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        comm = TorchComm("cpu")
        got = []
        for n in (1, 2, 3, 7, 64, 129):
            ids = np.arange(1000, 1000 + n, dtype=np.int32) * 3
            out = partitioned_prematch(HostMatcher(), ids, comm, None)
            rec = out.numpy().view(np.int64).reshape(-1, 2)
            got.append(rec[:n, 0].tolist())
        with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
            json.dump(got, f)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_ranks_gather_every_slice_in_order(tmp_path):
    world = 2
    mp.start_processes(_rank_main, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    outs = [json.load(open(tmp_path / f"r{r}.json")) for r in range(world)]
    for n, a, b in zip((1, 2, 3, 7, 64, 129), outs[0], outs[1]):
        want = (np.arange(1000, 1000 + n) * 3).tolist()
        assert a == want and b == want, n
