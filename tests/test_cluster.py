"""Multi-GPU D^2LPM protocol (paper_2501_14312_b200.cluster): the
replicated-dispatcher rounds must make exactly the decisions one dispatcher
with all workers in one process makes (tests/cluster_oracle.SingleCluster)."""
import json
import socket

import pytest
import torch.multiprocessing as mp

import cluster_oracle as co
from paper_2501_14312_b200.cluster import LocalComm


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def single():
    return {D: co.run_single(D) for D in (1, 2)}


@pytest.fixture(scope="module")
def single_pipe():
    return {D: co.run_single(D, pipelined=True) for D in (1, 2)}


def _check(rank_results, ref, D):
    assert rank_results[0]["seed"] == ref["seed"]
    for res in rank_results:
        assert res["seed"] == ref["seed"], "replicas disagree on the initial dispatch"
    for k, rr in enumerate(ref["rounds"]):
        for r, res in enumerate(rank_results):
            assert res["rounds"][k]["dispatched"] == rr["dispatched"], (k, r)
            assert res["rounds"][k]["admitted"] == rr["admitted"][r], (k, r)
    for res in rank_results:
        assert res["qsize"] == [int(x) for x in ref["qsize"]]


def test_workload_exercises_protocol(single):
    ref = single[2]
    adm = [sum(len(a) for a in rr["admitted"]) for rr in ref["rounds"]]
    assert all(a > 0 for a in adm)
    ws = set(ref["seed"]) | {w for rr in ref["rounds"] for w in rr["dispatched"]}
    assert ws == {0, 1}, "both workers must receive requests"
    assert ref["n_notices"] > 50, "eviction notices must flow through the exchange"


def test_local_rank_matches_single(single):
    q = co.workload()
    be = co.OracleRank(0, q, 1)
    res = co.run_rank(0, LocalComm(), be)
    res["qsize"] = [int(x) for x in be.dispatcher_state(co.SPEC.clients)[-1]]
    _check([res], single[1], 1)


def _spawn(world, kind, tmp_path, pipelined=False):
    port = _free_port()
    mp.start_processes(co.gloo_main, args=(world, port, str(tmp_path), kind, pipelined), nprocs=world, join=True,
                       start_method="spawn")
    return [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]


def test_gloo_two_ranks_oracle(single, tmp_path):
    _check(_spawn(2, "oracle", tmp_path), single[2], 2)


@pytest.mark.gpu
def test_gpu_rank_single(single):
    q = co.workload()
    be = co.make_gpu_rank(0, q, 1, "cuda:0")
    res = co.run_rank(0, LocalComm(), be)
    res["qsize"] = [int(x) for x in be.dispatcher_state(co.SPEC.clients)[-1]]
    _check([res], single[1], 1)


@pytest.mark.gpu
def test_gpu_two_ranks_gloo(single, tmp_path):
    """Two ranks (both on cuda:0 here; one per GPU in deployment) over gloo."""
    _check(_spawn(2, "gpu", tmp_path), single[2], 2)


def test_pipelined_differs_but_dispatches_alike(single, single_pipe):
    """Pipelining moves the local enqueue one round later: the schedules differ,
    the protocol still exercises every worker."""
    assert single_pipe[2]["rounds"] != single[2]["rounds"]
    ws = {w for rr in single_pipe[2]["rounds"] for w in rr["dispatched"]}
    assert ws == {0, 1}


def test_gloo_two_ranks_oracle_pipelined(single_pipe, tmp_path):
    _check(_spawn(2, "oracle", tmp_path, pipelined=True), single_pipe[2], 2)


@pytest.mark.gpu
def test_gpu_two_ranks_gloo_pipelined(single_pipe, tmp_path):
    """Pipelined rounds on the CUDA backend (dispatcher on its own stream)."""
    _check(_spawn(2, "gpu", tmp_path, pipelined=True), single_pipe[2], 2)
