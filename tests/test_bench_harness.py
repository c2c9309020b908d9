"""The bench's multi-rank path (replicas only) on CPU with gloo, world_size 2:
each rank runs its own sequence (no data-path collective), timing is barrier-bracketed and the
reported total is the max over ranks."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    import oracle
    import synth
    cfg = synth.CONFIGS["C1"]
    seq = synth.HostSequence(cfg)
    state = {"u": seq.initial(), "t": 0, "its": []}

    def step():  # one system of this rank's own sequence (the oracle stands in for the GPU here)
        state["t"] += 1
        A = oracle.Matrix.from_host(seq.matrix(state["t"], state["u"]))
        r = oracle.solve(A, seq.rhs(state["t"], state["u"]), m=cfg.m, tol=cfg.tol)
        state["u"] = r["x"]
        state["its"].append(r["iterations"])
        if rank == 1:  # make rank 1 measurably slower
            import time
            time.sleep(0.02)

    per, t_local, t_max = bench.timed_replicas(step, 3, 1, True, None, "cpu")
    out[rank] = (t_local, t_max, len(per), state["its"])
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_replicas_max_over_ranks():
    ws = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(ws, _free_port(), out), nprocs=ws, join=True)
    (l0, m0, n0, i0), (l1, m1, n1, i1) = out[0], out[1]
    assert n0 == n1 == 3
    assert m0 == m1 == max(l0, l1)          # every rank sees the max
    assert l1 > l0                           # rank 1 slept
    assert i0 == i1                          # independent replicas of the same sequence agree


def test_reduce_max_single_process_is_identity():
    import bench
    assert bench.reduce_max(1.5, False) == 1.5
