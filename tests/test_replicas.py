"""The N>1 plumbing of bench.py (replicas, max-over-ranks timing, whole-job
rate) on a world_size-2 gloo process group (CPU)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    from paper_2107_14758_b200 import replicas

    assert replicas.dist_env() == (rank, world, rank)
    assert replicas.init("gloo")
    t = 10.0 + 5.0 * rank  # per-rank timing (ms): the slow rank bounds the job
    tmax = replicas.max_over_ranks(t)
    replicas.barrier()
    out[rank] = (tmax, replicas.whole_job_rate(1000.0, world, tmax * 1e-3))
    replicas.finalize()


def test_two_rank_gloo_reduction():
    world, port = 2, _free_port()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0] == out[1]
    tmax, rate = out[0]
    assert tmax == 15.0 and rate == pytest.approx(2 * 1000.0 / 15e-3)


def test_single_process_is_identity():
    from paper_2107_14758_b200 import replicas

    assert replicas.max_over_ranks(3.5) == 3.5
    assert replicas.whole_job_rate(10.0, 1, 2.0) == 5.0
