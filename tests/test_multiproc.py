"""Multi-rank host logic of bench.py on CPU (gloo, world size 2): ranks run
independent replicas, the step time is the max over ranks, and the whole-job
value aggregates all ranks' bytes (weak scaling, no data-path collective)."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update({"RANK": str(rank), "LOCAL_RANK": str(rank), "WORLD_SIZE": str(world),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import bench
    import torch.distributed as dist

    w, r, _ = bench.dist_setup(world, backend="gloo")
    ms_local = 10.0 + 5.0 * r  # rank 1 is the slow replica
    ms = bench.dist_max(ms_local, w)
    bench.barrier(w)
    out[r] = (w, ms, bench.replica_value(bench.STEP_BYTES, w, ms))
    dist.destroy_process_group()


def test_two_rank_replicas_max_time_and_aggregate():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert set(res) == {0, 1}
    for r in (0, 1):
        w, ms, value = res[r]
        assert w == 2 and ms == 15.0  # both ranks see the slowest replica
        import bench

        assert value == pytest.approx(2 * bench.STEP_BYTES / 15e-3 / 1e9)
