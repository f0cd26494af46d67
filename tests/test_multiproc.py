"""The N>1 host logic of bench.py on CPU (gloo, world_size 2): replicas only -- each rank
runs the whole path on its own device; the only cross-rank traffic is the timing reduction
(max of per-rank times) and the sample count (sum), exactly as on NCCL."""
import os
import socket
import sys

import pytest

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, l = bench.dist_env()
    t = bench.max_over_ranks(10.0 + rank, w)
    s = bench.sum_over_ranks(100.0 * (rank + 1), w)
    bench.barrier(w)
    dist.destroy_process_group()
    q.put((r, w, l, t, s))


def test_replica_reductions_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert [x[0] for x in res] == [0, 1]
    assert all(x[1] == 2 for x in res)
    assert all(x[3] == 11.0 for x in res)   # max over ranks of the per-rank times
    assert all(x[4] == 300.0 for x in res)  # whole-job samples = sum over ranks


def test_reference_arm_nonzero_ranks_exit_quietly(capsys):
    sys.path.insert(0, ROOT)
    import bench

    class A:
        pass

    assert bench.run_reference_arm(A(), bench.CONFIGS["c2"], rank=1, world=2) == 0
    assert capsys.readouterr().out == ""
