"""Multi-process logic of bench.py on CPU (gloo, world_size 2): device times are max-reduced over
ranks and the whole-job value counts every rank's pixels (weak scaling, no data-path
collective: each rank filters its own image)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank), BF_BENCH_BACKEND="gloo")
    import bench
    w, r, _ = bench.dist_setup(world)
    t = 10.0 + 5.0 * r                       # rank 1 is slower
    tmax = bench.reduce_max(t, w)
    bench.barrier(w)
    import torch.distributed as dist
    dist.destroy_process_group()
    q.put((r, w, tmax))


@pytest.mark.timeout(120)
def test_reduce_max_over_two_gloo_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=90) for _ in procs)
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    assert [r for r, _, _ in res] == [0, 1]
    assert all(w == 2 and tmax == 15.0 for _, w, tmax in res)


def test_single_process_defaults():
    import bench
    os.environ.pop("WORLD_SIZE", None)
    w, r, l = bench.dist_setup(1)
    assert (w, r, l) == (1, 0, 0)
    assert bench.reduce_max(3.5, 1) == 3.5
