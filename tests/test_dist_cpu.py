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


def _shard_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank), BF_BENCH_BACKEND="gloo")
    import torch
    import torch.distributed as dist
    import bench
    import paper_1803_00004_b200 as pkg
    from synth import CONFIGS
    w, r, _ = bench.dist_setup(world)
    fr = bench.rank_frames(pkg, CONFIGS["cfg3"], w, r)          # this rank's frames of the stream
    mine = torch.zeros(CONFIGS["cfg3"].frames, dtype=torch.int64)
    mine[fr.start:fr.stop] = 1
    dist.all_reduce(mine)                                        # gloo: how many ranks took each frame
    single = bench.rank_frames(pkg, CONFIGS["cfg2"], w, r)      # single images: replicated
    dist.destroy_process_group()
    q.put((r, fr.start, fr.stop, mine.tolist(), list(single)))


@pytest.mark.timeout(120)
def test_cfg3_frames_sharded_over_two_gloo_ranks():
    """NEXT f4 (BASELINE configs[3]): a frame stream is sharded over the ranks (bf_shard_frames,
    contiguous blocks), every frame filtered by exactly one rank, with no data-path collective
    (the all_reduce here only checks the coverage); single images stay replicated per rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=90) for _ in procs)
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    assert [(a, b) for _, a, b, _, _ in res] == [(0, 32), (32, 64)]
    assert all(cov == [1] * 64 for _, _, _, cov, _ in res)
    assert all(single == [0] for *_, single in res)


@pytest.mark.parametrize("n,parts", [(64, 2), (64, 3), (64, 8), (5, 8), (0, 4), (1000, 7)])
def test_shard_frames_partition(n, parts):
    import paper_1803_00004_b200 as pkg
    blocks = [pkg.shard_frames(n, parts, p) for p in range(parts)]
    assert sum(c for _, c in blocks) == n
    pos = 0
    for first, count in blocks:
        assert first == pos and count >= 0
        pos += count
    counts = [c for _, c in blocks]
    assert max(counts) - min(counts) <= 1
