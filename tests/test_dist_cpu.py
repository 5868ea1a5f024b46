"""CPU, world_size 2 over gloo: the host side of the multi-process paths — the tensor-parallel handle
exchange (gather_tp_handles, rank order) as link_tp_processes uses it."""
import os

import pytest
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_05524_b200.specpar import gather_tp_handles
    mine = bytes([rank]) * 256
    flat = gather_tp_handles(mine)
    q.put((rank, flat))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_tp_handles_rank_order(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29650 + world
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = b"".join(bytes([r]) * 256 for r in range(world))
    assert all(v == want for v in got.values())


_CHILD = ("import os, sys; r, n, port = map(int, os.environ['DBL_TP_CHILD'].split(',')); "
          "assert 'RANK' not in os.environ and 'MASTER_PORT' not in os.environ; "
          "fail = os.environ.get('FAIL_RANK') == str(r); "
          "print('{\"rank\": %d, \"world\": %d}' % (r, n)); sys.exit(3 if fail else 0)")


def _bench_worker(rank, world, port, fail_rank, q):
    import sys
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["FAIL_RANK"] = str(fail_rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    line, err = bench.tp_children(None, rank, world, cmd=[sys.executable, "-c", _CHILD], timeout=120)
    q.put((rank, line, err, bench.all_max(rank + 1, world), bench.all_min(rank + 1, world)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,fail_rank", [(2, -1), (2, 1), (3, 0)])
def test_bench_tp_children_agree(world, fail_rank):
    """bench.py --gpus N (one process per GPU): every rank runs its tensor-parallel child; rank 0 prints
    its line only if every rank's child succeeded, otherwise all ranks fall back together (the first
    error recorded).  Timing is the max over ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + 10 * world + fail_rank + 1
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, fail_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {r: (line, err, mx, mn) for r, line, err, mx, mn in (q.get(timeout=180) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, (line, err, mx, mn) in got.items():
        assert mx == world and mn == 1
        if fail_rank < 0:
            assert err == ""
            assert line == ('{"rank": 0, "world": %d}' % world if r == 0 else "")
        else:
            assert line is None and err.startswith(f"rank {fail_rank}:")
