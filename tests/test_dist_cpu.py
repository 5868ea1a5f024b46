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
