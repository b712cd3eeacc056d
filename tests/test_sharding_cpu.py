"""Host-side logic of the multi-GPU decompositions, on CPU (gloo, world 2)."""
import os

import pytest

from paper_2312_02376_b200.sharding import excitation_shard, fft_columns, slab_planes


@pytest.mark.parametrize("n0,world", [(256, 8), (64, 3), (32, 4), (12, 4), (7, 2)])
def test_slab_planes_partition(n0, world):
    x = slab_planes(n0, world)
    assert x[0] == 0 and x[-1] == n0
    assert all(b >= a for a, b in zip(x, x[1:]))
    assert max(b - a for a, b in zip(x, x[1:])) - min(b - a for a, b in zip(x, x[1:])) <= 1


def test_fft_columns_partition():
    c = fft_columns(256, 256, 8)
    assert c[0] == 0 and c[-1] == 512 * 512
    assert len(set(b - a for a, b in zip(c, c[1:]))) == 1


def test_excitation_shard_covers_each_once():
    for world in (1, 2, 4, 8):
        got = sorted(e for r in range(world) for e in excitation_shard(64, world, r))
        assert got == list(range(64))


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # the NCCL unique-id exchange bench.py uses: rank 0's 128-byte blob to all ranks
    blob = [bytes(range(128))] if rank == 0 else [None]
    dist.broadcast_object_list(blob, src=0)
    mine = excitation_shard(64, world, rank)
    allx = [None] * world
    dist.all_gather_object(allx, mine)
    out.put((rank, blob[0] == bytes(range(128)), sorted(e for part in allx for e in part) == list(range(64)),
             slab_planes(256, world)))
    dist.destroy_process_group()


def test_gloo_world2_id_exchange_and_sharding():
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok_blob and ok_cover for _, ok_blob, ok_cover, _ in res)
    assert res[0][3] == res[1][3] == [0, 128, 256]
