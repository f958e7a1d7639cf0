"""CPU, world_size 2 over gloo: the multi-GPU orchestration of bench.py.

On N GPUs each rank renders the 64x64 super-tiles it owns (vxa_tile_owner)
straight into rank 0's framebuffer through a CUDA IPC peer mapping whose
64-byte handle rank 0 broadcasts. Here (no GPU) two gloo ranks check that
the ownership map splits the frame into disjoint, complete pixel sets and
that the handle exchange delivers rank 0's bytes to every rank.
"""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

W, H = 640, 360


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    import paper_1911_06001_b200 as vx

    lib = vx.vxa()
    owned = np.zeros((H, W), np.uint8)
    for y in range(H):
        for x in range(W):
            owned[y, x] = lib.vxa_tile_owner(x, y, W, H, world) == rank
    total = [None] * world
    dist.all_gather_object(total, owned)
    fake_handle = bytes(range(64)) if rank == 0 else bytes(64)
    got = bench.exchange_handle(dist, rank, fake_handle)
    out[rank] = (np.stack(total).sum(axis=0).tolist() if rank == 0 else None, got)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_partition_and_handle_exchange():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    cover = np.array(out[0][0])
    assert (cover == 1).all(), "every pixel owned by exactly one rank"
    for r in range(world):
        assert out[r][1] == bytes(range(64))
