"""World-size-2 gloo test of the multi-rank channel set-up on CPU.

Each process plays one rank of a (2,1,1) / (1,2,1) / (1,1,2) block grid,
publishes a fake arena record through the same exchange_table() the GPU
path uses (torch.distributed all_gather_object), links its put targets,
and the two ranks cross-check that every put lands exactly on the
neighbour's receive slot and flag for the opposite side — the
persistent-channel invariant that replaces per-message tags.
"""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, dims, pes, out):
    import sys

    sys.path.insert(0, ROOT)
    from paper_2102_12416_b200.halo import HaloBlock, exchange_table
    from paper_2102_12416_b200.jacobi3d import decompose

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    grid = decompose(dims, pes)
    fake_base = 0x7F0000000000 + rank * (1 << 36)
    b = HaloBlock(dims, grid, rank, device=0, allocate=False)
    table = exchange_table(dist, [(rank, b"h%d" % rank, fake_base, 0)])
    for d in b.nbr_dirs:
        b.link(d, table[b.neighbors[d]][1])
    mine = {"rank": rank, "base": fake_base,
            "puts": {d: (b.put_slot(d, 0), b.put_slot(d, 1), b.put_flag[d]) for d in b.nbr_dirs},
            "recv": {d: (b.slot_ptr(0, d, fake_base), b.slot_ptr(1, d, fake_base),
                         b.flag_ptr(d, fake_base)) for d in b.nbr_dirs},
            "neighbors": b.neighbors}
    everyone = [None] * world
    dist.all_gather_object(everyone, mine)
    if rank == 0:
        out.put(everyone)
    dist.destroy_process_group()


@pytest.mark.parametrize("dims", [(32, 16, 16), (16, 32, 16), (16, 16, 32)])
def test_two_rank_channel_setup(dims):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dims, 2, q)) for r in range(2)]
    for p in procs:
        p.start()
    everyone = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    by_rank = {e["rank"]: e for e in everyone}
    for e in everyone:
        for d, put in e["puts"].items():
            n = by_rank[e["neighbors"][d]]
            assert n["neighbors"][d ^ 1] == e["rank"]
            assert put == n["recv"][d ^ 1]  # both parity slots and the flag line up
