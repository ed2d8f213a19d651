"""torchrun worker for the multi-process (CUDA IPC) halo path.

    torchrun --nproc-per-node N tests/mp_halo_worker.py DX DY DZ ITERS OUT.json [MODE]
    HX_SAME_GPU=1 torchrun ...   (every rank on cuda:0: the 1-GPU IPC variant)

MODE: 0 = channel exchange, 1 = channel exchange + interior overlap,
fused = boundary sweep stores straight into the neighbours' ghost planes,
graph = fused, replayed from per-process CUDA graphs (no residuals),
nccl = the comparison path (pack, grouped NCCL send/recv, unpack; needs one
GPU per rank — NCCL refuses two ranks on one device).

One rank per GPU: HaloJacobi with local_ranks=[rank] opens its neighbours'
receive arenas through CUDA IPC handles exchanged once over gloo, runs
ITERS iterations of fused pack+put / wait+unpack / stencil, then rank 0
gathers the block interiors, compares the assembled field with the CPU
oracle bit for bit and writes the verdict to OUT.json.
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2102_12416_b200.halo import HaloJacobi

    dims = tuple(int(x) for x in sys.argv[1:4])
    iters = int(sys.argv[4])
    out = sys.argv[5]
    mode = sys.argv[6] if len(sys.argv) > 6 else "0"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    # HX_SAME_GPU=1: every rank on cuda:0 — CUDA IPC opens another process's
    # allocation on the same device, so a 1-GPU box runs the cross-process path
    same = os.environ.get("HX_SAME_GPU") == "1"
    local = 0 if same else int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    if mode == "nccl":  # the comparison exchange: NCCL send/recv on CUDA tensors, gloo for objects
        dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("gloo")
    exchange = {"fused": "fused", "graph": "fused", "nccl": "nccl"}.get(mode, "p2p")
    eng = HaloJacobi(dims, world, local_ranks=[rank], device_of=(lambda r: 0) if same else (lambda r: r),
                     dist=dist, timeout_s=20, overlap=mode == "1", exchange=exchange)
    if mode == "graph":
        eng.run_graph(iters)
    else:
        eng.run(iters, residual=True)
    eng.check_errors()
    if os.environ.get("HX_VERIFY") == "gpu":
        # bench-sized blocks: every rank checks its own block against the
        # single-array GPU sweep (the C/numpy oracle pins that sweep at
        # small sizes) instead of shipping fields to rank 0
        from paper_2102_12416_b200.jacobi3d import _block_coords, sequential_oracle

        want, _ = sequential_oracle(dims, iters, device=local)
        b = eng.blocks[rank]
        ix, iy, iz = _block_coords(rank, eng.grid)
        ref = want[ix * b.bx:(ix + 1) * b.bx, iy * b.by:(iy + 1) * b.by, iz * b.bz:(iz + 1) * b.bz]
        ok = bool(np.array_equal(eng.interior_host(rank), ref))
        allp = [None] * world
        dist.all_gather_object(allp, ok)
        if rank == 0:
            with open(out, "w") as f:
                json.dump({"bitwise": all(allp), "residuals": True, "grid": list(eng.grid),
                           "world": world}, f)
        eng.close()
        dist.barrier()
        dist.destroy_process_group()
        return
    mine = (rank, eng.interior_host(rank), eng.residuals(rank))
    allp = [None] * world
    dist.all_gather_object(allp, mine)
    if rank == 0:
        from oracle import jacobi_np

        parts = sorted(allp, key=lambda t: t[0])
        field = jacobi_np.assemble([p[1] for p in parts], dims, eng.grid)
        want, wres = jacobi_np.sequential(dims, iters)
        res = [max(col) for col in zip(*[p[2] for p in parts])]
        verdict = {"bitwise": field.tobytes() == want.tobytes(),
                   "residuals": mode == "graph" or res == wres,
                   "grid": list(eng.grid), "world": world,
                   "z_interior": any(eng.z_interior(b) for b in eng.blocks.values())
                   if exchange == "fused" else False}
        with open(out, "w") as f:
            json.dump(verdict, f)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
