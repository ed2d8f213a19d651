"""NCCL send/recv ping-pong and windowed bandwidth on 2 GPUs — the
comparison point the north star names for the persistent-channel path.

    torchrun --nproc-per-node 2 tools/nccl_osu.py [--out gpurun_out/nccl_osu.json]

Latency: one-way = device time of `iters` round trips / (2 iters), CUDA
events on the issuing stream (NCCL work is stream-ordered behind wait()).
Bandwidth: window of 64 isend/irecv of `size` bytes then an 8-byte ack.
"""
import argparse
import json
import os

import torch
import torch.distributed as dist


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/nccl_osu.json")
    args = ap.parse_args()
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    other = 1 - rank
    rows = []
    size = 8
    while size <= 4 << 20:
        buf = torch.full((size,), (size * 11) & 0xFF, dtype=torch.uint8, device="cuda")
        rbuf = torch.zeros_like(buf)
        iters = 200 if size <= 65536 else 50
        for _ in range(10):  # warm-up
            if rank == 0:
                dist.send(buf, other)
                dist.recv(rbuf, other)
            else:
                dist.recv(rbuf, other)
                dist.send(rbuf, other)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            if rank == 0:
                dist.send(buf, other)
                dist.recv(rbuf, other)
            else:
                dist.recv(rbuf, other)
                dist.send(rbuf, other)
        e1.record()
        torch.cuda.synchronize()
        lat_us = e0.elapsed_time(e1) * 1e3 / (2 * iters)
        window, reps = 64, 5
        ack = torch.zeros(8, dtype=torch.uint8, device="cuda")
        dist.barrier()
        torch.cuda.synchronize()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for rep in range(reps + 1):
            if rep == 1:
                e2.record()
            if rank == 0:
                ws = [dist.isend(buf, other) for _ in range(window)]
                for w in ws:
                    w.wait()
                dist.recv(ack, other)
            else:
                ws = [dist.irecv(rbuf, other) for _ in range(window)]
                for w in ws:
                    w.wait()
                dist.send(ack, other)
        e3.record()
        torch.cuda.synchronize()
        bw = reps * window * size / (e2.elapsed_time(e3) * 1e-3) / 1e9
        ok = bool((rbuf == ((size * 11) & 0xFF)).all().item())
        if rank == 0:
            rows.append({"size": size, "latency_us": lat_us, "bandwidth_gbps": bw, "verified": ok})
            print(json.dumps(rows[-1]), flush=True)
        size *= 2
    if rank == 0:
        with open(args.out, "w") as f:
            json.dump({"impl": "nccl", "version": ".".join(map(str, torch.cuda.nccl.version())),
                       "rows": rows}, f, indent=1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
