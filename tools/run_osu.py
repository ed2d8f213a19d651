"""OSU-style sweep on two GPUs (BASELINE.json configs[1]): 8 B - 4 MiB.

API level (the reference's measure_latency / measure_bandwidth procedures,
cl/bench.py:364-452, through the drop-in runtime): charm-channel,
charm-messaging and mpi, device mode, plus host-staging for contrast.
Persistent channel (pchannel: pre-registered slots, device-side counters,
per-GPU CUDA graphs): ping-pong latency and window bandwidth.
Device level: kernel-issued NVLink ping-pong (globaltimer) and windowed
peer-copy bandwidth (copy engine and SM stores, CUDA events).

    python tools/run_osu.py [--out gpurun_out/osu.json] [--quick]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "osu.json"))
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()

    import torch

    from paper_2102_12416_b200.osu import (channel_bandwidth, channel_latency, device_bandwidth,
                                           device_latency, measure_bandwidth, measure_latency,
                                           parse_sizes)

    ngpu = torch.cuda.device_count()
    sizes = parse_sizes("8:4194304:x2")
    if args.quick:
        sizes = [8, 4096, 1 << 20, 4 << 20]
    rows = []

    def emit(r):
        rows.append(r)
        print(json.dumps(r), flush=True)

    if ngpu >= 2:  # untimed warm-up: the first graph replays of a process run slow
        channel_latency(8, iters=500, warmup=50)
        device_latency(8, iters=500, warmup=50)
    for size in sizes:
        lat_iters = 200 if size <= 65536 else 50
        for api in ("charm-channel", "charm-messaging", "mpi"):
            r = measure_latency(api, "device", size, iters=lat_iters, warmup=5)
            emit({**r, "level": "api", "gpus": min(ngpu, 2)})
        r = measure_latency("charm-channel", "host", size, iters=lat_iters // 2, warmup=3)
        emit({**r, "level": "api", "gpus": min(ngpu, 2)})
        for api in ("charm-channel", "charm-messaging"):
            r = measure_bandwidth(api, "device", size, window=64, iters=5, warmup=2)
            emit({**r, "level": "api", "gpus": min(ngpu, 2)})
        if ngpu >= 2:
            emit(channel_latency(size, iters=1000 if size <= 65536 else 200, warmup=20))
            emit(channel_bandwidth(size, window=64, iters=5))  # 64 KiB slots: pull above
            if size > (64 << 10):  # slots as large as the message: push into the slot
                emit(channel_bandwidth(size, window=64, iters=5, slot_bytes=None))
            emit({**device_latency(size, iters=2000 if size <= 65536 else 200, warmup=50),
                  "level": "device"})
            for engine in ("ce", "sm", "sm-pull", "sm-window", "sm-pull-window"):
                emit({**device_bandwidth(size, window=64, iters=5, engine=engine),
                      "level": "device"})
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump({"gpus": ngpu, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
