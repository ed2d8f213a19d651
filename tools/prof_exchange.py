"""Break the persistent-channel exchange into its kernels on 2 GPUs
(in-process P2P): pack+put, wait+unpack, each timed with CUDA events.

    python tools/prof_exchange.py [--n 1536] [--reps 10]
"""

import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2102_12416_b200 import _lib
    from paper_2102_12416_b200.halo import HaloJacobi

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1536)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    n = args.n
    eng = HaloJacobi((2 * n, n, n), 2, device_of=lambda r: r, timeout_s=20, exchange="p2p")
    put_ms, wait_ms, both_ms = [], [], []
    for rep in range(args.reps + 2):
        ev = {}
        for b in eng.blocks.values():
            s = eng.stream_of(b)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[b.rank] = e
            _lib.call("hx_set_device", b.device)
            e[0].record(s)
            eng._put(b, eng.it)
            e[1].record(s)
        for b in eng.blocks.values():
            s = eng.stream_of(b)
            _lib.call("hx_set_device", b.device)
            eng._wait(b, eng.it)
            ev[b.rank][2].record(s)
        eng.it += 1
        eng.synchronize()
        if rep >= 2:
            for e in ev.values():
                put_ms.append(e[0].elapsed_time(e[1]))
                wait_ms.append(e[1].elapsed_time(e[2]))
                both_ms.append(e[0].elapsed_time(e[2]))
    eng.check_errors()
    face = n * n * 8
    out = {"face_bytes": face, "put_ms": statistics.median(put_ms),
           "wait_unpack_ms": statistics.median(wait_ms), "exchange_ms": statistics.median(both_ms)}
    out["put_GBps"] = face / (out["put_ms"] * 1e-3) / 1e9
    out["exchange_GBps"] = face / (out["exchange_ms"] * 1e-3) / 1e9
    print(json.dumps(out), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
