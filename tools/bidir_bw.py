"""Bidirectional NVLink bandwidth: both GPUs move a window at once
(push = SM stores to the peer, pull = SM loads from the peer)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2102_12416_b200 import _lib

    for a, b in ((0, 1), (1, 0)):
        _lib.call("hx_enable_peer", a, b)
    for size, window in ((1 << 20, 32), (4 << 20, 32), (16 << 20, 32), (19 << 20, 32), (19 << 20, 1)):
        for mode in ("push", "pull"):
            bufs = {g: (torch.ones(size, dtype=torch.uint8, device=f"cuda:{g}"),
                        torch.zeros(size, dtype=torch.uint8, device=f"cuda:{g}")) for g in (0, 1)}
            streams = {g: torch.cuda.Stream(device=g) for g in (0, 1)}
            ev = {}
            for rep in range(2):
                for g in (0, 1):
                    o = 1 - g
                    src, dst = (bufs[g][0], bufs[o][1]) if mode == "push" else (bufs[o][0], bufs[g][1])
                    _lib.call("hx_set_device", g)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    with torch.cuda.device(g):
                        e0.record(streams[g])
                        _lib.call("hx_copy_sm_window", dst.data_ptr(), src.data_ptr(), size, window,
                                  streams[g].cuda_stream)
                        e1.record(streams[g])
                    ev[g] = (e0, e1)
                for g in (0, 1):
                    streams[g].synchronize()
            res = {g: window * size / (ev[g][0].elapsed_time(ev[g][1]) * 1e-3) / 1e9 for g in (0, 1)}
            print(json.dumps({"size": size, "window": window, "mode": mode, "gpu0_GBps": res[0],
                              "gpu1_GBps": res[1]}),
                  flush=True)


if __name__ == "__main__":
    main()
