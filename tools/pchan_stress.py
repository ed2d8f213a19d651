"""Randomised persistent-channel schedules with separate send and receive
streams per endpoint; reports which configurations complete (diagnostics
for tests/test_gpu_multi.py::test_persistent_channel_random_schedules)."""
import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_12416_b200.pchannel import PersistentChannel  # noqa: E402


def run(seed, dirs=(0, 1), choices=(1, 8, 1000, 8192, 8193, 30000, 40000, 40001, 200000, 1 << 20),
        trunc=True, depth=1, n=30, fills=True, slot=40000):
    rng = np.random.default_rng(seed)
    ch = PersistentChannel(0, 1, slot_bytes=slot, depth=depth, timeout_s=2)
    send_s = [torch.cuda.Stream(device=e) for e in (0, 1)]
    recv_s = [torch.cuda.Stream(device=e) for e in (0, 1)]
    sizes = {e: [int(rng.choice(choices)) for _ in range(n)] for e in dirs}
    caps = {e: [int(rng.choice([s, s, s, max(1, s // 3), s + 7])) if trunc else s for s in sizes[e]]
            for e in dirs}
    shared = [torch.zeros(1 << 20, dtype=torch.uint8, device=f"cuda:{e}") for e in (0, 1)]
    srcs = {e: [torch.randint(0, 255, (s,), dtype=torch.uint8, device=f"cuda:{e}") for s in sizes[e]]
            for e in dirs}
    sinks = {e: [torch.zeros(max(c, 1), dtype=torch.uint8, device=f"cuda:{1 - e}") for c in caps[e]]
             for e in dirs}
    if os.environ.get("PCHAN_WARM_FILL", "1") == "1":  # see include/hx.h hx_preload
        for e in (0, 1):
            shared[e].fill_(1)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    for e in dirs:
        for k, size in enumerate(sizes[e]):
            src = srcs[e][k]
            if fills and rng.random() < 0.3:
                with torch.cuda.stream(send_s[e]):
                    shared[e].fill_(k)
                src = shared[e]
            ch.send(e, src, size, stream=send_s[e])
    for e in dirs:
        for k in range(n):
            ch.recv(1 - e, sinks[e][k], caps[e][k], stream=recv_s[1 - e])
    for s in send_s + recv_s:
        s.synchronize()
    try:
        ch.check()
        return "ok", ch.counters
    except RuntimeError:
        return "TIMEOUT", ch.counters


if __name__ == "__main__":
    for name, kw in [("both", {}), ("dir0", {"dirs": (0,)}), ("notrunc", {"trunc": False}),
                     ("nopull", {"choices": (1, 8, 1000, 8192, 8193, 30000, 40000)}),
                     ("pullonly", {"choices": (40001, 200000, 1 << 20)}),
                     ("nofills", {"fills": False}), ("depth3", {"depth": 3}),
                     ("dir0_nopull", {"dirs": (0,), "choices": (1, 8, 1000, 8192, 8193, 30000, 40000)}),
                     ("dir0_pull", {"dirs": (0,), "choices": (40001, 200000, 1 << 20)})]:
        print(name, run(0, **kw), flush=True)
