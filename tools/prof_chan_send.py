"""One-direction bulk sends for an ncu capture of chan_send_kernel: four
4 MiB sends into message-sized slots (depth 8), so no send waits for a
receive (kernels may be serialised by the profiler); the receives run
after the sends have completed.

    ncu --set full -k regex:chan_send -s 1 -c 1 python tools/prof_chan_send.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_12416_b200.pchannel import PersistentChannel  # noqa: E402

size, n = 4 << 20, 4
ch = PersistentChannel(0, 1, slot_bytes=size, depth=8, timeout_s=30)
src = torch.randint(0, 255, (size,), dtype=torch.uint8, device="cuda:0")
sink = torch.zeros(size, dtype=torch.uint8, device="cuda:1")
s0, s1 = torch.cuda.Stream(device=0), torch.cuda.Stream(device=1)
for _ in range(n):
    ch.send(0, src, size, stream=s0)
s0.synchronize()
for _ in range(n):
    ch.recv(1, sink, size, stream=s1)
s1.synchronize()
ch.check()
assert torch.equal(sink.cpu(), src.cpu())
print("ok", ch.counters)
