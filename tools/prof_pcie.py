"""Host <-> device copy rates on the GPU box: pinned D2H / H2D of 256 MB,
and first-touch vs warm memset of an 8 GB numpy array (one thread) — the
ingredients of run_jacobi's field read-back.

    python tools/prof_pcie.py
"""
import torch, time, json, os
x = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for pin in (True,):
    h = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=pin)
    for _ in range(3): h.copy_(x, non_blocking=True); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20): h.copy_(x, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(json.dumps({"d2h_GBps": 20 * (256 << 20) / dt / 1e9}))
    t = time.perf_counter()
    for _ in range(20): x.copy_(h, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(json.dumps({"h2d_GBps": 20 * (256 << 20) / dt / 1e9}))
# two staging buffers alternated with two streams
import numpy as np
out = np.empty(8 << 30, dtype=np.uint8)
t = time.perf_counter()
out[:] = 0
print(json.dumps({"first_touch_1thread_GBps": (8 << 30) / (time.perf_counter() - t) / 1e9}))
t = time.perf_counter()
out[:] = 1
print(json.dumps({"memset_warm_1thread_GBps": (8 << 30) / (time.perf_counter() - t) / 1e9}))
