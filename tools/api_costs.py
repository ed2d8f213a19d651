"""CPU cost (µs per call) of the CUDA operations on the per-message path,
measured on two GPUs: copy-engine vs SM-kernel peer copy of small payloads,
event record, cross-device stream wait, event query.

    python tools/api_costs.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2102_12416_b200 import _lib

    _lib.call("hx_enable_peer", 0, 1)
    _lib.call("hx_enable_peer", 1, 0)
    a = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda:0")
    b = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda:1")
    s1 = torch.cuda.Stream(device=1)
    s0 = torch.cuda.Stream(device=0)
    h1, h0 = s1.cuda_stream, s0.cuda_stream
    ev = _lib.ctypes.c_void_p()
    _lib.call("hx_set_device", 0)
    _lib.call("hx_event_create", _lib.ctypes.byref(ev), 0)
    out = {}

    def bench(name, fn, n=2000):
        for _ in range(50):
            fn()
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        t = time.perf_counter_ns()
        for _ in range(n):
            fn()
        out[name] = round((time.perf_counter_ns() - t) / n / 1000, 3)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)

    for size in (8, 4096, 65536):
        bench(f"memcpy_p2p_{size}", lambda: _lib.call("hx_memcpy", b.data_ptr(), a.data_ptr(), size, h1))
        _lib.call("hx_set_device", 1)  # a kernel launches on the current device
        bench(f"copy_sm_p2p_{size}", lambda: _lib.call("hx_copy_sm", b.data_ptr(), a.data_ptr(), size, h1))
        bench(f"set_device+copy_sm_{size}", lambda: (_lib.call("hx_set_device", 1),
                                                     _lib.call("hx_copy_sm", b.data_ptr(), a.data_ptr(), size, h1)))
        _lib.call("hx_set_device", 0)
    bench("event_record", lambda: _lib.call("hx_event_record", ev.value, h0))
    bench("stream_wait_cross_dev", lambda: _lib.call("hx_stream_wait_event", h1, ev.value))
    bench("stream_wait_same_dev", lambda: _lib.call("hx_stream_wait_event", h0, ev.value))
    bench("event_query", lambda: _lib.raw("hx_event_query")(ev.value))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
