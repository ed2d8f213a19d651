"""The fused shell kernel alone at 1536^2 (2 blocks on 2 GPUs): with and
without its NVLink stores, to see what bounds it."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2102_12416_b200 import _lib
    from paper_2102_12416_b200.halo import NDIRS, HaloJacobi

    n = 1536
    eng = HaloJacobi((2 * n, n, n), 2, device_of=lambda r: r, exchange="fused", timeout_s=20)
    eng.run(2)
    eng.synchronize()
    b = eng.blocks[0]
    c = eng.comm[b.device]
    _, shells = eng.boxes(b)
    flat = (ctypes.c_int * (6 * len(shells)))(*[v for box in shells for v in box])
    nxt = b.cur ^ 1
    for label, remote in (("with NVLink stores", [b.peer_fields[d][nxt] if d in b.nbr_dirs else None
                                                   for d in range(NDIRS)]),
                          ("local only", [None] * 6)):
        times = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            _lib.call("hx_set_device", b.device)
            e0.record(c)
            _lib.call("hx_shell_put", b.field_ptr(), b.field_ptr(nxt), b.bx, b.by, b.bz,
                      len(shells), flat, _lib.ptr_array(remote), _lib.ptr_array([None] * 6), 0,
                      _lib.ptr_array([None] * 6), 0, b.counters_ptr + 4, eng.timeout_ns,
                      b.err_ptr, None, None, c.cuda_stream)
            e1.record(c)
            c.synchronize()
            times.append(e0.elapsed_time(e1))
        print(json.dumps({"variant": label, "ms": sorted(times)[5]}), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
