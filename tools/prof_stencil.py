"""Time the stencil kernel alone (CUDA events) — the ncu target and the
chunk / variant sweep used to tune it.

    python tools/prof_stencil.py [--n 1536] [--reps 5] [--chunks 0,64,128] [--variant 0]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2102_12416_b200 import _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1536)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--chunks", default="0")
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--residual", action="store_true")
    ap.add_argument("--shape", default=None, help="bx,by,bz (default n,n,n)")
    ap.add_argument("--device", type=int, default=0)
    args = ap.parse_args()
    torch.cuda.set_device(args.device)
    _lib.call("hx_set_device", args.device)
    n = args.n
    bx, by, bz = (int(x) for x in args.shape.split(",")) if args.shape else (n, n, n)
    shape = (bx + 2, by + 2, bz + 2)
    a = torch.empty(shape, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    s = torch.cuda.current_stream().cuda_stream
    for t in (a, b):
        _lib.call("hx_init_block", t.data_ptr(), bx, by, bz, 1, 1.0, 0.0, 0.0, s)
    res = torch.zeros(1, dtype=torch.int64, device="cuda")
    rp = res.data_ptr() if args.residual else None
    _lib.raw("hx_stencil_set_variant")(args.variant)
    out = []
    for chunk in [int(c) for c in args.chunks.split(",")]:
        _lib.raw("hx_stencil_set_chunk")(chunk)
        for _ in range(2):
            _lib.call("hx_stencil", a.data_ptr(), b.data_ptr(), bx, by, bz, rp, s)
            a, b = b, a
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            _lib.call("hx_stencil", a.data_ptr(), b.data_ptr(), bx, by, bz, rp, s)
            a, b = b, a
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        gbs = 16 * bx * by * bz / (ms * 1e-3) / 1e9
        out.append({"shape": [bx, by, bz], "chunk": chunk, "variant": _lib.raw("hx_stencil_last_variant")(),
                    "ms": ms, "alg_GBps": gbs, "frac_of_6538.9": gbs / 6538.9})
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
