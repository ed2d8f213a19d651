"""Time the overlap split's kernels for one block with neighbours on the
given sides (default: +x, +y, +z — a rank of the 8-GPU (2,2,2) grid).

    python tools/prof_shell.py [--n 1536] [--sides 1,3,5]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2102_12416_b200 import _lib
    from paper_2102_12416_b200.halo import HaloBlock, HaloJacobi

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1536)
    ap.add_argument("--sides", default="1,3,5")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--shape", default=None, help="bx,by,bz (default n,n,n)")
    args = ap.parse_args()
    n = args.n
    bx_, by_, bz_ = (int(x) for x in args.shape.split(",")) if args.shape else (n, n, n)
    b = HaloBlock((bx_, by_, bz_), (1, 1, 1), 0, 0)
    b.neighbors = [0 if d in {int(x) for x in args.sides.split(",")} else None for d in range(6)]
    s = torch.cuda.current_stream().cuda_stream
    for f in b.fields:
        _lib.call("hx_init_block", f.data_ptr(), bx_, by_, bz_, 1, 1.0, 0.0, 0.0, s)
    inner, shells = HaloJacobi.boxes(None, b)
    out = {}
    for name, boxes in [("full", [(1, bx_ + 1, 1, by_ + 1, 1, bz_ + 1)]), ("interior", [inner])] + \
            [(f"shell{q}", [bx]) for q, bx in enumerate(shells)]:
        for _ in range(2):
            for bx in boxes:
                _lib.call("hx_stencil_box", b.fields[0].data_ptr(), b.fields[1].data_ptr(), bx_, by_,
                          bz_, *bx, None, s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            for bx in boxes:
                _lib.call("hx_stencil_box", b.fields[0].data_ptr(), b.fields[1].data_ptr(), bx_, by_,
                          bz_, *bx, None, s)
        e1.record()
        torch.cuda.synchronize()
        out[name] = {"box": boxes[0], "ms": e0.elapsed_time(e1) / args.reps,
                     "variant": _lib.raw("hx_stencil_last_variant")()}
        print(name, json.dumps(out[name]), flush=True)


if __name__ == "__main__":
    main()
