"""Compare one full sweep against the interior + shell split for a block
with the given neighbour sides; report the first mismatching box."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    from paper_2102_12416_b200 import _lib
    from paper_2102_12416_b200.halo import HaloBlock, HaloJacobi

    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="768,768,384")
    ap.add_argument("--sides", default="5")
    args = ap.parse_args()
    bx, by, bz = (int(x) for x in args.shape.split(","))
    b = HaloBlock((bx, by, bz), (1, 1, 1), 0, 0)
    b.neighbors = [0 if d in {int(x) for x in args.sides.split(",")} else None for d in range(6)]
    g = torch.Generator(device="cuda").manual_seed(7)
    cur = torch.randn((bx + 2, by + 2, bz + 2), dtype=torch.float64, device="cuda", generator=g)
    ref = torch.zeros_like(cur)
    out = torch.zeros_like(cur)
    s = torch.cuda.current_stream().cuda_stream
    _lib.call("hx_stencil", cur.data_ptr(), ref.data_ptr(), bx, by, bz, None, s)
    inner, shells = HaloJacobi.boxes(None, b)
    for box in [inner] + shells:
        _lib.call("hx_stencil_box", cur.data_ptr(), out.data_ptr(), bx, by, bz, *box, None, s)
        var = _lib.raw("hx_stencil_last_variant")()
        o = torch.zeros_like(cur)
        _lib.call("hx_stencil_box", cur.data_ptr(), o.data_ptr(), bx, by, bz, *box, None, s)
        i0, i1, j0, j1, k0, k1 = box
        a = o[i0:i1, j0:j1, k0:k1]
        r = ref[i0:i1, j0:j1, k0:k1]
        bad = (a != r).nonzero()
        print(box, "variant", var, "mismatches", bad.shape[0],
              (bad[:3] + torch.tensor([i0, j0, k0], device="cuda")).tolist() if bad.shape[0] else "")
    diff = (out[1:-1, 1:-1, 1:-1] != ref[1:-1, 1:-1, 1:-1]).sum().item()
    print("split vs full mismatching cells:", diff)


if __name__ == "__main__":
    main()
