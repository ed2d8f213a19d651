"""Standalone face pack / unpack throughput per direction (CUDA events).

Algorithmic bytes: 16 per face cell (8 read + 8 written). x and y faces are
rows of bz contiguous doubles; z faces are one double per (bz+2)-stride
row, so their field side touches one 32-byte sector per 8 bytes.

    python tools/prof_faces.py [--n 1536] [--reps 20]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2102_12416_b200 import _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1536)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    n = args.n
    _lib.call("hx_preload")  # (applies HX_L2_FETCH, if set)
    f = torch.randn((n + 2,) * 3, dtype=torch.float64, device="cuda")
    slot = torch.empty(n * n, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    rows = []
    for d in range(6):
        for fn in ("hx_pack", "hx_unpack"):
            for _ in range(3):
                _lib.call(fn, f.data_ptr(), n, n, n, d, slot.data_ptr(), s)
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.reps):
                _lib.call(fn, f.data_ptr(), n, n, n, d, slot.data_ptr(), s)
            z.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(z) / args.reps * 1e3
            rows.append({"dir": d, "op": fn[3:], "us": round(us, 2),
                         "alg_GBps": round(16 * n * n / (us * 1e-6) / 1e9, 1)})
            print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
