"""Rehearse the 8-GPU weak-scaling layout on 4 GPUs: 3072^3 in 8 blocks,
two per GPU, in one process (blocks sharing a GPU share its streams, so no
kernel ever waits on one launched after it).

Runs the B200 policy's (4,2,1) with the fused exchange and the reference
policy's (2,2,2), times a few steps of each, and checks decomposition
invariance: the two runs' fields must agree bit for bit at a few thousand
sampled global points (a 3072^3 single-array oracle does not fit one GPU).

    python tools/emulate8.py [--n 3072] [--iters 6]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def fill_global(eng, dims):
    """Overwrite every block (ghost layers too) with a smooth field defined
    on global coordinates, so boundary data crosses every block face from
    the first iteration and both decompositions start identical."""
    import torch

    from paper_2102_12416_b200.jacobi3d import _block_coords

    bx, by, bz = (dims[a] // eng.grid[a] for a in range(3))
    for r, b in eng.blocks.items():
        ix, iy, iz = _block_coords(r, eng.grid)
        dev = b.fields[0].device
        gj = torch.arange(iy * by - 1, iy * by + by + 1, device=dev, dtype=torch.float64)
        gk = torch.arange(iz * bz - 1, iz * bz + bz + 1, device=dev, dtype=torch.float64)
        yz = 0.5 * torch.cos(0.0021 * gj)[:, None] + 0.25 * torch.sin(0.0033 * gk)[None, :]
        with torch.cuda.device(dev):
            for li in range(bx + 2):
                v = yz + float(torch.sin(torch.tensor(0.0017 * (ix * bx + li - 1))))
                for f in b.fields:
                    f[li].copy_(v)
    for d in range(torch.cuda.device_count()):
        torch.cuda.synchronize(d)


def main():
    import numpy as np
    import torch

    from paper_2102_12416_b200.halo import HaloJacobi
    from paper_2102_12416_b200.jacobi3d import _block_coords

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=3072)
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--points", type=int, default=4096)
    args = ap.parse_args()
    n, ngpu = args.n, torch.cuda.device_count()
    dims = (n, n, n)
    rng = np.random.default_rng(5)
    pts = rng.integers(0, n, size=(args.points, 3))
    # half of the points sit on block faces of either layout
    faces = [0, 1, n // 4 - 1, n // 4, n // 2 - 1, n // 2, 3 * n // 4 - 1, 3 * n // 4, n - 1]
    q = args.points // 6
    for a in range(3):
        pts[a * q:(a + 1) * q, a] = rng.choice(faces, q)
    out = {"dims": dims, "gpus": ngpu}
    samples = {}
    for policy, exchange in (("b200", "fused"), ("reference", "fused")):
        eng = HaloJacobi(dims, 8, device_of=lambda r: r % ngpu, policy=policy, exchange=exchange,
                         timeout_s=60)
        fill_global(eng, dims)  # same global field (ghosts included) for both layouts
        eng.step()
        eng.synchronize()
        s0 = {d: torch.cuda.Event(enable_timing=True) for d in eng.streams}
        s1 = {d: torch.cuda.Event(enable_timing=True) for d in eng.streams}
        for d, s in eng.streams.items():
            s0[d].record(s)
        for _ in range(args.iters - 1):
            eng.step()
        for d, s in eng.streams.items():
            s1[d].record(s)
        eng.check_errors()
        ms = max(s0[d].elapsed_time(s1[d]) for d in eng.streams) / (args.iters - 1)
        vals = np.empty(len(pts))
        bx, by, bz = (dims[a] // eng.grid[a] for a in range(3))
        for r, b in eng.blocks.items():
            ix, iy, iz = _block_coords(r, eng.grid)
            sel = ((pts[:, 0] // bx == ix) & (pts[:, 1] // by == iy) & (pts[:, 2] // bz == iz))
            if sel.any():
                f = b.fields[b.cur]
                loc = torch.as_tensor(pts[sel] - [ix * bx, iy * by, iz * bz] + 1, device=f.device)
                vals[sel] = f[loc[:, 0], loc[:, 1], loc[:, 2]].cpu().numpy()
        samples[policy] = vals
        out[policy] = {"grid": list(eng.grid), "ms_per_step_8_blocks_on_%d_gpus" % ngpu: ms,
                       "glups": 8 * bx * by * bz / (ms * 1e-3) / 1e9,
                       "nonzero_samples": int((vals != 0).sum())}
        print(json.dumps(out[policy]), flush=True)
        eng.close()
        del eng
        torch.cuda.empty_cache()
    out["decomposition_invariant"] = bool(np.array_equal(samples["b200"], samples["reference"]))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
