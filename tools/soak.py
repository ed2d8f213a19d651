"""Soak test of the multi-GPU exchange protocols: many iterations of the
fused exchange (eager steps, CUDA-graph replays, persistent runs mixed) on
random fields, compared bit for bit with one block on one GPU (no exchange)
after the same number of iterations. Catches rare ordering races that the
short parity tests would miss.

    python tools/soak.py [--iters 3000] [--scale 1] [--sweep-exchange]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(dims, pes, device_of, schedule, policy, seed=None, init=None, sweepx=False):
    """Run ``schedule`` on a fresh engine whose initial interior is random
    (``seed``: per-block N(0,1)) or ``init`` (a global array); returns the
    initial and the final global interior."""
    import torch
    from paper_2102_12416_b200.halo import HaloJacobi

    eng = HaloJacobi(dims, pes, device_of=device_of, exchange="fused", policy=policy,
                     timeout_s=20)
    eng.xy_from_interior = sweepx
    if init is None:
        eng.fill_random(seed)
        eng.synchronize()
        init = eng.assemble()
    else:
        b = eng.blocks[0]
        with torch.cuda.device(b.device):
            b.fields[b.cur][1:-1, 1:-1, 1:-1].copy_(torch.from_numpy(init))
        torch.cuda.synchronize(b.device)
    for how, n in schedule:
        {"eager": eng.run, "graph": eng.run_graph, "persistent": eng.run_persistent}[how](n)
    eng.check_errors()
    out = eng.assemble()
    eng.close()
    return init, out, eng.grid


def main():
    import numpy as np
    import torch

    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=3000)
    ap.add_argument("--scale", type=int, default=1, help="multiply every extent")
    ap.add_argument("--sweep-exchange", action="store_true",
                    help="every face inside the interior sweep (HaloJacobi.xy_from_interior)")
    a = ap.parse_args()
    two = torch.cuda.device_count() >= 2
    dev2 = (lambda r: r % 2) if two else (lambda r: 0)
    n = a.iters
    cases = [
        ("x split, 2 blocks", (256, 128, 128), 2, "b200", [("eager", 5), ("graph", n), ("eager", 3)]),
        ("(2,2,1), 4 blocks", (128, 128, 64), 4, "b200", [("graph", n // 2), ("eager", 7), ("graph", n // 2)]),
        ("z split (1,2,2), 4 blocks", (64, 128, 128), 4, "reference",
         [("eager", 3), ("persistent", n // 2), ("graph", n // 2), ("persistent", 11)]),
        ("8 blocks (2,2,2)", (96, 96, 96), 8, "reference", [("persistent", n), ("eager", 2)]),
    ]
    ok = True
    for name, dims, pes, policy, sched in cases:
        dims = tuple(a.scale * e for e in dims)
        t = time.perf_counter()
        init, got, grid = run(dims, pes, dev2, sched, policy, seed=11, sweepx=a.sweep_exchange)
        iters = sum(k for _, k in sched)
        _, want, _ = run(dims, 1, lambda r: 0, [("eager", iters)], policy, init=init)
        same = got.tobytes() == want.tobytes()
        ok &= same
        print(json.dumps({"case": name, "grid": grid, "iters": iters, "gpus": 2 if two else 1,
                          "bitexact": same, "s": round(time.perf_counter() - t, 1)}), flush=True)
    print(json.dumps({"all_bitexact": ok}))
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
