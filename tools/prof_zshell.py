"""The fused exchange on a z split: one block's boundary kernel alone
(flags pre-satisfied, back-to-back launches) and full fused steps, with the
z faces produced by the interior sweep (default), by the boundary kernel
through the contiguous slots, or through the ghost columns.

    python tools/prof_zshell.py [--n 1536] [--two-gpus]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2102_12416_b200.halo import HaloJacobi

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1536)
    ap.add_argument("--two-gpus", action="store_true")
    a = ap.parse_args()
    n = a.n
    dev = (lambda r: r) if a.two_gpus else (lambda r: 0)
    eng = HaloJacobi((n, n, 2 * n), 2, device_of=dev, exchange="fused", policy="reference")
    assert eng.grid == (1, 1, 2), eng.grid
    out = {"n": n, "grid": eng.grid, "gpus": 2 if a.two_gpus else 1}
    for mode in ("interior", "slots", "ghost_columns"):
        zs = mode != "ghost_columns"
        eng.z_slots = zs
        eng.z_from_interior = mode == "interior"
        eng.xy_from_interior = mode == "interior"  # else the sweep would carry the z faces anyway
        eng.reset()
        for _ in range(3):
            eng.step()
        eng.synchronize()
        ms = eng.time_shell_alone(reps=7)
        s0 = eng.stream_of(eng.blocks[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        timing = {}
        e0.record(s0)
        for _ in range(10):
            eng.step(timing=timing)
        e1.record(s0)
        eng.synchronize()
        eng.check_errors()
        conc = [x.elapsed_time(y) for x, y in timing["exchange"]]
        out[mode] = {
            "shell_alone_ms": ms, "face_bytes": 8 * n * n,
            "nvlink_gbs": 8 * n * n / (ms * 1e-3) / 1e9,
            "step_ms": e0.elapsed_time(e1) / 10, "shell_concurrent_ms": sum(conc) / len(conc)}
    print(json.dumps(out), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
