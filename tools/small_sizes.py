"""Per-iteration time of small Jacobi problems through the public entry
points (launch/host-bound regime): run_jacobi(mode=channel-persistent) and
the reference-mode driver, 64^3 x 100 (config C1) at 1 and 8 PEs."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2102_12416_b200.jacobi3d import run_jacobi

    for mode in ("channel-persistent", "channel-device", "messaging-device"):
        for pes in (1, 8):
            run_jacobi(dims=(64, 64, 64), iters=5, mode=mode, pes=pes)
            t = time.perf_counter()
            r = run_jacobi(dims=(64, 64, 64), iters=100, mode=mode, pes=pes)
            wall = time.perf_counter() - t
            print(json.dumps({"mode": mode, "pes": pes, "ms_per_iter": r["total_ns"] / 100 / 1e6,
                              "wall_s": round(wall, 3)}), flush=True)


if __name__ == "__main__":
    main()
