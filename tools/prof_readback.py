"""Field read-back (the tail of run_jacobi's end-to-end time): a 1536^3
block's interior into a fresh numpy array, by HaloJacobi.interior_into with
HX_READBACK_THREADS host threads (the first call includes the pinned
staging allocation). Page-locking the output chunk by chunk
(cudaHostRegister) and copying into it directly was measured at 2.7 GB/s,
10x slower than staging, and dropped.

    python tools/prof_readback.py [--n 1536]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_2102_12416_b200.halo import HaloJacobi

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1536)
    a = ap.parse_args()
    n = a.n
    eng = HaloJacobi((n, n, n), 1, device_of=lambda r: 0, exchange="fused")
    eng.fill_random(1)
    eng.synchronize()
    print(json.dumps({"cores": len(os.sched_getaffinity(0)), "bytes": 8 * n ** 3}), flush=True)
    for th in (16, 8, 32):
        os.environ["HX_READBACK_THREADS"] = str(th)
        for rep in range(2):
            t = time.perf_counter()
            out = np.empty((n, n, n))
            eng.interior_into(0, out)
            dt = time.perf_counter() - t
            print(json.dumps({"how": "staging", "threads": th, "rep": rep, "s": round(dt, 3),
                              "GBps": round(8 * n ** 3 / dt / 1e9, 1)}), flush=True)
            del out
    eng.close()


if __name__ == "__main__":
    main()
