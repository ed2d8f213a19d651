"""Small blocks: µs per fused iteration for 64^3-class grids, eager steps vs
CUDA-graph replay vs the persistent kernel (one launch per block).

    python tools/prof_small.py [--dims 64,64,64] [--pes 2] [--iters 200] [--two-gpus]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2102_12416_b200.halo import HaloJacobi

    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="64,64,64")
    ap.add_argument("--pes", type=int, default=2)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--two-gpus", action="store_true")
    a = ap.parse_args()
    dims = tuple(int(x) for x in a.dims.split(","))
    dev = (lambda r: r % 2) if a.two_gpus else (lambda r: 0)
    out = {"dims": dims, "pes": a.pes, "gpus": 2 if a.two_gpus else 1}
    for how in ("eager", "graph", "persistent"):
        eng = HaloJacobi(dims, a.pes, device_of=dev, exchange="fused")
        run = {"eager": eng.run, "graph": eng.run_graph, "persistent": eng.run_persistent}[how]
        run(20)
        eng.synchronize()
        t = time.perf_counter()
        run(a.iters)
        eng.synchronize()
        out[how + "_us_per_iter"] = (time.perf_counter() - t) / a.iters * 1e6
        eng.check_errors()
        eng.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
