"""Phases of run_jacobi's end-to-end time at the bench size (the bench's
e2e_api leg): engine set-up (field allocation, init, peer set-up), the
iterations, the wait for the host pages' first touch, and the read-back.

    python tools/prof_e2e_api.py [--n 1536] [--iters 20]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2102_12416_b200 import halo

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1536)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--threads", type=int, default=16)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    for rep in range(a.reps):  # rep 0 pays the CUDA context and module loads
        once(a, rep)


def once(a, rep):
    import torch
    from paper_2102_12416_b200 import halo

    dims = (a.n,) * 3
    t = [time.perf_counter()]
    out, futs = halo.prefault_host(dims, a.threads)
    t.append(time.perf_counter())
    eng = halo.HaloJacobi(dims, 1, device_of=lambda r: 0, exchange="fused", policy="reference")
    eng.synchronize()
    t.append(time.perf_counter())
    eng.run(a.iters)
    eng.synchronize()
    t.append(time.perf_counter())
    for f in futs:
        f.result()
    t.append(time.perf_counter())
    eng.assemble(out)
    t.append(time.perf_counter())
    eng.close()
    del out
    torch.cuda.empty_cache()
    names = ["prefault_submit", "engine_setup", "iterations", "prefault_wait", "readback"]
    print(json.dumps({"rep": rep, "n": a.n, "iters": a.iters, "threads": a.threads,
                      **{k: round(t[i + 1] - t[i], 3) for i, k in enumerate(names)},
                      "total": round(t[-1] - t[0], 3)}), flush=True)


if __name__ == "__main__":
    main()
