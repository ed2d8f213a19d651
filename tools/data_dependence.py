"""Is HBM streaming speed data-dependent on B200?

Times (CUDA events, best and median of N) on 1536^3 fp64 fields:
  * the stencil (hx_stencil, TMA kernel) on zeros, on the hot wall, on a
    constant 1.0 field and on N(0,1) data;
  * a plain device copy (torch copy_) of 8 GiB of zeros, of 1.0 and of
    N(0,1) data — the roofline denominator measured on the same inputs.
Prints one JSON line per case.
"""

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2102_12416_b200 import _lib  # noqa: E402


def timeit(fn, reps=7):
    ts = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts = ts[1:]
    return min(ts), statistics.median(ts)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1536
    torch.cuda.set_device(0)
    shape = (n + 2,) * 3
    cur = torch.empty(shape, dtype=torch.float64, device="cuda")
    nxt = torch.empty_like(cur)
    s = torch.cuda.current_stream().cuda_stream
    _lib.call("hx_set_device", 0)
    alg = 16 * n ** 3

    def sweep():
        _lib.call("hx_stencil", cur.data_ptr(), nxt.data_ptr(), n, n, n, None, s)

    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    cases = {
        "zeros": lambda t: t.zero_(),
        "hotwall": lambda t: (t.zero_(), t[0].fill_(1.0)),
        "ones": lambda t: t.fill_(1.0),
        "normal": lambda t: t.normal_(generator=g),
        "uniform01": lambda t: t.uniform_(generator=g),
    }
    for name, fill in cases.items():
        fill(cur)
        fill(nxt)
        torch.cuda.synchronize()
        best, med = timeit(sweep)
        print(json.dumps({"kernel": "stencil", "data": name, "n": n, "best_ms": best,
                          "median_ms": med, "gbs_best": alg / best / 1e6}), flush=True)
    del cur, nxt
    torch.cuda.empty_cache()
    a = torch.empty(1 << 30, dtype=torch.float64, device="cuda")  # 8 GiB
    b = torch.empty_like(a)
    for name, fill in cases.items():
        if name == "hotwall":
            continue
        fill(a)
        b.zero_()
        torch.cuda.synchronize()
        best, med = timeit(lambda: b.copy_(a))
        print(json.dumps({"kernel": "torch copy_", "data": name, "bytes": 2 * a.numel() * 8,
                          "best_ms": best, "median_ms": med,
                          "gbs_best": 2 * a.numel() * 8 / best / 1e6}), flush=True)




def power_probe(n=1536, sweeps=300):
    """Power draw, SM clock and throttle reasons sampled every 20 ms while
    the stencil sweeps zeros, then N(0,1) data (one JSON line per case)."""
    import subprocess
    import time

    torch.cuda.set_device(0)
    shape = (n + 2,) * 3
    cur = torch.empty(shape, dtype=torch.float64, device="cuda")
    nxt = torch.empty_like(cur)
    s = torch.cuda.current_stream().cuda_stream
    _lib.call("hx_set_device", 0)
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    a8 = b8 = None
    for name, fill in (("zeros", lambda t: t.zero_()), ("normal", lambda t: t.normal_(generator=g)),
                       ("zeros-again", lambda t: t.zero_()), ("copy-zeros", None),
                       ("copy-normal", None)):
        if fill is None:  # plain device copies of 2 x 8 GiB on the same data
            if a8 is None:
                del cur, nxt
                torch.cuda.empty_cache()
                a8 = torch.empty(1 << 30, dtype=torch.float64, device="cuda")
                b8 = torch.empty_like(a8)
            (a8.zero_() if name == "copy-zeros" else a8.normal_(generator=g))
            b8.copy_(a8)
            torch.cuda.synchronize()
        else:
            fill(cur)
            fill(nxt)
            torch.cuda.synchronize()
        p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=power.draw,clocks.sm,clocks.mem,"
                              "clocks_event_reasons.active,temperature.gpu,temperature.memory",
                              "--format=csv,noheader,nounits", "-lms", "20"],
                             stdout=subprocess.PIPE, text=True)
        time.sleep(0.5)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(sweeps):
            if fill is None:
                b8.copy_(a8)
            else:
                _lib.call("hx_stencil", cur.data_ptr(), nxt.data_ptr(), n, n, n, None, s)
                cur, nxt = nxt, cur
        b.record()
        b.synchronize()
        p.terminate()
        rows = [r.split(", ") for r in p.communicate()[0].strip().splitlines()]
        rows = [r for r in rows if len(r) == 6][5:]
        def col(i):
            out = []
            for r in rows:
                try:
                    out.append(float(r[i]))
                except ValueError:
                    pass
            return out
        pw, sm = col(0), col(1)
        reasons = sorted({r[3] for r in rows})
        ms = a.elapsed_time(b) / sweeps
        alg = (2 * a8.numel() * 8) if fill is None else 16 * n ** 3
        print(json.dumps({"case": name, "ms_per_sweep": ms, "gbs": alg / ms / 1e6,
                          "power_w_median": statistics.median(pw) if pw else None,
                          "power_w_max": max(pw) if pw else None,
                          "sm_mhz_median": statistics.median(sm) if sm else None,
                          "sm_mhz_min": min(sm) if sm else None,
                          "reasons_bitmasks": reasons,
                          "temp_gpu_max": max(col(4)) if col(4) else None,
                          "temp_mem_max": max(col(5)) if col(5) else None,
                          "samples": len(rows)}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "power":
        power_probe(int(sys.argv[1]))
    else:
        main()
