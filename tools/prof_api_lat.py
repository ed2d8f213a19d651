"""Where the API-level 8-byte ping-pong spends its time: wall time per
one-way message, time inside libhx C calls (per entry point), and how many
times the scheduler polls CUDA events per message.

    python tools/prof_api_lat.py [--size 8] [--iters 2000] [--api charm-channel]
"""

import argparse
import collections
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=8)
    ap.add_argument("--iters", type=int, default=2000)
    ap.add_argument("--api", default="charm-channel")
    ap.add_argument("--bw", action="store_true", help="window bandwidth (64 x size) instead")
    args = ap.parse_args()

    from paper_2102_12416_b200 import _lib
    from paper_2102_12416_b200.osu import measure_latency

    measure_latency(args.api, "device", args.size, iters=50, warmup=5)  # warm pools
    spent = collections.Counter()
    calls = collections.Counter()
    real_call, real_raw = _lib.call, _lib.raw

    def call(fn, *a):
        t = time.perf_counter_ns()
        try:
            return real_call(fn, *a)
        finally:
            spent[fn] += time.perf_counter_ns() - t
            calls[fn] += 1

    def raw(fn):
        f = real_raw(fn)

        def wrapped(*a):
            t = time.perf_counter_ns()
            try:
                return f(*a)
            finally:
                spent[fn] += time.perf_counter_ns() - t
                calls[fn] += 1
        return wrapped

    _lib.call, _lib.raw = call, raw
    t0 = time.perf_counter_ns()
    if args.bw:
        from paper_2102_12416_b200.osu import measure_bandwidth

        r = measure_bandwidth(args.api, "device", args.size, window=64, iters=args.iters, warmup=1)
        msgs = 64 * (args.iters + 1)
    else:
        r = measure_latency(args.api, "device", args.size, iters=args.iters, warmup=5)
        msgs = 2 * (args.iters + 5)
    wall = time.perf_counter_ns() - t0
    _lib.call, _lib.raw = real_call, real_raw
    if args.bw:
        print(json.dumps({"api": args.api, "size": args.size, "window_gbps": r["value_gbps"],
                          "host_us_per_msg": wall / msgs / 1000,
                          "c_calls_us_per_msg": {k: round(spent[k] / msgs / 1000, 3) for k in spent},
                          "c_calls_per_msg": {k: round(calls[k] / msgs, 2) for k in calls},
                          "c_total_us_per_msg": round(sum(spent.values()) / msgs / 1000, 3)}),
              flush=True)
        return
    out = {"api": args.api, "size": args.size, "one_way_us": r["value_ns"] / 1000,
           "host_us_per_msg": wall / msgs / 1000,
           "c_calls_us_per_msg": {k: round(spent[k] / msgs / 1000, 3) for k in spent},
           "c_calls_per_msg": {k: round(calls[k] / msgs, 2) for k in calls}}
    out["c_total_us_per_msg"] = round(sum(spent.values()) / msgs / 1000, 3)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
