"""cProfile of the API-level OSU ping-pong (drop-in runtime path): where the
host time of one message goes.

    python tools/prof_api_cprofile.py [api] [size] [iters]
"""

import cProfile
import io
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    api = sys.argv[1] if len(sys.argv) > 1 else "charm-channel"
    size = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
    from paper_2102_12416_b200.osu import measure_bandwidth, measure_latency

    measure_latency(api, "device", size, iters=50, warmup=5)
    r = measure_latency(api, "device", size, iters=iters, warmup=5)
    print(f"{api} {size} B one-way {r['value_ns'] / 1e3:.2f} us (unprofiled)", flush=True)
    bw = measure_bandwidth(api, "device", 4 << 20, window=64, iters=3)
    print(f"{api} 4 MiB window bandwidth {bw['value_gbps']:.1f} GB/s (unprofiled)", flush=True)
    pr = cProfile.Profile()
    pr.enable()
    measure_latency(api, "device", size, iters=iters, warmup=5)
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(28)
    print(s.getvalue())


if __name__ == "__main__":
    main()
