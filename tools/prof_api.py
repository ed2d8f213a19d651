"""cProfile of the API-level ping-pong (where the host time goes)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_12416_b200.osu import measure_latency  # noqa: E402

for api, mode in (("charm-channel", "device"), ("charm-channel", "host"), ("charm-messaging", "device")):
    r = measure_latency(api, mode, 8, iters=300, warmup=20)
    print(api, mode, "one-way us", r["value_ns"] / 1000, flush=True)
pr = cProfile.Profile()
pr.enable()
measure_latency("charm-channel", "device", 8, iters=300, warmup=5)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

from paper_2102_12416_b200.osu import measure_bandwidth  # noqa: E402

for api in ("charm-channel", "charm-messaging"):
    r = measure_bandwidth(api, "device", 4 << 20, window=64, iters=3, warmup=1)
    print(api, "bw GB/s", r["value_gbps"], flush=True)
pr = cProfile.Profile()
pr.enable()
measure_bandwidth("charm-channel", "device", 4 << 20, window=64, iters=3, warmup=1)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
