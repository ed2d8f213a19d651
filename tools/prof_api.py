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
