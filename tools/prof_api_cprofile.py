"""cProfile of the API-level 8-byte Channel ping-pong (host time per call)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_12416_b200.osu import measure_latency  # noqa: E402

measure_latency("charm-channel", "device", 8, iters=100, warmup=5)
pr = cProfile.Profile()
pr.enable()
measure_latency("charm-channel", "device", 8, iters=1000, warmup=5)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
