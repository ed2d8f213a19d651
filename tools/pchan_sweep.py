"""Persistent-channel window bandwidth and ping-pong latency vs message size
(one JSON line per point), e.g. under HX_CHAN_SEND_CTAS / depth sweeps."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="65536,262144,1048576,4194304,16777216")
    ap.add_argument("--depths", default="8")
    ap.add_argument("--lat", action="store_true")
    a = ap.parse_args()
    from paper_2102_12416_b200.osu import channel_bandwidth, channel_latency
    for size in [int(x) for x in a.sizes.split(",")]:
        for depth in [int(x) for x in a.depths.split(",")]:
            r = channel_bandwidth(size, window=64, iters=5, depth=depth)
            r["depth"] = depth
            print(json.dumps(r), flush=True)
        if a.lat:
            print(json.dumps(channel_latency(size, iters=200, warmup=20)), flush=True)


if __name__ == "__main__":
    main()
