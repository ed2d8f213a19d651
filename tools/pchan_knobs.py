"""Sweep the persistent channel's copy shapes for the 64-message window
bandwidth; one JSON line each.
usage: pchan_knobs.py SEND_CTAS SEND_THREADS SIZES [RECV_THREADS]
(comma lists; HX_CHAN_SEND_CTAS, HX_CHAN_SEND_THREADS, HX_CHAN_RECV_THREADS)"""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_12416_b200.osu import channel_bandwidth  # noqa: E402


def arg(i, dflt):
    return sys.argv[i].split(",") if len(sys.argv) > i else dflt


ctas = arg(1, ["32"])
threads = arg(2, ["256"])
sizes = [int(x) for x in arg(3, [str(1 << 20), str(4 << 20), str(16 << 20)])]
recv_threads = arg(4, ["256"])
for c, t, rt in itertools.product(ctas, threads, recv_threads):
    os.environ.update(HX_CHAN_SEND_CTAS=c, HX_CHAN_SEND_THREADS=t, HX_CHAN_RECV_THREADS=rt)
    for size in sizes:
        r = channel_bandwidth(size, window=64, iters=5, depth=8)
        print(json.dumps({"send_ctas": c, "threads": t, "recv_threads": rt, "size": size,
                          "gbps": round(r["value_gbps"], 1), "ok": r["verified"]}), flush=True)
