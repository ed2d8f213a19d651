"""Sweep the persistent channel's copy grids (HX_CHAN_SEND_CTAS,
HX_CHAN_RECV_CTAS) for the 64-message window bandwidth; one JSON line each.
usage: pchan_knobs.py SEND_LIST RECV_LIST SIZE_LIST"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_12416_b200.osu import channel_bandwidth  # noqa: E402

sends = sys.argv[1].split(",") if len(sys.argv) > 1 else ["32", "64", "128"]
recvs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["296"]
sizes = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1 << 20, 4 << 20, 16 << 20]
for sc in sends:
    os.environ["HX_CHAN_SEND_CTAS"] = sc
    for rc in recvs:
        os.environ["HX_CHAN_RECV_CTAS"] = rc
        for size in sizes:
            r = channel_bandwidth(size, window=64, iters=5, depth=8)
            print(json.dumps({"send_ctas": sc, "recv_ctas": rc, "size": size,
                              "gbps": round(r["value_gbps"], 1), "ok": r["verified"]}), flush=True)
