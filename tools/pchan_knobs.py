"""Sweep the persistent channel's launch shapes for the 64-message window
bandwidth; one JSON line per (setting, size). The library reads its knobs
once per process, so every setting runs in its own subprocess.

usage: pchan_knobs.py SEND_CTAS SEND_THREADS SIZES [RECV_CTAS [FENCE [SLOT]]]
(comma lists: HX_CHAN_SEND_CTAS, HX_CHAN_SEND_THREADS, message sizes,
HX_CHAN_RECV_CTAS, HX_CHAN_DIAG_FENCE, slot bytes — 0 = as large as the
message; smaller: larger messages are pulled)"""
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def arg(i, dflt):
    return sys.argv[i].split(",") if len(sys.argv) > i else dflt


def child(sizes):
    sys.path.insert(0, ROOT)
    from paper_2102_12416_b200.osu import channel_bandwidth
    for size in sizes:
        slot = int(os.environ.get("PCHAN_SLOT", "0")) or None  # 0: slots as large as the message
        r = channel_bandwidth(size, window=64, iters=5, depth=8, slot_bytes=slot)
        print(json.dumps({k: os.environ.get(k) for k in KNOBS} |
                         {"size": size, "gbps": round(r["value_gbps"], 1), "ok": r["verified"]}),
              flush=True)


KNOBS = ("HX_CHAN_SEND_CTAS", "HX_CHAN_SEND_THREADS", "HX_CHAN_RECV_CTAS", "HX_CHAN_DIAG_FENCE",
         "PCHAN_SLOT")

if __name__ == "__main__":
    if sys.argv[1:2] == ["--child"]:
        child([int(x) for x in sys.argv[2].split(",")])
        sys.exit(0)
    sizes = arg(3, [str(1 << 20), str(4 << 20), str(16 << 20)])
    for setting in itertools.product(arg(1, ["64"]), arg(2, ["512"]), arg(4, ["0"]), arg(5, ["0"]),
                                     arg(6, ["0"])):
        env = dict(os.environ, **dict(zip(KNOBS, setting)))
        subprocess.run([sys.executable, __file__, "--child", ",".join(sizes)], env=env, check=True)
