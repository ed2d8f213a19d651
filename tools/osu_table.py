"""Render a tools/run_osu.py JSON as the markdown table kept in profiles/.

    python tools/osu_table.py gpurun_out/osu.json > profiles/rN_osu_2gpu_table.md
"""

import json
import sys


def main():
    d = json.load(open(sys.argv[1]))
    rows = d["rows"]
    sizes = sorted({r["size"] for r in rows})

    def pick(size, **kw):
        for r in rows:
            if r["size"] == size and all(r.get(k) == v for k, v in kw.items()):
                return r
        return None

    def lat(r):
        return f"{r['value_ns'] / 1000:.2f}" if r else "—"

    def bw(r):
        return f"{r['value_gbps']:.1f}" if r else "—"

    cols = [
        ("chan dev lat (µs)", lambda s: lat(pick(s, benchmark="latency", api="charm-channel", mode="device"))),
        ("msg dev lat", lambda s: lat(pick(s, benchmark="latency", api="charm-messaging", mode="device"))),
        ("mpi dev lat", lambda s: lat(pick(s, benchmark="latency", api="mpi", mode="device"))),
        ("chan host-staged lat", lambda s: lat(pick(s, benchmark="latency", api="charm-channel", mode="host"))),
        ("persistent chan lat (µs)", lambda s: lat(pick(s, benchmark="channel-latency"))),
        ("persistent chan bw (GB/s)", lambda s: bw(pick(s, benchmark="channel-bandwidth",
                                                        slot_bytes=65536))),
        ("persistent chan bw, message-sized slots", lambda s: bw(
            pick(s, benchmark="channel-bandwidth", protocol="slot", slot_bytes=max(s, 16)))
            if s > 65536 else "="),
        ("chan dev bw (GB/s)", lambda s: bw(pick(s, benchmark="bandwidth", api="charm-channel", mode="device"))),
        ("msg dev bw", lambda s: bw(pick(s, benchmark="bandwidth", api="charm-messaging", mode="device"))),
        ("device lat (µs)", lambda s: lat(pick(s, benchmark="device-latency"))),
        ("device bw CE", lambda s: bw(pick(s, benchmark="device-bandwidth", engine="ce"))),
        ("device bw pull (window kernel)", lambda s: bw(pick(s, benchmark="device-bandwidth", engine="sm-pull-window"))),
        ("device bw push (window kernel)", lambda s: bw(pick(s, benchmark="device-bandwidth", engine="sm-window"))),
    ]
    print("| size (B) | " + " | ".join(c for c, _ in cols) + " |")
    print("|---" * (len(cols) + 1) + "|")
    for s in sizes:
        print(f"| {s} | " + " | ".join(f(s) for _, f in cols) + " |")
    print()
    print("verified:", all(r.get("verified", True) for r in rows))


if __name__ == "__main__":
    main()
