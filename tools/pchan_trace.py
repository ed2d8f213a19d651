"""Per-message timeline of the persistent channel (hx_chan_trace stamps):
a 64-message window and a ping-pong, each replayed from CUDA graphs, at one
size. Prints median per-message intervals in microseconds."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2102_12416_b200 import _lib  # noqa: E402
from paper_2102_12416_b200.osu import _graph_pair, _replay_pair  # noqa: E402
from paper_2102_12416_b200.pchannel import PersistentChannel  # noqa: E402


def traces():
    t = [[torch.zeros(2048, dtype=torch.int64, device=f"cuda:{g}") for _ in (0, 1)] for g in (0, 1)]
    for g in (0, 1):
        _lib.call("hx_chan_trace", g, t[g][0].data_ptr(), t[g][1].data_ptr())
    return t


def show(name, a, n, cols):
    a = a[:n * 8].reshape(n, 8).astype(np.int64)
    print(f"-- {name}")
    base = a[:, 0:1]
    rel = (a - base) / 1e3
    for i, c in enumerate(cols):
        if i:
            print(f"   {c:>28}: median {np.median(rel[:, i]):8.2f} us after entry")
    ent = np.diff(a[:, 0]) / 1e3
    print(f"   {'entry-to-entry':>28}: median {np.median(ent):8.2f} us")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1048576")
    ap.add_argument("--window", type=int, default=64)
    ap.add_argument("--slot", type=int, default=0, help="0: as large as the message")
    ap.add_argument("--pingpong", action="store_true", help="latency timeline instead")
    a = ap.parse_args()
    for size in [int(x) for x in a.sizes.split(",")]:
        if a.pingpong:
            pingpong_timeline(size)
        else:
            run(a, size)


def run(a, size):
    ch = PersistentChannel(0, 1, slot_bytes=a.slot or max(size, 16), depth=8)
    src = torch.randint(0, 255, (size,), dtype=torch.uint8, device="cuda:0")
    sink = torch.zeros(size, dtype=torch.uint8, device="cuda:1")
    ack_tx = torch.zeros(8, dtype=torch.uint8, device="cuda:1")
    ack_rx = torch.zeros(8, dtype=torch.uint8, device="cuda:0")

    def sender(s):
        for _ in range(a.window):
            ch.send(0, src, size, stream=s)
        ch.recv(0, ack_rx, 8, stream=s)

    def drainer(s):
        for _ in range(a.window):
            ch.recv(1, sink, size, stream=s)
        ch.send(1, ack_tx, 8, stream=s)

    t = traces()  # before capture: the stamps' buffers are kernel arguments
    graphs, streams = _graph_pair((0, 1), sender, drainer)
    _replay_pair((0, 1), graphs, streams, 2)
    ms = _replay_pair((0, 1), graphs, streams, 1)
    ch.check()
    print(f"window of {a.window} x {size} B (slot {a.slot or size} B): {ms * 1e3:.1f} us, "
          f"{a.window * size / (ms * 1e6):.1f} GB/s")
    # message indices wrap in the 256 ring; show the last window only
    n = a.window
    send = t[0][0].cpu().numpy()
    recv = t[1][1].cpu().numpy()
    k0 = (ch.counters[0][0] - n) & 255
    idx = [(k0 + i) & 255 for i in range(n)]
    sa = np.concatenate([send[j * 8:(j + 1) * 8] for j in idx])
    ra = np.concatenate([recv[j * 8:(j + 1) * 8] for j in idx])
    show("send (GPU 0)", sa, n, ["entry", "claimed", "published", "pulled", "done"])
    show("recv (GPU 1)", ra, n, ["entry", "pred done", "header seen", "copied"])
    # cross-GPU (clocks roughly aligned): header seen - published
    sp = sa.reshape(n, 8)[:, 2]
    rh = ra.reshape(n, 8)[:, 2]
    print(f"   recv header seen - send published (cross-GPU clocks): median "
          f"{np.median((rh - sp) / 1e3):.2f} us")
    _lib.call("hx_chan_trace", 0, None, None)
    _lib.call("hx_chan_trace", 1, None, None)



def pingpong_timeline(size: int = 8, iters: int = 64):
    """Ping-pong (as osu.channel_latency) with stamps: for a few round
    trips, each GPU's channel events in time order, microseconds from that
    GPU's first event of the round trip (clocks are per GPU)."""
    ch = PersistentChannel(0, 1, slot_bytes=64 << 10, depth=2)
    src = torch.randint(0, 255, (max(size, 1),), dtype=torch.uint8, device="cuda:0")
    back = torch.zeros(max(size, 1), dtype=torch.uint8, device="cuda:0")
    mid = torch.zeros(max(size, 1), dtype=torch.uint8, device="cuda:1")
    t = traces()

    def leader(s):
        for _ in range(iters):
            ch.send(0, src, size, stream=s)
            ch.recv(0, back, size, stream=s)

    def echo(s):
        for _ in range(iters):
            ch.recv(1, mid, size, stream=s)
            ch.send(1, mid, size, stream=s)

    graphs, streams = _graph_pair((0, 1), leader, echo)
    _replay_pair((0, 1), graphs, streams, 1)
    ms = _replay_pair((0, 1), graphs, streams, 1)
    ch.check()
    print(f"ping-pong {size} B: {ms * 1e3 / iters / 2:.2f} us one-way")
    s0, r0 = (x.cpu().numpy()[:2048].reshape(256, 8) for x in t[0])
    s1, r1 = (x.cpu().numpy()[:2048].reshape(256, 8) for x in t[1])
    names_s = ["entry", "claimed", "published", "pulled", "done"]
    names_r = ["entry", "pred done", "header seen", "copied"]
    for k in range(2 * iters - 4, 2 * iters - 1):  # direction 0 message k, direction 1 message k
        kk = k & 255
        for gpu, (snd, rcv, who) in enumerate(((s0, r0, "leader"), (s1, r1, "echo"))):
            ev = [(snd[kk][i], f"send {names_s[i]}") for i in range(5) if snd[kk][i]]
            ev += [(rcv[kk][i], f"recv {names_r[i]}") for i in range(4) if rcv[kk][i]]
            ev.sort()
            base = ev[0][0]
            print(f"  k={k} {who}: " + ", ".join(f"{n} {(v - base) / 1e3:.2f}" for v, n in ev))


if __name__ == "__main__":
    main()
