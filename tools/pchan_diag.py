"""Diagnose a slow / stuck persistent-channel window: runs window tests in
one process with short device timeouts and prints per-replay times."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_12416_b200.osu import _graph_pair, _replay_pair  # noqa: E402
from paper_2102_12416_b200.pchannel import PersistentChannel  # noqa: E402


def window(size, depth=8, window=64, reps=3):
    t0 = time.time()
    ch = PersistentChannel(0, 1, slot_bytes=max(size, 16), depth=depth, timeout_s=0.2)
    src = torch.randint(0, 255, (size,), dtype=torch.uint8, device="cuda:0")
    sink = torch.zeros(size, dtype=torch.uint8, device="cuda:1")
    ack_tx = torch.zeros(8, dtype=torch.uint8, device="cuda:1")
    ack_rx = torch.zeros(8, dtype=torch.uint8, device="cuda:0")

    def sender(s):
        for _ in range(window):
            ch.send(0, src, size, stream=s)
        ch.recv(0, ack_rx, 8, stream=s)

    def drainer(s):
        for _ in range(window):
            ch.recv(1, sink, size, stream=s)
        ch.send(1, ack_tx, 8, stream=s)

    graphs, streams = _graph_pair((0, 1), sender, drainer)
    print(f"  size {size}: setup {time.time() - t0:.2f} s", flush=True)
    for r in range(reps):
        t1 = time.time()
        ms = _replay_pair((0, 1), graphs, streams, 1)
        try:
            ch.check()
            st = "ok"
        except RuntimeError as e:
            st = str(e)
        print(f"  rep {r}: {ms:.3f} ms device, {time.time() - t1:.2f} s wall, "
              f"{window * size / (ms * 1e6):.1f} GB/s, {st}, counters {ch.counters}", flush=True)
        if st != "ok":
            break
    same = torch.equal(sink.cpu(), src.cpu())
    print(f"  payload equal: {same}", flush=True)




def traced(size, depth=8):
    """One window with hx_chan_trace stamps; prints the first 12 messages'
    raw stamps (us from the first send entry; 0 = never written)."""
    from paper_2102_12416_b200 import _lib
    t = [[torch.zeros(2048 + 256 * 320, dtype=torch.int64, device=f"cuda:{g}") for _ in (0, 1)]
         for g in (0, 1)]
    for g in (0, 1):
        _lib.call("hx_chan_trace", g, t[g][0].data_ptr(), t[g][1].data_ptr())
    window(size, depth=depth, reps=1)
    torch.cuda.synchronize(0)
    claims = t[0][0].cpu().numpy()[2048:].reshape(256, 320)
    mixed = 0
    for row in range(256):
        v = claims[row][claims[row] > 0]
        if v.size and (v.min() != v.max()):
            mixed += 1
            if mixed <= 5:
                print(f"  launch serial {row}: CTAs claimed indices {sorted(set((v - 1).tolist()))[:8]}")
    print(f"  launches with CTAs on different indices: {mixed}")
    s = t[0][0].cpu().numpy()[:2048].reshape(256, 8)
    r = t[1][1].cpu().numpy()[:2048].reshape(256, 8)
    base = s[0, 0]
    for k in range(12):
        fs = " ".join(f"{(v - base) / 1e3:9.1f}" if v else "        -" for v in s[k][:5])
        fr = " ".join(f"{(v - base) / 1e3:9.1f}" if v else "        -" for v in r[k][:4])
        print(f"  k={k:2d} send[entry claim pub pull done] {fs} | recv[entry pred hdr copied] {fr}")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "trace":
        traced(int(sys.argv[1]))
    else:
        for s in [int(x) for x in sys.argv[1].split(",")]:
            window(s)
