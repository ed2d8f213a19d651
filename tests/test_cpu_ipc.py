"""World-size-2 gloo test of the process-per-GPU runtime backend ("ipc") on
CPU, host payloads only (the CUDA IPC data plane is covered on the GPU by
tests/test_gpu_ipc_runtime.py).

Two processes, four PEs (PE p in process p % 2). Checked:
* the TCP mesh hello (tag-layout digest) and envelope frames: a token
  passed around a ring of chares that alternates between the processes;
* futures fulfilled across processes (FutureRef frames) and callbacks;
* the Channel API with host payloads below and above the eager threshold,
  kth send meets kth receive, truncation reported as a status;
* the MPI facade (isend/irecv of numpy buffers, ANY_TAG) across processes,
  results gathered with the collective rank_result;
* run(until=...) followed by the drain, twice on one runtime.
"""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _app():
    """Chare classes, defined identically in every process (SPMD)."""
    import numpy as np  # noqa: F401

    from paper_2102_12416_b200.completion import Callback
    from paper_2102_12416_b200.runtime import Chare, entry

    class Ring(Chare):
        def __init__(self, n, laps):
            self.n, self.laps = n, laps
            self.hops = []
            self.answers = []
            self.finished = False
            self.ids = None

        @entry
        def start(self, ids):
            self.ids = ids
            if self.index == 0:
                self.proxy(ids[1]).token(1, [0])
            # a future answered by a chare in the other process
            other = ids[(self.index + 1) % self.n]
            fut = self.future()
            self.proxy(other).ask(fut.ref, self.index)
            v = yield fut
            self.answers.append(v)
            # a callback into this chare, fired by the remote chare
            self.proxy(other).call_back(Callback(self.id, "got", (self.index,)))

        @entry
        def ask(self, ref, x):
            self.fulfill(ref, 100 * x + self.index)

        @entry
        def call_back(self, cb):
            self.fulfill(cb, "cb-from-%d" % self.index)

        @entry
        def got(self, mine, value):
            self.answers.append((mine, value))
            self._maybe_done()

        @entry
        def token(self, hop, path):
            self.hops.append(hop)
            path = path + [self.index]
            if hop + 1 < self.laps * self.n:
                self.proxy(self.ids[(self.index + 1) % self.n]).token(hop + 1, path)
            else:
                for i in self.ids:
                    self.proxy(i).stop_ring(path)
            self._maybe_done()

        @entry
        def stop_ring(self, path):
            self.path = path
            self._maybe_done()

        def _maybe_done(self):
            if len(self.answers) == 2 and getattr(self, "path", None) is not None:
                self.finished = True

    class ChanPeer(Chare):
        def __init__(self, sizes):
            self.sizes = sizes
            self.got = []
            self.finished = False

        @entry
        def run(self, peer_id, leader):
            ch = self.channel(7, peer_id)
            for k, n in enumerate(self.sizes):
                payload = bytes((11 * i + n + k) & 0xFF for i in range(n))
                if leader:
                    ch.send(payload)
                    sink = bytearray(n)
                    comp = yield ch.recv(sink)
                    self.got.append((comp.status, comp.length, bytes(sink) == payload))
                else:
                    sink = bytearray(n)
                    comp = yield ch.recv(sink)
                    self.got.append((comp.status, comp.length, bytes(sink) == payload))
                    ch.send(bytes(sink))
            # truncation: a 64-byte payload into a 16-byte sink
            if leader:
                ch.send(b"x" * 64)
            else:
                comp = yield ch.recv(bytearray(16))
                self.got.append((comp.status, comp.length, None))
            self.finished = True

    return Ring, ChanPeer


def _worker(rank, world, port, out):
    import sys

    sys.path.insert(0, ROOT)
    import numpy as np

    from paper_2102_12416_b200.config import RuntimeConfig
    from paper_2102_12416_b200.mpi import ANY_TAG, mpi_run, rank_result
    from paper_2102_12416_b200.runtime import Runtime

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    Ring, ChanPeer = _app()
    cfg = RuntimeConfig(workers=4, backend="ipc")
    res = {"rank": rank}

    # ring + futures + callbacks
    rt = Runtime(cfg)
    rt.register(Ring)
    ids = rt.create(Ring, 4, args=(4, 3), placement=[0, 1, 2, 3])
    for cid in ids:
        rt.launch(cid, "start", list(ids))
    rt.start()
    mine = {cid.element: rt.pe(cid.home_pe).chares[(cid.collection, cid.element)]
            for cid in ids if rt.is_local(cid.home_pe)}
    rt.run(until=lambda: all(c.finished for c in mine.values()), timeout_s=60)
    res["ring"] = {e: (c.hops, c.answers, c.path) for e, c in mine.items()}
    rt.close()

    # channel API, host payloads (eager and rendezvous sizes), twice on one runtime
    rt = Runtime(cfg)
    rt.register(ChanPeer)
    sizes = [1, 8, 1000, 8192, 8193, 100_000]
    ids = rt.create(ChanPeer, 2, args=(sizes,), placement=[0, 1])
    rt.launch(ids[0], "run", ids[1], True)
    rt.launch(ids[1], "run", ids[0], False)
    rt.start()
    mine = {cid.element: rt.pe(cid.home_pe).chares[(0, cid.element)]
            for cid in ids if rt.is_local(cid.home_pe)}
    rt.run(until=lambda: all(c.finished for c in mine.values()), timeout_s=60)
    res["chan"] = {e: c.got for e, c in mine.items()}
    rt.close()

    # MPI facade: ring exchange of numpy buffers, ANY_TAG receive
    def main(comm):
        n = comm.size
        right, left = (comm.rank + 1) % n, (comm.rank - 1) % n
        send = np.arange(32, dtype=np.float64) + comm.rank
        recv = np.zeros(32)
        reqs = [comm.isend(send, right, tag=5), comm.irecv(recv, left, tag=ANY_TAG)]
        yield from comm.waitall(reqs)
        return float(recv[0]), float(recv.sum())

    rt = mpi_run(main, 4, cfg=cfg)
    res["mpi"] = [rank_result(rt, r) for r in range(4)]
    rt.close()

    everyone = [None] * world
    dist.all_gather_object(everyone, res)
    if rank == 0:
        out.put(everyone)
    dist.barrier()
    dist.destroy_process_group()


def test_ipc_backend_two_processes_host_payloads():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    everyone = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ring = {}
    for e in everyone:
        ring.update(e["ring"])
    assert sorted(ring) == [0, 1, 2, 3]
    hops = sorted(h for e in ring.values() for h in e[0])
    assert hops == list(range(1, 12))  # 3 laps of 4, every hop crossed a process boundary
    for e, (h, answers, path) in ring.items():
        assert path == [0, 1, 2, 3] * 3
        assert answers[0] == 100 * e + (e + 1) % 4  # future fulfilled by the next chare
        assert answers[1] == (e, "cb-from-%d" % ((e + 1) % 4))
    chan = {}
    for e in everyone:
        chan.update(e["chan"])
    sizes = [1, 8, 1000, 8192, 8193, 100_000]
    for side in (0, 1):
        got = chan[side]
        assert [g[:2] for g in got[:len(sizes)]] == [("ok", n) for n in sizes]
        assert all(g[2] for g in got[:len(sizes)])
    assert chan[1][-1][:2] == ("truncated", 64)
    mpi = everyone[0]["mpi"]
    assert mpi == everyone[1]["mpi"]
    for r, (first, total) in enumerate(mpi):
        left = (r - 1) % 4
        assert first == left and total == sum(range(32)) + 32 * left


@pytest.mark.parametrize("bad", [True])
def test_ipc_backend_needs_a_process_group(bad):
    import sys

    sys.path.insert(0, ROOT)
    from paper_2102_12416_b200.config import RuntimeConfig
    from paper_2102_12416_b200.transport import StartupError, TransportGroup

    if dist.is_initialized():
        pytest.skip("a process group is already initialised")
    with pytest.raises(StartupError):
        TransportGroup(RuntimeConfig(workers=2, backend="ipc"), backend="ipc")


def _mesh_worker(rank, world, port, digest, out):
    import sys

    sys.path.insert(0, ROOT)
    from paper_2102_12416_b200.wire import LayoutMismatchError, Mesh

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mesh = Mesh(rank, world, digest, dist, timeout_s=30)
    except LayoutMismatchError as e:
        out.put((rank, "mismatch", str(e)))
        dist.destroy_process_group()
        return
    sizes = [0, 1, 7, 1 << 16, (1 << 20) + 3, 3 << 20]  # across the 1 MiB receive chunks
    for k, n in enumerate(sizes):
        mesh.send(1 - rank, 4, (rank, k, bytes([(k + rank) % 251]) * n))
    got = []
    import time

    t0 = time.monotonic()
    while len(got) < len(sizes) and time.monotonic() - t0 < 60:
        got += mesh.poll()
    while not mesh.flushed:
        mesh.poll()
    ok = [p == 1 - rank and kind == 4 and b[0] == 1 - rank and b[1] == k and
          b[2] == bytes([(k + 1 - rank) % 251]) * sizes[k]
          for k, (p, kind, b) in enumerate(got)]
    dist.barrier()
    mesh.close()
    out.put((rank, "frames", (len(got), all(ok), mesh.frames_sent, mesh.frames_received)))
    dist.destroy_process_group()


@pytest.mark.parametrize("same_digest", [True, False])
def test_wire_mesh_frames_and_digest(same_digest):
    """wire.Mesh between two processes: frames of 0 B to 3 MiB (across the
    1 MiB receive chunks) arrive complete and in order both ways; a tag
    layout digest mismatch in the hello raises LayoutMismatchError
    (cl/transport.py:77-91)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    digests = [0x1234, 0x1234 if same_digest else 0x9999]
    procs = [ctx.Process(target=_mesh_worker, args=(r, 2, port, digests[r], q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    if same_digest:
        for rank, kind, val in res:
            assert kind == "frames" and val[0] == 6 and val[1], (rank, val)
            assert val[2] == 6 and val[3] == 6
    else:
        assert all(kind == "mismatch" for _, kind, _ in res)
