"""Tagged point-to-point transport with a B200 device data plane.

Mirror of cl/transport.py:1-636 (loopback backend): non-blocking tagged
sends and receives with masked matching — a receive (tag, mask) matches a
frame when ``frame.tag & mask == tag & mask``; arrivals match the earliest
posted receive, posts match the earliest unexpected frame, FIFO per
endpoint pair; eager (<= eager_threshold) vs rendezvous semantics.

What is B200-native (the only place device bytes move):
  * eager device payloads are snapshotted at send time into a device bounce
    buffer by a stream-ordered D2D copy (replaces read_wire at
    cl/transport.py:284-289), so the send completes immediately and the
    source is reusable, exactly as in the reference;
  * a matched rendezvous moves the payload with ONE direct device-to-device
    copy — local HBM or NVLink P2P — from the sender's region into the
    receiver's sink (replaces the PULL/PAYLOAD byte copies at
    cl/transport.py:449-465 and the write_wire at 430-432). It is enqueued
    on the sink owner's stream behind an event recorded on the sender's
    stream at send time, so no host staging and no extra copy;
  * host sinks / host payloads use pinned staging + cudaMemcpyAsync;
  * completions fire from progress() once the CUDA event recorded after the
    copy has completed (cl/transport.py:342-365), and ``idle`` reports
    in-flight GPU copies so the runtime never quiesces early
    (cl/transport.py:372-381, cl/runtime.py:530-542).
Backends: "loopback" — every worker in this process (cl/transport.py's
loopback); "ipc" — one process per GPU (the paper's setup),
the B200 form of the reference's TCP backend (cl/transport.py:469-586): the
workers of other processes are reached over a TCP mesh (wire.Mesh) that
carries only host frames — eager host payloads, envelopes, and for a device
payload a rendezvous frame holding the source allocation's CUDA IPC handle
and offset (the "IPC handles carried in the frames" of SURVEY §8f row 4).
The receiver opens the handle once (cached), copies straight from the
sender's HBM into its sink on its own stream, and acknowledges with a FIN
frame that completes the send. Device payloads never touch a socket or host
memory. Eager device payloads are snapshotted into a transport-owned bounce
buffer first (the send completes at once); rendezvous frames leave once the
source's stream has reached the send (a CUDA event, polled).
"""

from __future__ import annotations

import ctypes
import weakref
from collections import Counter, deque

import numpy as np
import torch

from . import _lib
from .completion import OK, TRANSPORT_ERROR, TRUNCATED, Completion, deliver
from .config import RuntimeConfig
from .device import DeviceBuffer, DeviceRegion, DeviceSpace, as_region
from .tags import EAGER, FULL_MASK, TagLayout
from .timebase import WallClock
from .wire import Mesh

# ipc backend frame kinds (wire.Mesh)
K_EAGER, K_RTS, K_FIN, K_RUNTIME = 1, 2, 3, 4


class TransportError(RuntimeError):
    pass


class StartupError(TransportError):
    pass


FRAME_EAGER = 0
FRAME_RTS = 1
_NAMES = {FRAME_EAGER: "eager", FRAME_RTS: "rts"}
_TX_KEY = {k: f"tx_{v}" for k, v in _NAMES.items()}
_RX_KEY = {k: f"rx_{v}" for k, v in _NAMES.items()}


class Frame:
    """One tagged message in flight. ``source`` is bytes (host) or a
    DeviceRegion (a bounce snapshot for eager, the sender's region for
    rendezvous); ``ready`` is the CUDA event after which it may be read."""

    __slots__ = ("kind", "tag", "length", "source", "ready", "src", "send_completion",
                 "keepalive", "seq")

    def __init__(self, kind, tag, length, source, ready, src, send_completion=None, keepalive=None):
        self.kind = kind
        self.tag = tag
        self.length = length
        self.source = source
        self.ready = ready
        self.src = src
        self.send_completion = send_completion
        self.keepalive = keepalive
        self.seq = 0

    @property
    def payload(self):
        return self.source if isinstance(self.source, bytes) else None

    def __repr__(self):
        return f"Frame({_NAMES[self.kind]}, tag=0x{self.tag:016x}, len={self.length}, src={self.src})"


class ReceiveRequest:
    __slots__ = ("tag", "mask", "capacity", "sink", "completion", "seq", "wildcard", "done")

    def __init__(self, tag, mask, capacity, sink, completion, seq, wildcard=False):
        self.tag = tag
        self.mask = mask
        self.capacity = capacity
        self.sink = sink
        self.completion = completion
        self.seq = seq
        self.wildcard = wildcard
        self.done = False

    def matches(self, frame_tag: int) -> bool:
        return (frame_tag & self.mask) == (self.tag & self.mask)


class Endpoint:
    __slots__ = ("worker", "peer", "failed")

    def __init__(self, worker, peer):
        self.worker = worker
        self.peer = peer
        self.failed = False


class _Inflight:
    """A GPU copy whose completion event gates one or more callbacks."""

    __slots__ = ("event", "fn")

    def __init__(self, event, fn):
        self.event = event
        self.fn = fn


def _is_device(x) -> bool:
    return isinstance(x, (DeviceBuffer, DeviceRegion))


class Worker:
    """Matching engine + device data plane for one PE (cl/transport.py:169-598)."""

    def __init__(self, group: "TransportGroup", worker_id: int):
        self.group = group
        self.id = worker_id
        self.cfg = group.cfg
        self.layout = group.layout
        self.clock = group.clocks[worker_id]
        self.posted: list[ReceiveRequest] = []
        self.unexpected: list[Frame] = []
        self.inbound: deque = deque()
        self.endpoints: dict[int, Endpoint] = {}
        self.stats: Counter = Counter()
        self.eager_handler = None
        self.eager_inbox: deque = deque()
        self._fired: deque = deque()
        self._inflight: list[_Inflight] = []
        self._post_seq = 0
        self._arrival_seq = 0
        self.hold = None
        self._held: list = []
        # ipc backend: sends to other processes in order (each waits for its
        # ready event), and rendezvous sends awaiting the receiver's FIN
        self._outbox: deque = deque()
        self._rdv: dict = {}

    # ------------------------------------------------------------- plumbing

    @property
    def space(self) -> DeviceSpace:
        return self.group.device_space

    @property
    def gpu(self) -> int:
        return self.group.gpu_of(self.id)

    @property
    def stream(self) -> torch.cuda.Stream:
        return self.space.stream_of(self.id)

    def connect(self, peer: int, address: str | None = None) -> Endpoint:
        ep = self.endpoints.get(peer)
        if ep is None:
            if peer not in self.group.workers:
                raise TransportError(f"no worker {peer} in this group")
            ep = self.endpoints[peer] = Endpoint(self, peer)
        return ep

    def _fire(self, handle, comp: Completion) -> None:
        self._fired.append((handle, comp))

    def _after(self, event, fn) -> None:
        self._inflight.append(_Inflight(event.acquire(), fn))

    # ---------------------------------------------------------------- sends

    def tag_send(self, ep: Endpoint, tag: int, payload, completion=None, length=None) -> None:
        """Non-blocking tagged send (cl/transport.py:258-295)."""
        if not 0 <= tag <= FULL_MASK:
            raise ValueError(f"tag 0x{tag:x} outside 64 bits")
        if ep.failed:
            self._fire(completion, Completion(status=TRANSPORT_ERROR, tag=tag,
                                              error=f"endpoint to {ep.peer} failed"))
            return
        if _is_device(payload):
            source = as_region(payload, length)
            nbytes = source.size
        else:
            data = bytes(payload)
            if length is not None:
                if length > len(data):
                    raise ValueError(f"length {length} exceeds payload of {len(data)}")
                data = data[:length]
            source, nbytes = data, len(data)
        if nbytes > self.cfg.max_message_bytes:
            raise ValueError(f"payload of {nbytes} bytes exceeds max message size "
                             f"{self.cfg.max_message_bytes}")
        peer = self.group.workers[ep.peer]
        if isinstance(peer, _RemoteWorker):
            self._send_remote(peer, tag, source, nbytes, completion)
            return
        if nbytes <= self.cfg.eager_threshold:
            ready, keep = None, None
            if isinstance(source, DeviceRegion):
                ready = self.space.record(source.buffer.owner)
                direct = Frame(FRAME_EAGER, tag, nbytes, source, ready, self.id)
                if peer._match_now(direct):
                    # the receive was already posted: one direct HBM/NVLink
                    # copy, and the sender's stream is ordered behind it, so
                    # the source is reusable at once (eager semantics)
                    self.stats["tx_eager"] += 1
                    self.stats["tx_direct"] += 1
                    self.stats["sends"] += 1
                    self._fire(completion, Completion(status=OK, length=nbytes, tag=tag))
                    return
                ready.release()
                source, ready, keep = self._snapshot(source)
            frame = Frame(FRAME_EAGER, tag, nbytes, source, ready, self.id, keepalive=keep)
            self._fire(completion, Completion(status=OK, length=nbytes, tag=tag))
        else:
            ready = None
            if isinstance(source, DeviceRegion):
                ready = self.space.record(source.buffer.owner)
            frame = Frame(FRAME_RTS, tag, nbytes, source, ready, self.id, send_completion=completion)
            if isinstance(source, DeviceRegion) and peer._match_now(frame):
                self.stats["tx_rts"] += 1
                self.stats["tx_direct"] += 1
                self.stats["sends"] += 1
                return
        self.stats[_TX_KEY[frame.kind]] += 1
        self.stats["sends"] += 1
        peer.inbound.append(frame)

    def _send_remote(self, peer, tag, source, nbytes, completion) -> None:
        """ipc backend: a send to a worker of another process. Host bytes go
        as an eager frame (the send completes at once); a device payload goes
        as a rendezvous frame carrying the source's IPC handle — eager-sized
        ones from a bounce snapshot (send complete at once, the bounce comes
        back with the FIN), larger ones straight from the source region (the
        FIN completes the send). Frames leave in send order."""
        self.stats["sends"] += 1
        if isinstance(source, bytes):
            self.stats["tx_eager"] += 1
            self._outbox.append((None, self.group.process_of(peer.id),
                                 (K_EAGER, (peer.id, self.id, tag, source))))
            self._fire(completion, Completion(status=OK, length=nbytes, tag=tag))
            self._flush_outbox()
            return
        sid = self.group.next_sid()
        if nbytes <= self.cfg.eager_threshold:
            self.stats["tx_eager"] += 1
            snap, ready, keep = self._snapshot(source)
            self._fire(completion, Completion(status=OK, length=nbytes, tag=tag))
            self._rdv[sid] = (None, tag, keep)
            addr = snap.addr
        else:
            self.stats["tx_rts"] += 1
            ready = self.space.record(source.buffer.owner)
            self._rdv[sid] = (completion, tag, None)
            addr = source.addr
        self._outbox.append((ready, self.group.process_of(peer.id),
                             (K_RTS, [peer.id, self.id, tag, nbytes, addr, sid])))
        self._flush_outbox()

    def _flush_outbox(self) -> None:
        while self._outbox:
            ready, proc_peer, (kind, body) = self._outbox[0]
            if ready is not None:
                if not ready.done():
                    return
                ready.release()
                handle, off = self.group.ipc_export(body[4])
                body = (body[0], body[1], body[2], body[3], handle, off, body[5])
            self._outbox.popleft()
            self.group.emit(proc_peer, kind, body)

    def _on_fin(self, sid: int, status: str, length: int, error) -> None:
        completion, tag, keep = self._rdv.pop(sid)
        if keep is not None:
            self.space.return_bounce(keep)
        if completion is not None:
            self._fire(completion, Completion(status=status, length=length, tag=tag, error=error))

    def _match_now(self, frame: Frame) -> bool:
        """Receiver side of a direct send: if a posted receive matches and no
        earlier frame from the same sender is still queued (FIFO per pair) or
        parked by a hold predicate, absorb the frame immediately."""
        if self.hold is not None or (self.inbound and any(f.src == frame.src for f in self.inbound)):
            return False
        for i, req in enumerate(self.posted):
            if req.matches(frame.tag):
                del self.posted[i]
                frame.seq = self._arrival_seq
                self._arrival_seq += 1
                self.stats[_RX_KEY[frame.kind]] += 1
                self._absorb(req, frame)
                return True
        return False

    def _snapshot(self, src: DeviceRegion):
        """Stream-ordered copy of an eager device payload into a pooled
        bounce buffer (returned to the pool once the receiver has read it)."""
        buf = src.buffer
        bounce = self.space.bounce(buf.gpu, src.size)
        ev = self.space.event(buf.gpu)
        _lib.call("hx_move", bounce.data_ptr(), src.addr, src.size, buf.gpu,
                  self.space.handle_of(buf.owner), None, ev.ptr, None)
        return _Bounce(bounce, src.size, buf.gpu, buf.owner), ev, bounce

    # ------------------------------------------------------------- receives

    def tag_recv(self, tag: int, mask: int = FULL_MASK, capacity: int = 0,
                 completion=None, sink=None) -> ReceiveRequest:
        """Post a tagged receive; matches queued unexpected frames first."""
        return self._post(tag, mask, capacity, sink, completion, wildcard=False)

    def _post(self, tag, mask, capacity, sink, completion, wildcard) -> ReceiveRequest:
        req = ReceiveRequest(tag, mask, capacity, sink, completion, self._post_seq, wildcard)
        self._post_seq += 1
        for i, frame in enumerate(self.unexpected):
            if req.matches(frame.tag):
                del self.unexpected[i]
                self._absorb(req, frame)
                return req
        self.posted.append(req)
        return req

    def tag_probe(self, tag: int, mask: int = FULL_MASK):
        for frame in self.unexpected:
            if (frame.tag & mask) == (tag & mask):
                return frame.tag, frame.length
        return None

    # ------------------------------------------------------------- progress

    def progress(self) -> int:
        """Drain arrivals, poll GPU copies, fire completions (cl/transport.py:342-362)."""
        if self.group.mesh is not None:
            self.group.poll()
            if self._outbox:
                self._flush_outbox()
        while self.inbound:
            frame = self.inbound.popleft()
            if self.hold is not None and self.hold(frame):
                self._held.append(frame)
                continue
            self._arrived(frame)
        if self._inflight:
            pending = []
            for op in self._inflight:
                if op.event.done():
                    op.fn()
                    op.event.release()
                else:
                    pending.append(op)
            self._inflight = pending
        fired = 0
        while self._fired:
            handle, comp = self._fired.popleft()
            if comp.timestamp is None:
                comp.timestamp = self.clock.now
            fired += 1
            if handle is not None:
                deliver(handle, comp)
        self.stats["completions"] += fired
        return fired

    def release_held(self) -> None:
        self.inbound.extendleft(reversed(self._held))
        self._held.clear()

    @property
    def idle(self) -> bool:
        """No arrivals, completions, or in-flight GPU copies."""
        return not (self.inbound or self._fired or self._inflight or self._outbox or self._rdv)

    def _arrived(self, frame: Frame) -> None:
        frame.seq = self._arrival_seq
        self._arrival_seq += 1
        self.stats[_RX_KEY[frame.kind]] += 1
        for i, req in enumerate(self.posted):
            if req.matches(frame.tag):
                del self.posted[i]
                self._absorb(req, frame)
                return
        self.unexpected.append(frame)

    def _absorb(self, req: ReceiveRequest, frame: Frame) -> None:
        """A request met a frame: move the bytes or truncate."""
        sender = self.group.workers[frame.src]
        if frame.length > req.capacity:
            self._fire(req.completion, Completion(
                status=TRUNCATED, length=frame.length, tag=frame.tag,
                error=f"frame of {frame.length} bytes exceeds capacity {req.capacity}"))
            if frame.kind == FRAME_RTS:  # the reference serves the pull anyway
                sender._fire(frame.send_completion, Completion(status=OK, length=frame.length,
                                                               tag=frame.tag))
            return
        try:
            self._move(req, frame, sender)
        except Exception as e:  # CUDA failure -> transport-error statuses
            err = Completion(status=TRANSPORT_ERROR, tag=frame.tag, error=repr(e))
            self._fire(req.completion, err)
            if frame.kind == FRAME_RTS:
                sender._fire(frame.send_completion, err)

    def _move(self, req: ReceiveRequest, frame: Frame, sender: "Worker") -> None:
        src, n, sink = frame.source, frame.length, req.sink
        if isinstance(sink, DeviceBuffer):
            sink = sink.region()

        def done(payload=None):
            comp = Completion(status=OK, length=n, tag=frame.tag, payload=payload)
            if req.wildcard:
                self._post(req.tag, req.mask, req.capacity, None, None, wildcard=True)
                if self.eager_handler is not None:
                    self.eager_handler(frame.tag, payload, self.clock.now)
                else:
                    self.eager_inbox.append((frame.tag, payload, self.clock.now))
                return
            self._fire(req.completion, comp)

        def send_done():
            if frame.kind == FRAME_RTS:
                sender._fire(frame.send_completion, Completion(status=OK, length=n, tag=frame.tag))

        if isinstance(src, bytes):
            if isinstance(sink, DeviceRegion):  # host -> device (pinned H2D)
                ev = self._h2d(sink, src)
                self._after(ev, done)
                ev.release()
                send_done()
            elif sink is None:
                done(src)
                send_done()
            else:
                sink[:n] = src
                done()
                send_done()
            return
        # device source: the sender's region (rdv) or a bounce snapshot (eager)
        if isinstance(sink, DeviceRegion):
            order = None
            if (frame.kind == FRAME_EAGER and isinstance(src, DeviceRegion)
                    and src.buffer.owner != sink.buffer.owner):
                # direct eager send: later work on the sender's stream must
                # not overwrite the source before the copy has read it
                order = self.space.handle_of(src.buffer.owner)
            ev = self._d2d(sink, src, n, frame.ready, order)
            keep = frame.keepalive

            def landed(keep=keep):
                done()
                send_done()
                if keep is not None:
                    self.space.return_bounce(keep)

            self._after(ev, landed)
            if frame.kind == FRAME_RTS:
                sender._after(ev, lambda: None)  # sender stays non-idle until the read ends
            ev.release()
        else:
            ev, stage = self._d2h(src, n, frame.ready)

            def landed_host(stage=stage, keep=frame.keepalive):
                data = stage.numpy()[:n].tobytes()
                if sink is None:
                    done(data)
                else:
                    sink[:n] = data
                    done()
                send_done()
                if keep is not None:
                    self.space.return_bounce(keep)

            self._after(ev, landed_host)
            ev.release()

    # ----------------------------------------------------------- GPU copies

    def _d2d(self, dst: DeviceRegion, src, n: int, ready, order=None):
        """Direct HBM / NVLink peer copy on the sink owner's stream: wait for
        the source, copy, record completion (and, if ``order`` is a stream,
        order it behind the copy) in one libhx call (hx_move)."""
        buf = dst.buffer
        ev = self.space.event(buf.gpu)
        _lib.call("hx_move", dst.addr, src.addr, n, buf.gpu, self.space.handle_of(buf.owner),
                  ready.ptr if ready is not None else None, ev.ptr, order)
        if ready is not None:
            ready.release()
        self.stats["d2d_copies"] += 1
        self.stats["d2d_bytes"] += n
        return ev

    def _h2d(self, dst: DeviceRegion, data: bytes):
        h = self.space.handle_of(dst.buffer.owner)
        stage = torch.empty(max(len(data), 1), dtype=torch.uint8, pin_memory=True)
        stage.numpy()[: len(data)] = np.frombuffer(data, dtype=np.uint8)
        if data:
            _lib.call("hx_memcpy", dst.addr, stage.data_ptr(), len(data), h)
        ev = self.space.record(dst.buffer.owner)
        self._after(ev, lambda stage=stage: None)  # keep the staging alive until landed
        return ev

    def _d2h(self, src, n: int, ready):
        owner = src.buffer.owner if isinstance(src, DeviceRegion) else src.owner
        h = self.space.handle_of(owner)
        if ready is not None:
            ready.wait_on(h)
            ready.release()
        stage = torch.empty(max(n, 1), dtype=torch.uint8, pin_memory=True)
        if n:
            _lib.call("hx_memcpy", stage.data_ptr(), src.addr, n, h)
        return self.space.record(owner), stage

    def close(self) -> None:
        pass


class _Bounce:
    """Device snapshot of an eager payload (owned by the transport)."""

    __slots__ = ("t", "addr", "size", "gpu", "owner")

    def __init__(self, t, size, gpu, owner):
        self.t = t
        self.addr = t.data_ptr()
        self.size = size
        self.gpu = gpu
        self.owner = owner


class _RemoteRegion:
    """A device payload living in another process's HBM, named by its
    allocation's CUDA IPC handle and offset; mapped (once per handle) into
    this process on first use."""

    __slots__ = ("group", "handle", "offset", "size", "owner", "_addr")

    def __init__(self, group, handle, offset, size, owner):
        self.group, self.handle, self.offset, self.size, self.owner = group, handle, offset, size, owner
        self._addr = None

    @property
    def addr(self) -> int:
        if self._addr is None:
            self._addr = self.group.ipc_open(self.handle, self.group.gpu_of(self.owner)) + self.offset
        return self._addr


class _FinToken:
    """Send completion of a remote rendezvous: firing it emits the FIN."""

    __slots__ = ("proc", "worker", "sid")

    def __init__(self, proc, worker, sid):
        self.proc, self.worker, self.sid = proc, worker, sid


class _RemoteWorker:
    """Stand-in for a worker of another process (ipc backend): what a local
    receiver does to "the sender" — fire its send completion, keep it busy —
    becomes a FIN frame, or nothing."""

    def __init__(self, group, worker_id: int):
        self.group = group
        self.id = worker_id

    def _fire(self, handle, comp: Completion) -> None:
        if isinstance(handle, _FinToken):
            self.group.emit(handle.proc, K_FIN, (handle.worker, handle.sid, comp.status,
                                                 comp.length, comp.error))

    def _after(self, event, fn) -> None:
        pass


class TransportGroup:
    """Process-local workers, wall clocks and the HBM device space
    (cl/transport.py:601-636). Enables NVLink peer access between every
    pair of GPUs the workers use.

    backend "ipc": one process per GPU under an initialised
    torch.distributed process group; worker w lives in process
    ``w % world`` (process_of). The other processes' workers appear as
    _RemoteWorker stand-ins, and the group owns the TCP mesh, the IPC handle
    caches (exported and opened) and the dispatch of arriving frames."""

    _live = weakref.WeakSet()  # diagnostics: debug_state() of every open group

    def __init__(self, cfg: RuntimeConfig | None = None, backend: str = "loopback"):
        TransportGroup._live.add(self)
        if backend not in ("loopback", "ipc"):
            raise StartupError(f"unknown backend {backend!r} (the B200 path offers 'loopback' "
                               "and 'ipc': one process per GPU, CUDA IPC data plane)")
        self.cfg = cfg or RuntimeConfig()
        self.backend = backend
        self.layout = TagLayout.from_spec(self.cfg.tag_layout)
        self.workers: dict = {}
        self.clocks: dict[int, WallClock] = {}
        self._device_space: DeviceSpace | None = None
        self._ngpu = None
        self.rank, self.world = 0, 1
        self.mesh = None
        self.runtime_handler = None  # ipc: callback(obj) for runtime frames
        self._sid = 0
        self._exported: dict = {}
        self._opened: dict = {}
        if backend == "ipc":
            import torch.distributed as dist

            if not dist.is_initialized():
                raise StartupError("backend 'ipc' needs an initialised torch.distributed process "
                                   "group (one process per GPU, e.g. under torchrun)")
            self.rank, self.world = dist.get_rank(), dist.get_world_size()
            self.mesh = Mesh(self.rank, self.world, self.layout.digest(), dist,
                             timeout_s=max(self.cfg.connect_timeout_s, 30.0))
            for w in range(self.cfg.workers):
                if not self.is_local(w):
                    self.workers[w] = _RemoteWorker(self, w)

    def debug_state(self) -> dict:
        """Queue depths of every local worker (diagnosing a stalled run)."""
        out = {"rank": self.rank, "world": self.world}
        for w, wk in self.workers.items():
            if isinstance(wk, Worker):
                out[w] = {"posted": [hex(r.tag) for r in wk.posted][:8],
                          "unexpected": [repr(f) for f in wk.unexpected][:8],
                          "inbound": len(wk.inbound), "fired": len(wk._fired),
                          "inflight": len(wk._inflight), "outbox": len(wk._outbox),
                          "rdv": sorted(wk._rdv)[:8], "stats": dict(wk.stats)}
        if self.mesh is not None:
            out["mesh"] = {p: (len(c.wbuf), len(c.rbuf), c.closed) for p, c in self.mesh.conns.items()}
        return out

    # ------------------------------------------------------------ ipc --

    def process_of(self, worker: int) -> int:
        return worker % self.world

    def is_local(self, worker: int) -> bool:
        return self.process_of(worker) == self.rank

    def local_workers(self) -> list:
        return [w for w in range(self.cfg.workers) if self.is_local(w)]

    def next_sid(self) -> int:
        self._sid += 1
        return self._sid

    def emit(self, proc: int, kind: int, body) -> None:
        self.mesh.send(proc, kind, body)

    def ipc_export(self, addr: int):
        """(IPC handle bytes, offset) of the allocation holding ``addr``,
        cached per allocation base."""
        b, n = ctypes.c_void_p(), ctypes.c_size_t(0)
        _lib.call("hx_alloc_range", addr, ctypes.byref(b), ctypes.byref(n))
        handle = self._exported.get((b.value, n.value))
        if handle is None:
            h = (ctypes.c_char * 64)()
            off = ctypes.c_size_t(0)
            _lib.call("hx_ipc_get", addr, h, ctypes.byref(off))
            handle = self._exported[(b.value, n.value)] = bytes(h)
        return handle, addr - b.value

    def ipc_open(self, handle: bytes, gpu: int) -> int:
        key = (handle, gpu)
        base = self._opened.get(key)
        if base is None:
            p = ctypes.c_void_p()
            _lib.call("hx_set_device", gpu)
            _lib.call("hx_ipc_open", handle, ctypes.byref(p))
            base = self._opened[key] = p.value
        return base

    def poll(self) -> None:
        """Deliver every frame that has arrived from the other processes."""
        for proc, kind, body in self.mesh.poll():
            if kind == K_EAGER:
                dst, src, tag, data = body
                self.workers[dst].inbound.append(
                    Frame(FRAME_EAGER, tag, len(data), data, None, src))
            elif kind == K_RTS:
                dst, src, tag, n, handle, off, sid = body
                region = _RemoteRegion(self, handle, off, n, dst)
                self.workers[dst].inbound.append(
                    Frame(FRAME_RTS, tag, n, region, None, src,
                          send_completion=_FinToken(proc, src, sid)))
            elif kind == K_FIN:
                worker, sid, status, length, error = body
                self.workers[worker]._on_fin(sid, status, length, error)
            elif kind == K_RUNTIME:
                if self.runtime_handler is None:
                    raise TransportError("runtime frame arrived but no runtime is attached")
                self.runtime_handler(body)
            else:
                raise TransportError(f"unknown frame kind {kind} from process {proc}")

    def gpu_of(self, worker: int) -> int:
        if self.cfg.gpus:
            return int(self.cfg.gpus[worker % len(self.cfg.gpus)])
        if self.backend == "ipc":
            return torch.cuda.current_device()  # one process per GPU
        if self._ngpu is None:
            self._ngpu = max(1, torch.cuda.device_count())
        return worker % self._ngpu

    def create_worker(self, worker_id: int, listen: str | None = None) -> Worker:
        if worker_id in self.workers:
            raise StartupError(f"duplicate worker id {worker_id} in process group")
        if not self.is_local(worker_id):
            raise StartupError(f"worker {worker_id} belongs to process "
                               f"{self.process_of(worker_id)}, not {self.rank}")
        self.clocks[worker_id] = WallClock()
        w = Worker(self, worker_id)
        self.workers[worker_id] = w
        return w

    @property
    def device_space(self) -> DeviceSpace:
        if self._device_space is None:
            self._device_space = DeviceSpace(self.gpu_of, self.clocks, self.cfg.device_capacity)
            gpus = sorted({self.gpu_of(w) for w in range(max(self.cfg.workers, 1))
                           if self.is_local(w)})
            for a in gpus:
                for b in gpus:
                    if a != b:
                        ok = ctypes.c_int(0)
                        _lib.call("hx_can_access_peer", a, b, ctypes.byref(ok))
                        if ok.value:
                            _lib.call("hx_enable_peer", a, b)
        return self._device_space

    def close(self) -> None:
        if self._device_space is not None:
            for s in self._device_space._streams.values():
                s.synchronize()
        for base in self._opened.values():
            _lib.raw("hx_ipc_close")(base)
        self._opened.clear()
        if self.mesh is not None:
            self.mesh.close()
            self.mesh = None
