"""Process mesh for the process-per-GPU backend: one TCP connection per
process pair carrying the runtime's control frames.

The reference's cross-process transport is its TCP backend
(cl/transport.py:469-586): a handshake of (magic, version, tag-layout
digest, worker id) (cl/transport.py:77-91), then length-prefixed frames,
delivered in send order per ordered pair. The B200 backend keeps that
shape for the HOST side only — envelopes, eager host payloads, rendezvous
announcements and their acknowledgements. Device payloads never cross a
socket: a device rendezvous frame carries the source allocation's CUDA
IPC handle and offset, and the receiver copies straight out of the
sender's HBM (NVLink P2P, or the same HBM when both processes share a GPU)
into its sink (transport.Worker._move). So the sockets see a few hundred
bytes per message whatever the payload size.

Set-up is collective: every process listens on 127.0.0.1 (ephemeral port),
the ports are all-gathered over the torch.distributed process group, each
process dials the lower ranks and accepts the higher ones, and the hello
is checked both ways (a tag-layout mismatch is a LayoutMismatchError, as
in the reference).
"""

from __future__ import annotations

import pickle
import socket
import struct
import time

MAGIC = b"HXW1"
PROTOCOL_VERSION = 1
_HELLO = struct.Struct("<4sHQI")   # magic, version, layout digest, process rank
_HEADER = struct.Struct("<4sBI")   # magic, kind, body length


class WireError(RuntimeError):
    pass


class LayoutMismatchError(WireError):
    pass


class _Conn:
    __slots__ = ("sock", "peer", "rbuf", "wbuf", "closed")

    def __init__(self, sock, peer):
        self.sock = sock
        self.peer = peer
        self.rbuf = bytearray()
        self.wbuf = bytearray()
        self.closed = False


def _recv_exact(sock, n: int, deadline: float) -> bytes:
    out = bytearray()
    while len(out) < n:
        if time.monotonic() > deadline:
            raise WireError("handshake timed out")
        chunk = sock.recv(n - len(out))
        if not chunk:
            raise WireError("peer closed during handshake")
        out += chunk
    return bytes(out)


class Mesh:
    """Full mesh of non-blocking TCP connections between ``world`` processes."""

    def __init__(self, rank: int, world: int, digest: int, dist, timeout_s: float = 30.0):
        self.rank, self.world = rank, world
        self.conns: dict[int, _Conn] = {}
        self.frames_sent = 0
        self.frames_received = 0
        self.eof_from: set = set()  # processes whose connection reached end of file
        if world == 1:
            return
        lst = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
        lst.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
        lst.bind(("127.0.0.1", 0))
        lst.listen(world)
        ports = [None] * world
        dist.all_gather_object(ports, lst.getsockname()[1])
        deadline = time.monotonic() + timeout_s
        hello = _HELLO.pack(MAGIC, PROTOCOL_VERSION, digest, rank)
        pending = []
        for peer in range(rank):  # dial the lower ranks (already listening)
            s = socket.create_connection(("127.0.0.1", ports[peer]), timeout=timeout_s)
            s.sendall(hello)
            pending.append(s)
        lst.settimeout(timeout_s)
        for _ in range(rank + 1, world):  # accept the higher ranks
            s, _ = lst.accept()
            s.sendall(hello)
            pending.append(s)
        lst.close()
        for s in pending:
            s.settimeout(timeout_s)
            magic, version, their_digest, peer = _HELLO.unpack(_recv_exact(s, _HELLO.size, deadline))
            if magic != MAGIC:
                raise WireError(f"bad handshake magic {magic!r}")
            if version != PROTOCOL_VERSION:
                raise WireError(f"protocol version mismatch: ours {PROTOCOL_VERSION}, "
                                f"theirs {version}")
            if their_digest != digest:
                raise LayoutMismatchError(f"tag layout digest mismatch: ours 0x{digest:016x}, "
                                          f"process {peer} sent 0x{their_digest:016x}")
            s.setblocking(False)
            s.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
            self.conns[peer] = _Conn(s, peer)
        if sorted(self.conns) != [p for p in range(world) if p != rank]:
            raise WireError(f"process {rank}: mesh incomplete ({sorted(self.conns)})")

    # ------------------------------------------------------------ frames --

    def send(self, peer: int, kind: int, obj) -> None:
        """Queue one frame (``obj`` pickled) to process ``peer`` and try to
        flush; frames to one peer leave in call order."""
        conn = self.conns.get(peer)
        if conn is None or conn.closed:
            raise WireError(f"no connection to process {peer}")
        body = pickle.dumps(obj, protocol=pickle.HIGHEST_PROTOCOL)
        conn.wbuf += _HEADER.pack(MAGIC, kind, len(body))
        conn.wbuf += body
        self.frames_sent += 1
        self._flush(conn)

    def _flush(self, conn: _Conn) -> None:
        while conn.wbuf:
            try:
                n = conn.sock.send(conn.wbuf)
            except BlockingIOError:
                return
            except OSError as e:
                conn.closed = True
                raise WireError(f"connection to process {conn.peer} failed: {e}") from e
            del conn.wbuf[:n]

    def poll(self) -> list:
        """Non-blocking: flush pending writes, return [(peer, kind, obj)] of
        every complete frame received since the last poll."""
        out = []
        for conn in self.conns.values():
            if conn.closed and not conn.rbuf:
                continue
            if conn.wbuf and not conn.closed:
                self._flush(conn)
            while not conn.closed:
                try:
                    chunk = conn.sock.recv(1 << 20)
                except BlockingIOError:
                    break
                except OSError as e:
                    conn.closed = True
                    raise WireError(f"connection to process {conn.peer} failed: {e}") from e
                if not chunk:  # the peer closed: frames already buffered still parse
                    conn.closed = True
                    self.eof_from.add(conn.peer)
                    break
                conn.rbuf += chunk
                if len(chunk) < (1 << 20):
                    break
            buf = conn.rbuf
            pos = 0
            while len(buf) - pos >= _HEADER.size:
                magic, kind, n = _HEADER.unpack_from(buf, pos)
                if magic != MAGIC:
                    conn.closed = True
                    raise WireError(f"bad frame magic {magic!r} from process {conn.peer}")
                if len(buf) - pos - _HEADER.size < n:
                    break
                start = pos + _HEADER.size
                out.append((conn.peer, kind, pickle.loads(bytes(buf[start:start + n]))))
                pos = start + n
            if pos:
                del buf[:pos]
        self.frames_received += len(out)
        return out

    @property
    def flushed(self) -> bool:
        return all(not c.wbuf for c in self.conns.values())

    def close(self) -> None:
        for c in self.conns.values():
            if not c.closed:
                c.closed = True
                try:
                    c.sock.close()
                except OSError:
                    pass
        self.conns.clear()
