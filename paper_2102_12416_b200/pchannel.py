"""Pre-registered device channels: the paper's Channel API in its B200 form.

The reference's Channel (cl/channels.py:33-102) is metadata-free: both ends
derive the kth transfer's tag from a per-direction counter, so no envelope
crosses. On B200 the same contract needs no host at all. Each direction owns
* a ring of ``depth`` slots in the receiver's HBM;
* the slots' lengths and an arrival counter next to them;
* a credit counter on the sender.
All of it is allocated and mapped once (NVLink P2P between the two GPUs).

``send`` is one kernel: wait for a free slot, write the payload into the
peer's slot over NVLink and publish its header (tag k + 1 and length in one
word; up to 8 KiB as LL words that carry the tag themselves, so no fence is
needed; payloads that fit a slot bulk-copied with the header
release-stored, so the sender may run ``depth`` messages ahead — and
consecutive sends on one stream overlap on the GPU, each in its own slot,
so a stream of them keeps NVLink busy across kernel boundaries; larger
payloads are not copied by the sender at all: the header publishes the
source address, the receiver copies straight out of it, and the send
completes when the slot comes back). ``recv`` is one kernel: wait for the
header tag, copy into the sink, hand the slot back (credit = k + 1). The
counters (k)
live on the device, so every operation is stream-ordered like an NCCL call,
and a sequence of them can be captured in a CUDA graph and replayed with no
host involvement (``osu.channel_latency`` / ``channel_bandwidth`` do exactly
that).

Kernels: hx_chan_send / hx_chan_recv (include/hx.h). The two endpoints are
normally on different GPUs: a receive spins until its matching send lands.
Both on one GPU (two streams) is opt-in (allow_same_gpu) and relies on the
spinning receive and the send being resident together, which the bounded
grids allow. A pulled send (larger than a slot) completes only after its
receive has run, so two pulled sends crossing in opposite directions must
not each sit in front of the receive the other one waits for on the same
stream (put one side's receives first, or on another stream).
"""

from __future__ import annotations

import torch

from . import _lib
from .completion import OK, TRUNCATED

LL_MAX = 8192  # include/hx.h HX_CHAN_LL_MAX: payloads up to this go as LL words
HDR = 128      # include/hx.h HX_CHAN_HDR: header block; the payload is 128-byte aligned


class PersistentChannel:
    """Bidirectional channel between endpoint 0 (``gpu_a``) and endpoint 1
    (``gpu_b``). Messages up to ``slot_bytes`` are staged in one of
    ``depth`` slots per direction; larger ones are pulled by the receiver
    straight from the sender's buffer."""

    def __init__(self, gpu_a: int, gpu_b: int, slot_bytes: int = 1 << 20, depth: int = 4,
                 timeout_s: float = 10.0, tickets: int = 4096, allow_same_gpu: bool = False):
        # Both ends on one GPU (allow_same_gpu, two streams) works when a
        # spinning receive and the send it waits for can be resident
        # together — true for the bounded grids used here, but not a
        # guarantee the hardware gives, so it is opt-in (tests on 1-GPU boxes).
        if gpu_a == gpu_b and not allow_same_gpu:
            raise ValueError("a persistent channel joins two different GPUs "
                             "(allow_same_gpu=True for two streams of one GPU)")
        if slot_bytes < 1 or depth < 1:
            raise ValueError("slot_bytes and depth must be positive")
        self.gpus = (gpu_a, gpu_b)
        self.slot_bytes = slot_bytes
        self.depth = depth
        self.timeout_ns = int(timeout_s * 1e9)
        if gpu_a != gpu_b:
            _lib.call("hx_enable_peer", gpu_a, gpu_b)
            _lib.call("hx_enable_peer", gpu_b, gpu_a)
        for g in sorted({gpu_a, gpu_b}):  # no lazy kernel load behind a spinning one
            _lib.call("hx_set_device", g)
            _lib.call("hx_preload")
        # a slot: header block, then the payload (LL words are 2x the bytes)
        ll = min(slot_bytes, LL_MAX)
        self.stride = -(-(HDR + max(slot_bytes, 8 * (-(-ll // 4)))) // 256) * 256
        self._dir = []
        for d in (0, 1):  # direction d: endpoint d sends, endpoint 1 - d receives
            tx, rx = self.gpus[d], self.gpus[1 - d]
            rdev, tdev = torch.device("cuda", rx), torch.device("cuda", tx)
            self._dir.append({
                "slots": torch.zeros(depth * self.stride, dtype=torch.uint8, device=rdev),
                # receive ticket (message index << 32 | CTAs of the current launch)
                "rseq": torch.zeros(1, dtype=torch.int64, device=rdev),
                # credit, ticket (message index << 32 | CTAs of the current launch)
                "tmeta": torch.zeros(2, dtype=torch.int64, device=tdev),
                "rctr": torch.zeros(2, dtype=torch.int32, device=rdev),   # counter, err
                # [_, err, one arrival counter per slot] (overlapping sends)
                "tctr": torch.zeros(2 + depth, dtype=torch.int32, device=tdev),
                "lens_out": torch.zeros(tickets, dtype=torch.int64, device=rdev),
                "posted": 0,
            })
        torch.cuda.synchronize(gpu_a)
        torch.cuda.synchronize(gpu_b)

    @staticmethod
    def _ptr(t: torch.Tensor, i: int = 0) -> int:
        return t.data_ptr() + i * t.element_size()

    def _stream(self, gpu: int, stream):
        return (stream if stream is not None else torch.cuda.current_stream(gpu)).cuda_stream

    def send(self, end: int, src: torch.Tensor, nbytes: int | None = None, stream=None) -> None:
        """Enqueue endpoint ``end``'s next send of ``src`` (a CUDA tensor on
        that endpoint's GPU) on ``stream``; the source may be reused by work
        later on the same stream."""
        d = self._dir[end]
        gpu = self.gpus[end]
        n = src.numel() * src.element_size() if nbytes is None else nbytes
        if src.device != torch.device("cuda", gpu):
            raise ValueError(f"endpoint {end} sends from cuda:{gpu}")
        _lib.call("hx_set_device", gpu)
        _lib.call("hx_chan_send", src.data_ptr(), n, d["slots"].data_ptr(), self.stride,
                  self.depth, self._ptr(d["tmeta"]), self._ptr(d["tmeta"], 1),
                  self._ptr(d["tctr"], 2), self.timeout_ns, self._ptr(d["tctr"], 1),
                  self._stream(gpu, stream))

    def recv(self, end: int, dst: torch.Tensor, capacity: int | None = None, stream=None) -> int:
        """Enqueue endpoint ``end``'s next receive into ``dst`` (a CUDA tensor
        on its GPU). Returns a ticket for ``completion``."""
        d = self._dir[1 - end]  # the direction whose receiver is ``end``
        gpu = self.gpus[end]
        cap = dst.numel() * dst.element_size() if capacity is None else capacity
        if dst.device != torch.device("cuda", gpu):
            raise ValueError(f"endpoint {end} receives into cuda:{gpu}")
        ticket = d["posted"]
        d["posted"] += 1
        _lib.call("hx_set_device", gpu)
        _lib.call("hx_chan_recv", dst.data_ptr(), cap, d["slots"].data_ptr(), self.stride,
                  self.depth, self._ptr(d["tmeta"]), self._ptr(d["rseq"]), self._ptr(d["rctr"]),
                  self._ptr(d["lens_out"], ticket % d["lens_out"].numel()), self.timeout_ns,
                  self._ptr(d["rctr"], 1), self._stream(gpu, stream))
        return ticket

    def completion(self, end: int, ticket: int, capacity: int) -> tuple:
        """(status, length) of a finished receive: OK or TRUNCATED (the
        reference's Completion statuses, cl/completion.py:14-16)."""
        d = self._dir[1 - end]
        torch.cuda.synchronize(self.gpus[end])
        n = int(d["lens_out"][ticket % d["lens_out"].numel()].item())
        return (TRUNCATED if n > capacity else OK), n

    def check(self) -> None:
        """Raise if a device-side wait of this channel timed out."""
        for d in self._dir:
            for t in (d["rctr"], d["tctr"]):
                err = int(t[1].item())
                if err:
                    raise RuntimeError(f"persistent channel: device error {err} "
                                       f"({_lib.error_string(err)})")

    @property
    def counters(self) -> list:
        """Per direction: (sent, received) message counts (device state)."""
        out = []
        for d in self._dir:
            out.append((int(d["tmeta"][1].item()) >> 32, int(d["rseq"][0].item()) >> 32))
        return out

    def close(self) -> None:
        self._dir.clear()


__all__ = ["PersistentChannel"]
