"""Persistent-channel Jacobi3D engine: one block per GPU, NVLink peer stores.

This is the B200 form of the paper's Channel API applied to the Jacobi3D
halo exchange (paper §3.2.2 + §4.3; reference loop cl/jacobi3d.py:246-279,
channels cl/channels.py:75-99). Each block owns an IPC-exportable arena in
HBM,

    [flags: 6 x u64][counters: 6 x u32][err: i32][pad][slot[parity][dir] ...]

and its two fields; both are exported once to the neighbours (CUDA IPC
handle cache across processes, plain P2P pointers inside one process). The
channel counter is a 64-bit flag value, so no tag or metadata ever crosses
(paper Fig. 6-7). Two exchanges share that set-up:

exchange="fused" (default). Per iteration it and block, with no host
involvement:
  * comm stream: ONE hx_shell_put — every CTA acquires its flags >= it + 1
    (the neighbours' boundary of it - 1 is in cur's ghost planes, and they
    have finished reading the ghost planes about to be written), relaxes the
    boundary shell and stores each neighbour-facing cell both into nxt and
    over NVLink straight into the neighbour's nxt ghost plane, then the last
    CTA release-stores flag = it + 2 in every neighbour's arena;
  * main stream, concurrently: the TMA sweep of the interior box, then a
    wait for the shell's event.
  One channel exchange (below) before the first step primes the ghosts.

exchange="p2p" (the channel kernels; overlap=True adds the interior /
boundary split):
  1. hx_pack_put: pack every neighbour-facing interior plane straight into
     the neighbour's slot[it & 1][d ^ 1] over NVLink and, once all CTAs have
     stored, release-store flag = it + 1 in the neighbour's arena;
  2. hx_wait_unpack: acquire own flags >= it + 1 and unpack the slots into
     the ghost planes;
  3. hx_stencil (TMA pipeline) cur -> nxt, optional fused residual.
  Two parity slots suffice: a neighbour can run at most one iteration ahead
  (cl/jacobi3d.py:146) because its put for it + 2 needs our flag for it + 1,
  which we publish only after unpacking iteration it.

Every device-side wait points at work of an EARLIER launch (another GPU's,
or one queued before it on the same stream): blocks hosted by one process
on one GPU share that GPU's streams and are driven in phase order, so no
kernel ever waits for one launched after it and no two waiting kernels need
to be co-resident.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _lib
from .jacobi3d import _block_coords, decompose, decompose_b200, neighbor_table

NDIRS = 6
_ALIGN = 256
_HDR = 256  # flags (48 B) + counters (24 B) + err (4 B), padded


def _round(n: int) -> int:
    return (n + _ALIGN - 1) // _ALIGN * _ALIGN


_STAGING: dict = {}


def _staging(nbytes: int, count: int) -> list:
    """Process-wide ring of ``count`` pinned byte buffers of at least
    ``nbytes`` (interior_into's read-back staging)."""
    ring = _STAGING.get(count)
    if ring is None or ring[0].numel() < nbytes:
        ring = _STAGING[count] = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
                                  for _ in range(count)]
    return ring


def _split(n: int, parts: int) -> list:
    """[r0, r1) ranges cutting range(n) into at most ``parts`` near-equal pieces."""
    parts = max(1, min(parts, n))
    return [(n * p // parts, n * (p + 1) // parts) for p in range(parts)]


def _copy_rows(out, host, i0: int, r0: int, r1: int, by: int) -> None:
    """Copy interior rows [r0, r1) (flattened (plane, row)) of the padded
    planes ``host`` (k, by + 2, bz + 2) into ``out[i0 + plane, row]``."""
    while r0 < r1:
        a, j0 = divmod(r0, by)
        j1 = min(by, j0 + (r1 - r0))
        np.copyto(out[i0 + a, j0:j1], host[a, 1 + j0:1 + j1, 1:-1])
        r0 += j1 - j0


def prefault_host(shape, threads: int = 16):
    """A float64 host array of ``shape`` whose pages are being touched by
    ``threads`` background threads (returns (array, futures)). First touch
    of fresh pages (the kernel zeroes them) is the slow part of reading a
    large field back (~6 GB/s per thread); run_jacobi starts it before the
    iterations so it overlaps the GPU work."""
    from concurrent.futures import ThreadPoolExecutor

    out = np.empty(shape)
    flat = out.reshape(-1)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1
    pool = ThreadPoolExecutor(max(1, min(threads, cores)))
    futs = [pool.submit(flat[a:b].fill, 0.0) for a, b in _split(flat.size, max(1, min(threads, cores)))]
    pool.shutdown(wait=False)
    return out, futs


class HaloBlock:
    """One block: two padded fields + its receive arena on one GPU."""

    def __init__(self, dims, grid, rank: int, device: int, allocate: bool = True):
        self.rank = rank
        self.grid = grid
        self.device = device
        self.bx, self.by, self.bz = dims[0] // grid[0], dims[1] // grid[1], dims[2] // grid[2]
        self.coords = _block_coords(rank, grid)
        self.neighbors = neighbor_table(grid, rank)
        self.nbr_dirs = [d for d in range(NDIRS) if self.neighbors[d] is not None]
        self.dir_mask = sum(1 << d for d in self.nbr_dirs)
        ext = (self.bx, self.by, self.bz)
        self.face_elems = [int(np.prod([ext[a] for a in range(3) if a != d // 2])) for d in range(NDIRS)]
        self.slot_off = {}
        off = _HDR
        for p in (0, 1):
            for d in range(NDIRS):
                self.slot_off[(p, d)] = off
                off += _round(self.face_elems[d] * 8)
        self.arena_bytes = off
        self.cur = 0
        self.fields, self.arena = [], None
        if allocate:
            dev = torch.device("cuda", device)
            shape = (self.bx + 2, self.by + 2, self.bz + 2)
            self.fields = [torch.empty(shape, dtype=torch.float64, device=dev) for _ in range(2)]
            self.arena = torch.zeros(self.arena_bytes, dtype=torch.uint8, device=dev)
            self.step_dev = torch.zeros(1, dtype=torch.int64, device=dev)  # graph replays
            # z faces from the interior sweep: its step counter (hx_zsignal advances it)
            self.zstep_dev = torch.zeros(1, dtype=torch.int64, device=dev)
        # filled by HaloJacobi.connect(): (neighbour arena base, its side)
        self.put_dst = [None] * NDIRS
        self.put_flag = [None] * NDIRS
        # exchange="fused": the neighbour's two field bases per direction
        self.peer_fields = [None] * NDIRS

    @property
    def base(self) -> int:
        return self.arena.data_ptr()

    def link(self, d: int, peer_base: int) -> None:
        """Point face d's put at the neighbour's arena: I send face d, the
        neighbour receives it on its side d ^ 1 (slot and flag)."""
        self.put_dst[d] = (peer_base, d ^ 1)
        self.put_flag[d] = self.flag_ptr(d ^ 1, peer_base)

    def put_slot(self, d: int, parity: int) -> int:
        base, side = self.put_dst[d]
        return base + self.slot_off[(parity, side)]

    def flag_ptr(self, d: int, base: int | None = None) -> int:
        return (self.base if base is None else base) + 8 * d

    @property
    def step_ptr(self) -> int:
        return self.step_dev.data_ptr()

    @property
    def counters_ptr(self) -> int:
        return self.base + 48

    @property
    def err_ptr(self) -> int:
        return self.base + 72

    def slot_ptr(self, parity: int, d: int, base: int | None = None) -> int:
        return (self.base if base is None else base) + self.slot_off[(parity, d)]

    def field_ptr(self, which: int | None = None) -> int:
        return self.fields[self.cur if which is None else which].data_ptr()

    @property
    def cells(self) -> int:
        return self.bx * self.by * self.bz


class _Marks:
    """CUDA event pairs per (name, block) for optional step timing. A timing
    dict holding the key "_only" (a set of names) records just those."""

    def __init__(self, timing):
        self.t = timing
        self.only = timing.get("_only") if timing is not None else None
        self.open = {}

    def begin(self, name, b, stream):
        if self.t is not None and (self.only is None or name in self.only):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            self.open[(name, b.rank)] = e

    def end(self, name, b, stream):
        if self.t is not None and (self.only is None or name in self.only):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            self.t.setdefault(name, []).append((self.open.pop((name, b.rank)), e))


def exchange_table(dist, mine):
    """All-gather each process's (rank, ipc handle, offset, device) arena
    records — the one-time persistent-channel set-up. Without a process
    group every block is local and the table is just ``mine``."""
    if dist is None:
        return {rec[0]: tuple(rec[1:]) for rec in mine}
    gathered = [None] * dist.get_world_size()
    dist.all_gather_object(gathered, mine)
    return {rec[0]: tuple(rec[1:]) for part in gathered for rec in part}


class HaloJacobi:
    """Jacobi3D over persistent NVLink channels.

    dims: global grid; pes: total blocks; local_ranks: blocks hosted by this
    process; device_of(rank) -> CUDA ordinal; dist: the initialised
    torch.distributed module (None when every block is local; used once to
    exchange IPC handles, and by the NCCL comparison path). policy "reference"
    uses cl/jacobi3d.py's decompose (bit-for-bit the reference's block
    layout); "b200" prefers not to split z on ties.

    exchange: "fused" (default) — the boundary sweep stores straight into
    the neighbours' ghost planes (hx_shell_put) while the interior sweeps;
    "p2p" — persistent-channel pack+put / wait+unpack kernels, with the
    interior/boundary split when overlap=True; "nccl" — the comparison
    path (pack, NCCL send/recv, unpack). overlap applies to "p2p" only.
    """

    e2e_ring_slots = 4096  # device residual slots of step_e2e (zeroed when the ring wraps)
    # fused, z neighbours: True (default) = the interior sweep produces and
    # consumes the z faces (hx_stencil_box_z: one launch whose edge tiles
    # wait for the z flags, take the ghost column from the slot and write the
    # face into the neighbour's slot; hx_zsignal releases the flags). The
    # sweep opens those DRAM pages anyway, so the z faces cost nothing extra:
    # 8.92 vs 9.07 ms per step for a 1536^3 block with a z split on 2 GPUs
    # (plain sweep 8.87). False = the boundary kernel's z tiles, which pay a
    # DRAM page activation per face cell (tools/prof_zshell.py,
    # profiles/r2_zface_dram.md).
    z_from_interior = True
    # fused: True (default) = every face (x / y as well as z) is produced and
    # consumed by the interior sweep's edge tiles (hx_stencil_exchange: one
    # launch per block and step, no boundary kernel, no comm stream), then
    # hx_exchange_signal releases the flags. Same box, 1536^3 per GPU:
    # N = 2 8.899 vs 8.907 ms per step, N = 4 8.910 vs 8.927
    # (profiles/r2_sweep_exchange_ab_*.jsonl). False = x / y faces by the
    # concurrent boundary kernel (hx_shell_put_z).
    xy_from_interior = True
    z_slots = True  # fused exchange: z faces through the contiguous arena slots (False: ghost columns)

    def __init__(self, dims, pes: int, local_ranks=None, device_of=None, dist=None,
                 policy: str = "reference", timeout_s: float = 30.0, overlap: bool = False,
                 exchange: str = "fused"):
        if exchange not in ("p2p", "fused", "nccl"):
            raise ValueError(f"exchange must be 'p2p', 'fused' or 'nccl', got {exchange!r}")
        if exchange == "nccl" and (dist is None or overlap):
            raise ValueError("the NCCL comparison path needs a process group and overlap=False")
        self.dims = tuple(dims)
        self.overlap = overlap
        self.exchange = exchange
        self.pes = pes
        self.grid = (decompose if policy == "reference" else decompose_b200)(self.dims, pes)
        self.local_ranks = list(range(pes)) if local_ranks is None else list(local_ranks)
        ndev = max(1, torch.cuda.device_count())
        self.device_of = device_of or (lambda r: r % ndev)
        self.dist = dist
        self.timeout_ns = int(timeout_s * 1e9)
        self.blocks = {r: HaloBlock(self.dims, self.grid, r, self.device_of(r)) for r in self.local_ranks}
        self.streams = {}
        self.comm = {}
        for b in self.blocks.values():
            if b.device not in self.streams:
                self.streams[b.device] = torch.cuda.Stream(device=b.device)
                # halo traffic on a high-priority stream so its few CTAs are
                # scheduled ahead of the queued interior-sweep CTAs
                self.comm[b.device] = torch.cuda.Stream(device=b.device, priority=-1)
        self.it = 0
        self._ipc_bases = []
        self._res = {}
        self._graphs = {}  # buffer parity -> {device: CUDAGraph} (run_graph)
        self.reset()
        if exchange in ("p2p", "fused"):
            self.connect()
        else:
            self._nccl_buffers()

    # ------------------------------------------------------------ set-up --

    def stream_of(self, b: HaloBlock) -> torch.cuda.Stream:
        return self.streams[b.device]

    def reset(self) -> None:
        """Dirichlet initial state (cl/jacobi3d.py:131-138) and zeroed flags."""
        for dev in sorted({b.device for b in self.blocks.values()}):
            _lib.call("hx_set_device", dev)
            _lib.call("hx_preload")  # no lazy kernel load behind a spinning one (include/hx.h)
        for b in self.blocks.values():
            s = self.stream_of(b).cuda_stream
            _lib.call("hx_set_device", b.device)
            for f in b.fields:
                _lib.call("hx_init_block", f.data_ptr(), b.bx, b.by, b.bz,
                          int(b.coords[0] == 0), 1.0, 0.0, 0.0, s)
            with torch.cuda.stream(self.stream_of(b)):
                b.arena[:_HDR].zero_()
                b.zstep_dev.zero_()
            b.cur = 0
        self.it = 0
        self._zstep_stale = False
        self.synchronize()

    def fill_random(self, seed: int = 0) -> None:
        """Seeded N(0,1) interior on both buffers of every local block; the
        ghost planes keep their Dirichlet values (cl/jacobi3d.py:131-138).
        Resets the step counter and the channel flags, so the next step
        re-primes the halo. Collective: every process calls it between two
        barriers (no step of any block may be in flight)."""
        self.reset()
        for b in self.blocks.values():
            g = torch.Generator(device=f"cuda:{b.device}")
            g.manual_seed(seed * 1000003 + b.rank)
            with torch.cuda.device(b.device), torch.cuda.stream(self.stream_of(b)):
                for f in b.fields:
                    f[1:-1, 1:-1, 1:-1].normal_(generator=g)
        self.synchronize()

    def connect(self) -> None:
        """Exchange receive-arena addresses once (the persistent channel set-up)."""
        fused = self.exchange == "fused"
        mine = []
        for r, b in self.blocks.items():
            rec = [r]
            for ptr in [b.base] + ([f.data_ptr() for f in b.fields] if fused else []):
                handle = (ctypes.c_char * 64)()
                off = ctypes.c_size_t(0)
                if self.dist is not None:
                    _lib.call("hx_set_device", b.device)
                    _lib.call("hx_ipc_get", ptr, handle, ctypes.byref(off))
                rec += [bytes(handle), off.value]
                if len(rec) == 3:
                    rec.append(b.device)
            mine.append(tuple(rec))
        table = exchange_table(self.dist, mine)
        bases, fields = {}, {}
        for r, b in self.blocks.items():
            for d in b.nbr_dirs:
                n = b.neighbors[d]
                if n in self.blocks:
                    bases[n] = self.blocks[n].base
                    fields[n] = [f.data_ptr() for f in self.blocks[n].fields]
                    if self.blocks[n].device != b.device:
                        _lib.call("hx_enable_peer", b.device, self.blocks[n].device)
                elif n not in bases:
                    rec = table[n]
                    _lib.call("hx_set_device", b.device)
                    bases[n] = self._open(rec[0], rec[1])
                    if fused:
                        fields[n] = [self._open(rec[3], rec[4]), self._open(rec[5], rec[6])]
                b.link(d, bases[n])
                if fused:
                    b.peer_fields[d] = fields[n]

    def _open(self, handle: bytes, offset: int) -> int:
        base = ctypes.c_void_p()
        _lib.call("hx_ipc_open", handle, ctypes.byref(base))
        self._ipc_bases.append(base.value)
        return base.value + offset

    # ------------------------------------------------------------- steps --

    def _put(self, b: HaloBlock, it: int) -> None:
        p = it & 1
        dst = [None] * NDIRS
        flg = [None] * NDIRS
        for d in b.nbr_dirs:
            dst[d] = b.put_slot(d, p)
            flg[d] = b.put_flag[d]
        _lib.call("hx_pack_put", b.field_ptr(), b.bx, b.by, b.bz, b.dir_mask, _lib.ptr_array(dst),
                  _lib.ptr_array(flg), it + 1, b.counters_ptr, self.stream_of(b).cuda_stream)

    def _wait(self, b: HaloBlock, it: int) -> None:
        p = it & 1
        src = [b.slot_ptr(p, d) if d in b.nbr_dirs else None for d in range(NDIRS)]
        flg = [b.flag_ptr(d) if d in b.nbr_dirs else None for d in range(NDIRS)]
        _lib.call("hx_wait_unpack", b.field_ptr(), b.bx, b.by, b.bz, b.dir_mask,
                  _lib.ptr_array(src), _lib.ptr_array(flg), it + 1, self.timeout_ns, b.err_ptr,
                  self.stream_of(b).cuda_stream)

    def _relax(self, b: HaloBlock, res_ptr) -> None:
        _lib.call("hx_stencil", b.field_ptr(), b.field_ptr(b.cur ^ 1), b.bx, b.by, b.bz, res_ptr,
                  self.stream_of(b).cuda_stream)
        b.cur ^= 1

    def _res_ptr(self, b: HaloBlock, it: int, residual):
        if isinstance(residual, dict):  # explicit per-block device u64 slots
            return residual.get(b.rank)
        if not residual:
            return None
        buf = self._res.setdefault(b.rank, [])
        if len(buf) <= it:
            # zero-filled on the block's main stream: every kernel that
            # accumulates into the slot is ordered after it (the comm stream
            # waits on the main stream's `ready` event, recorded later)
            with torch.cuda.stream(self.stream_of(b)):
                buf.append(torch.zeros(1, dtype=torch.int64, device=f"cuda:{b.device}"))
        return buf[it].data_ptr()

    def step(self, residual=False, timing: dict | None = None) -> None:
        """One iteration on every local block (enqueue only, no host sync).

        residual: False, True (per-step device slots, see residuals()) or a
        dict rank -> device u64 pointer accumulating max|nxt-cur|.
        timing (optional): dict of lists receiving CUDA event pairs per block
        — 'exchange' (put + wait + unpack), 'sweep' (all stencil work), and in
        overlap mode 'interior', 'exposed' (main stream stalled on the halo)
        and 'shell'."""
        if self.exchange == "nccl":
            return self._step_nccl(residual, timing)
        if self.exchange == "fused":
            return self._step_fused(residual, timing)
        if self.overlap:
            return self._step_overlap(residual, timing)
        it = self.it
        blocks = list(self.blocks.values())
        mark = _Marks(timing)
        for b in blocks:
            if b.nbr_dirs:
                _lib.call("hx_set_device", b.device)
                mark.begin("exchange", b, self.stream_of(b))
                self._put(b, it)
        for b in blocks:
            if b.nbr_dirs:
                _lib.call("hx_set_device", b.device)
                self._wait(b, it)
                mark.end("exchange", b, self.stream_of(b))
        for b in blocks:
            _lib.call("hx_set_device", b.device)
            mark.begin("sweep", b, self.stream_of(b))
            self._relax(b, self._res_ptr(b, it, residual))
            mark.end("sweep", b, self.stream_of(b))
        self.it += 1

    # ------------------------------------------------------- overlap mode --

    def boxes(self, b: HaloBlock):
        """Interior box (cells that read no neighbour-fed ghost) and the
        disjoint boundary slabs toward neighbours, 1-based [lo, hi) triples."""
        n = (b.bx, b.by, b.bz)
        nb = b.neighbors
        lo = [2 if nb[2 * a] is not None else 1 for a in range(3)]
        hi = [n[a] if nb[2 * a + 1] is not None else n[a] + 1 for a in range(3)]
        inner = (lo[0], hi[0], lo[1], hi[1], lo[2], hi[2])
        shells = []
        if nb[0] is not None:
            shells.append((1, 2, 1, b.by + 1, 1, b.bz + 1))
        if nb[1] is not None:
            shells.append((b.bx, b.bx + 1, 1, b.by + 1, 1, b.bz + 1))
        if nb[2] is not None:
            shells.append((lo[0], hi[0], 1, 2, 1, b.bz + 1))
        if nb[3] is not None:
            shells.append((lo[0], hi[0], b.by, b.by + 1, 1, b.bz + 1))
        if nb[4] is not None:
            shells.append((lo[0], hi[0], lo[1], hi[1], 1, 2))
        if nb[5] is not None:
            shells.append((lo[0], hi[0], lo[1], hi[1], b.bz, b.bz + 1))
        return inner, [x for x in shells if x[0] < x[1] and x[2] < x[3] and x[4] < x[5]]

    def z_interior(self, b: HaloBlock) -> bool:
        """Fused exchange with z neighbours: the interior TMA sweep spans
        whole z rows and produces / consumes the z faces itself
        (hx_stencil_box_z), so no kernel touches the z columns separately.
        Needs a TMA-describable block (even bz, 16-byte aligned field) and,
        with both z neighbours, bz > 64 (no tile holds both z faces)."""
        both = 4 in b.nbr_dirs and 5 in b.nbr_dirs
        return (self.z_from_interior and self.z_slots and (4 in b.nbr_dirs or 5 in b.nbr_dirs)
                and (b.bz + 2) % 2 == 0 and b.fields[0].data_ptr() % 16 == 0 and b.bz >= 2
                and not (both and b.bz <= 64))

    def sweep_exchange(self, b: HaloBlock) -> bool:
        """xy_from_interior applies to this block: the whole fused step is
        one hx_stencil_exchange sweep (TMA-describable block; no tile holds
        both faces of one axis: bz > 64 with both z neighbours, by > 32 with
        both y neighbours, bx >= 2 with both x neighbours)."""
        n = b.nbr_dirs
        return (self.xy_from_interior and self.z_slots and bool(n)
                and (b.bz + 2) % 2 == 0 and b.fields[0].data_ptr() % 16 == 0
                and not (4 in n and 5 in n and b.bz <= 64)
                and not (2 in n and 3 in n and b.by <= 32)
                and not (0 in n and 1 in n and b.bx < 2))

    def fused_boxes(self, b: HaloBlock):
        """(interior box, boundary slabs) of a fused step: boxes(), except
        that with z_interior the interior keeps whole z rows and the z slabs
        are dropped."""
        inner, shells = self.boxes(b)
        if not self.z_interior(b):
            return inner, shells
        inner = (inner[0], inner[1], inner[2], inner[3], 1, b.bz + 1)
        return inner, [x for x in shells if x[5] - x[4] > 1]

    def _box(self, b: HaloBlock, box, res_ptr, stream) -> None:
        if box[0] < box[1] and box[2] < box[3] and box[4] < box[5]:
            _lib.call("hx_stencil_box", b.field_ptr(), b.field_ptr(b.cur ^ 1), b.bx, b.by, b.bz,
                      *box, res_ptr, stream.cuda_stream)

    # ------------------------------------------- NCCL comparison exchange --

    def _nccl_buffers(self) -> None:
        self._sbuf, self._rbuf = {}, {}
        for r, b in self.blocks.items():
            dev = torch.device("cuda", b.device)
            self._sbuf[r] = {d: torch.empty(b.face_elems[d], dtype=torch.float64, device=dev)
                             for d in b.nbr_dirs}
            self._rbuf[r] = {d: torch.empty(b.face_elems[d], dtype=torch.float64, device=dev)
                             for d in b.nbr_dirs}

    def _step_nccl(self, residual, timing) -> None:
        """Baseline exchange (the north star's comparison point): pack into
        local buffers, grouped NCCL send/recv (batch_isend_irecv), unpack,
        sweep — the way a framework without persistent channels does it."""
        it = self.it
        mark = _Marks(timing)
        for b in self.blocks.values():
            s = self.stream_of(b)
            _lib.call("hx_set_device", b.device)
            with torch.cuda.stream(s):
                if b.nbr_dirs:
                    mark.begin("exchange", b, s)
                    for d in b.nbr_dirs:
                        _lib.call("hx_pack", b.field_ptr(), b.bx, b.by, b.bz, d,
                                  self._sbuf[b.rank][d].data_ptr(), s.cuda_stream)
                    ops = []
                    for d in b.nbr_dirs:
                        ops.append(self.dist.P2POp(self.dist.isend, self._sbuf[b.rank][d], b.neighbors[d]))
                        ops.append(self.dist.P2POp(self.dist.irecv, self._rbuf[b.rank][d], b.neighbors[d]))
                    for w in self.dist.batch_isend_irecv(ops):
                        w.wait()
                    for d in b.nbr_dirs:
                        _lib.call("hx_unpack", b.field_ptr(), b.bx, b.by, b.bz, d,
                                  self._rbuf[b.rank][d].data_ptr(), s.cuda_stream)
                    mark.end("exchange", b, s)
                mark.begin("sweep", b, s)
                self._relax(b, self._res_ptr(b, it, residual))
                mark.end("sweep", b, s)
        self.it += 1

    def _step_overlap(self, residual: bool, timing) -> None:
        """Interior sweep concurrent with the halo exchange (paper §4.3's
        overlap): comm stream = put, wait, unpack; main stream = interior
        box, then (after the halo event) the boundary slabs."""
        it, p = self.it, self.it & 1
        blocks = list(self.blocks.values())
        mark = _Marks(timing)
        halo_done = {}
        for b in blocks:  # phase 1: puts (comm stream, after the last sweep)
            if not b.nbr_dirs:
                continue
            _lib.call("hx_set_device", b.device)
            s, c = self.stream_of(b), self.comm[b.device]
            ready = torch.cuda.Event()
            ready.record(s)
            c.wait_event(ready)
            mark.begin("exchange", b, c)
            dst = [b.put_slot(d, p) if d in b.nbr_dirs else None for d in range(NDIRS)]
            flg = [b.put_flag[d] if d in b.nbr_dirs else None for d in range(NDIRS)]
            _lib.call("hx_pack_put", b.field_ptr(), b.bx, b.by, b.bz, b.dir_mask,
                      _lib.ptr_array(dst), _lib.ptr_array(flg), it + 1, b.counters_ptr,
                      c.cuda_stream)
        for b in blocks:  # phase 2: one-thread flag waits, then unpacks (comm stream)
            if not b.nbr_dirs:
                continue
            _lib.call("hx_set_device", b.device)
            c = self.comm[b.device]
            for d in b.nbr_dirs:
                _lib.call("hx_wait_flag", b.flag_ptr(d), it + 1, self.timeout_ns, b.err_ptr,
                          c.cuda_stream)
            for d in b.nbr_dirs:
                _lib.call("hx_unpack", b.field_ptr(), b.bx, b.by, b.bz, d, b.slot_ptr(p, d),
                          c.cuda_stream)
            mark.end("exchange", b, c)
            ev = torch.cuda.Event()
            ev.record(c)
            halo_done[b.rank] = ev
        for b in blocks:  # phase 3: interior boxes (main stream)
            _lib.call("hx_set_device", b.device)
            s = self.stream_of(b)
            inner, _ = self.boxes(b)
            rp = self._res_ptr(b, it, residual)
            mark.begin("sweep", b, s)
            mark.begin("interior", b, s)
            self._box(b, inner, rp, s)
            mark.end("interior", b, s)
        for b in blocks:  # phase 4: wait for the halo, boundary slabs
            _lib.call("hx_set_device", b.device)
            s = self.stream_of(b)
            _, shells = self.boxes(b)
            rp = self._res_ptr(b, it, residual)
            mark.begin("exposed", b, s)
            if b.rank in halo_done:
                s.wait_event(halo_done[b.rank])
            mark.end("exposed", b, s)
            mark.begin("shell", b, s)
            for box in shells:
                self._box(b, box, rp, s)
            mark.end("shell", b, s)
            mark.end("sweep", b, s)
            b.cur ^= 1
        self.it += 1

    # ------------------------------------------------------- fused mode --

    def _prime(self) -> None:
        """Before the first fused step: one channel exchange (pack_put +
        wait_unpack, flags -> 1) so cur's ghost planes hold the neighbours'
        initial boundary — afterwards every boundary value travels inside
        hx_shell_put."""
        for b in self.blocks.values():
            if b.nbr_dirs:
                _lib.call("hx_set_device", b.device)
                self._put(b, 0)
        for b in self.blocks.values():
            if b.nbr_dirs:
                _lib.call("hx_set_device", b.device)
                self._wait(b, 0)

    def _step_fused(self, residual, timing, devices=None, dev_step=False) -> None:
        """exchange="fused": per block, the comm stream runs ONE kernel that
        waits for the neighbours' previous boundary, relaxes the boundary
        shell and stores the neighbour-facing planes straight into the
        neighbours' nxt ghost planes over NVLink, then releases their flags
        (hx_shell_put); the main stream sweeps the interior concurrently.
        The step's work is complete on the main stream (it waits for the
        shell), so the next interior sees this step's boundary.

        devices: only the blocks on these GPUs (graph capture, one graph per
        GPU); dev_step: flag values come from each block's device step
        counter instead of the host's iteration number (graph replays)."""
        it = self.it
        if it == 0:
            self._prime()
        blocks = [b for b in self.blocks.values() if devices is None or b.device in devices]
        mark = _Marks(timing)
        shell_done = {}
        # residual slots first: a new slot is zero-filled on the main stream
        # before `ready` is recorded, so the shell's atomics follow the fill
        rps = {b.rank: self._res_ptr(b, it, residual) for b in blocks}
        if self._zstep_stale:  # a persistent run advanced the steps without hx_zsignal
            for b in self.blocks.values():
                with torch.cuda.stream(self.stream_of(b)):
                    b.zstep_dev.fill_(it)
            self._zstep_stale = False
        for b in blocks:
            if not b.nbr_dirs or self.sweep_exchange(b):
                continue
            _lib.call("hx_set_device", b.device)
            s, c = self.stream_of(b), self.comm[b.device]
            ready = torch.cuda.Event()
            ready.record(s)  # the previous interior (and shell) finished
            c.wait_event(ready)
            _, shells = self.fused_boxes(b)
            zint = self.z_interior(b)
            flat = (ctypes.c_int * (6 * len(shells)))(*[v for box in shells for v in box])
            nxt = b.cur ^ 1  # every block flips in lock step: the peer's nxt too
            remote = [b.peer_fields[d][nxt] if d in b.nbr_dirs else None for d in range(NDIRS)]
            wait = [b.flag_ptr(d) if d in b.nbr_dirs else None for d in range(NDIRS)]
            # with z_interior the z flags are released after both kernels (hx_zsignal)
            signal = [b.put_flag[d] if d in b.nbr_dirs and not (zint and d >= 4) else None
                      for d in range(NDIRS)]
            base = 0 if dev_step else it
            zin, zout = self._zslots(b, it)
            mark.begin("exchange", b, c)
            _lib.call("hx_shell_put_z", b.field_ptr(), b.field_ptr(nxt), b.bx, b.by, b.bz,
                      len(shells), flat, _lib.ptr_array(remote), _lib.ptr_array(wait), base + 1,
                      _lib.ptr_array(signal), base + 2, b.counters_ptr + 4, self.timeout_ns,
                      b.err_ptr, rps[b.rank], b.step_ptr if dev_step else None, zin, zout,
                      c.cuda_stream)
            mark.end("exchange", b, c)
            ev = torch.cuda.Event()
            ev.record(c)
            shell_done[b.rank] = ev
        # every local interior is enqueued before any main stream waits for
        # a shell, so blocks sharing a GPU do not serialise their interiors
        # behind each other's (spinning) boundary kernels
        for b in blocks:
            _lib.call("hx_set_device", b.device)
            s = self.stream_of(b)
            rp = rps[b.rank]
            mark.begin("sweep", b, s)
            mark.begin("interior", b, s)
            if self.sweep_exchange(b):  # the whole step: one sweep with every face
                nxt = b.cur ^ 1
                zin, zout = self._zslots(b, it)
                flags = [b.flag_ptr(d) if d in b.nbr_dirs else None for d in range(NDIRS)]
                peers = [b.peer_fields[d][nxt] if d in b.nbr_dirs and d < 4 else None
                         for d in range(NDIRS)]
                sig = [b.put_flag[d] if d in b.nbr_dirs else None for d in range(NDIRS)]
                # the sweep's last edge tile releases the flags (arena counter 2)
                _lib.call("hx_stencil_exchange", b.field_ptr(), b.field_ptr(nxt), b.bx, b.by,
                          b.bz, rp, _lib.ptr_array(flags), _lib.ptr_array(peers),
                          b.zstep_dev.data_ptr(), zin, zout, _lib.ptr_array(sig),
                          b.counters_ptr + 8, self.timeout_ns, b.err_ptr, s.cuda_stream)
            elif b.nbr_dirs and self.z_interior(b):
                inner, _ = self.fused_boxes(b)
                zin, zout = self._zslots(b, it)
                zflag = (ctypes.c_void_p * 2)(*[b.flag_ptr(d) if d in b.nbr_dirs else None
                                               for d in (4, 5)])
                _lib.call("hx_stencil_box_z", b.field_ptr(), b.field_ptr(b.cur ^ 1), b.bx, b.by,
                          b.bz, *inner, rp, zflag, b.zstep_dev.data_ptr(), zin, zout,
                          self.timeout_ns, b.err_ptr, s.cuda_stream)
            elif b.nbr_dirs:
                inner, _ = self.fused_boxes(b)
                self._box(b, inner, rp, s)
            else:
                _lib.call("hx_stencil", b.field_ptr(), b.field_ptr(b.cur ^ 1), b.bx, b.by, b.bz,
                          rp, s.cuda_stream)
            mark.end("interior", b, s)
        for b in blocks:
            _lib.call("hx_set_device", b.device)
            s = self.stream_of(b)
            mark.begin("exposed", b, s)
            if b.rank in shell_done:
                s.wait_event(shell_done[b.rank])
            mark.end("exposed", b, s)
            if self.sweep_exchange(b):
                pass  # the sweep released the flags itself (its last edge tile)
            elif b.nbr_dirs and self.z_interior(b):  # both kernels done: release the z flags
                zsig = (ctypes.c_void_p * 2)(*[b.put_flag[d] if d in b.nbr_dirs else None
                                              for d in (4, 5)])
                _lib.call("hx_zsignal", zsig, b.zstep_dev.data_ptr(), b.err_ptr, s.cuda_stream)
            mark.end("sweep", b, s)
            b.cur ^= 1
        self.it += 1

    def _zslots(self, b: HaloBlock, it: int):
        """z faces of the fused exchange travel through the arena slots
        (packed [i][j], contiguous) instead of the ghost columns: step it
        reads slot[it & 1] on each z side (filled by the neighbour's step
        it - 1, or by the priming exchange for it = 0) and writes the
        neighbour's slot[(it + 1) & 1]. The flag protocol is unchanged: the
        neighbour's flag >= it + 1 also says it finished reading the slot
        of that parity (its step it - 1)."""
        zin = (_lib.ctypes.c_void_p * 2)()
        zout = (_lib.ctypes.c_void_p * 2)()
        for h, d in enumerate((4, 5)):
            if d in b.nbr_dirs and self.z_slots:
                zin[h] = b.slot_ptr(it & 1, d)
                zout[h] = b.put_slot(d, (it + 1) & 1)
        return zin, zout

    def time_shell_alone(self, reps: int = 5) -> float | None:
        """Median ms of one block's hx_shell_put with nothing else running
        and no flag waits or releases: the fused exchange's own speed (its
        NVLink stores included). It rewrites exactly the boundary values the
        next step writes, so the run's state is unchanged."""
        b = next((b for b in self.blocks.values() if b.nbr_dirs), None)
        if b is None or self.exchange != "fused":
            return None
        _lib.call("hx_set_device", b.device)
        c = self.comm[b.device]
        self.synchronize()
        _, shells = self.fused_boxes(b)
        flat = (ctypes.c_int * (6 * len(shells)))(*[v for box in shells for v in box])
        nxt = b.cur ^ 1
        remote = [b.peer_fields[d][nxt] if d in b.nbr_dirs else None for d in range(NDIRS)]
        zin, zout = self._zslots(b, self.it)
        args = (b.field_ptr(), b.field_ptr(nxt), b.bx, b.by, b.bz, len(shells), flat,
                _lib.ptr_array(remote), _lib.ptr_array([None] * 6), 0, _lib.ptr_array([None] * 6),
                0, b.counters_ptr + 4, self.timeout_ns, b.err_ptr, None, None, zin, zout,
                c.cuda_stream)
        _lib.call("hx_shell_put_z", *args)  # warm (tensor maps, attributes)
        times = []
        back_to_back = 8  # launches per timing: the host's submit cost stays off the clock
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(c)
            for _ in range(back_to_back):
                _lib.call("hx_shell_put_z", *args)
            e1.record(c)
            c.synchronize()
            times.append(e0.elapsed_time(e1) / back_to_back)
        return sorted(times)[len(times) // 2]

    def run_graph(self, iters: int) -> None:
        """``iters`` fused iterations replayed from CUDA graphs: two steps
        (one buffer-parity period) of every local block are captured once
        per GPU, and each graph is replayed with the flag values taken from
        the blocks' device step counters, so the host enqueues one launch
        per GPU per two iterations. Same kernels and bits as run(); no
        residual or timing. GPUs synchronise only through the channel
        flags, whose waits always point at an earlier step."""
        if self.exchange != "fused":
            raise ValueError("run_graph needs exchange='fused'")
        if iters <= 0:
            return
        if self.it == 0:  # the priming exchange and step 0 stay outside the graph
            self.step()
            iters -= 1
        # the device step counters first: a capture must not record these fills
        for b in self.blocks.values():
            with torch.cuda.stream(self.stream_of(b)):
                b.step_dev.fill_(self.it)
                b.zstep_dev.fill_(self.it)
        self._zstep_stale = False
        parity = next(iter(self.blocks.values())).cur
        graphs = self._graphs.get(parity)
        if graphs is None:
            graphs = self._graphs[parity] = self._capture_pair()
        for _ in range(iters // 2):
            for d, g in graphs.items():
                with torch.cuda.device(d), torch.cuda.stream(self.streams[d]):
                    g.replay()
        self.it += 2 * (iters // 2)
        if iters % 2:
            self.step()

    def _capture_pair(self) -> dict:
        self.synchronize()
        graphs = {}
        for d, s in self.streams.items():
            g = torch.cuda.CUDAGraph()
            it0 = self.it
            with torch.cuda.device(d), torch.cuda.graph(g, stream=s):
                for _ in range(2):
                    self._step_fused(False, None, devices={d}, dev_step=True)
            self.it = it0  # capture only recorded the steps (each block flipped twice)
            graphs[d] = g
        return graphs

    def run_persistent(self, iters: int) -> None:
        """``iters`` fused iterations with ONE kernel launch per block
        (hx_persist_run: persistent CTAs, a grid barrier between
        iterations, the same neighbour flags as the fused steps). Meant for
        small blocks, where a step is ~1 us of HBM work and launches and
        their gaps dominate even in a graph replay. Blocks sharing a GPU run
        concurrently on their own streams with the SMs split between them
        (their kernels wait on each other's flags, so all must be resident).
        Same bits as run(); no residual."""
        if self.exchange != "fused":
            raise ValueError("run_persistent needs exchange='fused'")
        if iters <= 0:
            return
        if self.it == 0:  # the priming exchange and step 0 stay outside (as run_graph)
            self.step()
            iters -= 1
            if iters == 0:
                return
        per_dev = {}
        for b in self.blocks.values():
            per_dev.setdefault(b.device, []).append(b)
        st = getattr(self, "_persist", None)
        if st is None:
            st = self._persist = {}
        for b in self.blocks.values():  # every run starts after the last step's work ...
            if b.rank not in st:
                st[b.rank] = (torch.cuda.Stream(device=b.device),
                              torch.zeros(2, dtype=torch.int32, device=f"cuda:{b.device}"))
            st[b.rank][0].wait_stream(self.stream_of(b))
        for dev, blocks in per_dev.items():  # ... all are launched (they wait on each other) ...
            sms = _lib.ctypes.c_int(0)
            _lib.call("hx_set_device", dev)
            _lib.call("hx_sm_count", dev, _lib.ctypes.byref(sms))
            cap = max(1, sms.value // len(blocks))
            for b in blocks:
                s, bar = st[b.rank]
                fields = (_lib.ctypes.c_void_p * 2)(*[f.data_ptr() for f in b.fields])
                peer = (_lib.ctypes.c_void_p * 12)()
                for d in b.nbr_dirs:
                    peer[2 * d], peer[2 * d + 1] = b.peer_fields[d]
                wait = [b.flag_ptr(d) if d in b.nbr_dirs else None for d in range(NDIRS)]
                signal = [b.put_flag[d] if d in b.nbr_dirs else None for d in range(NDIRS)]
                zin = (_lib.ctypes.c_void_p * 4)()
                zout = (_lib.ctypes.c_void_p * 4)()
                for q in (0, 1):  # both slot parities (as _zslots, per iteration)
                    a, z = self._zslots(b, q)
                    zin[2 * q], zin[2 * q + 1], zout[2 * q], zout[2 * q + 1] = a[0], a[1], z[0], z[1]
                _lib.call("hx_persist_run", fields, peer, b.bx, b.by, b.bz, b.cur, self.it, iters,
                          _lib.ptr_array(wait), _lib.ptr_array(signal), zin, zout, bar.data_ptr(),
                          cap, self.timeout_ns, b.err_ptr, s.cuda_stream)
        for b in self.blocks.values():  # ... and later steps follow every run
            self.stream_of(b).wait_stream(st[b.rank][0])
        for b in self.blocks.values():
            b.cur ^= iters & 1
        self.it += iters
        self._zstep_stale = True

    def run(self, iters: int, residual: bool = False) -> None:
        for _ in range(iters):
            self.step(residual)

    # ------------------------------------------------- host-buffer steps --

    def step_e2e(self, host_wall=None, res_out=None) -> None:
        """One iteration fed from / reported to HOST memory (public API).

        host_wall: pinned fp64 host tensor of (by+2)*(bz+2) values, the
        Dirichlet x=0 ghost plane (cl/jacobi3d.py:137-138), uploaded into
        every local block on the global x=0 face; res_out: pinned int64 host
        tensor with one slot per local block receiving the bit pattern of
        that block's max|nxt-cur| (cl/jacobi3d.py:197).
        The upload for step it only has to wait for the sweep of it-2 (the
        last reader of that buffer's ghost plane), so it overlaps the sweep
        of it-1; the residual read-back trails the sweep on a copy stream.
        """
        it = self.it
        st = self._e2e_state()
        blocks = list(self.blocks.values())
        for b in blocks:
            if host_wall is not None and b.coords[0] == 0:
                if host_wall.numel() != (b.by + 2) * (b.bz + 2) or host_wall.dtype != torch.float64:
                    raise ValueError(f"host_wall must hold {(b.by + 2) * (b.bz + 2)} fp64 values")
                if not host_wall.is_pinned():
                    raise ValueError("host_wall must be pinned host memory")
                cs = st["up"][b.device]
                prev = st["sweep_done"].get((b.rank, it - 2))
                if prev is not None:
                    cs.wait_event(prev)
                _lib.call("hx_set_device", b.device)
                _lib.call("hx_memcpy", b.field_ptr(), host_wall.data_ptr(),
                          host_wall.numel() * 8, cs.cuda_stream)
                up = torch.cuda.Event()
                up.record(cs)
                st["uploaded"][b.rank] = up
        slots = {}
        for b in blocks:
            _lib.call("hx_set_device", b.device)
            s = self.stream_of(b)
            up = st["uploaded"].pop(b.rank, None)
            if up is not None:
                s.wait_event(up)  # the sweep reads the uploaded ghost plane
            ring = st["ring"][b.rank]
            slot = it % ring.numel()
            if slot == 0:
                # the ring wraps: the slots are about to be zeroed, so the
                # reads of every earlier step's residual must have finished.
                # The read-back stream is in order, so its latest event
                # covers all of them.
                last = st["read_done"].get(b.device)
                if last is not None:
                    s.wait_event(last)
                with torch.cuda.stream(s):
                    ring.zero_()
            slots[b.rank] = ring.data_ptr() + 8 * slot
        self.step(residual=slots)  # same (overlapped) sequence as step()
        for b in blocks:
            s = self.stream_of(b)
            done = torch.cuda.Event()
            done.record(s)
            st["sweep_done"][(b.rank, it)] = done
            st["sweep_done"].pop((b.rank, it - 3), None)
            if res_out is not None:
                cs = st["down"][b.device]  # separate from the upload stream, which
                cs.wait_event(done)        # must not queue behind this sweep
                _lib.call("hx_memcpy", res_out.data_ptr() + 8 * blocks.index(b), slots[b.rank], 8,
                          cs.cuda_stream)
                read = torch.cuda.Event()
                read.record(cs)
                st["read_done"][b.device] = read

    def drain_e2e(self) -> None:
        st = self._e2e_state()
        for cs in list(st["up"].values()) + list(st["down"].values()):
            cs.synchronize()
        self.synchronize()

    def _e2e_state(self):
        st = getattr(self, "_e2e", None)
        if st is None:
            st = self._e2e = {
                "up": {d: torch.cuda.Stream(device=d) for d in self.streams},
                "down": {d: torch.cuda.Stream(device=d) for d in self.streams},
                "ring": {r: torch.zeros(self.e2e_ring_slots, dtype=torch.int64,
                                        device=f"cuda:{b.device}")
                         for r, b in self.blocks.items()},
                "sweep_done": {}, "uploaded": {}, "read_done": {},
            }
        return st

    def synchronize(self) -> None:
        for s in self.streams.values():
            s.synchronize()

    def check_errors(self) -> None:
        self.synchronize()
        for b in self.blocks.values():
            err = int(b.arena[72:76].view(torch.int32).item())
            if err != 0:
                raise RuntimeError(f"block {b.rank}: device error {err} ({_lib.error_string(err)})")

    # ------------------------------------------------------------ results --

    def interior_host(self, rank: int) -> np.ndarray:
        b = self.blocks[rank]
        out = np.empty((b.bx, b.by, b.bz))
        self.interior_into(rank, out)
        return out

    def interior_into(self, rank: int, out: np.ndarray) -> None:
        """Copy block ``rank``'s current interior into the host array view
        ``out`` (shape (bx, by, bz), any strides): chunks of whole padded
        x planes (about 64 MB, contiguous in HBM, so one plain D2H each) go
        device -> pinned staging (a ring of three, so two chunks' host
        copies overlap the next chunk's transfer), and host threads spread
        each chunk's interior rows into ``out``. The staging ring is kept per process
        (pinned allocation is slow). 1536^3 (29 GB): ~1.0 s with 16 threads,
        against ~21 s for a pageable .cpu() plus a second host copy; the
        host side (first touch of the output's pages) is the bound, PCIe
        D2H runs at ~49 GB/s (tools/prof_readback.py, tools/prof_pcie.py)."""
        from concurrent.futures import ThreadPoolExecutor

        b = self.blocks[rank]
        field = b.fields[b.cur]  # whole padded planes are contiguous: one plain D2H per chunk
        s = self.stream_of(b)
        py, pz = b.by + 2, b.bz + 2
        plane = py * pz * 8
        per = max(1, min(b.bx, (64 << 20) // plane))
        stages = _staging(per * plane, 3)
        cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1
        nthreads = max(1, min(int(os.environ.get("HX_READBACK_THREADS", 16)), cores))
        with ThreadPoolExecutor(nthreads) as pool:
            pending = [[] for _ in stages]
            with torch.cuda.device(b.device), torch.cuda.stream(s):
                for c, i in enumerate(range(0, b.bx, per)):
                    k = min(per, b.bx - i)
                    q = c % len(stages)
                    for f in pending[q]:  # the staging buffer's previous chunk is out
                        f.result()
                    st = stages[q][: k * plane].view(torch.float64).view(k, py, pz)
                    st.copy_(field[1 + i:1 + i + k], non_blocking=True)
                    s.synchronize()
                    host = st.numpy()  # ghost rows and columns are dropped by the host copy
                    pending[q] = [pool.submit(_copy_rows, out, host, i, r0, r1, b.by)
                                  for r0, r1 in _split(k * b.by, nthreads)]
            for fs in pending:
                for f in fs:
                    f.result()

    def residuals(self, rank: int) -> list:
        self.synchronize()
        return [float(t.cpu().numpy().view(np.float64)[0]) for t in self._res.get(rank, [])]

    def assemble(self, out: np.ndarray | None = None) -> np.ndarray:
        """Global interior (all blocks must be local), each block copied
        straight into its slice of the result (``out``, if given: a float64
        array of the global shape, e.g. one whose pages were touched ahead
        of time by prefault_host)."""
        if out is None:
            out = np.empty(self.dims)
        elif out.shape != tuple(self.dims) or out.dtype != np.float64:
            raise ValueError(f"out must be float64 {tuple(self.dims)}, got {out.dtype} {out.shape}")
        bx, by, bz = (self.dims[a] // self.grid[a] for a in range(3))
        for r in range(self.pes):
            ix, iy, iz = _block_coords(r, self.grid)
            self.interior_into(r, out[ix * bx:(ix + 1) * bx, iy * by:(iy + 1) * by,
                                      iz * bz:(iz + 1) * bz])
        return out

    def close(self) -> None:
        self.synchronize()
        for base in self._ipc_bases:
            _lib.raw("hx_ipc_close")(base)
        self._ipc_bases = []
