"""GPU parity of the drop-in API: run_jacobi in all five modes, the
persistent-channel engine, Channel lockstep schedules, GPU Messaging
interleavings, the HBM device space and the OSU benches — the same
properties the reference's own tests pin (pkg/tests/test_jacobi.py,
test_channels.py, test_devmsg.py, test_devicesim.py, test_bench.py)."""

import hashlib
import json
import os
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def pkg(cuda):
    import paper_2102_12416_b200 as p

    return p


# ---------------------------------------------------------------- jacobi

@pytest.mark.parametrize("pes", [1, 2, 4, 8])
def test_run_jacobi_all_modes_match_reference_16(pkg, pes):
    from paper_2102_12416_b200.jacobi3d import MODES, run_jacobi

    for mode in MODES:
        r = run_jacobi(dims=(16, 16, 16), iters=5, mode=mode, pes=pes)
        assert sha(r["field"]) == GOLD["run_jacobi_sha256"][f"16x16x16/5/{pes}/{mode}"], mode


@pytest.mark.parametrize("pes", [2, 4])
def test_run_jacobi_all_modes_bitwise_32(pkg, pes):
    from paper_2102_12416_b200.jacobi3d import MODES, run_jacobi

    want = GOLD["seq_sha256"]["32x32x32/20"]
    for mode in MODES:
        r = run_jacobi(dims=(32, 32, 32), iters=20, mode=mode, pes=pes)
        assert sha(r["field"]) == want, mode


@pytest.mark.parametrize("pes", [1, 2, 4, 8])
def test_run_jacobi_persistent_mode(pkg, pes):
    """The B200 extension mode (persistent NVLink channels + overlap) through
    the reference's own entry point gives the reference's bits."""
    from paper_2102_12416_b200.jacobi3d import run_jacobi

    r = run_jacobi(dims=(16, 16, 16), iters=5, mode="channel-persistent", pes=pes, verify=True)
    assert sha(r["field"]) == GOLD["run_jacobi_sha256"][f"16x16x16/5/{pes}/channel-device"]
    assert r["max_err"] == 0.0 and r["total_ns"] > 0
    assert (r["comm_ns"] == 0.0) == (pes == 1)


def test_single_block_verify_and_no_comm(pkg):
    from paper_2102_12416_b200.jacobi3d import run_jacobi

    r = run_jacobi(dims=(16, 16, 16), iters=8, mode="channel-device", pes=1, verify=True)
    assert r["max_err"] == 0.0
    assert r["comm_ns"] == 0.0


def test_cli_csv(pkg, tmp_path):
    from paper_2102_12416_b200.jacobi3d import main

    out = tmp_path / "a.csv"
    assert main(["--dims", "16,16,16", "--iters", "5", "--mode", "channel-device", "--pes", "2",
                 "--verify", "--csv", str(out)]) == 0
    lines = out.read_text().strip().splitlines()
    assert lines[0] == "mode,pes,dims,iters,total_time,comm_time,unit,time_mode"
    row = lines[1].split(",")
    assert row[:4] == ["channel-device", "2", "16x16x16", "5"] and row[6:] == ["us", "wall"]
    assert main(["--dims", "64,64", "--iters", "1", "--pes", "1"]) == 2


@pytest.mark.parametrize("pes,dims,iters", [(1, (16, 16, 16), 5), (2, (16, 16, 16), 5),
                                            (4, (16, 16, 16), 5), (8, (16, 16, 16), 5),
                                            (2, (32, 32, 32), 20), (4, (32, 32, 32), 20)])
@pytest.mark.parametrize("exchange,overlap", [("p2p", False), ("p2p", True), ("fused", False)])
def test_halo_engine_matches_reference(pkg, pes, dims, iters, exchange, overlap):
    from paper_2102_12416_b200.halo import HaloJacobi

    eng = HaloJacobi(dims, pes, device_of=lambda r: 0, overlap=overlap, exchange=exchange)
    eng.run(iters)
    eng.check_errors()
    key = f"{dims[0]}x{dims[1]}x{dims[2]}/{iters}/{pes}/channel-device"
    want = GOLD["run_jacobi_sha256"].get(key) or GOLD["seq_sha256"][f"{dims[0]}x{dims[1]}x{dims[2]}/{iters}"]
    assert sha(eng.assemble()) == want
    eng.close()


@pytest.mark.parametrize("exchange,overlap", [("p2p", False), ("p2p", True), ("fused", False)])
def test_halo_engine_64_cubed_8_blocks_residuals(pkg, exchange, overlap):
    """Config C1 at 8 blocks: field sha and the full residual history
    (max over blocks) equal the reference's sequential oracle — with and
    without the interior/boundary overlap split."""
    from paper_2102_12416_b200.halo import HaloJacobi

    eng = HaloJacobi((64, 64, 64), 8, device_of=lambda r: 0, overlap=overlap, exchange=exchange)
    eng.run(100, residual=True)
    eng.check_errors()
    g = GOLD["seq_64_100"]
    assert sha(eng.assemble()) == g["sha256"]
    per_block = [eng.residuals(r) for r in range(8)]
    res = [max(col) for col in zip(*per_block)]
    assert [r.hex() for r in res] == g["residuals_hex"]
    eng.close()


@pytest.mark.parametrize("exchange,overlap", [("p2p", False), ("p2p", True), ("fused", False)])
def test_halo_engine_host_buffer_steps_match(pkg, exchange, overlap):
    """step_e2e (per-step pinned H2D of the hot wall, D2H of the residual)
    produces the reference's bits and residual history."""
    from paper_2102_12416_b200.halo import HaloJacobi

    eng = HaloJacobi((64, 64, 64), 2, device_of=lambda r: 0, overlap=overlap, exchange=exchange)
    assert eng.grid == (1, 1, 2)
    wall = torch.ones(66 * 34, dtype=torch.float64, pin_memory=True)
    host = torch.zeros(100, 2, dtype=torch.int64, pin_memory=True)
    for k in range(100):
        eng.step_e2e(wall, host[k])
    eng.drain_e2e()
    eng.check_errors()
    g = GOLD["seq_64_100"]
    assert sha(eng.assemble()) == g["sha256"]
    got = host.numpy().view(np.float64).max(axis=1)
    assert [float(r).hex() for r in got] == g["residuals_hex"]
    eng.close()


@pytest.mark.parametrize("exchange,overlap", [("p2p", False), ("p2p", True), ("fused", False)])
def test_halo_engine_b200_policy_8_blocks(pkg, exchange, overlap):
    """The 8-GPU bench layout under the B200 policy ((4,2,1), no z split)
    gives the reference's bits (decomposition invariance)."""
    from paper_2102_12416_b200.halo import HaloJacobi

    eng = HaloJacobi((32, 32, 32), 8, device_of=lambda r: 0, policy="b200", overlap=overlap,
                     exchange=exchange)
    assert eng.grid == (4, 2, 1)
    eng.run(20)
    eng.check_errors()
    assert sha(eng.assemble()) == GOLD["seq_sha256"]["32x32x32/20"]
    eng.close()


@pytest.mark.parametrize("pes,policy", [(2, "reference"), (2, "b200"), (4, "reference")])
@pytest.mark.parametrize("exchange", ["p2p", "fused"])
def test_halo_engine_overlap_at_scale(pkg, pes, policy, exchange):
    """Bench-sized blocks (512^3 split 2 or 4 ways), overlap on: the comm
    stream's face kernels share SMs with the TMA interior sweep for 30
    iterations, and the field must still equal the single-block sweep bit
    for bit (the small-size tests finish before kernels ever co-reside)."""
    from paper_2102_12416_b200.halo import HaloJacobi
    from paper_2102_12416_b200.jacobi3d import sequential_oracle

    dims = (512, 512, 512)
    want, _ = sequential_oracle(dims, 30)
    eng = HaloJacobi(dims, pes, device_of=lambda r: 0, policy=policy, overlap=exchange == "p2p",
                     exchange=exchange)
    eng.run(30)
    eng.check_errors()
    got = eng.assemble()
    eng.close()
    assert np.array_equal(got, want), int((got != want).sum())


@pytest.mark.parametrize("dims,pes", [((300, 301, 303), 2), ((260, 257, 255), 4)])
def test_fused_engine_odd_extents_at_scale(pkg, dims, pes):
    """Odd block extents (odd row pitch -> the row-pair TMA interior kernel,
    odd plane sizes, partial tiles) under the fused exchange for 25
    iterations equal the single-array sweep bit for bit."""
    from paper_2102_12416_b200.halo import HaloJacobi
    from paper_2102_12416_b200.jacobi3d import sequential_oracle

    want, _ = sequential_oracle(dims, 25)
    eng = HaloJacobi(dims, pes, device_of=lambda r: 0, policy="reference", exchange="fused")
    eng.run(25)
    eng.check_errors()
    got = eng.assemble()
    eng.close()
    assert np.array_equal(got, want), int((got != want).sum())


@pytest.mark.parametrize("exchange", ["p2p", "fused"])
def test_halo_engine_b200_policy_and_odd_sizes(pkg, exchange):
    from oracle import jacobi_np
    from paper_2102_12416_b200.halo import HaloJacobi

    dims = (24, 18, 30)
    eng = HaloJacobi(dims, 6, device_of=lambda r: 0, policy="b200", overlap=exchange == "p2p",
                     exchange=exchange)
    eng.run(9)
    eng.check_errors()
    want, _ = jacobi_np.sequential(dims, 9)
    assert eng.assemble().tobytes() == want.tobytes()
    eng.close()


# -------------------------------------------------------------- channels

def _content(direction, k, size):
    rng = random.Random(sum(direction.encode()) * 100003 + k)
    block = bytes(rng.randrange(256) for _ in range(64))
    return (block * ((size + 63) // 64))[:size]


def _streamer_cls(pkg):
    from paper_2102_12416_b200 import OK, Chare, entry

    class Streamer(Chare):
        def __init__(self):
            self.rbufs = {}
            self.done = False

        @entry
        def run_ops(self, cid, peer, ops, out_sizes, in_sizes, out_label, in_label):
            ch = self.channel(cid, peer)
            dev = self.runtime.device
            futs = []
            for kind, k, space in ops:
                if kind == "send":
                    data = _content(out_label, k, out_sizes[k])
                    if space == "dev":
                        buf = self.device_alloc(len(data))
                        dev.host_to_device(buf, data)
                        futs.append(ch.send(buf))
                    else:
                        futs.append(ch.send(data))
                else:
                    n = in_sizes[k]
                    if space == "dev":
                        sink = self.device_alloc(max(n, 1))
                        futs.append(ch.recv(sink, size=n))
                    else:
                        sink = bytearray(n)
                        futs.append(ch.recv(sink))
                    self.rbufs[k] = (space, sink, n)
            for f in futs:
                comp = yield f
                assert comp.status == OK
            self.done = True

        def read_back(self, k):
            space, sink, n = self.rbufs[k]
            if space == "dev":
                return self.runtime.device.device_to_host(sink, size=n) if n else b""
            return bytes(sink)

    return Streamer


@pytest.mark.parametrize("seed", range(12))
def test_channel_lockstep_random_schedules(pkg, seed):
    """cl/channels.py lockstep: kth recv gets kth send, any interleaving,
    host or HBM on either side, eager or rendezvous, zero envelopes."""
    from paper_2102_12416_b200 import Runtime, RuntimeConfig

    thr = 2048
    sizes_pool = (0, 1, 17, 300, thr - 1, thr, thr + 1, 9000, 40000)
    rng = random.Random(seed)

    def plan(n_out, n_in):
        kinds = ["send"] * n_out + ["recv"] * n_in
        rng.shuffle(kinds)
        ops, so, ro = [], 0, 0
        for kind in kinds:
            k = so if kind == "send" else ro
            ops.append((kind, k, rng.choice(("host", "dev"))))
            so, ro = (so + 1, ro) if kind == "send" else (so, ro + 1)
        return ops

    Streamer = _streamer_cls(pkg)
    rt = Runtime(RuntimeConfig(workers=2, eager_threshold=thr))
    rt.register(Streamer)
    placement = [0, 0] if seed % 4 == 3 else [0, 1]
    ids = rt.create(Streamer, 2, placement=placement)
    n_ab, n_ba = rng.randint(1, 8), rng.randint(0, 8)
    s_ab = [rng.choice(sizes_pool) for _ in range(n_ab)]
    s_ba = [rng.choice(sizes_pool) for _ in range(n_ba)]
    cid = rng.randrange(1 << 20)
    rt.launch(ids[0], "run_ops", cid, ids[1], plan(n_ab, n_ba), s_ab, s_ba, "ab", "ba")
    rt.launch(ids[1], "run_ops", cid, ids[0], plan(n_ba, n_ab), s_ba, s_ab, "ba", "ab")
    rt.run(timeout_s=60)
    a = rt.pe(placement[0]).chares[(0, 0)]
    b = rt.pe(placement[1]).chares[(0, 1)]
    assert a.done and b.done
    for k in range(n_ba):
        assert a.read_back(k) == _content("ba", k, s_ba[k])
    for k in range(n_ab):
        assert b.read_back(k) == _content("ab", k, s_ab[k])
    assert rt.total_envelopes_sent == 2  # the two launch seeds only; channels send none
    rt.close()


# --------------------------------------------------------- GPU messaging

def _msg_runtime(pkg, threshold=None):
    from paper_2102_12416_b200 import Chare, DeviceArg, Runtime, RuntimeConfig, entry

    class Sink(Chare):
        def __init__(self):
            self.heard = []
            self.stage = None

        def post_take(self, k, op, nbytes):
            self.stage = self.device_alloc(op.size)
            op.bind(self.stage)

        @entry
        def take(self, k, region, nbytes):
            self.heard.append((k, nbytes, self.runtime.device.device_to_host(region)))

    class Src(Chare):
        @entry
        def send_one(self, dest, k, nbytes):
            buf = self.device_alloc(nbytes)
            self.runtime.device.host_to_device(buf, bytes((k + i) % 256 for i in range(nbytes)))
            self.proxy(dest).take(k, DeviceArg(buf), nbytes)

    kw = {} if threshold is None else {"eager_threshold": threshold}
    rt = Runtime(RuntimeConfig(workers=2, **kw))
    rt.register(Sink)
    rt.register(Src)
    sinks = rt.create(Sink, 1, placement=[1])
    srcs = rt.create(Src, 1, placement=[0])
    rt.start()
    return rt, sinks[0], srcs[0]


@pytest.mark.parametrize("nbytes", [64, 65536])
def test_messaging_payload_first(pkg, nbytes):
    rt, sink, src = _msg_runtime(pkg)
    rt.launch(src, "send_one", sink, 3, nbytes)
    rt.run(timeout_s=30)
    obj = rt.pe(1).chares[(sink.collection, 0)]
    assert obj.heard == [(3, nbytes, bytes((3 + i) % 256 for i in range(nbytes)))]
    rt.close()


@pytest.mark.parametrize("nbytes", [64, 65536])
def test_messaging_envelope_first(pkg, nbytes):
    from paper_2102_12416_b200.tags import DEVICE

    rt, sink, src = _msg_runtime(pkg)
    w = rt.pe(1).worker
    w.hold = lambda frame: w.layout.kind_of(frame.tag) == DEVICE
    rt.launch(src, "send_one", sink, 7, nbytes)
    obj = rt.pe(1).chares[(sink.collection, 0)]
    rt.run(until=lambda: obj.stage is not None, timeout_s=10)
    assert obj.heard == [] and len(w._held) == 1
    w.hold = None
    w.release_held()
    rt.run(timeout_s=30)
    assert obj.heard == [(7, nbytes, bytes((7 + i) % 256 for i in range(nbytes)))]
    rt.close()


def test_messaging_entries_stay_in_send_order(pkg):
    from paper_2102_12416_b200 import Chare, DeviceArg, Runtime, RuntimeConfig, entry

    class Sink(Chare):
        def __init__(self):
            self.heard = []

        def post_take(self, k, op, n):
            op.bind(self.device_alloc(op.size))

        @entry
        def take(self, k, region, n):
            self.heard.append(k)

    class Burst(Chare):
        @entry
        def go(self, dest):
            big, small = self.device_alloc(200 * 1024), self.device_alloc(32)
            p = self.proxy(dest)
            p.take(1, DeviceArg(big), 1)
            p.take(2, DeviceArg(small), 2)

    rt = Runtime(RuntimeConfig(workers=2, eager_threshold=1024))
    rt.register(Sink)
    rt.register(Burst)
    s = rt.create(Sink, 1, placement=[1])
    b = rt.create(Burst, 1, placement=[0])
    rt.launch(b[0], "go", s[0])
    rt.run(timeout_s=30)
    assert rt.pe(1).chares[(s[0].collection, 0)].heard == [1, 2]
    rt.close()


def test_unbound_device_arg_aborts(pkg):
    from paper_2102_12416_b200 import Chare, DeviceArg, Runtime, RuntimeAbort, RuntimeConfig, entry

    class Lazy(Chare):
        def post_take(self, op):
            pass

        @entry
        def take(self, region):
            pass

    class Go(Chare):
        @entry
        def go(self, dest):
            self.proxy(dest).take(DeviceArg(self.device_alloc(16)))

    rt = Runtime(RuntimeConfig(workers=2))
    rt.register(Lazy)
    rt.register(Go)
    ids = rt.create(Lazy, 1, placement=[1])
    gs = rt.create(Go, 1, placement=[0])
    rt.launch(gs[0], "go", ids[0])
    with pytest.raises(RuntimeAbort, match="unbound"):
        rt.run(timeout_s=10)
    rt.close()


# ---------------------------------------------------------- device space

def test_device_space_registry_and_copies(pkg):
    from paper_2102_12416_b200.device import AllocationError, DeviceError, DeviceSpace

    space = DeviceSpace(lambda w: 0, capacity_per_worker=1 << 20)
    a = space.alloc(0, 100)
    b = space.alloc(1, 50)
    assert space.is_device_address(a.addr) and space.is_device_address(a.addr + 99)
    assert not space.is_device_address(a.addr - 1) and not space.is_device_address(0x1000)
    r = space.resolve(a.addr + 10, 20)
    assert r.buffer is a and r.offset == 10 and r.size == 20
    data = bytes(random.Random(3).randbytes(100))
    space.host_to_device(a, data)
    assert space.device_to_host(a) == data
    c = space.alloc(0, 100)
    space.device_to_device(c, a)
    assert space.device_to_host(c) == data
    with pytest.raises(DeviceError):
        space.host_to_device(b, bytes(51))
    with pytest.raises(AllocationError):
        space.alloc(0, 1 << 20)
    z = space.alloc(0, 0)
    assert space.is_device_address(z.addr)
    space.free(z)
    assert not space.is_device_address(z.addr)
    with pytest.raises(DeviceError):
        space.free(z)
    v = a.view(np.float64)
    v[:] = 1.5
    torch.cuda.synchronize()
    assert space.device_to_host(a)[:8] == np.float64(1.5).tobytes()


# ------------------------------------------------------------------ OSU

@pytest.mark.parametrize("api", ["charm-channel", "charm-messaging", "mpi"])
@pytest.mark.parametrize("mode", ["device", "host"])
def test_osu_latency_and_bandwidth_verify(pkg, api, mode):
    from paper_2102_12416_b200.osu import measure_bandwidth, measure_latency

    for size in (8, 65536):
        lat = measure_latency(api, mode, size, iters=4, warmup=1)
        assert lat["verified"] and lat["value_ns"] > 0
    bw = measure_bandwidth(api, mode, 1 << 20, window=8, iters=2, warmup=1)
    assert bw["verified"] and bw["value_gbps"] > 0


def test_osu_cli(pkg, tmp_path):
    from paper_2102_12416_b200.osu import main

    out = tmp_path / "b.csv"
    assert main(["--benchmark", "latency", "--api", "charm-channel", "--sizes", "8,4096",
                 "--iters", "3", "--csv", str(out)]) == 0
    assert out.read_text().splitlines()[0] == "benchmark,api,mode,size_bytes,metric,value,unit,time_mode"


@pytest.mark.parametrize("pes,dims,iters", [(1, (32, 32, 32), 9), (2, (64, 64, 64), 20),
                                            (8, (64, 64, 64), 21), (6, (24, 18, 30), 11)])
def test_fused_graph_replay_matches(pkg, pes, dims, iters):
    """HaloJacobi.run_graph (per-GPU CUDA graphs of two fused steps, flag
    values from device step counters) gives the eager path's bits, for odd
    and even iteration counts and after eager steps."""
    from oracle import jacobi_np
    from paper_2102_12416_b200.halo import HaloJacobi

    eng = HaloJacobi(dims, pes, device_of=lambda r: 0, policy="b200", exchange="fused")
    eng.run(3)
    eng.run_graph(iters - 5)
    eng.run(2)
    eng.check_errors()
    want, _ = jacobi_np.sequential(dims, iters)
    assert eng.assemble().tobytes() == want.tobytes()
    eng.close()


@pytest.mark.parametrize("dims,pes,policy", [((3, 2, 40), 6, "b200"), ((2, 3, 5), 6, "reference"),
                                             ((3, 4, 2), 12, "b200")])
@pytest.mark.parametrize("exchange,overlap", [("p2p", False), ("p2p", True), ("fused", False)])
def test_halo_engine_one_cell_thick_blocks(pkg, dims, pes, policy, exchange, overlap):
    """Blocks one or two cells thick: both faces of an axis on the same
    plane (the shells overlap, interior boxes are empty), every exchange."""
    from oracle import jacobi_np
    from paper_2102_12416_b200.halo import HaloJacobi

    eng = HaloJacobi(dims, pes, device_of=lambda r: 0, policy=policy, exchange=exchange,
                     overlap=overlap)
    eng.run(7)
    eng.check_errors()
    want, _ = jacobi_np.sequential(dims, 7)
    assert eng.assemble().tobytes() == want.tobytes()
    eng.close()


@pytest.mark.parametrize("dims,pes", [((48, 32, 40), 2), ((32, 32, 32), 8), ((30, 28, 26), 4),
                                      ((17, 19, 64), 2), ((64, 64, 64), 1)])
def test_persistent_kernel_run_bitexact(pkg, dims, pes):
    """HaloJacobi.run_persistent (one launch per block for many fused
    iterations: grid barriers, neighbour flags, peer ghost stores) gives the
    oracle's bits, alone and alternating with ordinary fused steps."""
    from oracle import jacobi_np
    from paper_2102_12416_b200.halo import HaloJacobi

    eng = HaloJacobi(dims, pes, device_of=lambda r: 0, exchange="fused", timeout_s=10)
    eng.run_persistent(9)
    eng.step()
    eng.run_persistent(6)
    eng.check_errors()
    want, _ = jacobi_np.sequential(dims, 16)
    assert eng.assemble().tobytes() == want.tobytes()
    eng.close()


@pytest.mark.parametrize("dims,pes,policy", [((128, 128, 64), 4, "b200"),
                                             ((64, 128, 128), 4, "reference")])
def test_exchange_soak_mixed_schedules_vs_one_block(pkg, dims, pes, policy):
    """Thousands of fused iterations on a random field — graph replays,
    persistent runs and eager steps alternating — on every visible GPU (round
    robin), bitwise equal to one block with no exchange after the same
    number of iterations (tools/soak.py runs the long version: 20 000
    iterations, profiles/r2_soak_2gpu.jsonl)."""
    import torch

    from paper_2102_12416_b200.halo import HaloJacobi

    ngpu = max(1, torch.cuda.device_count())
    eng = HaloJacobi(dims, pes, device_of=lambda r: r % ngpu, exchange="fused", policy=policy,
                     timeout_s=20)
    eng.fill_random(5)
    eng.synchronize()
    init = eng.assemble()
    sched = [("eager", 3), ("graph", 1000), ("persistent", 700), ("eager", 2), ("graph", 301)]
    for how, n in sched:
        {"eager": eng.run, "graph": eng.run_graph, "persistent": eng.run_persistent}[how](n)
    eng.check_errors()
    got = eng.assemble()
    eng.close()
    ref = HaloJacobi(dims, 1, device_of=lambda r: 0, exchange="fused", policy=policy)
    b = ref.blocks[0]
    b.fields[b.cur][1:-1, 1:-1, 1:-1].copy_(torch.from_numpy(init))
    torch.cuda.synchronize()
    ref.run(sum(n for _, n in sched))
    want = ref.assemble()
    ref.close()
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("dims,pes", [((48, 32, 40), 2), ((40, 96, 48), 2), ((64, 64, 64), 8),
                                      ((96, 96, 96), 27), ((40, 80, 136), 4), ((48, 40, 200), 3)])
def test_every_face_in_the_interior_sweep_bitexact(pkg, dims, pes):
    """HaloJacobi.xy_from_interior: the whole fused step is one sweep per
    block (hx_stencil_exchange: x / y faces stored straight into the
    neighbours' ghost planes / rows by the edge tiles, z faces through the
    slots) and hx_exchange_signal. Eager steps with the residual, graph
    replays and persistent runs alternate; (3,3,3) mixes blocks that qualify
    with middle blocks that do not (by = 32 with both y neighbours)."""
    from oracle import jacobi_np
    from paper_2102_12416_b200.halo import HaloJacobi

    eng = HaloJacobi(dims, pes, device_of=lambda r: 0, exchange="fused", timeout_s=10,
                     policy="reference")
    eng.xy_from_interior = True
    assert any(eng.sweep_exchange(b) for b in eng.blocks.values())
    eng.run(3, residual=True)
    eng.run_graph(4)
    eng.run_persistent(3)
    eng.run(2)
    eng.check_errors()
    want, wres = jacobi_np.sequential(dims, 12)
    assert eng.assemble().tobytes() == want.tobytes()
    got = [max(eng.residuals(r)[i] for r in eng.blocks) for i in range(3)]
    assert got == wres[:3]
    eng.close()


def test_persistent_kernel_timeout_stops_every_cta(pkg):
    """A neighbour that never runs: every CTA's flag wait times out, still
    arrives at the grid barrier, and the launch ends with HX_E_TIMEOUT in the
    block's error word instead of hanging the GPU."""
    import time

    from paper_2102_12416_b200.halo import HaloJacobi

    eng = HaloJacobi((48, 40, 32), 2, device_of=lambda r: 0, exchange="fused", timeout_s=0.5)
    eng.step()  # both blocks: flags for iteration 1 released
    both = eng.blocks
    eng.blocks = {0: both[0]}  # block 1 never runs: block 0 waits at iteration 2
    t0 = time.perf_counter()
    eng.run_persistent(4)
    eng.synchronize()
    elapsed = time.perf_counter() - t0
    eng.blocks = both
    assert elapsed < 20, elapsed
    with pytest.raises(RuntimeError, match="block 0: device error"):
        eng.check_errors()
    eng.close()


@pytest.mark.parametrize("dims,pes", [((32, 40, 64), 2), ((48, 48, 48), 8), ((40, 32, 96), 4),
                                      ((24, 32, 240), 3)])
def test_fused_z_faces_from_the_interior_sweep_bitexact(pkg, dims, pes):
    """The alternative z-face path (HaloJacobi.z_from_interior: hx_stencil_box_z
    edge tiles wait for the z flags, patch the ghost column from the slots
    and write the neighbour's slot; hx_zsignal releases the z flags) gives the
    oracle's bits, through eager steps, graph replays and persistent runs."""
    from oracle import jacobi_np
    from paper_2102_12416_b200.halo import HaloJacobi

    eng = HaloJacobi(dims, pes, device_of=lambda r: 0, exchange="fused", timeout_s=10,
                     policy="reference")
    eng.z_from_interior = True
    assert any(eng.z_interior(b) for b in eng.blocks.values())
    eng.run(3, residual=True)
    eng.run_graph(4)
    eng.run_persistent(3)
    eng.run(2)
    eng.check_errors()
    want, wres = jacobi_np.sequential(dims, 12)
    assert eng.assemble().tobytes() == want.tobytes()
    got = [max(eng.residuals(r)[i] for r in eng.blocks) for i in range(3)]
    assert got == wres[:3]
    eng.close()


def test_persistent_channel_two_streams_one_gpu(pkg):
    """pchannel.PersistentChannel with both endpoints on cuda:0 (two streams):
    LL, slot and pulled messages in both directions, interleaved, in order,
    bit-exact, with truncation — the device channel kernels on a 1-GPU box."""
    from paper_2102_12416_b200.completion import OK, TRUNCATED
    from paper_2102_12416_b200.pchannel import PersistentChannel

    rng = np.random.default_rng(5)
    slot = 70000
    ch = PersistentChannel(0, 0, slot_bytes=slot, depth=4, timeout_s=20, allow_same_gpu=True)
    s = [torch.cuda.Stream(device=0), torch.cuda.Stream(device=0)]
    # both directions at once: messages that fit a slot (a pulled send waits
    # for its receive, so two crossing pulls on two streams would each wait
    # behind the other's send); the pulled sizes go one way, below
    sizes = [8, 0, 4096, 8193, slot, 1, 65000, 17, 12345]
    msgs = [[torch.from_numpy(rng.integers(0, 256, n, dtype=np.uint8)).to("cuda:0") for n in sizes]
            for _ in (0, 1)]
    sinks = [[torch.zeros(max(sizes), dtype=torch.uint8, device="cuda:0") for _ in sizes]
             for _ in (0, 1)]
    tickets = [[], []]
    for k, n in enumerate(sizes):
        for e in (0, 1):
            ch.send(e, msgs[e][k], n, stream=s[e])
        for e in (0, 1):
            tickets[e].append(ch.recv(1 - e, sinks[e][k], max(sizes), stream=s[1 - e]))
    ch.check()
    for e in (0, 1):
        for k, n in enumerate(sizes):
            st, length = ch.completion(1 - e, tickets[e][k], max(sizes))
            assert st == OK and length == n, (e, k)
            assert torch.equal(sinks[e][k][:n].cpu(), msgs[e][k].cpu()), (e, k)
    small = torch.zeros(10, dtype=torch.uint8, device="cuda:0")
    ch.send(0, msgs[0][4], slot, stream=s[0])
    t = ch.recv(1, small, 10, stream=s[1])
    assert ch.completion(1, t, 10) == (TRUNCATED, slot)
    assert torch.equal(small.cpu(), msgs[0][4][:10].cpu())
    # pulled messages (larger than a slot), endpoint 0 -> 1, mixed with small ones
    big = [3 << 18, 8, 5 << 20, 70001]
    src = [torch.from_numpy(rng.integers(0, 256, n, dtype=np.uint8)).to("cuda:0") for n in big]
    dst = [torch.zeros(n, dtype=torch.uint8, device="cuda:0") for n in big]
    tk = []
    for k, n in enumerate(big):
        ch.send(0, src[k], n, stream=s[0])
        tk.append(ch.recv(1, dst[k], n, stream=s[1]))
    for k, n in enumerate(big):
        assert ch.completion(1, tk[k], n) == (OK, n)
        assert torch.equal(dst[k].cpu(), src[k].cpu()), k
    ch.check()
