"""Transport parity on the GPU: the B200 Worker's masked matching against a
brute-force matcher over randomized op schedules, the eager/rendezvous
split, truncation and failed endpoints.

Model (the reference's matching rules, cl/transport.py:258-465 and its
brute-force checker pkg/tests/matching_reference.py): an arriving frame
takes the earliest posted receive whose (tag & mask) agrees; a posted
receive takes the earliest queued frame that agrees; probes peek the
queue the same way; frames from one sender arrive in send order. Every
schedule mixes host and HBM payloads and sinks across two workers (two
GPUs when present, so device moves are NVLink peer copies), with sizes on
both sides of the eager threshold.
"""

import random

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


class Model:
    """Brute-force matcher for one receiving worker."""

    def __init__(self):
        self.posted = []  # (tag, mask, recv_id)
        self.queued = []  # (tag, send_id)

    def arrive(self, tag, send_id):
        for i, (rtag, mask, rid) in enumerate(self.posted):
            if (tag & mask) == (rtag & mask):
                del self.posted[i]
                return rid
        self.queued.append((tag, send_id))
        return None

    def post(self, tag, mask, rid):
        for i, (qtag, sid) in enumerate(self.queued):
            if (qtag & mask) == (tag & mask):
                del self.queued[i]
                return sid
        self.posted.append((tag, mask, rid))
        return None

    def probe(self, tag, mask):
        for qtag, _ in self.queued:
            if (qtag & mask) == (tag & mask):
                return qtag
        return None


def payload(send_id, size):
    head = send_id.to_bytes(4, "little")
    body = bytes((send_id * 7 + i) & 0xFF for i in range(max(0, size - 4)))
    return (head + body)[:size]


@pytest.fixture(scope="module")
def group(cuda):
    from paper_2102_12416_b200.config import RuntimeConfig
    from paper_2102_12416_b200.transport import TransportGroup

    g = TransportGroup(RuntimeConfig(workers=2))
    ws = [g.create_worker(0), g.create_worker(1)]
    eps = {(a, b): ws[a].connect(b) for a in (0, 1) for b in (0, 1)}
    return g, ws, eps


def pump(workers, limit=200000):
    for _ in range(limit):
        for w in workers:
            w.progress()
        if all(w.idle for w in workers):
            return
    raise AssertionError("transport did not quiesce")


@pytest.mark.parametrize("seed", range(25))
def test_matching_equals_brute_force(group, seed):
    """40 schedules x 24 ops per seed (1000 schedules, the reference's
    sweep size): every delivery pairs the same send and receive as the
    model, with the sender's exact bytes, and the leftovers agree."""
    from paper_2102_12416_b200.completion import OK
    from paper_2102_12416_b200.tags import FULL_MASK

    g, ws, eps = group
    space = g.device_space
    thr = g.cfg.eager_threshold
    sizes = [1, 7, 64, 1000, thr - 1, thr, thr + 1, 3 * thr + 5, 40000]
    rng = random.Random(1000 + seed)
    tags = [rng.getrandbits(64) & ~(0xF << 60) for _ in range(5)]
    masks = [FULL_MASK, FULL_MASK, 0xFFFF_FFFF_0000_0000, 0xFF, 0]
    for _ in range(40):
        models = [Model(), Model()]
        sends, recvs, delivered, expect = {}, {}, {}, {}
        keep = []
        for op in range(24):
            kind = rng.random()
            dst = rng.randrange(2)
            if kind < 0.45:  # send to dst
                src = rng.randrange(2)
                sid = len(sends)
                size = rng.choice(sizes)
                tag = rng.choice(tags)
                data = payload(sid, size)
                if rng.random() < 0.6:
                    buf = space.alloc(src, max(size, 1))
                    space.host_to_device(buf, data)
                    body = buf.region(0, size)
                    keep.append(buf)
                else:
                    body = data
                sends[sid] = (dst, tag, data)
                ws[src].tag_send(eps[(src, dst)], tag, body, completion=lambda c: None)
                rid = models[dst].arrive(tag, sid)
                if rid is not None:
                    expect[rid] = sid
            elif kind < 0.9:  # post a receive on dst
                rid = len(recvs)
                tag, mask = rng.choice(tags), rng.choice(masks)
                cap = max(sizes)
                if rng.random() < 0.5:
                    sink = space.alloc(dst, cap)
                    keep.append(sink)
                else:
                    sink = bytearray(cap)
                recvs[rid] = sink
                ws[dst].tag_recv(tag, mask, cap, completion=lambda c, r=rid: delivered.setdefault(r, c),
                                 sink=sink)
                sid = models[dst].post(tag, mask, rid)
                if sid is not None:
                    expect[rid] = sid
            else:  # probe dst's unexpected queue
                tag, mask = rng.choice(tags), rng.choice(masks)
                pump(ws)
                got = ws[dst].tag_probe(tag, mask)
                want = models[dst].probe(tag, mask)
                assert (got[0] if got else None) == want
            pump(ws)
        assert set(delivered) == set(expect), (sorted(delivered), sorted(expect))
        for rid, sid in expect.items():
            comp = delivered[rid]
            _, tag, data = sends[sid]
            assert comp.status == OK and comp.length == len(data) and comp.tag == tag
            sink = recvs[rid]
            got = (space.device_to_host(sink, size=len(data)) if not isinstance(sink, bytearray)
                   else bytes(sink[:len(data)]))
            assert got == data, (rid, sid)
        # leftovers: the unmatched receives stay posted, unmatched frames queued
        for w, m in zip(ws, models):
            assert [r.tag for r in w.posted] == [t for t, _, _ in m.posted]
            assert [f.tag for f in w.unexpected] == [t for t, _ in m.queued]
            w.posted.clear()
            w.unexpected.clear()
        for b in keep:
            space.free(b)


def test_eager_rendezvous_split_and_truncation(group):
    from paper_2102_12416_b200.completion import OK, TRUNCATED
    from paper_2102_12416_b200.tags import FULL_MASK

    g, ws, eps = group
    space = g.device_space
    thr = g.cfg.eager_threshold
    for size in (thr - 1, thr, thr + 1, 4 << 20):
        data = random.Random(size).randbytes(size)
        src = space.alloc(0, size)
        space.host_to_device(src, data)
        sink = space.alloc(1, size)
        eager0, rts0 = ws[0].stats["tx_eager"], ws[0].stats["tx_rts"]
        got, sent = [], []
        ws[0].tag_send(eps[(0, 1)], 77 + size, src, completion=sent.append)
        ws[1].tag_recv(77 + size, FULL_MASK, size, completion=got.append, sink=sink)
        pump(ws)
        assert got[0].status == OK and sent[0].status == OK
        assert space.device_to_host(sink) == data
        rendezvous = size > thr
        assert ws[0].stats["tx_rts"] - rts0 == int(rendezvous)
        assert ws[0].stats["tx_eager"] - eager0 == int(not rendezvous)
        space.free(src)
        space.free(sink)
    # a frame longer than the posted capacity completes TRUNCATED
    src = space.alloc(0, 4096)
    space.host_to_device(src, bytes(4096))
    got = []
    ws[1].tag_recv(5, FULL_MASK, 100, completion=got.append, sink=bytearray(100))
    ws[0].tag_send(eps[(0, 1)], 5, src, completion=lambda c: None)
    pump(ws)
    assert got[0].status == TRUNCATED and got[0].length == 4096
    space.free(src)


def test_failed_endpoint_reports_transport_error(group):
    from paper_2102_12416_b200.completion import TRANSPORT_ERROR

    g, ws, eps = group
    ep = eps[(0, 1)]
    ep.failed = True
    try:
        out = []
        ws[0].tag_send(ep, 9, b"abc", completion=out.append)
        pump(ws)
        assert out[0].status == TRANSPORT_ERROR
    finally:
        ep.failed = False
