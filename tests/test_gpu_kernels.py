"""GPU parity of the libhx kernels against the CPU oracle (bit-exact).

Calls the C ABI (include/hx.h) through paper_2102_12416_b200._lib on
seeded inputs: the 6-neighbour stencil (TMA and generic variants, odd and
even extents, sub-boxes), the fused residual, face pack/unpack in all six
directions, the fused pack+put+signal / wait+unpack pair, and the
sequential 64^3 x 100 golden run of the reference.
"""

import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import jacobi_c, jacobi_np  # noqa: E402

GOLD_DIR = os.path.join(os.path.dirname(__file__), "golden")
GOLD = json.load(open(os.path.join(GOLD_DIR, "golden.json")))
ARR = np.load(os.path.join(GOLD_DIR, "golden.npz"))

SHAPES = [(1, 1, 1), (2, 3, 4), (8, 6, 10), (6, 14, 11), (16, 16, 16), (33, 47, 64),
          (20, 70, 130), (64, 64, 64), (5, 40, 258)]


@pytest.fixture(scope="module")
def hx(cuda):
    from paper_2102_12416_b200 import _lib

    _lib.call("hx_set_device", 0)
    yield _lib
    _lib.raw("hx_stencil_set_variant")(0)


def stream():
    return torch.cuda.current_stream().cuda_stream


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run_stencil(hx, cur, variant, res=False, box=None):
    bx, by, bz = (s - 2 for s in cur.shape)
    rng = np.random.default_rng(99)
    nxt0 = rng.standard_normal(cur.shape)  # ghosts must survive untouched
    c, n = dev(cur), dev(nxt0)
    r = torch.zeros(1, dtype=torch.int64, device="cuda")
    hx.raw("hx_stencil_set_variant")(variant)
    rp = r.data_ptr() if res else None
    if box is None:
        hx.call("hx_stencil", c.data_ptr(), n.data_ptr(), bx, by, bz, rp, stream())
    else:
        hx.call("hx_stencil_box", c.data_ptr(), n.data_ptr(), bx, by, bz, *box, rp, stream())
    torch.cuda.synchronize()
    return nxt0, n.cpu().numpy(), float(r.cpu().numpy().view(np.float64)[0])


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("variant", [0, 2, 3, 5])
def test_stencil_bitexact_vs_oracle(hx, shape, variant):
    rng = np.random.default_rng(sum(shape))
    cur = rng.standard_normal(tuple(s + 2 for s in shape))
    nxt0, got, res = run_stencil(hx, cur, variant, res=True)
    want = nxt0.copy()
    wres = jacobi_c.stencil_residual(cur, want, nthreads=2)
    assert got.tobytes() == want.tobytes()
    assert res == wres
    if variant == 0:
        thin = shape[1] < 8 or shape[2] < 16
        expect = 3 if thin else (1 if (shape[2] + 2) % 2 == 0 else 5)
        # TMA for every thick even-z box, the row-pair TMA pipeline for odd z
        assert hx.raw("hx_stencil_last_variant")() == expect


def test_div6_matches_correctly_rounded_division(hx):
    """The stencil's division (RN(1/6) product + one FMA correction) equals
    the library's correctly rounded division on 2^27 random bit patterns
    per exponent band, plus zeros, subnormals, extremes and non-finites."""
    g = torch.Generator(device="cuda").manual_seed(1234)
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    n = 1 << 27
    for lo, hi in ((0x3C0, 0x440), (0x000, 0x7FF), (0x3FE, 0x402)):
        bits = torch.randint(0, 1 << 52, (n,), generator=g, device="cuda", dtype=torch.int64)
        exp = torch.randint(lo, hi, (n,), generator=g, device="cuda", dtype=torch.int64)
        sign = torch.randint(0, 2, (n,), generator=g, device="cuda", dtype=torch.int64)
        x = (bits | (exp << 52) | (sign << 63)).view(torch.float64)
        hx.call("hx_div6_check", x.data_ptr(), n, bad.data_ptr(), stream())
    special = torch.tensor([0.0, -0.0, 5e-324, -5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
                            -1.7976931348623157e308, float("inf"), float("-inf"), float("nan"), 6.0,
                            3.0, 1.0] + [float.fromhex(h) for h in (
                            "0x1p-960", "0x1p1020", "0x1.fffffffffffffp-961", "0x1.0000000000001p1020")], dtype=torch.float64, device="cuda")
    hx.call("hx_div6_check", special.data_ptr(), special.numel(), bad.data_ptr(), stream())
    torch.cuda.synchronize()
    assert int(bad.item()) == 0


def test_tma_forced_on_even_z(hx):
    rng = np.random.default_rng(5)
    cur = rng.standard_normal((40, 36, 66))
    nxt0, got, _ = run_stencil(hx, cur, 1)
    want = nxt0.copy()
    jacobi_np.stencil(cur, want)
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("chunk", [1, 3, 7, 1000])
def test_tma_chunking_is_invisible(hx, chunk):
    rng = np.random.default_rng(chunk)
    cur = rng.standard_normal((31, 40, 70))
    hx.raw("hx_stencil_set_chunk")(chunk)
    try:
        nxt0, got, res = run_stencil(hx, cur, 1, res=True)
    finally:
        hx.raw("hx_stencil_set_chunk")(0)
    want = nxt0.copy()
    assert res == jacobi_c.stencil_residual(cur, want)
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("variant", [1, 2, 5])
def test_box_plus_shells_equal_full_sweep(hx, variant):
    """Interior box + six boundary slabs (the overlap split) == one sweep."""
    rng = np.random.default_rng(11)
    cur = rng.standard_normal((22, 36, 68))
    bx, by, bz = 20, 34, 66
    inner = (2, bx, 2, by, 2, bz)
    slabs = [(1, 2, 1, by + 1, 1, bz + 1), (bx, bx + 1, 1, by + 1, 1, bz + 1),
             (2, bx, 1, 2, 1, bz + 1), (2, bx, by, by + 1, 1, bz + 1),
             (2, bx, 2, by, 1, 2), (2, bx, 2, by, bz, bz + 1)]
    c = dev(cur)
    nxt0 = rng.standard_normal(cur.shape)
    n = dev(nxt0)
    for box in [inner] + slabs:
        hx.raw("hx_stencil_set_variant")(variant if box is inner else 0)
        hx.call("hx_stencil_box", c.data_ptr(), n.data_ptr(), bx, by, bz, *box, None, stream())
    hx.raw("hx_stencil_set_variant")(0)
    want = nxt0.copy()
    jacobi_np.stencil(cur, want)
    assert n.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("shape,kcol", [((20, 70, 66), 1), ((20, 70, 66), 66), ((9, 40, 130), 2),
                                         ((9, 40, 130), 129), ((3, 33, 6), 6)])
def test_z_column_kernel(hx, shape, kcol):
    """Variant 4 (one z column, aligned quad loads + lane shuffles) over
    every j, including warp edges and partial warps, with the residual."""
    rng = np.random.default_rng(kcol)
    bx, by, bz = shape
    cur = rng.standard_normal((bx + 2, by + 2, bz + 2))
    nxt0 = rng.standard_normal(cur.shape)
    c, n = dev(cur), dev(nxt0)
    r = torch.zeros(1, dtype=torch.int64, device="cuda")
    hx.raw("hx_stencil_set_variant")(4)
    try:
        hx.call("hx_stencil_box", c.data_ptr(), n.data_ptr(), bx, by, bz, 1, bx + 1, 1, by + 1,
                kcol, kcol + 1, r.data_ptr(), stream())
    finally:
        hx.raw("hx_stencil_set_variant")(0)
    full = nxt0.copy()
    jacobi_np.stencil(cur, full)
    want = nxt0.copy()
    want[1:-1, 1:-1, kcol] = full[1:-1, 1:-1, kcol]
    assert n.cpu().numpy().tobytes() == want.tobytes()
    delta = np.abs(full[1:-1, 1:-1, kcol] - cur[1:-1, 1:-1, kcol]).max()
    assert float(r.cpu().numpy().view(np.float64)[0]) == delta


def test_sequential_64_cubed_matches_reference_golden(hx):
    from paper_2102_12416_b200.jacobi3d import sequential_oracle

    field, res = sequential_oracle((64, 64, 64), 100)
    g = GOLD["seq_64_100"]
    assert hashlib.sha256(field.tobytes()).hexdigest() == g["sha256"]
    assert [r.hex() for r in res] == g["residuals_hex"]


def test_sequential_custom_boundaries(hx):
    from paper_2102_12416_b200.jacobi3d import sequential_oracle

    f, _ = sequential_oracle((12, 10, 14), 7, hot=0.75, background=0.125, fill=0.5)
    assert f.tobytes() == ARR["seq_12x10x14_7_custom"].tobytes()


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_pack_unpack_match_reference_fixtures(hx, tag):
    meta = GOLD[f"block_{tag}"]
    field = ARR[f"pack_{tag}_field"]
    bx, by, bz = (s - 2 for s in field.shape)
    f = dev(field)
    for d in meta["nbr_dirs"]:
        want = ARR[f"pack_{tag}_face{d}"]
        out = torch.full((want.size,), float("nan"), dtype=torch.float64, device="cuda")
        hx.call("hx_pack", f.data_ptr(), bx, by, bz, d, out.data_ptr(), stream())
        assert out.cpu().numpy().tobytes() == want.tobytes()
    for d in meta["nbr_dirs"]:
        face = dev(ARR[f"unpack_{tag}_rstage{d}"])
        hx.call("hx_unpack", f.data_ptr(), bx, by, bz, d, face.data_ptr(), stream())
    assert f.cpu().numpy().tobytes() == ARR[f"unpack_{tag}_field"].tobytes()


@pytest.mark.parametrize("shape", [(3, 4, 5), (17, 9, 130), (64, 64, 64), (2, 2100, 3)])
def test_pack_unpack_all_dirs_random(hx, shape):
    rng = np.random.default_rng(len(shape) + sum(shape))
    field = rng.standard_normal(tuple(s + 2 for s in shape))
    f = dev(field)
    for d in range(6):
        want = jacobi_np.pack_face(field, d)
        out = torch.empty(want.size, dtype=torch.float64, device="cuda")
        hx.call("hx_pack", f.data_ptr(), *shape, d, out.data_ptr(), stream())
        assert out.cpu().numpy().tobytes() == want.tobytes(), d
        face = rng.standard_normal(want.shape)
        ref = field.copy()
        jacobi_np.unpack_face(ref, d, face)
        g = dev(field)
        hx.call("hx_unpack", g.data_ptr(), *shape, d, dev(face).data_ptr(), stream())
        assert g.cpu().numpy().tobytes() == ref.tobytes(), d


def test_fused_pack_put_wait_unpack_roundtrip(hx):
    """Two blocks on one stream: puts (with flag release) then waits."""
    import ctypes

    rng = np.random.default_rng(3)
    shape = (12, 10, 16)
    a = rng.standard_normal(tuple(s + 2 for s in shape))
    slots = torch.zeros(6 * 4096, dtype=torch.float64, device="cuda")
    flags = torch.zeros(8, dtype=torch.int64, device="cuda")
    ctr = torch.zeros(8, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    fa = dev(a)
    V = ctypes.c_void_p * 6
    dst = V(*[slots.data_ptr() + 8 * 4096 * d for d in range(6)])
    flg = V(*[flags.data_ptr() + 8 * d for d in range(6)])
    hx.call("hx_pack_put", fa.data_ptr(), *shape, 0b111111, dst, flg, 7, ctr.data_ptr(), stream())
    b = rng.standard_normal(a.shape)
    fb = dev(b)
    hx.call("hx_wait_unpack", fb.data_ptr(), *shape, 0b111111, dst, flg, 7, int(5e9),
            err.data_ptr(), stream())
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    assert flags.cpu().numpy()[:6].tolist() == [7] * 6
    assert ctr.cpu().numpy()[:6].tolist() == [0] * 6  # counters re-armed
    ref = b.copy()
    for d in range(6):
        jacobi_np.unpack_face(ref, d, jacobi_np.pack_face(a, d))
    assert fb.cpu().numpy().tobytes() == ref.tobytes()


def test_wait_times_out_instead_of_hanging(hx):
    flags = torch.zeros(1, dtype=torch.int64, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    hx.call("hx_wait_flag", flags.data_ptr(), 1, int(2e7), err.data_ptr(), stream())
    torch.cuda.synchronize()
    assert int(err.item()) == -2  # HX_E_TIMEOUT


def test_medium_block_vs_threaded_c_oracle(hx):
    """A 190 x 200 x 390 block (partial TMA tiles in j and k) over 3 sweeps."""
    rng = np.random.default_rng(17)
    cur = rng.standard_normal((192, 202, 392))
    c, n = dev(cur), dev(cur)
    h_cur, h_nxt = cur.copy(), cur.copy()
    for _ in range(3):
        hx.call("hx_stencil", c.data_ptr(), n.data_ptr(), 190, 200, 390, None, stream())
        c, n = n, c
        jacobi_c.stencil(h_cur, h_nxt)
        h_cur, h_nxt = h_nxt, h_cur
    assert c.cpu().numpy().tobytes() == h_cur.tobytes()


@pytest.mark.parametrize("k0", [1, 2])
def test_tma_stencil_under_concurrent_face_traffic(hx, k0):
    """Regression: face kernels on a second (high-priority) stream while the
    TMA stencil sweeps must not perturb its output. Before the prologue
    barrier consumed its shared loads, SM contention let the stage-0 refill
    overwrite plane 0 under a still-queued LDS (wrong first plane of a
    chunk, thousands of cells per 20 sweeps at this size)."""
    n = 512
    g = torch.Generator(device="cuda").manual_seed(3)
    cur = torch.randn((n + 2,) * 3, dtype=torch.float64, device="cuda", generator=g)
    other = torch.randn_like(cur)
    slot = torch.zeros(n * n * 6, dtype=torch.float64, device="cuda")
    box = (1, n + 1, 1, n + 1, k0, n + 1)
    hx.raw("hx_stencil_set_variant")(1)
    ref = torch.zeros_like(cur)
    hx.call("hx_stencil_box", cur.data_ptr(), ref.data_ptr(), n, n, n, *box, None, stream())
    torch.cuda.synchronize()
    S, C = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)
    bad = 0
    for _ in range(12):
        out = torch.zeros_like(cur)
        torch.cuda.synchronize()
        for _ in range(8):
            for d in range(6):
                hx.call("hx_pack", other.data_ptr(), n, n, n, d, slot.data_ptr(), C.cuda_stream)
                hx.call("hx_unpack", other.data_ptr(), n, n, n, d, slot.data_ptr(), C.cuda_stream)
        hx.call("hx_stencil_box", cur.data_ptr(), out.data_ptr(), n, n, n, *box, None, S.cuda_stream)
        torch.cuda.synchronize()
        bad += int((out != ref).sum().item())
    hx.raw("hx_stencil_set_variant")(0)
    assert bad == 0


def test_harmonic_fields_are_fixed_points(hx):
    """pkg/tests/test_jacobi.py:83-98's fixed-point property on the device:
    a constant field and an integer-valued linear field (harmonic, and every
    intermediate sum exact) come back bit-identical from one sweep."""
    for shape in ((16, 16, 16), (9, 20, 34)):
        i, j, k = np.meshgrid(*[np.arange(s + 2, dtype=np.float64) for s in shape], indexing="ij")
        for field in (np.full(i.shape, 0.5), i + 2 * j - 3 * k):
            _, out, _ = run_stencil(hx, field, 0)
            assert out[1:-1, 1:-1, 1:-1].tobytes() == field[1:-1, 1:-1, 1:-1].tobytes()


def test_residual_monotone_after_ten_iterations(hx):
    """Hot-wall run 64^3 x 60: the residual history is finite and never
    increases from iteration 10 on (pkg/tests/test_jacobi.py:83-98)."""
    from paper_2102_12416_b200.jacobi3d import sequential_oracle

    _, res = sequential_oracle((64, 64, 64), 60)
    assert all(np.isfinite(res)) and res[0] > 0
    assert all(b <= a for a, b in zip(res[10:], res[11:]))


@pytest.mark.parametrize("shape", [(40, 70, 129), (17, 65, 63), (5, 33, 1), (64, 64, 64), (9, 31, 33),
                                   (3, 2, 65)])
@pytest.mark.parametrize("chunk", [0, 1, 5])
def test_row_pipeline_odd_z_and_chunks(hx, shape, chunk):
    """Variant 5 (parity-class tensor maps: even and odd rows staged by two
    boxes with their own alignment shifts) on odd row pitches and odd plane
    sizes, partial tiles and chunkings, with the residual."""
    rng = np.random.default_rng(sum(shape) + chunk)
    cur = rng.standard_normal(tuple(s + 2 for s in shape))
    hx.raw("hx_stencil_set_chunk")(chunk)
    try:
        nxt0, got, res = run_stencil(hx, cur, 5, res=True)
    finally:
        hx.raw("hx_stencil_set_chunk")(0)
    want = nxt0.copy()
    assert res == jacobi_c.stencil_residual(cur, want)
    assert got.tobytes() == want.tobytes()


def test_row_pipeline_odd_z_sub_boxes(hx):
    """Interior box + shells of an odd-z block through the auto selection
    (row-pair TMA interior) equal one sweep."""
    rng = np.random.default_rng(21)
    bx, by, bz = 20, 40, 67
    cur = rng.standard_normal((bx + 2, by + 2, bz + 2))
    boxes = [(2, bx, 2, by, 2, bz), (1, 2, 1, by + 1, 1, bz + 1), (bx, bx + 1, 1, by + 1, 1, bz + 1),
             (2, bx, 1, 2, 1, bz + 1), (2, bx, by, by + 1, 1, bz + 1), (2, bx, 2, by, 1, 2),
             (2, bx, 2, by, bz, bz + 1)]
    c = dev(cur)
    nxt0 = rng.standard_normal(cur.shape)
    n = dev(nxt0)
    hx.raw("hx_stencil_set_variant")(0)
    for box in boxes:
        hx.call("hx_stencil_box", c.data_ptr(), n.data_ptr(), bx, by, bz, *box, None, stream())
        if box is boxes[0]:
            assert hx.raw("hx_stencil_last_variant")() == 5
    want = nxt0.copy()
    jacobi_np.stencil(cur, want)
    assert n.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("variant", [0, 2, 5])
def test_residual_propagates_nan_like_numpy(hx, variant):
    """max|nxt - cur| with a NaN in the field is NaN, as numpy's max makes it
    in the reference (cl/jacobi3d.py:197-198); the C oracle agrees. Without
    one, the residual is unchanged by the integer-pipe max."""
    rng = np.random.default_rng(7)
    shape = (12, 20, 35) if variant == 5 else (12, 20, 34)
    cur = rng.standard_normal(tuple(s + 2 for s in shape))
    _, _, clean = run_stencil(hx, cur, variant, res=True)
    want = cur.copy()
    assert clean == jacobi_c.stencil_residual(cur, want, nthreads=2) == jacobi_np.residual(cur, want)
    cur[5, 7, 9] = np.nan
    nxt0, got, res = run_stencil(hx, cur, variant, res=True)
    want = nxt0.copy()
    assert np.isnan(res)
    assert np.isnan(jacobi_c.stencil_residual(cur, want, nthreads=2))
    assert np.isnan(jacobi_np.residual(cur, want))
    # NaN payloads may differ between the GPU's and the host's arithmetic
    assert np.array_equal(got, want, equal_nan=True)
