"""CPU-only checks: the C-ABI library loads and exports every symbol
include/hx.h declares; host-side logic (tags, config, decomposition,
neighbour tables, arena layout, size parsing) matches the reference's
golden vectors. No compute calls (no GPU here)."""

import ctypes
import json
import os
import re

import pytest

from paper_2102_12416_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "hx.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char \*)\s*(hx_\w+)\s*\(", header, re.M))
    assert declared == set(_lib.EXPORTS)
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert _lib.load().hx_abi_version() == 1
    assert _lib.error_string(-2) == "hx: device flag wait timed out"


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass  # the stencil stages planes with TMA


def test_tag_codec_matches_reference():
    from paper_2102_12416_b200.tags import TagLayout

    lay = TagLayout()
    for cid, d, c, want in GOLD["tags"]["channel"]:
        assert lay.encode_channel(cid, d, c) == want
        dec = lay.decode(want)
        assert (dec.channel_id, dec.direction, dec.counter) == (cid, d, c)
    for kind, pe, c, want in GOLD["tags"]["messaging"]:
        assert lay.encode_messaging(kind, pe, c) == want
    assert lay.digest() == GOLD["tags"]["digest"]


def test_decompose_neighbors_match_reference():
    from paper_2102_12416_b200.jacobi3d import JacobiError, decompose, neighbor_table

    for key, want in GOLD["decompose"].items():
        dims_s, n = key.rsplit("/", 1)
        dims = tuple(int(x) for x in dims_s.strip("()").split(","))
        if want is None:
            with pytest.raises(JacobiError):
                decompose(dims, int(n))
        else:
            assert list(decompose(dims, int(n))) == want, key
    for g_s, tables in GOLD["neighbors"].items():
        grid = tuple(int(x) for x in g_s.strip("()").split(","))
        for r, want in enumerate(tables):
            assert neighbor_table(grid, r) == want


def test_b200_policy_minimises_weighted_face_cost():
    from paper_2102_12416_b200.jacobi3d import (_triples, decompose, decompose_b200,
                                                weighted_face_cost)

    for dims in ((64, 64, 64), (128, 64, 64), (3072, 3072, 3072), (96, 48, 24), (3072, 1536, 1536)):
        for n in (1, 2, 4, 8, 16):
            try:
                a, b = decompose(dims, n), decompose_b200(dims, n)
            except Exception:
                continue
            assert weighted_face_cost(dims, b) <= weighted_face_cost(dims, a)
            legal = [g for g in _triples(n) if all(dims[i] % g[i] == 0 for i in range(3))]
            assert weighted_face_cost(dims, b) == min(weighted_face_cost(dims, g) for g in legal)
    # the bench configurations
    assert decompose_b200((3072, 1536, 1536), 2) == (2, 1, 1)
    assert decompose_b200((3072, 3072, 1536), 4) == (2, 2, 1)
    assert decompose_b200((3072, 3072, 3072), 4) == (2, 2, 1)   # reference: (1, 2, 2)
    assert decompose_b200((3072, 3072, 3072), 8) == (4, 2, 1)   # reference: (2, 2, 2)
    assert decompose((64, 64, 64), 2) == (1, 1, 2)              # reference splits z
    assert decompose_b200((64, 64, 64), 2) == (2, 1, 1)


def test_config_rejects_virtual_time():
    from paper_2102_12416_b200.config import ConfigError, RuntimeConfig

    with pytest.raises(ConfigError):
        RuntimeConfig(time_mode="virtual")
    assert RuntimeConfig().time_mode == "wall"


def test_parse_sizes():
    from paper_2102_12416_b200.osu import BenchError, parse_sizes

    assert parse_sizes("1:4194304:x2")[-1] == 4194304 and len(parse_sizes("8:4194304:x2")) == 20
    assert parse_sizes("8,64,4096") == [8, 64, 4096]
    assert parse_sizes("1:10:+4") == [1, 5, 9]
    with pytest.raises(BenchError):
        parse_sizes("1:10:y2")


def test_readback_row_split_and_prefault():
    """The read-back helpers of HaloJacobi.interior_into: _split cuts the
    rows evenly, _copy_rows drops the staged planes' ghost rows / columns
    into any strided view of the result, prefault_host returns a touched
    (zero) array of the global shape."""
    import numpy as np

    from paper_2102_12416_b200.halo import _copy_rows, _split, prefault_host

    assert _split(10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert _split(2, 16) == [(0, 1), (1, 2)]
    assert _split(0, 4) == [(0, 0)]
    rng = np.random.default_rng(3)
    k, by, bz = 3, 5, 7
    host = rng.standard_normal((k, by + 2, bz + 2))
    glob = np.zeros((4 * k, 2 * by, 3 * bz))
    view = glob[k:2 * k, by:2 * by, bz:2 * bz]  # a block's slice of the global field
    for r0, r1 in _split(k * by, 4):
        _copy_rows(view, host, 0, r0, r1, by)
    assert np.array_equal(view, host[:, 1:-1, 1:-1])
    assert glob.sum() == view.sum()
    out, futs = prefault_host((6, 5, 4), threads=3)
    for f in futs:
        f.result()
    assert out.shape == (6, 5, 4) and out.dtype == np.float64 and not out.any()


def test_exchange_edge_item_count_matches_the_kernel_rule():
    """hx_exchange_edge_items (how many work items of the one-sweep fused
    step hold a face; its last edge tile releases the step, so a wrong count
    would hang the neighbours until the flag timeout) against a brute-force
    enumeration of the kernel's own schedule and classification
    (stencil_tma_kernel: tiles of TY x TZ, x chunks of 4 planes)."""
    import itertools
    import random

    TY, TZ, CHUNK = 32, 64, 4

    def brute(bx, by, bz, mask):
        chunk = min(CHUNK, bx)
        n = 0
        for jb in range(1, by + 1, TY):
            for kb in range(1, bz + 1, TZ):
                for ib in range(1, bx + 1, chunk):
                    last = min(ib + chunk, bx + 1) - 1
                    zlo = mask & 16 and kb == 1
                    zhi = mask & 32 and kb <= bz < kb + TZ
                    xy = ((mask & 1 and ib == 1) or (mask & 2 and last == bx)
                          or (mask & 4 and jb == 1) or (mask & 8 and jb <= by < jb + TY))
                    n += bool(zlo or zhi or xy)
        return n

    rng = random.Random(7)
    shapes = [(1, 1, 2), (4, 32, 64), (5, 33, 65), (8, 64, 130), (96, 96, 96), (13, 70, 200)]
    shapes += [(rng.randint(1, 40), rng.randint(1, 100), 2 * rng.randint(1, 120)) for _ in range(30)]
    got = ctypes.c_uint(0)
    fn = _lib.raw("hx_exchange_edge_items")
    for (bx, by, bz), mask in itertools.product(shapes, [1, 2, 3, 4, 8, 12, 16, 32, 48, 63, 21, 42]):
        assert fn(bx, by, bz, mask, ctypes.byref(got)) == 0
        assert got.value == brute(bx, by, bz, mask), (bx, by, bz, mask)
    assert fn(0, 4, 4, 1, ctypes.byref(got)) != 0


def test_hot_kernels_do_not_spill():
    """ptxas report of the shipped build (csrc/build/hx_stencil.ptxas.log):
    the stencil sweeps (plain TMA, odd-z pair, and the one-sweep fused step
    without the residual — the bench's step) and the exchange kernels keep
    everything in registers at their occupancy. A spill in these inner loops
    costs HBM-roofline fraction, so it fails here, before any GPU run."""
    import re

    log = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_2102_12416_b200", "csrc", "build", "hx_stencil.ptxas.log")
    if not os.path.exists(log):
        pytest.skip("no ptxas log (library not built here)")
    text = open(log).read()
    found = {}
    for entry in text.split("Compiling entry function '")[1:]:
        name = entry.split("'")[0]
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", entry)
        if m:
            found[name] = (int(m.group(1)), int(m.group(2)))
    must = [n for n in found if "stencil_tma_kernelILb0" in n or "stencil_pair_kernel" in n
            or "face_tma_kernel" in n or "persist_kernel" in n
            or ("stencil_tma_kernelILb1" in n and "Lb0EE" in n)]
    assert len(must) >= 8, sorted(found)
    for n in must:
        assert found[n] == (0, 0), (n, found[n])
