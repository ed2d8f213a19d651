"""CPU checks of the oracle itself against golden vectors frozen from the
reference (tests/golden/make_golden.py). No GPU needed."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import jacobi_c, jacobi_np

GOLD_DIR = os.path.join(os.path.dirname(__file__), "golden")
GOLD = json.load(open(os.path.join(GOLD_DIR, "golden.json")))
ARR = np.load(os.path.join(GOLD_DIR, "golden.npz"))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_numpy_oracle_pins_reference_64_cubed():
    f, res = jacobi_np.sequential((64, 64, 64), 100)
    g = GOLD["seq_64_100"]
    assert sha(f) == g["sha256"]
    assert [r.hex() for r in res] == g["residuals_hex"]


def test_c_oracle_bitwise_equals_reference_64_cubed():
    f, res = jacobi_c.sequential((64, 64, 64), 100, nthreads=3)
    g = GOLD["seq_64_100"]
    assert sha(f) == g["sha256"]
    assert [r.hex() for r in res] == g["residuals_hex"]


def test_small_fields_and_custom_boundaries():
    f, res = jacobi_np.sequential((16, 16, 16), 8)
    assert np.array_equal(f, ARR["seq_16_8"])
    assert [r.hex() for r in res] == GOLD["seq_16_8_residuals_hex"]
    f2, _ = jacobi_c.sequential((12, 10, 14), 7, hot=0.75, background=0.125, fill=0.5)
    assert np.array_equal(f2, ARR["seq_12x10x14_7_custom"])


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_pack_unpack_update_match_reference(tag):
    meta = GOLD[f"block_{tag}"]
    field = ARR[f"pack_{tag}_field"].copy()
    for d in meta["nbr_dirs"]:
        want = ARR[f"pack_{tag}_face{d}"]
        assert jacobi_np.pack_face(field, d).tobytes() == want.tobytes()
        assert jacobi_c.pack(field, d).tobytes() == want.tobytes()
    f_np, f_c = field.copy(), field.copy()
    for d in meta["nbr_dirs"]:
        face = ARR[f"unpack_{tag}_rstage{d}"]
        jacobi_np.unpack_face(f_np, d, face)
        jacobi_c.unpack(f_c, d, face)
    assert f_np.tobytes() == ARR[f"unpack_{tag}_field"].tobytes()
    assert f_c.tobytes() == ARR[f"unpack_{tag}_field"].tobytes()
    # the update writes the other buffer's interior only: start from the
    # golden buffer with a poisoned interior, so ghosts must stay untouched
    want = ARR[f"update_{tag}_next"]
    nxt = want.copy()
    nxt[1:-1, 1:-1, 1:-1] = np.nan
    nxt_c = nxt.copy()
    jacobi_np.stencil(f_np, nxt)
    assert nxt.tobytes() == want.tobytes()
    jacobi_c.stencil(f_c, nxt_c, nthreads=2)
    assert nxt_c.tobytes() == want.tobytes()


def test_decompose_and_neighbors_match_reference():
    for key, want in GOLD["decompose"].items():
        dims_s, n = key.rsplit("/", 1)
        dims = tuple(int(x) for x in dims_s.strip("()").split(","))
        got = jacobi_np.decompose(dims, int(n))
        assert (list(got) if got is not None else None) == want, key
    for g_s, tables in GOLD["neighbors"].items():
        grid = tuple(int(x) for x in g_s.strip("()").split(","))
        for r, want in enumerate(tables):
            assert jacobi_np.neighbors(grid, r) == want


@pytest.mark.parametrize("pes", [1, 2, 4, 8])
def test_blocked_oracle_matches_reference_run_jacobi(pes):
    f = jacobi_np.blocked((16, 16, 16), 5, pes)
    for mode in ("channel-device", "messaging-device", "host-staging", "mpi-device"):
        assert sha(f) == GOLD["run_jacobi_sha256"][f"16x16x16/5/{pes}/{mode}"]


def test_pattern_matches_reference():
    for s, h in GOLD["pattern_sha256"].items():
        assert hashlib.sha256(jacobi_np.pattern(int(s))).hexdigest() == h
