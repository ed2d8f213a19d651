"""Property-based checks of the host logic and the CPU oracle (hypothesis).

The golden tables pin the reference's answers at fixed inputs
(test_oracle.py, test_cpu_host.py). These tests sweep random inputs against
independent brute-force restatements of the same rules:
* decomposition: minimal internal face area, ties to the smallest (px, py),
  cl/jacobi3d.py:45-76 (the reference's tests use the same idea,
  pkg/tests/test_jacobi.py:19-35);
* the B200 policy: minimal weighted cost;
* neighbour tables: d and d ^ 1 are mutual;
* the tag codec: channel and messaging round trips;
* face pack / unpack: packing face d of one block and unpacking it on the
  neighbour's side d ^ 1 moves exactly the boundary plane;
* the numpy and threaded-C oracles agree bit for bit on random fields.
"""

import itertools

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import jacobi_c, jacobi_np
from paper_2102_12416_b200.jacobi3d import (FACE_COST, JacobiError, decompose, decompose_b200,
                                            neighbor_table, weighted_face_cost)

DIM = st.integers(min_value=1, max_value=96)
PES = st.integers(min_value=1, max_value=24)


def _factorisations(dims, n):
    for px in range(1, n + 1):
        if n % px:
            continue
        for py in range(1, n // px + 1):
            if (n // px) % py:
                continue
            pz = n // (px * py)
            if all(d % p == 0 for d, p in zip(dims, (px, py, pz))):
                yield px, py, pz


def _area(dims, g):
    nx, ny, nz = dims
    px, py, pz = g
    return (px - 1) * ny * nz + (py - 1) * nx * nz + (pz - 1) * nx * ny


@settings(max_examples=300, deadline=None)
@given(st.tuples(DIM, DIM, DIM), PES)
def test_reference_decomposition_is_the_brute_force_minimum(dims, n):
    cands = list(_factorisations(dims, n))
    if not cands:
        try:
            decompose(dims, n)
        except JacobiError:
            return
        raise AssertionError("decompose accepted an impossible tiling")
    best = min(cands, key=lambda g: (_area(dims, g), g[0], g[1]))
    assert decompose(dims, n) == best


@settings(max_examples=300, deadline=None)
@given(st.tuples(DIM, DIM, DIM), PES)
def test_b200_policy_minimises_weighted_cost(dims, n):
    cands = list(_factorisations(dims, n))
    if not cands:
        return
    g = decompose_b200(dims, n)
    assert g in cands
    assert weighted_face_cost(dims, g) == min(weighted_face_cost(dims, c) for c in cands)
    assert FACE_COST[2] >= FACE_COST[0]


@settings(max_examples=200, deadline=None)
@given(st.tuples(st.integers(1, 5), st.integers(1, 5), st.integers(1, 5)))
def test_neighbour_tables_are_mutual(grid):
    n = grid[0] * grid[1] * grid[2]
    tables = [neighbor_table(grid, r) for r in range(n)]
    for r, nb in enumerate(tables):
        for d in range(6):
            if nb[d] is not None:
                assert tables[nb[d]][d ^ 1] == r
        for a in range(3):  # domain edges have no neighbour, interior ones both
            coord = (r % grid[0], (r // grid[0]) % grid[1], r // (grid[0] * grid[1]))[a]
            assert (nb[2 * a] is None) == (coord == 0)
            assert (nb[2 * a + 1] is None) == (coord == grid[a] - 1)


@settings(max_examples=300, deadline=None)
@given(st.integers(0, (1 << 28) - 1), st.integers(0, 1), st.integers(0, (1 << 31) - 1),
       st.integers(0, 2), st.integers(0, (1 << 28) - 1), st.integers(0, (1 << 28) - 1))
def test_tag_codec_round_trips(cid, direction, ctr, kind_i, pe, mctr):
    from paper_2102_12416_b200.tags import DEVICE, EAGER, PROBE, TagError, TagLayout

    lay = TagLayout()
    try:
        tag = lay.encode_channel(cid, direction, ctr)
    except TagError:
        pass
    else:
        d = lay.decode(tag)
        assert (d.channel_id, d.direction, d.counter) == (cid, direction, ctr)
        assert 0 <= tag < (1 << 64)
    kind = (EAGER, PROBE, DEVICE)[kind_i]
    try:
        tag = lay.encode_messaging(kind, pe, mctr)
    except TagError:
        return
    d = lay.decode(tag)
    assert (d.kind, d.source_pe, d.counter) == (kind, pe, mctr)


@settings(max_examples=60, deadline=None)
@given(st.tuples(st.integers(1, 9), st.integers(1, 9), st.integers(1, 9)), st.integers(0, 5),
       st.integers(0, 2 ** 32 - 1))
def test_pack_then_unpack_moves_the_boundary_plane(shape, d, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(tuple(s + 2 for s in shape))
    b = rng.standard_normal(a.shape)
    before = b.copy()
    face = jacobi_np.pack_face(a, d)
    jacobi_np.unpack_face(b, d ^ 1, face)
    axis = d // 2
    src = [slice(1, -1)] * 3
    dst = [slice(1, -1)] * 3
    src[axis] = 1 if d % 2 == 0 else shape[axis]
    dst[axis] = shape[axis] + 1 if d % 2 == 0 else 0
    assert np.array_equal(b[tuple(dst)], a[tuple(src)])
    mask = np.ones(b.shape, dtype=bool)
    mask[tuple(dst)] = False
    assert np.array_equal(b[mask], before[mask])  # nothing else moved


@settings(max_examples=40, deadline=None)
@given(st.tuples(st.integers(1, 12), st.integers(1, 12), st.integers(1, 12)),
       st.integers(0, 2 ** 32 - 1))
def test_numpy_and_c_oracles_agree(shape, seed):
    rng = np.random.default_rng(seed)
    cur = rng.standard_normal(tuple(s + 2 for s in shape)) * 10.0 ** rng.integers(-300, 300)
    a, b = cur.copy(), cur.copy()
    jacobi_np.stencil(cur, a)
    jacobi_c.stencil(cur, b, nthreads=2)
    assert a.tobytes() == b.tobytes()
    assert jacobi_np.residual(cur, a) == jacobi_c.stencil_residual(cur, b.copy(), nthreads=1)


def test_factorisations_helper_is_complete():
    # the brute-force reference above must see every (px, py, pz) triple
    dims, n = (12, 12, 12), 12
    got = set(_factorisations(dims, n))
    want = {g for g in itertools.product(range(1, 13), repeat=3)
            if g[0] * g[1] * g[2] == n and all(d % p == 0 for d, p in zip(dims, g))}
    assert got == want
