"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference Jacobi3D path.

Every function cites the reference (``/root/reference/pkg/src/charmlet/``,
abbreviated ``cl/``) line it restates. The arithmetic is plain IEEE fp64
elementwise addition followed by a true division by 6.0, evaluated in the
reference's left-to-right order, so the result is bit-identical across numpy
versions. Pinned against tests/golden/ (generated from the reference itself).
"""

from __future__ import annotations

import numpy as np

NDIRS = 6  # 0=-x 1=+x 2=-y 3=+y 4=-z 5=+z; d ^ 1 flips (cl/jacobi3d.py:35)


# ---------------------------------------------------------------- geometry

def face_area(dims, grid) -> int:
    """Internal face area of a block grid (cl/jacobi3d.py:55-59)."""
    nx, ny, nz = dims
    px, py, pz = grid
    return (px - 1) * ny * nz + (py - 1) * nx * nz + (pz - 1) * nx * ny


def decompose(dims, nblocks: int):
    """Minimum-face-area factorisation, ties to smallest (px, py)
    (cl/jacobi3d.py:62-76). Returns None when nothing tiles."""
    best = None
    for px in range(1, nblocks + 1):
        if nblocks % px:
            continue
        for py in range(1, nblocks // px + 1):
            if (nblocks // px) % py:
                continue
            pz = nblocks // px // py
            if dims[0] % px or dims[1] % py or dims[2] % pz:
                continue
            key = (face_area(dims, (px, py, pz)), px, py)
            if best is None or key < best[0]:
                best = (key, (px, py, pz))
    return None if best is None else best[1]


def block_coords(rank: int, grid):
    """rank -> (ix, iy, iz), x fastest (cl/jacobi3d.py:79-81)."""
    return rank % grid[0], (rank // grid[0]) % grid[1], rank // (grid[0] * grid[1])


def neighbors(grid, rank: int):
    """Neighbour rank per direction or None (cl/jacobi3d.py:84-97)."""
    c = block_coords(rank, grid)
    out = []
    for d in range(NDIRS):
        a = d // 2
        cc = list(c)
        cc[a] += 1 if d & 1 else -1
        out.append(cc[0] + grid[0] * (cc[1] + grid[1] * cc[2])
                   if 0 <= cc[a] < grid[a] else None)
    return out


def face_index(d: int, interior: bool):
    """Plane selector of a padded block (cl/jacobi3d.py:102-112): first/last
    interior plane when packing, ghost plane when unpacking; the other two
    axes span the interior only."""
    idx = [slice(1, -1), slice(1, -1), slice(1, -1)]
    if d & 1:
        idx[d // 2] = -2 if interior else -1
    else:
        idx[d // 2] = 1 if interior else 0
    return tuple(idx)


# ---------------------------------------------------------------- kernels

def pack_face(field: np.ndarray, d: int) -> np.ndarray:
    """Contiguous C-order copy of face d (cl/jacobi3d.py:157-158)."""
    return np.ascontiguousarray(field[face_index(d, True)])


def unpack_face(field: np.ndarray, d: int, face: np.ndarray) -> None:
    """Write a received face into ghost plane d (cl/jacobi3d.py:160-163)."""
    field[face_index(d, False)] = face


def stencil(cur: np.ndarray, nxt: np.ndarray) -> None:
    """Six-neighbour average into nxt's interior, ghosts untouched
    (cl/jacobi3d.py:165-172): (((((x- + x+) + y-) + y+) + z-) + z+) / 6."""
    acc = cur[:-2, 1:-1, 1:-1] + cur[2:, 1:-1, 1:-1]
    acc += cur[1:-1, :-2, 1:-1]
    acc += cur[1:-1, 2:, 1:-1]
    acc += cur[1:-1, 1:-1, :-2]
    acc += cur[1:-1, 1:-1, 2:]
    nxt[1:-1, 1:-1, 1:-1] = acc / 6.0


def residual(cur: np.ndarray, nxt: np.ndarray) -> float:
    """max |nxt - cur| over the interior (cl/jacobi3d.py:197-198)."""
    return float(np.max(np.abs(nxt[1:-1, 1:-1, 1:-1] - cur[1:-1, 1:-1, 1:-1])))


def init_global(dims, hot=1.0, background=0.0, fill=0.0) -> np.ndarray:
    """Padded single-block field (cl/jacobi3d.py:186-188)."""
    g = np.full((dims[0] + 2, dims[1] + 2, dims[2] + 2), background, dtype=np.float64)
    g[1:-1, 1:-1, 1:-1] = fill
    g[0, :, :] = hot
    return g


def sequential(dims, iters: int, hot=1.0, background=0.0, fill=0.0):
    """Single-array run; returns (interior copy, residual history)
    (cl/jacobi3d.py:181-200)."""
    g = init_global(dims, hot, background, fill)
    n = g.copy()
    res = []
    for _ in range(iters):
        stencil(g, n)
        res.append(residual(g, n))
        g, n = n, g
    return g[1:-1, 1:-1, 1:-1].copy(), res


def init_block(dims, grid, rank) -> np.ndarray:
    """Padded block field: zeros, hot wall 1.0 on the whole x=0 ghost plane
    when the block touches the global x=0 face (cl/jacobi3d.py:131-138)."""
    bx, by, bz = dims[0] // grid[0], dims[1] // grid[1], dims[2] // grid[2]
    f = np.zeros((bx + 2, by + 2, bz + 2))
    if block_coords(rank, grid)[0] == 0:
        f[0, :, :] = 1.0
    return f


def blocked(dims, iters: int, pes: int):
    """All blocks in lockstep: pack, exchange, unpack, update
    (cl/jacobi3d.py:246-279). Returns the assembled interior."""
    grid = decompose(dims, pes)
    if grid is None:
        raise ValueError(f"{pes} blocks cannot tile {dims}")
    cur = [init_block(dims, grid, r) for r in range(pes)]
    nxt = [init_block(dims, grid, r) for r in range(pes)]
    nbrs = [neighbors(grid, r) for r in range(pes)]
    for _ in range(iters):
        faces = [{d: pack_face(cur[r], d) for d in range(NDIRS) if nbrs[r][d] is not None}
                 for r in range(pes)]
        for r in range(pes):
            for d in range(NDIRS):
                src = nbrs[r][d]
                if src is not None:
                    unpack_face(cur[r], d, faces[src][d ^ 1])
        for r in range(pes):
            stencil(cur[r], nxt[r])
        cur, nxt = nxt, cur
    return assemble([c[1:-1, 1:-1, 1:-1] for c in cur], dims, grid)


def assemble(fields, dims, grid) -> np.ndarray:
    """Place block interiors in the global array (cl/jacobi3d.py:324-332)."""
    out = np.empty(dims)
    bx, by, bz = dims[0] // grid[0], dims[1] // grid[1], dims[2] // grid[2]
    for r, f in enumerate(fields):
        ix, iy, iz = block_coords(r, grid)
        out[ix * bx:(ix + 1) * bx, iy * by:(iy + 1) * by, iz * bz:(iz + 1) * bz] = f
    return out


def pattern(size: int) -> bytes:
    """OSU payload (cl/bench.py:36-37): byte i = (11 i + size) & 0xFF."""
    return ((np.arange(size, dtype=np.int64) * 11 + size) & 0xFF).astype(np.uint8).tobytes()
