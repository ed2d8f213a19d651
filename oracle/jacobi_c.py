"""TEST INFRASTRUCTURE ONLY — ctypes wrapper over oracle/build/liboracle_jacobi.so.

The threaded C restatement (oracle/jacobi_c.c) of the reference stencil
(cl/jacobi3d.py:165-172), residual (197-198), pack/unpack (157-163) and
sequential oracle (181-200). Used by tests as a second checker and by
bench.py as the timed CPU baseline on the host cores.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "build", "liboracle_jacobi.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile the C oracle with the committed Makefile."""
    src = os.path.join(_HERE, "jacobi_c.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_stencil.argtypes = [_dp, _dp, ctypes.c_long, ctypes.c_long, ctypes.c_long, ctypes.c_int]
        L.orc_stencil.restype = None
        L.orc_stencil_residual.argtypes = L.orc_stencil.argtypes
        L.orc_stencil_residual.restype = ctypes.c_double
        L.orc_pack.argtypes = [_dp, ctypes.c_long, ctypes.c_long, ctypes.c_long, ctypes.c_int, _dp]
        L.orc_unpack.argtypes = L.orc_pack.argtypes
        L.orc_sequential.argtypes = [ctypes.c_long, ctypes.c_long, ctypes.c_long, ctypes.c_int,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double, _dp, _dp,
                                     ctypes.c_int]
        L.orc_sequential.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def max_threads() -> int:
    return lib().orc_max_threads()


def stencil(cur: np.ndarray, nxt: np.ndarray, nthreads: int = 0) -> None:
    bx, by, bz = (s - 2 for s in cur.shape)
    lib().orc_stencil(_ptr(cur), _ptr(nxt), bx, by, bz, nthreads)


def stencil_residual(cur: np.ndarray, nxt: np.ndarray, nthreads: int = 0) -> float:
    bx, by, bz = (s - 2 for s in cur.shape)
    return lib().orc_stencil_residual(_ptr(cur), _ptr(nxt), bx, by, bz, nthreads)


def face_shape(shape, d: int):
    ext = [s - 2 for s in shape]
    return tuple(ext[a] for a in range(3) if a != d // 2)


def pack(field: np.ndarray, d: int) -> np.ndarray:
    out = np.empty(face_shape(field.shape, d))
    bx, by, bz = (s - 2 for s in field.shape)
    lib().orc_pack(_ptr(field), bx, by, bz, d, _ptr(out))
    return out


def unpack(field: np.ndarray, d: int, face: np.ndarray) -> None:
    face = np.ascontiguousarray(face, dtype=np.float64)
    bx, by, bz = (s - 2 for s in field.shape)
    lib().orc_unpack(_ptr(field), bx, by, bz, d, _ptr(face))


def sequential(dims, iters: int, hot=1.0, background=0.0, fill=0.0, nthreads: int = 0):
    out = np.empty(tuple(dims))
    res = np.empty(max(iters, 1))
    rc = lib().orc_sequential(dims[0], dims[1], dims[2], iters, hot, background, fill,
                              _ptr(out), _ptr(res), nthreads)
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    return out, [float(r) for r in res[:iters]]
