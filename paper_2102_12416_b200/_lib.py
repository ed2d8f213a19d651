"""ctypes binding of libhx.so (include/hx.h), the package's only compute path.

There is no CPU fallback: if the shared library is missing the import
fails loudly, and every compute call requires a CUDA device. The binding
mirrors include/hx.h one to one; callers pass raw device pointers (ints)
and raw cudaStream_t handles.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
# HX_LIB_PATH: load another build of the same ABI (A/B experiments in tools/)
LIB_PATH = os.environ.get("HX_LIB_PATH") or os.path.join(_HERE, "libhx.so")
CSRC = os.path.join(_HERE, "csrc")

HX_E_INVALID = -1
HX_E_TIMEOUT = -2
HX_E_NODRIVER = -3
HX_E_TMA = -4

# Every symbol include/hx.h declares (checked by the CPU test suite).
EXPORTS = (
    "hx_abi_version", "hx_error_string", "hx_device_count", "hx_set_device", "hx_get_device",
    "hx_sm_count", "hx_device_synchronize", "hx_stream_create", "hx_stream_destroy",
    "hx_stream_synchronize", "hx_event_create", "hx_event_destroy", "hx_event_record",
    "hx_event_query", "hx_event_synchronize", "hx_event_elapsed_ms", "hx_stream_wait_event",
    "hx_malloc", "hx_free", "hx_malloc_host", "hx_free_host", "hx_can_access_peer",
    "hx_enable_peer", "hx_ipc_get", "hx_ipc_open", "hx_ipc_close", "hx_alloc_range", "hx_memcpy",
    "hx_memcpy_peer", "hx_copy_sm", "hx_move", "hx_copy_sm_window", "hx_fill_f64", "hx_stencil", "hx_stencil_box",
    "hx_stencil_set_variant", "hx_stencil_last_variant", "hx_stencil_set_chunk", "hx_div6_check",
    "hx_init_block", "hx_pack", "hx_unpack", "hx_pack_put", "hx_wait_unpack", "hx_shell_put",
    "hx_shell_put_z", "hx_persist_run", "hx_stencil_box_z", "hx_zsignal",
    "hx_stencil_exchange", "hx_exchange_signal", "hx_exchange_edge_items",
    "hx_chan_send", "hx_chan_recv", "hx_chan_trace", "hx_preload",
    "hx_signal",
    "hx_wait_flag", "hx_read_u64", "hx_pingpong", "hx_pingpong_ll",
)


class HxError(RuntimeError):
    """A libhx call returned a non-zero status."""

    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed ({code}): {msg}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile libhx.so for sm_100a with the committed Makefile."""
    if force:
        subprocess.run(["make", "-s", "-C", CSRC, "clean"], check=True)
    subprocess.run(["make", "-s", "-C", CSRC], check=True)
    return LIB_PATH


_V = ctypes.c_void_p
_I = ctypes.c_int
_U64 = ctypes.c_ulonglong
_SZ = ctypes.c_size_t
_D = ctypes.c_double

_SIGS = {
    "hx_abi_version": ([], _I),
    "hx_error_string": ([_I], ctypes.c_char_p),
    "hx_device_count": ([ctypes.POINTER(_I)], _I),
    "hx_set_device": ([_I], _I),
    "hx_get_device": ([ctypes.POINTER(_I)], _I),
    "hx_sm_count": ([_I, ctypes.POINTER(_I)], _I),
    "hx_device_synchronize": ([], _I),
    "hx_stream_create": ([ctypes.POINTER(_V)], _I),
    "hx_stream_destroy": ([_V], _I),
    "hx_stream_synchronize": ([_V], _I),
    "hx_event_create": ([ctypes.POINTER(_V), _I], _I),
    "hx_event_destroy": ([_V], _I),
    "hx_event_record": ([_V, _V], _I),
    "hx_event_query": ([_V], _I),
    "hx_event_synchronize": ([_V], _I),
    "hx_event_elapsed_ms": ([_V, _V, ctypes.POINTER(ctypes.c_float)], _I),
    "hx_stream_wait_event": ([_V, _V], _I),
    "hx_malloc": ([ctypes.POINTER(_V), _SZ], _I),
    "hx_free": ([_V], _I),
    "hx_malloc_host": ([ctypes.POINTER(_V), _SZ], _I),
    "hx_free_host": ([_V], _I),
    "hx_can_access_peer": ([_I, _I, ctypes.POINTER(_I)], _I),
    "hx_enable_peer": ([_I, _I], _I),
    "hx_ipc_get": ([_V, _V, ctypes.POINTER(_SZ)], _I),
    "hx_ipc_open": ([_V, ctypes.POINTER(_V)], _I),
    "hx_ipc_close": ([_V], _I),
    "hx_alloc_range": ([_V, ctypes.POINTER(_V), ctypes.POINTER(_SZ)], _I),
    "hx_memcpy": ([_V, _V, _SZ, _V], _I),
    "hx_memcpy_peer": ([_V, _I, _V, _I, _SZ, _V], _I),
    "hx_copy_sm": ([_V, _V, _SZ, _V], _I),
    "hx_move": ([_V, _V, _SZ, _I, _V, _V, _V, _V], _I),
    "hx_copy_sm_window": ([_V, _V, _SZ, _I, _V], _I),
    "hx_fill_f64": ([_V, _SZ, _D, _V], _I),
    "hx_stencil": ([_V, _V, _I, _I, _I, _V, _V], _I),
    "hx_stencil_box": ([_V, _V, _I, _I, _I, _I, _I, _I, _I, _I, _I, _V, _V], _I),
    "hx_stencil_set_variant": ([_I], _I),
    "hx_stencil_last_variant": ([], _I),
    "hx_stencil_set_chunk": ([_I], _I),
    "hx_div6_check": ([_V, _SZ, _V, _V], _I),
    "hx_init_block": ([_V, _I, _I, _I, _I, _D, _D, _D, _V], _I),
    "hx_pack": ([_V, _I, _I, _I, _I, _V, _V], _I),
    "hx_unpack": ([_V, _I, _I, _I, _I, _V, _V], _I),
    "hx_pack_put": ([_V, _I, _I, _I, _I, ctypes.POINTER(_V), ctypes.POINTER(_V), _U64, _V, _V], _I),
    "hx_wait_unpack": ([_V, _I, _I, _I, _I, ctypes.POINTER(_V), ctypes.POINTER(_V), _U64, _U64,
                        _V, _V], _I),
    "hx_shell_put": ([_V, _V, _I, _I, _I, _I, _V, ctypes.POINTER(_V), ctypes.POINTER(_V), _U64,
                      ctypes.POINTER(_V), _U64, _V, _U64, _V, _V, _V, _V], _I),
    "hx_persist_run": ([ctypes.POINTER(_V), ctypes.POINTER(_V), _I, _I, _I, _I, _U64, _I,
                        ctypes.POINTER(_V), ctypes.POINTER(_V), ctypes.POINTER(_V),
                        ctypes.POINTER(_V), _V, _I, _U64, _V, _V], _I),
    "hx_stencil_box_z": ([_V, _V, _I, _I, _I, _I, _I, _I, _I, _I, _I, _V, ctypes.POINTER(_V), _V,
                          ctypes.POINTER(_V), ctypes.POINTER(_V), _U64, _V, _V], _I),
    "hx_zsignal": ([ctypes.POINTER(_V), _V, _V, _V], _I),
    "hx_stencil_exchange": ([_V, _V, _I, _I, _I, _V, ctypes.POINTER(_V), ctypes.POINTER(_V), _V,
                             ctypes.POINTER(_V), ctypes.POINTER(_V), ctypes.POINTER(_V), _V,
                             _U64, _V, _V], _I),
    "hx_exchange_signal": ([ctypes.POINTER(_V), _V, _V, _V], _I),
    "hx_exchange_edge_items": ([_I, _I, _I, _I, ctypes.POINTER(ctypes.c_uint)], _I),
    "hx_shell_put_z": ([_V, _V, _I, _I, _I, _I, _V, ctypes.POINTER(_V), ctypes.POINTER(_V), _U64,
                        ctypes.POINTER(_V), _U64, _V, _U64, _V, _V, _V, ctypes.POINTER(_V),
                        ctypes.POINTER(_V), _V], _I),
    "hx_chan_send": ([_V, _SZ, _V, _SZ, _I, _V, _V, _V, _U64, _V, _V], _I),
    "hx_chan_recv": ([_V, _SZ, _V, _SZ, _I, _V, _V, _V, _V, _U64, _V, _V], _I),
    "hx_chan_trace": ([_I, _V, _V], _I),
    "hx_preload": ([], _I),
    "hx_signal": ([_V, _U64, _V], _I),
    "hx_wait_flag": ([_V, _U64, _U64, _V, _V], _I),
    "hx_read_u64": ([_V, ctypes.POINTER(_U64)], _I),
    "hx_pingpong": ([_I, _V, _V, _SZ, _V, _V, _I, _I, _U64, _V, _V, _V], _I),
    "hx_pingpong_ll": ([_I, _V, _V, _V, _V, _SZ, _I, _I, _U64, _V, _V, _V], _I),
}

_lib = None


def load():
    """Load libhx.so (raises if it is missing — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (make -C paper_2102_12416_b200/csrc). There is no CPU fallback.")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def error_string(code: int) -> str:
    return load().hx_error_string(code).decode()


def call(name: str, *args) -> int:
    """Invoke hx_<name>; raise HxError on a non-zero status."""
    rc = getattr(load(), name)(*args)
    if rc != 0:
        raise HxError(name, rc, error_string(rc))
    return rc


def raw(name: str):
    return getattr(load(), name)


def ptr_array(ptrs) -> ctypes.Array:
    """A void*[6] from a sequence of 6 ints/None."""
    arr = (_V * 6)()
    for i, p in enumerate(ptrs):
        arr[i] = p or None
    return arr


def device_count() -> int:
    n = _I(0)
    rc = load().hx_device_count(ctypes.byref(n))
    return n.value if rc == 0 else 0
