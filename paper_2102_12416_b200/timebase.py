"""Per-worker clocks (mirror of cl/timebase.py:34-59, wall mode only).

The reference's VirtualClock exists to model a simulated device; on B200
every time is measured: host wall time (monotonic ns) for API-level
numbers, CUDA events / %globaltimer for device-level ones.
"""

from __future__ import annotations

import time


class WallClock:
    __slots__ = ()

    virtual = False

    @property
    def now(self) -> int:
        return time.monotonic_ns()

    def charge(self, ns: int) -> int:
        return time.monotonic_ns()

    def merge(self, ts: int) -> int:
        return time.monotonic_ns()


def make_clock(time_mode: str):
    if time_mode != "wall":
        raise ValueError(f"time mode {time_mode!r} is not available on the B200 path")
    return WallClock()
