"""Time the fused exchange (hx_shell_put) on its own and inside a step.

Two blocks of an (2n, n, n) grid on GPUs 0 and 1 (or both on GPU 0 with
--one-gpu), exchange="fused". Reports, per block:
  * the shell kernel alone on an idle GPU (flags pre-satisfied): time, HBM
    bytes (3 planes read + 1 written per x-plane cell = 32 B) and the NVLink
    bytes it stores into the neighbour (8 B per face cell);
  * full fused steps: step time, interior sweep, the concurrent shell.

    python tools/prof_fused.py [--n 1536] [--reps 10] [--one-gpu] [--steps-only]
"""

import argparse
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2102_12416_b200 import _lib
    from paper_2102_12416_b200.halo import NDIRS, HaloJacobi

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1536)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--one-gpu", action="store_true")
    ap.add_argument("--steps-only", action="store_true")
    ap.add_argument("--exchange", default="fused", choices=("fused", "p2p"))
    ap.add_argument("--iso-only", action="store_true", help="skip the full steps (for ncu)")
    ap.add_argument("--remote", default="peer", choices=("peer", "none"),
                    help="none: the shell alone without its NVLink stores (diagnostics)")
    args = ap.parse_args()
    n = args.n
    two = torch.cuda.device_count() >= 2 and not args.one_gpu
    eng = HaloJacobi((2 * n, n, n), 2, device_of=(lambda r: r) if two else (lambda r: 0),
                     exchange=args.exchange, overlap=args.exchange == "p2p", timeout_s=20)
    for _ in range(3):
        eng.step()
    eng.synchronize()
    out = {"n": n, "gpus": 2 if two else 1}

    if not args.steps_only and args.exchange == "fused":
        iso = []
        for _ in range(args.reps):
            for b in eng.blocks.values():
                _lib.call("hx_set_device", b.device)
                c = eng.comm[b.device]
                _, shells = eng.boxes(b)
                flat = (ctypes.c_int * (6 * len(shells)))(*[v for box in shells for v in box])
                nxt = b.cur ^ 1
                remote = [b.peer_fields[d][nxt] if d in b.nbr_dirs and args.remote == "peer"
                          else None for d in range(NDIRS)]
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(c)
                for _ in range(8):  # back to back: the host's submit cost stays off the clock
                    _lib.call("hx_shell_put", b.field_ptr(), b.field_ptr(nxt), b.bx, b.by, b.bz,
                              len(shells), flat, _lib.ptr_array(remote), _lib.ptr_array([None] * 6),
                              0, _lib.ptr_array([None] * 6), 0, b.counters_ptr + 4, eng.timeout_ns,
                              b.err_ptr, None, None, c.cuda_stream)
                e1.record(c)
                c.synchronize()
                iso.append(e0.elapsed_time(e1) / 8)
        b = eng.blocks[0]
        cells = sum((x[1] - x[0]) * (x[3] - x[2]) * (x[5] - x[4]) for x in eng.boxes(b)[1])
        face = b.by * b.bz
        ms = statistics.median(iso)
        out["shell_alone"] = {"ms": ms, "remote": args.remote, "all_ms": [round(x, 4) for x in iso], "cells": cells, "hbm_bytes": 32 * cells,
                              "hbm_gbs": 32 * cells / (ms * 1e-3) / 1e9,
                              "nvlink_bytes": 8 * face,
                              "nvlink_gbs": 8 * face / (ms * 1e-3) / 1e9}

    if args.iso_only:
        print(json.dumps(out), flush=True)
        eng.close()
        return
    timing: dict = {}
    s0 = eng.stream_of(eng.blocks[0])
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.synchronize()
    a.record(s0)
    for _ in range(args.reps):
        eng.step(timing=timing)
    z.record(s0)
    eng.synchronize()
    eng.check_errors()

    def mean(name):
        p = timing.get(name, [])
        if not p:
            return None
        k = len(eng.blocks)  # pairs are appended block by block each step
        return [round(statistics.mean(x.elapsed_time(y) for x, y in p[r::k]), 4) for r in range(k)]

    out["step_ms"] = a.elapsed_time(z) / args.reps
    out["interior_ms"] = mean("interior")
    out["shell_concurrent_ms"] = mean("exchange")
    out["exposed_ms"] = mean("exposed")
    print(json.dumps(out), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
