"""torchrun worker for the process-per-GPU runtime backend ("ipc").

    torchrun --nproc-per-node 2 tests/mp_runtime_worker.py OUT.json [quick]
    HX_SAME_GPU=1 torchrun ...   (both processes on cuda:0: the 1-GPU variant)

Every process builds the same runtime with RuntimeConfig(backend="ipc");
PE p runs in process p % 2. Checked, bit for bit / byte for byte:
* run_jacobi in all five reference modes and channel-persistent at 2 and 4
  PEs against the reference's sequential_oracle sha (32^3 x 20, and the
  acceptance config 64^3 x 100 at 2 PEs): halos cross the process boundary
  as Channel sends, GPU Messaging DeviceArgs, MPI device messages, host-
  staged blobs, or the fused engine's IPC-mapped stores;
* the OSU benches (both runtime APIs and MPI, device and host modes) at
  eager and rendezvous sizes: verified payloads, positive times.
Rank 0 writes {"ok": bool, "failures": [...], "osu": [...]} to OUT.json.
"""

import faulthandler
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2102_12416_b200 import osu
    from paper_2102_12416_b200.config import RuntimeConfig
    from paper_2102_12416_b200.jacobi3d import ALL_MODES, run_jacobi

    import signal

    from paper_2102_12416_b200.transport import TransportGroup

    def dump(signum, frame):  # a stalled case prints every open group's queues
        for g in list(TransportGroup._live):
            print(f"[{dist.get_rank()}] STALL {g.debug_state()}", flush=True)

    signal.signal(signal.SIGALRM, dump)
    out = sys.argv[1]
    quick = len(sys.argv) > 2 and sys.argv[2] == "quick"
    same = os.environ.get("HX_SAME_GPU") == "1"
    local = 0 if same else int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
    cfg = RuntimeConfig(backend="ipc")
    failures = []

    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()

    cases = [((32, 32, 32), 20, pes, gold["seq_sha256"]["32x32x32/20"]) for pes in (2, 4)]
    if not quick:
        cases.append(((64, 64, 64), 100, 2, gold["seq_64_100"]["sha256"]))
    for dims, iters, pes, want in cases:
        for mode in ALL_MODES:
            # a hung case dumps every thread's stack and exits (never a silent hang)
            faulthandler.dump_traceback_later(120, exit=True)
            signal.alarm(100)
            print(f"[{rank}] run_jacobi {dims} x {iters} {mode} pes={pes}", flush=True)
            try:
                r = run_jacobi(dims, iters, mode, pes, cfg=cfg)
                if sha(r["field"]) != want:
                    failures.append(f"run_jacobi {dims} x {iters} {mode} pes={pes}: field differs")
                if r["total_ns"] <= 0 or r["comm_ns"] <= 0:
                    failures.append(f"run_jacobi {mode} pes={pes}: times {r['total_ns']}, "
                                    f"{r['comm_ns']}")
            except Exception as e:  # noqa: BLE001 - report every failing case
                failures.append(f"run_jacobi {dims} {mode} pes={pes}: {type(e).__name__}: {e}")

    osu_rows = []
    sizes = (8, 8193) if quick else (8, 8192, 8193, 1 << 20)
    bcfg = osu.bench_config(base=cfg)
    for api in osu.APIS:
        for mode in osu.MODES:
            for size in sizes:
                faulthandler.dump_traceback_later(120, exit=True)
                signal.alarm(100)
                print(f"[{rank}] osu {api}/{mode}/{size}", flush=True)
                try:
                    lat = osu.measure_latency(api, mode, size, iters=10, warmup=2, cfg=bcfg)
                    bw = osu.measure_bandwidth(api, mode, size, window=8, iters=2, cfg=bcfg)
                    osu_rows.append({"api": api, "mode": mode, "size": size,
                                     "latency_us": lat["value_ns"] / 1e3,
                                     "bandwidth_gbs": bw["value_gbps"]})
                    if not (lat["verified"] and bw["verified"]):
                        failures.append(f"osu {api}/{mode}/{size}: payload not verified")
                    if not (lat["value_ns"] > 0 and bw["value_gbps"] > 0):
                        failures.append(f"osu {api}/{mode}/{size}: non-positive result")
                except Exception as e:  # noqa: BLE001
                    failures.append(f"osu {api}/{mode}/{size}: {type(e).__name__}: {e}")

    faulthandler.cancel_dump_traceback_later()
    signal.alarm(0)
    everyone = [None] * dist.get_world_size()
    dist.all_gather_object(everyone, failures)
    if rank == 0:
        allf = [f"process {p}: {f}" for p, fs in enumerate(everyone) for f in fs]
        with open(out, "w") as f:
            json.dump({"ok": not allf, "failures": allf, "osu": osu_rows,
                       "world": dist.get_world_size(), "same_gpu": same}, f, indent=1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
