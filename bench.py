"""Jacobi3D weak-scaling bench on B200 (BASELINE.json configs[2]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

Workload: 1536^3 fp64 cells per GPU, global grid 1536 x (1,1,1)/(2,1,1)/
(2,2,1)/(2,2,2) at N = 1/2/4/8 (x, y, z doubling),
decomposed by the reference's decompose (cl/jacobi3d.py:62-76). A step is
one full iteration over all ranks: fused pack+NVLink put+flag, wait+unpack,
TMA stencil (paper_2102_12416_b200/halo.py). Inputs (two 29 GB fields per
GPU) are far larger than L2, so no flush is needed between steps.

Printed JSON line (rank 0): value = whole-job GLUP/s (interior cells x
steps / max-over-ranks device time), roofline of the stencil kernel vs the
measured HBM copy peak, cpu_baseline (the C oracle on the host cores, a
bounded slab sample), e2e through the public API with host buffers
(per-step H2D of the Dirichlet hot-wall plane from pinned memory, per-step
D2H of the residual), clocks sampled during the timed region.

Also on the line: data_alt (the same timed steps on a seeded N(0,1)
interior: speed must not come from the hot wall's zeros) and, at N=1,
e2e_api (the reference's entry point run_jacobi(mode="channel-persistent")
end to end, field read-back included).

--impl reference: the reference's OWN code (charmlet, installed unmodified
into baseline/_ref): _BlockCore.update (numpy, cl/jacobi3d.py:165-173) in
one pinned process per host core, each on a 16-plane slab block of the
per-GPU cross-section; plus its run_jacobi 64^3 x 100 and OSU 8 B / 4 MiB
numbers in wall mode (reference_api). Falls back to the bit-identical C
restatement in oracle/ when baseline/_ref is absent.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Jacobi3D ms/iter & GLUP/s at 1/2/4/8 B200; p2p halo GB/s & 8B latency"
UNIT = "GLUP/s"
BLOCK = 1536
ALG_BYTES_PER_CELL = 16  # 8 B read + 8 B written per interior cell
NVLINK_GBS = 900.0


def global_dims(n: int, block: int):
    doubling = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}
    if n not in doubling:
        raise SystemExit(f"--gpus must be 1, 2, 4 or 8 (got {n})")
    return tuple(block * f for f in doubling[n])


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(alg_bytes):
    """(dram bytes per stencil launch, capture's traffic / algorithmic ratio)
    from the committed ncu --set full summary. The bytes are reported only
    when the capture is of a launch of this size (same algorithmic bytes);
    a capture of another block size is not this launch's traffic."""
    try:
        with open(os.path.join(ROOT, "profiles", "stencil_ncu_summary.json")) as f:
            d = json.load(f)
    except Exception:
        return None, None
    ratio = d.get("traffic_over_alg")
    for cap in [d] + d.get("other_captures", []):
        cap_alg = cap.get("alg_bytes_per_launch")
        if cap_alg and abs(cap_alg - alg_bytes) <= 0.001 * cap_alg:
            return cap.get("dram_bytes_per_launch"), ratio
    return None, ratio


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
         "utilization.gpu")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.5)  # let the sampler attach before the timed region
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        self._p.terminate()
        try:
            out = self._p.communicate(timeout=10)[0]
        except Exception:
            self._p.kill()
            out = ""
        for line in out.splitlines():
            cols = [c.strip() for c in line.split(",")]
            if len(cols) >= 9:
                self.rows.append(cols)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        busy = [r for r in self.rows if (num(r[8]) or 0) >= 50] or self.rows
        sm = [num(r[1]) for r in busy if num(r[1]) is not None]
        mx = [num(r[2]) for r in self.rows if num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in busy for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples_under_load": len(busy), "samples": len(self.rows)}


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_sample(block: int, seconds: float):
    """The C oracle (all host cores) on a bounded slab of the per-GPU block:
    64 x-planes of the full block cross-section, swept until ~seconds pass."""
    import numpy as np

    from oracle import jacobi_c

    planes = 64
    cur = np.zeros((planes + 2, block + 2, block + 2))
    cur[0] = 1.0
    nxt = cur.copy()
    nth = cpu_threads()
    jacobi_c.stencil(cur, nxt, nth)  # warm
    sweeps, t0 = 0, time.perf_counter()
    while True:
        jacobi_c.stencil(cur, nxt, nth)
        cur, nxt = nxt, cur
        sweeps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    cells = planes * block * block
    return {"value": cells * sweeps / el / 1e9, "unit": UNIT, "cores": nth, "kind": "port",
            "sample": f"C oracle (oracle/jacobi_c.c, {nth} pthreads) on a {planes}x{block}x{block} "
                      f"slab of the {block}^3 block, {sweeps} sweeps in {el:.1f} s"}


# ------------------------------------------------------------- reference arm

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "charmlet"))


def _ref_update_worker(core_id, planes, block, steps, conn):
    """One host core: the reference's own _BlockCore.update (numpy,
    cl/jacobi3d.py:165-173) on a (planes, block, block) slab block, one
    update per step when the parent says go."""
    try:
        os.sched_setaffinity(0, {core_id})
    except Exception:
        pass
    sys.path.insert(0, REF_DIR)
    from charmlet.devicesim import DeviceSpace
    from charmlet.jacobi3d import _BlockCore

    space = DeviceSpace(None, {}, 1 << 42)
    core = _BlockCore((planes, block, block), (1, 1, 1), 0, lambda n: space.alloc(0, n))
    core.update()  # first touch of every page + numpy temporaries
    conn.send("ready")
    for _ in range(steps):
        conn.recv()
        t0 = time.perf_counter()
        core.update()
        conn.send(time.perf_counter() - t0)
    conn.close()


def reference_update_sample(block: int, steps: int, warmup: int, planes: int = 16):
    """Aggregate GLUP/s of the reference's numpy stencil on every host core:
    one pinned process per core, each sweeping its own slab of the per-GPU
    block's cross-section; a step = one update in every process, started
    together, timed to the last one to finish."""
    import multiprocessing as mp

    ctx = mp.get_context("fork")
    cores = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else list(
        range(os.cpu_count() or 1))
    # each process holds two slab fields plus numpy's temporaries (~7 field
    # sizes); keep the sample within half of the available host memory
    per_proc = 8 * (planes + 2) * (block + 2) ** 2 * 8
    try:
        import psutil

        avail = psutil.virtual_memory().available
        cores = cores[:max(1, min(len(cores), int(avail * 0.5) // per_proc))]
    except Exception:
        cores = cores[:32]
    procs, pipes = [], []
    for c in cores:
        a, b = ctx.Pipe()
        p = ctx.Process(target=_ref_update_worker, args=(c, planes, block, warmup + steps, b))
        p.start()
        procs.append(p)
        pipes.append(a)
    for a in pipes:
        assert a.recv() == "ready"
    times = []
    for k in range(warmup + steps):
        t0 = time.perf_counter()
        for a in pipes:
            a.send("go")
        for a in pipes:
            a.recv()
        if k >= warmup:
            times.append(time.perf_counter() - t0)
    for p in procs:
        p.join()
    cells = len(cores) * planes * block * block
    t = statistics.median(times)
    return {"value": cells / t / 1e9, "unit": UNIT, "cores": len(cores), "kind": "reference",
            "step_s": t,
            "sample": f"reference charmlet _BlockCore.update (numpy, baseline/_ref) in {len(cores)} "
                      f"processes pinned one per core, each on its own {planes}x{block}x{block} "
                      f"slab block; step = one update in every process (median of {steps})"}


def reference_api_sample():
    """The reference's own drivers in wall mode on one core:
    run_jacobi 64^3 x 100 (channel-device, 1/2/4/8 PEs) and the OSU 8 B
    latency / 4 MiB window bandwidth of both APIs (cl/jacobi3d.py:335-379,
    cl/bench.py:364-452)."""
    sys.path.insert(0, REF_DIR)
    from charmlet import bench as rbench
    from charmlet.config import RuntimeConfig
    from charmlet.jacobi3d import run_jacobi as rjacobi

    out = {"run_jacobi_64x100_ms_per_iter": {}, "osu": {}}
    for pes in (1, 2, 4, 8):
        r = rjacobi((64, 64, 64), 100, "channel-device", pes, cfg=RuntimeConfig(time_mode="wall"))
        out["run_jacobi_64x100_ms_per_iter"][str(pes)] = r["total_ns"] / 100 / 1e6
    cfg = rbench.bench_config(time_mode="wall")
    for api in ("charm-channel", "charm-messaging"):
        lat = rbench.measure_latency(api, "device", 8, cfg=cfg)
        bw = rbench.measure_bandwidth(api, "device", 4 << 20, cfg=cfg)
        out["osu"][api] = {"latency_8B_us": lat["value_ns"] / 1e3,
                           "bandwidth_4MiB_gbs": bw["value_gbps"],
                           "verified": lat["verified"] and bw["verified"]}
    out["cores"] = 1
    return out


def run_reference(args, rank: int) -> int:
    if rank != 0:
        return 0
    n = args.gpus
    dims = global_dims(n, args.block)
    if reference_available():
        cpu = reference_update_sample(args.block, args.steps, args.warmup)
        v = cpu["value"]
        extra = {"reference_api": reference_api_sample()}
    else:  # the reference install is missing: its bit-identical C restatement
        per_step = max(1.0, args.ref_seconds / max(1, args.steps))
        for _ in range(args.warmup):
            cpu_sample(args.block, min(per_step, 2.0))
        vals = [cpu_sample(args.block, per_step) for _ in range(args.steps)]
        v = statistics.median(x["value"] for x in vals)
        cpu = dict(vals[0], value=v)
        extra = {}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": args.block ** 3 * n / (v * 1e9) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (Dirichlet hot wall, cl/jacobi3d.py:131-138)",
            "config": {"workload": f"Jacobi3D {args.block}^3 per GPU fp64 weak scaling",
                       "global_dims": list(dims), "block": [args.block] * 3},
            "cpu_baseline": {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "ms_per_step extrapolates the measured per-cell rate to the whole per-GPU "
                    "block (1536^3 does not fit the reference's numpy path in host RAM)"}
    line.update(extra)
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm

def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--block", type=int, default=BLOCK,
                    help="weak scaling: per-GPU block edge (configs[2]: 1536, configs[4]: 768)")
    ap.add_argument("--dims", default=None,
                    help="strong scaling: fixed global grid, e.g. 3072,3072,3072 (configs[3])")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-seconds", type=float, default=60.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-p2p", action="store_true", help="skip the GPU 0 <-> 1 OSU probe")
    ap.add_argument("--data", choices=("hotwall", "random"), default="hotwall",
                    help="hotwall: the reference's Dirichlet input (interior 0, x=0 plane 1.0); "
                         "random: seeded N(0,1) interior, same walls. The line also carries a "
                         "data_alt leg timed on the other input (--no-data-alt skips it)")
    ap.add_argument("--no-data-alt", action="store_true")
    ap.add_argument("--no-e2e-api", action="store_true",
                    help="skip the run_jacobi end-to-end leg (N=1 only)")
    ap.add_argument("--policy", choices=("b200", "reference"), default="b200",
                    help="block decomposition: reference = cl/jacobi3d.py:62-76 exactly; b200 = "
                         "same face area, ties broken away from splitting z (strided faces)")
    ap.add_argument("--exchange", choices=("p2p", "fused", "nccl"), default="fused",
                    help="p2p: persistent NVLink channels (pack+put / wait+unpack kernels); "
                         "fused: the boundary sweep stores into the neighbours' ghost planes "
                         "itself (hx_shell_put); nccl: grouped NCCL send/recv comparison "
                         "(implies --overlap 0)")
    ap.add_argument("--sweep-exchange", type=int, default=1,
                    help="fused: 1 (default) = every face produced and consumed by the interior "
                         "sweep (hx_stencil_exchange, no boundary kernel); 0 = x / y faces by "
                         "the boundary kernel, z faces by the sweep")
    ap.add_argument("--overlap", type=int, default=1,
                    help="1: interior sweep concurrent with the halo exchange (default)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}; launch N>1 with torchrun")
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")

    import torch
    import torch.distributed as dist

    from paper_2102_12416_b200 import _lib
    from paper_2102_12416_b200.halo import HaloJacobi

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.dims:
        dims = tuple(int(x) for x in args.dims.replace("x", ",").split(","))
        scaling, workload = "strong", f"Jacobi3D {dims[0]}x{dims[1]}x{dims[2]} fp64 strong scaling"
    else:
        dims = global_dims(world, args.block)
        scaling = "weak"
        workload = f"Jacobi3D {args.block}^3 per GPU fp64 weak scaling"
    eng = HaloJacobi(dims, world, local_ranks=[rank], device_of=lambda r: local,
                     dist=dist if world > 1 else None,
                     overlap=bool(args.overlap) and args.exchange == "p2p",
                     policy=args.policy, exchange=args.exchange if world > 1 else "p2p")
    eng.xy_from_interior = bool(args.sweep_exchange)
    b = eng.blocks[rank]
    s = eng.stream_of(b)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-timed steps (inputs resident in HBM)
    data_desc = {"hotwall": "synthetic (Dirichlet hot wall, cl/jacobi3d.py:131-138)",
                 "random": "synthetic (seeded N(0,1) interior, Dirichlet hot-wall ghost planes)"}
    if args.data == "random":
        barrier()
        eng.fill_random(seed=1)
        barrier()
    live, t_local, clk = timed_steps(eng, b, args.steps, args.warmup, barrier, local)
    timing: dict = {}
    for _ in range(min(args.steps, 10)):
        eng.step(timing=timing)
    barrier()
    eng.check_errors()
    for name in ("interior", "sweep"):  # the roofline kernel: live timings from the timed steps
        if name in live:
            timing[name] = live[name]

    def mean_ms(name):
        pairs = timing.get(name, [])
        return statistics.mean(a.elapsed_time(z) for a, z in pairs) if pairs else 0.0

    t_ms = max_over_ranks(t_local)
    sweep_cells = b.cells  # cells the timed TMA launch relaxes
    if (eng.overlap or eng.exchange == "fused") and b.nbr_dirs:
        inner = (eng.fused_boxes(b) if eng.exchange == "fused" else eng.boxes(b))[0]
        sweep_cells = (inner[1] - inner[0]) * (inner[3] - inner[2]) * (inner[5] - inner[4])
        if eng.exchange == "fused" and eng.sweep_exchange(b):
            sweep_cells = b.cells  # the sweep relaxes the whole block
        sten_ms = mean_ms("interior")  # the TMA interior launch alone
        exposed_ms = max_over_ranks(mean_ms("exposed"))
        if eng.exchange == "fused" and eng.sweep_exchange(b):
            launches_per_step = 1  # the sweep with every face; its last edge tile releases
        elif eng.exchange == "fused":
            # interior sweep + boundary kernel; with z neighbours the sweep
            # carries the z faces and hx_zsignal follows
            launches_per_step = 2 + (1 if eng.z_interior(b) else 0)
        else:
            launches_per_step = 1 + len(eng.boxes(b)[1]) + 1 + 2 * len(b.nbr_dirs)
    else:
        sten_ms = mean_ms("sweep")
        exposed_ms = max_over_ranks(mean_ms("exchange"))
        per_face = 2 * len(b.nbr_dirs)  # nccl: pack + unpack per face (+ NCCL's own kernels)
        launches_per_step = 1 + (per_face if eng.exchange == "nccl" else (2 if b.nbr_dirs else 0))
    xch_ms = max_over_ranks(mean_ms("exchange"))
    launches = args.steps * launches_per_step * world
    cells = b.cells
    total_cells = cells * world
    value = total_cells * args.steps / (t_ms * 1e-3) / 1e9
    peak, peak_kind = hbm_peak()
    achieved = ALG_BYTES_PER_CELL * sweep_cells / (sten_ms * 1e-3) / 1e9
    traffic, traffic_ratio = ncu_traffic(ALG_BYTES_PER_CELL * sweep_cells)
    face_bytes = sum(b.face_elems[d] * 8 for d in b.nbr_dirs)
    # with z faces produced by the interior sweep (HaloJacobi.z_interior), the
    # boundary kernel (the timed exchange) carries only the x / y faces
    zint = world > 1 and eng.exchange == "fused" and eng.z_interior(b)
    swx = world > 1 and eng.exchange == "fused" and eng.sweep_exchange(b)
    # (with every face inside the sweep the boundary kernel still times the
    # x / y exchange alone: its isolated rate is the NVLink figure below)
    shell_bytes = sum(b.face_elems[d] * 8 for d in b.nbr_dirs if not (zint and d >= 4))

    # ---- the exchange alone (not sharing HBM with an interior sweep): a few
    # untimed-for-value steps with the overlap split off, for the NVLink fraction
    iso_ms = None
    if world > 1 and eng.exchange == "fused":
        barrier()
        one = eng.time_shell_alone()
        barrier()
        iso_ms = max_over_ranks(one) if one is not None else None
    if world > 1 and eng.exchange == "p2p":
        saved, eng.overlap = eng.overlap, False
        iso: dict = {}
        for _ in range(5):
            eng.step(timing=iso)
        barrier()
        eng.overlap = saved
        pairs = iso.get("exchange", [])
        iso_ms = max_over_ranks(statistics.median(a.elapsed_time(z) for a, z in pairs)) if pairs else None

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(eng, b, args, world, barrier, max_over_ranks, total_cells)

    # ---- the same steps on the other input (speed must not depend on zeros)
    alt = None
    if not args.no_data_alt:
        other = "random" if args.data == "hotwall" else "hotwall"
        barrier()
        if other == "random":
            eng.fill_random(seed=1)
        else:
            eng.reset()
        barrier()
        live_a, t_a, clk_a = timed_steps(eng, b, args.steps, args.warmup, barrier, local)
        eng.check_errors()
        t_a = max_over_ranks(t_a)
        name = "interior" if "interior" in live_a else "sweep"
        k_ms = statistics.mean(x.elapsed_time(y) for x, y in live_a[name])
        ach = ALG_BYTES_PER_CELL * sweep_cells / (k_ms * 1e-3) / 1e9
        v_a = total_cells * args.steps / (t_a * 1e-3) / 1e9
        alt = {"data": data_desc[other], "value": v_a, "unit": UNIT,
               "ms_per_step": t_a / args.steps, "rel_to_line": v_a / value,
               "roofline": {"achieved": ach, "peak": peak, "frac": ach / peak, "kernel_ms": k_ms},
               "clocks": clk_a}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample(args.block, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": data_desc[args.data],
            "config": {"workload": workload,
                       "global_dims": list(dims), "grid": list(eng.grid), "policy": args.policy,
                       "exchange": ("fused, every face inside the interior sweep" if swx
                                    else eng.exchange) if world > 1 else "none (single block)",
                       "block": [b.bx, b.by, b.bz], "parallelism": f"3d-blocks x{world}",
                       "l2": f"inputs > L2 (2 x {(b.bx + 2) * (b.by + 2) * (b.bz + 2) * 8 / 1e9:.1f} GB "
                             "fields per GPU vs 126 MB L2), no flush needed"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_over_alg_1536_capture": traffic_ratio,
                         "kernel": "stencil_tma_kernel", "peak_kind": peak_kind,
                         "kernel_ms": sten_ms,
                         "alg_bytes_per_launch": ALG_BYTES_PER_CELL * sweep_cells},
            "halo": ({"bytes_out_per_rank": face_bytes,
                      "boundary_kernel_bytes": shell_bytes,
                      "z_faces_in_interior_sweep": bool(zint or swx),
                      "all_faces_in_interior_sweep": bool(swx),
                      "exchange_ms": xch_ms,
                      # (with every face inside the sweep, exchange_ms is only the flag
                      # release left outside it: no rate is derived from it)
                      "exchange_gbs": shell_bytes / (xch_ms * 1e-3) / 1e9
                      if xch_ms and not swx else None,
                      "nvlink_frac": shell_bytes / (xch_ms * 1e-3) / 1e9 / NVLINK_GBS
                      if xch_ms and not swx else None,
                      "overlap": eng.overlap, "exposed_ms": exposed_ms,
                      "interior_ms": mean_ms("interior"), "shell_ms": mean_ms("shell"),
                      "non_overlapped_frac": exposed_ms / (t_ms / args.steps),
                      "isolated_exchange_ms": iso_ms,
                      "isolated_exchange_kernel": "hx_shell_put_z alone (the boundary kernel: "
                                                  "x / y faces, relax + local and NVLink stores)",
                      "isolated_exchange_gbs": (shell_bytes / (iso_ms * 1e-3) / 1e9)
                      if iso_ms and shell_bytes else None,
                      "isolated_nvlink_frac": (shell_bytes / (iso_ms * 1e-3) / 1e9 / NVLINK_GBS)
                      if iso_ms and shell_bytes else None} if world > 1 else None),
            "gpu_launches": launches,
            "clocks": clk,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "data_alt": alt,
        }
    eng.close()
    del eng, b
    torch.cuda.empty_cache()
    if world == 1 and not args.no_e2e_api and not args.dims:
        line["e2e_api"] = run_e2e_api(dims, args.steps)
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        # after the other ranks are done with the GPUs: the metric's "p2p
        # halo GB/s & 8B latency" between GPUs 0 and 1 (untimed by the step)
        line["p2p"] = None if args.no_p2p else p2p_probe()
        print(json.dumps(line), flush=True)
    return 0


def timed_steps(eng, b, steps, warmup, barrier, local):
    """W untimed steps, then K steps bracketed by barrier + synchronize and
    one CUDA event pair on the block's main stream, nvidia-smi sampling the
    clocks throughout. The dominant kernel (the interior / full sweep) is
    timed live inside the timed steps by one event pair per step on its own
    stream; returns (live kernel events, step time in ms, clock summary)."""
    import torch

    s = eng.stream_of(b)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        for _ in range(warmup):
            eng.step()
        barrier()
        split = (eng.overlap or eng.exchange == "fused") and bool(b.nbr_dirs)
        live = {"_only": {"interior" if split else "sweep"}}
        start.record(s)
        for _ in range(steps):
            eng.step(timing=live)
        stop.record(s)
        barrier()
    live.pop("_only")
    return live, start.elapsed_time(stop), clk.summary()


def run_e2e_api(dims, iters):
    """The reference's own entry point, end to end: run_jacobi(dims, iters,
    mode="channel-persistent") (cl/jacobi3d.py:335-379) — block allocation
    and Dirichlet init in HBM, the iterations (two eager, the rest replayed
    from CUDA graphs), and the whole field read back into the returned numpy
    array. Wall clock around the call."""
    from paper_2102_12416_b200.jacobi3d import run_jacobi

    t0 = time.perf_counter()
    r = run_jacobi(dims, iters, mode="channel-persistent", pes=1)
    wall = time.perf_counter() - t0
    cells = dims[0] * dims[1] * dims[2]
    field_bytes = r["field"].nbytes
    del r["field"]
    return {"value": cells * iters / wall / 1e9, "unit": UNIT, "wall_s": wall,
            "iterations_ms_per_iter": r["total_ns"] / iters / 1e6,
            "iterations_value": cells * iters / (r["total_ns"] * 1e-9) / 1e9,
            "d2h_bytes": field_bytes, "h2d_bytes": 0, "iters": iters,
            "api": "paper_2102_12416_b200.jacobi3d.run_jacobi(mode='channel-persistent')",
            "note": "includes block allocation, init and the one-time read-back of the whole "
                    "field (the reference's return value); iterations_* is the loop alone"}


def p2p_probe() -> dict | None:
    """OSU-style point to point between GPUs 0 and 1 (configs[1]): 8-byte
    one-way latency and 4 MiB window bandwidth, device level (one kernel
    per side: LL ping-pong; pull window) and through the pre-registered
    persistent channel (graph-replayed send/recv; 64 KiB slots, so the
    4 MiB messages are pulled by the receive). None on a 1-GPU box."""
    import torch

    if torch.cuda.device_count() < 2:
        return None
    if os.environ.get("CUDA_INJECTION64_PATH"):
        # under ncu / a tool: kernels are serialised, and the two sides of a
        # ping-pong must run concurrently on different GPUs
        return {"skipped": "profiler attached (kernels serialised)"}
    from paper_2102_12416_b200 import osu

    try:
        osu.device_latency(8, iters=500, warmup=50)  # warm-up (clocks, first replays)
        osu.channel_latency(8, iters=200, warmup=20)
        lat = osu.device_latency(8, iters=2000, warmup=200)
        bw = osu.device_bandwidth(4 << 20, window=64, iters=5, engine="sm-pull-window")
        clat = osu.channel_latency(8, iters=1000, warmup=50)
        cbw = osu.channel_bandwidth(4 << 20, window=64, iters=5)
    except Exception as e:  # the Jacobi line stands on its own
        return {"error": f"{type(e).__name__}: {e}"}
    return {"gpus": [0, 1], "nvlink_peak_gbs": NVLINK_GBS,
            "latency_8B_us": {"device_ll": lat["value_ns"] / 1e3,
                              "persistent_channel": clat["value_ns"] / 1e3},
            "bandwidth_4MiB_gbs": {"device_pull_window": bw["value_gbps"],
                                   "persistent_channel": cbw["value_gbps"]},
            "frac_of_nvlink_4MiB": {"device_pull_window": bw["value_gbps"] / NVLINK_GBS,
                                    "persistent_channel": cbw["value_gbps"] / NVLINK_GBS},
            "verified": all(r["verified"] for r in (lat, bw, clat, cbw)),
            "tool": "paper_2102_12416_b200.osu (tools/run_osu.py has the full 8 B-4 MiB sweep)"}


def run_e2e(eng, b, args, world, barrier, max_over_ranks, total_cells):
    """Public-API steps with host buffers: each step uploads the Dirichlet
    hot-wall plane (ranks on the global x=0 face) from pinned memory and
    reads the step's residual back to pinned host memory."""
    import torch

    hot = b.coords[0] == 0
    plane = (b.by + 2) * (b.bz + 2)
    host_wall = torch.ones(plane, dtype=torch.float64, pin_memory=True)
    res_host = torch.zeros(args.steps + args.warmup, dtype=torch.int64, pin_memory=True)
    for k in range(args.warmup):
        eng.step_e2e(host_wall if hot else None, res_host[k:k + 1])
    barrier()
    t0 = time.perf_counter()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    s = eng.stream_of(b)
    start.record(s)
    for k in range(args.warmup, args.warmup + args.steps):
        eng.step_e2e(host_wall if hot else None, res_host[k:k + 1])
    eng.drain_e2e()
    stop.record(s)
    barrier()
    wall_ms = (time.perf_counter() - t0) * 1e3
    dev_ms = start.elapsed_time(stop)
    t_ms = max_over_ranks(max(dev_ms, wall_ms))
    eng.check_errors()
    h2d = torch.tensor([plane * 8 if hot else 0], dtype=torch.int64)
    h2d_total = int(h2d.item()) * (world // eng.grid[0])  # ranks on the x=0 face
    res = res_host.numpy().view("float64")
    return {"value": total_cells * args.steps / (t_ms * 1e-3) / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": h2d_total, "d2h_bytes_per_step": 8 * world,
            "ms_per_step": t_ms / args.steps, "last_residual": float(res[-1]),
            "device_ms_per_step": dev_ms / args.steps, "wall_ms_per_step": wall_ms / args.steps,
            "api": "paper_2102_12416_b200.halo.HaloJacobi.step_e2e"}


if __name__ == "__main__":
    sys.exit(main())
