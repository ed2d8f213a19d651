"""Parity at the bench's own sizes, the reference's acceptance configuration,
and the cross-process (CUDA IPC) halo path on one GPU.

* Bench configs (BASELINE configs[2] / configs[4] at N = 1: 1536^3 and 768^3
  single blocks, the exact HaloJacobi path bench.py times) on a seeded
  N(0,1) field — not the ~98 %-zero hot wall — for two sweeps with the
  fused residual. Each sweep is checked bit for bit against the C oracle
  (oracle/jacobi_c.c, pinned to the reference's goldens in test_oracle.py)
  slab by slab: planes [i0-1, i1+1) of the sweep's input go to the host,
  the oracle relaxes them, and planes [i0, i1) of the GPU output must be
  identical. Host memory stays bounded (two pinned 66-plane slabs); the
  bitwise comparison of uint64 patterns runs on the GPU.
* Multi-block at scale on one GPU (the fused NVLink-store exchange, every
  block's peer on the same device): the 768^3-per-GPU weak configs at
  N = 2 (x split) and N = 4 (2,2,1), and a z split — checked against the
  oracle applied to the global field assembled slab by slab from the
  blocks (internal ghosts come from the neighbours' interiors, so a stale
  or misplaced halo fails).
* run_jacobi((64,)*3, 100) in every mode at 1/2/4/8 PEs against the
  reference's sequential_oracle sha (pkg/tests/test_acceptance.py:330-358).
* Two processes on cuda:0 under torchrun: HaloJacobi's CUDA IPC handles,
  cross-process flags and peer stores, bit-exact against the numpy oracle.
"""

import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
SLAB = 64


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def oracle_c(cuda):
    from oracle import jacobi_c

    jacobi_c.build()
    return jacobi_c


class _SlabChecker:
    """Pinned host slabs reused across the sweep. The input slab is read
    back from the GPU, the C oracle relaxes it on the host cores, and the
    oracle's output goes back up so the bitwise comparison (on the uint64
    bit patterns) runs on the GPU — host memory traffic stays small."""

    def __init__(self, eng):
        nx, ny, nz = eng.dims
        self.eng = eng
        self.dev = next(iter(eng.blocks.values())).device
        self.cur = torch.empty((SLAB + 2, ny + 2, nz + 2), dtype=torch.float64, pin_memory=True)
        self.want = torch.empty_like(self.cur, pin_memory=True)

    def gather(self, which, g0, g1):
        """Global padded planes [g0, g1) of every block's buffer ``which``
        ("cur" or "nxt" relative to each block's state) into the pinned
        input slab. Each global cell comes from exactly one block: interiors
        from their owner, a domain-face ghost from the block on that face.
        Internal ghosts are never copied — they are the neighbours' interior
        cells — so a stale or misplaced halo on the GPU makes its output
        differ from the oracle's."""
        out = self.cur[:g1 - g0]
        for b in self.eng.blocks.values():
            f = b.fields[b.cur if which == "cur" else b.cur ^ 1]
            ext = (b.bx, b.by, b.bz)
            lo = [0 if b.coords[a] == 0 else 1 for a in range(3)]
            hi = [ext[a] + 2 if b.coords[a] == self.eng.grid[a] - 1 else ext[a] + 1 for a in range(3)]
            org = [b.coords[a] * ext[a] for a in range(3)]
            a, z = max(g0, org[0] + lo[0]), min(g1, org[0] + hi[0])
            if a < z:
                out[a - g0:z - g0, org[1] + lo[1]:org[1] + hi[1], org[2] + lo[2]:org[2] + hi[2]].copy_(
                    f[a - org[0]:z - org[0], lo[1]:hi[1], lo[2]:hi[2]])
        torch.cuda.synchronize(self.dev)
        return out

    def check(self, oracle_c, before):
        """After one eng.step(residual=True): every block's output interior
        equals the oracle applied to the assembled global input (``before``
        names the buffer parity each block read: its 'nxt' after the flip).
        Returns the oracle's max|nxt - cur| over the whole domain."""
        eng = self.eng
        nx = eng.dims[0]
        res = 0.0
        for i0 in range(1, nx + 1, SLAB):
            i1 = min(i0 + SLAB, nx + 1)
            cur = self.gather(before, i0 - 1, i1 + 1).numpy()
            want = self.want[:i1 - i0 + 2].numpy()
            res = max(res, oracle_c.stencil_residual(cur, want))
            want_d = self.want[:i1 - i0 + 2].to(f"cuda:{self.dev}", non_blocking=False)
            for b in eng.blocks.values():
                org = [b.coords[a] * (b.bx, b.by, b.bz)[a] for a in range(3)]
                a, z = max(i0, org[0] + 1), min(i1, org[0] + b.bx + 1)
                if a >= z:
                    continue
                got = b.fields[b.cur][a - org[0]:z - org[0], 1:-1, 1:-1]
                ref = want_d[a - i0 + 1:z - i0 + 1, org[1] + 1:org[1] + b.by + 1,
                             org[2] + 1:org[2] + b.bz + 1]
                assert torch.equal(got.view(torch.int64), ref.to(got.device).view(torch.int64)), \
                    f"block {b.rank}: x planes [{a}, {z}) differ from the C oracle"
            del want_d
        return res


def _randomise(eng, seed):
    g = torch.Generator(device=f"cuda:{next(iter(eng.blocks.values())).device}")
    g.manual_seed(seed)
    for b in eng.blocks.values():
        for f in b.fields:
            f.normal_(generator=g)
    torch.cuda.synchronize()


@pytest.mark.parametrize("n", [1536, 768])
def test_bench_config_random_field_bitexact_vs_c_oracle(oracle_c, n):
    """bench.py's N=1 path (HaloJacobi, one block, TMA sweep + fused residual)
    at the full 1536^3 / 768^3 block on a random field, 2 sweeps."""
    from paper_2102_12416_b200.halo import HaloJacobi

    eng = HaloJacobi((n,) * 3, 1, device_of=lambda r: 0)
    _randomise(eng, 7 + n)
    chk = _SlabChecker(eng)
    for sweep in range(2):
        eng.step(residual=True)
        want_res = chk.check(oracle_c, "nxt")
        got_res = eng.residuals(0)[sweep]
        assert got_res == want_res, (sweep, got_res, want_res)
    eng.check_errors()
    eng.close()
    del eng
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dims,pes,grid", [
    ((1536, 768, 768), 2, (2, 1, 1)),     # configs[4] at N = 2
    ((1536, 1536, 768), 4, (2, 2, 1)),    # configs[4] at N = 4
    ((768, 768, 1536), 2, (1, 1, 2)),     # a z split: z faces through the arena slots
    ((1536, 1536, 1536), 8, (2, 2, 2)),   # the paper's (2,2,2) layout: every face, edge, corner
])
def test_fused_exchange_at_scale_random_field_vs_c_oracle(oracle_c, dims, pes, grid):
    """The default multi-GPU exchange (hx_shell_put: boundary relax + peer
    ghost-plane stores + flags, concurrent with the TMA interior) with all
    blocks on cuda:0, 768^3-class blocks, random field, 2 steps."""
    from paper_2102_12416_b200.halo import HaloJacobi

    eng = HaloJacobi(dims, pes, device_of=lambda r: 0, exchange="fused", timeout_s=30)
    assert eng.grid == grid
    _randomise(eng, 11 * pes)
    chk = _SlabChecker(eng)
    for step in range(2):
        eng.step(residual=True)
        want_res = chk.check(oracle_c, "nxt")
        got_res = max(eng.residuals(r)[step] for r in eng.blocks)
        assert got_res == want_res, (step, got_res, want_res)
    eng.check_errors()
    eng.close()
    del eng
    torch.cuda.empty_cache()


@pytest.mark.parametrize("pes", [1, 2, 4, 8])
def test_reference_acceptance_64cubed_100_iters_all_modes(cuda, pes):
    """pkg/tests/test_acceptance.py:330-358: 64^3 x 100 iterations, every
    mode (plus the persistent-channel mode) at 1/2/4/8 PEs, bitwise equal to
    the reference's sequential_oracle (sha frozen from the reference)."""
    from paper_2102_12416_b200.jacobi3d import ALL_MODES, run_jacobi

    want = GOLD["seq_64_100"]["sha256"]
    for mode in ALL_MODES:
        r = run_jacobi(dims=(64, 64, 64), iters=100, mode=mode, pes=pes)
        assert sha(r["field"]) == want, (mode, pes)
        assert (r["comm_ns"] == 0.0) == (pes == 1), (mode, pes)


@pytest.mark.parametrize("pes", [1, 2])
def test_run_jacobi_large_field_prefaulted_readback_vs_c_oracle(oracle_c, pes):
    """run_jacobi on a field above the prefault threshold (512^3 = 1.07 GB):
    the result array is touched on host threads while the GPU iterates, then
    read back chunk by chunk through the pinned staging ring; it must equal
    the C oracle's sequential sweep bit for bit."""
    from paper_2102_12416_b200 import jacobi3d

    dims, iters = (512, 512, 512), 4
    assert 8 * 512 ** 3 >= jacobi3d._PREFAULT_MIN_BYTES
    r = jacobi3d.run_jacobi(dims=dims, iters=iters, mode="channel-persistent", pes=pes)
    want, _ = oracle_c.sequential(dims, iters)
    assert r["field"].shape == dims
    assert np.array_equal(r["field"].view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("mode,dims", [("0", (40, 24, 32)), ("fused", (40, 24, 32)),
                                       ("graph", (40, 24, 32)), ("fused", (24, 32, 80)),
                                       ("graph", (24, 32, 80))])
def test_ipc_engine_two_processes_one_gpu(cuda, tmp_path, mode, dims):
    """torchrun, 2 ranks, both on cuda:0: arenas and fields exported with
    cudaIpcGetMemHandle, opened by the other process, flags and peer stores
    across processes; bit-exact vs the numpy oracle (+ residual history).
    (24, 32, 80) splits z: the z faces go through IPC-mapped slots, produced
    and consumed by each process's interior sweep."""
    out = tmp_path / "verdict.json"
    env = dict(os.environ, HX_SAME_GPU="1")
    port = 29633 + ["0", "fused", "graph"].index(mode) + (10 if dims[2] == 80 else 0)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "mp_halo_worker.py"), *map(str, dims), "8", str(out), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    v = json.loads(out.read_text())
    assert v["bitwise"] and v["residuals"], v
    assert v["world"] == 2
    if dims[2] == 80:
        assert v["grid"] == [1, 1, 2] and v["z_interior"], v


def test_step_e2e_residual_ring_wraps(cuda):
    """step_e2e's device residual ring, shrunk to 4 slots and run for 11
    steps: every step's host residual equals the plain engine's, including
    the steps right before and after each wrap."""
    from paper_2102_12416_b200.halo import HaloJacobi

    dims, iters = (24, 20, 16), 11
    ref = HaloJacobi(dims, 2, device_of=lambda r: 0)
    ref.run(iters, residual=True)
    want = [max(ref.residuals(r)[i] for r in ref.blocks) for i in range(iters)]
    ref.close()

    eng = HaloJacobi(dims, 2, device_of=lambda r: 0)
    eng.e2e_ring_slots = 4
    host_wall = torch.ones((dims[1] + 2) * (dims[2] + 2), dtype=torch.float64, pin_memory=True)
    res = torch.zeros((iters, 2), dtype=torch.int64, pin_memory=True)
    for i in range(iters):
        eng.step_e2e(host_wall, res[i])
    eng.drain_e2e()
    got = [float(v) for v in res.numpy().view(np.float64).max(axis=1)]
    assert got == want
    eng.close()
