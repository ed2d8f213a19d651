"""Process-per-GPU runtime backend ("ipc") on the GPU: the reference's
drivers (run_jacobi in every mode, the OSU benches over both runtime APIs
and MPI) with PE p in process p % 2 under torchrun, device payloads moved
between processes through CUDA IPC handles carried in the rendezvous frames
(cl/transport.py:77-91, 469-555's TCP backend, B200 form).

The 1-GPU variant puts both processes on cuda:0 (an IPC handle opens in
another process on the same device), so a single-GPU box runs the whole
cross-process path; with two GPUs the same worker runs one process per GPU
over NVLink."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tmp_path, same_gpu, port, quick):
    out = tmp_path / "verdict.json"
    env = dict(os.environ)
    if same_gpu:
        env["HX_SAME_GPU"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "mp_runtime_worker.py"), str(out)] + (["quick"] if quick else [])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-4000:]
    v = json.loads(out.read_text())
    assert v["ok"], v["failures"]
    assert v["world"] == 2
    return v


def test_ipc_runtime_two_processes_one_gpu(cuda, tmp_path):
    v = _run(tmp_path, True, 29711, quick=False)
    assert len(v["osu"]) == 3 * 2 * 4


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_ipc_runtime_one_process_per_gpu(cuda, tmp_path):
    v = _run(tmp_path, False, 29712, quick=True)
    assert len(v["osu"]) == 3 * 2 * 2
