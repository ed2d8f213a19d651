# quick 2-GPU regression: the multi-GPU tests and the N=2 bench line
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ipc_runtime.py -q 2>&1 | tail -2
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2_end_n2.json 2> gpurun_out/r2_end_n2.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2_end_n2.json").read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ("value", "ms_per_step", "roofline", "halo", "p2p", "clocks", "gpu_launches")})[:2500])
PY
